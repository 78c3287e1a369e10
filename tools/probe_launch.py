"""Host-overhead probe: eager FISTA inner loop vs CUDA-graph replay at config-0 size."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2305_06482_b200 import synth
from paper_2305_06482_b200.cartesian import CartesianKernel
from paper_2305_06482_b200.plan import cartesian_plan
from paper_2305_06482_b200.recon import SketchedReconEngine
from paper_2305_06482_b200.sketching import SketchConfig
dims = (256, 256); C = 16
rng = np.random.default_rng(0)
pts = synth.mask_points(synth.vd_poisson_mask(dims, 4.0, 24, 0))
kern = CartesianKernel(dims, [cartesian_plan(dims, pts)])
maps = torch.from_numpy(synth.gaussian_coil_maps(dims, C, rng).astype(np.complex64)).cuda().unsqueeze(0)
y = kern.forward(maps, torch.from_numpy(synth.random_ellipses(dims, 10, rng).ravel().astype(np.complex64)).cuda().view(1, -1))
eng = SketchedReconEngine(kern, maps, y, dims=dims, sketch=SketchConfig(8, 4, 4, rademacher_scale=12 ** -0.5), lam=1e-3)
res = eng.run(2, 10)  # warm + capture
smaps = eng._smaps_buf
for name, fn in [("eager", lambda: eng._fista(smaps, 10)), ("graph", lambda: eng._graph.replay())]:
    for _ in range(3): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20): fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
    print(name, "ms per 10 FISTA iterations:", dt * 1e3)
t = time.perf_counter(); g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    eng._fista(smaps, 10)
torch.cuda.synchronize(); print("capture ms", (time.perf_counter() - t) * 1e3)
t = time.perf_counter(); eng.power_lambda(smaps); torch.cuda.synchronize(); print("power iteration ms", (time.perf_counter() - t) * 1e3)
t = time.perf_counter(); eng.objective(eng.x); eng.true_gradient(eng.d); torch.cuda.synchronize(); print("objective+gradient ms", (time.perf_counter() - t) * 1e3)
