"""Wall time of repeated config-0 coil_sketching_recon calls (host clock around a synchronised
call), graph replay on / off: checks call-to-call stability of the captured path."""
import sys, time, gc
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2305_06482_b200.recon as R
from oracle import sketch_oracle as O
from paper_2305_06482_b200 import coil_sketch as cs, forward_model as fm, linops as lo, sketching as sk, solvers as so, synth
CFG = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(0)
kw = {}
if CFG == 0:
    dims, C, T, K, lam = (256, 256), 16, 10, 10, 1e-3
    pts = synth.mask_points(synth.vd_poisson_mask(dims, 4.0, 24, 0))
    traj = lo.Trajectory(pts, "cartesian-mask")
    okern = O.CartesianKernel(dims, pts)
else:
    from paper_2305_06482_b200.nufft import GriddedKernel
    dims, C, T, K, lam = (320, 320), 16, 15, 8, 5e-4
    pts = synth.golden_angle_radial(128, 640, dims)
    traj = lo.Trajectory(pts, "non-cartesian")
    okern = O.GriddedKernel(dims, pts, 2.0, 4)
    kw = dict(weights=fm.radial_density_weights(traj), kernel=GriddedKernel(dims, pts, 2.0, 4))
truth = synth.random_ellipses(dims, 10, rng).ravel()
maps = synth.gaussian_coil_maps(dims, C, rng)
clean = O.Sense(maps, okern).forward(truth).reshape(C, -1)
data = clean + synth.complex_noise(clean.shape, 0.01 * np.abs(clean).max(), rng)
shape = lo.GridShape(dims)
reg = so.make_regularizer("l1-wavelet", lam, shape)
cfg = cs.CoilSketchConfig(C, sk.SketchConfig(8, 4, 4, rademacher_scale=12 ** -0.5), reg, T, K)
for mode in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,0,1").split(",")]:
    R.OUTER_GRAPH = bool(mode)
    ts = []
    for _ in range(8):
        torch.cuda.synchronize(); t = time.perf_counter()
        cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg, **kw)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
    print("graph" if mode else "eager", " ".join("%.1f" % v for v in ts), flush=True)
# instrumented: host time of every capture and of run() per call (graph mode)
R.OUTER_GRAPH = True
ocap = R._capture
caps = []
def cap(fn, dev):
    t = time.perf_counter(); r = ocap(fn, dev); caps.append((time.perf_counter() - t) * 1e3); return r
R._capture = cap
orun = R.SketchedReconEngine.run
marks = {}
def run(self, *a, **k):
    t = time.perf_counter(); res = orun(self, *a, **k); marks["run"] = (time.perf_counter() - t) * 1e3; return res
R.SketchedReconEngine.run = run
for _ in range(8):
    caps.clear()
    gc_t = time.perf_counter(); gc.collect(); gc_ms = (time.perf_counter() - gc_t) * 1e3
    torch.cuda.synchronize(); t = time.perf_counter()
    cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg, **kw)
    torch.cuda.synchronize()
    print("call %.1f ms, run %.1f, captures %s, gc before %.1f" % ((time.perf_counter() - t) * 1e3, marks["run"],
          ["%.1f" % c for c in caps], gc_ms), flush=True)
# allocations inside the captures (0 = the graphs own no pool memory)
alloc = []
def cap2(fn, dev):
    torch.cuda.synchronize(); m0 = torch.cuda.memory_allocated()
    r = ocap(fn, dev)
    torch.cuda.synchronize(); alloc.append(torch.cuda.memory_allocated() - m0); return r
R._capture = cap2
cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg, **kw)
print("bytes allocated by the captures:", alloc, flush=True)
