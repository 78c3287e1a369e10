"""Wall time of repeated config-0 coil_sketching_recon calls (host clock around a synchronised
call), graph replay on / off: checks call-to-call stability of the captured path."""
import sys, time, gc
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2305_06482_b200.recon as R
from oracle import sketch_oracle as O
from paper_2305_06482_b200 import coil_sketch as cs, forward_model as fm, linops as lo, sketching as sk, solvers as so, synth
dims, C = (256, 256), 16
rng = np.random.default_rng(0)
pts = synth.mask_points(synth.vd_poisson_mask(dims, 4.0, 24, 0))
traj = lo.Trajectory(pts, "cartesian-mask")
truth = synth.random_ellipses(dims, 10, rng).ravel()
maps = synth.gaussian_coil_maps(dims, C, rng)
clean = O.Sense(maps, O.CartesianKernel(dims, pts)).forward(truth).reshape(C, -1)
data = clean + synth.complex_noise(clean.shape, 0.01 * np.abs(clean).max(), rng)
shape = lo.GridShape(dims)
reg = so.make_regularizer("l1-wavelet", 1e-3, shape)
cfg = cs.CoilSketchConfig(C, sk.SketchConfig(8, 4, 4, rademacher_scale=12 ** -0.5), reg, 10, 10)
for mode in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,0,1").split(",")]:
    R.OUTER_GRAPH = bool(mode)
    ts = []
    for _ in range(8):
        torch.cuda.synchronize(); t = time.perf_counter()
        cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg)
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
    cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg)
    torch.cuda.synchronize()
    print("call %.1f ms, run %.1f, captures %s, gc before %.1f" % ((time.perf_counter() - t) * 1e3, marks["run"],
          ["%.1f" % c for c in caps], gc_ms), flush=True)
