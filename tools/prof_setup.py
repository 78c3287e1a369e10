"""cProfile of the host-side setup of one config-0 coil_sketching_recon call (everything before
the engine's run), sorted by cumulative time."""
import cProfile, pstats, sys
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
for _ in range(3):
    cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg)
torch.cuda.synchronize()
R.SketchedReconEngine.run = lambda self, *a, **k: (_ for _ in ()).throw(StopIteration())
pr = cProfile.Profile()
pr.enable()
try:
    cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg)
except StopIteration:
    pass
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
