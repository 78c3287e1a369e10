import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from oracle import sketch_oracle as O
from paper_2305_06482_b200 import coil_sketch as cs, forward_model as fm, linops as lo, sketching as sk, solvers as so, synth
from paper_2305_06482_b200.forward_model import coil_compress_device, SenseOperator
dims, C = (256, 256), 16
rng = np.random.default_rng(0)
pts = synth.mask_points(synth.vd_poisson_mask(dims, 4.0, 24, 0))
traj = lo.Trajectory(pts, "cartesian-mask")
truth = synth.random_ellipses(dims, 10, rng).ravel()
maps = synth.gaussian_coil_maps(dims, C, rng)
clean = O.Sense(maps, O.CartesianKernel(dims, pts)).forward(truth).reshape(C, -1)
data = clean + synth.complex_noise(clean.shape, 0.01 * np.abs(clean).max(), rng)
shape = lo.GridShape(dims)
kd, sm = fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps)
def T(f):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, (time.perf_counter() - t) * 1e3
for _ in range(4):
    (m0, d0, _, e), t1 = T(lambda: coil_compress_device(kd, sm, 16))
    a, t2 = T(lambda: SenseOperator(m0, traj, None, shape=shape))
    _, t3 = T(lambda: fm.KSpaceData(traj, data))
    _, t4 = T(lambda: torch.from_numpy(data).cuda())
    _, t5 = T(lambda: torch.from_numpy(maps).cuda())
    print("compress %.2f  sense_op %.2f  kspacedata %.2f  up_data %.2f  up_maps %.2f ms" % (t1, t2, t3, t4, t5))
