import sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2305_06482_b200 import synth, linops as lo
from paper_2305_06482_b200.forward_model import SenseOperator
from paper_2305_06482_b200.plan import cartesian_plan
from paper_2305_06482_b200.cartesian import CartesianKernel
dims = (256, 256)
pts = synth.mask_points(synth.vd_poisson_mask(dims, 4.0, 24, 0))
traj = lo.Trajectory(pts, "cartesian-mask")
m0 = torch.randn(16, 65536, dtype=torch.complex64, device="cuda")
shape = lo.GridShape(dims)
for _ in range(3): SenseOperator(m0, traj, None, shape=shape)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(10): SenseOperator(m0, traj, None, shape=shape)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
