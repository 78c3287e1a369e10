"""A/B: host SVD coil compression vs device QR compression on config-3 inputs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from oracle import sketch_oracle as O
from paper_2305_06482_b200 import forward_model as fm, linops as lo, synth
from paper_2305_06482_b200 import _device as dv

rng = np.random.default_rng(0)
dims, C = (320, 320), 16
pts = synth.golden_angle_radial(128, 640, dims)
traj = lo.Trajectory(pts, "non-cartesian")
weights = fm.radial_density_weights(traj)
okern = O.GriddedKernel(dims, pts, 2.0, 4)
truth = synth.random_ellipses(dims, 10, rng).ravel()
maps = synth.gaussian_coil_maps(dims, C, rng)
clean = O.Sense(maps, okern).forward(truth).reshape(C, -1)
data = clean + synth.complex_noise(clean.shape, 0.01 * np.abs(clean).max(), rng)
D, M = fm.KSpaceData(traj, data), fm.SensitivityMaps(lo.GridShape(dims), maps)
d0, m0, comp, en = fm.coil_compress_svd(D, M, C)
m0d, d0d, compd, end = fm.coil_compress_device(D, M, C)
s = np.linalg.svd(data, compute_uv=False)
print("sv", s[:3], s[-4:], "gaps", np.diff(s)[-4:] / s[0])
print("comp diff per row", np.abs(comp - compd).max(axis=1))
print("maps0 rel", np.linalg.norm(dv.to_numpy128(m0d) - m0.coils) / np.linalg.norm(m0.coils))
print("data0 rel", np.linalg.norm(dv.to_numpy128(d0d) - d0.coils) / np.linalg.norm(d0.coils))
