#!/usr/bin/env python3
"""Host-side (Python) profile of one config-0 coil_sketching_recon call: where the CPU time
between kernel launches goes (cProfile, cumulative), after a warm-up call."""
import cProfile
import pstats
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import sketch_oracle as O  # noqa: E402  (input generation only)
from paper_2305_06482_b200 import coil_sketch as cs, forward_model as fm, linops as lo, sketching as sk  # noqa: E402
from paper_2305_06482_b200 import solvers as so, synth  # noqa: E402

dims, C = (256, 256), 16
rng = np.random.default_rng(0)
pts = synth.mask_points(synth.vd_poisson_mask(dims, 4.0, 24, 0))
traj = lo.Trajectory(pts, "cartesian-mask")
shape = lo.GridShape(dims)
truth = synth.random_ellipses(dims, 10, rng).ravel()
maps = synth.gaussian_coil_maps(dims, C, rng)
clean = O.Sense(maps, O.CartesianKernel(dims, pts)).forward(truth).reshape(C, -1)
data = clean + synth.complex_noise(clean.shape, 0.01 * np.abs(clean).max(), rng)
cfg = cs.CoilSketchConfig(C, sk.SketchConfig(8, 4, 4, rademacher_scale=12 ** -0.5),
                          so.make_regularizer("l1-wavelet", 1e-3, shape), 10, 10)
args = (fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg)
cs.coil_sketching_recon(*args)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
cs.coil_sketching_recon(*args)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
