#!/usr/bin/env python3
"""Config-3 NUFFT normal-op probe (320^2 golden-angle radial 128 x 640, KB 2x / w4, 8 coils):
per-apply device time for gridding bin sizes (CUDA events), and agreement between them."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_06482_b200 import synth  # noqa: E402
from paper_2305_06482_b200.nufft import GriddedKernel  # noqa: E402

dims = (320, 320)
pts = synth.golden_angle_radial(128, 640, dims)
rng = np.random.default_rng(0)
maps = torch.from_numpy(synth.gaussian_coil_maps(dims, 8, rng).astype(np.complex64)).cuda().unsqueeze(0)
x = torch.from_numpy(synth.random_ellipses(dims, 10, rng).ravel().astype(np.complex64)).cuda().view(1, -1)
r = np.linalg.norm(pts, axis=1)
w = torch.from_numpy(np.sqrt(r / r.max()).astype(np.float32)).cuda()
ref = None
for bs in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "16,4").split(",")]:
    kern = GriddedKernel(dims, pts, 2.0, 4, binsize=bs)
    out = torch.empty_like(x)
    for _ in range(3):
        kern.normal(maps, x, out, w=w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        kern.normal(maps, x, out, w=w)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    print(json.dumps({"binsize": bs, "nchunks": kern.nchunks, "normal_us": e0.elapsed_time(e1) / 50 * 1e3,
                      "rel_vs_first": float(torch.linalg.vector_norm(out - ref) / torch.linalg.vector_norm(ref))}),
          flush=True)
