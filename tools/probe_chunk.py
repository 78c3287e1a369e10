"""Gridding chunk size (samples per CTA, <= 256) vs the config-3 / config-4 NUFFT normal-op time."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2305_06482_b200 import synth
from paper_2305_06482_b200.nufft import GriddedKernel

def run(dims, pts, os_, C, sizes):
    rng = np.random.default_rng(0)
    maps = torch.randn(1, C, int(np.prod(dims)), dtype=torch.complex64, device="cuda") * 0.2
    x = torch.from_numpy(synth.random_ellipses(dims, 10, rng).ravel().astype(np.complex64)).cuda().view(1, -1)
    r = np.linalg.norm(pts, axis=1)
    w = torch.from_numpy(np.sqrt(r / r.max()).astype(np.float32)).cuda()
    ref = None
    for ch in sizes:
        GriddedKernel.BIN_CHUNK = ch
        kern = GriddedKernel(dims, pts, os_, 4)
        out = torch.empty_like(x)
        for _ in range(3):
            kern.normal(maps, x, out, w=w)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            kern.normal(maps, x, out, w=w)
        e1.record()
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        print(json.dumps({"dims": dims, "chunk": ch, "nchunks": kern.nchunks, "normal_ms": e0.elapsed_time(e1) / n,
                          "rel": float(torch.linalg.vector_norm(out - ref) / torch.linalg.vector_norm(ref))}), flush=True)

run((320, 320), synth.golden_angle_radial(128, 640, (320, 320)), 2.0, 8, [256, 128, 64, 32])
d3 = (256, 256, 160)
run(d3, synth.cones_3d(d3, n_readouts=18000, n_samples=512), 1.25, 16, [256, 128, 64])
