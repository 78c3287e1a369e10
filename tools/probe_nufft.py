#!/usr/bin/env python3
"""Config-4 NUFFT normal-op probe: plan build time and per-apply device time of the sketched
normal op (16 coils) on the full cones trajectory; used for ncu captures of the gridding kernels.

  python tools/probe_nufft.py [--scale 1.0] [--coils 16] [--steps 5] [--device-plan 0|1]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2305_06482_b200 import synth
from paper_2305_06482_b200.nufft import GriddedKernel


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--coils", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--binsize", type=int, default=0)
    ap.add_argument("--compare", action="store_true", help="relative difference vs the per-sample "
                    "(unbinned, float atomics) path on the same plan geometry")
    args = ap.parse_args()
    dims = tuple(int(round(n * args.scale)) for n in (256, 256, 160))
    pts = synth.cones_3d(dims, n_readouts=int(18000 * args.scale ** 2), n_samples=int(512 * args.scale))
    torch.cuda.init()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kern = GriddedKernel(dims, pts, 1.25, 4, binsize=args.binsize or None)
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    D = kern.D
    maps = torch.randn(1, args.coils, D, dtype=torch.complex64, device="cuda") * 0.2
    x = torch.from_numpy(synth.random_ellipses(dims, 20, rng).ravel().astype(np.complex64)).cuda().view(1, -1)
    r = np.linalg.norm(pts, axis=1)
    w = torch.from_numpy((r / r.max()).astype(np.float32)).cuda()
    out = torch.empty_like(x)
    for _ in range(2):
        kern.normal(maps, x, out, w=w)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        kern.normal(maps, x, out, w=w)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    extra = {}
    if args.compare:
        ref = GriddedKernel(dims, pts, 1.25, 4, binned=False)
        out2 = torch.empty_like(x)
        ref.normal(maps, x, out2, w=w)
        extra["rel_vs_unbinned"] = float(torch.linalg.vector_norm(out - out2) / torch.linalg.vector_norm(out2))
    print(json.dumps({"dims": dims, "N": int(len(pts)), "coils": args.coils, "plan_s": t_plan,
                      "nchunks": kern.nchunks, "normal_ms": ms, **extra,
                      "checksum": float(torch.linalg.vector_norm(out).item())}), flush=True)


if __name__ == "__main__":
    main()
