#!/usr/bin/env python3
"""K1 single-pass cluster schedule vs the three-launch schedule on the config-1 workload.

Prints JSON lines: relative L2 difference of the two schedules (plain and with the FISTA
epilogue / anchor), and ms per apply of each (CUDA events, 20 applies after 3 warm-ups).
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_06482_b200 import _lib  # noqa: E402


def rel(a, b):
    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--min-batch", type=int, default=16)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = bench.build_workload(0, dev)
    kern, smaps, x = w["kern"], w["smaps"], w["x"]
    out3 = torch.empty_like(x)
    outc = torch.empty_like(x)
    _lib.call("sr_cart_tune_cluster", 0)
    kern.normal(smaps, x, out3, chunk=0)
    _lib.call("sr_cart_tune_cluster", args.min_batch)
    kern.normal(smaps, x, outc, chunk=0)
    torch.cuda.synchronize()
    print(json.dumps({"check": "plain", "rel_l2": rel(outc, out3)}), flush=True)
    # epilogue + anchor
    g = torch.Generator(dev).manual_seed(3)
    a = torch.randn(x.shape, dtype=torch.complex64, device=dev, generator=g) * 0.1
    dd = torch.randn(x.shape, dtype=torch.complex64, device=dev, generator=g)
    coef = torch.tensor([[0.7, -0.3, 0.2, 0.0]] * x.shape[0], dtype=torch.float32, device=dev)
    _lib.call("sr_cart_tune_cluster", 0)
    kern.normal(smaps, x, out3, anchor=a, coef=coef, u=x, d=dd, chunk=0)
    _lib.call("sr_cart_tune_cluster", args.min_batch)
    kern.normal(smaps, x, outc, anchor=a, coef=coef, u=x, d=dd, chunk=0)
    torch.cuda.synchronize()
    print(json.dumps({"check": "epilogue", "rel_l2": rel(outc, out3)}), flush=True)
    prof = torch.zeros(7, dtype=torch.int64, device=dev)
    _lib.call("sr_cart_tune_cluster", args.min_batch)
    _lib.call("sr_cart_cluster_profile", prof.data_ptr())
    kern.normal(smaps, x, outc, chunk=0)
    torch.cuda.synchronize()
    _lib.call("sr_cart_cluster_profile", None)
    names = ["F_inv", "F_fwd", "R", "C", "X", "C_inv", "R_inv"]
    tot = float(prof.sum())
    nct = x.shape[0] * 4
    print(json.dumps({"phase_kcycles_per_cta": {n: round(float(v) / nct / 1e3, 1) for n, v in zip(names, prof.tolist())},
                      "share": {n: round(float(v) / tot, 3) for n, v in zip(names, prof.tolist())}}), flush=True)
    for mb in (0, args.min_batch):
        _lib.call("sr_cart_tune_cluster", mb)
        t = bench.time_applies(lambda: kern.normal(smaps, x, outc, chunk=0), args.steps, 3, torch.cuda.synchronize)
        print(json.dumps({"schedule": "cluster" if mb else "three-pass", "ms_per_apply": t * 1e3 / args.steps}),
              flush=True)


if __name__ == "__main__":
    main()
