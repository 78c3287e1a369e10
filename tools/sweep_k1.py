#!/usr/bin/env python3
"""Sweep K1 (fused Cartesian normal op) settings on the config-1 workload.

Prints one JSON line per setting with ms/apply.  Knobs of the three-launch schedule: slice
chunks (L2 residency of the coil workspace), column-pass coils per CTA, next-coil register
prefetch, shared-memory carveout, row-pass store mode.  (The persistent / group / split
schedules of round 1 were removed in round 2; their measurements are in DESIGN.md.)
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", default="0,32,16")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--coljc", default="", help="comma list of column-pass coils per CTA (0 = generic)")
    ap.add_argument("--colpf", default="", help="comma list of column-pass prefetch modes (1 / 0)")
    ap.add_argument("--carveout", default="", help="comma list of column-pass shared-memory carveouts (percent, "
                                                   "-1 = default); each runs the colpf list")
    ap.add_argument("--rows", default="", help="semicolon list of bulk,min_n row-pass store modes")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = bench.build_workload(0, dev)
    kern, smaps, x = w["kern"], w["smaps"], w["x"]
    out = torch.empty_like(x)
    from paper_2305_06482_b200 import _lib

    def run(**tag):
        t = bench.time_applies(lambda: kern.normal(smaps, x, out, chunk=tag.get("chunk", 0)), args.steps, 3,
                               torch.cuda.synchronize)
        print(json.dumps({**tag, "ms_per_apply": t * 1e3 / args.steps}), flush=True)

    for cv in [int(c) for c in args.carveout.split(",") if c] or [None]:
        if cv is not None:
            _lib.call("sr_cart_tune_carveout", cv)
        for pf in [int(c) for c in args.colpf.split(",") if c]:
            _lib.call("sr_cart_tune_colpf", pf)
            run(carveout=cv, colpf=pf)
    _lib.call("sr_cart_tune_colpf", 1)
    _lib.call("sr_cart_tune_carveout", -1)
    for jc in [int(c) for c in args.coljc.split(",") if c]:
        _lib.call("sr_cart_tune", jc)
        run(coljc=jc)
    _lib.call("sr_cart_tune", 4)
    for cfg in [c for c in args.rows.split(";") if c]:
        bulk, min_n = (int(v) for v in cfg.split(","))
        _lib.call("sr_cart_tune_rows", bulk, min_n)
        run(rows=[bulk, min_n])
    _lib.call("sr_cart_tune_rows", 2, 0)
    for ch in [int(c) for c in args.chunks.split(",") if c]:
        run(chunk=ch)


if __name__ == "__main__":
    main()
