#!/usr/bin/env python3
"""Sweep K1 (fused Cartesian normal op) settings on the config-1 workload.

Prints one line per setting with ms/apply and algorithmic GB/s.  Used to pick
the slice-chunk size (L2 residency of the coil workspace); not part of bench.
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
    ap.add_argument("--fused", default="", help="semicolon list of lagB,lagC,slots,tile configs of the persistent launch")
    ap.add_argument("--coljc", default="", help="comma list of column-pass coils per CTA (0 = generic)")
    ap.add_argument("--group", default="", help="comma list of group sizes G for chunk -2")
    ap.add_argument("--stats", action="store_true", help="collect fused-kernel wait/item statistics")
    ap.add_argument("--colpf", default="", help="comma list of column-pass prefetch modes (1 / 0)")
    ap.add_argument("--carveout", default="", help="comma list of shared-memory carveouts (percent, -1 = default); "
                                                   "each runs the colpf list")
    ap.add_argument("--split", default="", help="semicolon list of jc,ja settings of the split-column schedule (chunk -3)")
    ap.add_argument("--multistream", default="", help="semicolon list of chunk,streams for the three-pass schedule")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = bench.build_workload(0, dev)
    kern, smaps, x = w["kern"], w["smaps"], w["x"]
    out = torch.empty_like(x)
    from paper_2305_06482_b200 import _lib
    for cv in [int(c) for c in args.carveout.split(",") if c] or [None]:
        if cv is not None:
            _lib.call("sr_cart_tune_carveout", cv)
        for pf in [int(c) for c in args.colpf.split(",") if c]:
            _lib.call("sr_cart_tune_colpf", pf)
            t = bench.time_applies(lambda: kern.normal(smaps, x, out, chunk=0), args.steps, 3, torch.cuda.synchronize)
            print(json.dumps({"carveout": cv, "colpf": pf, "ms_per_apply": t * 1e3 / args.steps}), flush=True)
    _lib.call("sr_cart_tune_colpf", 1)
    for cfg in [c for c in args.split.split(";") if c]:
        jc, ja = (int(v) for v in cfg.split(","))
        _lib.call("sr_split_tune", jc, ja)
        t = bench.time_applies(lambda: kern.normal(smaps, x, out, chunk=-3), args.steps, 3, torch.cuda.synchronize)
        print(json.dumps({"split_jc": jc, "split_ja": ja, "ms_per_apply": t * 1e3 / args.steps}), flush=True)
    for cfg in [c for c in args.fused.split(";") if c]:
        lb, lc, sl, tl = (int(v) for v in cfg.split(","))
        _lib.call("sr_fused_config", lb, lc, sl, tl)
        kern._ws = None
        t = bench.time_applies(lambda: kern.normal(smaps, x, out, chunk=-1), args.steps, 3, torch.cuda.synchronize)
        ms = t / args.steps * 1e3
        rec = {"fused": cfg, "ms_per_apply": ms, "alg_GBps": bench.algorithmic_bytes() / (ms * 1e-3) / 1e9}
        if args.stats:
            st = torch.zeros(8, dtype=torch.int64, device=dev)
            _lib.call("sr_fused_stats", st.data_ptr())
            kern.normal(smaps, x, out, chunk=-1)
            torch.cuda.synchronize()
            _lib.call("sr_fused_stats", None)
            rec["stats"] = st.cpu().tolist()
        print(json.dumps(rec), flush=True)
    for cfg in [c for c in args.multistream.split(";") if c]:
        ch, ns = (int(v) for v in cfg.split(","))
        ms = multistream(kern, smaps, x, out, ch, ns)
        print(json.dumps({"multistream": cfg, "ms_per_apply": ms}), flush=True)
    for jc in [int(c) for c in args.coljc.split(",") if c]:
        _lib.call("sr_cart_tune", jc)
        t = bench.time_applies(lambda: kern.normal(smaps, x, out, chunk=0), args.steps, 3, torch.cuda.synchronize)
        ms = t / args.steps * 1e3
        print(json.dumps({"coljc": jc, "ms_per_apply": ms, "alg_GBps": bench.algorithmic_bytes() / (ms * 1e-3) / 1e9}),
              flush=True)
    if args.coljc:
        _lib.call("sr_cart_tune", 4)
    for g in [int(c) for c in args.group.split(",") if c]:
        _lib.call("sr_group_select", g)
        t = bench.time_applies(lambda: kern.normal(smaps, x, out, chunk=-2), args.steps, 3, torch.cuda.synchronize)
        ms = t / args.steps * 1e3
        print(json.dumps({"group": g, "ngroups": _lib.lib().sr_group_ngroups(kern.ny, kern.nx), "ms_per_apply": ms,
                          "alg_GBps": bench.algorithmic_bytes() / (ms * 1e-3) / 1e9}), flush=True)
    _lib.call("sr_group_select", 0)
    for ch in [int(c) for c in args.chunks.split(",") if c]:
        t = bench.time_applies(lambda: kern.normal(smaps, x, out, chunk=ch), args.steps, 3, torch.cuda.synchronize)
        ms = t / args.steps * 1e3
        print(json.dumps({"chunk": ch, "ms_per_apply": ms,
                          "alg_GBps": bench.algorithmic_bytes() / (ms * 1e-3) / 1e9}), flush=True)





def multistream(kern, smaps, x, out, chunk, nstreams, steps=20):
    """Three-pass K1 over slice chunks spread round-robin over `nstreams` streams (L2 experiment)."""
    import torch
    ncoils = smaps.shape[1]
    B = kern.batch
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    wss = [torch.empty(chunk * ncoils * kern.D, dtype=torch.complex64, device=x.device) for _ in range(nstreams)]
    cur = torch.cuda.current_stream()

    def once():
        for s in streams:
            s.wait_stream(cur)
        for i, b0 in enumerate(range(0, B, chunk)):
            k = i % nstreams
            kern._normal_range(smaps, x, out, b0, min(B, b0 + chunk), wss[k], streams[k].cuda_stream)
        for s in streams:
            cur.wait_stream(s)

    t = bench.time_applies(once, steps, 3, torch.cuda.synchronize)
    return t / steps * 1e3


if __name__ == "__main__":
    main()
