#!/usr/bin/env python3
"""e2e (host buffers) throughput of the config-1 normal op vs slice-chunk count."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    w = bench.build_workload(0, dev)
    kern, smaps, x = w["kern"], w["smaps"], w["x"]
    x_host = x.cpu().pin_memory()
    out_host = torch.empty_like(x_host).pin_memory()
    stage = (torch.empty_like(x), torch.empty_like(x))
    for spec in (sys.argv[1] if len(sys.argv) > 1 else "8:1,8:2,16:2,16:3").split(","):
        # "n:lanes" (n equal chunks) or "s1/s2/.../sk:lanes" (explicit slice counts)
        c, lanes = spec.split(":")
        ch = [int(v) for v in c.split("/")] if "/" in c else int(c)
        lanes = int(lanes)
        steps = 20
        for ov in (False, True):
            t = bench.time_applies(lambda: kern.normal_host(smaps, x_host, out_host, chunks=ch, buffers=stage,
                                                            lanes=lanes, overlap_prev=ov), steps, 3,
                                   torch.cuda.synchronize)
            print(json.dumps({"chunks": ch, "lanes": lanes, "overlap_prev": ov, "e2e_applies_per_s": steps / t,
                              "ms": t / steps * 1e3}), flush=True)
    # raw copy bandwidth
    xd = stage[0]
    for name, fn in [("h2d", lambda: xd.copy_(x_host, non_blocking=True)),
                     ("d2h", lambda: out_host.copy_(xd, non_blocking=True))]:
        t = bench.time_applies(fn, 20, 3, torch.cuda.synchronize)
        print(json.dumps({name: x_host.numel() * 8 * 20 / t / 1e9, "unit": "GB/s"}), flush=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    x_host2 = torch.empty_like(x_host).pin_memory()

    def duplex():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            xd.copy_(x_host, non_blocking=True)
        with torch.cuda.stream(s2):
            x_host2.copy_(stage[1], non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    t = bench.time_applies(duplex, 20, 3, torch.cuda.synchronize)
    print(json.dumps({"duplex_ms": t / 20 * 1e3, "each_GBps": x_host.numel() * 8 * 20 / t / 1e9}), flush=True)


if __name__ == "__main__":
    main()
