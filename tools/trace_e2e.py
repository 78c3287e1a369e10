#!/usr/bin/env python3
"""Timeline of the config-1 e2e step (pinned host in -> K1 over slice chunks -> pinned host out)
from the torch profiler: per-stream copy / kernel intervals of one step, to see where the PCIe
pipeline idles.  usage: trace_e2e.py [chunks e.g. 8 or 2/6/8/8/8/8/8/8/4/2/2] [lanes]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402


def main():
    spec = sys.argv[1] if len(sys.argv) > 1 else "8"
    lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    chunks = [int(v) for v in spec.split("/")] if "/" in spec else int(spec)
    dev = torch.device("cuda", 0)
    w = bench.build_workload(0, dev)
    kern, smaps, x = w["kern"], w["smaps"], w["x"]
    x_host = x.cpu().pin_memory()
    out_host = torch.empty_like(x_host).pin_memory()
    stage = (torch.empty_like(x), torch.empty_like(x))
    for _ in range(3):
        kern.normal_host(smaps, x_host, out_host, chunks=chunks, buffers=stage, lanes=lanes, overlap_prev=True)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            kern.normal_host(smaps, x_host, out_host, chunks=chunks, buffers=stage, lanes=lanes, overlap_prev=True)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    # last of the three steps
    n = len(evs) // 3
    step = evs[-n:]
    s0 = step[0].time_range.start
    for e in step:
        name = e.name[:40]
        print(f"{(e.time_range.start - s0):8.1f} {(e.time_range.end - s0):8.1f} us  {name}")
    print("step span us:", step[-1].time_range.end - s0, " 3-step span us:", evs[-1].time_range.end - t0)


if __name__ == "__main__":
    main()
