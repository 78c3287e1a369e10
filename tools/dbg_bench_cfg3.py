"""Why does config 3 read 50-110 ms inside bench.py and 42-46 ms alone?  Stage the bench process
step by step and time run_2d(3) after each stage."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
import torch
import bench
import bench_configs as bc

def t3(tag):
    torch.cuda.init(); st0 = torch.cuda.memory_stats()
    r = bc.run_2d(3, False)
    st1 = torch.cuda.memory_stats()
    print(tag, [round(v * 1e3, 1) for v in r["gpu_wall_s_runs"]],
          "cudaMalloc", st1.get("num_device_alloc", 0) - st0.get("num_device_alloc", 0),
          "cudaFree", st1.get("num_device_free", 0) - st0.get("num_device_free", 0),
          "reserved MB", st1.get("reserved_bytes.all.current", 0) >> 20, flush=True)

dev = torch.device("cuda", 0)
t3("fresh process")
w = bench.build_workload(0, dev)
t3("after build_workload")
kern, smaps, x = w["kern"], w["smaps"], w["x"]
out = torch.empty_like(x)
bench.time_applies(lambda: kern.normal(smaps, x, out), 20, 3, torch.cuda.synchronize)
t3("after K1 timing")
x_host = x.cpu().pin_memory(); out_host = torch.empty_like(x_host).pin_memory()
stage = (torch.empty_like(x), torch.empty_like(x))
bench.time_applies(lambda: kern.normal_host(smaps, x_host, out_host, chunks=8, buffers=stage, overlap_prev=True), 10, 2, torch.cuda.synchronize)
t3("after e2e")
with bench.ClockSampler(0) if hasattr(bench, "ClockSampler") else open("/dev/null") as s:
    pass
t3("after sampler")
