"""Kernel-time table (torch profiler) of the config-2 batched reconstruction (256 slices)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
import torch
from torch.profiler import ProfilerActivity, profile
import bench_configs as B
B.run_cfg2(False, 256, 0)  # warm-up
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    line = B.run_cfg2(False, 256, 0)
    torch.cuda.synchronize()
print(line.get("gpu_wall_s"), line.get("gpu_solve_s"), line.get("compression_s"))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
