import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch
from torch.profiler import ProfilerActivity, profile
import bench_configs as B
B.run_cfg4(False, outer=1, inner=1)  # warm-up
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    line = B.run_cfg4(False, outer=3, inner=10)
    torch.cuda.synchronize()
print(line.get("recon_wall_s"), line.get("sketched_normal_apply_s"))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18))
