"""Which allocations happen inside the engine's CUDA-graph captures (config-3 recon)?"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
import torch
import paper_2305_06482_b200.recon as R
import bench_configs as bc

orig = R._capture
def traced(fn, *a, **k):
    torch.cuda.memory._record_memory_history(max_entries=100000)
    out = orig(fn, *a, **k)
    snap = torch.cuda.memory._snapshot()
    torch.cuda.memory._record_memory_history(enabled=None)
    for ev in snap["device_traces"][0]:
        if ev["action"] in ("alloc", "segment_alloc"):
            fr = [f"{f['filename'].split('/')[-1]}:{f['line']}:{f['name']}" for f in ev.get("frames", []) if "paper_2305" in f["filename"]][:4]
            print(ev["action"], ev["size"], fr, flush=True)
    return out
R._capture = traced
bc.run_2d(int(sys.argv[1]) if len(sys.argv) > 1 else 3, False)
