"""3-D DB4 prox (config 4 volume 256 x 256 x 160, 4 levels): per-call time."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2305_06482_b200.wavelet import WaveletEngine
dims = (256, 256, 160)
eng = WaveletEngine(dims, None, batch=1)
D = dims[0] * dims[1] * dims[2]
v = torch.randn(1, D, dtype=torch.complex64, device="cuda")
out, z, xo = torch.empty_like(v), torch.empty_like(v), torch.randn_like(v)
th = torch.full((1,), 0.1, device="cuda")
for _ in range(3):
    eng.prox(v, out, thresh=th, zout=z, xold=xo, beta=0.3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    eng.prox(v, out, thresh=th, zout=z, xold=xo, beta=0.3)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"levels": eng.levels, "prox_ms": e0.elapsed_time(e1) / 10, "checksum": float(out.abs().sum())}))
