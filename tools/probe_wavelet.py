"""DB4 2-D prox on a batch of slices (config 2: 256 slices of 256 x 160, 4 levels): per-call time."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2305_06482_b200.wavelet import WaveletEngine
B, dims = (int(sys.argv[1]) if len(sys.argv) > 1 else 256), (256, 160)
eng = WaveletEngine(dims, None, batch=B)
v = torch.randn(B, dims[0] * dims[1], dtype=torch.complex64, device="cuda")
out, z, xo = torch.empty_like(v), torch.empty_like(v), torch.randn_like(v)
th = torch.full((B,), 0.1, device="cuda")
for _ in range(3):
    eng.prox(v, out, thresh=th, zout=z, xold=xo, beta=0.3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    eng.prox(v, out, thresh=th, zout=z, xold=xo, beta=0.3)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
mb = B * dims[0] * dims[1] * 8 / 1e6
print(json.dumps({"batch": B, "levels": eng.levels, "prox_ms": ms, "image_MB": mb,
                  "GBps_2x_image_per_direction": 4 * mb / ms}))
