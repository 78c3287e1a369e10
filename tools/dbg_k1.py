"""Debug: run each K1/K2 entry point once per geometry with a sync after each (CUDA_LAUNCH_BLOCKING)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2305_06482_b200.cartesian import CartesianKernel
from paper_2305_06482_b200.plan import cartesian_plan

for dims in [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]:
    rng = np.random.default_rng(7)
    B, C = 3, 5
    D = dims[0] * dims[1]
    plans = [cartesian_plan(dims, np.argwhere(rng.random(dims) < 0.2) - np.array([n // 2 for n in dims]))
             for _ in range(B)]
    kern = CartesianKernel(dims, plans)
    md = torch.randn(B, C, D, dtype=torch.complex64, device="cuda")
    xd = torch.randn(B, D, dtype=torch.complex64, device="cuda")
    for name, fn in [("normal0", lambda: kern.normal(md, xd, torch.empty_like(xd), chunk=0)),
                     ("forward", lambda: kern.forward(md, xd))]:
        try:
            fn()
            torch.cuda.synchronize()
            print(dims, name, "ok", flush=True)
        except Exception as e:  # noqa: BLE001
            print(dims, name, "FAIL", str(e)[:80], flush=True)
            try:
                torch.cuda.synchronize()
            except Exception as e2:  # noqa: BLE001
                print("  sync:", str(e2)[:200], flush=True)
            sys.exit(1)
