#!/usr/bin/env python3
"""K1 at a given geometry with the rowfwd TMA bulk store on/off (tuning of sr_cart_tune_rows)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_06482_b200 import _lib  # noqa: E402
from paper_2305_06482_b200.cartesian import CartesianKernel  # noqa: E402
from paper_2305_06482_b200.plan import cartesian_plan  # noqa: E402


def main():
    for spec in sys.argv[1:]:
        ny, nx, B, C = (int(v) for v in spec.split("x"))
        rng = np.random.default_rng(0)
        dims = (ny, nx)
        pts = np.argwhere(rng.random(dims) < 0.2) - np.array([ny // 2, nx // 2])
        kern = CartesianKernel(dims, [cartesian_plan(dims, pts)], batch=B)
        maps = torch.randn(B, C, ny * nx, dtype=torch.complex64, device="cuda")
        x = torch.randn(B, ny * nx, dtype=torch.complex64, device="cuda")
        out = torch.empty_like(x)
        for bulk in (0, 1):
            _lib.call("sr_cart_tune_rows", bulk, 0)
            t = bench.time_applies(lambda: kern.normal(maps, x, out, chunk=0), 20, 3, torch.cuda.synchronize)
            print(json.dumps({"dims": dims, "B": B, "C": C, "bulk": bulk, "ms": t / 20 * 1e3}), flush=True)
    _lib.call("sr_cart_tune_rows", 2, 0)


if __name__ == "__main__":
    main()
