"""Debug: 3-D NUFFT normal (fused path) vs adjoint(forward) (unfused) vs oracle."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from oracle import sketch_oracle as O
from paper_2305_06482_b200 import synth
from paper_2305_06482_b200.nufft import GriddedKernel


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


for dims in [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]:
    rng = np.random.default_rng(13)
    D = int(np.prod(dims))
    pts = synth.cones_3d(dims, n_readouts=60, n_samples=200)
    maps = (rng.standard_normal((2, D)) + 1j * rng.standard_normal((2, D))) / 3
    x = rng.standard_normal(D) + 1j * rng.standard_normal(D)
    ok = O.GriddedKernel(dims, pts, 1.25, 4)
    ref = O.Sense(maps, ok).normal(x)
    kern = GriddedKernel(dims, pts, 1.25, 4)
    md = torch.from_numpy(maps.astype(np.complex64)).cuda().unsqueeze(0)
    xd = torch.from_numpy(x.astype(np.complex64)).cuda().view(1, -1)
    out = torch.empty_like(xd)
    kern.normal(md, xd, out)
    y = kern.forward(md, xd)
    adj = torch.empty_like(xd)
    kern.adjoint(md, y, adj)
    yref = O.Sense(maps, ok).forward(x)
    print(dims, "gdims", kern.gdims, "normal", rel(out.cpu().numpy(), ref), "adj(fwd)", rel(adj.cpu().numpy(), ref),
          "fwd", rel(y.cpu().numpy(), yref), flush=True)

if len(sys.argv) == 1 or True:
    dims = (16, 24, 32)
    rng = np.random.default_rng(13)
    D = int(np.prod(dims))
    pts = synth.cones_3d(dims, n_readouts=60, n_samples=200)
    maps = np.ones((1, D), dtype=np.complex128)
    x = rng.standard_normal(D) + 1j * rng.standard_normal(D)
    ok = O.GriddedKernel(dims, pts, 1.25, 4)
    yref = O.Sense(maps, ok).forward(x)
    kern = GriddedKernel(dims, pts, 1.25, 4)
    y = kern.forward(torch.from_numpy(maps.astype(np.complex64)).cuda().unsqueeze(0),
                     torch.from_numpy(x.astype(np.complex64)).cuda().view(1, -1)).cpu().numpy().ravel()
    err = np.abs(y - yref) / np.abs(yref).max()
    r = np.linalg.norm(pts / (np.array(dims) / 2.0), axis=1)
    print("pts range", pts.min(axis=0), pts.max(axis=0), "dims/2", np.array(dims) / 2)
    order = np.argsort(-err)[:8]
    for i in order:
        print(" err %.2e  pt %s  r %.3f" % (err[i], pts[i], r[i]))
    for lo_, hi_ in [(0, 0.5), (0.5, 0.9), (0.9, 0.99), (0.99, 2)]:
        m = (r >= lo_) & (r < hi_)
        if m.any():
            print(" r in [%.2f,%.2f): n=%d max err %.2e" % (lo_, hi_, m.sum(), err[m].max()))
