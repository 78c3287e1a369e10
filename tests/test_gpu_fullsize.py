"""GPU tests at BASELINE.json's full sizes, through size-independent properties of the sketched
normal operator N = A_s^H A_s (and direct oracle parity on a sample of slices where the oracle
finishes in seconds):

* self-adjoint: <y, N x> = conj(<x, N y>)           (N = sum_j C_j^H F^H W F C_j is Hermitian)
* positive semidefinite: <x, N x> real and >= 0
* linear: N(a x + b y) = a N x + b N y
* additive over coils: N with C_hat maps = sum of the C_hat single-coil normal ops
* slice independence (Cartesian batch): a slice's result does not depend on the rest of the batch

Tolerances: the operator bar of north_star (1e-4) for oracle parity; 1e-5 for the float32
identities (the kernels compute in complex64; every identity here is exact in real arithmetic).
"""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import rel
from oracle import sketch_oracle as O

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

pytestmark = pytest.mark.gpu

OP_TOL = 1e-4
ID_TOL = 1e-5


def _dot(a: torch.Tensor, b: torch.Tensor) -> complex:
    """<a, b> = sum conj(a) b in float64 on the device."""
    return complex(torch.vdot(a.reshape(-1).to(torch.complex128), b.reshape(-1).to(torch.complex128)).item())


def _check_identities(apply, x, y, ncoils_apply=None):
    nx_, ny_ = apply(x), apply(y)
    # self-adjoint
    lhs, rhs = _dot(y, nx_), np.conj(_dot(x, ny_))
    scale = float(torch.linalg.vector_norm(nx_) * torch.linalg.vector_norm(y))
    assert abs(lhs - rhs) / scale < ID_TOL
    # positive semidefinite
    q = _dot(x, nx_)
    assert q.real > 0 and abs(q.imag) / abs(q) < ID_TOL
    # linear
    a, b = 2.0 - 0.5j, -3.0j
    lin = apply(a * x + b * y)
    assert rel(lin.cpu().numpy(), (a * nx_ + b * ny_).cpu().numpy()) < ID_TOL
    return nx_


@pytest.fixture(scope="module")
def cfg1():
    import bench
    w = bench.build_workload(0, torch.device("cuda", 0))
    yield w
    del w
    torch.cuda.empty_cache()


def test_config1_full_size_properties(cuda, cfg1):
    """Config 1 at full size: 64 slices of 320^2, C_hat = 12 sketched maps (the bench workload)."""
    kern, smaps, x = cfg1["kern"], cfg1["smaps"], cfg1["x"]
    g = torch.Generator("cuda").manual_seed(3)
    y = torch.randn(x.shape, dtype=torch.complex64, device="cuda", generator=g)

    def apply(v):
        out = torch.empty_like(v)
        kern.normal(smaps, v.contiguous(), out)
        return out

    nx_ = _check_identities(apply, x, y)
    # additive over coils (a checksum of per-coil operators)
    acc = torch.zeros(x.shape, dtype=torch.complex128, device="cuda")
    for j in range(smaps.shape[1]):
        acc += apply_coils(kern, smaps[:, j:j + 1].contiguous(), x).to(torch.complex128)
    assert rel(nx_.cpu().numpy(), acc.cpu().numpy()) < ID_TOL
    # slice independence: slices 5 and 37 alone (batch-1 kernels) equal their batch results
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.plan import cartesian_plan
    for b in (5, 37):
        k1 = CartesianKernel(kern.dims, [cartesian_plan(kern.dims, cfg1["pts"][b])])
        o1 = torch.empty_like(x[b:b + 1])
        k1.normal(smaps[b:b + 1].contiguous(), x[b:b + 1].contiguous(), o1)
        assert rel(o1.cpu().numpy(), nx_[b:b + 1].cpu().numpy()) < 1e-6


def apply_coils(kern, maps, x):
    out = torch.empty_like(x)
    kern.normal(maps, x, out)
    return out


def test_config1_full_size_oracle_slices(cuda, cfg1):
    """Direct parity at full size on two sampled slices (oracle: numpy complex128, ~1 s)."""
    kern, smaps, x = cfg1["kern"], cfg1["smaps"], cfg1["x"]
    out = torch.empty_like(x)
    kern.normal(smaps, x, out)
    for b in (0, 63):
        ref = O.Sense(smaps[b].cpu().numpy().astype(np.complex128),
                      O.CartesianKernel(kern.dims, cfg1["pts"][b])).normal(x[b].cpu().numpy().astype(np.complex128))
        assert rel(out[b].cpu().numpy(), ref) < OP_TOL


def test_config2_shape_full_batch(cuda):
    """Config-2 slice geometry at full batch: 256 slices of 256x160, C_hat = 12, one shared ky-kz
    Poisson mask (R = 8, 20x20 centre): identities on the batch, oracle parity on two slices."""
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.plan import cartesian_plan
    dims, B, C = (256, 160), 256, 12
    D = dims[0] * dims[1]
    mask = synth.vd_poisson_mask(dims, 8.0, 20, 0)
    pts = synth.mask_points(mask)
    kern = CartesianKernel(dims, [cartesian_plan(dims, pts)], batch=B)
    g = torch.Generator("cuda").manual_seed(9)
    maps = (torch.randn(B, C, D, dtype=torch.complex64, device="cuda", generator=g) * 0.25).contiguous()
    x = torch.randn(B, D, dtype=torch.complex64, device="cuda", generator=g)
    y = torch.randn(B, D, dtype=torch.complex64, device="cuda", generator=g)

    def apply(v):
        out = torch.empty_like(v)
        kern.normal(maps, v.contiguous(), out)
        return out

    nx_ = _check_identities(apply, x, y)
    for b in (0, 255):
        ref = O.Sense(maps[b].cpu().numpy().astype(np.complex128),
                      O.CartesianKernel(dims, pts)).normal(x[b].cpu().numpy().astype(np.complex128))
        assert rel(nx_[b].cpu().numpy(), ref) < OP_TOL


def test_config4_full_size_nufft_properties(cuda):
    """Config 4 at full size: 256x256x160, 3-D cones N = 9.2 M, KB 1.25x / w4, 16 sketched coils,
    density weights.  Identities, coil additivity, and agreement of the binned fixed-point gridding
    with the per-sample float-atomic path (no shared-memory tiles, no fixed point)."""
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.nufft import GriddedKernel
    dims = (256, 256, 160)
    pts = synth.cones_3d(dims, n_readouts=18000, n_samples=512)
    assert len(pts) > 9_000_000
    kern = GriddedKernel(dims, pts, 1.25, 4)
    D = kern.D
    g = torch.Generator("cuda").manual_seed(4)
    maps = (torch.randn(1, 16, D, dtype=torch.complex64, device="cuda", generator=g) * 0.25).contiguous()
    r = np.linalg.norm(pts, axis=1)
    sw = torch.from_numpy(np.sqrt(r / r.max())).cuda()
    rng = np.random.default_rng(0)
    x = torch.from_numpy(synth.random_ellipses(dims, 20, rng).ravel().astype(np.complex64)).cuda().view(1, -1)
    y = torch.randn(1, D, dtype=torch.complex64, device="cuda", generator=g)

    def apply(v, m=maps, k=kern):
        out = torch.empty_like(v)
        k.normal(m, v.contiguous(), out, w=sw)
        return out

    nx_ = _check_identities(apply, x, y)
    acc = apply(x, maps[:, :8].contiguous()).to(torch.complex128) + apply(x, maps[:, 8:].contiguous())
    assert rel(nx_.cpu().numpy(), acc.cpu().numpy()) < ID_TOL
    ref = GriddedKernel(dims, pts, 1.25, 4, binned=False)
    assert rel(nx_.cpu().numpy(), apply(x, maps, ref).cpu().numpy()) < ID_TOL


def test_config4_geometry_half_scale_vs_oracle(cuda):
    """Config-4 cones geometry at half scale per axis (128x128x80, N = 1.15 M, KB 1.25x / w4),
    one sketched coil with density weights: device normal op vs the oracle (bounded-memory
    chunked kernel).  tools/bench_configs.py --config 4 --oracle runs the same check at full size
    (measured rel L2 1.8e-6)."""
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.nufft import GriddedKernel
    dims = (128, 128, 80)
    pts = synth.cones_3d(dims, n_readouts=4500, n_samples=256)
    r = np.linalg.norm(pts, axis=1)
    w = r / r.max()
    rng = np.random.default_rng(21)
    D = int(np.prod(dims))
    m = (rng.standard_normal(D) + 1j * rng.standard_normal(D)) * 0.3
    x = synth.random_ellipses(dims, 20, rng).ravel()
    kern = GriddedKernel(dims, pts, 1.25, 4)
    out = torch.empty(1, D, dtype=torch.complex64, device="cuda")
    kern.normal(torch.from_numpy(m.astype(np.complex64)).cuda().view(1, 1, -1),
                torch.from_numpy(x.astype(np.complex64)).cuda().view(1, -1), out,
                w=torch.from_numpy(np.sqrt(w)).cuda())
    ref = O.Sense(m[None, :], O.ChunkedGriddedKernel(dims, pts, 1.25, 4), w).normal(x)
    assert rel(out[0].cpu().numpy(), ref) < OP_TOL
