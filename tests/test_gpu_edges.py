"""GPU edge cases of the operator path: empty and ragged sample sets, a single coil, a zero
update, unsupported sizes and malformed arguments (errors raised, never a silent fallback)."""

import numpy as np
import pytest
import torch

from conftest import rel
from oracle import sketch_oracle as O

pytestmark = pytest.mark.gpu

OP_TOL = 1e-4


def _kern(dims, pts_list):
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.plan import cartesian_plan
    return CartesianKernel(dims, [cartesian_plan(dims, p) for p in pts_list])


def _c64(a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(np.complex64)).cuda()


def test_empty_and_ragged_masks(cuda):
    """Slice 0 has no samples (A^H A = 0), slice 1 a handful, slice 2 a dense mask."""
    rng = np.random.default_rng(4)
    dims, C = (48, 40), 3
    D = dims[0] * dims[1]
    half = np.array([n // 2 for n in dims])
    pts = [np.zeros((0, 2), dtype=np.int64),
           np.argwhere(rng.random(dims) < 0.01) - half,
           np.argwhere(rng.random(dims) < 0.5) - half]
    kern = _kern(dims, pts)
    maps = (rng.standard_normal((3, C, D)) + 1j * rng.standard_normal((3, C, D))) / 2
    x = rng.standard_normal((3, D)) + 1j * rng.standard_normal((3, D))
    out = torch.full((3, D), float("nan"), dtype=torch.complex64, device="cuda")
    kern.normal(_c64(maps), _c64(x), out)
    got = out.cpu().numpy()
    assert np.all(got[0] == 0)
    for b in (1, 2):
        ref = O.Sense(maps[b], O.CartesianKernel(dims, pts[b])).normal(x[b])
        assert rel(got[b], ref) < OP_TOL
    y = kern.forward(_c64(maps), _c64(x))
    assert y.shape[-1] == max(len(p) for p in pts)
    assert np.all(y[0].cpu().numpy() == 0)


def test_single_coil_and_zero_update(cuda):
    """C = 1, and x == anchor gives exactly the epilogue's d term."""
    rng = np.random.default_rng(5)
    dims = (32, 32)
    D = dims[0] * dims[1]
    pts = [np.argwhere(rng.random(dims) < 0.3) - 16]
    kern = _kern(dims, pts)
    maps = rng.standard_normal((1, 1, D)) + 1j * rng.standard_normal((1, 1, D))
    x = rng.standard_normal((1, D)) + 1j * rng.standard_normal((1, D))
    out = torch.empty(1, D, dtype=torch.complex64, device="cuda")
    kern.normal(_c64(maps), _c64(x), out)
    ref = O.Sense(maps[0], O.CartesianKernel(dims, pts[0])).normal(x[0])
    assert rel(out.cpu().numpy()[0], ref) < OP_TOL
    d = rng.standard_normal((1, D)) + 1j * rng.standard_normal((1, D))
    coef = torch.tensor([[0.7, 0.0, 1.0, 0.0]], dtype=torch.float32, device="cuda")
    xt = _c64(x)
    kern.normal(_c64(maps), xt, out, anchor=xt, coef=coef, d=_c64(d))
    np.testing.assert_allclose(out.cpu().numpy(), d.astype(np.complex64), rtol=0, atol=0)


def test_unsupported_size_and_bad_arguments(cuda):
    from paper_2305_06482_b200 import _lib
    assert _lib.lib().sr_fft_size_supported(14) == 0  # 2 x 7: no 7-point codelet
    with pytest.raises(ValueError):
        _kern((14, 16), [np.zeros((1, 2), dtype=np.int64)])
    kern = _kern((32, 32), [np.zeros((1, 2), dtype=np.int64)])
    x = torch.zeros(1, 1024, dtype=torch.complex64, device="cuda")
    out = torch.empty_like(x)
    with pytest.raises(ValueError):  # maps of the wrong length
        kern.normal(torch.zeros(1, 2, 1000, dtype=torch.complex64, device="cuda"), x, out)
    with pytest.raises(ValueError):  # wrong dtype
        kern.normal(torch.zeros(1, 2, 1024, dtype=torch.complex128, device="cuda"), x, out)
    with pytest.raises(ValueError):  # density weights are not defined for Cartesian masks
        kern.normal(torch.zeros(1, 2, 1024, dtype=torch.complex64, device="cuda"), x, out,
                    w=torch.ones(1, device="cuda"))
    # the C ABI rejects bad shapes itself (no launch)
    with pytest.raises(ValueError):
        _lib.call("sr_cart_normal", x.data_ptr(), None, x.data_ptr(), 0, None, 0, out.data_ptr(), None,
                  0, 1, 32, 32, None, None, None, 0, 0)


def test_nufft_without_samples(cuda):
    """A trajectory with no points: the gridded operator is the zero map."""
    from paper_2305_06482_b200.nufft import GriddedKernel
    dims = (32, 32)
    kern = GriddedKernel(dims, np.zeros((0, 2)), 2.0, 4)
    D = 32 * 32
    maps = torch.ones(1, 2, D, dtype=torch.complex64, device="cuda")
    x = torch.ones(1, D, dtype=torch.complex64, device="cuda")
    out = torch.full_like(x, float("nan"))
    kern.normal(maps, x, out)
    assert torch.all(out == 0)


@pytest.mark.parametrize("dims", [(320, 320), (256, 160), (240, 200)])
def test_row_pass_store_modes_agree(cuda, dims):
    """The row FFT pass's TMA bulk stores and its copy-out pass write identical workspaces."""
    from paper_2305_06482_b200 import _lib
    rng = np.random.default_rng(8)
    D = dims[0] * dims[1]
    half = np.array([n // 2 for n in dims])
    kern = _kern(dims, [np.argwhere(rng.random(dims) < 0.2) - half for _ in range(2)])
    maps = _c64((rng.standard_normal((2, 3, D)) + 1j * rng.standard_normal((2, 3, D))) / 2)
    x = _c64(rng.standard_normal((2, D)) + 1j * rng.standard_normal((2, D)))
    outs = []
    try:
        for mode in (0, 1):
            _lib.call("sr_cart_tune_rows", mode, 0)
            o = torch.empty_like(x)
            kern.normal(maps, x, o)
            outs.append(o.cpu().numpy())
    finally:
        _lib.call("sr_cart_tune_rows", 2, 0)
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("dims", [(320, 320), (256, 160), (256, 256)])
def test_column_pass_prefetch_modes_agree(cuda, dims):
    """The coil-looped column pass with and without the register prefetch of the next coil's
    strip (sr_cart_tune_colpf) computes identical results (same arithmetic, different schedule)."""
    from paper_2305_06482_b200 import _lib
    rng = np.random.default_rng(12)
    D = dims[0] * dims[1]
    half = np.array([n // 2 for n in dims])
    kern = _kern(dims, [np.argwhere(rng.random(dims) < 0.2) - half for _ in range(2)])
    maps = _c64((rng.standard_normal((2, 6, D)) + 1j * rng.standard_normal((2, 6, D))) / 2)
    x = _c64(rng.standard_normal((2, D)) + 1j * rng.standard_normal((2, D)))
    outs = []
    try:
        for pf in (1, 0):
            _lib.call("sr_cart_tune_colpf", pf)
            o = torch.empty_like(x)
            kern.normal(maps, x, o)
            outs.append(o.cpu().numpy())
    finally:
        _lib.call("sr_cart_tune_colpf", 1)
    np.testing.assert_array_equal(outs[0], outs[1])
    with pytest.raises(ValueError):
        _lib.call("sr_cart_tune_colpf", 2)


@pytest.mark.parametrize("B,C,chat,D", [(3, 32, 12, 4096), (1, 16, 8, 1000), (2, 9, 5, 64), (1, 40, 32, 128)])
def test_real_sketch_contraction_matches_complex_path(cuda, B, C, chat, D):
    """K5 with a real coefficient matrix (2 FMAs per MAC, two voxels per thread) equals the
    general complex-coefficient kernel bit for bit (same fused multiply-adds, zero imaginary part)."""
    from paper_2305_06482_b200.sketching import coil_contract
    rng = np.random.default_rng(B * 100 + C)
    maps = _c64(rng.standard_normal((B, C, D)) + 1j * rng.standard_normal((B, C, D)))
    S = rng.standard_normal((chat, C))
    S[:2] = 0
    S[0, 0] = S[1, 1] = 1.0  # identity rows copy exactly
    got = coil_contract(maps, S)
    ref = coil_contract(maps, S.astype(np.complex128))
    np.testing.assert_array_equal(got.cpu().numpy(), ref.cpu().numpy())
    np.testing.assert_array_equal(got[:, :2].cpu().numpy(), maps[:, :2].cpu().numpy())


@pytest.mark.parametrize("dims,C", [((320, 320), 5), ((256, 160), 4), ((64, 40), 3), ((60,), 2)])
def test_fused_sample_io_matches_separate_passes(cuda, dims, C):
    """K2 with the sample gather / scatter inside the column pass equals the separate
    gather / scatter launches: ragged per-slice sample sets, duplicated bins (last write wins),
    residual against measured data and its per-block squared norms."""
    rng = np.random.default_rng(len(dims) * 10 + C)
    D = int(np.prod(dims))
    half = np.array([n // 2 for n in dims])
    pts_l = []
    for frac in (0.3, 0.05, 0.0 if len(dims) == 2 else 0.2):
        pts = np.argwhere(rng.random(dims) < frac) - half
        if len(pts):
            pts = np.concatenate([pts, pts[: max(1, len(pts) // 7)]])  # duplicates
        pts_l.append(pts.reshape(-1, len(dims)))
    kern = _kern(dims, pts_l)
    B = len(pts_l)
    maps = _c64((rng.standard_normal((B, C, D)) + 1j * rng.standard_normal((B, C, D))) / 2)
    x = _c64(rng.standard_normal((B, D)) + 1j * rng.standard_normal((B, D)))
    ymeas = _c64(rng.standard_normal((B, C, kern.nmax)) + 1j * rng.standard_normal((B, C, kern.nmax)))
    outs = {}
    for fused in (False, True):
        kern.fused_io = fused
        part = torch.zeros(kern.partial_shape(C), dtype=torch.float64, device="cuda")
        y = kern.forward(maps, x, ymeas=ymeas, partial=part)
        adj = torch.empty_like(x)
        kern.adjoint(maps, y, adj)
        outs[fused] = (y.cpu().numpy(), adj.cpu().numpy(), part.sum(dim=-1).cpu().numpy())
    kern.fused_io = True
    for b in range(B):  # equal up to the FMA contraction of the scale-and-subtract (~1 ulp)
        n = kern.n_points_per_slice[b]
        np.testing.assert_allclose(outs[True][0][b, :, :n], outs[False][0][b, :, :n], rtol=0, atol=2e-6)
    assert np.abs(outs[True][1] - outs[False][1]).max() <= 1e-6 * max(1.0, np.abs(outs[False][1]).max())
    np.testing.assert_allclose(outs[True][2], outs[False][2], rtol=1e-7)


@pytest.mark.parametrize("S,N,C", [(4, 5119, 32), (3, 700, 12), (2, 40, 40 // 2), (1, 33, 32),
                                   (1, 16384, 16), (1, 81920, 16), (1, 5000, 32)])
def test_tsqr_r_matches_lapack(cuda, S, N, C):
    """Batched tall-skinny Householder R (csrc/tsqr.cu) equals LAPACK's zgeqrf R (numpy.linalg.qr,
    mode "r") including the signs of its real diagonal; a zero column takes the tau = 0 path.  Single
    large blocks take the many-CTA kernel (grid barriers)."""
    from paper_2305_06482_b200 import _device as dv
    from paper_2305_06482_b200 import _lib
    rng = np.random.default_rng(S * N + C)
    A = (rng.standard_normal((S, N, C)) + 1j * rng.standard_normal((S, N, C))) * np.exp(rng.standard_normal((S, 1, C)))
    A[0, :, min(3, C - 1)] = 0.0
    At = torch.from_numpy(A).cuda().contiguous()
    R = torch.empty(S, C, C, dtype=torch.complex128, device="cuda")
    _lib.call("sr_tsqr_r", At.data_ptr(), N, C, N * C, S, R.data_ptr(), dv.stream())
    R = R.cpu().numpy()
    for s in range(S):
        ref = np.linalg.qr(A[s], mode="r")
        np.testing.assert_allclose(R[s], ref, rtol=0, atol=1e-10 * np.abs(ref).max())


def test_c_abi_plans_reject_out_of_range_coordinates(cuda):
    """sr_cart_plan_create / sr_nufft_plan_create return SR_EINVAL (ValueError) for a coordinate
    outside [-n/2, n/2), as Trajectory.validate_for (linops.py:130-140) rejects it, instead of
    wrapping it modulo n."""
    import ctypes
    from paper_2305_06482_b200 import _device as dv
    from paper_2305_06482_b200 import _lib
    dims = (32, 40)
    cdims = (ctypes.c_int * 2)(*dims)
    for bad in ([16.0, 0.0], [-17.0, 0.0], [0.0, 20.0], [0.0, float("nan")]):
        pts = np.array([[0.0, 0.0], bad], dtype=np.float64)
        counts = (ctypes.c_longlong * 1)(2)
        plan = ctypes.c_void_p()
        with pytest.raises(ValueError):
            _lib.call("sr_cart_plan_create", pts.ctypes.data, counts, 1, 2, cdims, 0, ctypes.byref(plan), dv.stream())
        nplan = ctypes.c_void_p()
        with pytest.raises(ValueError):
            _lib.call("sr_nufft_plan_create", pts.ctypes.data, 2, 2, cdims, 2.0, 4, 0, ctypes.byref(nplan),
                      dv.stream())
    # the edge values themselves are accepted
    pts = np.array([[-16.0, -20.0], [15.0, 19.0]], dtype=np.float64)
    counts = (ctypes.c_longlong * 1)(2)
    plan = ctypes.c_void_p()
    _lib.call("sr_cart_plan_create", pts.ctypes.data, counts, 1, 2, cdims, 0, ctypes.byref(plan), dv.stream())
    _lib.call("sr_cart_plan_destroy", plan)
    nplan = ctypes.c_void_p()
    _lib.call("sr_nufft_plan_create", pts.ctypes.data, 2, 2, cdims, 2.0, 4, 0, ctypes.byref(nplan), dv.stream())
    _lib.call("sr_nufft_plan_destroy", nplan)

