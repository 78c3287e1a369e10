"""GPU parity: the sm_100a path (through the C ABI) against the oracle and the
reference's golden vectors.  Bars (BASELINE.json north_star): per-operator
relative L2 <= 1e-4, final-image NRMSE <= 1e-3; integer/index work exact.
"""

import numpy as np
import pytest
import torch

from conftest import golden, rel
from oracle import sketch_oracle as O

pytestmark = pytest.mark.gpu

OP_TOL = 1e-4      # per-operator relative L2 (north_star)
IMG_TOL = 1e-3     # final-image NRMSE (north_star)


def _api():
    from paper_2305_06482_b200 import coil_sketch, forward_model, linops, sketching, solvers
    return coil_sketch, forward_model, linops, sketching, solvers


@pytest.mark.parametrize("name", ["sense_cart", "sense_cart_b", "sense_cart_1d"])
def test_sense_operator_matches_reference(cuda, name):
    cs, fm, lo, sk, so = _api()
    g = golden(name)
    shape = lo.GridShape(tuple(g["dims"]))
    traj = lo.Trajectory(g["points"], "cartesian-mask")
    a = fm.build_sense(fm.SensitivityMaps(shape, g["maps"]), traj)
    assert rel(a.forward(g["x"]), g["Ax"]) < OP_TOL
    assert rel(a.adjoint(g["y"]), g["AHy"]) < OP_TOL
    assert rel(a.adjoint(a.forward(g["x"])), g["AHAx"]) < OP_TOL
    S = sk.SketchMatrix(g["S"], sk.SketchConfig(3, 2, 1))
    a_s = sk.build_sketched_operator(a, S)
    assert rel(a_s.adjoint(a_s.forward(g["x"])), g["AsHAsx"]) < OP_TOL
    # fused normal entry point
    x = torch.from_numpy(g["x"].astype(np.complex64)).cuda().view(1, -1)
    out = torch.empty_like(x)
    a_s.normal_into(x, out)
    assert rel(out.cpu().numpy().ravel(), g["AsHAsx"]) < OP_TOL
    # V identity rows of the sketch are bit-exact copies of the (fp32) maps
    np.testing.assert_array_equal(a_s.maps_dev[0, :2].cpu().numpy(), g["maps"][:2].astype(np.complex64))
    lam = so.normal_max_eig(a_s)
    assert abs(lam - float(g["lam_max"])) <= 1e-5 * float(g["lam_max"])
    # counters: forward + adjoint + adjoint(forward) on the full op = 4C; sketched pair + fused normal
    # = 2*3 + 2*3; the power iteration is paused (linops.py:774)
    assert a.counts["coil_transform"] == 4 * a.n_coils + 12


def test_kernel_plugin_protocol(cuda):
    """The device kernel honours the reference plugin protocol (apply / apply_adjoint)."""
    from paper_2305_06482_b200.cartesian import CartesianKernel
    g = golden("sense_cart")
    dims = tuple(g["dims"])
    kern = CartesianKernel.from_points(dims, g["points"])
    ok = O.CartesianKernel(dims, g["points"])
    rng = np.random.default_rng(0)
    b = rng.standard_normal((4, int(np.prod(dims)))) + 1j * rng.standard_normal((4, int(np.prod(dims))))
    yb = rng.standard_normal((4, ok.n_points)) + 1j * rng.standard_normal((4, ok.n_points))
    assert kern.n_points == ok.n_points
    assert rel(kern.apply(b), ok.apply(b)) < OP_TOL
    assert rel(kern.apply_adjoint(yb), ok.apply_adjoint(yb)) < OP_TOL
    # and plugged into the oracle's SENSE operator (the reference's seam, FM:134)
    a = O.Sense(g["maps"], kern)
    assert rel(a.normal(g["x"]), g["AHAx"]) < OP_TOL


@pytest.mark.parametrize("name", ["wavelet_32x32", "wavelet_40x16", "wavelet_20x24", "wavelet_3d", "wavelet_1d"])
def test_wavelet_and_prox(cuda, name):
    cs, fm, lo, sk, so = _api()
    g = golden(name)
    shape = lo.GridShape(tuple(g["dims"]))
    w = lo.WaveletOp(shape)
    assert w.levels == int(g["levels"])
    assert rel(w.forward(g["x"]), g["fwd"]) < OP_TOL
    assert rel(w.adjoint(g["x"]), g["adj"]) < OP_TOL
    reg = so.make_regularizer("l1-wavelet", 0.3, shape)
    assert rel(reg.prox(g["x"], 0.7), g["prox"]) < OP_TOL
    assert abs(reg.value(g["x"]) - float(g["value"])) < 1e-5 * float(g["value"])


@pytest.mark.parametrize("dims", [(320, 320), (256, 256), (256, 160), (64, 64), (64, 40), (200, 80), (240, 180),
                                  (90, 150), (36, 30)])
def test_batched_normal_op_vs_oracle(cuda, dims):
    """K1 at BASELINE geometries (a few slices, per-slice masks and maps)."""
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.plan import cartesian_plan
    rng = np.random.default_rng(7)
    B, C = 3, 5
    D = dims[0] * dims[1]
    plans, pts_all = [], []
    for b in range(B):
        m = rng.random(dims) < 0.2
        pts = np.argwhere(m) - np.array([n // 2 for n in dims])
        pts_all.append(pts)
        plans.append(cartesian_plan(dims, pts))
    kern = CartesianKernel(dims, plans)
    maps = (rng.standard_normal((B, C, D)) + 1j * rng.standard_normal((B, C, D))) / 3
    x = rng.standard_normal((B, D)) + 1j * rng.standard_normal((B, D))
    md = torch.from_numpy(maps.astype(np.complex64)).cuda()
    xd = torch.from_numpy(x.astype(np.complex64)).cuda()
    out = torch.empty_like(xd)
    kern.normal(md, xd, out)
    got = out.cpu().numpy()
    refs = [O.Sense(maps[b], O.CartesianKernel(dims, pts_all[b])).normal(x[b]) for b in range(B)]
    for b in range(B):
        assert rel(got[b], refs[b]) < OP_TOL, b
    # the chunked three-pass schedule of the same operator
    for ch in (2,):
        out2 = torch.full_like(xd, float("nan"))
        kern.normal(md, xd, out2, chunk=ch)
        got2 = out2.cpu().numpy()
        for b in range(B):
            assert rel(got2[b], refs[b]) < OP_TOL, (ch, b)
    # forward / adjoint with ragged per-slice samples
    y = kern.forward(md, xd)
    for b in range(B):
        a = O.Sense(maps[b], O.CartesianKernel(dims, pts_all[b]))
        n = len(pts_all[b])
        assert rel(y[b, :, :n].cpu().numpy().ravel(), a.forward(x[b])) < OP_TOL
    adj = torch.empty_like(xd)
    kern.adjoint(md, y, adj)
    for b in range(B):
        a = O.Sense(maps[b], O.CartesianKernel(dims, pts_all[b]))
        n = len(pts_all[b])
        assert rel(adj[b].cpu().numpy(), a.adjoint(y[b, :, :n].cpu().numpy().astype(np.complex128).ravel())) < OP_TOL


def test_fused_fista_epilogue(cuda):
    """out = z - step (N(z - a) + d) in one K1 call (coil_sketch.py:196-197, solvers.py:291)."""
    from paper_2305_06482_b200.cartesian import CartesianKernel
    g = golden("sense_cart_b")
    dims = tuple(g["dims"])
    kern = CartesianKernel.from_points(dims, g["points"])
    rng = np.random.default_rng(3)
    D = int(np.prod(dims))
    z, a, d = (rng.standard_normal(D) + 1j * rng.standard_normal(D) for _ in range(3))
    step = 0.37
    ref = z - step * (O.Sense(g["maps"], O.CartesianKernel(dims, g["points"])).normal(z - a) + d)
    t = lambda v: torch.from_numpy(v.astype(np.complex64)).cuda().view(1, -1)  # noqa: E731
    coef = torch.tensor([[-step, 1.0, -step, 0.0]], dtype=torch.float32, device="cuda")
    zt = t(z)
    out = torch.empty_like(zt)
    kern.normal(torch.from_numpy(g["maps"].astype(np.complex64)).cuda().unsqueeze(0), zt, out,
                anchor=t(a), coef=coef, u=zt, d=t(d))
    assert rel(out.cpu().numpy().ravel(), ref) < OP_TOL


def test_reductions_are_deterministic(cuda):
    from paper_2305_06482_b200.solvers import dev_norm2, dev_vdot
    rng = np.random.default_rng(5)
    a = torch.from_numpy((rng.standard_normal((4, 100003)) + 1j * rng.standard_normal((4, 100003))).astype(np.complex64)).cuda()
    b = torch.roll(a, 1, dims=1).contiguous()
    r1, r2 = dev_norm2(a).cpu().numpy(), dev_norm2(a).cpu().numpy()
    np.testing.assert_array_equal(r1, r2)
    np.testing.assert_array_equal(dev_vdot(a, b).cpu().numpy(), dev_vdot(a, b).cpu().numpy())
    an = a.cpu().numpy().astype(np.complex128)
    np.testing.assert_allclose(r1, np.sum(np.abs(an) ** 2, axis=1), rtol=1e-12)


def _recon_inputs(g):
    cs, fm, lo, sk, so = _api()
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    nufft = float(g["oversamp"]) > 0
    traj = lo.Trajectory(g["points"], "non-cartesian" if nufft else "cartesian-mask")
    return cs, fm, lo, sk, so, dims, shape, traj, nufft


@pytest.mark.parametrize("name,solver,kind", [("recon_cart", "fista", "l1-wavelet"),
                                              ("recon_cart_pm1", "fista", "l1-wavelet"),
                                              ("recon_cart_cg", "cg", "l2"),
                                              ("recon_cart_tv", "pdhg", "l1-tv")])
def test_coil_sketching_recon_matches_reference(cuda, name, solver, kind):
    g = golden(name)
    cs, fm, lo, sk, so, dims, shape, traj, nufft = _recon_inputs(g)
    reg = so.make_regularizer(kind, float(g["lam"]), shape)
    v, s = int(g["v"]), int(g["s"])
    cfg = cs.CoilSketchConfig(int(g["chat0"]), sk.SketchConfig(v + s, v, s, "rademacher", 0,
                                                               rademacher_scale=float(g["scale"])),
                              reg, int(g["outer"]), int(g["inner"]), solver=solver)
    rep = cs.coil_sketching_recon(fm.KSpaceData(traj, g["data"]), fm.SensitivityMaps(shape, g["maps"]), cfg)
    x = rep.x_final.values
    ref = g["x_final"]
    nrmse = np.linalg.norm(np.abs(x) - np.abs(ref)) / np.linalg.norm(ref)
    assert nrmse <= IMG_TOL
    assert rel(x, ref) <= IMG_TOL
    np.testing.assert_allclose([r.objective for r in rep.per_outer], g["objectives"], rtol=1e-4)
    assert rep.counts["coil_transform"] == int(g["counts"]) == int(g["expected"])
    assert rep.diverged == bool(g["diverged"])


def test_tv_operators_match_reference(cuda):
    """Finite differences, their adjoint, the dual clamp, the TV value and the TV prox on the
    device against the reference's (linops.py:717-741, solvers.py:61-69,138-164)."""
    cs, fm, lo, sk, so = _api()
    from paper_2305_06482_b200 import _lib
    g = golden("tv_ops")
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v).astype(np.complex64)).cuda()  # noqa: E731
    fd = lo.FiniteDiffOp(shape)
    assert rel(fd.forward(g["x"]), g["fwd"]) < OP_TOL
    assert rel(fd.adjoint(g["y"]), g["adj"]) < OP_TOL
    p = t(g["y"])
    z = torch.zeros(shape.size, dtype=torch.complex64, device="cuda")
    sig = torch.ones(1, dtype=torch.float32, device="cuda")
    import ctypes
    _lib.call("sr_tv_dual", p.data_ptr(), z.data_ptr(), (ctypes.c_int * 2)(*dims), 2, 0, sig.data_ptr(), 0.8, 1, 0)
    torch.cuda.synchronize()
    assert rel(p.cpu().numpy(), g["clamp"]) < OP_TOL
    reg = so.make_regularizer("l1-tv", 0.3, shape)
    assert abs(reg.value(g["x"]) - float(g["value"])) < 1e-4 * float(g["value"])
    ref_prox = O.finite_diff_forward  # the oracle's TV prox below restates solvers.py:152-164
    v = g["x"]
    x, z_, pp = v.copy(), v.copy(), np.zeros(2 * v.size, complex)
    sg = tau = 1.0 / (2.0 * np.sqrt(2.0))
    for _ in range(10):
        pp = O.clamp_magnitude(pp + sg * ref_prox(z_, dims), 0.7 * 0.3)
        xn = (x - tau * O.finite_diff_adjoint(pp, dims) + tau * v) / (1.0 + tau)
        z_, x = 2.0 * xn - x, xn
    assert rel(reg.prox(v, 0.7), x) < OP_TOL


# ----------------------------------------------------------------------------- NUFFT (K3/K4)
@pytest.mark.parametrize("name", ["nufft_2x_w4", "nufft_125_w4", "nufft_125_w6", "nufft3d"])
def test_gridded_nufft_kernel_matches_reference(cuda, name):
    from paper_2305_06482_b200.nufft import GriddedKernel
    g = golden(name)
    dims = tuple(int(n) for n in g["dims"])
    k = GriddedKernel(dims, g["points"], float(g["oversamp"]), int(g["width"]))
    assert k.n_points == len(g["points"])
    assert rel(k.apply(g["batch"]), g["fwd"]) < OP_TOL
    assert rel(k.apply_adjoint(g["y"]), g["adj"]) < OP_TOL


@pytest.mark.parametrize("name", ["nufft_2x_w4", "nufft_125_w4", "nufft_125_w6"])
def test_nufft_sense_normal_with_density_weights(cuda, name):
    cs, fm, lo, sk, so = _api()
    from paper_2305_06482_b200.nufft import GriddedKernel
    g = golden(name)
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    traj = lo.Trajectory(g["points"], "non-cartesian")
    w = fm.radial_density_weights(traj)
    assert rel(w.w, g["weights"]) < 1e-14
    kern = GriddedKernel(dims, g["points"], float(g["oversamp"]), int(g["width"]))
    a = fm.SenseOperator(fm.SensitivityMaps(shape, g["maps"]), traj, w, kernel=kern)
    assert rel(a.adjoint(a.forward(g["x"])), g["AHAx"]) < OP_TOL
    x = torch.from_numpy(g["x"].astype(np.complex64)).cuda().view(1, -1)
    out = torch.empty_like(x)
    a.normal_into(x, out)
    assert rel(out.cpu().numpy().ravel(), g["AHAx"]) < OP_TOL


def test_nufft_large_2d_vs_oracle(cuda):
    """config-3 geometry (320^2, 2x grid, w4, 128 golden-angle spokes x 640) against the oracle."""
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.nufft import GriddedKernel
    dims = (320, 320)
    pts = synth.golden_angle_radial(128, 640, dims)
    rng = np.random.default_rng(11)
    maps = synth.gaussian_coil_maps(dims, 3, rng)
    x = synth.random_ellipses(dims, 6, rng).ravel()
    w = O.radial_density_weights(pts)
    ok = O.GriddedKernel(dims, pts, 2.0, 4)
    ref = O.Sense(maps, ok, w).normal(x)
    kern = GriddedKernel(dims, pts, 2.0, 4)
    md = torch.from_numpy(maps.astype(np.complex64)).cuda().unsqueeze(0)
    xd = torch.from_numpy(x.astype(np.complex64)).cuda().view(1, -1)
    sw = torch.from_numpy(np.sqrt(w)).cuda()
    out = torch.empty_like(xd)
    kern.normal(md, xd, out, w=sw)
    assert rel(out.cpu().numpy().ravel(), ref) < OP_TOL
    y = kern.forward(md, xd, w=sw)
    assert rel(y.cpu().numpy().ravel(), O.Sense(maps, ok, w).forward(x)) < OP_TOL


def test_nufft_3d_dense_centre_runs_vs_oracle(cuda):
    """Many samples per grid cell (dense cone centre): the spread merges runs of samples that
    share a first-tap cell in registers before the shared atomics; the normal op, forward and
    adjoint must still match the oracle."""
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.nufft import GriddedKernel
    dims = (24, 24, 16)
    rng = np.random.default_rng(5)
    pts = synth.cones_3d(dims, n_readouts=400, n_samples=256)
    D = int(np.prod(dims))
    maps = (rng.standard_normal((2, D)) + 1j * rng.standard_normal((2, D))) / 3
    x = rng.standard_normal(D) + 1j * rng.standard_normal(D)
    w = O.radial_density_weights(pts)
    ok = O.GriddedKernel(dims, pts, 1.25, 4)
    kern = GriddedKernel(dims, pts, 1.25, 4)
    g = [np.ceil(pts[:, a] * (kern.gdims[a] / dims[a]) - 2.0) for a in range(3)]
    assert len(pts) / len(np.unique(np.stack(g), axis=1).T) > 4  # long runs
    md = torch.from_numpy(maps.astype(np.complex64)).cuda().unsqueeze(0)
    xd = torch.from_numpy(x.astype(np.complex64)).cuda().view(1, -1)
    sw = torch.from_numpy(np.sqrt(w)).cuda()
    out = torch.empty_like(xd)
    kern.normal(md, xd, out, w=sw)
    e_n = rel(out.cpu().numpy().ravel(), O.Sense(maps, ok, w).normal(x))
    y = kern.forward(md, xd, w=sw)
    yr = O.Sense(maps, ok, w).forward(x)
    e_f = rel(y.cpu().numpy().ravel(), yr)
    adj = torch.empty_like(xd)
    kern.adjoint(md, torch.from_numpy(yr.astype(np.complex64)).cuda().view(1, 2, -1), adj, w=sw)
    e_a = rel(adj.cpu().numpy().ravel(), O.Sense(maps, ok, w).adjoint(yr))
    print(f"dense-centre 3-D: normal {e_n:.2e} forward {e_f:.2e} adjoint {e_a:.2e}")
    assert max(e_n, e_f, e_a) < OP_TOL


def test_nufft_3d_fused_row_passes_vs_oracle(cuda):
    """3-D grid large enough (n0 n1 >= 9472 image rows) for the fused embed/row-FFT and
    row-IFFT/crop/coil-sum kernels and the pruned strided passes, with density weights and the
    FISTA epilogue, against the oracle."""
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.nufft import GriddedKernel
    dims = (96, 128, 32)
    rng = np.random.default_rng(13)
    pts = synth.cones_3d(dims, n_readouts=60, n_samples=200)
    D = int(np.prod(dims))
    maps = (rng.standard_normal((3, D)) + 1j * rng.standard_normal((3, D))) / 3
    x = rng.standard_normal(int(np.prod(dims))) + 1j * rng.standard_normal(int(np.prod(dims)))
    w = O.radial_density_weights(pts)
    ok = O.GriddedKernel(dims, pts, 1.25, 4)
    ref = O.Sense(maps, ok, w).normal(x)
    kern = GriddedKernel(dims, pts, 1.25, 4)
    assert kern.dims[0] * kern.dims[1] >= 9472
    md = torch.from_numpy(maps.astype(np.complex64)).cuda().unsqueeze(0)
    xd = torch.from_numpy(x.astype(np.complex64)).cuda().view(1, -1)
    sw = torch.from_numpy(np.sqrt(w)).cuda()
    out = torch.empty_like(xd)
    kern.normal(md, xd, out, w=sw)
    assert rel(out.cpu().numpy().ravel(), ref) < OP_TOL
    # epilogue: out = 0.5 N(x - a) + u - 0.25 d
    a, d = (rng.standard_normal(x.size) + 1j * rng.standard_normal(x.size) for _ in range(2))
    coef = torch.tensor([[0.5, 1.0, -0.25, 0.0]], dtype=torch.float32, device="cuda")
    t = lambda v: torch.from_numpy(v.astype(np.complex64)).cuda().view(1, -1)  # noqa: E731
    kern.normal(md, xd, out, anchor=t(a), coef=coef, u=xd, d=t(d), w=sw)
    ref2 = 0.5 * O.Sense(maps, ok, w).normal(x - a) + x - 0.25 * d
    assert rel(out.cpu().numpy().ravel(), ref2) < OP_TOL


@pytest.mark.parametrize("name", ["recon_radial", "recon_cones3d"])
def test_coil_sketching_recon_noncartesian_matches_reference(cuda, name):
    g = golden(name)
    cs, fm, lo, sk, so, dims, shape, traj, nufft = _recon_inputs(g)
    from paper_2305_06482_b200.nufft import GriddedKernel
    reg = so.make_regularizer("l1-wavelet", float(g["lam"]), shape)
    v, s = int(g["v"]), int(g["s"])
    cfg = cs.CoilSketchConfig(int(g["chat0"]), sk.SketchConfig(v + s, v, s, rademacher_scale=float(g["scale"])),
                              reg, int(g["outer"]), int(g["inner"]))
    kern = GriddedKernel(dims, g["points"], float(g["oversamp"]), int(g["width"]))
    rep = cs.coil_sketching_recon(fm.KSpaceData(traj, g["data"]), fm.SensitivityMaps(shape, g["maps"]), cfg,
                                  weights=fm.DensityWeights(g["weights"]), kernel=kern)
    x, ref = rep.x_final.values, g["x_final"]
    assert np.linalg.norm(np.abs(x) - np.abs(ref)) / np.linalg.norm(ref) <= IMG_TOL
    np.testing.assert_allclose([r.objective for r in rep.per_outer], g["objectives"], rtol=1e-4)
    assert rep.counts["coil_transform"] == int(g["counts"])


# ----------------------------------------------------------------------------- config 2 path
def test_readout_decoupling_matches_3d_reference_convention(cuda):
    """K8: centered IDFT along the readout of 3-D Cartesian data == per-slice 2-D SENSE data,
    with the 3-D data produced by the oracle's 3-D Cartesian operator (argwhere order, kx-major)."""
    from paper_2305_06482_b200.parallel_recon import ReadoutDecoupler
    rng = np.random.default_rng(4)
    nx, ny, nz, C = 16, 12, 10, 3
    m2 = rng.random((ny, nz)) < 0.4
    m3 = np.broadcast_to(m2, (nx, ny, nz))
    pts3 = np.argwhere(m3) - np.array([nx // 2, ny // 2, nz // 2])
    maps = (rng.standard_normal((C, nx, ny, nz)) + 1j * rng.standard_normal((C, nx, ny, nz))) / 2
    vol = rng.standard_normal((nx, ny, nz)) + 1j * rng.standard_normal((nx, ny, nz))
    k3 = O.Sense(maps.reshape(C, -1), O.CartesianKernel((nx, ny, nz), pts3)).forward(vol.ravel())
    k3 = k3.reshape(C, nx, -1)
    dec = ReadoutDecoupler(nx)
    got = dec(torch.from_numpy(k3.astype(np.complex64)).cuda()).cpu().numpy()  # (nx, C, Nyz)
    pts2 = np.argwhere(m2) - np.array([ny // 2, nz // 2])
    for x in range(nx):
        ref = O.Sense(maps[:, x].reshape(C, -1), O.CartesianKernel((ny, nz), pts2)).forward(vol[x].ravel())
        assert rel(got[x].ravel(), ref) < OP_TOL, x


def test_batched_slice_recon_matches_per_slice_oracle(cuda):
    """Config-2 style: S independent slices (own PCA compression, shared ky-kz mask) in one
    batched engine run, each against the oracle's per-slice Algorithm 1."""
    cs, fm, lo, sk, so = _api()
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.parallel_recon import compress_slices
    from paper_2305_06482_b200.plan import cartesian_plan
    rng = np.random.default_rng(9)
    S, C, dims = 3, 8, (32, 40)
    mask = synth.vd_poisson_mask(dims, 3.0, 8, 5)
    pts = synth.mask_points(mask)
    maps = np.stack([synth.gaussian_coil_maps(dims, C, rng) for _ in range(S)])
    imgs = np.stack([synth.random_ellipses(dims, 4, rng).ravel() for _ in range(S)])
    okern = O.CartesianKernel(dims, pts)
    data = np.stack([O.Sense(maps[s], okern).forward(imgs[s]).reshape(C, -1) for s in range(S)])
    data = data + synth.complex_noise(data.shape, 0.01 * np.abs(data).max(), rng)
    kern = CartesianKernel(dims, [cartesian_plan(dims, pts)], batch=S)
    comp = np.stack([np.linalg.svd(data[s], full_matrices=False)[0].conj().T for s in range(S)])
    maps0, y0, _ = compress_slices(torch.from_numpy(maps.astype(np.complex64)).cuda(),
                                   torch.from_numpy(data.astype(np.complex64)).cuda(), C, comp=comp)
    reg = so.make_regularizer("l1-wavelet", 1e-3, lo.GridShape(dims))
    cfg = cs.CoilSketchConfig(C, sk.SketchConfig(4, 2, 2, rademacher_scale=12 ** -0.5), reg, 3, 4)
    res = cs.coil_sketching_recon_batched(kern, maps0, y0, cfg, dims)
    x = res.x.cpu().numpy()
    for s in range(S):
        ref = O.coil_sketching_recon(data[s], maps[s], dims, lambda: okern, c_hat0=C, v=2, s=2, lam=1e-3,
                                     outer=3, inner=4, rademacher_scale=12 ** -0.5)
        nrmse = np.linalg.norm(np.abs(x[s]) - np.abs(ref.x_final)) / np.linalg.norm(ref.x_final)
        assert nrmse <= IMG_TOL, (s, nrmse)
        np.testing.assert_allclose(res.objectives[:, s], ref.objectives, rtol=1e-4)


def test_normal_host_pipelined_matches_device(cuda):
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.plan import cartesian_plan
    rng = np.random.default_rng(12)
    dims, B, C = (64, 40), 5, 3
    plans = [cartesian_plan(dims, np.argwhere(rng.random(dims) < 0.3) - np.array([32, 20])) for _ in range(B)]
    kern = CartesianKernel(dims, plans)
    D = dims[0] * dims[1]
    maps = torch.from_numpy((rng.standard_normal((B, C, D)) + 1j * rng.standard_normal((B, C, D))).astype(np.complex64)).cuda()
    x = torch.from_numpy((rng.standard_normal((B, D)) + 1j * rng.standard_normal((B, D))).astype(np.complex64))
    ref = torch.empty(B, D, dtype=torch.complex64, device="cuda")
    kern.normal(maps, x.cuda(), ref)
    out = torch.empty(B, D, dtype=torch.complex64).pin_memory()
    kern.normal_host(maps, x.pin_memory(), out, chunks=3)
    torch.cuda.synchronize()
    assert rel(out.numpy(), ref.cpu().numpy()) < 1e-6
    # consecutive calls overlap (the next call's copies start during the previous call's tail):
    # many back-to-back calls on distinct inputs / outputs with shared staging buffers
    stage = (torch.empty(B, D, dtype=torch.complex64, device="cuda"),
             torch.empty(B, D, dtype=torch.complex64, device="cuda"))
    xs = [torch.from_numpy((rng.standard_normal((B, D)) + 1j * rng.standard_normal((B, D))).astype(np.complex64))
          .pin_memory() for _ in range(6)]
    outs = [torch.empty(B, D, dtype=torch.complex64).pin_memory() for _ in range(6)]
    for xi, oi in zip(xs, outs):
        kern.normal_host(maps, xi, oi, chunks=3, buffers=stage, overlap_prev=True)
    torch.cuda.synchronize()
    for xi, oi in zip(xs, outs):
        r = torch.empty(B, D, dtype=torch.complex64, device="cuda")
        kern.normal(maps, xi.cuda(), r)
        assert rel(oi.numpy(), r.cpu().numpy()) < 1e-6
    # default (no overlap): work on the current stream that reads the staging input between two
    # calls sees the first call's input, not the second call's (the H2D waits for the stream)
    seen = torch.empty(B, D, dtype=torch.complex64, device="cuda")
    o1 = torch.empty(B, D, dtype=torch.complex64).pin_memory()
    kern.normal_host(maps, xs[0], o1, chunks=3, buffers=stage)
    torch.cuda._sleep(2_000_000)  # keep the stream busy so a racing H2D would land first
    seen.copy_(stage[0])
    kern.normal_host(maps, xs[1], o1, chunks=3, buffers=stage, sync=True)
    torch.cuda.synchronize()
    assert torch.equal(seen.cpu(), xs[0])


@pytest.mark.parametrize("binned", [True, False])
def test_nufft_binned_and_per_sample_paths_agree(cuda, binned):
    """Both gridding schedules (binned shared-memory tiles / per-sample atomics) vs the oracle."""
    from paper_2305_06482_b200.nufft import GriddedKernel
    for name in ("nufft_2x_w4", "nufft3d"):
        g = golden(name)
        dims = tuple(int(n) for n in g["dims"])
        k = GriddedKernel(dims, g["points"], float(g["oversamp"]), int(g["width"]), binned=binned, binsize=4)
        assert rel(k.apply(g["batch"]), g["fwd"]) < OP_TOL
        assert rel(k.apply_adjoint(g["y"]), g["adj"]) < OP_TOL


def test_slice_compression_matches_host_svd(cuda):
    """Device QR + C x C host SVD gives the reference's comp = U^H (forward_model.py:262-267)."""
    from paper_2305_06482_b200.parallel_recon import slice_compression
    rng = np.random.default_rng(21)
    S, C, N = 3, 12, 700
    y = (rng.standard_normal((S, C, N)) + 1j * rng.standard_normal((S, C, N))) * np.exp(rng.standard_normal((S, C, 1)))
    y = y.astype(np.complex64)
    comp = slice_compression(torch.from_numpy(y).cuda(), C)
    for s in range(S):
        u = np.linalg.svd(y[s].astype(np.complex128), full_matrices=False)[0]
        np.testing.assert_allclose(comp[s], u.conj().T, atol=1e-9)


def test_coil_compress_device_matches_host(cuda):
    """Device compression (QR of Y^H + C x C SVD, complex128 rotations) == host coil_compress_svd."""
    _, fm, lo, _, _ = _api()
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200 import _device as dv
    rng = np.random.default_rng(5)
    dims, C, keep = (24, 20), 10, 6
    pts = synth.mask_points(synth.vd_poisson_mask(dims, 2.5, 6, 1))
    traj = lo.Trajectory(pts, "cartesian-mask")
    data = fm.KSpaceData(traj, rng.standard_normal((C, len(pts))) + 1j * rng.standard_normal((C, len(pts))))
    maps = fm.SensitivityMaps(lo.GridShape(dims), synth.gaussian_coil_maps(dims, C, rng))
    d0, m0, comp, energy = fm.coil_compress_svd(data, maps, keep)
    m0d, d0d, comp_d, energy_d = fm.coil_compress_device(data, maps, keep)
    np.testing.assert_allclose(comp_d, comp, atol=1e-9)
    assert abs(energy - energy_d) < 1e-12
    assert rel(dv.to_numpy128(m0d), m0.coils) < 1e-6
    assert rel(dv.to_numpy128(d0d), d0.coils) < 1e-6


@pytest.mark.parametrize("reg,solver,reuse", [("l1-wavelet", "fista", True), ("l1-wavelet", "fista", False),
                                               ("l2", "fista", True), ("l2", "cg", True), ("l1-tv", "pdhg", True)])
def test_graphed_outer_loop_matches_eager(cuda, reg, solver, reuse):
    """The CUDA-graph replay of the outer iterations (t >= 2) launches the same kernels on the same
    buffers as the eager loop: iterates, objectives, Lipschitz constants and counters are bitwise
    those of the eager run (every sub-solver, and the per-outer power iteration)."""
    cs, fm, lo, sk, so = _api()
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.plan import cartesian_plan
    from paper_2305_06482_b200.recon import SketchedReconEngine
    rng = np.random.default_rng(13)
    C, dims = 8, (48, 40)
    pts = synth.mask_points(synth.vd_poisson_mask(dims, 3.0, 8, 2))
    maps = torch.from_numpy(synth.gaussian_coil_maps(dims, C, rng).astype(np.complex64)).cuda().view(1, C, -1)
    kern = CartesianKernel(dims, [cartesian_plan(dims, pts)], batch=1)
    y = torch.zeros(1, C, kern.nmax, dtype=torch.complex64, device="cuda")
    y[:, :, : len(pts)] = torch.from_numpy(
        (rng.standard_normal((C, len(pts))) + 1j * rng.standard_normal((C, len(pts)))).astype(np.complex64)).cuda()
    res = []
    for graph in (False, True):
        eng = SketchedReconEngine(kern, maps, y, dims=dims, sketch=sk.SketchConfig(4, 2, 2), lam=1e-3,
                                  reg=reg, solver=solver, use_graph=graph, cg_iters=3)
        res.append(eng.run(4, 5, reuse_step_size=reuse))
    assert torch.equal(res[0].x, res[1].x)
    np.testing.assert_array_equal(np.asarray(res[0].objectives), np.asarray(res[1].objectives))
    np.testing.assert_array_equal(res[0].lipschitz, res[1].lipschitz)
    assert res[0].counts == res[1].counts and res[0].per_outer_counts == res[1].per_outer_counts


def _plan_cases():
    from paper_2305_06482_b200 import synth
    cases = []
    for name in ("nufft_2x_w4", "nufft_125_w4", "nufft_125_w6", "nufft3d"):
        g = golden(name)
        cases.append((name, tuple(g["dims"]), g["points"], float(g["oversamp"]), int(g["width"])))
    # equatorial cone samples lie on grid lines up to 1e-16 (support-edge nudging)
    cases.append(("cones", (40, 48, 24), synth.cones_3d((40, 48, 24), n_readouts=200, n_samples=160), 1.25, 4))
    cases.append(("radial", (64, 80), synth.golden_angle_radial(40, 128, (64, 80)), 2.0, 4))
    cases.append(("grid_lines", (32, 32), np.round(np.random.default_rng(2).uniform(-16, 16, (4000, 2)) * 2) / 2
                  * (2 * np.pi / 32), 2.0, 4))
    return cases


def test_device_plan_equals_host_plan(cuda):
    """The device plan (csrc/nufft_plan.cu: fp64 tap geometry, support-edge alignment, sort key,
    gather, chunk list) is bit-identical to the NumPy plan, and both give the same operator."""
    from paper_2305_06482_b200.nufft import GriddedKernel
    for name, dims, pts, os_, w in _plan_cases():
        for bs in (None, 4):
            kd = GriddedKernel(dims, pts, os_, w, binsize=bs, plan="device")
            kh = GriddedKernel(dims, pts, os_, w, binsize=bs, plan="host")
            for f in ("base", "frac", "orig", "chunks"):
                a, b = getattr(kd, f), getattr(kh, f)
                assert a.shape == b.shape and a.dtype == b.dtype, (name, f)
                assert torch.equal(a, b), (name, bs, f)
            assert kd.nchunks == kh.nchunks


def test_device_plan_empty_trajectory(cuda):
    from paper_2305_06482_b200.nufft import GriddedKernel
    k = GriddedKernel((16, 16), np.zeros((0, 2)), 2.0, 4, plan="device")
    assert k.n_points == 0 and k.nchunks == 0
    with pytest.raises(ValueError):
        GriddedKernel((16, 16), np.zeros((5, 2)), 2.0, 4, plan="gpu")


def _solver_inputs(name):
    cs, fm, lo, sk, so = _api()
    g = golden(name)
    dims = tuple(int(v) for v in g["dims"])
    shape = lo.GridShape(dims)
    a = fm.build_sense(fm.SensitivityMaps(shape, g["maps"]), lo.Trajectory(g["points"], "cartesian-mask"))
    return g, so, lo, shape, a


def test_full_operator_pdhg_tv_matches_reference(cuda):
    """reconstruct(l1-tv) -> device PDHG (fused dual/primal TV kernels, inner CG on the fused
    normal operator) against the reference's result on the same inputs; counters exact."""
    g, so, lo, shape, a = _solver_inputs("solve_pdhg_tv")
    cfg = so.SolverConfig(max_iters=int(g["iters"]), tol=0.0, inner_cg_iters=int(g["cg_iters"]))
    res = so.reconstruct(a, g["y"], so.make_regularizer("l1-tv", float(g["lam"]), shape), cfg)
    x = res.x.values.cpu().numpy() if isinstance(res.x.values, torch.Tensor) else res.x.values
    assert res.iterations_run == int(g["iterations"])
    assert res.coil_transform_count == int(g["counts"])
    assert rel(x, g["x"]) < IMG_TOL


def test_accproxsgd_matches_reference(cuda):
    """AccProxSGD over coil batches: the reference's coil draws, device sub-operators, wavelet prox."""
    g, so, lo, shape, a = _solver_inputs("solve_accproxsgd")
    x0 = lo.Image(shape, np.zeros(shape.size, dtype=np.complex128))
    res = so.accproxsgd(a, g["y"], so.make_regularizer("l1-wavelet", float(g["lam"]), shape), int(g["batch"]),
                        float(g["alpha0"]), float(g["beta"]), float(g["beta_min"]), x0,
                        so.SolverConfig(max_iters=int(g["iters"]), tol=0.0), seed=int(g["seed"]))
    x = res.x.values.cpu().numpy() if isinstance(res.x.values, torch.Tensor) else res.x.values
    assert res.iterations_run == int(g["iterations"])
    assert res.coil_transform_count == int(g["counts"])
    assert rel(x, g["x"]) < IMG_TOL
    with pytest.raises(ValueError):
        so.accproxsgd(a, g["y"], so.make_regularizer("l1-wavelet", 1e-3, shape), 0, 1.0, 0.9, 0.1, x0,
                      so.SolverConfig(max_iters=1))


def test_opaque_c_plan_equals_python_plan(cuda):
    """sr_nufft_plan_create (the C-ABI plan a non-Python caller uses: grid, betas, apodisation,
    tap geometry, CUB radix sort, chunk list -- all in the library) equals GriddedKernel's plan
    array for array, and sr_nufft_plan_normal equals GriddedKernel.normal bit for bit."""
    import ctypes
    from paper_2305_06482_b200 import _device as dv
    from paper_2305_06482_b200 import _lib, synth
    from paper_2305_06482_b200.nufft import GriddedKernel
    lib = _lib.lib()
    cases = [((40, 48, 24), synth.cones_3d((40, 48, 24), n_readouts=200, n_samples=160), 1.25, 4),
             ((64, 80), synth.golden_angle_radial(40, 128, (64, 80)), 2.0, 4)]
    g = golden("nufft_125_w6")
    cases.append((tuple(int(v) for v in g["dims"]), g["points"], 1.25, 6))
    for dims, pts, os_, w in cases:
        kern = GriddedKernel(dims, pts, os_, w)
        nd = len(dims)
        pts64 = np.ascontiguousarray(pts, dtype=np.float64)
        plan = ctypes.c_void_p()
        _lib.call("sr_nufft_plan_create", pts64.ctypes.data, len(pts64), nd, (ctypes.c_int * nd)(*dims), os_, w, 0,
                  ctypes.byref(plan), dv.stream())
        try:
            d3, g3, b3 = (ctypes.c_int * 3)(), (ctypes.c_int * 3)(), (ctypes.c_float * 3)()
            n, nch = ctypes.c_longlong(), ctypes.c_longlong()
            ptrs = [ctypes.c_void_p() for _ in range(7)]
            _lib.call("sr_nufft_plan_info", plan, d3, g3, b3, ctypes.byref(n), ctypes.byref(nch),
                      *[ctypes.byref(p) for p in ptrs])
            assert list(d3) == kern.dims3.tolist() and list(g3) == kern.gdims3.tolist()
            assert np.array_equal(np.array(list(b3), dtype=np.float32), kern.betas3.numpy())
            assert n.value == kern.n_points and nch.value == kern.nchunks

            def fetch(ptr, like):
                t = torch.empty_like(like)
                _lib.call("sr_memcpy_d2d", t.data_ptr(), ptr, t.numel() * t.element_size(), dv.stream())
                return t
            for ptr, ref in zip(ptrs[:4], (kern.base, kern.frac, kern.orig, kern.chunks)):
                assert torch.equal(fetch(ptr.value, ref), ref)
            for ptr, ref in zip(ptrs[4:], kern.ia):
                assert torch.equal(fetch(ptr.value, ref), ref)
            rng = np.random.default_rng(7)
            D = kern.D
            maps = torch.from_numpy((rng.standard_normal((2, D)) + 1j * rng.standard_normal((2, D))).astype(
                np.complex64)).cuda().unsqueeze(0)
            x = torch.from_numpy((rng.standard_normal(D) + 1j * rng.standard_normal(D)).astype(np.complex64)).cuda()
            x = x.view(1, -1)
            o1, o2 = torch.empty_like(x), torch.empty_like(x)
            kern.normal(maps, x, o1)
            grids = torch.empty(2 * 2 * kern.G, dtype=torch.complex64, device="cuda")
            _lib.call("sr_nufft_plan_normal", plan, x.data_ptr(), None, maps.data_ptr(), 2, None, o2.data_ptr(),
                      grids.data_ptr(), None, None, None, dv.stream())
            assert rel(o2.cpu().numpy(), o1.cpu().numpy()) < 1e-6
        finally:
            _lib.call("sr_nufft_plan_destroy", plan)


def test_opaque_cartesian_plan_equals_python_plan(cuda):
    """sr_cart_plan_create (the library-built Cartesian tables of the C ABI) equals CartesianKernel's
    tables array for array, and the plan's normal / forward / adjoint equal the kernel methods."""
    import ctypes
    from paper_2305_06482_b200 import _device as dv
    from paper_2305_06482_b200 import _lib
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.plan import cartesian_plan
    rng = np.random.default_rng(31)
    cases = []
    for dims, B, shared in (((320, 320), 3, False), ((256, 160), 4, True), ((60,), 2, False), ((64, 40), 1, False)):
        half = np.array([n // 2 for n in dims])
        pl = []
        for b in range(1 if shared else B):
            pts = np.argwhere(rng.random(dims) < 0.2 + 0.1 * b) - half
            pts = np.concatenate([pts, pts[: max(1, len(pts) // 9)]]).astype(np.float64)  # duplicates
            pl.append(pts)
        cases.append((dims, B, shared, pl))
    for dims, B, shared, pl in cases:
        kern = CartesianKernel(dims, [cartesian_plan(dims, p) for p in pl], batch=B)
        allp = np.ascontiguousarray(np.concatenate(pl), dtype=np.float64)
        counts = (ctypes.c_longlong * len(pl))(*[len(p) for p in pl])
        plan = ctypes.c_void_p()
        _lib.call("sr_cart_plan_create", allp.ctypes.data, counts, B, len(dims), (ctypes.c_int * len(dims))(*dims),
                  1 if shared else 0, ctypes.byref(plan), dv.stream())
        try:
            ny, nx, nblk = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
            nmax, tot, wtot = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_longlong()
            ptrs = [ctypes.c_void_p() for _ in range(10)]
            _lib.call("sr_cart_plan_info", plan, ctypes.byref(ny), ctypes.byref(nx), ctypes.byref(nmax),
                      ctypes.byref(tot), ctypes.byref(wtot), ctypes.byref(nblk), *[ctypes.byref(p) for p in ptrs])
            assert (ny.value, nx.value, nmax.value, nblk.value) == (kern.ny, kern.nx, kern.nmax, kern.nblk)

            def fetch(ptr, like):
                t = torch.empty_like(like)
                _lib.call("sr_memcpy_d2d", t.data_ptr(), ptr, t.numel() * t.element_size(), dv.stream())
                return t
            refs = (kern.spos, kern.ph, kern.soff, kern.wlist, kern.woff, kern.maskT, kern.g_ptr, kern.g_idx,
                    kern.s_ptr, kern.s_idx)
            for name, ptr, ref in zip(("spos", "ph", "soff", "wlist", "woff", "maskT", "g_ptr", "g_idx", "s_ptr",
                                       "s_idx"), ptrs, refs):
                assert torch.equal(fetch(ptr.value, ref.contiguous()), ref), (dims, name)
            C = 3
            D = kern.D
            maps = torch.from_numpy(((rng.standard_normal((B, C, D)) + 1j * rng.standard_normal((B, C, D))) / 2)
                                    .astype(np.complex64)).cuda()
            x = torch.from_numpy((rng.standard_normal((B, D)) + 1j * rng.standard_normal((B, D))).astype(np.complex64)).cuda()
            ws = torch.empty((_lib.lib().sr_cart_plan_ws_bytes(plan, C) + 7) // 8, dtype=torch.complex64, device="cuda")
            o1, o2 = torch.empty_like(x), torch.empty_like(x)
            kern.normal(maps, x, o1)
            _lib.call("sr_cart_plan_normal", plan, x.data_ptr(), None, maps.data_ptr(), C * D, C, o2.data_ptr(),
                      ws.data_ptr(), None, None, None, dv.stream())
            assert torch.equal(o1, o2)
            y1 = kern.forward(maps, x)
            y2 = torch.zeros_like(y1)
            _lib.call("sr_cart_plan_forward", plan, x.data_ptr(), maps.data_ptr(), C * D, C, y2.data_ptr(),
                      y2.shape[-1], None, None, 0, ws.data_ptr(), dv.stream())
            assert torch.equal(y1, y2)
            a1, a2 = torch.empty_like(x), torch.empty_like(x)
            kern.adjoint(maps, y1, a1)
            _lib.call("sr_cart_plan_adjoint", plan, y1.data_ptr(), y1.shape[-1], maps.data_ptr(), C * D, C,
                      a2.data_ptr(), ws.data_ptr(), None, None, None, dv.stream())
            assert torch.equal(a1, a2)
        finally:
            _lib.call("sr_cart_plan_destroy", plan)
