"""Drop-in semantics of the reference API on the device, against fixtures made by the real
reference (tests/golden/make_golden.py): 3-D Cartesian masks, FISTA/PDHG early stopping
(tol > 0), per-outer step sizes, the classical-sketch initialisation, duck-typed host
kernels, the full-coil reconstruct() pairings, the centered FFT KATs and the pseudo-replica
g-factor."""

import numpy as np
import pytest
import torch

from conftest import golden, rel
from oracle import sketch_oracle as O

pytestmark = pytest.mark.gpu

OP_TOL = 1e-4
IMG_TOL = 1e-3


def _api():
    from paper_2305_06482_b200 import coil_sketch as cs
    from paper_2305_06482_b200 import forward_model as fm
    from paper_2305_06482_b200 import linops as lo
    from paper_2305_06482_b200 import sketching as sk
    from paper_2305_06482_b200 import solvers as so
    return cs, fm, lo, sk, so


def test_centered_fft_op_kats(cuda):
    """CenteredFFTOp (linops.py:316-329) against the reference's fft fixture (SPEC 50-52 KATs)."""
    cs, fm, lo, sk, so = _api()
    g = golden("fft")
    op8 = lo.CenteredFFTOp(lo.GridShape((8, 8)))
    d8 = np.zeros((8, 8), complex)
    d8[4, 4] = 1
    assert rel(op8.forward(d8.ravel()), g["delta8"]) < OP_TOL
    assert rel(op8.forward(np.ones(64, complex)), g["ones8"]) < OP_TOL
    op = lo.CenteredFFTOp(lo.GridShape((16, 12)))
    assert rel(op.forward(g["x"].ravel()), g["fx"]) < OP_TOL
    assert rel(op.adjoint(g["x"].ravel()), g["ifx"]) < OP_TOL


def test_cartesian_3d_sense_matches_reference(cuda):
    """SenseOperator on a 3-D Cartesian mask (linops.py:332-364; duplicated bins) vs the fixture."""
    cs, fm, lo, sk, so = _api()
    g = golden("sense_cart3d")
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    traj = lo.Trajectory(g["points"], "cartesian-mask")
    a = fm.build_sense(fm.SensitivityMaps(shape, g["maps"]), traj)
    from paper_2305_06482_b200.cartesian3d import Cartesian3DKernel
    assert isinstance(a.kernel, Cartesian3DKernel)
    assert rel(a.forward(g["x"]), g["Ax"]) < OP_TOL
    assert rel(a.adjoint(g["y"]), g["AHy"]) < OP_TOL
    assert rel(a.adjoint(a.forward(g["x"])), g["AHAx"]) < OP_TOL
    xd = torch.from_numpy(g["x"].astype(np.complex64)).cuda().view(1, -1)
    out = torch.empty_like(xd)
    a.normal_into(xd, out)
    assert rel(out.cpu().numpy().ravel(), g["AHAx"]) < OP_TOL
    a_s = sk.build_sketched_operator(a, sk.SketchMatrix(g["S"], sk.SketchConfig(3, 2, 1)))
    assert rel(a_s.adjoint(a_s.forward(g["x"])), g["AsHAsx"]) < OP_TOL
    # the plugin protocol (host numpy) matches the oracle kernel
    ok = O.CartesianKernel(dims, g["points"])
    b = g["maps"] * g["x"][None, :]
    assert rel(a.kernel.apply(b), ok.apply(b)) < OP_TOL
    yy = g["y"].reshape(4, -1)
    assert rel(a.kernel.apply_adjoint(yy), ok.apply_adjoint(yy)) < OP_TOL
    # a 3-D CenteredFFTOp is the same kernel over every bin
    op = lo.CenteredFFTOp(shape)
    xg = g["x"].reshape(dims)
    assert rel(op.forward(g["x"]), O.centered_dft(xg, 3).ravel()) < OP_TOL
    assert rel(op.adjoint(g["x"]), O.centered_dft(xg, 3, inverse=True).ravel()) < OP_TOL


def _recon_cfg(g, cs, sk, so, shape, solver="fista", kind="l1-wavelet"):
    reg = so.make_regularizer(kind, float(g["lam"]), shape)
    v, s = int(g["v"]), int(g["s"])
    return cs.CoilSketchConfig(int(g["chat0"]), sk.SketchConfig(v + s, v, s, "rademacher", 0,
                                                                rademacher_scale=float(g["scale"])),
                               reg, int(g["outer"]), int(g["inner"]), solver=solver,
                               reuse_step_size=bool(g["reuse"]), use_init=bool(g["use_init"]))


@pytest.mark.parametrize("name", ["recon_cart3d", "recon_cart_tol", "recon_cart_noreuse", "recon_cart_init"])
def test_recon_options_match_reference(cuda, name):
    """coil_sketching_recon with the default device compression: 3-D mask, tol > 0 early stops
    (per-outer counters below the closed form), reuse_step_size=False, use_init=True."""
    cs, fm, lo, sk, so = _api()
    g = golden(name)
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    traj = lo.Trajectory(g["points"], "cartesian-mask")
    cfg = _recon_cfg(g, cs, sk, so, shape)
    scfg = so.SolverConfig(max_iters=int(g["max_iters"]), tol=float(g["tol"]))
    rep = cs.coil_sketching_recon(fm.KSpaceData(traj, g["data"]), fm.SensitivityMaps(shape, g["maps"]), cfg,
                                  solver_cfg=scfg)
    x, ref = rep.x_final.values, g["x_final"]
    assert np.linalg.norm(np.abs(x) - np.abs(ref)) / np.linalg.norm(ref) <= IMG_TOL
    assert rel(x, ref) <= IMG_TOL
    np.testing.assert_allclose([r.objective for r in rep.per_outer], g["objectives"], rtol=1e-4)
    assert [r.coil_transforms for r in rep.per_outer] == list(g["per_outer_counts"])
    assert rep.counts["coil_transform"] == int(g["counts"])
    assert rep.init_coil_transforms == int(g["init_counts"])


def test_duck_typed_host_kernel(cuda):
    """A host kernel object with only n_points / apply / apply_adjoint (the reference's plugin
    protocol, forward_model.py:134,147-148) is accepted by SenseOperator and by
    coil_sketching_recon, and gives the reference's results."""
    cs, fm, lo, sk, so = _api()
    g = golden("sense_cart")
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    traj = lo.Trajectory(g["points"], "cartesian-mask")
    host = O.CartesianKernel(dims, g["points"])
    a = fm.SenseOperator(fm.SensitivityMaps(shape, g["maps"]), traj, kernel=host)
    assert rel(a.forward(g["x"]), g["Ax"]) < OP_TOL
    assert rel(a.adjoint(g["y"]), g["AHy"]) < OP_TOL
    assert rel(a.adjoint(a.forward(g["x"])), g["AHAx"]) < OP_TOL
    a_s = sk.build_sketched_operator(a, sk.SketchMatrix(g["S"], sk.SketchConfig(3, 2, 1)))
    assert rel(a_s.adjoint(a_s.forward(g["x"])), g["AsHAsx"]) < OP_TOL
    gr = golden("recon_cart")
    dims = tuple(int(n) for n in gr["dims"])
    shape = lo.GridShape(dims)
    traj = lo.Trajectory(gr["points"], "cartesian-mask")
    cfg = cs.CoilSketchConfig(int(gr["chat0"]), sk.SketchConfig(int(gr["v"]) + int(gr["s"]), int(gr["v"]),
                                                                 int(gr["s"]), "rademacher", 0,
                                                                 rademacher_scale=float(gr["scale"])),
                              so.make_regularizer("l1-wavelet", float(gr["lam"]), shape), int(gr["outer"]),
                              int(gr["inner"]))
    rep = cs.coil_sketching_recon(fm.KSpaceData(traj, gr["data"]), fm.SensitivityMaps(shape, gr["maps"]), cfg,
                                  kernel=O.CartesianKernel(dims, gr["points"]))
    assert rel(rep.x_final.values, gr["x_final"]) <= IMG_TOL
    assert rep.counts["coil_transform"] == int(gr["counts"])


def test_full_coil_reconstruct_matches_reference(cuda):
    """reconstruct() l1-wavelet -> FISTA and l2 -> CG, fixed count (with the recorded history) and
    tol stops, against the reference (solvers.py:232-308, 434-500)."""
    cs, fm, lo, sk, so = _api()
    g = golden("solve_full")
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    traj = lo.Trajectory(g["points"], "cartesian-mask")
    a = fm.build_sense(fm.SensitivityMaps(shape, g["maps"]), traj)
    wav = so.make_regularizer("l1-wavelet", 1e-3, shape)
    l2 = so.make_regularizer("l2", 1e-2, shape)
    r = so.reconstruct(a, g["y"], wav, so.SolverConfig(max_iters=12, tol=0.0, record_history=True))
    assert rel(np.asarray(r.x.values), g["fista_x"]) <= IMG_TOL
    np.testing.assert_allclose(r.objective_history, g["fista_hist"], rtol=1e-4)
    assert r.coil_transform_count == int(g["fista_counts"])
    r = so.reconstruct(a, g["y"], wav, so.SolverConfig(max_iters=40, tol=3e-3))
    assert r.iterations_run == int(g["fista_tol_iters"])
    assert rel(np.asarray(r.x.values), g["fista_tol_x"]) <= IMG_TOL
    r = so.reconstruct(a, g["y"], l2, so.SolverConfig(max_iters=10, tol=0.0, record_history=True))
    assert rel(np.asarray(r.x.values), g["cg_x"]) <= IMG_TOL
    np.testing.assert_allclose(r.objective_history, g["cg_hist"], rtol=1e-4)
    assert r.coil_transform_count == int(g["cg_counts"])
    r = so.reconstruct(a, g["y"], l2, so.SolverConfig(max_iters=50, tol=1e-3))
    assert r.iterations_run == int(g["cg_tol_iters"])
    assert rel(np.asarray(r.x.values), g["cg_tol_x"]) <= IMG_TOL


def test_gfactor_montecarlo_matches_reference(cuda):
    """Pseudo-replica inverse g-factor with the device CG-l2 reconstruction (metrics.py:157-211)."""
    cs, fm, lo, sk, so = _api()
    from paper_2305_06482_b200 import metrics
    g = golden("gfactor")
    dims = tuple(int(n) for n in g["dims"])
    shape = lo.GridShape(dims)
    smaps = fm.SensitivityMaps(shape, g["maps"])
    a_full = fm.build_sense(smaps, lo.Trajectory(g["full_points"], "cartesian-mask"))
    a_under = fm.build_sense(smaps, lo.Trajectory(g["under_points"], "cartesian-mask"))
    reg = so.make_regularizer("l2", float(g["lam"]), shape)
    iters = int(g["iters"])

    def recon(op, y):
        return so.reconstruct(op, y, reg, so.SolverConfig(max_iters=iters, tol=0.0)).x

    gm = metrics.gfactor_montecarlo(recon, a_full, a_under, lo.Image(shape, g["truth"]), float(g["sigma"]),
                                    int(g["trials"]), float(g["R"]), int(g["seed"]))
    np.testing.assert_array_equal(gm.mask, g["mask"])
    assert rel(gm.inverse_g, g["inverse_g"]) < 1e-3
