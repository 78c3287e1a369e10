"""Pin the CPU oracle against golden vectors produced by the real reference.

tests/golden/*.npz come from tests/golden/make_golden.py, which imports
/root/reference/pkg/src/sketchrecon and runs it on seeded inputs.
"""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import sketch_oracle as O

TOL = 1e-10


def test_rng_and_sketch_draws():
    g = golden("rng")
    assert [O.child_seed(0, t) for t in range(1, 6)] == list(g["child_seeds"])
    # SURVEY 8c survey-time values
    assert list(g["child_seeds"][:3]) == [3964924996, 3141116543, 2613022947]
    m = O.gen_sketch_matrix(12, 6, 6, 32, int(g["child_seeds"][0]))
    np.testing.assert_array_equal(m, g["sketch_12_6_6_c32"])
    np.testing.assert_array_equal(m[6, 6:16], [-1, 1, 1, -1, -1, -1, 1, -1, -1, 1])
    np.testing.assert_array_equal(O.gen_sketch_matrix(4, 2, 2, 9, 7, "gaussian"), g["sketch_gauss"])
    gs = O.seed_stream(0, 0)
    v0 = gs.standard_normal(50) + 1j * gs.standard_normal(50)
    np.testing.assert_array_equal(v0, g["power_v0"])


def test_centered_fft_kats():
    g = golden("fft")
    d8 = np.zeros((8, 8), complex)
    d8[4, 4] = 1
    assert rel(O.centered_dft(d8, 2).ravel(), g["delta8"]) < TOL
    np.testing.assert_allclose(g["delta8"], 1 / 8)
    assert rel(O.centered_dft(np.ones((8, 8), complex), 2).ravel(), g["ones8"]) < TOL
    assert rel(O.centered_dft(g["x"], 2).ravel(), g["fx"]) < TOL
    assert rel(O.centered_dft(g["x"], 2, inverse=True).ravel(), g["ifx"]) < TOL


@pytest.mark.parametrize("name", ["sense_cart", "sense_cart_b", "sense_cart_1d"])
def test_cartesian_sense(name):
    g = golden(name)
    dims = tuple(g["dims"])
    k = O.CartesianKernel(dims, g["points"])
    a = O.Sense(g["maps"], k)
    assert rel(a.forward(g["x"]), g["Ax"]) < TOL
    assert rel(a.adjoint(g["y"]), g["AHy"]) < TOL
    assert rel(a.normal(g["x"]), g["AHAx"]) < TOL
    smaps = g["S"] @ g["maps"]
    assert rel(smaps, g["smaps"]) < TOL
    a_s = O.Sense(smaps, k)
    assert rel(a_s.normal(g["x"]), g["AsHAsx"]) < TOL
    lam = O.power_max_eig(a_s.normal, int(np.prod(dims)))
    assert abs(lam - float(g["lam_max"])) < 1e-10 * abs(float(g["lam_max"]))


@pytest.mark.parametrize("name", ["wavelet_32x32", "wavelet_40x16", "wavelet_20x24", "wavelet_3d", "wavelet_1d"])
def test_wavelet(name):
    g = golden(name)
    dims = tuple(g["dims"])
    assert O.wavelet_levels(dims) == int(g["levels"])
    assert rel(O.wavelet_forward(g["x"], dims), g["fwd"]) < TOL
    assert rel(O.wavelet_adjoint(g["x"], dims), g["adj"]) < TOL
    assert rel(O.wavelet_prox(g["x"], dims, 0.7, 0.3), g["prox"]) < TOL
    assert abs(O.wavelet_l1(g["x"], dims, 0.3) - float(g["value"])) < 1e-10 * float(g["value"])
    # unitary round trip (SPEC 68-70)
    assert rel(O.wavelet_adjoint(O.wavelet_forward(g["x"], dims), dims), g["x"]) < 1e-12


@pytest.mark.parametrize("name", ["nufft_2x_w4", "nufft_125_w4", "nufft_125_w6", "nufft3d"])
def test_gridded_nufft(name):
    g = golden(name)
    dims = tuple(g["dims"])
    k = O.GriddedKernel(dims, g["points"], float(g["oversamp"]), int(g["width"]))
    assert rel(k.apply(g["batch"]), g["fwd"]) < TOL
    assert rel(k.apply_adjoint(g["y"]), g["adj"]) < TOL
    if "AHAx" in g:
        w = O.radial_density_weights(g["points"])
        assert rel(w, g["weights"]) < 1e-14
        a = O.Sense(g["maps"], k, w)
        assert rel(a.normal(g["x"]), g["AHAx"]) < TOL


def test_coil_compression():
    g = golden("compress")
    d, m, comp, en = O.coil_compress_svd(g["data"], g["maps"], 4)
    assert rel(comp, g["comp"]) < TOL
    assert rel(d, g["cdata"]) < TOL and rel(m, g["cmaps"]) < TOL
    assert abs(en - float(g["energy"])) < 1e-12


def _kernel_for(g):
    dims = tuple(g["dims"])
    if float(g["oversamp"]) > 0:
        return lambda: O.GriddedKernel(dims, g["points"], float(g["oversamp"]), int(g["width"]))
    return lambda: O.CartesianKernel(dims, g["points"])


@pytest.mark.parametrize("name,solver,reg", [("recon_cart", "fista", "l1-wavelet"),
                                             ("recon_cart_pm1", "fista", "l1-wavelet"),
                                             ("recon_cart_cg", "cg", "l2"),
                                             ("recon_cart_tv", "pdhg", "l1-tv"),
                                             ("recon_radial", "fista", "l1-wavelet"),
                                             ("recon_cones3d", "fista", "l1-wavelet")])
def test_recon_end_to_end(name, solver, reg):
    g = golden(name)
    dims = tuple(g["dims"])
    w = g["weights"] if g["weights"].size else None
    res = O.coil_sketching_recon(g["data"], g["maps"], dims, _kernel_for(g), c_hat0=int(g["chat0"]),
                                 v=int(g["v"]), s=int(g["s"]), lam=float(g["lam"]), outer=int(g["outer"]),
                                 inner=int(g["inner"]), seed=0, weights=w,
                                 rademacher_scale=float(g["scale"]), solver=solver, reg=reg)
    assert rel(res.x_final, g["x_final"]) < 1e-9
    np.testing.assert_allclose(res.objectives, g["objectives"], rtol=1e-9)
    assert res.counts["coil_transform"] == int(g["counts"]) == int(g["expected"])
    assert res.diverged == bool(g["diverged"])


def test_tv_operators():
    g = golden("tv_ops")
    dims = tuple(int(n) for n in g["dims"])
    assert rel(O.finite_diff_forward(g["x"], dims), g["fwd"]) < 1e-13
    assert rel(O.finite_diff_adjoint(g["y"], dims), g["adj"]) < 1e-13
    assert rel(O.clamp_magnitude(g["y"], 0.8), g["clamp"]) < 1e-14
    assert abs(O.tv_norm_value(g["x"], dims, 0.3) - float(g["value"])) < 1e-12 * float(g["value"])


def _solver_case(name):
    g = golden(name)
    dims = tuple(int(v) for v in g["dims"])
    a = O.Sense(g["maps"], O.CartesianKernel(dims, g["points"]))
    return g, dims, a


def test_full_operator_pdhg_tv():
    """reconstruct(l1-tv) -> PDHG with the inner-CG data prox (solvers.py:315-362, 470-500)."""
    g, dims, a = _solver_case("solve_pdhg_tv")
    x, it = O.pdhg_reconstruct_tv(a, g["y"], dims, float(g["lam"]), int(g["iters"]), int(g["cg_iters"]))
    assert it == int(g["iterations"])
    assert rel(x, g["x"]) < TOL
    assert a.counter.counts["coil_transform"] == int(g["counts"])


def test_accproxsgd():
    """Accelerated proximal SGD over coil batches (solvers.py:369-427)."""
    g, dims, a = _solver_case("solve_accproxsgd")
    lam = float(g["lam"])
    x, it = O.accproxsgd(a, g["y"], lambda v, s: O.wavelet_prox(v, dims, s, lam), int(g["batch"]),
                         float(g["alpha0"]), float(g["beta"]), float(g["beta_min"]),
                         np.zeros(int(np.prod(dims)), complex), int(g["iters"]), seed=int(g["seed"]))
    assert it == int(g["iterations"])
    assert rel(x, g["x"]) < TOL
    assert a.counter.counts["coil_transform"] == int(g["counts"])


def test_chunked_gridded_kernel_equals_gridded_kernel():
    """The bounded-memory oracle kernel (per-chunk tap tables, used to time the CPU path at
    config-4 size) computes exactly what the whole-table oracle does (pinned to the fixtures)."""
    g = golden("nufft3d")
    dims = tuple(int(v) for v in g["dims"])
    k = O.ChunkedGriddedKernel(dims, g["points"], float(g["oversamp"]), int(g["width"]), chunk=7)
    assert rel(k.apply(g["batch"]), g["fwd"]) < TOL
    assert rel(k.apply_adjoint(g["y"]), g["adj"]) < TOL


def test_cartesian_sense_3d():
    """3-D Cartesian mask SENSE (linops.py:332-364 on a 3-D grid), duplicated bins."""
    g = golden("sense_cart3d")
    dims = tuple(int(n) for n in g["dims"])
    k = O.CartesianKernel(dims, g["points"])
    a = O.Sense(g["maps"], k)
    assert rel(a.forward(g["x"]), g["Ax"]) < TOL
    assert rel(a.adjoint(g["y"]), g["AHy"]) < TOL
    assert rel(a.normal(g["x"]), g["AHAx"]) < TOL
    assert rel(O.Sense(g["S"] @ g["maps"], k).normal(g["x"]), g["AsHAsx"]) < TOL


@pytest.mark.parametrize("name", ["recon_cart3d", "recon_cart_tol", "recon_cart_noreuse", "recon_cart_init"])
def test_recon_options(name):
    """Algorithm 1 with a 3-D mask, FISTA early stopping (tol > 0), per-outer step sizes and the
    classical-sketch initialisation (coil_sketch.py:148-159, 220-306; solvers.py:300)."""
    g = golden(name)
    dims = tuple(int(n) for n in g["dims"])
    res = O.coil_sketching_recon(g["data"], g["maps"], dims, _kernel_for(g), c_hat0=int(g["chat0"]),
                                 v=int(g["v"]), s=int(g["s"]), lam=float(g["lam"]), outer=int(g["outer"]),
                                 inner=int(g["inner"]), seed=0, rademacher_scale=float(g["scale"]),
                                 tol=float(g["tol"]), reuse_step_size=bool(g["reuse"]),
                                 use_init=bool(g["use_init"]), init_iters=int(g["max_iters"]))
    assert rel(res.x_final, g["x_final"]) < 1e-9
    np.testing.assert_allclose(res.objectives, g["objectives"], rtol=1e-9)
    assert res.counts["coil_transform"] == int(g["counts"])
    assert res.per_outer_counts == list(g["per_outer_counts"])
    assert res.init_count == int(g["init_counts"])
    if float(g["tol"]) > 0:
        assert int(g["counts"]) < int(g["expected"])  # the early stop fired


def test_full_coil_reconstruct():
    """reconstruct(): l1-wavelet -> FISTA, l2 -> CG, fixed count and tol stops (solvers.py:232-500)."""
    g = golden("solve_full")
    dims = tuple(int(n) for n in g["dims"])
    k = O.CartesianKernel(dims, g["points"])
    a = O.Sense(g["maps"], k)
    x, it, hist, cnt = O.reconstruct(a, g["y"], dims, "l1-wavelet", 1e-3, 12)
    assert rel(x, g["fista_x"]) < 1e-9 and cnt == int(g["fista_counts"])
    np.testing.assert_allclose(hist, g["fista_hist"], rtol=1e-9)
    x, it, _, _ = O.reconstruct(a, g["y"], dims, "l1-wavelet", 1e-3, 40, tol=3e-3)
    assert rel(x, g["fista_tol_x"]) < 1e-9 and it == int(g["fista_tol_iters"])
    x, it, hist, cnt = O.reconstruct(a, g["y"], dims, "l2", 1e-2, 10)
    assert rel(x, g["cg_x"]) < 1e-9 and cnt == int(g["cg_counts"])
    np.testing.assert_allclose(hist, g["cg_hist"], rtol=1e-9)
    x, it, _, _ = O.reconstruct(a, g["y"], dims, "l2", 1e-2, 50, tol=1e-3)
    assert rel(x, g["cg_tol_x"]) < 1e-9 and it == int(g["cg_tol_iters"])


def test_gfactor_montecarlo():
    """Pseudo-replica inverse g-factor with a CG-l2 recon (metrics.py:157-211)."""
    g = golden("gfactor")
    dims = tuple(int(n) for n in g["dims"])
    a_full = O.Sense(g["maps"], O.CartesianKernel(dims, g["full_points"]))
    a_under = O.Sense(g["maps"], O.CartesianKernel(dims, g["under_points"]))
    lam, iters = float(g["lam"]), int(g["iters"])

    def recon(op, y):
        return O.reconstruct(op, y, dims, "l2", lam, iters)[0]

    inv, mask = O.gfactor_montecarlo(recon, a_full, a_under, g["truth"], float(g["sigma"]), int(g["trials"]),
                                     float(g["R"]), int(g["seed"]))
    np.testing.assert_array_equal(mask, g["mask"])
    assert rel(inv, g["inverse_g"]) < 1e-9
