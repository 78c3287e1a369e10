"""End-to-end reconstruction parity at BASELINE.json's full configuration sizes, through the
DEFAULT drop-in path (device PCA compression), against the CPU oracle on identical seeded
inputs (north_star: final-image NRMSE <= 1e-3 after the fixed iteration count; per-outer
objectives within rtol 1e-4; coil-transform counters equal to the closed form,
coil_sketch.py:318-330).

* config 0: 256^2, 16 coils -> 4 PCA + 4 Rademacher(+-1/sqrt 12), VD Poisson R=4, 10 x 10, lam 1e-3
* config 3: 320^2 golden-angle radial 128 x 640, KB 2x / w4, ramp DCF, 16 -> 4+4, 15 x 8, lam 5e-4
* config 2: a 16-slice batch of the readout-decoupled 256 x 160 slices (32 -> 6+6, R=8, 10 x 10)
  through the batched device path, each slice against its own oracle reconstruction.
"""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import sketch_oracle as O

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-3


def _nrmse(x, ref):
    return float(np.linalg.norm(np.abs(x) - np.abs(ref)) / np.linalg.norm(ref))


def _run_2d(cfgid):
    from paper_2305_06482_b200 import coil_sketch as cs
    from paper_2305_06482_b200 import forward_model as fm
    from paper_2305_06482_b200 import linops as lo
    from paper_2305_06482_b200 import sketching as sk
    from paper_2305_06482_b200 import solvers as so
    from paper_2305_06482_b200 import synth
    rng = np.random.default_rng(0)
    if cfgid == 0:
        dims, C, v, s, lam, T, K = (256, 256), 16, 4, 4, 1e-3, 10, 10
        pts = synth.mask_points(synth.vd_poisson_mask(dims, 4.0, 24, 0))
        traj = lo.Trajectory(pts, "cartesian-mask")
        weights, okern, kern = None, O.CartesianKernel(dims, pts), None
    else:
        from paper_2305_06482_b200.nufft import GriddedKernel
        dims, C, v, s, lam, T, K = (320, 320), 16, 4, 4, 5e-4, 15, 8
        pts = synth.golden_angle_radial(128, 640, dims)
        traj = lo.Trajectory(pts, "non-cartesian")
        weights = fm.radial_density_weights(traj)
        okern, kern = O.GriddedKernel(dims, pts, 2.0, 4), GriddedKernel(dims, pts, 2.0, 4)
    shape = lo.GridShape(dims)
    truth = synth.random_ellipses(dims, 10, rng).ravel()
    maps = synth.gaussian_coil_maps(dims, C, rng)
    clean = O.Sense(maps, okern).forward(truth).reshape(C, -1)
    data = clean + synth.complex_noise(clean.shape, 0.01 * np.abs(clean).max(), rng)
    reg = so.make_regularizer("l1-wavelet", lam, shape)
    cfg = cs.CoilSketchConfig(C, sk.SketchConfig(v + s, v, s, rademacher_scale=12 ** -0.5), reg, T, K)
    rep = cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg,
                                  weights=weights, kernel=kern)
    ref = O.coil_sketching_recon(data, maps, dims, lambda: okern, c_hat0=C, v=v, s=s, lam=lam, outer=T,
                                 inner=K, weights=None if weights is None else weights.w,
                                 rademacher_scale=12 ** -0.5)
    return rep, ref, cs.expected_coil_transforms(cfg, so.SolverConfig(tol=0.0))


@pytest.mark.parametrize("cfgid", [0, 3])
def test_full_config_recon_matches_oracle(cuda, cfgid):
    rep, ref, expected = _run_2d(cfgid)
    nr = _nrmse(rep.x_final.values, ref.x_final)
    print(f"config {cfgid}: NRMSE {nr:.3e}")
    assert nr <= IMG_TOL
    np.testing.assert_allclose([r.objective for r in rep.per_outer], ref.objectives, rtol=1e-4)
    assert rep.counts["coil_transform"] == ref.counts["coil_transform"] == expected
    assert rep.diverged == ref.diverged


def test_config2_slice_batch_matches_oracle(cuda):
    """16 readout-decoupled config-2 slices (256 x 160, 32 coils -> 6+6) in one batched device
    reconstruction (batched device QR compression, shared mask), each vs its oracle recon."""
    from paper_2305_06482_b200 import coil_sketch as cs
    from paper_2305_06482_b200 import linops as lo
    from paper_2305_06482_b200 import sketching as sk
    from paper_2305_06482_b200 import solvers as so
    from paper_2305_06482_b200 import synth
    from paper_2305_06482_b200.cartesian import CartesianKernel
    from paper_2305_06482_b200.parallel_recon import compress_slices
    from paper_2305_06482_b200.plan import cartesian_plan
    dev = torch.device("cuda", 0)
    NX, NY, NZ, C, V, S, B = 256, 256, 160, 32, 6, 6, 16
    dims = (NY, NZ)
    D = NY * NZ
    rng = np.random.default_rng(0)
    pts = synth.mask_points(synth.vd_poisson_mask(dims, 8.0, 20, 0))
    vol = synth.random_ellipses((NX, NY, NZ), 20, rng)
    maps3 = synth.coil_maps_cylinder((NX, NY, NZ), C, rng, xp=torch, device=dev)
    x0 = NX // 2 - B // 2  # central slab (the object's extent)
    maps = maps3.view(C, NX, D)[:, x0:x0 + B].permute(1, 0, 2).contiguous()
    del maps3
    x_true = torch.from_numpy(vol.reshape(NX, D)[x0:x0 + B].astype(np.complex64)).to(dev)
    kern = CartesianKernel(dims, [cartesian_plan(dims, pts)], batch=B)
    y = kern.forward(maps, x_true)
    gen = torch.Generator(dev).manual_seed(1234)
    y = y + torch.randn(y.shape, dtype=torch.complex64, device=dev, generator=gen) * (0.01 * float(torch.abs(y).max()))
    maps0, y0, comp = compress_slices(maps, y, C)
    reg = so.make_regularizer("l1-wavelet", 1e-3, lo.GridShape(dims))
    cfg = cs.CoilSketchConfig(C, sk.SketchConfig(V + S, V, S, rademacher_scale=12 ** -0.5), reg, 10, 10)
    res = cs.coil_sketching_recon_batched(kern, maps0, y0, cfg, dims)
    xs = res.x.cpu().numpy()
    yh = y.cpu().numpy().astype(np.complex128)
    mh = maps.cpu().numpy().astype(np.complex128)
    okern = O.CartesianKernel(dims, pts)
    worst = 0.0
    for sl in range(B):
        ref = O.coil_sketching_recon(yh[sl], mh[sl], dims, lambda: okern, c_hat0=C, v=V, s=S, lam=1e-3,
                                     outer=10, inner=10, rademacher_scale=12 ** -0.5)
        worst = max(worst, _nrmse(xs[sl], ref.x_final))
        np.testing.assert_allclose(res.objectives[:, sl], ref.objectives, rtol=1e-4)
    print(f"config 2 (16 slices): worst NRMSE {worst:.3e}")
    assert worst <= IMG_TOL
    assert res.counts["coil_transform"] == cs.expected_coil_transforms(cfg, so.SolverConfig(tol=0.0))
