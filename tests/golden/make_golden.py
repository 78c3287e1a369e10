#!/usr/bin/env python3
"""Generate golden vectors by running the REAL reference `sketchrecon`.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [fixture names ...]

(with names, only those fixtures are rewritten; all fixtures are always computed, in order,
so the shared RNG stream and therefore every fixture stays the same)

Every fixture stores the seeded inputs and the reference outputs (complex128)
in tests/golden/<name>.npz.  The oracle (oracle/sketch_oracle.py) is pinned
against these in tests/test_oracle_golden.py, and the GPU path is checked
against both.  Inputs are small so the fixtures stay a few hundred KB.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _imports():
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    import sketchrecon.coil_sketch as cs
    import sketchrecon.forward_model as fm
    import sketchrecon.linops as lo
    import sketchrecon.rng as rng
    import sketchrecon.sketching as sk
    import sketchrecon.solvers as so
    return cs, fm, lo, rng, sk, so


def crandn(g, *shape):
    return g.standard_normal(shape) + 1j * g.standard_normal(shape)


def random_mask_points(g, dims, frac, center=4):
    """Integer bins in argwhere (row-major) order of a random mask with a full centre."""
    m = g.random(dims) < frac
    sl = tuple(slice(n // 2 - center // 2, n // 2 - center // 2 + center) for n in dims)
    m[sl] = True
    return np.argwhere(m).astype(np.float64) - np.array([n // 2 for n in dims])


def smooth_maps(g, dims, ncoils):
    """Smooth random complex maps normalised to SOS = 1."""
    grids = np.meshgrid(*[np.linspace(-1, 1, n, endpoint=False) for n in dims], indexing="ij")
    maps = []
    for _ in range(ncoils):
        c = g.uniform(-1.2, 1.2, size=len(dims))
        r2 = sum((gg - cc) ** 2 for gg, cc in zip(grids, c))
        ph = g.uniform(0, 2 * np.pi) + sum(g.uniform(-2, 2) * gg for gg in grids)
        maps.append(np.exp(-r2 / 0.8) * np.exp(1j * ph))
    maps = np.array(maps).reshape(ncoils, -1)
    return maps / np.sqrt(np.sum(np.abs(maps) ** 2, axis=0, keepdims=True))


def radial_points(nspokes, nread, dims, golden=True):
    ang = np.arange(nspokes) * (np.pi * 0.6180339887498949 if golden else np.pi / nspokes)
    r = (np.arange(nread) - nread // 2) / nread  # in [-1/2, 1/2)
    kmax = np.array(dims, dtype=np.float64) / 2
    pts = np.stack([np.outer(np.cos(ang), r).ravel() * 2 * kmax[0],
                    np.outer(np.sin(ang), r).ravel() * 2 * kmax[1]], axis=1)
    return np.clip(pts, -kmax, kmax - 1e-9)


def scaled_gen(sk, scale):
    base = sk.gen_sketch_matrix

    def gen(cfg, n_coils):
        m = base(cfg, n_coils)
        mat = m.mat.copy()
        mat[cfg.v:, cfg.v:] *= scale
        return sk.SketchMatrix(mat, cfg)
    return gen


def main():
    cs, fm, lo, rng, sk, so = _imports()
    g = np.random.default_rng(20230511)
    out = {}

    # --- rng / sketch draws (rng.py, sketching.py:69-94)
    seeds = np.array([rng.child_seed(0, t) for t in range(1, 6)], dtype=np.int64)
    cfg = sk.SketchConfig(12, 6, 6, "rademacher", int(seeds[0]))
    out["rng"] = dict(child_seeds=seeds, sketch_12_6_6_c32=sk.gen_sketch_matrix(cfg, 32).mat,
                      sketch_gauss=sk.gen_sketch_matrix(sk.SketchConfig(4, 2, 2, "gaussian", 7), 9).mat,
                      power_v0=(lambda r: r.standard_normal(50) + 1j * r.standard_normal(50))(rng.seed_stream(0, 0)))

    # --- centered FFT KATs (linops.py:304-329, SPEC 50-52)
    d8 = np.zeros((8, 8), complex); d8[4, 4] = 1
    x = crandn(g, 16, 12)
    out["fft"] = dict(delta8=lo.fft_centered(lo.Image.from_grid(d8)),
                      ones8=lo.fft_centered(lo.Image.from_grid(np.ones((8, 8), complex))),
                      x=x, fx=lo.fft_centered(lo.Image.from_grid(x)),
                      ifx=lo.CenteredFFTOp(lo.GridShape((16, 12))).adjoint(x.ravel()))

    # --- Cartesian SENSE operator, full + sketched (forward_model.py:119-213, sketching.py:97-129)
    for name, dims, C, frac in [("sense_cart", (24, 20), 6, 0.35), ("sense_cart_b", (32, 40), 8, 0.25),
                                ("sense_cart_1d", (40,), 3, 0.5)]:
        shape = lo.GridShape(dims)
        pts = random_mask_points(g, dims, frac)
        if name == "sense_cart":  # duplicated bins (adjoint keeps the last write)
            pts = np.concatenate([pts, pts[:5]], axis=0)
        traj = lo.Trajectory(pts, "cartesian-mask")
        maps = smooth_maps(g, dims, C)
        a = fm.build_sense(fm.SensitivityMaps(shape, maps), traj)
        xx = crandn(g, shape.size)
        yy = crandn(g, C * traj.n_points)
        S = sk.gen_sketch_matrix(sk.SketchConfig(3, 2, 1, "rademacher", rng.child_seed(0, 1)), C)
        a_s = sk.build_sketched_operator(a, S)
        out[name] = dict(dims=np.array(dims), points=pts, maps=maps, x=xx, y=yy,
                         Ax=a.forward(xx), AHy=a.adjoint(yy), AHAx=a.adjoint(a.forward(xx)),
                         S=S.mat, smaps=a_s.maps.coils, AsHAsx=a_s.adjoint(a_s.forward(xx)),
                         lam_max=so.normal_max_eig(a_s), counts=np.array(a.counts["coil_transform"]))

    # --- wavelet + prox (linops.py:593-702, solvers.py:71-81,129-135)
    for name, dims in [("wavelet_32x32", (32, 32)), ("wavelet_40x16", (40, 16)), ("wavelet_20x24", (20, 24))]:
        shape = lo.GridShape(dims)
        w = lo.WaveletOp(shape)
        xx = crandn(g, shape.size)
        reg = so.make_regularizer("l1-wavelet", 0.3, shape)
        out[name] = dict(dims=np.array(dims), levels=np.array(w.levels), x=xx, fwd=w.forward(xx),
                         adj=w.adjoint(xx), prox=reg.prox(xx, 0.7), value=np.array(reg.value(xx)))

    # --- gridded NUFFT (linops.py:404-516)
    for name, dims, os_, wd in [("nufft_2x_w4", (16, 20), 2.0, 4), ("nufft_125_w4", (16, 16), 1.25, 4),
                                ("nufft_125_w6", (12, 16), 1.25, 6)]:
        shape = lo.GridShape(dims)
        pts = radial_points(12, 24, dims)
        traj = lo.Trajectory(pts, "non-cartesian")
        kern = lo._GriddedNUFFTKernel(shape, traj, os_, wd)
        b = crandn(g, 2, shape.size)
        yy = crandn(g, 2, traj.n_points)
        wts = fm.radial_density_weights(traj).w
        maps = smooth_maps(g, dims, 3)
        a = fm.SenseOperator(fm.SensitivityMaps(shape, maps), traj, fm.DensityWeights(wts), kernel=kern)
        xx = crandn(g, shape.size)
        out[name] = dict(dims=np.array(dims), points=pts, oversamp=np.array(os_), width=np.array(wd),
                         batch=b, y=yy, fwd=kern.apply(b), adj=kern.apply_adjoint(yy), weights=wts,
                         maps=maps, x=xx, AHAx=a.adjoint(a.forward(xx)))
    # 3-D gridded NUFFT
    dims = (8, 12, 6)
    shape = lo.GridShape(dims)
    pts = np.stack([g.uniform(-n / 2, n / 2 - 1e-6, 60) for n in dims], axis=1)
    traj = lo.Trajectory(pts, "non-cartesian")
    kern = lo._GriddedNUFFTKernel(shape, traj, 1.25, 4)
    b = crandn(g, 2, shape.size)
    yy = crandn(g, 2, traj.n_points)
    out["nufft3d"] = dict(dims=np.array(dims), points=pts, oversamp=np.array(1.25), width=np.array(4),
                          batch=b, y=yy, fwd=kern.apply(b), adj=kern.apply_adjoint(yy))

    # --- coil compression (forward_model.py:245-272)
    dims = (16, 16)
    shape = lo.GridShape(dims)
    pts = random_mask_points(g, dims, 0.4)
    traj = lo.Trajectory(pts, "cartesian-mask")
    maps = smooth_maps(g, dims, 6)
    data = crandn(g, 6, traj.n_points)
    nd, nm, comp, en = fm.coil_compress_svd(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), 4)
    out["compress"] = dict(data=data, maps=maps, cdata=nd.coils, cmaps=nm.coils, comp=comp, energy=np.array(en))

    # --- end-to-end coil-sketched reconstructions (coil_sketch.py:220-330)
    def recon_case(name, dims, C, chat0, v, s, lam, T, K, scale, solver="fista", kind="l1-wavelet",
                   nufft=None, solver_cfg=None, reuse=True, use_init=False):
        shape = lo.GridShape(dims)
        maps = smooth_maps(g, dims, C)
        img = np.zeros(dims, complex)
        grids = np.meshgrid(*[np.linspace(-1, 1, n, endpoint=False) for n in dims], indexing="ij")
        for _ in range(4):
            c = g.uniform(-0.4, 0.4, len(dims)); ax = g.uniform(0.1, 0.5, len(dims))
            img += g.uniform(0.2, 1.0) * (sum(((gg - cc) / aa) ** 2 for gg, cc, aa in zip(grids, c, ax)) <= 1)
        img = img * np.exp(1j * np.pi * 0.3 * grids[0])
        weights = None
        if nufft is None:
            pts = random_mask_points(g, dims, 0.3)
            traj = lo.Trajectory(pts, "cartesian-mask")
            kern = None
        else:
            pts = radial_points(nufft[0], nufft[1], dims)
            traj = lo.Trajectory(pts, "non-cartesian")
            kern = lo._GriddedNUFFTKernel(shape, traj, nufft[2], nufft[3])
            weights = fm.radial_density_weights(traj)
        a = fm.SenseOperator(fm.SensitivityMaps(shape, maps), traj, kernel=kern)
        clean = a.forward_unweighted(img.ravel()).reshape(C, -1)
        sigma = 0.01 * np.abs(clean).max()
        noise = (g.standard_normal(clean.shape) + 1j * g.standard_normal(clean.shape)) * sigma / np.sqrt(2)
        data = clean + noise
        orig_gen = cs.gen_sketch_matrix
        orig_mk = fm.make_fourier_kernel
        cs.gen_sketch_matrix = scaled_gen(sk, scale)
        if kern is not None:
            fm.make_fourier_kernel = lambda sh, tr, method="auto": lo._GriddedNUFFTKernel(sh, tr, nufft[2], nufft[3])
        try:
            reg = so.make_regularizer(kind, lam, shape)
            cfg = cs.CoilSketchConfig(chat0, sk.SketchConfig(v + s, v, s, "rademacher", 0), reg, T, K,
                                      solver=solver, reuse_step_size=reuse, use_init=use_init)
            rep = cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg,
                                          weights=weights, solver_cfg=solver_cfg)
        finally:
            cs.gen_sketch_matrix = orig_gen
            fm.make_fourier_kernel = orig_mk
        out[name] = dict(dims=np.array(dims), points=pts, maps=maps, data=data, truth=img.ravel(),
                         chat0=np.array(chat0), v=np.array(v), s=np.array(s), lam=np.array(lam),
                         outer=np.array(T), inner=np.array(K), scale=np.array(scale),
                         x_final=rep.x_final.values, objectives=np.array([r.objective for r in rep.per_outer]),
                         counts=np.array(rep.counts.get("coil_transform", 0)),
                         expected=np.array(cs.expected_coil_transforms(cfg, so.SolverConfig(tol=0.0))),
                         diverged=np.array(rep.diverged),
                         weights=np.zeros(0) if weights is None else weights.w,
                         oversamp=np.array(0.0 if nufft is None else nufft[2]),
                         width=np.array(0 if nufft is None else nufft[3]),
                         tol=np.array(0.0 if solver_cfg is None else solver_cfg.tol),
                         max_iters=np.array(100 if solver_cfg is None else solver_cfg.max_iters),
                         reuse=np.array(reuse), use_init=np.array(use_init),
                         init_counts=np.array(rep.init_coil_transforms),
                         per_outer_counts=np.array([r.coil_transforms for r in rep.per_outer]))

    recon_case("recon_cart", (32, 32), 8, 8, 2, 2, 1e-3, 3, 4, 1.0 / np.sqrt(12))
    recon_case("recon_cart_pm1", (40, 32), 6, 6, 2, 1, 5e-3, 2, 5, 1.0)
    recon_case("recon_cart_cg", (24, 24), 6, 6, 2, 2, 1e-2, 2, 4, 1.0, solver="cg", kind="l2")
    recon_case("recon_radial", (16, 16), 4, 4, 2, 1, 5e-4, 2, 3, 1.0 / np.sqrt(12),
               nufft=(16, 32, 2.0, 4))

    # --- 1-D / 3-D wavelets (appended: earlier fixtures keep their RNG stream)
    for name, dims in [("wavelet_3d", (16, 12, 8)), ("wavelet_1d", (64,))]:
        shape = lo.GridShape(dims)
        w = lo.WaveletOp(shape)
        xx = crandn(g, shape.size)
        reg = so.make_regularizer("l1-wavelet", 0.3, shape)
        out[name] = dict(dims=np.array(dims), levels=np.array(w.levels), x=xx, fwd=w.forward(xx),
                         adj=w.adjoint(xx), prox=reg.prox(xx, 0.7), value=np.array(reg.value(xx)))
    # --- 3-D non-Cartesian (config-4 style, reduced) end to end
    recon_case_3d = dict(dims=(16, 16, 12), C=4, chat0=4, v=2, s=2, lam=1e-3, T=2, K=3)
    dims = recon_case_3d["dims"]
    shape = lo.GridShape(dims)
    C = recon_case_3d["C"]
    maps = smooth_maps(g, dims, C)
    grids = np.meshgrid(*[np.linspace(-1, 1, n, endpoint=False) for n in dims], indexing="ij")
    img = np.zeros(dims, complex)
    for _ in range(3):
        c = g.uniform(-0.3, 0.3, 3); ax = g.uniform(0.2, 0.5, 3)
        img += g.uniform(0.2, 1.0) * (sum(((gg - cc) / aa) ** 2 for gg, cc, aa in zip(grids, c, ax)) <= 1)
    # cones-like: random points on shells, kept inside [-n/2, n/2)
    npts = 1500
    rad = g.uniform(0, 1, npts) ** 0.7
    th = np.arccos(g.uniform(-1, 1, npts)); ph = g.uniform(0, 2 * np.pi, npts)
    half = np.array(dims) / 2 * 0.999
    pts = np.stack([rad * np.cos(th), rad * np.sin(th) * np.cos(ph), rad * np.sin(th) * np.sin(ph)], 1) * half
    traj = lo.Trajectory(pts, "non-cartesian")
    weights = fm.radial_density_weights(traj)
    kern = lo._GriddedNUFFTKernel(shape, traj, 1.25, 4)
    a = fm.SenseOperator(fm.SensitivityMaps(shape, maps), traj, kernel=kern)
    clean = a.forward_unweighted(img.ravel()).reshape(C, -1)
    data = clean + (g.standard_normal(clean.shape) + 1j * g.standard_normal(clean.shape)) * 0.01 * np.abs(clean).max() / np.sqrt(2)
    orig_gen, orig_mk = cs.gen_sketch_matrix, fm.make_fourier_kernel
    cs.gen_sketch_matrix = scaled_gen(sk, 1.0 / np.sqrt(12))
    fm.make_fourier_kernel = lambda sh, tr, method="auto": lo._GriddedNUFFTKernel(sh, tr, 1.25, 4)
    try:
        reg = so.make_regularizer("l1-wavelet", 1e-3, shape)
        cfg = cs.CoilSketchConfig(4, sk.SketchConfig(4, 2, 2, "rademacher", 0), reg, 2, 3)
        rep = cs.coil_sketching_recon(fm.KSpaceData(traj, data), fm.SensitivityMaps(shape, maps), cfg,
                                      weights=weights)
    finally:
        cs.gen_sketch_matrix, fm.make_fourier_kernel = orig_gen, orig_mk
    out["recon_cones3d"] = dict(dims=np.array(dims), points=pts, maps=maps, data=data, truth=img.ravel(),
                                chat0=np.array(4), v=np.array(2), s=np.array(2), lam=np.array(1e-3),
                                outer=np.array(2), inner=np.array(3), scale=np.array(1.0 / np.sqrt(12)),
                                x_final=rep.x_final.values,
                                objectives=np.array([r.objective for r in rep.per_outer]),
                                counts=np.array(rep.counts.get("coil_transform", 0)),
                                expected=np.array(cs.expected_coil_transforms(cfg, so.SolverConfig(tol=0.0))),
                                diverged=np.array(rep.diverged), weights=weights.w,
                                oversamp=np.array(1.25), width=np.array(4))

    # --- TV / PDHG sub-solver (appended last: earlier fixtures keep their RNG stream)
    recon_case("recon_cart_tv", (24, 20), 6, 6, 2, 2, 2e-3, 2, 3, 1.0, solver="pdhg", kind="l1-tv")
    tv_shape = lo.GridShape((12, 10))
    xx = crandn(g, tv_shape.size)
    fd = lo.FiniteDiffOp(tv_shape)
    yy = crandn(g, fd.out_dim)
    out["tv_ops"] = dict(dims=np.array((12, 10)), x=xx, y=yy, fwd=fd.forward(xx), adj=fd.adjoint(yy),
                         clamp=so._clamp_magnitude(yy, 0.8),
                         value=np.array(so.make_regularizer("l1-tv", 0.3, tv_shape).value(xx)))

    # --- full-coil solver baselines (appended last): reconstruct(l1-tv -> pdhg) and accproxsgd
    #     (solvers.py:315-362, 369-427, 434-500)
    dims = (24, 20)
    shape = lo.GridShape(dims)
    maps = smooth_maps(g, dims, 6)
    pts = random_mask_points(g, dims, 0.35)
    traj = lo.Trajectory(pts, "cartesian-mask")
    a = fm.build_sense(fm.SensitivityMaps(shape, maps), traj)
    grids = np.meshgrid(*[np.linspace(-1, 1, n, endpoint=False) for n in dims], indexing="ij")
    img = np.zeros(dims, complex)
    for _ in range(3):
        c = g.uniform(-0.4, 0.4, 2); ax = g.uniform(0.15, 0.5, 2)
        img += g.uniform(0.2, 1.0) * (sum(((gg - cc) / aa) ** 2 for gg, cc, aa in zip(grids, c, ax)) <= 1)
    clean = a.forward(img.ravel())
    y = clean + (g.standard_normal(clean.shape) + 1j * g.standard_normal(clean.shape)) * 0.01 * np.abs(clean).max()
    n0 = a.counts["coil_transform"]
    cfg_tv = so.SolverConfig(max_iters=6, tol=0.0, inner_cg_iters=4)
    res = so.reconstruct(a, y, so.make_regularizer("l1-tv", 2e-3, shape), cfg_tv)
    out["solve_pdhg_tv"] = dict(dims=np.array(dims), points=pts, maps=maps, y=y, lam=np.array(2e-3),
                                iters=np.array(6), cg_iters=np.array(4), x=res.x.values,
                                iterations=np.array(res.iterations_run),
                                counts=np.array(res.coil_transform_count))
    L = so.normal_max_eig(a)
    reg_w = so.make_regularizer("l1-wavelet", 1e-3, shape)
    x0 = lo.Image(shape, np.zeros(shape.size, dtype=np.complex128))
    res2 = so.accproxsgd(a, y, reg_w, 2, 1.0 / L, 0.95, 0.25 / L, x0, so.SolverConfig(max_iters=8, tol=0.0), seed=3)
    out["solve_accproxsgd"] = dict(dims=np.array(dims), points=pts, maps=maps, y=y, lam=np.array(1e-3),
                                   batch=np.array(2), alpha0=np.array(1.0 / L), beta=np.array(0.95),
                                   beta_min=np.array(0.25 / L), iters=np.array(8), seed=np.array(3),
                                   x=res2.x.values, iterations=np.array(res2.iterations_run),
                                   counts=np.array(res2.coil_transform_count), unused_n0=np.array(n0))

    # --- round 2 (appended last: earlier fixtures keep their RNG stream)
    # 3-D Cartesian mask SENSE operator (linops.py:332-364 on a 3-D grid), duplicated bins
    dims = (12, 10, 8)
    shape = lo.GridShape(dims)
    pts = random_mask_points(g, dims, 0.3)
    pts = np.concatenate([pts, pts[:7]], axis=0)
    traj = lo.Trajectory(pts, "cartesian-mask")
    maps = smooth_maps(g, dims, 4)
    a = fm.build_sense(fm.SensitivityMaps(shape, maps), traj)
    xx = crandn(g, shape.size)
    yy = crandn(g, 4 * traj.n_points)
    S = sk.gen_sketch_matrix(sk.SketchConfig(3, 2, 1, "rademacher", rng.child_seed(0, 2)), 4)
    a_s = sk.build_sketched_operator(a, S)
    out["sense_cart3d"] = dict(dims=np.array(dims), points=pts, maps=maps, x=xx, y=yy, Ax=a.forward(xx),
                               AHy=a.adjoint(yy), AHAx=a.adjoint(a.forward(xx)), S=S.mat,
                               AsHAsx=a_s.adjoint(a_s.forward(xx)))
    # Algorithm 1 on a 3-D Cartesian mask; FISTA early stopping (tol > 0, solvers.py:300);
    # per-outer step sizes (reuse_step_size=False, coil_sketch.py:281); classical-sketch init
    # (use_init, coil_sketch.py:148-159, 268-272)
    recon_case("recon_cart3d", (16, 12, 10), 4, 4, 2, 1, 1e-3, 2, 3, 1.0 / np.sqrt(12))
    recon_case("recon_cart_tol", (32, 24), 6, 6, 2, 2, 2e-3, 3, 12, 1.0,
               solver_cfg=so.SolverConfig(tol=0.02))
    recon_case("recon_cart_noreuse", (24, 32), 6, 6, 2, 2, 1e-3, 3, 4, 1.0 / np.sqrt(12), reuse=False)
    recon_case("recon_cart_init", (24, 24), 6, 6, 2, 2, 1e-3, 2, 3, 1.0,
               solver_cfg=so.SolverConfig(max_iters=6, tol=0.0), use_init=True)
    # full-coil reconstruct(): l1-wavelet -> FISTA, l2 -> CG (solvers.py:434-500), incl. tol stops
    dims = (24, 20)
    shape = lo.GridShape(dims)
    maps = smooth_maps(g, dims, 5)
    pts = random_mask_points(g, dims, 0.4)
    traj = lo.Trajectory(pts, "cartesian-mask")
    a = fm.build_sense(fm.SensitivityMaps(shape, maps), traj)
    grids = np.meshgrid(*[np.linspace(-1, 1, n, endpoint=False) for n in dims], indexing="ij")
    img = np.zeros(dims, complex)
    for _ in range(3):
        c = g.uniform(-0.4, 0.4, 2); ax = g.uniform(0.15, 0.5, 2)
        img += g.uniform(0.2, 1.0) * (sum(((gg - cc) / aa) ** 2 for gg, cc, aa in zip(grids, c, ax)) <= 1)
    clean = a.forward(img.ravel())
    y = clean + (g.standard_normal(clean.shape) + 1j * g.standard_normal(clean.shape)) * 0.01 * np.abs(clean).max()
    res_f = so.reconstruct(a, y, so.make_regularizer("l1-wavelet", 1e-3, shape),
                           so.SolverConfig(max_iters=12, tol=0.0, record_history=True))
    res_ft = so.reconstruct(a, y, so.make_regularizer("l1-wavelet", 1e-3, shape),
                            so.SolverConfig(max_iters=40, tol=3e-3))
    res_c = so.reconstruct(a, y, so.make_regularizer("l2", 1e-2, shape), so.SolverConfig(max_iters=10, tol=0.0,
                                                                                         record_history=True))
    res_ct = so.reconstruct(a, y, so.make_regularizer("l2", 1e-2, shape), so.SolverConfig(max_iters=50, tol=1e-3))
    out["solve_full"] = dict(dims=np.array(dims), points=pts, maps=maps, y=y,
                             fista_x=res_f.x.values, fista_hist=res_f.objective_history,
                             fista_counts=np.array(res_f.coil_transform_count),
                             fista_tol_x=res_ft.x.values, fista_tol_iters=np.array(res_ft.iterations_run),
                             cg_x=res_c.x.values, cg_hist=res_c.objective_history,
                             cg_counts=np.array(res_c.coil_transform_count),
                             cg_tol_x=res_ct.x.values, cg_tol_iters=np.array(res_ct.iterations_run))
    # pseudo-replica inverse g-factor with a CG-l2 reconstruction (metrics.py:157-211)
    import sketchrecon.metrics as met
    dims = (20, 16)
    shape = lo.GridShape(dims)
    maps = smooth_maps(g, dims, 4)
    full_pts = np.argwhere(np.ones(dims, bool)).astype(np.float64) - np.array([n // 2 for n in dims])
    under_pts = full_pts[(full_pts[:, 0] % 2 == 0) | (np.abs(full_pts[:, 0]) < 3)]
    a_full = fm.build_sense(fm.SensitivityMaps(shape, maps), lo.Trajectory(full_pts, "cartesian-mask"))
    a_under = fm.build_sense(fm.SensitivityMaps(shape, maps), lo.Trajectory(under_pts, "cartesian-mask"))
    img = np.zeros(dims, complex)
    grids = np.meshgrid(*[np.linspace(-1, 1, n, endpoint=False) for n in dims], indexing="ij")
    img += 1.0 * ((grids[0] / 0.7) ** 2 + (grids[1] / 0.6) ** 2 <= 1)
    reg2 = so.make_regularizer("l2", 1e-3, shape)
    recon = lambda op, yy: so.reconstruct(op, yy, reg2, so.SolverConfig(max_iters=8, tol=0.0)).x  # noqa: E731
    R = full_pts.shape[0] / under_pts.shape[0]
    gm = met.gfactor_montecarlo(recon, a_full, a_under, lo.Image(shape, img.ravel()), 0.05, 4, R, 11)
    out["gfactor"] = dict(dims=np.array(dims), maps=maps, full_points=full_pts, under_points=under_pts,
                          truth=img.ravel(), sigma=np.array(0.05), trials=np.array(4), R=np.array(R),
                          seed=np.array(11), lam=np.array(1e-3), iters=np.array(8),
                          inverse_g=gm.inverse_g, mask=gm.mask)

    only = set(sys.argv[1:])
    written = []
    for k, v in out.items():
        if only and k not in only:
            continue
        np.savez_compressed(OUT / f"{k}.npz", **v)
        written.append(k)
    print("wrote", ", ".join(sorted(written)))


if __name__ == "__main__":
    main()
