"""Coil-sketched reconstruction (Algorithm 1), mirroring coil_sketch.py of the reference.

``coil_sketching_recon`` keeps the reference signature and report
(/root/reference/pkg/src/sketchrecon/coil_sketch.py:220-306) and runs the
outer/inner loops in the batched device engine (recon.SketchedReconEngine)
with B = 1.  ``coil_sketching_recon_batched`` runs many independent slices
(e.g. readout-decoupled 3-D Cartesian data, BASELINE config 2) in lock step.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from .forward_model import (DensityWeights, KSpaceData, SenseOperator, SensitivityMaps, build_sense,
                            coil_compress_device, coil_compress_svd)
from .linops import Image, make_fourier_kernel
from .recon import DIVERGENCE_FACTOR, SketchedReconEngine, _gc_paused
from .rng import child_seed
from .sketching import SketchConfig, SketchMatrix, apply_sketch_to_data, build_sketched_operator, gen_sketch_matrix
from .solvers import Regularizer, SolverConfig, composite_objective, reconstruct

__all__ = ["CoilSketchConfig", "SketchSubproblem", "OuterRecord", "ReconReport", "true_gradient",
           "sketched_objective_grad", "sketched_objective_value", "classical_sketch_solve",
           "coil_sketching_recon", "coil_sketching_recon_batched", "solver_apps_per_inner",
           "expected_coil_transforms", "DIVERGENCE_FACTOR"]


@dataclass(frozen=True)
class CoilSketchConfig:
    """Outer-loop parameters (coil_sketch.py:64-91)."""

    c_hat0: int
    sketch: SketchConfig
    reg: Regularizer
    outer_iters: int = 10
    inner_iters: int = 20
    use_init: bool = False
    reuse_step_size: bool = True
    solver: str = "fista"

    def __post_init__(self):
        if self.c_hat0 < 1:
            raise ValueError("c_hat0 must be >= 1")
        if self.sketch.c_hat > self.c_hat0:
            raise ValueError("sketch c_hat cannot exceed c_hat0")
        if self.outer_iters < 1:
            raise ValueError("outer_iters must be >= 1")
        if self.inner_iters < 1:
            raise ValueError("inner_iters must be >= 1")
        if self.solver not in ("cg", "fista", "pdhg"):
            raise ValueError(f"unknown solver {self.solver!r}")
        if self.solver == "cg" and self.reg.kind != "l2":
            raise ValueError("cg sub-solver requires the l2 regularizer")
        if self.solver == "pdhg" and self.reg.kind != "l1-tv":
            raise ValueError("pdhg sub-solver requires the l1-tv regularizer")


@dataclass(frozen=True)
class SketchSubproblem:
    anchor: object
    true_grad: object
    sketched_op: SenseOperator
    reg: Regularizer


@dataclass(frozen=True)
class OuterRecord:
    outer_index: int
    distance: float
    objective: float
    coil_transforms: int
    wall_time: float


@dataclass
class ReconReport:
    x_final: Image
    per_outer: list = field(default_factory=list)
    diverged: bool = False
    init_coil_transforms: int = 0
    counts: dict = field(default_factory=dict)
    energy_fraction: float = 1.0


def true_gradient(a: SenseOperator, x, y):
    """d = A^H (A x - y) (coil_sketch.py:123-126)."""
    vec = x.values if isinstance(x, Image) else x
    host = not isinstance(vec, torch.Tensor)
    r = a._forward(dv.c64(vec)) - dv.c64(y)
    g = a._adjoint(r)
    return dv.to_numpy128(g) if host else g


def sketched_objective_grad(sub: SketchSubproblem, x):
    """A_S^H A_S (x - x^t) + d (coil_sketch.py:129-133), fused K1 epilogue."""
    vec = x.values if isinstance(x, Image) else x
    host = not isinstance(vec, torch.Tensor)
    xv = dv.c64(vec).view(1, -1)
    out = torch.empty_like(xv)
    one = torch.tensor([[1.0, 0.0, 1.0, 0.0]], dtype=torch.float32, device=xv.device)
    sub.sketched_op.normal_into(xv, out, anchor=dv.c64(sub.anchor).view(1, -1), coef=one,
                                d=dv.c64(sub.true_grad).view(1, -1))
    return dv.to_numpy128(out[0]) if host else out[0]


def sketched_objective_value(sub: SketchSubproblem, x, include_reg: bool = True) -> float:
    """0.5 ||A_S (x - x^t)||^2 + Re<d, x> (+ g) (coil_sketch.py:136-145)."""
    vec = dv.c64(x.values if isinstance(x, Image) else x)
    a_s = sub.sketched_op
    with a_s.paused_counts():
        q = a_s._forward(vec - dv.c64(sub.anchor))
    val = 0.5 * float(torch.linalg.vector_norm(q.to(torch.complex128)) ** 2)
    val += float(torch.real(torch.vdot(dv.c64(sub.true_grad).to(torch.complex128), vec.to(torch.complex128))))
    if include_reg:
        val += sub.reg.value(vec)
    return val


def classical_sketch_solve(a: SenseOperator, y, sk: SketchMatrix, reg: Regularizer,
                           solver_cfg: SolverConfig, solver: str | None = None) -> Image:
    """One-shot min 0.5||S A x - S y||^2 + g(x) (coil_sketch.py:148-159)."""
    a_s = build_sketched_operator(a, sk)
    y_s = apply_sketch_to_data(np.asarray(y), sk, a.n_points)
    return reconstruct(a_s, y_s, reg, solver_cfg, solver=solver).x


def _reg_kind(reg: Regularizer) -> str:
    return reg.kind


def coil_sketching_recon(data: KSpaceData, maps: SensitivityMaps, cfg: CoilSketchConfig,
                         weights: DensityWeights | None = None, solver_cfg: SolverConfig | None = None,
                         x_ref: Image | None = None, x0: Image | None = None, method: str = "auto",
                         kernel=None, compress: str = "device") -> ReconReport:
    """Full coil-sketched reconstruction on the device (coil_sketch.py:220-306); see
    _coil_sketching_recon.  Python's cyclic garbage collector is paused for the call."""
    with _gc_paused():
        return _coil_sketching_recon(data, maps, cfg, weights, solver_cfg, x_ref, x0, method, kernel, compress)


def _coil_sketching_recon(data: KSpaceData, maps: SensitivityMaps, cfg: CoilSketchConfig,
                          weights: DensityWeights | None = None, solver_cfg: SolverConfig | None = None,
                          x_ref: Image | None = None, x0: Image | None = None, method: str = "auto",
                          kernel=None, compress: str = "device") -> ReconReport:
    """Full coil-sketched reconstruction on the device (coil_sketch.py:220-306).

    ``kernel`` optionally injects the Fourier kernel (e.g. a GriddedKernel with
    BASELINE's oversampling/width), where the reference builds its own.
    ``compress``: "device" (default) takes the PCA basis from a device Householder QR of
    Y^H plus a C x C host SVD; "lapack" runs numpy's SVD of Y on the host as the reference
    does.  Both give the same singular subspaces, but LAPACK fixes each singular vector's
    phase by rounding-level details of its own bidiagonalisation, so on some inputs a few
    PCA coils come out with a different (equally valid) phase, which changes the Rademacher
    combinations and moves the iterates by ~1e-4 NRMSE.
    """
    if cfg.c_hat0 > data.n_coils:
        raise ValueError(f"c_hat0 = {cfg.c_hat0} exceeds the {data.n_coils} available coils")
    kind = _reg_kind(cfg.reg)
    if compress not in ("device", "lapack"):
        raise ValueError(f"compress must be 'device' or 'lapack', got {compress!r}")
    if compress == "device":
        maps0_dev, data0_dev, _, energy = coil_compress_device(data, maps, cfg.c_hat0)
        a = SenseOperator(maps0_dev, data.traj, weights, method=method, kernel=kernel, shape=maps.shape)
        y = data0_dev
        if weights is not None and not data.weights_applied:
            y = y * a.sqrt_w_dev.to(torch.complex64)
        y = y.view(1, cfg.c_hat0, a.n_points)
    else:
        data0, maps0, _, energy = coil_compress_svd(data, maps, cfg.c_hat0)
        a = SenseOperator(maps0, data0.traj, weights, method=method, kernel=kernel)
        y = dv.c64(a.measurement_vector(data0)).view(1, cfg.c_hat0, a.n_points)
    solver_cfg = solver_cfg or SolverConfig(tol=0.0)
    ypad = torch.zeros(1, cfg.c_hat0, a.kernel.nmax, dtype=torch.complex64, device=y.device)
    ypad[:, :, : a.n_points] = y
    init_count = 0
    x0_dev = None
    if x0 is not None:
        x0_dev = dv.c64(x0.values).view(1, -1)
    if cfg.use_init:
        before = a.counts.get("coil_transform", 0)
        sk0 = gen_sketch_matrix(cfg.sketch.with_seed(child_seed(cfg.sketch.seed, 0)), cfg.c_hat0)
        x0_dev = dv.c64(classical_sketch_solve(a, dv.to_numpy128(y.reshape(-1)), sk0, cfg.reg, solver_cfg,
                                               cfg.solver).values).view(1, -1)
        init_count = a.counts.get("coil_transform", 0) - before
    eng = SketchedReconEngine(a.kernel, a.maps_dev, ypad, dims=maps.shape.dims, sketch=cfg.sketch,
                              lam=cfg.reg.lam, reg=kind, solver=cfg.solver,
                              step_scale=solver_cfg.step_scale, sqrt_w=a.sqrt_w_dev,
                              wavelet_levels=getattr(cfg.reg.transform, "levels", None), counter=a.counter,
                              pdhg_ratio=solver_cfg.pdhg_sigma_tau_ratio, cg_iters=solver_cfg.inner_cg_iters)
    ref = None if x_ref is None else dv.c64(x_ref.values).view(1, -1)
    # the reference passes tol to the FISTA / PDHG sub-solvers; its CG sub-solver always runs
    # the full budget (coil_sketch.py:182-191)
    tol = solver_cfg.tol if cfg.solver in ("fista", "pdhg") else 0.0
    res = eng.run(cfg.outer_iters, cfg.inner_iters, x0=x0_dev, x_ref=ref, tol=tol,
                  reuse_step_size=cfg.reuse_step_size)
    report = ReconReport(x_final=Image(maps.shape, dv.to_numpy128(res.x[0])), energy_fraction=energy,
                         init_coil_transforms=init_count)
    for t in range(len(res.objectives)):
        report.per_outer.append(OuterRecord(t + 1, float(res.per_outer_dist[t][0]), float(res.objectives[t][0]),
                                            int(res.per_outer_counts[t]), float(res.per_outer_wall[t])))
    report.diverged = bool(res.diverged[0])
    report.counts = a.counts
    report.lipschitz = float(res.lipschitz[0])
    return report


def coil_sketching_recon_batched(kernel, maps0: torch.Tensor, y: torch.Tensor, cfg: CoilSketchConfig,
                                 dims, solver_cfg: SolverConfig | None = None, sqrt_w=None,
                                 x0: torch.Tensor | None = None):
    """B independent (already coil-compressed) slices in lock step on one device.

    maps0: (B, C0, D) complex64; y: (B, C0, nmax) weighted measurements.
    Returns the engine result (x: (B, D) device tensor, per-slice objectives).
    """
    solver_cfg = solver_cfg or SolverConfig(tol=0.0)
    eng = SketchedReconEngine(kernel, maps0, y, dims=dims, sketch=cfg.sketch, lam=cfg.reg.lam,
                              reg=_reg_kind(cfg.reg), solver=cfg.solver, step_scale=solver_cfg.step_scale,
                              sqrt_w=sqrt_w, wavelet_levels=getattr(cfg.reg.transform, "levels", None),
                              pdhg_ratio=solver_cfg.pdhg_sigma_tau_ratio, cg_iters=solver_cfg.inner_cg_iters)
    return eng.run(cfg.outer_iters, cfg.inner_iters, x0=x0)


def solver_apps_per_inner(solver: str, solver_cfg: SolverConfig) -> int:
    """Operator applications per inner iteration (coil_sketch.py:309-315)."""
    if solver in ("cg", "fista"):
        return 2
    if solver == "pdhg":
        return 2 * (solver_cfg.inner_cg_iters + 1)
    raise ValueError(f"unknown solver {solver!r}")


def expected_coil_transforms(cfg: CoilSketchConfig, solver_cfg: SolverConfig, init_count: int = 0,
                             outer_iters: int | None = None) -> int:
    """init + T (2 C0 + inner k C_hat) (coil_sketch.py:318-330)."""
    t = cfg.outer_iters if outer_iters is None else outer_iters
    k = solver_apps_per_inner(cfg.solver, solver_cfg)
    return init_count + t * (2 * cfg.c_hat0 + cfg.inner_iters * k * cfg.sketch.c_hat)
