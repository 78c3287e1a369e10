"""Iterative solvers and proximal maps (mirrors solvers.py of the reference).

Same signatures and semantics as /root/reference/pkg/src/sketchrecon/solvers.py
for the pairings on the sketched-operator path (l2 -> CG, l1-wavelet ->
FISTA).  Callbacks receive and return complex64 CUDA tensors; vector algebra
runs in the device kernels of csrc/vecops.cu, norms/dots are fixed-order
device reductions.  The l1-TV / PDHG / AccProxSGD pairings are outside the
hot-path scope and raise
NotImplementedError.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .forward_model import SenseOperator
from .linops import FiniteDiffOp, GridShape, IdentityOp, Image, LinOp, WaveletOp, max_eig_power

__all__ = ["Regularizer", "SolverConfig", "SolveResult", "make_regularizer", "prox_l1", "cg_normal",
           "fista", "reconstruct", "normal_max_eig", "composite_objective", "pdhg", "accproxsgd"]


# --------------------------------------------------------------------- device helpers
def _reduce(mode: int, a: torch.Tensor, b: torch.Tensor | None = None) -> torch.Tensor:
    """Fixed-order reduction of (B, n) tensors -> (B, 2) float64 device tensor."""
    a2 = a.reshape(a.shape[0], -1) if a.dim() > 1 else a.reshape(1, -1)
    B, n = a2.shape
    nparts = _lib.lib().sr_reduce_nparts()
    part = torch.empty(B, nparts, 2, dtype=torch.float64, device=a.device)
    res = torch.empty(B, 2, dtype=torch.float64, device=a.device)
    _lib.call("sr_reduce", mode, dv.ptr(a2), dv.ptr(b), n, n, B, dv.ptr(part), dv.ptr(res), dv.stream())
    return res


def dev_norm2(a) -> torch.Tensor:
    return _reduce(0, a.contiguous())[:, 0]


def dev_abs_sum(a) -> torch.Tensor:
    """sum |a_i| per row (complex magnitudes), (B,) float64."""
    return _reduce(2, a.contiguous())[:, 0]


def dev_vdot(a, b) -> torch.Tensor:
    """sum conj(a) b, (B, 2) [re, im]."""
    return _reduce(1, a.contiguous(), b.contiguous())


def lincomb(out, X, Y=None, Z=None, cx=1.0, cy=0.0, cz=0.0, coef=None):
    """out = cx X + cy Y + cz Z (host scalars) or per-slice device coef (B, 4)."""
    X2 = X.reshape(X.shape[0], -1) if X.dim() > 1 else X.reshape(1, -1)
    B, n = X2.shape
    _lib.call("sr_lincomb", dv.ptr(out), dv.ptr(X), dv.ptr(Y), dv.ptr(Z), dv.ptr(coef), float(cx),
              float(cy), float(cz), n, n, B, dv.stream())
    return out


# --------------------------------------------------------------------- regularizers
@dataclass(frozen=True)
class Regularizer:
    """g(x) = lam/2 ||x||^2 or lam ||Psi x||_1 (solvers.py:47-81)."""

    kind: str
    lam: float
    transform: LinOp

    def __post_init__(self):
        if self.kind not in ("l2", "l1-wavelet", "l1-tv"):
            raise ValueError(f"unknown regularizer kind {self.kind!r}")
        if self.lam < 0:
            raise ValueError("lambda must be nonnegative")

    def value(self, x) -> float:
        """g(x) without advancing cost counters (solvers.py:61-69)."""
        if self.lam == 0.0:
            return 0.0
        xt = dv.c64(x)
        if self.kind == "l2":
            return 0.5 * self.lam * float(dev_norm2(xt.view(1, -1))[0])
        if self.kind == "l1-wavelet":
            return self.lam * float(self.transform.engine.l1_norm(xt.view(1, -1))[0])
        with self.transform.paused_counts():
            tx = self.transform.forward(xt.reshape(-1))
        return self.lam * float(dev_abs_sum(tx.view(1, -1))[0])

    def prox(self, v, step: float, tv_iters: int = 10):
        """prox_{step g}(v) (solvers.py:71-81); numpy in -> numpy out, tensor -> tensor."""
        host = not isinstance(v, torch.Tensor)
        vt = dv.c64(v)
        if self.lam == 0.0:
            out = vt.clone()
        elif self.kind == "l2":
            out = vt / (1.0 + step * self.lam)
        elif self.kind == "l1-wavelet":
            out = torch.empty_like(vt)
            self.transform.engine.prox(vt.view(1, -1), out.view(1, -1), hthresh=step * self.lam)
        else:
            out = tv_prox(vt.reshape(1, -1), step * self.lam, self.transform.shape, tv_iters).reshape(vt.shape)
        return dv.to_numpy128(out) if host else out


def make_regularizer(kind: str, lam: float, shape: GridShape, wavelet_levels: int | None = None):
    """Regularizer with its transform (solvers.py:84-97)."""
    if kind == "l2":
        return Regularizer(kind, lam, IdentityOp(shape.size))
    if kind == "l1-wavelet":
        return Regularizer(kind, lam, WaveletOp(shape, wavelet_levels))
    if kind == "l1-tv":
        return Regularizer(kind, lam, FiniteDiffOp(shape))
    raise ValueError(f"unknown regularizer kind {kind!r}")


def tv_op_norm(ndim: int) -> float:
    """||D|| = 2 sqrt(ndim) for circular finite differences (solvers.py:145-148)."""
    return 2.0 * float(np.sqrt(ndim))


def tv_prox(v: torch.Tensor, weight: float, shape: GridShape, iters: int) -> torch.Tensor:
    """argmin_u 0.5||u - v||^2 + weight ||D u||_1 by the reference's short PDHG loop
    (_tv_prox, solvers.py:152-164), batched over rows of v (B, D) on the device."""
    import ctypes
    B, D = v.shape
    dims = (ctypes.c_int * shape.ndim)(*shape.dims)
    sigma = tau = 1.0 / max(tv_op_norm(shape.ndim), 1e-12)
    st = dv.stream()
    sig_t = torch.full((B,), sigma, dtype=torch.float32, device=v.device)
    tau_t = torch.full((B,), tau, dtype=torch.float32, device=v.device)
    x = v.clone()
    z = x.clone()
    t = torch.empty_like(x)
    p = torch.zeros(B, shape.ndim * D, dtype=torch.complex64, device=v.device)
    for _ in range(int(iters)):
        _lib.call("sr_tv_dual", dv.ptr(p), dv.ptr(z), dims, shape.ndim, 0, dv.ptr(sig_t), float(weight), B, st)
        _lib.call("sr_tv_primal", dv.ptr(t), dv.ptr(x), dv.ptr(p), dims, shape.ndim, dv.ptr(tau_t), B, st)
        xn = torch.empty_like(x)
        lincomb(xn, t, v, None, 1.0 / (1.0 + tau), tau / (1.0 + tau), 0.0)
        lincomb(z, xn, x, None, 2.0, -1.0, 0.0)
        x = xn
    return x


@dataclass(frozen=True)
class SolverConfig:
    """(solvers.py:100-117)"""

    max_iters: int = 100
    tol: float = 1e-6
    step_scale: float = 0.9
    pdhg_sigma_tau_ratio: float = 1.0
    inner_cg_iters: int = 8
    record_history: bool = False

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.tol < 0:
            raise ValueError("tol must be nonnegative")
        if not 0 < self.step_scale <= 1:
            raise ValueError("step_scale must be in (0, 1]")
        if self.inner_cg_iters < 1:
            raise ValueError("inner_cg_iters must be >= 1")


@dataclass
class SolveResult:
    x: Image
    iterations_run: int
    objective_history: np.ndarray
    coil_transform_count: int
    wall_time: float


def prox_l1(v, thresh: float):
    """Complex soft threshold; zeros stay zero (solvers.py:129-135)."""
    if thresh < 0:
        raise ValueError("threshold must be nonnegative")
    if isinstance(v, torch.Tensor):
        mag = torch.abs(v)
        scale = torch.clamp(mag - thresh, min=0.0) / torch.where(mag > 0, mag, torch.ones_like(mag))
        return v * scale
    mag = np.abs(v)
    return v * (np.maximum(mag - thresh, 0.0) / np.where(mag > 0, mag, 1.0))


class _NormalOp(LinOp):
    """A^H A sharing A's counters; fused K1 when A is a SenseOperator (solvers.py:167-180)."""

    def __init__(self, a: LinOp):
        super().__init__(a.in_dim, a.in_dim)
        self._a = a

    def _forward(self, x):
        if isinstance(self._a, SenseOperator):
            out = torch.empty(1, self.in_dim, dtype=torch.complex64, device=x.device)
            self._a.normal_into(x.view(1, -1).contiguous(), out)
            return out[0]
        return self._a._adjoint(self._a._forward(x))

    _adjoint = _forward

    def _counters(self):
        return self._a._counters() + (self.counter,)


def normal_max_eig(a: LinOp, iters: int = 30, seed: int = 0) -> float:
    """lambda_max(A^H A) by power iteration, counters paused (solvers.py:183-185)."""
    return max_eig_power(_NormalOp(a), iters=iters, seed=seed)


def composite_objective(a: LinOp, y, reg: Regularizer | None, x) -> float:
    """0.5 ||A x - y||^2 + g(x), counters paused (solvers.py:188-195)."""
    yt = dv.c64(y)
    with a.paused_counts():
        r = a._forward(dv.c64(x)) - yt
    obj = 0.5 * float(dev_norm2(r.view(1, -1))[0])
    if reg is not None:
        obj += reg.value(x)
    return obj


def _coil_count(a) -> int:
    return a.counts.get("coil_transform", 0)


def _cg_loop(matvec, b, x0, max_iters, tol_abs, history=None):
    """Plain CG on M x = b (solvers.py:206-229); device tensors, fixed-order dots."""
    x = dv.c64(x0).clone()
    b = dv.c64(b)
    r = b - matvec(x) if bool(torch.any(x != 0)) else b.clone()
    p = r.clone()
    rs = float(dev_norm2(r.view(1, -1))[0])
    res = [math.sqrt(rs)]
    it = 0
    for it in range(1, max_iters + 1):
        if math.sqrt(rs) <= tol_abs:
            it -= 1
            break
        mp = matvec(p)
        denom = float(dev_vdot(p.view(1, -1), mp.view(1, -1))[0, 0])
        if denom <= 0:
            break
        alpha = rs / denom
        lincomb(x, x, p, cx=1.0, cy=alpha)
        lincomb(r, r, mp, cx=1.0, cy=-alpha)
        rs_new = float(dev_norm2(r.view(1, -1))[0])
        res.append(math.sqrt(rs_new))
        lincomb(p, r, p, cx=1.0, cy=rs_new / rs)
        rs = rs_new
    return x, it, np.array(res)


def cg_normal(a: LinOp, y, lam: float, x0: Image, cfg: SolverConfig) -> SolveResult:
    """(A^H A + lam I) x = A^H y by CG (solvers.py:232-257)."""
    if lam < 0:
        raise ValueError("lambda must be nonnegative")
    t0 = time.perf_counter()
    n0 = _coil_count(a)
    b = a._adjoint(dv.c64(y))
    tol_abs = cfg.tol * math.sqrt(float(dev_norm2(b.view(1, -1))[0]))
    nop = _NormalOp(a)

    def matvec(v):
        return nop._forward(v) + lam * v

    x, iters, res = _cg_loop(matvec, b, x0.values, cfg.max_iters, tol_abs)
    return SolveResult(Image(x0.shape, x), iters, res if cfg.record_history else np.empty(0),
                       _coil_count(a) - n0, time.perf_counter() - t0)


def fista(grad, prox, L: float, x0: Image, cfg: SolverConfig, objective=None,
          op_for_count: LinOp | None = None) -> SolveResult:
    """FISTA with Nesterov momentum (solvers.py:264-308); grad/prox act on device tensors."""
    if L <= 0:
        raise ValueError("Lipschitz constant must be positive")
    t0 = time.perf_counter()
    n0 = _coil_count(op_for_count) if op_for_count is not None else 0
    step = 1.0 / L
    x = dv.c64(x0.values)
    z = x.clone()
    t_k = 1.0
    hist = []
    iters = 0
    for iters in range(1, cfg.max_iters + 1):
        v = z - step * grad(z)
        x_new = prox(v, step)
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t_k * t_k))
        z = torch.empty_like(x_new)
        lincomb(z, x_new, x, cx=1.0 + (t_k - 1.0) / t_next, cy=-(t_k - 1.0) / t_next)
        need = cfg.tol > 0
        if need:
            diff = torch.empty_like(x_new)
            lincomb(diff, x_new, x, cx=1.0, cy=-1.0)
            delta = math.sqrt(float(dev_norm2(diff.view(1, -1))[0]))
            x_norm = math.sqrt(float(dev_norm2(x.view(1, -1))[0]))
        x = x_new
        t_k = t_next
        if cfg.record_history and objective is not None:
            hist.append(objective(x))
        if need and x_norm > 0 and delta / x_norm < cfg.tol:
            break
    return SolveResult(Image(x0.shape, x), iters, np.array(hist),
                       (_coil_count(op_for_count) - n0) if op_for_count is not None else 0,
                       time.perf_counter() - t0)


def reconstruct(a: SenseOperator, y, reg: Regularizer, cfg: SolverConfig, x0: Image | None = None,
                solver: str | None = None, lipschitz: float | None = None) -> SolveResult:
    """min 0.5 ||A x - y||^2 + g(x) with the paired solver (solvers.py:434-500)."""
    if x0 is None:
        x0 = Image(a.shape, np.zeros(a.in_dim, dtype=np.complex128))
    solver = solver or {"l2": "cg", "l1-wavelet": "fista", "l1-tv": "pdhg"}[reg.kind]
    if solver == "cg":
        if reg.kind != "l2":
            raise ValueError("cg solves the l2-regularized problem")
        return cg_normal(a, y, reg.lam, x0, cfg)
    if solver == "fista":
        if lipschitz is None:
            lipschitz = normal_max_eig(a) / cfg.step_scale
        yt = dv.c64(y)
        nop = _NormalOp(a)
        with a.paused_counts():
            aty = a._adjoint(yt)  # A^H y once; each grad() still tallies 2C like the reference

        def grad(v):
            return nop._forward(v) - aty

        def prox(v, step):
            return reg.prox(v, step)

        return fista(grad, prox, lipschitz, x0, cfg,
                     objective=lambda v: composite_objective(a, y, reg, v), op_for_count=a)
    if solver == "pdhg":
        raise NotImplementedError("PDHG (l1-tv) is outside the sketched-operator hot-path scope")
    raise ValueError(f"unknown solver {solver!r}")


def pdhg(*args, **kwargs):
    raise NotImplementedError("PDHG is outside the sketched-operator hot-path scope (SURVEY.md 2, row 9b)")


def accproxsgd(*args, **kwargs):
    raise NotImplementedError("AccProxSGD is outside the sketched-operator hot-path scope (SURVEY.md 2, row 9b)")
