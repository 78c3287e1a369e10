"""Iterative solvers and proximal maps (mirrors solvers.py of the reference).

Same signatures and semantics as /root/reference/pkg/src/sketchrecon/solvers.py
for the three regularizer pairings (l2 -> CG, l1-wavelet -> FISTA, l1-tv -> PDHG
with the inner-CG data prox) and the AccProxSGD baseline over coil batches.
Callbacks receive and return complex64 CUDA tensors; vector algebra runs in the
device kernels of csrc/vecops.cu and csrc/tv.cu, norms/dots are fixed-order
device reductions.
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
    """Plain CG on M x = b (solvers.py:206-229) on the device: per iteration the caller's matvec
    and the fused vector step of csrc/vecops.cu (sr_cg_step: alpha, x/r update, |r|^2, beta,
    p update, fixed-order reductions).  The reference's breaks (sqrt(rs) <= tol_abs before an
    iteration, p^H M p <= 0 inside it) freeze the device state instead of returning early, so the
    loop never reads a scalar back; the iteration count and the residual history are read once
    at the end."""
    x = dv.c64(x0).clone().view(1, -1)
    b = dv.c64(b).view(1, -1)
    D = x.shape[1]
    r = (b - matvec(x[0]).view(1, -1)) if bool(torch.any(x != 0)) else b.clone()
    p = r.clone()
    st = dv.stream()
    nparts = _lib.lib().sr_reduce_nparts()
    pdot = torch.empty(1, nparts, 2, dtype=torch.float64, device=x.device)
    prs = torch.empty_like(pdot)
    rs0 = torch.empty(1, 2, dtype=torch.float64, device=x.device)
    _lib.call("sr_reduce", 0, dv.ptr(r), None, D, D, 1, dv.ptr(pdot), dv.ptr(rs0), st)
    state = torch.zeros(1, 4, dtype=torch.float64, device=x.device)
    state[:, 0] = rs0[:, 0]
    state[:, 2] = 1.0
    hist = torch.full((1, max_iters + 1), float("nan"), dtype=torch.float64, device=x.device)
    hist[:, 0] = torch.sqrt(rs0[:, 0])
    for it in range(max_iters):
        mp = matvec(p[0]).view(1, -1).contiguous()
        _lib.call("sr_cg_step", dv.ptr(x), dv.ptr(r), dv.ptr(p), dv.ptr(mp), dv.ptr(pdot), dv.ptr(prs),
                  dv.ptr(state), dv.ptr(hist), max_iters, D, D, 1, it & 1, float(tol_abs), st)
    iters = int(state[0, 3].item())
    # one history entry per completed update (a p^H M p <= 0 break counts the iteration but
    # appends nothing); entries never written stay NaN
    h = hist[0].cpu().numpy()
    return x[0], iters, h[~np.isnan(h)]


def _shifted_normal(a: LinOp, shift: float):
    """v -> A^H A v + shift v; for a SenseOperator one fused K1 call with the epilogue
    {1, shift} (no separate vector op), counting 2C coil transforms like adjoint(forward)."""
    if isinstance(a, SenseOperator):
        coef = torch.tensor([[1.0, float(shift), 0.0, 0.0]], dtype=torch.float32, device=a.maps_dev.device)

        def mv(v):
            vv = v.view(1, -1).contiguous()
            out = torch.empty_like(vv)
            a.normal_into(vv, out, coef=coef, u=vv)
            return out[0]
        return mv
    nop = _NormalOp(a)

    def mv(v):
        out = nop._forward(v)
        return out + shift * v if shift else out
    return mv


def cg_normal(a: LinOp, y, lam: float, x0: Image, cfg: SolverConfig) -> SolveResult:
    """(A^H A + lam I) x = A^H y by CG (solvers.py:232-257)."""
    if lam < 0:
        raise ValueError("lambda must be nonnegative")
    t0 = time.perf_counter()
    n0 = _coil_count(a)
    b = a._adjoint(dv.c64(y))
    tol_abs = cfg.tol * math.sqrt(float(dev_norm2(b.view(1, -1))[0]))
    matvec = _shifted_normal(a, lam)

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
        v = torch.empty_like(x)  # fresh: a caller's prox may return its argument
        lincomb(v, z, grad(z), cx=1.0, cy=-step)
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
        with a.paused_counts():
            aty = a._adjoint(yt).view(1, -1)  # A^H y once; each grad() still tallies 2C like the reference
        if isinstance(a, SenseOperator):
            gcoef = torch.tensor([[1.0, 0.0, -1.0, 0.0]], dtype=torch.float32, device=aty.device)

            def grad(v):  # A^H A v - A^H y in one fused K1 call (epilogue {1, 0, -1})
                vv = v.view(1, -1).contiguous()
                out = torch.empty_like(vv)
                a.normal_into(vv, out, coef=gcoef, d=aty)
                return out[0]
        else:
            nop = _NormalOp(a)

            def grad(v):
                return nop._forward(v) - aty[0]

        def prox(v, step):
            return reg.prox(v, step)

        return fista(grad, prox, lipschitz, x0, cfg,
                     objective=lambda v: composite_objective(a, y, reg, v), op_for_count=a)
    if solver == "pdhg":
        if reg.kind != "l1-tv":
            raise ValueError("pdhg is paired with the l1-tv regularizer")
        return _pdhg_tv(a, y, reg, x0, cfg)
    raise ValueError(f"unknown solver {solver!r}")


def _pdhg_steps(norm_K: float, cfg: SolverConfig) -> tuple[float, float]:
    ratio = math.sqrt(cfg.pdhg_sigma_tau_ratio)
    sigma = ratio / norm_K * cfg.step_scale
    tau = 1.0 / (ratio * norm_K) * cfg.step_scale
    if sigma * tau * norm_K ** 2 > 1.0 + 1e-12:
        raise ValueError("step-size product violates sigma*tau*||K||^2 <= 1")
    return sigma, tau


def pdhg(K: LinOp, prox_fdual, prox_g, x0: Image, cfg: SolverConfig, norm_K: float | None = None,
         objective=None, op_for_count: LinOp | None = None) -> SolveResult:
    """Chambolle-Pock primal-dual iteration for min_x g(x) + f(K x) (solvers.py:315-362).

    K acts on device tensors; prox_fdual(p, sigma) / prox_g(v, tau) receive and return complex64
    CUDA tensors.  The axpys run in the sr_lincomb kernel, norms in the fixed-order reductions."""
    t0 = time.perf_counter()
    n0 = _coil_count(op_for_count) if op_for_count is not None else 0
    if norm_K is None:
        norm_K = math.sqrt(max(normal_max_eig(K, iters=30, seed=0), 1e-30))
    sigma, tau = _pdhg_steps(norm_K, cfg)
    x = dv.c64(x0.values).reshape(-1).clone()
    z = x.clone()
    p = torch.zeros(K.out_dim, dtype=torch.complex64, device=x.device)
    hist = []
    iters = 0
    for iters in range(1, cfg.max_iters + 1):
        kz = K.forward(z)
        lincomb(kz, p, kz, cx=1.0, cy=sigma)
        p = prox_fdual(kz, sigma)
        ka = K.adjoint(p)
        lincomb(ka, x, ka, cx=1.0, cy=-tau)
        x_new = prox_g(ka, tau)
        z = torch.empty_like(x_new)
        lincomb(z, x_new, x, cx=2.0, cy=-1.0)
        done = False
        if cfg.tol > 0:
            diff = torch.empty_like(x_new)
            lincomb(diff, x_new, x, cx=1.0, cy=-1.0)
            delta = math.sqrt(float(dev_norm2(diff.view(1, -1))[0]))
            x_norm = math.sqrt(float(dev_norm2(x.view(1, -1))[0]))
            done = x_norm > 0 and delta / x_norm < cfg.tol
        x = x_new
        if cfg.record_history and objective is not None:
            hist.append(objective(x))
        if done:
            break
    return SolveResult(Image(x0.shape, x), iters, np.array(hist),
                       (_coil_count(op_for_count) - n0) if op_for_count is not None else 0,
                       time.perf_counter() - t0)


def clamp_magnitude(p: torch.Tensor, radius: float, shape: GridShape) -> torch.Tensor:
    """Project each complex entry of a (ndim * D) dual variable onto |p| <= radius
    (_clamp_magnitude, solvers.py:138-142), in place, by the dual-step kernel with sigma = 0."""
    import ctypes
    dims = (ctypes.c_int * shape.ndim)(*shape.dims)
    zero_img = torch.zeros(shape.size, dtype=torch.complex64, device=p.device)
    sig0 = torch.zeros(1, dtype=torch.float32, device=p.device)
    _lib.call("sr_tv_dual", dv.ptr(p), dv.ptr(zero_img), dims, shape.ndim, 0, dv.ptr(sig0), float(radius), 1,
              dv.stream())
    return p


def _pdhg_tv(a: SenseOperator, y, reg: Regularizer, x0: Image, cfg: SolverConfig) -> SolveResult:
    """reconstruct(l1-tv) -> PDHG with K = D, f* prox = clamp to lam, and the data prox
    v + argmin_w from inner CG on (A^H A + I/tau) w = A^H (y - A v) (solvers.py:470-500).
    The dual step p = clamp(p + sigma D z, lam) and the primal step v = x - tau D^H p are
    single fused kernels (csrc/tv.cu); the CG matvec is the fused normal operator."""
    import ctypes
    shape = reg.transform.shape
    nd, D = shape.ndim, shape.size
    dims = (ctypes.c_int * nd)(*shape.dims)
    sigma, tau = _pdhg_steps(tv_op_norm(nd), cfg)
    t0 = time.perf_counter()
    n0 = _coil_count(a)
    yt = dv.c64(y).reshape(-1)
    x = dv.c64(x0.values).reshape(1, D).clone()
    z = x.clone()
    v = torch.empty_like(x)
    p = torch.zeros(1, nd * D, dtype=torch.complex64, device=x.device)
    sig_t = torch.full((1,), sigma, dtype=torch.float32, device=x.device)
    tau_t = torch.full((1,), tau, dtype=torch.float32, device=x.device)
    st = dv.stream()
    matvec = _shifted_normal(a, 1.0 / tau)  # one fused K1 call per CG matvec

    hist = []
    iters = 0
    for iters in range(1, cfg.max_iters + 1):
        _lib.call("sr_tv_dual", dv.ptr(p), dv.ptr(z), dims, nd, 0, dv.ptr(sig_t), float(reg.lam), 1, st)
        _lib.call("sr_tv_primal", dv.ptr(v), dv.ptr(x), dv.ptr(p), dims, nd, dv.ptr(tau_t), 1, st)
        r = a._forward(v.reshape(-1))
        lincomb(r, yt, r, cx=1.0, cy=-1.0)
        rhs = a._adjoint(r)
        w, _, _ = _cg_loop(matvec, rhs, torch.zeros_like(rhs), cfg.inner_cg_iters, 0.0)
        x_new = torch.empty_like(x)
        lincomb(x_new, v, w.view(1, -1), cx=1.0, cy=1.0)
        lincomb(z, x_new, x, cx=2.0, cy=-1.0)
        done = False
        if cfg.tol > 0:
            diff = torch.empty_like(x)
            lincomb(diff, x_new, x, cx=1.0, cy=-1.0)
            delta = math.sqrt(float(dev_norm2(diff)[0]))
            x_norm = math.sqrt(float(dev_norm2(x)[0]))
            done = x_norm > 0 and delta / x_norm < cfg.tol
        x = x_new
        if cfg.record_history:
            hist.append(composite_objective(a, yt, reg, x.reshape(-1)))
        if done:
            break
    return SolveResult(Image(x0.shape, x.reshape(-1)), iters, np.array(hist), _coil_count(a) - n0,
                       time.perf_counter() - t0)


def accproxsgd(op: SenseOperator, y, reg: Regularizer, batch: int, alpha0: float, beta: float,
               beta_min: float, x0: Image, cfg: SolverConfig, seed: int = 0, objective=None) -> SolveResult:
    """Accelerated proximal SGD over random coil batches (solvers.py:369-427).

    The coil draws are the reference's (seed_stream(seed, 0).choice, sorted) on the host; each
    iteration's sub-operator (coil_subset, sharing kernel and counter) runs one forward and one
    adjoint on the device (2 * batch coil transforms), the prox and momentum are device kernels."""
    from .rng import seed_stream
    n_coils = op.n_coils
    if not 1 <= batch <= n_coils:
        raise ValueError(f"batch must be in [1, {n_coils}], got {batch}")
    t0 = time.perf_counter()
    n0 = _coil_count(op)
    rng = seed_stream(seed, 0)
    y_mat = dv.c64(y).reshape(n_coils, op.n_points)
    scale = n_coils / batch
    x = dv.c64(x0.values).reshape(-1).clone()
    z = x.clone()
    t_k = 1.0
    hist = []
    iters = 0
    for iters in range(1, cfg.max_iters + 1):
        idx = np.sort(rng.choice(n_coils, size=batch, replace=False))
        sub = op.coil_subset(idx)
        ysub = y_mat.index_select(0, torch.as_tensor(idx, device=y_mat.device)).reshape(-1)
        resid = sub._forward(z)
        lincomb(resid, resid, ysub, cx=1.0, cy=-1.0)
        g = sub._adjoint(resid)
        alpha = max(beta ** iters * alpha0, beta_min)
        v = torch.empty_like(z)
        lincomb(v, z, g, cx=1.0, cy=-alpha * scale)
        x_new = reg.prox(v, alpha)
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t_k * t_k))
        z = torch.empty_like(x_new)
        lincomb(z, x_new, x, cx=1.0 + (t_k - 1.0) / t_next, cy=-(t_k - 1.0) / t_next)
        done = False
        if cfg.tol > 0:
            diff = torch.empty_like(x_new)
            lincomb(diff, x_new, x, cx=1.0, cy=-1.0)
            delta = math.sqrt(float(dev_norm2(diff.view(1, -1))[0]))
            x_norm = math.sqrt(float(dev_norm2(x.view(1, -1))[0]))
            done = x_norm > 0 and delta / x_norm < cfg.tol
        x = x_new
        t_k = t_next
        if cfg.record_history and objective is not None:
            hist.append(objective(x))
        if done:
            break
    return SolveResult(Image(x0.shape, x), iters, np.array(hist), _coil_count(op) - n0,
                       time.perf_counter() - t0)
