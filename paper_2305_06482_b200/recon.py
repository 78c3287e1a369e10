"""Batched device engine for Algorithm 1 (coil-sketched reconstruction).

Runs B independent slices in lock step (one slice = the reference's
``coil_sketching_recon``, /root/reference/pkg/src/sketchrecon/coil_sketch.py:220-306):

  per outer t:  d = A^H (A x - y)            (residual from the previous objective, K2)
                S^t drawn on the host          (coil_sketch.py:276-278, bit-identical)
                c_hat = S^t c                  (K5)
                [t == 1] L = lambda_max / s    (30 fused power steps, K1 + K7)
                inner FISTA / CG               (K1 with fused gradient epilogue, K6 prox
                                                with fused momentum, K7)
                objective 0.5||A x - y||^2 + lam ||Psi x||_1 -> residual for t+1
                divergence check (one host sync per outer)

No host synchronisation inside an inner loop (tol = 0 as in coil_sketch.py:246).
Counters follow the reference tally per slice: 2*C0 per true gradient,
2*C_hat per inner iteration; power iteration and objectives are paused.
"""

from __future__ import annotations

import contextlib
import ctypes
import gc

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .linops import CostCounter
from .rng import child_seed, seed_stream
from .sketching import SketchConfig, coil_contract, gen_sketch_matrix
from .wavelet import WaveletEngine

DIVERGENCE_FACTOR = 10.0  # coil_sketch.py:61


@dataclass
class EngineResult:
    x: torch.Tensor                 # (B, D) complex64, non-finite entries scrubbed
    objectives: np.ndarray          # (T_run, B)
    obj0: np.ndarray                # (B,)
    diverged: np.ndarray            # (B,) bool
    outer_run: np.ndarray           # (B,) outer iterations completed per slice
    lipschitz: np.ndarray           # (B,)
    counts: dict = field(default_factory=dict)
    per_outer_counts: list = field(default_factory=list)
    per_outer_wall: list = field(default_factory=list)
    per_outer_dist: list = field(default_factory=list)


_POWER_V0: dict = {}
# use_graph=None: replay the outer iterations of fixed-count runs with >= 3 outers as a CUDA graph
OUTER_GRAPH = os.environ.get("SR_OUTER_GRAPH", "1") != "0"
GRAPH_MAX_PIXELS = 1 << 21
# image-plane slabs of the coil-sharded NUFFT normal op whose all-reduces overlap the next slab
SHARD_SLABS = 4
@contextlib.contextmanager
def _gc_paused():
    """Python's cyclic collector off for the duration of a reconstruction: a full collection walks
    every tracked object of the process (~185 K with torch imported, ~33 ms) and lands at a random
    point of the launch stream; the engine itself creates almost no cyclic garbage."""
    was = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if was:
            gc.enable()


_SIDE_STREAMS: dict = {}


def _capture(fn, dev):
    """Capture fn() as a CUDA graph on a side stream (private memory pool); returns (graph, fn())."""
    g = torch.cuda.CUDAGraph()
    side = _SIDE_STREAMS.get(str(dev))
    if side is None:
        side = _SIDE_STREAMS[str(dev)] = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        # capture_begin/end directly: torch.cuda.graph() would empty the allocator cache
        g.capture_begin()
        out = fn()
        g.capture_end()
    torch.cuda.current_stream().wait_stream(side)
    return g, out


def _power_start(seed: int, d: int, dev) -> torch.Tensor:
    """Unit start vector of the power iteration (linops.py:766-782), cached per (seed, D, device):
    generating 2 D normals on the host dominates small-slice setup otherwise."""
    key = (int(seed), int(d), str(dev))
    v = _POWER_V0.get(key)
    if v is None:
        g = seed_stream(seed, 0)
        v0 = g.standard_normal(d) + 1j * g.standard_normal(d)
        v = dv.c64(v0 / np.linalg.norm(v0)).view(1, d).to(dev)
        if len(_POWER_V0) > 16:
            _POWER_V0.clear()
        _POWER_V0[key] = v
    return v


class SketchedReconEngine:
    """Device state of B slices sharing one grid, one Fourier kernel and one sketch design."""

    def __init__(self, kernel, maps0: torch.Tensor, y: torch.Tensor, *, dims, sketch: SketchConfig,
                 lam: float, reg: str = "l1-wavelet", solver: str = "fista", step_scale: float = 0.9,
                 sqrt_w: torch.Tensor | None = None, wavelet_levels: int | None = None,
                 counter: CostCounter | None = None, shard=None, use_graph: bool | None = None,
                 pdhg_ratio: float = 1.0, cg_iters: int = 8):
        self.kernel = kernel
        self.maps0 = maps0.contiguous()          # (B, C0, D) all compressed coils (sketch input)
        self.B, self.C0, self.D = self.maps0.shape
        # coil sharding (config 4): this rank applies the full operator over its coil block and
        # the sketched operator over its block of sketched coils; partials are all-reduced
        self.shard = shard if (shard is not None and shard.world > 1) else None
        if self.shard is not None:
            lo, hi = self.shard.coils(self.C0)
            self.maps_full = self.maps0[:, lo:hi].contiguous()
            y = y[:, lo:hi]
        else:
            self.maps_full = self.maps0
        self.y = y.contiguous()                  # (B, C0 or local coils, nmax) weighted measurements
        self.sketch = sketch
        self.lam = float(lam)
        self.reg = reg
        self.solver = solver
        self.step_scale = float(step_scale)
        self.sqrt_w = sqrt_w
        if sqrt_w is not None and hasattr(kernel, "prepare_weights"):
            kernel.prepare_weights(sqrt_w)  # not inside a graph capture (its first normal() may be captured)
        self.dims = tuple(dims)
        self.counter = counter if counter is not None else CostCounter()
        self.dev = self.maps0.device
        if reg not in ("l1-wavelet", "l2", "l1-tv"):
            raise ValueError(f"unknown regularizer {reg!r}")
        if solver == "cg" and reg != "l2":
            raise ValueError("cg sub-solver requires the l2 regularizer")
        if solver == "pdhg" and reg != "l1-tv":
            raise ValueError("pdhg sub-solver requires the l1-tv regularizer")
        if solver not in ("fista", "cg", "pdhg"):
            raise ValueError(f"unknown solver {solver!r}")
        if reg == "l1-tv" and solver != "pdhg":
            raise NotImplementedError("l1-tv is solved by the pdhg sub-solver (coil_sketch.py:200-216)")
        self.pdhg_ratio = float(pdhg_ratio)
        self.cg_iters = int(cg_iters)
        self.ndim = len(self.dims)
        self._cdims = (ctypes.c_int * self.ndim)(*self.dims)
        self.wav = WaveletEngine(self.dims, wavelet_levels, batch=self.B) if reg == "l1-wavelet" else None
        B, D = self.B, self.D
        mk = lambda: torch.zeros(B, D, dtype=torch.complex64, device=self.dev)  # noqa: E731
        self.x, self.z, self.v, self.d, self.anchor = mk(), mk(), mk(), mk(), mk()
        self.r = torch.zeros_like(self.y)
        self.partial = torch.zeros(kernel.partial_shape(max(1, self.maps_full.shape[1])), dtype=torch.float64,
                                   device=self.dev)
        self.tmp = mk() if self.shard is not None else None
        if reg == "l1-tv":  # dual variable and scratch of the PDHG sub-solver
            self.p = torch.zeros(B, self.ndim * D, dtype=torch.complex64, device=self.dev)
            self.wbuf, self.rhs, self.xn = mk(), mk(), mk()
        # every outer iteration after the first launches the same kernels on the same buffers, so a
        # fixed-count run captures it once as a CUDA graph and replays it (run(); None = auto)
        self.use_graph = use_graph if use_graph is None else bool(use_graph)
        if self.shard is not None:
            self.use_graph = False
        self.step = None       # (B,) float64 device
        self.fcoef = torch.zeros(B, 4, dtype=torch.float32, device=self.dev)
        self.thresh = torch.zeros(B, dtype=torch.float32, device=self.dev)
        self._bufs: dict = {}

    # ------------------------------------------------------------ pieces
    def _buf(self, name: str, shape, dtype, fill=None) -> torch.Tensor:
        """Persistent scratch tensor of the engine (allocated on first use, reused after): the
        outer iteration allocates nothing, so its CUDA graph owns no pool memory (freeing a graph's
        private pool synchronises the device whenever the garbage collector gets to it)."""
        shape = tuple(int(v) for v in shape)
        t = self._bufs.get(name)
        if t is None or tuple(t.shape) != shape or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, device=self.dev)
            if fill is not None:
                t.fill_(fill)
            self._bufs[name] = t
        return t

    def _normal(self, maps, x, out, anchor=None, coef=None, u=None, d=None):
        if self.shard is None:
            return self.kernel.normal(maps, x, out, w=self.sqrt_w, anchor=anchor, coef=coef, u=u, d=d)
        # partial over this rank's sketched coils, all-reduce, then the epilogue.  With a kernel
        # that finishes its image in slabs of planes (3-D NUFFT), each slab's all-reduce starts as
        # soon as its launches are queued and runs under the next slab's inverse passes.
        nplanes = self.kernel.slab_planes() if hasattr(self.kernel, "slab_planes") else 0
        if nplanes >= 2 * SHARD_SLABS and self.shard.world > 1 and self.B == 1:
            # every rank issues the same slab collectives (a rank without sketched coils sends zeros)
            bounds = [(nplanes * k // SHARD_SLABS, nplanes * (k + 1) // SHARD_SLABS) for k in range(SHARD_SLABS)]
            plane = self.D // nplanes
            works = []

            def slab_done(a, b):
                works.append(self.shard.all_reduce_async(self.tmp[:, a * plane:b * plane]))

            if maps.shape[1] > 0:
                self.kernel.normal_slabs(maps, x, self.tmp, bounds, slab_done, w=self.sqrt_w, anchor=anchor)
            else:
                self.tmp.zero_()
                for a, b in bounds:
                    slab_done(a, b)
            for wk in works:
                wk.wait()
        else:
            if maps.shape[1] > 0:
                self.kernel.normal(maps, x, self.tmp, w=self.sqrt_w, anchor=anchor)
            else:
                self.tmp.zero_()
            self.shard.all_reduce_(self.tmp)
        if coef is None:
            out.copy_(self.tmp)
        else:
            _lib.call("sr_lincomb", dv.ptr(out), dv.ptr(self.tmp), dv.ptr(u), dv.ptr(d), dv.ptr(coef), 0.0, 0.0,
                      0.0, self.D, self.D, self.B, dv.stream())
        return out

    def _sketch(self, mat: np.ndarray) -> torch.Tensor:
        """This rank's rows of S^t @ maps0 (all rows without sharding)."""
        if self.shard is None:
            return coil_contract(self.maps0, mat, out=self._buf("smaps", (self.B, mat.shape[-2], self.D),
                                                                   torch.complex64))
        lo, hi = self.shard.coils(mat.shape[0])
        if hi == lo:
            return torch.zeros(self.B, 0, self.D, dtype=torch.complex64, device=self.dev)
        return coil_contract(self.maps0, mat[lo:hi])

    def objective(self, x) -> torch.Tensor:
        """Per-slice 0.5||A x - y||^2 + g(x) (float64 device); leaves A x - y in self.r."""
        return self._objective_into(x, torch.empty(self.B, dtype=torch.float64, device=self.dev))

    def _objective_into(self, x, out) -> torch.Tensor:
        """objective(x) written into `out` (B,) with the engine's scratch only (no allocation);
        the same operations in the same order as the reference-shaped formula."""
        B = self.B
        if self.maps_full.shape[1] > 0:
            self.kernel.forward(self.maps_full, x, self.r, ymeas=self.y, partial=self.partial, w=self.sqrt_w)
        else:
            self.partial.zero_()
        if self.shard is not None:
            self.shard.all_reduce_(self.partial)
        torch.sum(self.partial.view(B, -1), dim=1, out=out)
        out.mul_(0.5)
        if self.lam != 0.0:
            reg = self._buf("obj_reg", (B,), torch.float64)
            if self.reg == "l1-wavelet":
                self.wav.l1_norm(x, out=reg, tmp=self._buf("obj_tmp", (B,), torch.float64))
                reg.mul_(self.lam)
            elif self.reg == "l1-tv":
                _lib.call("sr_tv_dual", dv.ptr(self.p), dv.ptr(x), self._cdims, self.ndim, 1, None, 0.0, self.B,
                          dv.stream())
                self._reduce_into(2, self.p, reg)
                reg.mul_(self.lam)
            else:
                self._reduce_into(0, x, reg)
                reg.mul_(0.5 * self.lam)
            out.add_(reg)
        return out

    def _reduce_into(self, mode: int, a, out) -> torch.Tensor:
        """out (B,) = the fixed-order device reduction `mode` of a (B, n) (sr_reduce), no allocation."""
        n = a.numel() // self.B
        nparts = _lib.lib().sr_reduce_nparts()
        part = self._buf("red_part", (self.B, nparts, 2), torch.float64)
        res = self._buf("red_res", (self.B, 2), torch.float64)
        _lib.call("sr_reduce", mode, dv.ptr(a), None, n, n, self.B, dv.ptr(part), dv.ptr(res), dv.stream())
        out.copy_(res[:, 0])
        return out

    def true_gradient(self, out):
        """d = A^H r with r = A x - y from the last objective (coil_sketch.py:123-126)."""
        self.counter.add("coil_transform", 2 * self.C0)
        if self.maps_full.shape[1] > 0:
            self.kernel.adjoint(self.maps_full, self.r, out, w=self.sqrt_w)
        else:
            out.zero_()
        if self.shard is not None:
            self.shard.all_reduce_(out)
        return out

    def power_lambda(self, smaps, iters: int = 30, seed: int = 0) -> torch.Tensor:
        """lambda_max(A_s^H A_s) per slice (linops.py:766-782), counters paused."""
        B, D = self.B, self.D
        v = self._buf("pw_v", (B, D), torch.complex64)
        v.copy_(_power_start(seed, D, self.dev).expand(B, D))  # v is updated in place
        w = self._buf("pw_w", (B, D), torch.complex64)
        nparts = _lib.lib().sr_reduce_nparts()
        part = self._buf("pw_part", (B, nparts, 2), torch.float64)
        r0 = self._buf("pw_r0", (B, 2), torch.float64)
        r1 = self._buf("pw_r1", (B, 2), torch.float64)
        lam = self._buf("pw_lam", (B,), torch.float64)
        lam.zero_()
        coef = self._buf("pw_coef", (B, 4), torch.float32)
        coef.zero_()
        flags = self._buf("pw_flags", (B,), torch.int32)
        flags.zero_()

        def step():
            st = dv.stream()
            self._normal(smaps, v, w)
            _lib.call("sr_reduce", 0, dv.ptr(w), None, self.D, self.D, self.B, dv.ptr(part), dv.ptr(r0), st)
            _lib.call("sr_reduce", 1, dv.ptr(v), dv.ptr(w), self.D, self.D, self.B, dv.ptr(part), dv.ptr(r1), st)
            _lib.call("sr_scalar_op", 0, dv.ptr(r0), dv.ptr(r1), dv.ptr(lam), dv.ptr(coef), None,
                      dv.ptr(flags), self.B, st)
            _lib.call("sr_lincomb", dv.ptr(v), dv.ptr(w), None, None, dv.ptr(coef), 0.0, 0.0, 0.0,
                      self.D, self.D, self.B, st)

        # launch-bound sizes replay one captured iteration (identical kernels on the same buffers)
        if self._graphable() and not torch.cuda.is_current_stream_capturing() and iters > 2:
            g, _ = _capture(step, self.dev)
            for _ in range(int(iters)):
                g.replay()
        else:
            for _ in range(int(iters)):
                step()
        return lam

    def _graphable(self) -> bool:
        """Launch-bound problem on a device kernel without collectives: CUDA graphs pay off."""
        auto = self.use_graph if self.use_graph is not None else (OUTER_GRAPH and self.B * self.D <= GRAPH_MAX_PIXELS)
        return bool(auto) and self.shard is None and getattr(self.kernel, "graph_capturable", True)

    def _fista(self, smaps, inner: int, tol: float = 0.0):
        """Warm-started FISTA on the anchored sub-problem (coil_sketch.py:192-199, solvers.py:284-301).

        tol > 0 (B = 1): the reference's relative-change stop `||x_new - x|| / ||x|| < tol`
        (solvers.py:296-301), evaluated with the fixed-order device reductions and one host
        read per inner iteration.  Returns the number of inner iterations run."""
        self.x.copy_(self.anchor)
        self.z.copy_(self.anchor)
        t_k = 1.0
        if tol > 0.0:
            xold = torch.empty_like(self.x)
        it = 0
        for it in range(1, inner + 1):
            if tol > 0.0:
                xold.copy_(self.x)
            self.counter.add("coil_transform", 2 * self.chat)
            # v = z - step * (A_s^H A_s (z - anchor) + d)
            self._normal(smaps, self.z, self.v, anchor=self.anchor, coef=self.fcoef, u=self.z, d=self.d)
            t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t_k * t_k))
            beta = (t_k - 1.0) / t_next
            if self.reg == "l1-wavelet":
                if self.lam == 0.0:
                    _lincomb(self.z, self.v, self.x, None, 1.0 + beta, -beta, 0.0, self.B, self.D)
                    self.x.copy_(self.v)
                else:
                    self.wav.prox(self.v, self.x, thresh=self.thresh, zout=self.z, xold=self.x, beta=beta)
            else:  # l2 prox v / (1 + step lam), then momentum
                _lincomb(self.v, self.v, None, None, 1.0, 0.0, 0.0, self.B, self.D, coef=self.l2coef)
                _lincomb(self.z, self.v, self.x, None, 1.0 + beta, -beta, 0.0, self.B, self.D)
                self.x.copy_(self.v)
            t_k = t_next
            if tol > 0.0 and self._rel_change_stop(self.x, xold, tol):
                break
        return it

    def _step_size(self, smaps):
        """Power iteration on this outer's sketched operator and the FISTA coefficients that follow
        from it (coil_sketch.py:279-283); device tensors only."""
        B = self.B
        f64 = torch.float64
        lam_max = self.power_lambda(smaps)
        lip = torch.div(lam_max, self.step_scale, out=self._buf("st_lip", (B,), f64))
        step = torch.reciprocal(lip, out=self._buf("st_step", (B,), f64))
        t = torch.neg(step, out=self._buf("st_t", (B,), f64))
        self.fcoef[:, 0] = t
        self.fcoef[:, 1] = 1.0
        self.fcoef[:, 2] = t
        self.thresh.copy_(torch.mul(step, self.lam, out=t))
        if self.reg == "l2":
            if getattr(self, "l2coef", None) is None:
                self.l2coef = torch.zeros(B, 4, dtype=torch.float32, device=self.dev)
            torch.mul(step, self.lam, out=t)
            t.add_(1.0)
            self.l2coef[:, 0] = torch.reciprocal(t, out=t)
        return lip

    def _outer_body(self, mat, inner: int, tol: float, power: bool):
        """One outer iteration of Algorithm 1 up to its objective: d = A^H r, the sketched maps of
        `mat`, (the step size), the anchored sub-solve and the objective.  Returns (obj, finite,
        lip or None); nothing in it reads the host when tol == 0, so it can be a CUDA graph."""
        self.true_gradient(self.d)
        smaps = self._sketch(mat)
        lip = self._step_size(smaps) if power else None
        self.anchor.copy_(self.x)
        if self.solver == "fista":
            self._fista(smaps, inner, tol)
        elif self.solver == "pdhg":
            self._pdhg(smaps, inner, tol)
        else:
            self._cg(smaps, inner)
        # x is finite iff sum |x|^2 is (fp64 accumulation of float32 squares cannot overflow)
        B = self.B
        n2 = self._reduce_into(0, self.x, self._buf("x_norm2", (B,), torch.float64))
        finite = torch.lt(n2, float("inf"), out=self._buf("x_finite", (B,), torch.bool))
        obj = self._objective_into(self.x, self._buf("obj_val", (B,), torch.float64))
        obj = torch.where(finite, obj, self._buf("obj_inf", (B,), torch.float64, fill=float("inf")),
                          out=self._buf("obj_out", (B,), torch.float64))
        return obj, finite, lip

    def _capture_outer(self, mat_buf, inner: int, power: bool):
        """Capture _outer_body on the persistent sketch buffer `mat_buf` as one CUDA graph (its
        temporaries live in the shared graph pool; the engine's buffers and the kernels'
        workspaces exist from the eager first outer, so replays touch the same memory)."""
        with self.counter.paused():
            return _capture(lambda: self._outer_body(mat_buf, inner, 0.0, power), self.dev)

    def _cg_solve(self, smaps, sol, rhs, shift_coef, iters: int):
        """sol = `iters` CG steps on (A_s^H A_s + shift I) sol = rhs from sol = 0 (_cg_loop,
        solvers.py:206-229); shift_coef (B, 4) = {1, shift, 0, 0} is the K1 epilogue of the matvec.
        Per iteration: K1 with the shift epilogue, then the fused vector step (csrc/vecops.cu
        sr_cg_step: <p, Mp>, x/r update with |r|^2, p update; fixed-order reductions).  A slice
        whose residual vanishes or whose curvature p^H M p <= 0 stops updating, as the reference's
        loop breaks (state kept on the device, no host sync)."""
        B, D, st = self.B, self.D, dv.stream()
        sol.zero_()
        r = self._buf("cg_r", rhs.shape, rhs.dtype)
        r.copy_(rhs)
        p = self._buf("cg_p", rhs.shape, rhs.dtype)
        p.copy_(r)
        mp = self._buf("cg_mp", rhs.shape, rhs.dtype)
        nparts = _lib.lib().sr_reduce_nparts()
        pdot = self._buf("cg_pdot", (B, nparts, 2), torch.float64)
        prs = self._buf("cg_prs", (B, nparts, 2), torch.float64)
        rs = self._buf("cg_rs", (B, 2), torch.float64)
        state = self._buf("cg_state", (B, 4), torch.float64)
        state.zero_()
        _lib.call("sr_reduce", 0, dv.ptr(r), None, D, D, B, dv.ptr(pdot), dv.ptr(rs), st)
        state[:, 0] = rs[:, 0]
        state[:, 2] = 1.0
        for it in range(iters):
            self.counter.add("coil_transform", 2 * self.chat)
            self._normal(smaps, p, mp, coef=shift_coef, u=p)
            _lib.call("sr_cg_step", dv.ptr(sol), dv.ptr(r), dv.ptr(p), dv.ptr(mp), dv.ptr(pdot), dv.ptr(prs),
                      dv.ptr(state), None, 0, D, D, B, it & 1, 0.0, st)
        return sol

    def _cg(self, smaps, inner: int):
        """(A_s^H A_s + lam I) delta = -d - lam x^t, x = x^t + delta (coil_sketch.py:182-191)."""
        B, D = self.B, self.D
        delta = self._buf("cgo_delta", self.x.shape, self.x.dtype)
        delta.zero_()
        rhs = self._buf("cgo_rhs", self.x.shape, self.x.dtype)
        _lincomb(rhs, self.d, self.anchor, None, -1.0, -self.lam, 0.0, B, D)
        lcoef = self._buf("cgo_lcoef", (B, 4), torch.float32)
        lcoef.zero_()
        lcoef[:, 0] = 1.0
        lcoef[:, 1] = self.lam
        self._cg_solve(smaps, delta, rhs, lcoef, inner)
        _lincomb(self.x, self.anchor, delta, None, 1.0, 1.0, 0.0, B, D)

    def _rel_change_stop(self, new, old, tol: float) -> bool:
        """||new - old|| / ||old|| < tol (solvers.py:300, 354) for B = 1, fixed-order device
        reductions, one host read."""
        st = dv.stream()
        if getattr(self, "_tolbuf", None) is None:
            nparts = _lib.lib().sr_reduce_nparts()
            self._tolbuf = (torch.empty_like(self.x), torch.empty(1, nparts, 2, dtype=torch.float64, device=self.dev),
                            torch.empty(2, 2, dtype=torch.float64, device=self.dev))
        diff, part, rd = self._tolbuf
        _lincomb(diff, new, old, None, 1.0, -1.0, 0.0, 1, self.D)
        _lib.call("sr_reduce", 0, dv.ptr(diff), None, self.D, self.D, 1, dv.ptr(part), dv.ptr(rd[0:1]), st)
        _lib.call("sr_reduce", 0, dv.ptr(old), None, self.D, self.D, 1, dv.ptr(part), dv.ptr(rd[1:2]), st)
        h = rd[:, 0].cpu().numpy()
        delta, x_norm = math.sqrt(max(h[0], 0.0)), math.sqrt(max(h[1], 0.0))
        return x_norm > 0 and delta / x_norm < tol

    def _pdhg(self, smaps, inner: int, tol: float = 0.0):
        """Chambolle-Pock on min_x 0.5||A_s(x - x^t)||^2 + Re<d, x> + lam ||D x||_1 with K = D
        (coil_sketch.py:200-216, solvers.py:315-362): per iteration p = clamp(p + sigma D z, lam),
        v = x - tau D^H p, x' = v + CG_k((A_s^H A_s + I/tau) w = -d - A_s^H A_s (v - x^t)),
        z = 2 x' - x.  sigma tau ||D||^2 = step_scale^2 with ||D|| = 2 sqrt(ndim)."""
        B, D, st = self.B, self.D, dv.stream()
        norm_k = 2.0 * math.sqrt(self.ndim)
        ratio = math.sqrt(self.pdhg_ratio)
        sigma = ratio / norm_k * self.step_scale
        tau = 1.0 / (ratio * norm_k) * self.step_scale
        sig_t = self._buf("pd_sig", (B,), torch.float32)
        sig_t.fill_(sigma)
        tau_t = self._buf("pd_tau", (B,), torch.float32)
        tau_t.fill_(tau)
        shift = self._buf("pd_shift", (B, 4), torch.float32)
        shift.zero_()
        shift[:, 0] = 1.0
        shift[:, 1] = 1.0 / tau
        rcoef = self._buf("pd_rcoef", (B, 4), torch.float32)
        rcoef.zero_()
        rcoef[:, 0] = -1.0
        rcoef[:, 2] = -1.0
        self.x.copy_(self.anchor)
        self.z.copy_(self.anchor)
        self.p.zero_()
        x_buf = self.x
        for _ in range(inner):
            _lib.call("sr_tv_dual", dv.ptr(self.p), dv.ptr(self.z), self._cdims, self.ndim, 0, dv.ptr(sig_t),
                      self.lam, B, st)
            _lib.call("sr_tv_primal", dv.ptr(self.v), dv.ptr(self.x), dv.ptr(self.p), self._cdims, self.ndim,
                      dv.ptr(tau_t), B, st)
            self.counter.add("coil_transform", 2 * self.chat)
            self._normal(smaps, self.v, self.rhs, anchor=self.anchor, coef=rcoef, d=self.d)  # -N(v - a) - d
            self._cg_solve(smaps, self.wbuf, self.rhs, shift, self.cg_iters)
            _lincomb(self.xn, self.v, self.wbuf, None, 1.0, 1.0, 0.0, B, D)
            _lincomb(self.z, self.xn, self.x, None, 2.0, -1.0, 0.0, B, D)
            stop = tol > 0.0 and self._rel_change_stop(self.xn, self.x, tol)
            self.x, self.xn = self.xn, self.x
            if stop:
                break
        if self.x is not x_buf:
            # the iterate ends in the buffer it started in (a captured outer replays on fixed pointers)
            x_buf.copy_(self.x)
            self.x, self.xn = x_buf, self.x

    # ------------------------------------------------------------ Algorithm 1
    def run(self, outer: int, inner: int, x0: torch.Tensor | None = None,
            x_ref: torch.Tensor | None = None, tol: float = 0.0, reuse_step_size: bool = True) -> EngineResult:
        """Algorithm 1 (see _run), with the Python cyclic garbage collector paused."""
        with _gc_paused():
            return self._run(outer, inner, x0=x0, x_ref=x_ref, tol=tol, reuse_step_size=reuse_step_size)

    def _run(self, outer: int, inner: int, x0: torch.Tensor | None = None,
             x_ref: torch.Tensor | None = None, tol: float = 0.0, reuse_step_size: bool = True) -> EngineResult:
        """Algorithm 1 (coil_sketch.py:220-306).  tol > 0: FISTA inner solves stop on the relative
        change (solvers.py:300; B = 1); reuse_step_size=False re-runs the power iteration on
        every outer's sketched operator (coil_sketch.py:281)."""
        B = self.B
        tol = float(tol)
        if tol > 0.0 and (B != 1 or self.solver == "cg"):
            raise ValueError("inner-solver early stopping (tol > 0) runs FISTA / PDHG one slice at a time")
        t_start = time.perf_counter()
        ev_start = torch.cuda.Event(enable_timing=True)
        ev_start.record()
        if x0 is not None:
            self.x.copy_(x0)
        else:
            self.x.zero_()
        # With a fixed inner count (tol = 0) nothing inside the loop needs a host decision: the
        # sketch draws are made up front (host RNG, bit-identical, one upload), the divergence
        # test, the frozen copy of a diverged slice, the objectives and the distances stay on the
        # device, and everything is read back once at the end (CUDA events time the outers).
        # A slice that diverges keeps its frozen image; the outers after the last live one are
        # trimmed from the records and their coil transforms removed from the counter, so the
        # report equals the reference's early exit (coil_sketch.py:300-302).  tol > 0 needs a
        # host read per inner iteration anyway and keeps the per-outer checks on the host.
        deferred = tol == 0.0
        obj0_d = self.objective(self.x)
        alive_d = torch.ones(B, dtype=torch.bool, device=self.dev)
        outer_run_d = torch.zeros(B, dtype=torch.int64, device=self.dev)
        frozen = self.x.clone()
        obj_hist = torch.full((outer, B), float("inf"), dtype=torch.float64, device=self.dev)
        dist_hist = torch.full((outer, B), float("nan"), dtype=torch.float64, device=self.dev)
        cnts, evs = [], []
        lip = None
        ref_norm = None
        if x_ref is not None:
            ref_norm = torch.linalg.vector_norm(x_ref.to(torch.complex128), dim=1)
        mats = [gen_sketch_matrix(self.sketch.with_seed(child_seed(self.sketch.seed, t)), self.C0).mat
                for t in range(1, outer + 1)]
        mats_d = torch.from_numpy(np.ascontiguousarray(np.stack(mats), dtype=np.float32)).to(self.dev)
        self.chat = mats[0].shape[0]
        t_done = 0
        # From the second outer on, a fixed-count run replays the whole outer iteration as one CUDA
        # graph (captured once): the host issues a sketch-row copy, the replay and the bookkeeping
        # instead of ~150 launches per outer.  The first outer runs eagerly: it sizes every
        # workspace and (reuse_step_size) runs the power iteration whose step the replays keep.
        graph = self.use_graph
        if graph is None:
            # launch-bound problems only: a batch of large slices (config 2) gains nothing and its
            # capture would allocate the sketched maps again in the graph's private pool
            graph = OUTER_GRAPH and outer >= 3 and B * self.D <= GRAPH_MAX_PIXELS
        graph = bool(graph) and deferred and self.shard is None and getattr(self.kernel, "graph_capturable", True)
        power_each = self.solver == "fista" and not reuse_step_size
        captured = None
        mat_buf = None
        per_outer = None
        for t in range(1, outer + 1):
            if graph and t >= 2:
                if captured is None:
                    mat_buf = mats_d[t - 1].clone()
                    captured = self._capture_outer(mat_buf, inner, power_each)
                else:
                    mat_buf.copy_(mats_d[t - 1])
                captured[0].replay()
                obj, finite, lip_t = captured[1]
                if lip_t is not None:
                    lip = lip_t
                for tag, n in per_outer.items():
                    self.counter.add(tag, n)
            else:
                c_before = self.counter.asdict()
                obj, finite, lip_t = self._outer_body(mats_d[t - 1], inner, tol,
                                                      self.solver == "fista" and (lip is None or power_each))
                if lip_t is not None:
                    lip = lip_t
                c_after = self.counter.asdict()
                per_outer = {k: v - c_before.get(k, 0) for k, v in c_after.items() if v != c_before.get(k, 0)}
            obj_hist[t - 1] = obj
            cnts.append(self.counter.value("coil_transform"))
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            evs.append(ev)
            if x_ref is not None:
                dist_hist[t - 1] = torch.linalg.vector_norm((self.x - x_ref).to(torch.complex128), dim=1) / ref_norm
            newly = alive_d & ((~finite) | (obj > DIVERGENCE_FACTOR * obj0_d))
            outer_run_d = torch.where(alive_d, torch.full_like(outer_run_d, t), outer_run_d)
            fr = torch.view_as_real(frozen)
            fr.copy_(torch.where(newly.view(B, 1, 1), torch.view_as_real(self.x), fr))
            alive_d = alive_d & ~newly
            t_done = t
            if not deferred and not bool(alive_d.any()):
                break
        # the one host read of the run
        obj_h = obj_hist[:t_done].cpu().numpy()
        outer_run = outer_run_d.cpu().numpy()
        diverged = ~alive_d.cpu().numpy()
        obj0 = obj0_d.cpu().numpy()
        dists = list(dist_hist[:t_done].cpu().numpy())
        walls = [ev_start.elapsed_time(e) / 1e3 for e in evs]
        t_last = int(outer_run.max()) if B else t_done
        if t_last < t_done:  # every slice stopped at t_last: drop the outers run past it
            self.counter.add("coil_transform", cnts[t_last - 1] - cnts[t_done - 1])
            obj_h, cnts, walls, dists = obj_h[:t_last], cnts[:t_last], walls[:t_last], dists[:t_last]
        x = self.x.clone()
        if diverged.any():
            idx = torch.as_tensor(np.nonzero(diverged)[0], device=self.dev)
            x.index_copy_(0, idx, frozen.index_select(0, idx))
        xr = torch.view_as_real(x)
        x = torch.view_as_complex(torch.where(torch.isfinite(xr), xr, torch.zeros_like(xr)).contiguous())
        return EngineResult(x, obj_h, obj0, diverged, outer_run,
                            np.full(B, np.nan) if lip is None else lip.cpu().numpy(),
                            self.counter.asdict(), cnts, walls, dists)


def _abs_sum(x) -> torch.Tensor:
    B = x.shape[0]
    n = x.numel() // B
    nparts = _lib.lib().sr_reduce_nparts()
    part = torch.empty(B, nparts, 2, dtype=torch.float64, device=x.device)
    res = torch.empty(B, 2, dtype=torch.float64, device=x.device)
    _lib.call("sr_reduce", 2, dv.ptr(x), None, n, n, B, dv.ptr(part), dv.ptr(res), dv.stream())
    return res[:, 0]


def _norm2(x) -> torch.Tensor:
    B, D = x.shape
    nparts = _lib.lib().sr_reduce_nparts()
    part = torch.empty(B, nparts, 2, dtype=torch.float64, device=x.device)
    res = torch.empty(B, 2, dtype=torch.float64, device=x.device)
    _lib.call("sr_reduce", 0, dv.ptr(x), None, D, D, B, dv.ptr(part), dv.ptr(res), dv.stream())
    return res[:, 0]


def _lincomb(out, X, Y, Z, cx, cy, cz, B, D, coef=None):
    _lib.call("sr_lincomb", dv.ptr(out), dv.ptr(X), dv.ptr(Y), dv.ptr(Z), dv.ptr(coef), float(cx),
              float(cy), float(cz), D, D, B, dv.stream())
