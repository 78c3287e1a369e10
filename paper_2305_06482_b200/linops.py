"""Operator algebra mirroring ``sketchrecon.linops`` on the device.

Reference: /root/reference/pkg/src/sketchrecon/linops.py.  Same types and
contracts (GridShape/Image/Trajectory validation, CostCounter tags and pause
semantics, LinOp shape checks raising ValueError), but operators act on
device tensors:

* ``forward``/``adjoint`` accept a numpy vector (coerced like linops.py:205,
  computed on the GPU in complex64, returned as complex128 numpy) or a CUDA
  tensor (returned as a complex64 CUDA tensor, no host round trip).
"""

from __future__ import annotations

import ctypes

import contextlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .rng import seed_stream
from .wavelet import WaveletEngine, default_wavelet_levels

__all__ = [
    "GridShape", "Image", "Trajectory", "CostCounter", "LinOp", "IdentityOp", "DiagonalOp",
    "ComposeOp", "CenteredFFTOp", "CartesianMaskOp", "WaveletOp", "FiniteDiffOp", "make_fourier_kernel",
    "default_wavelet_levels", "max_eig_power", "dot_test",
]


@dataclass(frozen=True)
class GridShape:
    """Rectangular 1-3 axis grid (linops.py:53-73)."""

    dims: tuple

    def __post_init__(self):
        dims = tuple(int(n) for n in self.dims)
        object.__setattr__(self, "dims", dims)
        if not 1 <= len(dims) <= 3:
            raise ValueError(f"grid must have 1-3 axes, got {dims}")
        if any(n < 2 for n in dims):
            raise ValueError(f"every grid dim must be >= 2, got {dims}")

    @property
    def size(self) -> int:
        return int(np.prod(self.dims))

    @property
    def ndim(self) -> int:
        return len(self.dims)


@dataclass(frozen=True)
class Image:
    """Complex image vector with its grid (linops.py:76-100)."""

    shape: GridShape
    values: np.ndarray

    def __post_init__(self):
        v = self.values
        if isinstance(v, torch.Tensor):
            v = dv.to_numpy128(v)
        v = np.ascontiguousarray(v, dtype=np.complex128)
        if v.ndim != 1 or v.size != self.shape.size:
            raise ValueError(f"values must be a flat vector of length {self.shape.size}, "
                             f"got shape {np.shape(self.values)}")
        if not np.all(np.isfinite(v)):
            raise ValueError("image contains non-finite entries")
        object.__setattr__(self, "values", v)

    @classmethod
    def from_grid(cls, arr) -> "Image":
        arr = np.asarray(arr)
        return cls(GridShape(tuple(arr.shape)), arr.ravel())

    @property
    def grid(self) -> np.ndarray:
        return self.values.reshape(self.shape.dims)


@dataclass(frozen=True)
class Trajectory:
    """k-space samples in cycles/FOV, one row per sample (linops.py:103-140)."""

    points: np.ndarray
    kind: str

    def __post_init__(self):
        pts = np.atleast_2d(np.asarray(self.points, dtype=np.float64))
        object.__setattr__(self, "points", pts)
        if pts.ndim != 2 or pts.shape[0] < 1:
            raise ValueError("trajectory needs at least one point")
        if not np.all(np.isfinite(pts)):
            raise ValueError("trajectory contains non-finite coordinates")
        if self.kind not in ("cartesian-mask", "non-cartesian"):
            raise ValueError(f"unknown trajectory kind {self.kind!r}")
        if self.kind == "cartesian-mask" and not np.all(pts == np.round(pts)):
            raise ValueError("cartesian-mask trajectories must have integer coordinates")

    @property
    def n_points(self) -> int:
        return self.points.shape[0]

    @property
    def ndim(self) -> int:
        return self.points.shape[1]

    def validate_for(self, shape: GridShape) -> None:
        if self.ndim != shape.ndim:
            raise ValueError(f"trajectory is {self.ndim}-D but grid is {shape.ndim}-D")
        for a, n in enumerate(shape.dims):
            col = self.points[:, a]
            if col.min() < -n / 2 or col.max() >= n / 2:
                raise ValueError(f"trajectory axis {a} coordinates outside [{-n / 2}, {n / 2}) "
                                 f"for grid {shape.dims}")


class CostCounter:
    """Tagged application tallies with nestable pause (linops.py:147-178)."""

    def __init__(self):
        self._counts: dict[str, int] = {}
        self._pause_depth = 0

    def add(self, tag: str, n: int = 1) -> None:
        if self._pause_depth == 0:
            self._counts[tag] = self._counts.get(tag, 0) + int(n)

    def value(self, tag: str) -> int:
        return self._counts.get(tag, 0)

    def asdict(self) -> dict[str, int]:
        return dict(self._counts)

    def reset(self) -> None:
        self._counts.clear()

    @contextlib.contextmanager
    def paused(self):
        self._pause_depth += 1
        try:
            yield
        finally:
            self._pause_depth -= 1


class LinOp:
    """C^in -> C^out with exact adjoint, on the device (linops.py:185-244)."""

    def __init__(self, in_dim: int, out_dim: int, counter: CostCounter | None = None):
        self.in_dim = int(in_dim)
        self.out_dim = int(out_dim)
        self.counter = counter if counter is not None else CostCounter()

    # subclasses implement on (dim,) complex64 CUDA tensors
    def _forward(self, x: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError

    def _adjoint(self, y: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError

    @staticmethod
    def _io(v, dim: int, fn):
        if isinstance(v, torch.Tensor):
            if tuple(v.shape) != (dim,):
                raise ValueError(f"expected input of shape ({dim},), got {tuple(v.shape)}")
            return fn(dv.c64(v))
        v = np.ascontiguousarray(v, dtype=np.complex128)
        if v.shape != (dim,):
            raise ValueError(f"expected input of shape ({dim},), got {v.shape}")
        return dv.to_numpy128(fn(dv.c64(v)))

    def forward(self, x):
        return self._io(x, self.in_dim, self._forward)

    def adjoint(self, y):
        return self._io(y, self.out_dim, self._adjoint)

    def normal(self, x):
        return self.adjoint(self.forward(x))

    def _counters(self):
        return (self.counter,)

    @property
    def counts(self) -> dict[str, int]:
        merged: dict[str, int] = {}
        for c in {id(c): c for c in self._counters()}.values():
            for tag, n in c.asdict().items():
                merged[tag] = merged.get(tag, 0) + n
        return merged

    def reset_counts(self) -> None:
        for c in {id(c): c for c in self._counters()}.values():
            c.reset()

    @contextlib.contextmanager
    def paused_counts(self):
        with contextlib.ExitStack() as stack:
            for c in {id(c): c for c in self._counters()}.values():
                stack.enter_context(c.paused())
            yield

    def __matmul__(self, other: "LinOp") -> "ComposeOp":
        return ComposeOp(self, other)


class IdentityOp(LinOp):
    def __init__(self, dim: int):
        super().__init__(dim, dim)

    def _forward(self, x):
        return x.clone()

    def _adjoint(self, y):
        return y.clone()


class DiagonalOp(LinOp):
    """Pointwise multiplication by a fixed vector (linops.py:258-272)."""

    def __init__(self, diag, counter: CostCounter | None = None):
        d = np.ascontiguousarray(diag, dtype=np.complex128)
        if d.ndim != 1:
            raise ValueError("diagonal must be a flat vector")
        super().__init__(d.size, d.size, counter)
        self.diag = d
        self._d = dv.c64(d)

    def _forward(self, x):
        return self._d * x

    def _adjoint(self, y):
        return torch.conj(self._d) * y


class ComposeOp(LinOp):
    """outer @ inner (linops.py:275-294)."""

    def __init__(self, outer: LinOp, inner: LinOp):
        if inner.out_dim != outer.in_dim:
            raise ValueError(f"cannot compose: inner out_dim {inner.out_dim} != outer in_dim {outer.in_dim}")
        super().__init__(inner.in_dim, outer.out_dim)
        self.outer, self.inner = outer, inner

    def _forward(self, x):
        return self.outer._forward(self.inner._forward(x))

    def _adjoint(self, y):
        return self.inner._adjoint(self.outer._adjoint(y))

    def _counters(self):
        return self.outer._counters() + self.inner._counters() + (self.counter,)


class CartesianMaskOp(LinOp):
    """Centered unitary FFT sampled at integer bins, one coil (linops.py:534-549)."""

    def __init__(self, shape: GridShape, traj: Trajectory, counter: CostCounter | None = None):
        from .cartesian import CartesianKernel
        if traj.kind != "cartesian-mask":
            raise ValueError("Cartesian kernel needs a cartesian-mask trajectory")
        traj.validate_for(shape)
        self.kernel = CartesianKernel.from_points(shape.dims, traj.points)
        super().__init__(shape.size, traj.n_points, counter)
        self.shape = shape
        self._ones = torch.ones(1, 1, shape.size, dtype=torch.complex64, device=self.kernel.device)

    def _forward(self, x):
        self.counter.add("fourier")
        return self.kernel.forward(self._ones, x.view(1, -1))[0, 0, : self.out_dim].clone()

    def _adjoint(self, y):
        self.counter.add("fourier")
        out = torch.empty(1, self.in_dim, dtype=torch.complex64, device=y.device)
        return self.kernel.adjoint(self._ones, y.view(1, 1, -1), out)[0]


class CenteredFFTOp(CartesianMaskOp):
    """Unitary DC-centered FFT over the full grid (linops.py:316-329)."""

    def __init__(self, shape: GridShape, counter: CostCounter | None = None):
        axes = [np.arange(n) - n // 2 for n in shape.dims]
        pts = np.stack([m.ravel() for m in np.meshgrid(*axes, indexing="ij")], axis=1)
        super().__init__(shape, Trajectory(pts, "cartesian-mask"), counter)


class WaveletOp(LinOp):
    """Multilevel orthogonal DB4, periodic, in-place [lo|hi] layout (linops.py:654-702)."""

    def __init__(self, shape: GridShape, levels: int | None = None, counter: CostCounter | None = None):
        super().__init__(shape.size, shape.size, counter)
        self.shape = shape
        self.engine = WaveletEngine(shape.dims, levels, batch=1)
        self.levels = self.engine.levels

    def _forward(self, x):
        self.counter.add("wavelet")
        out = torch.empty(1, self.in_dim, dtype=torch.complex64, device=x.device)
        return self.engine.forward(x.view(1, -1).contiguous(), out)[0]

    def _adjoint(self, y):
        self.counter.add("wavelet")
        out = torch.empty(1, self.in_dim, dtype=torch.complex64, device=y.device)
        return self.engine.adjoint(y.view(1, -1).contiguous(), out)[0]


class FiniteDiffOp(LinOp):
    """Per-axis circular forward differences stacked over axes, D -> ndim*D (linops.py:717-738),
    on the device (csrc/tv.cu)."""

    def __init__(self, shape: GridShape, counter: CostCounter | None = None):
        super().__init__(shape.size, shape.ndim * shape.size, counter)
        self.shape = shape
        self._dims = (ctypes.c_int * shape.ndim)(*shape.dims)

    def _forward(self, x):
        self.counter.add("finite_diff")
        out = torch.empty(self.out_dim, dtype=torch.complex64, device=x.device)
        _lib.call("sr_tv_dual", dv.ptr(out), dv.ptr(x), self._dims, self.shape.ndim, 1, None, 0.0, 1, dv.stream())
        return out

    def _adjoint(self, y):
        self.counter.add("finite_diff")
        out = torch.empty(self.in_dim, dtype=torch.complex64, device=y.device)
        zero = torch.zeros(self.in_dim, dtype=torch.complex64, device=y.device)
        tau = torch.full((1,), -1.0, dtype=torch.float32, device=y.device)  # out = 0 - (-1) D^H y
        _lib.call("sr_tv_primal", dv.ptr(out), dv.ptr(zero), dv.ptr(y), self._dims, self.shape.ndim, dv.ptr(tau), 1,
                  dv.stream())
        return out


def make_fourier_kernel(shape: GridShape, traj: Trajectory, method: str = "auto",
                        oversamp: float = 1.25, width: int = 6):
    """Pick the device Fourier kernel (linops.py:519-531).

    Cartesian masks -> CartesianKernel; non-Cartesian -> Kaiser-Bessel gridding
    (`oversamp`/`width` are exposed here, where the reference hard-codes 1.25/6).
    """
    if traj.kind == "cartesian-mask":
        from .cartesian import CartesianKernel
        traj.validate_for(shape)
        return CartesianKernel.from_points(shape.dims, traj.points)
    if method in ("auto", "gridded"):
        from .nufft import GriddedKernel
        traj.validate_for(shape)
        return GriddedKernel(shape.dims, traj.points, oversamp, width)
    if method == "direct":
        raise ValueError("the direct O(N D) NUDFT is oracle-only (oracle/sketch_oracle.py)")
    raise ValueError(f"unknown NUFFT method {method!r}")


def max_eig_power(op: LinOp, iters: int = 30, seed: int = 0) -> float:
    """Power iteration on a self-adjoint PSD operator (linops.py:766-782)."""
    if op.in_dim != op.out_dim:
        raise ValueError("power iteration needs a square operator")
    g = seed_stream(seed, 0)
    v0 = g.standard_normal(op.in_dim) + 1j * g.standard_normal(op.in_dim)
    v = dv.c64(v0 / np.linalg.norm(v0))
    lam = 0.0
    with op.paused_counts():
        for _ in range(int(iters)):
            w = op._forward(v)
            nw = float(torch.linalg.vector_norm(w.to(torch.complex128)))
            if nw == 0.0:
                return 0.0
            lam = float(torch.real(torch.vdot(v.to(torch.complex128), w.to(torch.complex128))))
            v = (w / nw).to(torch.complex64)
    return lam


def dot_test(op: LinOp, rng: np.random.Generator, trials: int = 10) -> float:
    """Max relative adjointness gap over random draws (linops.py:785-795)."""
    worst = 0.0
    for _ in range(trials):
        u = rng.standard_normal(op.in_dim) + 1j * rng.standard_normal(op.in_dim)
        v = rng.standard_normal(op.out_dim) + 1j * rng.standard_normal(op.out_dim)
        lhs = np.vdot(v, op.forward(u))
        rhs = np.vdot(op.adjoint(v), u)
        worst = max(worst, abs(lhs - rhs) / (np.linalg.norm(u) * np.linalg.norm(v)))
    return worst
