"""Host-side layout planning for the Cartesian kernels (pure NumPy, no GPU).

The kernels keep spectra in "perm order": an axis of length n = P*Q (split
queried from the native library) stores frequency k at P*(k % Q) + k // Q,
the natural output order of the two-level in-register FFT (csrc/fft2step.cuh).
This module turns a reference-style integer trajectory
(``Trajectory.points``, centered bins in [-n/2, n/2), linops.py:103-140) into
the index/phase tables the kernels consume:

* ``spos``  - offset of each sample in the perm-order (ny, nx) spectrum
* ``ph``    - per-sample centering phase exp(2 pi i (n//2) f / n) per axis, which
              replaces the ifftshift/fftshift pair of linops.py:348-351
* ``maskT`` - the sampled-bin indicator, transposed [pos_x][pos_y]
* ``wlist`` - sample indices written by the adjoint scatter: for duplicated
              bins only the LAST occurrence, as numpy fancy assignment
              (linops.py:357) keeps the last value.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


def perm_positions(n: int) -> np.ndarray:
    """pos[k] for frequency index k in [0, n)."""
    p, q = _lib.fft_split(n)
    k = np.arange(n, dtype=np.int64)
    return p * (k % q) + k // q


def grid2d(dims: tuple[int, ...]) -> tuple[int, int]:
    """(ny, nx) of the kernels for a 1-D or 2-D reference grid."""
    if len(dims) == 1:
        return 1, int(dims[0])
    if len(dims) == 2:
        return int(dims[0]), int(dims[1])
    raise NotImplementedError("the 2-D Cartesian kernels take 1-D/2-D grids; 3-D grids use Cartesian3DKernel")


@dataclass(frozen=True)
class CartesianPlan:
    ny: int
    nx: int
    n_points: int
    spos: np.ndarray   # (N,) int32
    ph: np.ndarray     # (N,) complex64
    maskT: np.ndarray  # (nx*ny,) uint8, [pos_x][pos_y]
    wlist: np.ndarray  # (Nw,) int32

    @property
    def D(self) -> int:
        return self.ny * self.nx


def cartesian_plan(dims: tuple[int, ...], points: np.ndarray) -> CartesianPlan:
    ny, nx = grid2d(dims)
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != len(dims):
        raise ValueError("trajectory dimensionality does not match the grid")
    f = np.rint(pts).astype(np.int64)
    if len(dims) == 1:
        fy = np.zeros(f.shape[0], dtype=np.int64)
        fx = f[:, 0]
    else:
        fy, fx = f[:, 0], f[:, 1]
    ky, kx = np.mod(fy, ny), np.mod(fx, nx)
    py = perm_positions(ny) if ny > 1 else np.zeros(1, dtype=np.int64)
    px = perm_positions(nx)
    pos_y, pos_x = py[ky], px[kx]
    spos = (pos_y * nx + pos_x).astype(np.int32)
    # exp(2 pi i (n//2) f / n) per axis, evaluated on f mod n in float64
    ang = 2.0 * np.pi * ((ny // 2) * ky / ny + (nx // 2) * kx / nx)
    ang = np.mod(ang, 2.0 * np.pi)
    ph = np.exp(1j * ang).astype(np.complex64)
    maskT = np.zeros(nx * ny, dtype=np.uint8)
    maskT[pos_x * ny + pos_y] = 1
    # last occurrence of every distinct bin: a stable sort by bin (radix sort on int32) keeps the
    # samples of a bin in trajectory order, so the last of each run is the last occurrence
    order = np.argsort(spos, kind="stable").astype(np.int32)
    s = spos[order]
    last = np.ones(len(s), dtype=bool)
    last[:-1] = s[1:] != s[:-1]
    wlist = np.sort(order[last], kind="stable").astype(np.int32)
    return CartesianPlan(ny, nx, int(pts.shape[0]), spos, ph, maskT, wlist)


def to_perm_spectrum(spec: np.ndarray, ny: int, nx: int) -> np.ndarray:
    """Reorder a natural-order (.., ny, nx) spectrum into perm order (test helper)."""
    out = np.empty_like(spec)
    py = perm_positions(ny) if ny > 1 else np.zeros(1, dtype=np.int64)
    px = perm_positions(nx)
    out[..., py[:, None], px[None, :]] = spec
    return out
