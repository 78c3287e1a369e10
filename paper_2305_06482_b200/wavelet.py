"""Device Daubechies-4 wavelet engine (K6): analysis, synthesis, fused L1 prox.

Reference: WaveletOp (linops.py:654-702), default_wavelet_levels
(linops.py:609-616), Regularizer.prox / value (solvers.py:61-81), prox_l1
(solvers.py:129-135).  2-D grids use the tiled one-launch-per-level kernels
(csrc/wavelet.cu); 1-D and 3-D grids (config 4 volume) one launch per axis and
level (csrc/wavelet_nd.cu).
"""

from __future__ import annotations

import math

import torch

from . import _device as dv
from . import _lib


def default_wavelet_levels(dims, cap: int = 4) -> int:
    """Largest level count <= cap with every dim halvable (linops.py:609-616)."""
    levels, d = 0, [int(n) for n in dims]
    while levels < cap and all(n % 2 == 0 and n // 2 >= 1 for n in d):
        d = [n // 2 for n in d]
        levels += 1
    return levels


def np_prod(dims) -> int:
    return int(math.prod(int(n) for n in dims))


class WaveletEngine:
    """Batched (B, ny, nx) multilevel DB4 on the device."""

    def __init__(self, dims, levels: int | None = None, batch: int = 1):
        dims = tuple(int(n) for n in dims)
        if not 1 <= len(dims) <= 3:
            raise ValueError("grid must have 1-3 axes")
        if levels is None:
            levels = default_wavelet_levels(dims)
        levels = int(levels)
        if levels < 1:
            raise ValueError("levels must be >= 1")
        for n in dims:
            if n % (1 << levels) != 0:
                raise ValueError(f"grid dims {dims} not divisible by 2^{levels}")
        self.dims, self.levels, self.batch = dims, levels, int(batch)
        self.generic = len(dims) != 2
        self.dims3 = (1,) * (3 - len(dims)) + dims
        self.axes = list(range(3 - len(dims), 3))
        self.ny, self.nx = (self.dims3[0] * self.dims3[1], self.dims3[2])
        self.D = int(np_prod(dims))
        self.device = dv.require_cuda()
        self.buf = [torch.empty(self.batch, self.D, dtype=torch.complex64, device=self.device)
                    for _ in range(2)]
        if self.generic:
            self.tmp = [torch.empty(self.batch, self.D, dtype=torch.complex64, device=self.device)
                        for _ in range(2)]
            self.nblocks = [_lib.lib().sr_wavelet_axis_nblocks()] * levels
        else:
            self.nblocks = [_lib.lib().sr_wavelet_ana2_nblocks(self.ny >> l, self.nx >> l)
                            for l in range(levels)]
        # one contiguous (B, nblocks_l) partial-sum buffer per level (the kernel indexes b * nblocks + blk)
        self.l1parts = [torch.zeros(self.batch, nb, dtype=torch.float64, device=self.device)
                        for nb in self.nblocks]

    def _region(self, l):
        return self.ny >> l, self.nx >> l

    def _region3(self, l):
        return tuple((n >> l) if a in self.axes else 1 for a, n in enumerate(self.dims3))

    def _ana(self, src, dst, l, thresh=None, hthresh=-1.0, l1=None):
        if self.generic:
            return self._ana_axes(src, dst, l, thresh, hthresh, l1)
        h, w = self._region(l)
        _lib.call("sr_wavelet_ana2", dv.ptr(src), dv.ptr(dst), h, w, self.nx, self.D, self.batch,
                  dv.ptr(thresh), float(hthresh), int(l == self.levels - 1), dv.ptr(l1), dv.stream())

    def _syn(self, src, dst, l, zout=None, xold=None, beta=0.0):
        if self.generic:
            return self._syn_axes(src, dst, l, zout, xold, beta)
        h, w = self._region(l)
        _lib.call("sr_wavelet_syn2", dv.ptr(src), dv.ptr(dst), h, w, self.nx, self.D, self.batch,
                  dv.ptr(zout), dv.ptr(xold), float(beta), dv.stream())

    def _ana_axes(self, src, dst, l, thresh, hthresh, l1):
        """Axes 0..d-1 of level l (linops.py:683-685), threshold on the last axis."""
        h = self._region3(l)
        cur = src
        for i, ax in enumerate(self.axes):
            last = i == len(self.axes) - 1
            out = dst if last else self.tmp[i % 2]
            _lib.call("sr_wavelet_axis", dv.ptr(cur), dv.ptr(out), h[0], h[1], h[2], self.dims3[1],
                      self.dims3[2], self.D, self.batch, ax, 0, dv.ptr(thresh) if last else None,
                      float(hthresh) if last else -1.0, int(last), int(l == self.levels - 1),
                      dv.ptr(l1) if last else None, None, None, 0.0, dv.stream())
            cur = out

    def _syn_axes(self, src, dst, l, zout, xold, beta):
        """Axes d-1..0 of level l (linops.py:699-700), momentum epilogue on the last launch."""
        h = self._region3(l)
        cur = src
        axes = list(reversed(self.axes))
        for i, ax in enumerate(axes):
            last = i == len(axes) - 1
            out = dst if last else self.tmp[i % 2]
            _lib.call("sr_wavelet_axis", dv.ptr(cur), dv.ptr(out), h[0], h[1], h[2], self.dims3[1],
                      self.dims3[2], self.D, self.batch, ax, 1, None, -1.0, 0, 0, None,
                      dv.ptr(zout) if last else None, dv.ptr(xold) if last else None, float(beta),
                      dv.stream())
            cur = out


    # ------------------------------------------------------------- hot path
    def prox(self, v, out, thresh=None, hthresh=-1.0, zout=None, xold=None, beta=0.0):
        """out = Psi^H soft(Psi v, t); optional z = out + beta (out - xold).

        thresh: device (B,) float32 thresholds or None with host `hthresh`.
        v must not alias out, self.buf.  out may alias xold.
        """
        if not self.generic:  # 2-D: every level's launches from one C call (sr_wavelet_prox2)
            _lib.call("sr_wavelet_prox2", dv.ptr(v), dv.ptr(out), dv.ptr(self.buf[0]), dv.ptr(self.buf[1]),
                      self.ny, self.nx, self.D, self.batch, self.levels, dv.ptr(thresh), float(hthresh),
                      dv.ptr(zout), dv.ptr(xold), float(beta), dv.stream())
            return out
        src = v
        for l in range(self.levels):
            dst = self.buf[l % 2]
            self._ana(src, dst, l, thresh, hthresh)
            src = dst
        for l in range(self.levels - 1, -1, -1):
            dst = out if l == 0 else self.buf[(l - 1) % 2]
            if l == 0:
                self._syn(self.buf[0], dst, 0, zout, xold, beta)
            else:
                self._syn(self.buf[l % 2], dst, l)
        return out

    def l1_norm(self, x, out=None, tmp=None) -> torch.Tensor:
        """sum |Psi x| per slice as a (B,) float64 device tensor (no host sync).  With `out` and `tmp`
        ((B,) float64) nothing is allocated: the per-level block sums are added in level order, as
        the generator sum does."""
        src = x
        for l in range(self.levels):
            dst = self.buf[l % 2]
            self._ana(src, dst, l, None, -1.0, self.l1parts[l])
            src = dst
        if out is None:
            return sum(p.sum(dim=1) for p in self.l1parts)
        torch.sum(self.l1parts[0], dim=1, out=out)
        for p in self.l1parts[1:]:
            out.add_(torch.sum(p, dim=1, out=tmp))
        return out

    # ------------------------------------------------- reference-layout API
    def _corner(self, t, l):
        h = self._region3(l)
        return t.view((self.batch,) + self.dims3)[:, : h[0], : h[1], : h[2]]

    def forward(self, x, out):
        """Coefficients in the reference in-place [lo|hi] layout (linops.py:677-687)."""
        self._ana(x, out, 0)
        tmp = self.buf[0]
        for l in range(1, self.levels):
            self._ana(out, tmp, l)
            self._corner(out, l).copy_(self._corner(tmp, l))
        return out

    def adjoint(self, c, out):
        """Inverse/adjoint (linops.py:689-702)."""
        work = self.buf[1]
        work.copy_(c)
        tmp = self.buf[0]
        for l in range(self.levels - 1, 0, -1):
            self._syn(work, tmp, l)
            self._corner(work, l).copy_(self._corner(tmp, l))
        self._syn(work, out, 0)
        return out
