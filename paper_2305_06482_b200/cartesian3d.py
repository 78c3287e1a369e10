"""3-D Cartesian mask kernel on the device.

Drop-in for the reference plugin ``_CartesianMaskKernel`` on a 3-D grid
(/root/reference/pkg/src/sketchrecon/linops.py:332-364), which accepts a mask of any
dimensionality; the 2-D K1/K2 kernels (cartesian.py) cover 1-D and 2-D grids.  The
operator runs the per-axis grid pipeline of the gridded NUFFT (csrc/nufft.cu) with an
oversampled grid equal to the image grid and unit apodisation: the embed places pixel r
at index r mod n (the reference's ifftshift), the axis FFTs leave axes 0 and 1 in perm order
and axis 2 in natural order, and the sample at centered bin f sits at
perm(f_0) n_1 n_2 + perm(f_1) n_2 + f_2 (all mod n_a), so
no centering phase is needed.  The normal op multiplies the spectrum by the sampled-bin
indicator / D between the forward and the inverse passes.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .plan import perm_positions


class Cartesian3DKernel:
    """Device tables of one 3-D Cartesian sampling pattern (B = 1, coils batched)."""

    def __init__(self, dims, points):
        self.dims = tuple(int(n) for n in dims)
        if len(self.dims) != 3:
            raise ValueError("Cartesian3DKernel needs a 3-D grid")
        for n in self.dims:
            if n > 1 and not _lib.lib().sr_fft_size_supported(n):
                raise ValueError(f"grid axis {n} has no sm_100a FFT instantiation")
        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != 3:
            raise ValueError("trajectory dimensionality does not match the grid")
        for a, n in enumerate(self.dims):
            if pts.size and (pts[:, a].min() < -n / 2 or pts[:, a].max() >= n / 2):
                raise ValueError(f"trajectory axis {a} coordinates outside [{-n / 2}, {n / 2}) for grid {self.dims}")
        self.batch = 1
        self.D = int(np.prod(self.dims))
        self.n_points = int(pts.shape[0])
        self.nmax = self.n_points
        # reference bin (linops.py:341): idx = (points + n//2).astype(intp), i.e. f = idx - n//2
        idx = (pts + np.array([n // 2 for n in self.dims])).astype(np.int64)
        f = idx - np.array([n // 2 for n in self.dims])
        n0, n1, n2 = self.dims
        pos = []
        for a, n in enumerate(self.dims):
            if a == 2:  # the grid pipeline keeps the contiguous axis in natural order
                pos.append(np.mod(f[:, a], n))
                continue
            pp = perm_positions(n) if n > 1 else np.zeros(1, dtype=np.int64)
            pos.append(pp[np.mod(f[:, a], n)])
        spos = (pos[0] * n1 * n2 + pos[1] * n2 + pos[2]).astype(np.int64)
        mask = np.zeros(self.D, dtype=np.uint8)
        mask[spos] = 1
        rev = spos[::-1]
        _, first_in_rev = np.unique(rev, return_index=True)
        wlist = np.sort(len(spos) - 1 - first_in_rev).astype(np.int32)
        dev = dv.require_cuda()
        self.device = dev
        self.spos = dv.host_to_dev(spos.astype(np.int32), torch.int32, dev)
        self.mask = dv.host_to_dev(mask, torch.uint8, dev)
        self.wlist = dv.host_to_dev(wlist, torch.int32, dev)
        self.nw = int(wlist.size)
        self._ones = [torch.ones(n, dtype=torch.float32, device=dev) for n in self.dims]
        self._dims_h = (ctypes.c_int * 3)(*self.dims)
        self._grids = None
        self.nparts = int(_lib.lib().sr_cart3_partial_blocks(self.n_points, 64))

    def workspace(self, ncoils: int, batch: int | None = None, chunk: int = 0, normal: bool = True):
        need = ncoils * self.D
        if self._grids is None or self._grids.numel() < need:
            self._grids = torch.empty(need, dtype=torch.complex64, device=self.device)
        return self._grids

    def partial_shape(self, ncoils: int) -> tuple:
        return (1, int(_lib.lib().sr_cart3_partial_blocks(self.n_points, max(1, ncoils))))

    def _maps(self, maps):
        if maps.dim() != 3 or maps.shape[0] != 1 or maps.shape[2] != self.D:
            raise ValueError(f"maps must be (1, C, {self.D})")
        return maps.shape[1]

    def _ones_ptrs(self):
        return tuple(dv.ptr(o) for o in self._ones)

    def normal(self, maps, x, out, *, anchor=None, coef=None, u=None, d=None, w=None, chunk=None):
        if w is not None:
            raise ValueError("density weights are not used with Cartesian masks")
        C = self._maps(maps)
        grids = self.workspace(C)
        _lib.call("sr_cart3_normal", dv.ptr(x), dv.ptr(anchor), dv.ptr(maps), C, self._dims_h, *self._ones_ptrs(),
                  dv.ptr(self.mask), dv.ptr(out), dv.ptr(grids), dv.ptr(coef), dv.ptr(u), dv.ptr(d), dv.stream())
        return out

    def forward(self, maps, x, y=None, *, ymeas=None, partial=None, partial_blocks=None, w=None):
        if w is not None:
            raise ValueError("density weights are not used with Cartesian masks")
        C = self._maps(maps)
        if y is None:
            y = torch.zeros(1, C, self.n_points, dtype=torch.complex64, device=self.device)
        if partial is not None and partial.numel() < _lib.lib().sr_cart3_partial_blocks(self.n_points, C):
            raise ValueError("partial buffer too small")
        grids = self.workspace(C)
        _lib.call("sr_cart3_forward", dv.ptr(x), dv.ptr(maps), C, self._dims_h, *self._ones_ptrs(),
                  dv.ptr(self.spos), self.n_points, dv.ptr(y), y.shape[-1], dv.ptr(ymeas), dv.ptr(partial),
                  dv.ptr(grids), dv.stream())
        return y

    def adjoint(self, maps, y, out, *, coef=None, u=None, d=None, w=None):
        if w is not None:
            raise ValueError("density weights are not used with Cartesian masks")
        C = self._maps(maps)
        if y.dim() != 3 or y.shape[1] != C or y.shape[2] < self.n_points:
            raise ValueError("y must be (1, C, >= n_points)")
        grids = self.workspace(C)
        _lib.call("sr_cart3_adjoint", dv.ptr(y), y.shape[-1], dv.ptr(maps), C, self._dims_h, *self._ones_ptrs(),
                  dv.ptr(self.spos), dv.ptr(self.wlist), self.nw, dv.ptr(out), dv.ptr(grids), dv.ptr(coef),
                  dv.ptr(u), dv.ptr(d), dv.stream())
        return out

    # ------------------------------------------------- reference plugin protocol
    def apply(self, batch: np.ndarray) -> np.ndarray:
        """(C, D) coil images -> (C, N) samples (linops.py:344-352)."""
        b = dv.c64(np.asarray(batch).reshape(-1, self.D))
        ones = torch.ones(1, self.D, dtype=torch.complex64, device=self.device)
        y = self.forward(b.unsqueeze(0).contiguous(), ones)
        return dv.to_numpy128(y[0])

    def apply_adjoint(self, batch: np.ndarray) -> np.ndarray:
        """(C, N) samples -> (C, D) coil images (linops.py:354-364)."""
        b = dv.c64(np.asarray(batch).reshape(-1, self.n_points))
        ones = torch.ones(1, 1, self.D, dtype=torch.complex64, device=self.device)
        outs = []
        for c in range(b.shape[0]):
            out = torch.empty(1, self.D, dtype=torch.complex64, device=self.device)
            self.adjoint(ones, b[c].reshape(1, 1, -1).contiguous(), out)
            outs.append(out[0])
        return dv.to_numpy128(torch.stack(outs))
