"""Adapter for duck-typed host Fourier kernels.

The reference's SenseOperator accepts any object with ``n_points`` and host
``apply((C, D)) -> (C, N)`` / ``apply_adjoint((C, N)) -> (C, D)``
(/root/reference/pkg/src/sketchrecon/forward_model.py:134, 147-148).  The device
operator and engine call batched device entry points (``normal`` / ``forward`` /
``adjoint`` on complex64 CUDA tensors); this adapter provides them for such a
user kernel: the coil images are formed on the device, moved to the host for the
user's transform, and the coil-conjugate sum / solver epilogue run on the device
again.  It exists for API parity with third-party kernels, not for speed: the
repository's own kernels (CartesianKernel, Cartesian3DKernel, GriddedKernel) never
take this path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dv


class HostKernelAdapter:
    def __init__(self, kernel, D: int, device=None):
        if not (hasattr(kernel, "apply") and hasattr(kernel, "apply_adjoint") and hasattr(kernel, "n_points")):
            raise TypeError("kernel must provide n_points, apply and apply_adjoint")
        self.host = kernel
        self.D = int(D)
        self.n_points = int(kernel.n_points)
        self.nmax = self.n_points
        self.batch = 1
        self.device = device or dv.require_cuda()
        # the user's transform runs on the host: the engine cannot capture it in a CUDA graph
        self.graph_capturable = False

    # engine / operator protocol ------------------------------------------------
    def workspace(self, ncoils: int, batch: int | None = None, chunk: int = 0, normal: bool = True):
        return None

    def partial_shape(self, ncoils: int) -> tuple:
        return (1, 1)

    def _check(self, maps):
        if maps.dim() != 3 or maps.shape[0] != 1 or maps.shape[2] != self.D:
            raise ValueError(f"maps must be (1, C, {self.D})")
        return maps.shape[1]

    def _fwd_host(self, maps, x, w):
        imgs = dv.to_numpy128(maps[0] * x.reshape(1, self.D))
        k = np.asarray(self.host.apply(imgs), dtype=np.complex128).reshape(maps.shape[1], self.n_points)
        kd = dv.c64(k, self.device)
        if w is not None:
            kd = kd * w.to(kd.device, torch.float32).view(1, -1)
        return kd

    def _adj_host(self, maps, y, w, out, coef=None, u=None, d=None):
        k = y.reshape(maps.shape[1], -1)[:, : self.n_points]
        if w is not None:
            k = k * w.to(k.device, torch.float32).view(1, -1)
        imgs = np.asarray(self.host.apply_adjoint(dv.to_numpy128(k)), dtype=np.complex128)
        acc = (torch.conj(maps[0]) * dv.c64(imgs.reshape(maps.shape[1], self.D), self.device)).sum(dim=0)
        return self._epilogue(acc.view(1, -1), out, coef, u, d)

    @staticmethod
    def _epilogue(acc, out, coef, u, d):
        """out = s_acc acc + s_u u + s_d d with coef[b] = {s_acc, s_u, s_d, -} (sr_cart_normal)."""
        if coef is None:
            out.copy_(acc)
            return out
        c = coef.to(torch.float32).view(-1, 4)
        r = c[:, 0:1] * acc
        if u is not None:
            r = r + c[:, 1:2] * u
        if d is not None:
            r = r + c[:, 2:3] * d
        out.copy_(r)
        return out

    def normal(self, maps, x, out, *, anchor=None, coef=None, u=None, d=None, w=None, chunk=None):
        self._check(maps)
        xv = x if anchor is None else x - anchor
        k = self._fwd_host(maps, xv, w)
        return self._adj_host(maps, k, w, out, coef, u, d)

    def forward(self, maps, x, y=None, *, ymeas=None, partial=None, partial_blocks=None, w=None):
        C = self._check(maps)
        k = self._fwd_host(maps, x, w)
        if y is None:
            y = torch.zeros(1, C, self.n_points, dtype=torch.complex64, device=self.device)
        if ymeas is not None:
            k = k - ymeas.reshape(C, -1)[:, : self.n_points]
        y.view(C, -1)[:, : self.n_points].copy_(k)
        if partial is not None:
            partial.zero_()
            if ymeas is not None:
                partial.view(-1)[0] = float(torch.sum(torch.abs(k.to(torch.complex128)) ** 2))
        return y

    def adjoint(self, maps, y, out, *, coef=None, u=None, d=None, w=None):
        self._check(maps)
        return self._adj_host(maps, y, w, out, coef, u, d)

    # reference plugin protocol -------------------------------------------------
    def apply(self, batch):
        return self.host.apply(batch)

    def apply_adjoint(self, batch):
        return self.host.apply_adjoint(batch)
