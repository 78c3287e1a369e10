"""Cartesian Fourier kernel on the device (K1 normal op, K2 forward/adjoint).

Drop-in for the reference plugin ``_CartesianMaskKernel``
(/root/reference/pkg/src/sketchrecon/linops.py:332-364): it exposes the same
``n_points`` / ``apply`` / ``apply_adjoint`` protocol (host numpy, used when it
is plugged into a reference ``SenseOperator``) and, for the performance path,
batched device entry points that fuse the map multiply, both FFT passes, the
mask and the conjugate coil sum (``normal``), plus ``forward``/``adjoint``
with compact samples in trajectory order.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .plan import CartesianPlan, cartesian_plan, grid2d


def _no_weights(w):
    if w is not None:
        raise ValueError("density weights are not used with Cartesian masks")


class CartesianKernel:
    """Device tables for B slices sharing one grid (one mask per slice or shared).

    ``plans`` holds one CartesianPlan per slice (len B) or a single shared plan.
    """

    def __init__(self, dims, plans: list[CartesianPlan], batch: int | None = None):
        self.dims = tuple(int(n) for n in dims)
        self.ny, self.nx = grid2d(self.dims)
        for n in (self.ny, self.nx):
            if n > 1 and not _lib.lib().sr_fft_size_supported(n):
                raise ValueError(f"grid axis {n} has no sm_100a FFT instantiation")
        self.D = self.ny * self.nx
        self.batch = int(batch if batch is not None else len(plans))
        if len(plans) not in (1, self.batch):
            raise ValueError("need one plan per slice or one shared plan")
        self.shared_mask = len(plans) == 1
        per_slice = plans if len(plans) == self.batch else plans * self.batch
        self.n_points_per_slice = [p.n_points for p in per_slice]
        self.n_points = per_slice[0].n_points
        self.nmax = max(self.n_points_per_slice)
        dev = dv.require_cuda()
        self.device = dev
        self.maskT = dv.host_to_dev(np.stack([p.maskT for p in plans]), torch.uint8, dev)
        self.mask_bstride = 0 if self.shared_mask else self.D
        self.spos = dv.host_to_dev(np.concatenate([p.spos for p in per_slice]), torch.int32, dev)
        self.ph = dv.c64(np.concatenate([p.ph for p in per_slice]), dev)
        soff = np.zeros(self.batch + 1, dtype=np.int64)
        soff[1:] = np.cumsum(self.n_points_per_slice)
        self.soff = dv.host_to_dev(soff, torch.int64, dev)
        self.wlist = dv.host_to_dev(np.concatenate([p.wlist for p in per_slice]), torch.int32, dev)
        woff = np.zeros(self.batch + 1, dtype=np.int64)
        woff[1:] = np.cumsum([len(p.wlist) for p in per_slice])
        self.woff = dv.host_to_dev(woff, torch.int64, dev)
        # per-column-block sample lists: K2 gathers / scatters inside the column pass
        cb = int(_lib.lib().sr_cart_col_block(self.ny))
        self.nblk = (self.nx + cb - 1) // cb if cb > 0 else 0
        self.fused_io = cb > 0
        if self.fused_io:
            g_idx, g_ptr, s_idx, s_ptr = [], [], [], []
            g_base = s_base = 0
            for p in per_slice:
                # small block ids (uint16): numpy's stable sort is a radix sort for them
                blk = ((p.spos.astype(np.int64) % self.nx) // cb).astype(np.uint16)
                order = np.argsort(blk, kind="stable").astype(np.int32)
                g_idx.append(order)
                g_ptr.append(g_base + np.r_[0, np.cumsum(np.bincount(blk, minlength=self.nblk))])
                g_base += len(order)
                wb = blk[p.wlist]
                worder = p.wlist[np.argsort(wb, kind="stable")].astype(np.int32)
                s_idx.append(worder)
                s_ptr.append(s_base + np.r_[0, np.cumsum(np.bincount(wb, minlength=self.nblk))])
                s_base += len(worder)
            self.g_idx = dv.host_to_dev(np.concatenate(g_idx), torch.int32, dev)
            self.g_ptr = dv.host_to_dev(np.stack(g_ptr), torch.int32, dev)
            self.s_idx = dv.host_to_dev(np.concatenate(s_idx), torch.int32, dev)
            self.s_ptr = dv.host_to_dev(np.stack(s_ptr), torch.int32, dev)
        self._ws = None
        self.chunk = 0  # sr_cart_normal schedule: 0 three launches, >0 chunked, -1 persistent fused
        self._plans = plans
        self._replicas: dict[int, "CartesianKernel"] = {}

    @classmethod
    def from_points(cls, dims, points):
        """Kernel for one trajectory; a 3-D grid gets the grid-pipeline Cartesian3DKernel."""
        if len(tuple(dims)) == 3:
            from .cartesian3d import Cartesian3DKernel
            return Cartesian3DKernel(dims, points)
        return cls(dims, [cartesian_plan(tuple(dims), points)])

    # ------------------------------------------------------------------ device
    def workspace(self, ncoils: int, batch: int | None = None, chunk: int = -1) -> torch.Tensor:
        """Coil workspace (complex64) large enough for sr_cart_normal(chunk) and the K2 passes."""
        nbytes = max(8 * (batch or self.batch) * ncoils * self.D,
                     _lib.lib().sr_cart_ws_bytes(self.batch, ncoils, self.ny, self.nx, chunk))
        need = (nbytes + 7) // 8
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.complex64, device=self.device)
        return self._ws

    def _maps_stride(self, maps: torch.Tensor) -> tuple[int, int]:
        if maps.dim() != 3 or maps.shape[2] != self.D or maps.shape[0] not in (1, self.batch):
            raise ValueError(f"maps must be (1 or {self.batch}, C, {self.D}), got {tuple(maps.shape)}")
        if maps.dtype != torch.complex64 or not maps.is_contiguous():
            raise ValueError("maps must be contiguous complex64")
        ncoils = maps.shape[1]
        return ncoils, (0 if maps.shape[0] == 1 else ncoils * self.D)

    def _check_img(self, t, name):
        if t is None:
            return
        if t.shape != (self.batch, self.D) or t.dtype != torch.complex64 or not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous complex64 ({self.batch}, {self.D})")

    def normal(self, maps, x, out, *, anchor=None, coef=None, u=None, d=None, w=None, chunk=None):
        """out = e(sum_j conj(c_j) F^H M F (c_j (x - anchor)))  (K1).

        chunk: None -> self.chunk; 0 -> three launches over the batch; > 0 -> three launches
        per group of `chunk` slices.
        """
        _no_weights(w)
        ncoils, mbs = self._maps_stride(maps)
        for t, n in ((x, "x"), (out, "out"), (anchor, "anchor"), (u, "u"), (d, "d")):
            self._check_img(t, n)
        chunk = self.chunk if chunk is None else int(chunk)
        ws = self.workspace(ncoils, chunk=chunk)
        _lib.call("sr_cart_normal", dv.ptr(x), dv.ptr(anchor), dv.ptr(maps), mbs,
                  dv.ptr(self.maskT), self.mask_bstride, dv.ptr(out), dv.ptr(ws), self.batch,
                  ncoils, self.ny, self.nx, dv.ptr(coef), dv.ptr(u), dv.ptr(d), chunk, dv.stream())
        return out

    def _normal_range(self, maps, x, out, b0: int, b1: int, ws, stream: int):
        """K1 over slices [b0, b1) of the batch (device pointers offset, three-launch schedule)."""
        ncoils, mbs = self._maps_stride(maps)
        item = 8  # bytes per complex64
        xo = b0 * self.D * item
        _lib.call("sr_cart_normal", dv.ptr(x) + xo, None, dv.ptr(maps) + b0 * mbs * item, mbs,
                  dv.ptr(self.maskT) + b0 * self.mask_bstride, self.mask_bstride, dv.ptr(out) + xo,
                  dv.ptr(ws), b1 - b0, ncoils, self.ny, self.nx, None, None, None, 0, stream)

    def normal_host(self, maps, x_host, out_host, *, chunks: int = 8, buffers=None, lanes: int = 1,
                    overlap_prev: bool = False, sync: bool = False):
        """A^H A on HOST (pinned) buffers, pipelined: slice chunks are copied in, applied and
        copied out so PCIe transfers overlap the K1 launches.  Chunk i runs its K1 on compute
        lane i % lanes (own stream and workspace), so two small-grid K1 launches share the GPU.

        x_host/out_host: pinned (B, D) complex64 CPU tensors.  The call is asynchronous: it returns
        out_host once the copies are enqueued and makes the current stream wait for them, so the
        caller must synchronise (``torch.cuda.current_stream().synchronize()``, or pass
        ``sync=True``) before reading out_host or rewriting x_host.
        `chunks` = number of equal chunks, or a sequence of slice counts summing to B (a small
        last chunk shortens the pipeline drain: its K1 + D2H are all that follow the last H2D).
        `buffers` = (x_dev, out_dev) device staging tensors to reuse across calls.
        `overlap_prev` = True lets this call's host-to-device copies start while the previous
        call's last chunks still compute (they wait only for the previous call's K1 events on
        the same staging buffers, not for the current stream).  Only valid when this kernel
        instance owns `buffers` exclusively: no other stream work may read or write them
        between calls.  Default False: the copies wait for the current stream.
        """
        import torch
        if x_host.device.type != "cpu" or out_host.device.type != "cpu":
            raise ValueError("normal_host takes host tensors")
        ncoils, _ = self._maps_stride(maps)
        B = self.batch
        if isinstance(chunks, (list, tuple)):
            sizes = [int(c) for c in chunks]
            if sum(sizes) != B or min(sizes) < 1:
                raise ValueError("chunk sizes must be positive and sum to the batch")
            edges = np.cumsum([0] + sizes)
            bounds = [(int(edges[i]), int(edges[i + 1])) for i in range(len(sizes))]
        else:
            nch = max(1, min(int(chunks), B))
            bounds = [(B * i // nch, B * (i + 1) // nch) for i in range(nch)]
        lanes = max(1, min(int(lanes), len(bounds)))
        if buffers is None:
            buffers = (torch.empty(B, self.D, dtype=torch.complex64, device=self.device),
                       torch.empty(B, self.D, dtype=torch.complex64, device=self.device))
        xd, od = buffers
        nb = max(b1 - b0 for b0, b1 in bounds)
        need = 8 * nb * ncoils * self.D
        if getattr(self, "_host_ws", None) is None or len(self._host_ws) < lanes or \
                self._host_ws[0].numel() * 8 < need:
            self._host_ws = [torch.empty((need + 7) // 8, dtype=torch.complex64, device=self.device)
                             for _ in range(lanes)]
        cur = torch.cuda.current_stream()
        if getattr(self, "_host_streams", None) is None or len(self._host_streams[2]) < lanes:
            self._host_streams = (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device),
                                  [torch.cuda.Stream(self.device) for _ in range(lanes)])
        s_in, s_out, s_k = self._host_streams
        for st in (s_out, *s_k[:lanes]):
            st.wait_stream(cur)
        # The host-to-device copies depend on no device work of the caller; they only must not
        # overwrite a staging chunk the previous call's K1 still reads.  So consecutive calls
        # pipeline: this call's copies start while the previous call's last chunks compute and
        # copy back (same chunking and staging buffers: per-chunk events; otherwise a full wait).
        prev = getattr(self, "_host_prev", None)
        if overlap_prev and prev is not None and prev[0] == bounds and prev[1] is xd:
            for ev in prev[2]:
                s_in.wait_event(ev)
        else:
            s_in.wait_stream(cur)
        done_in = []
        for b0, b1 in bounds:
            with torch.cuda.stream(s_in):
                xd[b0:b1].copy_(x_host[b0:b1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
                done_in.append(e)
        done_k = []
        for i, ((b0, b1), e) in enumerate(zip(bounds, done_in)):
            sk = s_k[i % lanes]
            sk.wait_event(e)
            self._normal_range(maps, xd, od, b0, b1, self._host_ws[i % lanes], sk.cuda_stream)
            ec = torch.cuda.Event()
            ec.record(sk)
            done_k.append(ec)
            s_out.wait_event(ec)
            with torch.cuda.stream(s_out):
                out_host[b0:b1].copy_(od[b0:b1], non_blocking=True)
        self._host_prev = (bounds, xd, done_k)
        cur.wait_stream(s_out)
        for st in s_k[:lanes]:
            cur.wait_stream(st)
        if sync:
            s_out.synchronize()
        return out_host

    def partial_shape(self, ncoils: int) -> tuple:
        """Shape of the residual partial-sum buffer `forward(partial=...)` fills."""
        return (self.batch, ncoils, 64)

    def forward(self, maps, x, y=None, *, ymeas=None, partial=None, partial_blocks=64, w=None):
        """y[b, j, :N_b] = A_b x_b  (- ymeas);  partial sums of |y|^2 if requested (K2)."""
        _no_weights(w)
        ncoils, mbs = self._maps_stride(maps)
        self._check_img(x, "x")
        if y is None:
            y = torch.zeros(self.batch, ncoils, self.nmax, dtype=torch.complex64, device=self.device)
        ws = self.workspace(ncoils)
        fused = self.fused_io
        _lib.call("sr_cart_forward", dv.ptr(x), dv.ptr(maps), mbs, dv.ptr(self.spos),
                  dv.ptr(self.ph), dv.ptr(self.soff), dv.ptr(y), y.shape[-1], dv.ptr(ymeas),
                  dv.ptr(partial), partial_blocks, dv.ptr(ws), self.batch, ncoils, self.ny,
                  self.nx, dv.ptr(self.g_ptr) if fused else None, dv.ptr(self.g_idx) if fused else None,
                  self.nblk, dv.stream())
        return y

    def adjoint(self, maps, y, out, *, coef=None, u=None, d=None, w=None):
        """out_b = sum_j conj(c_j) A_j^H y_bj  (K2)."""
        _no_weights(w)
        ncoils, mbs = self._maps_stride(maps)
        self._check_img(out, "out")
        if y.dim() != 3 or y.shape[0] != self.batch or y.shape[1] != ncoils or y.shape[2] < self.nmax:
            raise ValueError("y must be (B, C, >= nmax)")
        ws = self.workspace(ncoils)
        _lib.call("sr_cart_adjoint", dv.ptr(y), y.shape[-1], dv.ptr(maps), mbs, dv.ptr(self.spos),
                  dv.ptr(self.ph), dv.ptr(self.soff), dv.ptr(self.wlist), dv.ptr(self.woff),
                  dv.ptr(out), dv.ptr(ws), self.batch, ncoils, self.ny, self.nx, dv.ptr(coef),
                  dv.ptr(u), dv.ptr(d), dv.ptr(self.s_ptr) if self.fused_io else None,
                  dv.ptr(self.s_idx) if self.fused_io else None, self.nblk, dv.stream())
        return out

    # ------------------------------------------------- reference plugin protocol
    def _replica(self, c: int) -> "CartesianKernel":
        if self.batch != 1:
            raise ValueError("the host plugin protocol is single-slice")
        if c == 1:
            return self
        if c not in self._replicas:
            self._replicas[c] = CartesianKernel(self.dims, self._plans, batch=c)
        return self._replicas[c]

    def apply(self, batch: np.ndarray) -> np.ndarray:
        """(C, D) coil images -> (C, N) samples (linops.py:344-352)."""
        b = np.asarray(batch)
        k = self._replica(b.shape[0])
        ones = torch.ones(1, 1, self.D, dtype=torch.complex64, device=self.device)
        y = k.forward(ones, dv.c64(b.reshape(b.shape[0], self.D)))
        return dv.to_numpy128(y[:, 0, : self.n_points])

    def apply_adjoint(self, batch: np.ndarray) -> np.ndarray:
        """(C, N) samples -> (C, D) coil images (linops.py:354-364)."""
        b = np.asarray(batch)
        k = self._replica(b.shape[0])
        ones = torch.ones(1, 1, self.D, dtype=torch.complex64, device=self.device)
        out = torch.empty(b.shape[0], self.D, dtype=torch.complex64, device=self.device)
        k.adjoint(ones, dv.c64(b.reshape(b.shape[0], 1, -1)), out)
        return dv.to_numpy128(out)
