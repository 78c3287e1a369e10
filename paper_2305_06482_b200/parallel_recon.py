"""Multi-GPU partitioning of the sketched reconstruction.

* Config 2 (readout-decoupled 3-D Cartesian): the readout IDFT (K8) turns the
  volume into independent 2-D slices; ranks own contiguous slice blocks and run
  the batched engine with NO data-path collective (weak scaling); rank 0 gathers
  the slices at the end.
* Config 4 (3-D non-Cartesian): ranks own coil blocks; every operator call on
  the coil dimension (sketched normal op, true gradient, objective residual)
  produces a partial image / partial sum that is all-reduced (NCCL over
  NVLink on the GPU box, gloo in the CPU tests), FISTA state is replicated.

The reference has no distributed code; this module is
new.  The partition arithmetic is pure and tested on CPU with world size 2.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _lib


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items for `rank`; the first n % world ranks get one more."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class CoilShard:
    """Which coils / sketched coils one rank owns (config 4)."""

    rank: int
    world: int
    group: object = None  # torch.distributed process group (None = default)

    def coils(self, n: int) -> tuple[int, int]:
        return shard_range(n, self.rank, self.world)

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over ranks (no-op for world 1)."""
        if self.world > 1:
            import torch.distributed as dist
            if t.is_complex():
                dist.all_reduce(torch.view_as_real(t), group=self.group)
            else:
                dist.all_reduce(t, group=self.group)
        return t

    def all_reduce_async(self, t: torch.Tensor):
        """Start an in-place sum over ranks of a contiguous tensor (view); returns a handle whose
        .wait() makes the current stream wait for the collective.  NCCL runs it on its own stream,
        so kernels queued on the current stream after this call overlap it."""
        import torch.distributed as dist
        if self.world == 1:
            return _Done()
        v = torch.view_as_real(t) if t.is_complex() else t
        if not v.is_contiguous():
            raise ValueError("all_reduce_async needs a contiguous view")
        return dist.all_reduce(v, group=self.group, async_op=True)


class _Done:
    def wait(self):
        return True


def sharded_normal(partial_fn, x: torch.Tensor, shard: CoilShard) -> torch.Tensor:
    """sum_ranks partial_fn(x): each rank applies A_r^H A_r over its coils, then all-reduce."""
    return shard.all_reduce_(partial_fn(x))


def gather_slices(x_local: torch.Tensor, n_total: int, rank: int, world: int) -> torch.Tensor | None:
    """Concatenate per-rank slice blocks on rank 0 (returns None elsewhere)."""
    if world == 1:
        return x_local
    import torch.distributed as dist
    lo, hi = shard_range(n_total, rank, world)
    maxn = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world))
    pad = torch.zeros((maxn,) + tuple(x_local.shape[1:]), dtype=x_local.dtype, device=x_local.device)
    pad[: hi - lo] = x_local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    if rank != 0:
        return None
    parts = []
    for r in range(world):
        a, b = shard_range(n_total, r, world)
        parts.append(bufs[r][: b - a])
    return torch.cat(parts, dim=0)


# --------------------------------------------------------------------------- K8
def readout_phases(n: int) -> tuple[np.ndarray, np.ndarray]:
    """Centered unitary IDFT as pre * IDFT_unnorm * post (readout.cu header), fp64."""
    h = n // 2
    k = np.arange(n, dtype=np.float64)
    pre = np.exp(-2j * np.pi * ((k * h) % n) / n)
    post = np.exp(2j * np.pi * ((h * h) % n) / n) * np.exp(-2j * np.pi * ((h * k) % n) / n) / math.sqrt(n)
    return pre, post


class ReadoutDecoupler:
    """K8: (C, n_readout, N_yz) 3-D k-space -> (n_readout, C, N_yz) per-slice 2-D data."""

    def __init__(self, n_readout: int, device=None):
        self.n = int(n_readout)
        if not _lib.lib().sr_fft_size_supported(self.n):
            raise ValueError(f"readout length {self.n} has no sm_100a FFT instantiation")
        pre, post = readout_phases(self.n)
        self.device = device or dv.require_cuda()
        self.pre = dv.c64(pre, self.device)
        self.post = dv.c64(post, self.device)

    def __call__(self, kdata: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if kdata.dim() != 3 or kdata.shape[1] != self.n:
            raise ValueError(f"k-space must be (C, {self.n}, N_yz)")
        kdata = kdata.contiguous()
        C, n, inner = kdata.shape
        if out is None:
            out = torch.empty(n, C, inner, dtype=torch.complex64, device=kdata.device)
        _lib.call("sr_readout_idft", dv.ptr(kdata), dv.ptr(out), dv.ptr(self.pre), dv.ptr(self.post), C, n,
                  inner, dv.stream())
        return out


# --------------------------------------------------------------------------- per-slice prep
def slice_compression(y: torch.Tensor, keep: int, valid_n=None, threads: int | None = None) -> np.ndarray:
    """comp[s] = U_s[:, :keep]^H of each slice's (C, N) data, as coil_compress_svd computes it
    (forward_model.py:262-267) but without the N-long host SVD: numpy's SVD of a wide C x N
    matrix goes through the LQ factor, and svd(Y).U == svd(R^H).U for R from the (LAPACK /
    cuSOLVER-convention) Householder QR of Y^H (agreement ~1e-13, checked on the box).  So the
    QR runs batched on the device in complex128 and only the C x C SVDs run on the host.
    Zero padding of ragged slices leaves R unchanged."""
    import concurrent.futures as cf
    import os
    S, C, N = y.shape
    if valid_n is not None:
        y = y.clone()
        for s in range(S):
            y[s, :, int(valid_n[s]):] = 0
    if N < C:
        raise ValueError("compression needs at least as many samples as coils")
    A = y.to(torch.complex128).conj().transpose(1, 2).contiguous()
    if C <= 32:
        # batched tall-skinny Householder kernel (csrc/tsqr.cu), one CTA per slice
        from . import _device as dv
        from . import _lib
        Rt = torch.empty(S, C, C, dtype=torch.complex128, device=y.device)
        _lib.call("sr_tsqr_r", A.data_ptr(), N, C, N * C, S, Rt.data_ptr(), dv.stream())
        R = Rt.cpu().numpy()
    else:
        a, _ = torch.geqrf(A)
        R = torch.triu(a[:, :C, :]).cpu().numpy()

    def one(s):
        u, _, _ = np.linalg.svd(R[s].conj().T, full_matrices=False)
        return u[:, :keep].conj().T

    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    # one BLAS thread per worker: a multi-threaded BLAS inside every worker oversubscribes the host
    # (the compression step varied 38-140 ms between runs)
    try:
        from threadpoolctl import threadpool_limits
        limit = threadpool_limits(limits=1)
    except ImportError:  # pragma: no cover - threadpoolctl ships with the image
        limit = None
    try:
        with cf.ThreadPoolExecutor(max_workers=threads or max(1, min(S, ncpu))) as ex:
            return np.stack(list(ex.map(one, range(S))))
    finally:
        if limit is not None:
            limit.restore_original_limits()


def compress_slices(maps: torch.Tensor, y: torch.Tensor, keep: int, valid_n=None, comp=None):
    """(maps0, y0, comp): per-slice PCA rotation of maps (S, C, D) and data (S, C, N) on the device (K5).

    `comp` (S, keep, C) may be given, e.g. from the SVD of the complex128 host data: the
    low-energy singular vectors are ill-conditioned, so parity with the reference needs
    the SVD of exactly the reference's data, not of its complex64 copy."""
    from .sketching import coil_contract
    if comp is None:
        comp = slice_compression(y, keep, valid_n)
    maps0 = coil_contract(maps.contiguous(), comp)
    y0 = coil_contract(y.contiguous(), comp)
    return maps0, y0, comp
