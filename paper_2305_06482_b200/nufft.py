"""Kaiser-Bessel gridded NUFFT kernel on the device (K3/K4).

Drop-in for the reference plugin ``_GriddedNUFFTKernel``
(/root/reference/pkg/src/sketchrecon/linops.py:424-516): same oversampled grid
(g = 2 ceil(n os / 2), linops.py:438), Beatty beta (linops.py:440-445),
apodisation (linops.py:413-421, 447-452), tap rule base = ceil(u - w/2) with
the unnormalised KB window (linops.py:404-410, 464-492), D^-1/2 scaling and G
factor of the adjoint (linops.py:500-516).  The host builds the plan in fp64
(tap bases, offsets, apodisation); the device evaluates the KB weights on the
fly, so no N x G sparse matrix is ever materialised.  Samples are stored in a
locality-sorted order; forward/adjoint map back to trajectory order.  The plan
(tap bases, offsets, sort, chunk list) is built on the device by default
(csrc/nufft_plan.cu); the NumPy construction is kept as plan="host".
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _device as dv
from . import _lib

C_INT = ctypes.c_int


def oversampled_dims(dims, oversamp: float) -> tuple[int, ...]:
    return tuple(int(math.ceil(n * oversamp / 2) * 2) for n in dims)


def beatty_beta(n: int, g: int, width: int) -> float:
    s = g / n
    return math.pi * math.sqrt((width / s) ** 2 * (s - 0.5) ** 2 - 0.8)


def kb_apodization(r_over_g: np.ndarray, width: int, beta: float) -> np.ndarray:
    z2 = beta ** 2 - (math.pi * width * r_over_g) ** 2
    z = np.sqrt(np.abs(z2))
    out = np.empty_like(z)
    pos = z2 > 0
    out[pos] = np.sinh(z[pos]) / z[pos]
    out[~pos] = np.sinc(z[~pos] / np.pi)
    return width * out


def support_safe_frac(u: np.ndarray, b: np.ndarray, w: int) -> np.ndarray:
    """fp32 tap offsets t = u - b whose device-side KB support decisions equal the reference's.

    The reference evaluates tap k at d = u - (b + k) in float64 and keeps it iff
    1 - (2 d / w)^2 > 0 (linops.py:404-410).  The unnormalised kernel jumps from I0(0) = 1 to 0
    at |d| = w/2, so a sample that lies on a grid line up to 1e-16 (cos(pi/2) in a synthetic
    trajectory) keeps a tap with weight ~1 in float64 that a plain float32 offset drops.  The
    device tests |2 (t - k) / w| < 1 in float32 (kb_weight, nufft.cu); where that disagrees with
    float64 the offset is moved by one float32 ulp towards (or away from) the tap, which changes
    the other taps' weights by ~1e-7 relative.
    """
    u = np.asarray(u, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    t_all = (u - b).astype(np.float32)
    # only offsets within a few float32 ulps of a support edge (t - k = +-w/2) can disagree
    edge = np.abs((u - b) * 2.0 - np.round((u - b) * 2.0)) < 1e-5
    if not edge.any():
        return t_all
    idx = np.flatnonzero(edge)
    u, b = u[idx], b[idx]
    t32 = t_all[idx]
    one, two, wf = np.float32(1.0), np.float32(2.0), np.float32(w)
    for _ in range(8):
        moved = False
        for k in range(w):
            d64 = u - (b + k)
            ref = (1.0 - (2.0 * d64 / w) ** 2) > 0
            dev = np.abs((two * (t32 - np.float32(k))) / wf) < one
            bad = ref != dev
            if bad.any():
                tb = t32[bad]
                toward = np.where(ref[bad], np.sign(np.float32(k) - tb), np.sign(tb - np.float32(k)))
                toward = np.where(toward == 0, 1.0, toward).astype(np.float32)
                t32[bad] = np.nextafter(tb, tb + toward * np.float32(np.inf)).astype(np.float32)
                moved = True
        if not moved:
            t_all[idx] = t32
            return t_all
    raise RuntimeError("could not align float32 KB support decisions with float64")


class GriddedKernel:
    """Device NUFFT plan for one image grid (2-D or 3-D)."""

    BIN_CHUNK = 256  # samples per CTA of the binned gridding kernels (nufft.cu)

    def __init__(self, dims, points, oversamp: float = 1.25, width: int = 6, binned: bool = True,
                 binsize: int | None = None, plan: str = "device"):
        """plan: "device" builds the tap geometry, sort and chunk list on the GPU
        (csrc/nufft_plan.cu); "host" is the NumPy construction.  Both give identical plans."""
        self.dims = tuple(int(n) for n in dims)
        nd = len(self.dims)
        if nd not in (2, 3):
            raise NotImplementedError("device NUFFT implements 2-D and 3-D grids")
        if isinstance(points, torch.Tensor):
            pts = points.detach()
            if pts.dtype != torch.float64:
                raise ValueError("trajectory must be float64")
        else:
            pts = np.asarray(points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != nd:
            raise ValueError("trajectory dimensionality does not match the grid")
        if plan not in ("device", "host"):
            raise ValueError("plan must be 'device' or 'host'")
        self.width = int(width)
        if not 1 <= self.width <= 8:
            raise ValueError("KB width must be in [1, 8]")
        self.gdims = oversampled_dims(self.dims, oversamp)
        for g in self.gdims:
            if not _lib.lib().sr_fft_size_supported(g):
                raise ValueError(f"oversampled grid axis {g} has no sm_100a FFT instantiation")
        self.betas = [beatty_beta(n, g, self.width) for n, g in zip(self.dims, self.gdims)]
        self.n_points = int(pts.shape[0])
        self.batch = 1
        self.D = int(np.prod(self.dims))
        self.G = int(np.prod(self.gdims))
        self.nmax = self.n_points
        # bins: tile of binsize^d grid cells holding each sample's first tap; samples sorted by bin
        # and, inside a bin, by first-tap cell
        self.binsize = int(binsize or (8 if nd == 3 else 16))
        self.binned = bool(binned)
        dev = dv.require_cuda()
        self.device = dev
        pad = 3 - nd
        if plan == "device":
            self.base, self.frac, self.orig, chunks = self._plan_device(pts)
        else:
            self.base, self.frac, self.orig, chunks = self._plan_host(
                pts.cpu().numpy() if isinstance(pts, torch.Tensor) else pts)
        self.nchunks = int(chunks.shape[0])
        self.chunks = chunks
        self.dims3 = torch.tensor([1] * pad + list(self.dims), dtype=torch.int32)
        self.gdims3 = torch.tensor([1] * pad + list(self.gdims), dtype=torch.int32)
        self.betas3 = torch.tensor([0.0] * pad + self.betas, dtype=torch.float32)
        self._dims3_d = self.dims3.to(dev)
        self._gdims3_d = self.gdims3.to(dev)
        self._betas3_d = self.betas3.to(dev)
        ia = [np.ones(1)] * pad
        for n, g, beta in zip(self.dims, self.gdims, self.betas):
            r = np.arange(n, dtype=np.float64) - n // 2
            ia.append(1.0 / kb_apodization(r / g, self.width, beta))
        self.ia = [dv.host_to_dev(v.astype(np.float32), torch.float32, dev) for v in ia]
        self._grids = None
        self._pp = None  # (coil count, clean spread grid) of the ping-pong normal op
        self._wcache: dict = {}
        self.nparts = max(_lib.lib().sr_nufft_partial_blocks(self.n_points), self.nchunks)

    def _plan_host(self, pts: np.ndarray):
        """NumPy plan: tap bases / offsets per axis in fp64 (linops.py:472-476); the fp32 offsets
        keep the reference's fp64 support decisions (see support_safe_frac)."""
        nd, w, B = len(self.dims), self.width, self.binsize
        bases, fracs = [], []
        for a, (n, g) in enumerate(zip(self.dims, self.gdims)):
            u = pts[:, a] * (g / n)
            b = np.ceil(u - w / 2.0)
            bases.append(b.astype(np.int64))
            fracs.append(support_safe_frac(u, b, w))
        bpos = [np.mod(bases[a], g) for a, g in enumerate(self.gdims)]
        nbins = [-(-g // B) for g in self.gdims]
        binid = np.zeros(self.n_points, dtype=np.int64)
        local = np.zeros(self.n_points, dtype=np.int64)
        for a in range(nd):
            binid = binid * nbins[a] + bpos[a] // B
            local = local * B + bpos[a] % B
        # within a bin, samples sharing a first-tap cell are adjacent: the spread merges such
        # runs in registers before its shared atomics (about 3 samples per cell at config 4)
        order = np.argsort(binid * B ** nd + local, kind="stable")
        chunks = []
        if self.n_points:
            sb = binid[order]
            starts = np.flatnonzero(np.r_[True, sb[1:] != sb[:-1]])
            ends = np.r_[starts[1:], self.n_points]
            for st, en in zip(starts, ends):
                bid = int(sb[st])
                coords = []
                for a in range(nd - 1, -1, -1):
                    coords.append((bid % nbins[a]) * B)
                    bid //= nbins[a]
                coords = [0] * (3 - nd) + coords[::-1]
                for c0 in range(st, en, self.BIN_CHUNK):
                    chunks.append(coords + [c0, min(self.BIN_CHUNK, en - c0)])
        pad = 3 - nd
        base3 = np.zeros((3, self.n_points), dtype=np.int32)
        frac3 = np.zeros((3, self.n_points), dtype=np.float32)
        for a in range(nd):
            base3[pad + a] = bases[a][order]
            frac3[pad + a] = fracs[a][order]
        dev = self.device
        return (dv.host_to_dev(base3, torch.int32, dev), dv.host_to_dev(frac3, torch.float32, dev),
                dv.host_to_dev(order.astype(np.int32), torch.int32, dev),
                dv.host_to_dev(np.asarray(chunks, dtype=np.int32).reshape(-1, 5), torch.int32, dev))

    def _plan_device(self, pts):
        """Device plan (csrc/nufft_plan.cu): per-sample geometry and sort key in a kernel, a stable
        device radix sort, a gather by the order, and the chunk list from the bin boundaries."""
        nd, B, N, dev = len(self.dims), self.binsize, self.n_points, self.device
        CH = self.BIN_CHUNK
        if isinstance(pts, torch.Tensor):
            pts_d = pts.to(dev).contiguous()
        else:
            pts_d = torch.from_numpy(np.ascontiguousarray(pts)).pin_memory().to(dev, non_blocking=True)
        base_u = torch.empty(3, N, dtype=torch.int32, device=dev)
        frac_u = torch.empty(3, N, dtype=torch.float32, device=dev)
        key = torch.empty(N, dtype=torch.int64, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        dims_h = (C_INT * nd)(*self.dims)
        gdims_h = (C_INT * nd)(*self.gdims)
        _lib.call("sr_nufft_plan_geom", dv.ptr(pts_d), N, nd, dims_h, gdims_h, self.width, B, dv.ptr(base_u),
                  dv.ptr(frac_u), dv.ptr(key), dv.ptr(err), dv.stream())
        skey, order = torch.sort(key, stable=True)
        base = torch.empty_like(base_u)
        frac = torch.empty_like(frac_u)
        orig = torch.empty(N, dtype=torch.int32, device=dev)
        _lib.call("sr_nufft_plan_permute", dv.ptr(base_u), dv.ptr(frac_u), dv.ptr(order), N, dv.ptr(base),
                  dv.ptr(frac), dv.ptr(orig), dv.stream())
        del base_u, frac_u, key, order
        if N == 0:
            chunks = torch.zeros(0, 5, dtype=torch.int32, device=dev)
        else:
            binid = skey // (B ** nd)
            change = torch.ones(N, dtype=torch.bool, device=dev)
            change[1:] = binid[1:] != binid[:-1]
            starts = torch.nonzero(change).flatten()
            ends = torch.cat([starts[1:], torch.tensor([N], device=dev)])
            nch = (ends - starts + CH - 1) // CH
            owner = torch.repeat_interleave(torch.arange(len(starts), device=dev), nch)
            first = torch.cumsum(nch, 0) - nch
            c0 = starts[owner] + (torch.arange(len(owner), device=dev) - first[owner]) * CH
            cnt = torch.minimum(torch.full_like(c0, CH), ends[owner] - c0)
            bid = binid[starts][owner]
            nbins = [-(-g // B) for g in self.gdims]
            coords = []
            for a in range(nd - 1, -1, -1):
                coords.append((bid % nbins[a]) * B)
                bid = bid // nbins[a]
            cols = [torch.zeros_like(c0)] * (3 - nd) + coords[::-1] + [c0, cnt]
            chunks = torch.stack(cols, dim=1).to(torch.int32).contiguous()
        if int(err.item()):
            raise RuntimeError("could not align float32 KB support decisions with float64")
        return base, frac, orig, chunks

    # ------------------------------------------------------------ helpers
    # spread grids of at least this many bytes are zeroed off the critical path (sr_nufft_normal_pp)
    PP_MIN_BYTES = 1 << 28

    def workspace(self, ncoils: int, batch: int | None = None, chunk: int = 0, normal: bool = True, slots: int = 2):
        need = (slots if normal else 1) * ncoils * self.G
        if self._grids is None or self._grids.numel() < need:
            self._grids = torch.empty(need, dtype=torch.complex64, device=self.device)
        self._pp = None  # whoever asked may write anywhere in the workspace
        return self._grids

    def _geom(self):
        # dims / gdims / betas are HOST arrays (read into the kernel argument struct);
        # the inverse apodisation vectors are device arrays
        return (self.dims3.data_ptr(), self.gdims3.data_ptr(), self.betas3.data_ptr(), self.width,
                dv.ptr(self.ia[0]), dv.ptr(self.ia[1]), dv.ptr(self.ia[2]))

    def _weights(self, sqrt_w, squared: bool):
        """Per-sample weights in the sorted order: sqrt(w) (fwd/adj) or w (normal)."""
        if sqrt_w is None:
            return None
        key = (id(sqrt_w), squared)
        if key not in self._wcache:
            # one weight vector at a time: entries of an earlier one are dropped (a kernel reused over
            # many reconstructions would otherwise keep every vector it has seen)
            for k in [k for k in self._wcache if k[0] != id(sqrt_w)]:
                del self._wcache[k]
            sw = sqrt_w.to(torch.float64)
            v = (sw * sw) if squared else sw
            self._wcache[key] = (sqrt_w, v[self.orig.long()].to(torch.float32).contiguous())
        return self._wcache[key][1]

    def prepare_weights(self, sqrt_w) -> None:
        """Build the sorted-order weight vectors now (w for the normal op, sqrt(w) for forward /
        adjoint), so that a caller about to capture CUDA graphs does not allocate them inside a capture
        (memory of a graph's private pool is not returned to the allocator's cache)."""
        self._weights(sqrt_w, True)
        self._weights(sqrt_w, False)

    def _maps(self, maps):
        if maps.dim() != 3 or maps.shape[0] != 1 or maps.shape[2] != self.D:
            raise ValueError(f"maps must be (1, C, {self.D})")
        if maps.dtype != torch.complex64 or not maps.is_contiguous():
            raise ValueError("maps must be contiguous complex64")
        return maps.shape[1]

    def partial_shape(self, ncoils: int) -> tuple:
        return (1, self.nparts)

    def _bins(self):
        if self.binned:
            return dv.ptr(self.chunks), self.nchunks, self.binsize
        return None, 0, 0

    # ------------------------------------------------------------ device API
    def normal(self, maps, x, out, *, anchor=None, coef=None, u=None, d=None, w=None, chunk=None):
        C = self._maps(maps)
        if self.binned and 8 * C * self.G >= self.PP_MIN_BYTES and not torch.cuda.is_current_stream_capturing():
            # large grids: two spread grids used in turn, the idle one zeroed while the gridding kernel
            # runs (the state is the pair (coil count, clean spread grid); any other workspace user
            # resets it)
            pp, before = self._pp, self._grids
            grids = self.workspace(C, normal=True, slots=3)
            idx, clean = (pp[1], 1) if pp is not None and pp[0] == C and grids is before else (0, 0)
            _lib.call("sr_nufft_normal_pp", dv.ptr(x), dv.ptr(anchor), dv.ptr(maps), C, *self._geom()[:4],
                      *self._geom()[4:], dv.ptr(self.base), dv.ptr(self.frac), dv.ptr(self._weights(w, True)),
                      self.n_points, dv.ptr(out), dv.ptr(grids), dv.ptr(coef), dv.ptr(u), dv.ptr(d), *self._bins(),
                      idx, clean, dv.stream())
            self._pp = (C, 1 - idx)
            return out
        grids = self.workspace(C, normal=True)
        _lib.call("sr_nufft_normal", dv.ptr(x), dv.ptr(anchor), dv.ptr(maps), C, *self._geom()[:4],
                  *self._geom()[4:], dv.ptr(self.base), dv.ptr(self.frac), dv.ptr(self._weights(w, True)),
                  self.n_points, dv.ptr(out), dv.ptr(grids), dv.ptr(coef), dv.ptr(u), dv.ptr(d), *self._bins(),
                  dv.stream())
        return out

    def slab_planes(self) -> int:
        """Image planes along axis 0 that normal_slabs can split (0: no split for this grid)."""
        return int(self.dims3[0]) if _lib.lib().sr_nufft_normal_slabs_ok(self.dims3.data_ptr()) else 0

    def normal_slabs(self, maps, x, out, bounds, on_slab, *, anchor=None, coef=None, u=None, d=None, w=None):
        """normal() with the inverse tail issued one slab of image planes at a time: bounds =
        [(i0a, i0b), ...] covering [0, n0); after each slab's launches, on_slab(i0a, i0b) is called
        (the coil-sharded engine starts that slab's all-reduce there while the next slab computes)."""
        C = self._maps(maps)
        grids = self.workspace(C, normal=True)
        _lib.call("sr_nufft_normal_head", dv.ptr(x), dv.ptr(anchor), dv.ptr(maps), C, *self._geom(),
                  dv.ptr(self.base), dv.ptr(self.frac), dv.ptr(self._weights(w, True)), self.n_points,
                  dv.ptr(grids), *self._bins(), dv.stream())
        for a, b in bounds:
            _lib.call("sr_nufft_normal_tail", dv.ptr(maps), C, *self._geom(), dv.ptr(out), dv.ptr(grids),
                      dv.ptr(coef), dv.ptr(u), dv.ptr(d), int(a), int(b), dv.stream())
            on_slab(a, b)
        return out

    def forward(self, maps, x, y=None, *, ymeas=None, partial=None, partial_blocks=None, w=None):
        C = self._maps(maps)
        if y is None:
            y = torch.zeros(1, C, self.n_points, dtype=torch.complex64, device=self.device)
        if partial is not None and partial.numel() < self.nparts:
            raise ValueError("partial buffer too small")
        grids = self.workspace(C, normal=False)
        _lib.call("sr_nufft_forward", dv.ptr(x), dv.ptr(maps), C, *self._geom(), dv.ptr(self.base),
                  dv.ptr(self.frac), dv.ptr(self._weights(w, False)), dv.ptr(self.orig), self.n_points,
                  dv.ptr(y), dv.ptr(ymeas), dv.ptr(partial), dv.ptr(grids), *self._bins(), dv.stream())
        return y

    def adjoint(self, maps, y, out, *, coef=None, u=None, d=None, w=None):
        C = self._maps(maps)
        grids = self.workspace(C, normal=False)
        _lib.call("sr_nufft_adjoint", dv.ptr(y), dv.ptr(maps), C, *self._geom(), dv.ptr(self.base),
                  dv.ptr(self.frac), dv.ptr(self._weights(w, False)), dv.ptr(self.orig), self.n_points,
                  dv.ptr(out), dv.ptr(grids), dv.ptr(coef), dv.ptr(u), dv.ptr(d), *self._bins(), dv.stream())
        return out

    # ------------------------------------------------- reference plugin protocol
    def apply(self, batch: np.ndarray) -> np.ndarray:
        """(C, D) images -> (C, N) samples (linops.py:494-505)."""
        b = dv.c64(np.asarray(batch).reshape(-1, self.D))
        ones = torch.ones(1, self.D, dtype=torch.complex64, device=self.device)
        y = self.forward(b.unsqueeze(0).contiguous(), ones)
        return dv.to_numpy128(y[0])

    def apply_adjoint(self, batch: np.ndarray) -> np.ndarray:
        """(C, N) samples -> (C, D) images (linops.py:507-516)."""
        b = dv.c64(np.asarray(batch).reshape(-1, self.n_points))
        ones = torch.ones(1, 1, self.D, dtype=torch.complex64, device=self.device)
        outs = []
        for c in range(b.shape[0]):
            out = torch.empty(1, self.D, dtype=torch.complex64, device=self.device)
            self.adjoint(ones, b[c].reshape(1, 1, -1).contiguous(), out)
            outs.append(out[0])
        return dv.to_numpy128(torch.stack(outs))
