"""CPU ORACLE -- test infrastructure only, never the product path.

A NumPy restatement (complex128) of the reference algorithm for the sketched
SENSE normal-operator path of `sketchrecon`
(/root/reference/pkg/src/sketchrecon).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import it, and only as
the checker or the timed CPU baseline.  Every function cites the reference
lines it restates.  It is pinned against golden vectors produced by the real
reference (tests/golden/make_golden.py -> tests/golden/*.npz,
tests/test_oracle_golden.py).

Third-party arithmetic the reference relies on (pinned by the golden vectors,
generated with numpy 2.3.5 / scipy 1.18.1): numpy.fft (pocketfft),
numpy.random.SeedSequence + PCG64, numpy.linalg.svd (LAPACK gesdd),
scipy.special.i0.  This oracle uses the same numpy/scipy routines for those.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import i0 as bessel_i0

# --------------------------------------------------------------------------
# RNG streams  (rng.py:14-30)


def seed_stream(seed: int, index: int = 0) -> np.random.Generator:
    """Generator for stream `index` of root `seed` (rng.py:14-23)."""
    if seed < 0 or index < 0:
        raise ValueError("seed and index must be non-negative")
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), int(index)])))


def child_seed(seed: int, index: int) -> int:
    """First 32-bit word of SeedSequence((seed, index)) (rng.py:26-30)."""
    if seed < 0 or index < 0:
        raise ValueError("seed and index must be non-negative")
    return int(np.random.SeedSequence([int(seed), int(index)]).generate_state(1)[0])


# --------------------------------------------------------------------------
# centered unitary DFT  (linops.py:300-313, 332-364)


def _axes(a: np.ndarray, nd: int) -> tuple[int, ...]:
    return tuple(range(a.ndim - nd, a.ndim))


def centered_dft(grid: np.ndarray, nd: int, inverse: bool = False) -> np.ndarray:
    """DC-centered unitary DFT over the trailing `nd` axes (linops.py:304-309).

    Index i holds coordinate i - n//2 in both domains; implemented as
    roll-to-origin, plain FFT, roll-back.
    """
    ax = _axes(grid, nd)
    dims = [grid.shape[a] for a in ax]
    to_origin = [-(n // 2) for n in dims]
    back = [n // 2 for n in dims]
    g = np.roll(grid, to_origin, axis=ax)
    g = np.fft.ifftn(g, axes=ax, norm="ortho") if inverse else np.fft.fftn(g, axes=ax, norm="ortho")
    return np.roll(g, back, axis=ax)


def cartesian_bins(dims: tuple[int, ...], points: np.ndarray) -> np.ndarray:
    """Flat index of each integer trajectory bin on the centered grid (linops.py:341-342)."""
    pts = np.asarray(points, dtype=np.float64)
    if not np.all(pts == np.round(pts)):
        raise ValueError("cartesian-mask trajectories must have integer coordinates")
    for a, n in enumerate(dims):
        if pts[:, a].min() < -n / 2 or pts[:, a].max() >= n / 2:
            raise ValueError("trajectory outside [-n/2, n/2)")
    idx = np.rint(pts).astype(np.int64) + np.array([n // 2 for n in dims])
    flat = np.zeros(len(pts), dtype=np.int64)
    for a, n in enumerate(dims):
        flat = flat * n + idx[:, a]
    return flat


class CartesianKernel:
    """Oracle of _CartesianMaskKernel (linops.py:332-364): (C, D) <-> (C, N)."""

    def __init__(self, dims, points):
        self.dims = tuple(int(n) for n in dims)
        self.bins = cartesian_bins(self.dims, points)
        self.n_points = len(self.bins)

    def apply(self, batch: np.ndarray) -> np.ndarray:
        g = np.asarray(batch, dtype=np.complex128).reshape((-1,) + self.dims)
        spec = centered_dft(g, len(self.dims)).reshape(g.shape[0], -1)
        return spec[:, self.bins]

    def apply_adjoint(self, batch: np.ndarray) -> np.ndarray:
        b = np.asarray(batch, dtype=np.complex128)
        spec = np.zeros((b.shape[0], int(np.prod(self.dims))), dtype=np.complex128)
        spec[:, self.bins] = b  # duplicate bins: last write wins, as the reference
        g = centered_dft(spec.reshape((-1,) + self.dims), len(self.dims), inverse=True)
        return g.reshape(b.shape[0], -1)


# --------------------------------------------------------------------------
# Kaiser-Bessel gridded NUFFT  (linops.py:404-516)


def kb_window(u: np.ndarray, width: int, beta: float) -> np.ndarray:
    """I0(beta sqrt(1 - (2u/w)^2)) inside |u| < w/2, 0 outside (linops.py:404-410)."""
    t = 1.0 - (2.0 * np.asarray(u, dtype=np.float64) / width) ** 2
    return np.where(t > 0, bessel_i0(beta * np.sqrt(np.maximum(t, 0.0))), 0.0)


def kb_apod(r_over_g: np.ndarray, width: int, beta: float) -> np.ndarray:
    """w * sinh(z)/z, z = sqrt(beta^2 - (pi w r/g)^2) (sin for imaginary z) (linops.py:413-421)."""
    z2 = beta * beta - (math.pi * width * np.asarray(r_over_g, dtype=np.float64)) ** 2
    z = np.sqrt(np.abs(z2))
    safe = np.where(z == 0, 1.0, z)
    val = np.where(z2 > 0, np.sinh(safe) / safe, np.sin(safe) / safe)
    val = np.where(z == 0, 1.0, val)
    return width * val


def beatty_beta(n: int, g: int, width: int) -> float:
    """beta = pi sqrt((w/s)^2 (s - 1/2)^2 - 0.8), s = g/n (linops.py:441-445)."""
    s = g / n
    return math.pi * math.sqrt((width / s) ** 2 * (s - 0.5) ** 2 - 0.8)


def oversampled_dims(dims, oversamp: float) -> tuple[int, ...]:
    return tuple(int(math.ceil(n * oversamp / 2) * 2) for n in dims)  # linops.py:438


class GriddedKernel:
    """Oracle of _GriddedNUFFTKernel (linops.py:424-516).

    The interpolator is kept as dense per-sample tap tables (N, w^d) instead of
    a sparse matrix; duplicate grid columns of one sample are summed by the
    scatter/gather arithmetic exactly as CSR sum_duplicates does.
    """

    def __init__(self, dims, points, oversamp: float = 1.25, width: int = 6):
        self.dims = tuple(int(n) for n in dims)
        self.gdims = oversampled_dims(self.dims, oversamp)
        self.width = int(width)
        pts = np.asarray(points, dtype=np.float64)
        for a, n in enumerate(self.dims):
            if pts[:, a].min() < -n / 2 or pts[:, a].max() >= n / 2:
                raise ValueError("trajectory outside [-n/2, n/2)")
        self.n_points = pts.shape[0]
        self.betas = [beatty_beta(n, g, self.width) for n, g in zip(self.dims, self.gdims)]
        apod = np.ones(1)
        for n, g, beta in zip(self.dims, self.gdims, self.betas):
            r = np.arange(n, dtype=np.float64) - n // 2
            apod = np.multiply.outer(apod, kb_apod(r / g, self.width, beta)).reshape(-1)
        self.apod = apod
        # per-axis taps
        w = self.width
        cols_all, vals_all = [], []
        for a, (n, g, beta) in enumerate(zip(self.dims, self.gdims, self.betas)):
            u = pts[:, a] * (g / n)
            base = np.ceil(u - w / 2).astype(np.int64)
            cols = base[:, None] + np.arange(w)[None, :]
            vals_all.append(kb_window(u[:, None] - cols, w, beta))
            cols_all.append(np.mod(cols + g // 2, g))
        # tensor product, row-major over axes
        idx = np.zeros((self.n_points, 1), dtype=np.int64)
        val = np.ones((self.n_points, 1))
        for a in range(len(self.dims)):
            stride = int(np.prod(self.gdims[a + 1:]))
            idx = (idx[:, :, None] + stride * cols_all[a][:, None, :]).reshape(self.n_points, -1)
            val = (val[:, :, None] * vals_all[a][:, None, :]).reshape(self.n_points, -1)
        self.tap_idx = idx
        self.tap_val = val
        self.scale = 1.0 / math.sqrt(int(np.prod(self.dims)))
        self.G = int(np.prod(self.gdims))
        self.lo = [g // 2 - n // 2 for n, g in zip(self.dims, self.gdims)]

    def _embed(self, imgs):
        c = imgs.shape[0]
        grid = np.zeros((c,) + self.gdims, dtype=np.complex128)
        sl = (slice(None),) + tuple(slice(l, l + n) for l, n in zip(self.lo, self.dims))
        grid[sl] = imgs
        return grid

    def apply(self, batch: np.ndarray) -> np.ndarray:
        b = np.asarray(batch, dtype=np.complex128)
        c = b.shape[0]
        pre = (b / self.apod).reshape((c,) + self.dims)
        grid = self._embed(pre)
        nd = len(self.dims)
        ax = _axes(grid, nd)
        # unnormalised centered DFT on the oversampled grid
        spec = np.roll(np.fft.fftn(np.roll(grid, [-(g // 2) for g in self.gdims], axis=ax), axes=ax),
                       [g // 2 for g in self.gdims], axis=ax).reshape(c, -1)
        vals = np.einsum("nt,cnt->cn", self.tap_val, spec[:, self.tap_idx])
        return vals * self.scale

    def apply_adjoint(self, batch: np.ndarray) -> np.ndarray:
        b = np.asarray(batch, dtype=np.complex128)
        c = b.shape[0]
        spec = np.zeros((c, self.G), dtype=np.complex128)
        contrib = b[:, :, None] * self.tap_val[None, :, :]  # real weights: conj = same
        for ci in range(c):
            np.add.at(spec[ci], self.tap_idx.ravel(), contrib[ci].ravel())
        spec = spec.reshape((c,) + self.gdims)
        nd = len(self.dims)
        ax = _axes(spec, nd)
        grid = np.roll(np.fft.ifftn(np.roll(spec, [-(g // 2) for g in self.gdims], axis=ax), axes=ax),
                       [g // 2 for g in self.gdims], axis=ax) * self.G
        sl = (slice(None),) + tuple(slice(l, l + n) for l, n in zip(self.lo, self.dims))
        sub = grid[sl].reshape(c, -1)
        return sub / self.apod * self.scale


class ChunkedGriddedKernel(GriddedKernel):
    """GriddedKernel with the per-sample tap tables built per chunk of samples on the fly instead
    of stored for the whole trajectory (same arithmetic, bounded memory: config 4's 9.2 M samples
    x 64 taps would need ~9.4 GB of tables).  Used to time the CPU reference path at full size."""

    def __init__(self, dims, points, oversamp: float = 1.25, width: int = 6, chunk: int = 1 << 20):
        pts = np.asarray(points, dtype=np.float64)
        super().__init__(dims, pts[:1], oversamp, width)  # geometry, betas, apodisation
        for a, n in enumerate(self.dims):
            if pts[:, a].min() < -n / 2 or pts[:, a].max() >= n / 2:
                raise ValueError("trajectory outside [-n/2, n/2)")
        self.points = pts
        self.n_points = pts.shape[0]
        self.chunk = int(chunk)
        del self.tap_idx, self.tap_val

    def _taps(self, p):
        w = self.width
        idx = np.zeros((p.shape[0], 1), dtype=np.int64)
        val = np.ones((p.shape[0], 1))
        for a, (n, g, beta) in enumerate(zip(self.dims, self.gdims, self.betas)):
            u = p[:, a] * (g / n)
            base = np.ceil(u - w / 2).astype(np.int64)
            cols = base[:, None] + np.arange(w)[None, :]
            stride = int(np.prod(self.gdims[a + 1:]))
            idx = (idx[:, :, None] + stride * np.mod(cols + g // 2, g)[:, None, :]).reshape(p.shape[0], -1)
            val = (val[:, :, None] * kb_window(u[:, None] - cols, w, beta)[:, None, :]).reshape(p.shape[0], -1)
        return idx, val

    def apply(self, batch: np.ndarray) -> np.ndarray:
        b = np.asarray(batch, dtype=np.complex128)
        c = b.shape[0]
        grid = self._embed((b / self.apod).reshape((c,) + self.dims))
        ax = _axes(grid, len(self.dims))
        spec = np.roll(np.fft.fftn(np.roll(grid, [-(g // 2) for g in self.gdims], axis=ax), axes=ax),
                       [g // 2 for g in self.gdims], axis=ax).reshape(c, -1)
        out = np.empty((c, self.n_points), dtype=np.complex128)
        for s0 in range(0, self.n_points, self.chunk):
            idx, val = self._taps(self.points[s0:s0 + self.chunk])
            out[:, s0:s0 + idx.shape[0]] = np.einsum("nt,cnt->cn", val, spec[:, idx])
        return out * self.scale

    def apply_adjoint(self, batch: np.ndarray) -> np.ndarray:
        b = np.asarray(batch, dtype=np.complex128)
        c = b.shape[0]
        spec = np.zeros((c, self.G), dtype=np.complex128)
        for s0 in range(0, self.n_points, self.chunk):
            idx, val = self._taps(self.points[s0:s0 + self.chunk])
            fi = idx.ravel()
            for ci in range(c):
                contrib = (b[ci, s0:s0 + idx.shape[0], None] * val).ravel()
                # duplicate columns summed like CSR^H (np.bincount: same sums as np.add.at, faster)
                spec[ci] += np.bincount(fi, contrib.real, self.G) + 1j * np.bincount(fi, contrib.imag, self.G)
        spec = spec.reshape((c,) + self.gdims)
        ax = _axes(spec, len(self.dims))
        grid = np.roll(np.fft.ifftn(np.roll(spec, [-(g // 2) for g in self.gdims], axis=ax), axes=ax),
                       [g // 2 for g in self.gdims], axis=ax) * self.G
        sl = (slice(None),) + tuple(slice(l, l + n) for l, n in zip(self.lo, self.dims))
        return grid[sl].reshape(c, -1) / self.apod * self.scale


# --------------------------------------------------------------------------
# SENSE operator  (forward_model.py:119-213)


@dataclass
class Counter:
    """Tagged tallies with pause depth (linops.py:147-178)."""

    counts: dict = field(default_factory=dict)
    depth: int = 0

    def add(self, tag, n=1):
        if self.depth == 0:
            self.counts[tag] = self.counts.get(tag, 0) + int(n)


class Sense:
    """A = W^1/2 F C over a Fourier kernel (forward_model.py:119-180)."""

    def __init__(self, maps: np.ndarray, kernel, weights: np.ndarray | None = None,
                 counter: Counter | None = None):
        self.maps = np.asarray(maps, dtype=np.complex128)
        self.kernel = kernel
        self.sqrt_w = None if weights is None else np.sqrt(np.asarray(weights, dtype=np.float64))
        self.counter = counter if counter is not None else Counter()

    @property
    def n_coils(self):
        return self.maps.shape[0]

    def forward(self, x):
        self.counter.add("coil_transform", self.n_coils)
        k = self.kernel.apply(self.maps * np.asarray(x, dtype=np.complex128)[None, :])
        if self.sqrt_w is not None:
            k = k * self.sqrt_w[None, :]
        return k.reshape(-1)

    def forward_unweighted(self, x):
        self.counter.add("coil_transform", self.n_coils)
        return self.kernel.apply(self.maps * np.asarray(x, dtype=np.complex128)[None, :]).reshape(-1)

    def adjoint(self, y):
        k = np.asarray(y, dtype=np.complex128).reshape(self.n_coils, -1)
        if self.sqrt_w is not None:
            k = k * self.sqrt_w[None, :]
        self.counter.add("coil_transform", self.n_coils)
        imgs = self.kernel.apply_adjoint(k)
        return np.einsum("cd,cd->d", np.conj(self.maps), imgs)

    def normal(self, x):
        return self.adjoint(self.forward(x))

    def weight_data(self, k):
        if self.sqrt_w is None:
            return np.array(k, dtype=np.complex128)
        return np.asarray(k, dtype=np.complex128) * self.sqrt_w[None, :]


def radial_density_weights(points: np.ndarray) -> np.ndarray:
    """Ramp |f| with DC fix-up, max-normalised (forward_model.py:227-242)."""
    r = np.sqrt(np.sum(np.asarray(points, dtype=np.float64) ** 2, axis=1))
    nz = r > 1e-12 * max(r.max(), 1.0)
    if not nz.any():
        return np.ones_like(r)
    w = np.where(nz, r, 0.5 * r[nz].min())
    return w / w.max()


def coil_compress_svd(data: np.ndarray, maps: np.ndarray, keep: int):
    """SVD compression of (C, N) data, maps rotated alike (forward_model.py:245-272)."""
    c = data.shape[0]
    if not 1 <= keep <= c:
        raise ValueError("keep out of range")
    u, s, _ = np.linalg.svd(np.asarray(data, dtype=np.complex128), full_matrices=False)
    comp = np.conj(u[:, :keep]).T
    total = float(np.sum(s ** 2))
    energy = float(np.sum(s[:keep] ** 2) / total) if total > 0 else 1.0
    return comp @ data, comp @ maps, comp, energy


# --------------------------------------------------------------------------
# structured sketch  (sketching.py:69-129)


def gen_sketch_matrix(c_hat: int, v: int, s: int, n_coils: int, seed: int,
                      distribution: str = "rademacher", rademacher_scale: float = 1.0) -> np.ndarray:
    """[I_v 0; 0 R] with R s x (C - v) random (sketching.py:69-94).

    `rademacher_scale` = 1 is the reference; BASELINE configs use 1/sqrt(12).
    """
    if v > n_coils or s > n_coils - v or c_hat > n_coils or c_hat != v + s:
        raise ValueError("invalid sketch shape")
    mat = np.zeros((c_hat, n_coils))
    mat[:v, :v] = np.eye(v)
    if s > 0:
        g = seed_stream(seed, 0)
        if distribution == "gaussian":
            blk = g.standard_normal((s, n_coils - v)) / s
        else:
            blk = (g.integers(0, 2, size=(s, n_coils - v)) * 2.0 - 1.0) * rademacher_scale
        mat[v:, v:] = blk
    return mat


# --------------------------------------------------------------------------
# Daubechies-4 wavelet  (linops.py:593-702)

DB4_LO = np.array([
    -0.010597401785069032105, 0.032883011666885199735, 0.030841381835560763627,
    -0.18703481171909308408, -0.027983769416859854211, 0.63088076792985890788,
    0.71484657055291564709, 0.23037781330889650086])
DB4_HI = np.array([DB4_LO[7 - k] * (-1.0 if k % 2 else 1.0) for k in range(8)])


def wavelet_levels(dims, cap: int = 4) -> int:
    """Largest level count (<= cap) with every dim halvable (linops.py:609-616)."""
    lv, d = 0, list(dims)
    while lv < cap and all(n % 2 == 0 and n // 2 >= 1 for n in d):
        d = [n // 2 for n in d]
        lv += 1
    return lv


def _split_axis(a: np.ndarray, axis: int) -> np.ndarray:
    """lo[i] = sum_k h[k] a[(2i+k) mod n], hi likewise; [lo | hi] (linops.py:619-635)."""
    a = np.moveaxis(a, axis, -1)
    n = a.shape[-1]
    if n % 2:
        raise ValueError("odd axis")
    lo = np.zeros(a.shape[:-1] + (n // 2,), dtype=np.complex128)
    hi = np.zeros_like(lo)
    for k in range(8):
        sh = np.take(a, (2 * np.arange(n // 2) + k) % n, axis=-1)
        lo += DB4_LO[k] * sh
        hi += DB4_HI[k] * sh
    return np.moveaxis(np.concatenate([lo, hi], axis=-1), -1, axis)


def _merge_axis(a: np.ndarray, axis: int) -> np.ndarray:
    """Transpose of _split_axis (linops.py:638-651)."""
    a = np.moveaxis(a, axis, -1)
    n = a.shape[-1]
    lo, hi = a[..., : n // 2], a[..., n // 2:]
    out = np.zeros(a.shape, dtype=np.complex128)
    for k in range(8):
        pos = (2 * np.arange(n // 2) + k) % n
        # scatter-add: x[pos] += h[k] lo
        np.add.at(out, (Ellipsis, pos), DB4_LO[k] * lo + DB4_HI[k] * hi)
    return np.moveaxis(out, -1, axis)


def wavelet_forward(x: np.ndarray, dims, levels: int | None = None) -> np.ndarray:
    """Multilevel analysis, [lo|hi] per axis, recurse on the low corner (linops.py:677-687)."""
    levels = wavelet_levels(dims) if levels is None else levels
    out = np.asarray(x, dtype=np.complex128).reshape(dims).copy()
    ext = list(dims)
    for _ in range(levels):
        sl = tuple(slice(0, e) for e in ext)
        blk = out[sl]
        for ax in range(len(dims)):
            blk = _split_axis(blk, ax)
        out[sl] = blk
        ext = [(e + 1) // 2 for e in ext]
    return out.reshape(-1)


def wavelet_adjoint(c: np.ndarray, dims, levels: int | None = None) -> np.ndarray:
    """Inverse (= adjoint) of wavelet_forward (linops.py:689-702)."""
    levels = wavelet_levels(dims) if levels is None else levels
    out = np.asarray(c, dtype=np.complex128).reshape(dims).copy()
    exts = []
    ext = list(dims)
    for _ in range(levels):
        exts.append(list(ext))
        ext = [(e + 1) // 2 for e in ext]
    for ext in reversed(exts):
        sl = tuple(slice(0, e) for e in ext)
        blk = out[sl]
        for ax in reversed(range(len(dims))):
            blk = _merge_axis(blk, ax)
        out[sl] = blk
    return out.reshape(-1)


def prox_l1(v: np.ndarray, t: float) -> np.ndarray:
    """Complex soft threshold (solvers.py:129-135)."""
    if t < 0:
        raise ValueError("threshold must be nonnegative")
    m = np.abs(v)
    return v * (np.maximum(m - t, 0.0) / np.where(m > 0, m, 1.0))


def wavelet_prox(v: np.ndarray, dims, step: float, lam: float, levels=None) -> np.ndarray:
    """prox of step*lam*||Psi x||_1 (solvers.py:71-80)."""
    if lam == 0.0:
        return np.array(v, dtype=np.complex128)
    return wavelet_adjoint(prox_l1(wavelet_forward(v, dims, levels), step * lam), dims, levels)


def wavelet_l1(x: np.ndarray, dims, lam: float, levels=None) -> float:
    """lam ||Psi x||_1 (solvers.py:61-69)."""
    if lam == 0.0:
        return 0.0
    return lam * float(np.sum(np.abs(wavelet_forward(x, dims, levels))))


# --------------------------------------------------------------------------
# solvers  (linops.py:766-782, solvers.py:188-308)


def power_max_eig(apply, dim: int, iters: int = 30, seed: int = 0) -> float:
    """Power iteration with v0 ~ CN(0, I) from seed_stream(seed, 0) (linops.py:766-782)."""
    g = seed_stream(seed, 0)
    v = g.standard_normal(dim) + 1j * g.standard_normal(dim)
    v = v / np.linalg.norm(v)
    lam = 0.0
    for _ in range(int(iters)):
        w = apply(v)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0
        lam = float(np.real(np.vdot(v, w)))
        v = w / nw
    return lam


# --------------------------------------------------------------------------
# total variation (linops.py:717-741) and the PDHG sub-solver (solvers.py:138-149, 315-362)


def finite_diff_forward(x: np.ndarray, dims) -> np.ndarray:
    """Per-axis circular forward differences stacked over axes, D -> ndim*D (linops.py:724-729)."""
    g = np.asarray(x, dtype=np.complex128).reshape(dims)
    return np.concatenate([(np.roll(g, -1, axis=a) - g).ravel() for a in range(g.ndim)])


def finite_diff_adjoint(y: np.ndarray, dims) -> np.ndarray:
    """Adjoint: sum_a roll(part_a, +1, a) - part_a (linops.py:731-738)."""
    d = int(np.prod(dims))
    acc = np.zeros(dims, dtype=np.complex128)
    for a in range(len(dims)):
        part = np.asarray(y[a * d:(a + 1) * d]).reshape(dims)
        acc += np.roll(part, 1, axis=a) - part
    return acc.ravel()


def tv_norm_value(x: np.ndarray, dims, lam: float) -> float:
    """lam ||D x||_1, complex magnitudes (solvers.py:61-69 with FiniteDiffOp)."""
    if lam == 0.0:
        return 0.0
    return lam * float(np.sum(np.abs(finite_diff_forward(x, dims))))


def clamp_magnitude(p: np.ndarray, radius: float) -> np.ndarray:
    """Project every complex entry onto the disc of the given radius (solvers.py:138-142)."""
    mag = np.abs(p)
    factor = np.where(mag > radius, radius / np.where(mag > 0, mag, 1.0), 1.0)
    return p * factor


def pdhg_tv(normal_s, dvec: np.ndarray, anchor: np.ndarray, dims, lam: float, iters: int,
            cg_iters: int, ratio: float = 1.0, step_scale: float = 0.9) -> np.ndarray:
    """Chambolle-Pock on min_x 0.5||A_s(x - a)||^2 + Re<d, x> + lam||D x||_1, K = D
    (coil_sketch.py:200-216 over solvers.py:315-362); ||D|| = 2 sqrt(ndim) (solvers.py:145-148);
    the data prox solves (A_s^H A_s + I/tau) w = -d - A_s^H A_s (v - a) by cg_iters CG steps."""
    norm_k = 2.0 * math.sqrt(len(dims))
    r = math.sqrt(ratio)
    sigma = r / norm_k * step_scale
    tau = 1.0 / (r * norm_k) * step_scale
    x = np.array(anchor, dtype=np.complex128)
    z = x.copy()
    p = np.zeros(len(dims) * x.size, dtype=np.complex128)
    for _ in range(iters):
        p = clamp_magnitude(p + sigma * finite_diff_forward(z, dims), lam)
        v = x - tau * finite_diff_adjoint(p, dims)
        rhs = -dvec - normal_s(v - anchor)
        w = cg(lambda u: normal_s(u) + u / tau, rhs, np.zeros_like(v), cg_iters)
        x_new = v + w
        z = 2.0 * x_new - x
        x = x_new
    return x


def pdhg_reconstruct_tv(a: "Sense", y: np.ndarray, dims, lam: float, iters: int, cg_iters: int,
                        ratio: float = 1.0, step_scale: float = 0.9, tol: float = 0.0) -> tuple[np.ndarray, int]:
    """Full-operator l1-TV reconstruction, reconstruct(..., solver="pdhg") (solvers.py:470-500):
    Chambolle-Pock with K = D (solvers.py:315-362), f* prox = clamp to |p| <= lam, and the data
    prox argmin_u 0.5||Au - y||^2 + ||u - v||^2/(2 tau) = v + w, w from cg_iters CG steps on
    (A^H A + I/tau) w = A^H (y - A v) started at 0.  Returns (x, iterations run)."""
    norm_k = 2.0 * math.sqrt(len(dims))
    r = math.sqrt(ratio)
    sigma = r / norm_k * step_scale
    tau = 1.0 / (r * norm_k) * step_scale
    x = np.zeros(int(np.prod(dims)), dtype=np.complex128)
    z = x.copy()
    p = np.zeros(len(dims) * x.size, dtype=np.complex128)
    it = 0
    for it in range(1, iters + 1):
        p = clamp_magnitude(p + sigma * finite_diff_forward(z, dims), lam)
        v = x - tau * finite_diff_adjoint(p, dims)
        rhs = a.adjoint(y - a.forward(v))
        w = cg(lambda u: a.adjoint(a.forward(u)) + u / tau, rhs, np.zeros_like(v), cg_iters)
        x_new = v + w
        z = 2.0 * x_new - x
        delta = float(np.linalg.norm(x_new - x))
        xnorm = float(np.linalg.norm(x))
        x = x_new
        if xnorm > 0 and delta / xnorm < tol:
            break
    return x, it


def accproxsgd(a: "Sense", y: np.ndarray, prox, batch: int, alpha0: float, beta: float, beta_min: float,
               x0: np.ndarray, iters: int, seed: int = 0, tol: float = 0.0) -> tuple[np.ndarray, int]:
    """Accelerated proximal SGD over coil batches (solvers.py:369-427): per iteration `batch`
    coils drawn without replacement from seed_stream(seed, 0) (sorted), gradient
    (C/batch) A_S^H (A_S z - y_S), step max(beta^t alpha0, beta_min), prox, Nesterov momentum.
    The coil subset shares the kernel and counter (forward_model.py:198-203)."""
    C = a.n_coils
    if not 1 <= batch <= C:
        raise ValueError(f"batch must be in [1, {C}], got {batch}")
    rng = seed_stream(seed, 0)
    y_mat = np.asarray(y, dtype=np.complex128).reshape(C, -1)
    scale = C / batch
    x = np.array(x0, dtype=np.complex128)
    z = x.copy()
    t = 1.0
    it = 0
    for it in range(1, iters + 1):
        idx = np.sort(rng.choice(C, size=batch, replace=False))
        w = None if a.sqrt_w is None else a.sqrt_w ** 2
        sub = Sense(a.maps[idx], a.kernel, w, a.counter)
        g = scale * sub.adjoint(sub.forward(z) - y_mat[idx].ravel())
        alpha = max(beta ** it * alpha0, beta_min)
        xn = prox(z - alpha * g, alpha)
        tn = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
        z = xn + ((t - 1.0) / tn) * (xn - x)
        delta = float(np.linalg.norm(xn - x))
        xnorm = float(np.linalg.norm(x))
        x = xn
        t = tn
        if xnorm > 0 and delta / xnorm < tol:
            break
    return x, it


def power_start_vector(dim: int, seed: int = 0) -> np.ndarray:
    g = seed_stream(seed, 0)
    v = g.standard_normal(dim) + 1j * g.standard_normal(dim)
    return v / np.linalg.norm(v)


def fista(grad, prox, L: float, x0: np.ndarray, iters: int, tol: float = 0.0, objective=None,
          full: bool = False):
    """FISTA, t_{k+1} = (1 + sqrt(1 + 4 t_k^2))/2 (solvers.py:264-308).  full=True returns
    (x, iterations run, objective history)."""
    step = 1.0 / L
    x = np.array(x0, dtype=np.complex128)
    z = x.copy()
    t = 1.0
    hist = []
    it = 0
    for it in range(1, iters + 1):
        xn = prox(z - step * grad(z), step)
        tn = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
        z = xn + ((t - 1.0) / tn) * (xn - x)
        delta = float(np.linalg.norm(xn - x))
        xnorm = float(np.linalg.norm(x))
        x = xn
        t = tn
        if objective is not None:
            hist.append(objective(x))
        if xnorm > 0 and delta / xnorm < tol:
            break
    return (x, it, np.array(hist)) if full else x


def cg(matvec, b, x0, iters: int, tol_abs: float = 0.0, full: bool = False):
    """Plain CG on M x = b (solvers.py:206-229).  full=True returns (x, iterations, residual
    norms)."""
    x = np.array(x0, dtype=np.complex128)
    r = b - matvec(x) if np.any(x) else np.array(b, dtype=np.complex128)
    p = r.copy()
    rs = float(np.real(np.vdot(r, r)))
    res = [math.sqrt(rs)]
    it = 0
    for it in range(1, iters + 1):
        if math.sqrt(rs) <= tol_abs:
            it -= 1
            break
        mp = matvec(p)
        den = float(np.real(np.vdot(p, mp)))
        if den <= 0:
            break
        a = rs / den
        x = x + a * p
        r = r - a * mp
        rn = float(np.real(np.vdot(r, r)))
        res.append(math.sqrt(rn))
        p = r + (rn / rs) * p
        rs = rn
    return (x, it, np.array(res)) if full else x


def reconstruct(a: "Sense", y: np.ndarray, dims, reg: str, lam: float, iters: int, tol: float = 0.0,
                step_scale: float = 0.9):
    """Full-coil min 0.5||A x - y||^2 + g(x) (solvers.py:434-500): l2 -> cg_normal
    (solvers.py:232-257, stop at tol * ||A^H y||), l1-wavelet -> FISTA with L from the power
    iteration and the composite objective recorded per iteration.  Returns (x, iterations,
    history, coil transforms)."""
    n0 = a.counter.counts.get("coil_transform", 0)
    D = int(np.prod(dims))
    x0 = np.zeros(D, dtype=np.complex128)
    if reg == "l2":
        b = a.adjoint(y)
        x, it, hist = cg(lambda u: a.adjoint(a.forward(u)) + lam * u, b, x0, iters, tol * float(np.linalg.norm(b)),
                         full=True)
    else:
        a.counter.depth += 1
        L = power_max_eig(a.normal, D) / step_scale
        a.counter.depth -= 1

        def objective(v):
            a.counter.depth += 1
            r = a.forward(v) - y
            a.counter.depth -= 1
            return 0.5 * float(np.linalg.norm(r) ** 2) + wavelet_l1(v, dims, lam)

        x, it, hist = fista(lambda v: a.adjoint(a.forward(v) - y), lambda v, st: wavelet_prox(v, dims, st, lam),
                            L, x0, iters, tol, objective=objective, full=True)
    return x, it, hist, a.counter.counts.get("coil_transform", 0) - n0


def gfactor_montecarlo(recon, a_full: "Sense", a_under: "Sense", x_true: np.ndarray, noise_sigma: float,
                       trials: int, R: float, seed: int, support_rel_threshold: float = 1e-3):
    """Pseudo-replica inverse g-factor (metrics.py:157-211): per trial i, noise from
    seed_stream(seed, i) (full data first, then undersampled), both reconstructed by recon(op, y);
    inverse_g = std_full sqrt(R) / std_under on the support (|x| > thr max|x|) where the
    undersampled std is not degenerate.  Returns (inverse_g, mask)."""
    if trials < 2:
        raise ValueError("need at least 2 trials")
    clean_full = a_full.forward_unweighted(x_true)
    clean_under = a_under.forward_unweighted(x_true)
    scale = noise_sigma / math.sqrt(2.0)
    rf = np.empty((trials, x_true.size), dtype=np.complex128)
    ru = np.empty_like(rf)
    for i in range(trials):
        g = seed_stream(seed, i)
        n_full = scale * (g.standard_normal(clean_full.shape) + 1j * g.standard_normal(clean_full.shape))
        n_under = scale * (g.standard_normal(clean_under.shape) + 1j * g.standard_normal(clean_under.shape))
        rf[i] = recon(a_full, a_full.weight_data(clean_full + n_full))
        ru[i] = recon(a_under, a_under.weight_data(clean_under + n_under))
    sf, su = np.std(rf, axis=0), np.std(ru, axis=0)
    mag = np.abs(x_true)
    mask = (mag > support_rel_threshold * mag.max()) & ~(su <= np.finfo(float).tiny)
    inv = np.zeros(x_true.size)
    inv[mask] = sf[mask] * math.sqrt(R) / su[mask]
    return inv, mask


# --------------------------------------------------------------------------
# Algorithm 1: coil-sketched reconstruction  (coil_sketch.py:220-330)


@dataclass
class ReconResult:
    x_final: np.ndarray
    objectives: list
    counts: dict
    diverged: bool
    lipschitz: float
    init_count: int = 0
    per_outer_counts: list = field(default_factory=list)


def coil_sketching_recon(data: np.ndarray, maps: np.ndarray, dims, make_kernel, *,
                         c_hat0: int, v: int, s: int, lam: float, outer: int, inner: int,
                         seed: int = 0, weights=None, rademacher_scale: float = 1.0,
                         solver: str = "fista", reg: str = "l1-wavelet",
                         step_scale: float = 0.9, distribution: str = "rademacher",
                         cg_iters: int = 8, pdhg_ratio: float = 1.0, tol: float = 0.0,
                         reuse_step_size: bool = True, use_init: bool = False,
                         init_iters: int = 100) -> ReconResult:
    """Outer true-gradient + fresh sketch + warm-started inner solve (coil_sketch.py:220-306).

    make_kernel() builds the Fourier kernel (shared by full and sketched ops).
    reg: 'l1-wavelet' (FISTA), 'l2' (CG, coil_sketch.py:182-191) or 'l1-tv' (PDHG with an
    inner CG of cg_iters steps, coil_sketch.py:200-216).
    tol: FISTA relative-change stop of the inner solves (solvers.py:300, passed through
    coil_sketch.py:171-178); reuse_step_size=False re-estimates the Lipschitz constant every
    outer (coil_sketch.py:281); use_init runs the classical-sketch solve of
    coil_sketch.py:148-159, 268-272 (init_iters = SolverConfig.max_iters) before the loop.
    """
    d0, m0, _, _ = coil_compress_svd(data, maps, c_hat0)
    counter = Counter()
    kern = make_kernel()
    a = Sense(m0, kern, weights, counter)
    y = a.weight_data(d0).reshape(-1)
    D = int(np.prod(dims))

    def reg_value(x):
        if reg == "l2":
            return 0.5 * lam * float(np.linalg.norm(x) ** 2) if lam else 0.0
        if reg == "l1-tv":
            return tv_norm_value(x, dims, lam)
        return wavelet_l1(x, dims, lam)

    def objective(x):
        counter.depth += 1
        r = a.forward(x) - y
        counter.depth -= 1
        return 0.5 * float(np.linalg.norm(r) ** 2) + reg_value(x)

    x = np.zeros(D, dtype=np.complex128)
    obj0 = objective(x)
    objs = []
    diverged = False
    L = None
    init_count = 0
    if use_init:
        before = counter.counts.get("coil_transform", 0)
        S0 = gen_sketch_matrix(v + s, v, s, c_hat0, child_seed(seed, 0), distribution, rademacher_scale)
        x = classical_sketch_solve(a, y, S0, m0, kern, weights, counter, dims, lam, reg, solver, init_iters,
                                   tol, step_scale)
        init_count = counter.counts.get("coil_transform", 0) - before
    per_outer = []
    for t in range(1, outer + 1):
        dvec = a.adjoint(a.forward(x) - y)
        S = gen_sketch_matrix(v + s, v, s, c_hat0, child_seed(seed, t), distribution,
                              rademacher_scale)
        a_s = Sense(S @ m0, kern, weights, counter)
        anchor = x

        def normal_s(u):
            return a_s.adjoint(a_s.forward(u))

        if solver == "fista":
            if L is None or not reuse_step_size:
                counter.depth += 1
                L = power_max_eig(normal_s, D) / step_scale
                counter.depth -= 1

            def grad(z):
                return normal_s(z - anchor) + dvec

            def prox(vv, st):
                return wavelet_prox(vv, dims, st, lam) if reg == "l1-wavelet" else (
                    vv / (1.0 + st * lam) if lam else vv.copy())

            x = fista(grad, prox, L, anchor, inner, tol)
        elif solver == "cg":
            b = -dvec - lam * anchor
            delta = cg(lambda u: normal_s(u) + lam * u, b, np.zeros(D, dtype=np.complex128), inner)
            x = anchor + delta
        elif solver == "pdhg":
            x = pdhg_tv(normal_s, dvec, anchor, dims, lam, inner, cg_iters, pdhg_ratio, step_scale)
        else:
            raise ValueError(solver)
        finite = bool(np.all(np.isfinite(x)))
        obj = objective(x) if finite else math.inf
        objs.append(obj)
        per_outer.append(counter.counts.get("coil_transform", 0))
        if not finite or obj > 10.0 * obj0:
            diverged = True
            break
    return ReconResult(np.where(np.isfinite(x), x, 0.0), objs, dict(counter.counts), diverged,
                       float(L) if L is not None else float("nan"), init_count, per_outer)


def classical_sketch_solve(a: "Sense", y: np.ndarray, S: np.ndarray, m0: np.ndarray, kern, weights, counter,
                           dims, lam: float, reg: str, solver: str, iters: int, tol: float,
                           step_scale: float) -> np.ndarray:
    """One-shot min 0.5||S A x - S y||^2 + g(x) (coil_sketch.py:148-159) through reconstruct
    (solvers.py:434-500): the sketched data is S applied per sample (sketching.py:106-109)."""
    a_s = Sense(S @ m0, kern, weights, counter)
    y_s = (S @ y.reshape(m0.shape[0], -1)).ravel()
    D = int(np.prod(dims))
    x0 = np.zeros(D, dtype=np.complex128)
    if solver == "cg":
        b = a_s.adjoint(y_s)
        return cg(lambda u: a_s.adjoint(a_s.forward(u)) + lam * u, b, x0, iters,
                  tol * float(np.linalg.norm(b)))
    counter.depth += 1
    L = power_max_eig(lambda u: a_s.adjoint(a_s.forward(u)), D) / step_scale
    counter.depth -= 1

    def grad(z):
        return a_s.adjoint(a_s.forward(z) - y_s)

    def prox(vv, st):
        return wavelet_prox(vv, dims, st, lam) if reg == "l1-wavelet" else (
            vv / (1.0 + st * lam) if lam else vv.copy())

    return fista(grad, prox, L, x0, iters, tol)
