"""Seeded synthetic inputs with the shapes and value distributions of BASELINE.json.

The reference's own generators (simulate.py) only draw Shepp-Logan phantoms,
1-D line masks and radial spokes; the BASELINE configs need random-ellipse
phantoms, Gaussian ring/cylinder coils, variable-density Poisson-disc masks
(SURVEY.md Appendix A).  Everything here is deterministic given the seed, and
the same arrays are handed to the GPU path and to the oracle.
Coordinates follow the reference convention: normalised [-1, 1) per axis
(simulate.py:99-105), FOV = 2 normalised units.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib


def _axes(dims):
    return [(np.arange(n) - (n - 1) / 2.0) * (2.0 / n) for n in dims]


def random_ellipses(dims, n_ellipses: int, rng: np.random.Generator, smooth_phase: bool = True,
                    planes: tuple[int, int] | None = None) -> np.ndarray:
    """Sum of random ellipses/ellipsoids: intensity U[0.2,1], semi-axes U[0.05,0.4]*FOV,
    random rotation; times exp(i pi (0.5 x^2 + 0.3 y)) (BASELINE config 0).
    planes = (lo, hi) evaluates only those indices of axis 0 (same draws, same values):
    a rank builds just its slab of a sharded volume."""
    axes = _axes(dims)
    if planes is not None:
        axes[0] = axes[0][planes[0]:planes[1]]
    grids = np.meshgrid(*axes, indexing="ij")
    img = np.zeros(tuple(len(a) for a in axes))
    fov = 2.0
    for _ in range(n_ellipses):
        amp = rng.uniform(0.2, 1.0)
        semi = rng.uniform(0.05, 0.4, size=len(dims)) * fov
        cen = rng.uniform(-0.4, 0.4, size=len(dims))
        coords = [g - c for g, c in zip(grids, cen)]
        if len(dims) == 2:
            th = rng.uniform(0, np.pi)
            u = math.cos(th) * coords[0] + math.sin(th) * coords[1]
            v = -math.sin(th) * coords[0] + math.cos(th) * coords[1]
            inside = (u / semi[0]) ** 2 + (v / semi[1]) ** 2 <= 1.0
        else:
            th = rng.uniform(0, np.pi)
            u = math.cos(th) * coords[1] + math.sin(th) * coords[2]
            v = -math.sin(th) * coords[1] + math.cos(th) * coords[2]
            inside = (coords[0] / semi[0]) ** 2 + (u / semi[1]) ** 2 + (v / semi[2]) ** 2 <= 1.0
        img = img + amp * inside
    if smooth_phase:
        x, y = grids[-1], grids[-2]
        return img * np.exp(1j * np.pi * (0.5 * x ** 2 + 0.3 * y))
    return img.astype(np.complex128)


def coil_centres(n_coils: int, ndim: int, rng: np.random.Generator, radius: float = 1.5):
    """Coil centres on a circle (2-D) / cylinder (3-D) of radius `radius` FOV."""
    fov = 2.0
    ang = 2 * np.pi * np.arange(n_coils) / n_coils + rng.uniform(0, 2 * np.pi / n_coils)
    cen = np.zeros((n_coils, ndim))
    cen[:, -1] = radius * fov * np.cos(ang) / 2
    cen[:, -2] = radius * fov * np.sin(ang) / 2
    if ndim == 3:
        cen[:, 0] = rng.uniform(-0.5, 0.5, n_coils)
    phase = rng.uniform(0, 2 * np.pi, n_coils)
    return cen, phase


def gaussian_coil_maps(dims, n_coils: int, rng: np.random.Generator, radius: float = 1.5,
                       sigma: float = 0.6, xp=np, device=None):
    """Gaussian coils, sigma = 0.6 FOV, random phase each, SOS normalised to 1.

    xp = numpy (host, complex128) or torch (device, complex64; for large batches).
    """
    cen, phase = coil_centres(n_coils, len(dims), rng, radius)
    s = sigma * 2.0
    if xp is np:
        grids = np.meshgrid(*_axes(dims), indexing="ij")
        maps = np.empty((n_coils,) + tuple(dims), dtype=np.complex128)
        for c in range(n_coils):
            r2 = sum((g - cc) ** 2 for g, cc in zip(grids, cen[c]))
            maps[c] = np.exp(-r2 / (2 * s * s)) * np.exp(1j * phase[c])
        maps /= np.sqrt(np.sum(np.abs(maps) ** 2, axis=0, keepdims=True))
        return maps.reshape(n_coils, -1)
    import torch
    axes = [torch.as_tensor(a, dtype=torch.float32, device=device) for a in _axes(dims)]
    grids = torch.meshgrid(*axes, indexing="ij")
    out = torch.empty((n_coils,) + tuple(dims), dtype=torch.complex64, device=device)
    for c in range(n_coils):
        r2 = sum((g - float(cc)) ** 2 for g, cc in zip(grids, cen[c]))
        mag = torch.exp(-r2 / (2 * s * s))
        out[c] = torch.polar(mag, torch.full_like(mag, float(phase[c])))
    out /= torch.sqrt(torch.sum(torch.abs(out) ** 2, dim=0, keepdim=True))
    return out.reshape(n_coils, -1)


def vd_poisson_mask(dims, accel: float, calib: int, seed: int) -> np.ndarray:
    """Variable-density Poisson-disc mask (bool, dims) via the native host generator."""
    ny, nx = dims
    m = np.zeros(ny * nx, dtype=np.uint8)
    n = _lib.lib().sr_host_vd_poisson(int(ny), int(nx), float(accel), int(calib), int(seed) & (2 ** 64 - 1),
                                       m.ctypes.data)
    if n < 0:
        raise ValueError("bad mask arguments")
    return m.reshape(ny, nx).astype(bool)


def vd_poisson_masks(dims, accel: float, calib: int, seeds) -> list[np.ndarray]:
    """Many masks in parallel host threads (the native generator releases the GIL)."""
    import concurrent.futures as cf
    import os
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(seeds), os.cpu_count() or 1))) as ex:
        return list(ex.map(lambda s: vd_poisson_mask(dims, accel, calib, s), seeds))


def mask_points(mask: np.ndarray) -> np.ndarray:
    """Integer centered bins of a mask in argwhere (row-major) order (cartesian-mask trajectory)."""
    return np.argwhere(mask).astype(np.float64) - np.array([n // 2 for n in mask.shape], dtype=np.float64)


def golden_angle_radial(n_spokes: int, n_read: int, dims) -> np.ndarray:
    """Golden-angle radial spokes, k in [-pi, pi) rad = [-n/2, n/2) cycles/FOV (simulate.py:267-289)."""
    ga = 0.6180339887498949 * np.pi
    ang = np.arange(n_spokes) * ga
    r = (np.arange(n_read) - n_read // 2) / n_read  # [-1/2, 1/2)
    pts = np.stack([np.outer(np.sin(ang), r).ravel() * dims[0],
                    np.outer(np.cos(ang), r).ravel() * dims[1]], axis=1)
    lim = np.array(dims, dtype=np.float64) / 2
    return np.clip(pts, -lim, lim * (1 - 1e-9))


def complex_noise(shape, sigma: float, rng: np.random.Generator) -> np.ndarray:
    """Complex Gaussian noise, std sigma/sqrt(2) per component (simulate.py:347-352)."""
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * (sigma / math.sqrt(2.0))


def cones_3d(dims, n_cones: int = 32, n_readouts: int = 18000, n_samples: int = 512,
             turns: float = 4.0, seed: int = 0) -> np.ndarray:
    """3-D conical-spiral trajectory (BASELINE config 4), cycles/FOV per axis.

    `n_cones` polar angles uniform in (0, pi/2], mirrored to both hemispheres;
    interleaves per cone proportional to sin(theta) (about `n_readouts` in total);
    each readout a conical spiral of `n_samples` samples whose radius grows
    linearly to k_max = pi rad.  The cone axis is the last image axis.  k is
    scaled by (1 - 1e-6) so every coordinate lies in [-n/2, n/2) as
    Trajectory.validate_for requires (linops.py:130-140).
    """
    rng = np.random.default_rng(seed)
    th = np.arange(1, n_cones + 1) * (np.pi / 2) / n_cones
    weights = np.sin(th)
    per = np.maximum(1, np.round(weights / weights.sum() * (n_readouts / 2))).astype(int)
    t = np.arange(n_samples) / n_samples  # radius fraction in [0, 1)
    out = []
    for theta, n_il in zip(th, per):
        for sign in (1.0, -1.0):
            phi0 = rng.uniform(0, 2 * np.pi) + 2 * np.pi * np.arange(n_il)[:, None] / n_il
            phi = phi0 + 2 * np.pi * turns * t[None, :]
            r = np.pi * t[None, :]
            kz = sign * r * np.cos(theta)
            kx = r * np.sin(theta) * np.cos(phi)
            ky = r * np.sin(theta) * np.sin(phi)
            out.append(np.stack([kx.ravel(), ky.ravel(), np.broadcast_to(kz, kx.shape).ravel()], axis=1))
    k = np.concatenate(out, axis=0) * (1 - 1e-6)
    n = np.asarray(dims, dtype=np.float64)
    return k * n / (2 * np.pi)


def coil_maps_cylinder(dims, n_coils: int, rng: np.random.Generator, radius: float = 1.5, sigma: float = 0.6,
                       xp=np, device=None):
    """3-D Gaussian coils on a cylinder around the last axis (BASELINE configs 2, 4)."""
    return gaussian_coil_maps(dims, n_coils, rng, radius=radius, sigma=sigma, xp=xp, device=device)
