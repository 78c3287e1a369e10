"""Pseudo-replica inverse g-factor on the device (metrics.py:157-211 of the reference).

The reference draws, per trial i, complex Gaussian noise from ``seed_stream(seed, i)``
(full data first, then undersampled), adds it to the clean full / undersampled
k-space, reconstructs both with a deterministic ``recon(op, y) -> Image`` and returns
``sigma_full * sqrt(R) / sigma_under`` on the object support.  Here the clean data come
from the device forward operators, the per-trial reconstructions are whatever device
reconstruction ``recon`` runs (e.g. ``solvers.reconstruct`` with the l2 regulariser ->
the device CG), and the pixelwise standard deviations are accumulated on the device in
float64.  The noise draws stay on the host so they are bit-identical to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from .linops import Image
from .rng import seed_stream

__all__ = ["GFactorMap", "gfactor_montecarlo"]


@dataclass
class GFactorMap:
    inverse_g: np.ndarray  # (D,) nonnegative, zero outside the mask
    mask: np.ndarray       # (D,) bool: support with nondegenerate variance
    trials: int
    R: float


def gfactor_montecarlo(recon, a_full, a_under, x_true: Image, noise_sigma: float, trials: int, R: float,
                       seed: int, support_rel_threshold: float = 1e-3) -> GFactorMap:
    """Inverse g-factor map by pseudo-replicas (metrics.py:157-211)."""
    if trials < 2:
        raise ValueError("need at least 2 trials")
    if noise_sigma <= 0:
        raise ValueError("noise_sigma must be positive")
    dev = dv.require_cuda()
    xt = dv.c64(x_true.values, dev)
    clean_full = dv.to_numpy128(a_full.forward_unweighted(xt))
    clean_under = dv.to_numpy128(a_under.forward_unweighted(xt))
    scale = noise_sigma / np.sqrt(2.0)
    D = x_true.shape.size
    recs = [[], []]
    for i in range(trials):
        g = seed_stream(seed, i)
        n_full = scale * (g.standard_normal(clean_full.shape) + 1j * g.standard_normal(clean_full.shape))
        n_under = scale * (g.standard_normal(clean_under.shape) + 1j * g.standard_normal(clean_under.shape))
        y_full = a_full.weight_data(clean_full + n_full)
        y_under = a_under.weight_data(clean_under + n_under)
        for k, (op, y) in enumerate(((a_full, y_full), (a_under, y_under))):
            r = recon(op, y)
            v = r.values if isinstance(r, Image) else r
            recs[k].append(dv.c64(v, dev).to(torch.complex128))
    # two-pass (mean, then squared deviations) like np.std, in float64
    std = []
    for k in range(2):
        st = torch.stack(recs[k])
        mean = st.mean(dim=0)
        std.append(torch.sqrt(torch.mean(torch.abs(st - mean) ** 2, dim=0)))
    std_full, std_under = std
    mag = torch.abs(xt.to(torch.complex128))
    support = mag > support_rel_threshold * mag.max()
    degenerate = std_under <= np.finfo(float).tiny
    mask = support & ~degenerate
    inv = torch.zeros(D, dtype=torch.float64, device=dev)
    inv[mask] = std_full[mask] * np.sqrt(R) / std_under[mask]
    return GFactorMap(inverse_g=inv.cpu().numpy(), mask=mask.cpu().numpy(), trials=trials, R=R)
