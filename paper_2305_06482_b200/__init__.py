"""B200-native (sm_100a) sketched SENSE normal operator and coil-sketched reconstruction.

Drop-in for the operator / solver API of the reference package ``sketchrecon``
(arXiv 2305.06482 reference implementation, /root/reference/pkg/src/sketchrecon):
same class and function names, argument meaning and errors; the arithmetic
runs in hand-written CUDA kernels (csrc/, C ABI in include/sketchrecon_b200.h)
on device-resident complex64 data.  There is no CPU fallback.

Import is light: the native library and torch CUDA state are touched on first use.
"""

from .linops import (CartesianMaskOp, CenteredFFTOp, ComposeOp, CostCounter, DiagonalOp, GridShape,
                     IdentityOp, Image, LinOp, Trajectory, WaveletOp, dot_test, make_fourier_kernel,
                     max_eig_power)
from .rng import child_seed, seed_stream

__all__ = [
    "GridShape", "Image", "Trajectory", "LinOp", "CostCounter", "IdentityOp", "DiagonalOp", "ComposeOp",
    "CenteredFFTOp", "CartesianMaskOp", "WaveletOp", "make_fourier_kernel", "max_eig_power", "dot_test",
    "seed_stream", "child_seed",
]
