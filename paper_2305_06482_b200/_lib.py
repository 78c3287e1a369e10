"""ctypes binding of the C ABI in include/sketchrecon_b200.h.

The shared library is built in-tree by ``paper_2305_06482_b200.build``.  There
is no fallback: if the library is missing every operator raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# SR_LIB_PATH: an alternative build of the same library (A/B measurements of a kernel change in
# one process's box session, tools only); unset -> the in-tree build
LIB_PATH = Path(os.environ.get("SR_LIB_PATH") or Path(__file__).resolve().parent / "_native" / "libsketchrecon_b200.so")

_vp = C.c_void_p
_i = C.c_int
_ll = C.c_longlong
_f = C.c_float

# name -> argtypes (restype is always int status, except the pure queries)
SIGNATURES = {
    "sr_fft_size_supported": [_i],
    "sr_fft_split": [_i, C.POINTER(_i), C.POINTER(_i)],
    "sr_cart_normal": [_vp, _vp, _vp, _ll, _vp, _ll, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp],
    "sr_cart_forward": [_vp, _vp, _ll, _vp, _vp, _vp, _vp, _ll, _vp, _vp, _i, _vp, _i, _i, _i, _i,
                        _vp, _vp, _i, _vp],
    "sr_cart_col_block": [_i],
    "sr_cart_plan_create": [_vp, _vp, _i, _i, _vp, _i, _vp, _vp],
    "sr_cart_plan_destroy": [_vp],
    "sr_cart_plan_info": [_vp] + [_vp] * 16,
    "sr_cart_plan_ws_bytes": [_vp, _i],
    "sr_cart_plan_normal": [_vp, _vp, _vp, _vp, _ll, _i, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_cart_plan_forward": [_vp, _vp, _vp, _ll, _i, _vp, _ll, _vp, _vp, _i, _vp, _vp],
    "sr_cart_plan_adjoint": [_vp, _vp, _ll, _vp, _ll, _i, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_cart_adjoint": [_vp, _ll, _vp, _ll, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i,
                        _vp, _vp, _vp, _vp, _vp, _i, _vp],
    "sr_coil_contract": [_vp, _vp, _vp, _ll, _i, _i, _i, _ll, _ll, _ll, _vp],
    "sr_coil_contract_real": [_vp, _vp, _vp, _ll, _i, _i, _i, _ll, _ll, _ll, _vp],
    "sr_wavelet_ana2": [_vp, _vp, _i, _i, _i, _ll, _i, _vp, _f, _i, _vp, _vp],
    "sr_wavelet_ana2_nblocks": [_i, _i],
    "sr_wavelet_syn2": [_vp, _vp, _i, _i, _i, _ll, _i, _vp, _vp, _f, _vp],
    "sr_wavelet_prox2": [_vp, _vp, _vp, _vp, _i, _i, _ll, _i, _i, _vp, _f, _vp, _vp, _f, _vp],
    "sr_wavelet_levels_max": [],
    "sr_wavelet_axis": [_vp, _vp, _i, _i, _i, _i, _i, _ll, _i, _i, _i, _vp, _f, _i, _i, _vp, _vp, _vp, _f, _vp],
    "sr_wavelet_axis_nblocks": [],
    "sr_reduce": [_i, _vp, _vp, _ll, _ll, _i, _vp, _vp, _vp],
    "sr_reduce_nparts": [],
    "sr_lincomb": [_vp, _vp, _vp, _vp, _vp, _f, _f, _f, _ll, _ll, _i, _vp],
    "sr_tv_dual": [_vp, _vp, _vp, _i, _i, _vp, _f, _i, _vp],
    "sr_tv_primal": [_vp, _vp, _vp, _vp, _i, _vp, _i, _vp],
    "sr_scalar_op": [_i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp],
    "sr_host_vd_poisson": [_i, _i, C.c_double, _i, C.c_ulonglong, _vp],
    "sr_cart_ws_bytes": [_i, _i, _i, _i, _i],
    "sr_cart_tune": [_i],
    "sr_cart_tune_colpf": [_i],
    "sr_cart_tune_carveout": [_i],
    "sr_cart_tune_rows": [_i, _i],
    "sr_nufft_normal": [_vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp,
                        _vp, _vp, _vp, _vp, _i, _i, _vp],
    "sr_nufft_normal_pp": [_vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp,
                           _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp],
    "sr_nufft_normal_head": [_vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp, _i,
                             _i, _vp],
    "sr_nufft_normal_tail": [_vp, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp],
    "sr_nufft_normal_slabs_ok": [_vp],
    "sr_nufft_forward": [_vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp,
                         _vp, _vp, _vp, _i, _i, _vp],
    "sr_nufft_adjoint": [_vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp,
                         _vp, _vp, _vp, _vp, _i, _i, _vp],
    "sr_nufft_partial_blocks": [_ll],
    "sr_cg_step": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _ll, _ll, _i, _i, C.c_double, _vp],
    "sr_cart3_normal": [_vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_cart3_forward": [_vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _ll, _vp, _vp, _vp, _vp],
    "sr_cart3_adjoint": [_vp, _ll, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_cart3_partial_blocks": [_ll, _i],
    "sr_nufft_plan_geom": [_vp, _ll, _i, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp],
    "sr_nufft_plan_permute": [_vp, _vp, _vp, _ll, _vp, _vp, _vp, _vp],
    "sr_nufft_plan_create": [_vp, _ll, _i, _vp, C.c_double, _i, _i, _vp, _vp],
    "sr_nufft_plan_destroy": [_vp],
    "sr_nufft_plan_info": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_nufft_plan_normal": [_vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_memcpy_d2d": [_vp, _vp, _ll, _vp],
    "sr_tsqr_r": [_vp, _ll, _i, _ll, _i, _vp, _vp],
    "sr_fft_axis": [_vp, _ll, _i, _ll, _i, _vp],
    "sr_readout_idft": [_vp, _vp, _vp, _vp, _i, _i, _ll, _vp],
}
RESTYPES = {"sr_host_vd_poisson": C.c_longlong, "sr_cart_ws_bytes": C.c_longlong,
            "sr_cart_plan_ws_bytes": C.c_longlong}

_ERRORS = {1: ValueError, 2: ValueError, 3: RuntimeError}
_MESSAGES = {1: "invalid argument or shape", 2: "unsupported transform length",
             3: "CUDA launch/runtime error"}


class NativeLibraryMissing(ImportError):
    pass


_lib = None


def lib():
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeLibraryMissing(
                f"{LIB_PATH} not built; run `python -m paper_2305_06482_b200.build` "
                "(there is no CPU fallback)")
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        for name, args in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = RESTYPES.get(name, C.c_int)
        _lib = handle
    return _lib


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise _ERRORS.get(rc, RuntimeError)(f"{name}: {_MESSAGES.get(rc, f'error {rc}')}")


def fft_split(n: int) -> tuple[int, int]:
    p, q = C.c_int(0), C.c_int(0)
    rc = lib().sr_fft_split(int(n), C.byref(p), C.byref(q))
    if rc != 0:
        raise ValueError(f"FFT length {n} is not supported by the sm_100a kernels")
    return p.value, q.value


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
