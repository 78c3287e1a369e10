"""Device plumbing: torch owns device memory and streams; kernels are ours."""

from __future__ import annotations

import numpy as np
import torch


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2305_06482_b200 runs its operators on a CUDA device (sm_100a); "
            "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream() -> int:
    """Raw cudaStream_t of the current stream of the current device.  torch's public
    current_stream() goes through device-index and availability checks (~14 us per call on the
    box, ~1000 calls per config-0 reconstruction), so the raw accessor is used when present."""
    if _raw_stream is not None:
        return _raw_stream(torch._C._cuda_getDevice())
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def c64(a, device=None) -> torch.Tensor:
    """Contiguous complex64 CUDA tensor from a numpy array / tensor."""
    device = device or require_cuda()
    if isinstance(a, torch.Tensor):
        t = a.to(device=device, dtype=torch.complex64)
    elif isinstance(a, np.ndarray) and a.dtype == np.complex128 and a.size >= (1 << 16):
        # large complex128 arrays (maps, k-space data): copy as they are and round on the device
        # (same IEEE rounding as numpy's astype, without the host pass over the array)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device).to(torch.complex64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex64)).to(device)
    return t.contiguous()


def to_numpy128(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().astype(np.complex128)


def host_to_dev(a: np.ndarray, dtype, device=None) -> torch.Tensor:
    device = device or require_cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype).contiguous()
