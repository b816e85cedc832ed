"""Host-side tensor plumbing: accept torch CUDA tensors (the fast path) or
host arrays (numpy float32/float64/bfloat16, as a reference user passes
them), move host inputs to the device as bf16, and hand results back in
the caller's flavour."""

from __future__ import annotations

import numpy as np
import torch


def is_host(x) -> bool:
    return isinstance(x, np.ndarray) or (isinstance(x, torch.Tensor) and not x.is_cuda)


def to_device_bf16(x, name: str, device=None) -> torch.Tensor:
    """bf16, contiguous, on CUDA.  Host numpy arrays are rounded to bf16
    with round-to-nearest-even (the storage dtype of the hot path)."""
    if isinstance(x, np.ndarray):
        if x.dtype.name == "bfloat16":
            t = torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16)
        else:
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
        x = t
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor or numpy array, got {type(x).__name__}")
    if x.dtype != torch.bfloat16:
        x = x.to(torch.bfloat16)
    if not x.is_cuda:
        x = x.pin_memory().to(device or "cuda", non_blocking=True)
    return x.contiguous()


def to_host_like(t: torch.Tensor, bf16: bool):
    """Device result -> numpy (bf16 via ml_dtypes when requested)."""
    if bf16:
        import ml_dtypes
        return t.contiguous().view(torch.int16).cpu().numpy().view(ml_dtypes.bfloat16)
    return t.cpu().numpy()


def dtype_of(x) -> str:
    if isinstance(x, np.ndarray):
        return x.dtype.name
    return str(x.dtype).replace("torch.", "")
