"""numpy <-> device plumbing for the drop-in API.

Functions accept numpy arrays (the reference's types) or torch tensors.
numpy inputs are copied to the current CUDA device and results come back as
numpy; torch CUDA inputs stay on their device and results are torch CUDA
tensors.  Nothing here computes -- all arithmetic is in the sm_100a library.
"""

from __future__ import annotations

import numpy as np
import torch

_NP2T = {np.dtype(np.complex64): torch.complex64, np.dtype(np.complex128): torch.complex128,
         np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def device_of(*xs) -> torch.device:
    for x in xs:
        if is_torch(x) and x.is_cuda:
            return x.device
    if not torch.cuda.is_available():
        from .errors import NativeLibraryError
        raise NativeLibraryError("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def shape(x) -> tuple:
    return tuple(x.shape)


def np_dtype(x) -> np.dtype:
    if is_torch(x):
        return np.dtype({torch.complex64: np.complex64, torch.complex128: np.complex128,
                         torch.float64: np.float64, torch.float32: np.float32}[x.dtype])
    return np.asarray(x).dtype


def complex_type(*xs) -> np.dtype:
    """numpy's promotion of the operands, lifted to complex (the reference
    multiplies complex arrays by these, so the result is complex)."""
    dt = np.result_type(*[np_dtype(x) for x in xs])
    return np.dtype(np.complex64) if dt in (np.complex64, np.float32) else np.dtype(np.complex128)


def to_dev(x, dtype: np.dtype, device: torch.device) -> torch.Tensor:
    tdt = _NP2T[np.dtype(dtype)]
    if is_torch(x):
        t = x.to(device=device)
        if not t.is_complex() and tdt.is_complex:
            t = t.to(torch.float64 if tdt == torch.complex128 else torch.float32)
        return t.to(tdt).contiguous()
    a = np.ascontiguousarray(np.asarray(x).astype(dtype, copy=False))
    return torch.from_numpy(a).to(device, non_blocking=False)


def out(t: torch.Tensor, as_numpy: bool, dtype: np.dtype | None = None):
    if dtype is not None and np.dtype(dtype) != np_dtype(t):
        want = _NP2T[np.dtype(dtype)]
        t = t.real.to(want) if (t.is_complex() and not want.is_complex) else t.to(want)
    return t.cpu().numpy() if as_numpy else t
