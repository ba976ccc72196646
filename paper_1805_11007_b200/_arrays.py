"""Host/device array plumbing for the function-level API.

Every public op accepts numpy arrays or torch tensors.  Host inputs are
uploaded, the op runs on the device, and the result comes back as numpy; CUDA
tensor inputs stay on the device and the result is a CUDA tensor.
"""

from __future__ import annotations

import numpy as np

from . import _native


def is_tensor(a) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(a, torch.Tensor)


def on_device(a) -> bool:
    return is_tensor(a) and a.device.type == "cuda"


def dev(a, dtype=None):
    """CUDA tensor view/copy of `a` (contiguous, optional dtype)."""
    t, _ = _native.to_device(a, dtype)
    return t


def float_dtype_of(a):
    import torch
    if is_tensor(a):
        return a.dtype if a.dtype in (torch.float32, torch.float64) else torch.float64
    a = np.asarray(a)
    return torch.float32 if a.dtype == np.float32 else torch.float64


def back(t, host: bool):
    return t.cpu().numpy() if host else t


def empty(shape, dtype):
    torch = _native.require_cuda()
    return torch.empty(shape, dtype=dtype, device="cuda")


def zeros(shape, dtype):
    torch = _native.require_cuda()
    return torch.zeros(shape, dtype=dtype, device="cuda")


def to_numpy(a):
    if is_tensor(a):
        return a.detach().cpu().numpy()
    return np.asarray(a)
