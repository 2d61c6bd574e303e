"""Host <-> device plumbing for the drop-in API.

numpy inputs are copied to the current CUDA device and results come back as
numpy (the reference's contract); torch tensors stay on the device.
"""
from __future__ import annotations

import numpy as np
import torch

from .engine import require_device


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


_NP2T = {np.dtype(np.float32): torch.float32, np.dtype(np.int8): torch.int8,
         np.dtype(np.uint8): torch.uint8, np.dtype(np.int32): torch.int32,
         np.dtype(np.bool_): torch.bool, np.dtype(np.float64): torch.float64,
         np.dtype(np.int64): torch.int64}


def np_dtype(x) -> np.dtype:
    if is_torch(x):
        return np.dtype(str(x.dtype).replace("torch.", "").replace("bool", "bool_"))
    return np.asarray(x).dtype


def to_device(x, dtype=None) -> torch.Tensor:
    """Contiguous CUDA tensor of `dtype` (numpy dtype or None to keep)."""
    dev = require_device()
    if is_torch(x):
        t = x
        if dtype is not None:
            t = t.to(_NP2T[np.dtype(dtype)])
        return t.to(dev).contiguous()
    a = np.asarray(x)
    if dtype is not None:
        a = a.astype(dtype, copy=False)
    a = np.ascontiguousarray(a)
    if a.dtype == np.bool_:
        return torch.from_numpy(a.view(np.uint8)).to(dev).to(torch.bool)
    return torch.from_numpy(a).to(dev)


def to_host(t: torch.Tensor, like_numpy: bool):
    if not like_numpy:
        return t
    return t.detach().cpu().numpy()
