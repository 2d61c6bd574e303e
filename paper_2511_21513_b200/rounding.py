"""Round-half-away-from-zero, the library-wide rounding rule (reference
rounding.py:12-21).  Kernels realise it as floorf(|t| + 0.5f) with the sign
restored (f32, csrc/quantize.cu) and (2n + d) // (2d) for integers
(csrc/params.cuh); this host/tensor helper evaluates it in the input dtype.
"""
from __future__ import annotations

import numpy as np
import torch


def round_half_away(x):
    """Nearest integer, ties away from zero, returned in the input's float dtype.

    The tie is decided on the value of |x| + 0.5 as computed in that dtype.
    Accepts numpy arrays/scalars and torch tensors (computed where they live).
    """
    if isinstance(x, torch.Tensor):
        return torch.copysign(torch.floor(torch.abs(x) + 0.5), x)
    a = np.asarray(x)
    half = a.dtype.type(0.5) if a.dtype.kind == "f" else 0.5
    return np.copysign(np.floor(np.abs(a) + half), a)
