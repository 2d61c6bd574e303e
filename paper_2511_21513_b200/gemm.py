"""Exact integer GEMMs on tcgen05 (reference gemm.py).

``matmul_int8`` / ``gemm_qk`` / ``gemm_pv`` run csrc/gemm_i8.cu
(``tcgen05.mma.kind::i8``, s32 accumulation in TMEM): exact by construction,
where the reference reaches exactness through float BLAS with a mantissa bound
(gemm.py:45-59).  These are the stage-level operators; ``int_attention``
never materialises their L x L outputs (csrc/attention.cu fuses them).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import engine as E
from ._tensors import is_torch, np_dtype, to_device, to_host
from .quantize import PER_TENSOR, QuantizedMatrix

MAX_HEAD_DIM = 131070  # d * 127 * 127 fits int32 (gemm.py:25)
MAX_SEQ_LEN = 65536    # L * 255 * 127 fits int32 (gemm.py:26)


@dataclass(frozen=True)
class LogitMatrix:
    """Exact int32 logits ``values[i, j] = q_i . k_j`` and alpha = s_q s_k / sqrt(d)."""

    values: object
    alpha: float


def matmul_int8(a_values, b_t_values, threads=None):
    """Exact int32 ``a @ b_t.T`` of two int8 matrices (gemm.py:70-85).

    ``threads`` is accepted for API compatibility; the GPU ignores it.
    """
    if np_dtype(a_values) != np.int8 or np_dtype(b_t_values) != np.int8:
        raise ValueError("matmul_int8 expects int8 operands")
    if a_values.shape[1] != b_t_values.shape[1]:
        raise ValueError(f"inner dimensions differ: {tuple(a_values.shape)} vs {tuple(b_t_values.shape)}")
    if a_values.shape[1] > MAX_HEAD_DIM:
        raise ValueError(f"head dimension exceeds accumulator bound {MAX_HEAD_DIM}")
    numpy_in = not is_torch(a_values)
    a = to_device(a_values)
    b = to_device(b_t_values)
    return to_host(E.gemm_i8(a, b, a_signed=True), numpy_in)


def gemm_qk(qhat, khat, threads=None):
    """Logit GEMM plus alpha (gemm.py:88-106); per-tensor scales only."""
    for name, m in (("qhat", qhat), ("khat", khat)):
        if not isinstance(m, QuantizedMatrix):
            raise TypeError(f"{name} must be a QuantizedMatrix")
        if m.granularity.kind != PER_TENSOR:
            raise ValueError("gemm_qk requires per-tensor scales; use matmul_int8 plus "
                             "index_softmax_grouped for grouped quantization")
    values = matmul_int8(qhat.values, khat.values)
    d = qhat.values.shape[1]
    sq = float(qhat.scales[0])
    sk = float(khat.scales[0])
    return LogitMatrix(values=values, alpha=sq * sk / math.sqrt(d))


def gemm_pv(phat, vhat, threads=None):
    """Exact int32 ``phat @ vhat`` (gemm.py:109-133): phat uint8 (or int8 in the
    INT8X127 ablation) [L, L], vhat int8 [L, d]."""
    values = vhat.values if isinstance(vhat, QuantizedMatrix) else vhat
    pdt = np_dtype(phat)
    if pdt not in (np.dtype(np.uint8), np.dtype(np.int8)):
        raise ValueError(f"phat must be uint8 or int8, got {pdt}")
    if np_dtype(values) != np.int8:
        raise ValueError("vhat must hold int8 values")
    if len(phat.shape) != 2 or phat.shape[0] != phat.shape[1]:
        raise ValueError(f"phat must be square, got {tuple(phat.shape)}")
    if phat.shape[1] != values.shape[0]:
        raise ValueError(f"dimension mismatch: {tuple(phat.shape)} @ {tuple(values.shape)}")
    if phat.shape[1] > MAX_SEQ_LEN:
        raise ValueError(f"sequence length exceeds accumulator bound {MAX_SEQ_LEN}")
    numpy_in = not is_torch(phat)
    p = to_device(phat)
    v = to_device(values)
    out = E.gemm_i8(p, v.t().contiguous(), a_signed=(pdt == np.dtype(np.int8)))
    return to_host(out, numpy_in)


def gemm_real(a, b_transposed, threads=None):
    """f32 ``a @ b_transposed.T`` for the reference pipelines (gemm.py:136-143);
    cuBLAS fp32 on the device (TF32 disabled).  Not on the integer path."""
    numpy_in = not is_torch(a)
    x = to_device(a, np.float32)
    y = to_device(b_transposed, np.float32)
    if x.shape[1] != y.shape[1]:
        raise ValueError(f"inner dimensions differ: {tuple(x.shape)} vs {tuple(y.shape)}")
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        out = x @ y.T
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return to_host(out, numpy_in)
