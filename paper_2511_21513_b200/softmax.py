"""IndexSoftmax on the GPU (reference softmax.py).

    delta  = rowmax(A) - A;  delta' = min(delta, c_int)
    idx    = round(delta' (2^b - 1) / c_int)       (exact integer rounding)
    e      = lut[idx];  p = round(255 e / rowsum(e))

``index_softmax`` runs csrc/softmax_rows.cu over a materialised int32 logit
matrix (the stage operator); the fused attention kernel (csrc/attention.cu)
runs the same integer map on logits held in TMEM.  The per-element division is
the exact magic-number form documented in csrc/params.cuh.  ``build_lut`` and
``compute_c_int`` are per-call host constants (f64), exactly as the reference
computes them; every per-element operation is device work.
"""
from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import engine as E
from .gemm import MAX_SEQ_LEN, LogitMatrix
from ._tensors import is_torch, np_dtype, to_device, to_host

_C_INT_CAP = 1 << 52  # softmax.py:47


class PFormat(Enum):
    """Probability format; the value is the fixed denominator scale."""

    UINT8X255 = 255
    INT8X127 = 127


@dataclass(frozen=True)
class ExpLut:
    """2^b uint8 entries approximating 255*exp(-x) on [0, c]; last entry 0."""

    b: int
    c: float
    entries: np.ndarray


@dataclass(frozen=True)
class ClipThreshold:
    """max(1, round(c / alpha)) in logit units."""

    c_int: int


@dataclass(frozen=True)
class ProbMatrix:
    """8-bit probabilities with their fixed denominator (255 or 127)."""

    values: object
    denom_scale: int


def build_lut(b, c):
    """entries[i] = round_half_away(255 exp(-c i / (2^b - 1))), entries[-1] = 0
    (softmax.py:88-102).  Host constant, f64, as in the reference."""
    if not isinstance(b, int) or not 2 <= b <= 8:
        raise ValueError(f"b must be an int in [2, 8], got {b!r}")
    if not (math.isfinite(c) and c > 0):
        raise ValueError(f"c must be positive and finite, got {c!r}")
    return ExpLut(b=b, c=float(c), entries=E.lut_bytes(b, float(c)))


def _c_int_from_alpha(c, alpha):
    r = float(c) / float(alpha)
    ci = int(math.copysign(math.floor(abs(r) + 0.5), r))
    return max(1, min(ci, _C_INT_CAP))


def compute_c_int(c, d, s_q, s_k):
    """max(1, round(c sqrt(d) / (s_q s_k))) via alpha = s_q s_k / sqrt(d)
    (softmax.py:105-121)."""
    for name, val in (("c", c), ("d", d), ("s_q", s_q), ("s_k", s_k)):
        if not (math.isfinite(float(val)) and float(val) > 0):
            raise ValueError(f"{name} must be positive and finite, got {val!r}")
    alpha = float(s_q) * float(s_k) / math.sqrt(d)
    return ClipThreshold(c_int=_c_int_from_alpha(c, alpha))


# ---------------------------------------------------------------- dataflow audit
_audit_sink = None


@contextlib.contextmanager
def dataflow_audit(sink):
    """Collect (tag, dtype) records of tensors crossing the softmax stage
    (softmax.py:207-228), in the reference's order: logits, index_table, lut,
    [mask], prob (+ pv_in from int_attention, pipeline.py:248); grouped:
    surrogates, prob.  For the fused kernel the logits / prob / pv_in records are
    the dtypes its instruction encodings fix for the on-chip buffers (s32 TMEM
    accumulator of tcgen05.mma kind::i8; u8 / s8 A operand of the P.V MMA)."""
    global _audit_sink
    prev = _audit_sink
    _audit_sink = sink
    try:
        yield sink
    finally:
        _audit_sink = prev


_TORCH_NP = {torch.int32: np.int32, torch.uint8: np.uint8, torch.int8: np.int8,
             torch.int64: np.int64, torch.float32: np.float32}


def _note(tag, x):
    """Record (tag, dtype) of ``x``: an observed array / tensor, or -- for a buffer
    that lives only on chip inside the fused kernel (TMEM logits, smem P^) -- the
    dtype the kernel's instruction encoding fixes for it."""
    if _audit_sink is not None:
        if isinstance(x, torch.Tensor):
            dt = np.dtype(_TORCH_NP[x.dtype])
        elif isinstance(x, np.ndarray):
            dt = x.dtype
        else:
            dt = np.dtype(x)
        _audit_sink.append((tag, dt))


def _check_lut(lut):
    if not isinstance(lut, ExpLut):
        raise TypeError("lut must be an ExpLut")
    if lut.entries[0] != 255 or lut.entries[-1] != 0:
        raise ValueError("lookup table endpoints must be 255 and 0")


def _logit_values(logits):
    values = logits.values if isinstance(logits, LogitMatrix) else logits
    if not is_torch(values):
        values = np.asarray(values)
    if np_dtype(values) != np.int32 or len(values.shape) != 2:
        raise ValueError("logits must be an int32 matrix")
    if values.shape[0] != values.shape[1]:
        raise ValueError(f"logits must be square, got {tuple(values.shape)}")
    if values.shape[0] > MAX_SEQ_LEN:
        raise ValueError(f"sequence length exceeds {MAX_SEQ_LEN}")
    return values


def _prep_mask(mask, shape):
    m = to_device(mask)
    if tuple(m.shape) != tuple(shape):
        raise ValueError(f"mask shape {tuple(m.shape)} does not match logits {tuple(shape)}")
    return m.to(torch.bool)


def index_softmax(logits, c_int, lut, mask=None, p_format=PFormat.UINT8X255, threads=1):
    """Integer softmax surrogate (softmax.py:265-299) on the GPU.

    ``mask`` (bool L x L, True = excluded) removes positions from the row max
    and gives them probability 0; a fully masked row is all zero.
    """
    values = _logit_values(logits)
    _check_lut(lut)
    ci = c_int.c_int if isinstance(c_int, ClipThreshold) else int(c_int)
    if ci < 1:
        raise ValueError("c_int must be >= 1")
    ci = min(ci, _C_INT_CAP)
    numpy_in = not is_torch(values)
    lv = to_device(values, np.int32)
    _note("logits", lv)
    # the reference's u8 index table (softmax.py:124-128, :280-282) is an exact
    # magic-number division here (csrc/params.cuh); its entries are u8 indices
    _note("index_table", np.uint8)
    _note("lut", lut.entries)
    m = None
    if mask is not None:
        m = _prep_mask(mask, lv.shape)
        _note("mask", np.uint8)  # staged as u8, then bit-packed (engine.pack_mask)
    out = E.index_softmax_dev(lv, ci, lut.entries, m, p_format.value)
    if p_format is PFormat.INT8X127:
        out = out.view(torch.int8)
    _note("prob", out)
    return ProbMatrix(values=to_host(out, numpy_in), denom_scale=p_format.value)


def index_softmax_grouped(logits, group_of_column, alphas, c, lut, mask=None,
                          p_format=PFormat.UINT8X255, common_max=False, threads=1):
    """Grouped-key IndexSoftmax (softmax.py:302-399): per-group clip threshold
    c_int^(g) = max(1, round(c / alpha_g)) and, by default, a per-group row max.

    The default (per-group max) mode runs the grouped row kernel
    (csrc/softmax_rows.cu, ia_index_softmax_grouped; <= 4096 groups).  The
    diagnostic ``common_max`` mode (f64 rescaling onto the finest group's grid,
    "not part of the integer runtime path", softmax.py:324-326) and > 4096
    groups are composed from exact int64 / f64 torch ops on the device.  A single
    group is bit-identical to ``index_softmax``.
    """
    values = _logit_values(logits)
    _check_lut(lut)
    numpy_in = not is_torch(values)
    v = to_device(values, np.int32).to(torch.int64)
    n = v.shape[0]
    groups = np.asarray(group_of_column.cpu() if is_torch(group_of_column) else group_of_column)
    if groups.shape != (n,):
        raise ValueError(f"group_of_column must have shape ({n},)")
    groups = groups.astype(np.int64)
    alphas = [float(a) for a in alphas]
    if not alphas:
        raise ValueError("alphas must be non-empty")
    for g, a in enumerate(alphas):
        if not (math.isfinite(a) and a > 0):
            raise ValueError(f"alpha for group {g} must be positive, got {a!r}")
    if groups.min() < 0 or groups.max() >= len(alphas):
        raise ValueError("every column must map to a group in [0, len(alphas))")
    dev = v.device
    if not common_max and len(alphas) <= 4096:
        m = _prep_mask(mask, v.shape) if mask is not None else None
        cis = [min(_c_int_from_alpha(c, a), _C_INT_CAP) for a in alphas]
        _note("surrogates", np.uint8)
        out = E.index_softmax_grouped_dev(to_device(values, np.int32), groups, cis, lut.entries,
                                          m, p_format.value)
        if p_format is PFormat.INT8X127:
            out = out.view(torch.int8)
        _note("prob", np.int8 if p_format is PFormat.INT8X127 else np.uint8)
        return ProbMatrix(values=to_host(out, numpy_in), denom_scale=p_format.value)
    k = len(lut.entries) - 1
    lut_t = torch.as_tensor(lut.entries.astype(np.int64), device=dev)
    m8 = _prep_mask(mask, v.shape) if mask is not None else None
    e = torch.zeros(v.shape, dtype=torch.int64, device=dev)
    neg = torch.tensor(-(1 << 62), dtype=torch.int64, device=dev)
    if common_max:
        a_star = min(alphas)
        ratio = torch.as_tensor(np.array([a / a_star for a in alphas], np.float64), device=dev)
        g_t = torch.as_tensor(groups, device=dev)
        x = v.to(torch.float64) * ratio[g_t][None, :]
        resc = torch.copysign(torch.floor(torch.abs(x) + 0.5), x)
        if float(resc.abs().max()) >= float(1 << 62):
            raise ValueError("group scale ratios too large to rescale exactly")
        resc = resc.to(torch.int64)
        ci = _c_int_from_alpha(c, a_star)
        work = torch.where(m8, neg, resc) if m8 is not None else resc
        mx = work.max(dim=1).values
        delta = torch.clamp(mx[:, None] - resc, min=0)
        idx = (2 * torch.clamp(delta, max=ci) * k + ci) // (2 * ci)
        e = lut_t[idx]
    else:
        for g, alpha in enumerate(alphas):
            cols = torch.as_tensor(np.flatnonzero(groups == g), device=dev)
            if cols.numel() == 0:
                continue
            sub = v[:, cols]
            ci = _c_int_from_alpha(c, alpha)
            work = torch.where(m8[:, cols], neg, sub) if m8 is not None else sub
            mx = work.max(dim=1).values
            delta = torch.clamp(mx[:, None] - sub, min=0)
            idx = (2 * torch.clamp(delta, max=ci) * k + ci) // (2 * ci)
            e[:, cols] = lut_t[idx]
    if m8 is not None:
        e = e.masked_fill(m8, 0)
    _note("surrogates", np.uint8)
    scale = p_format.value
    s = e.sum(dim=1, keepdim=True)  # < 2^32 (L <= 65536, e <= 255)
    out = ((e * (2 * scale) + s) // torch.clamp(2 * s, min=1)).to(torch.uint8)
    if p_format is PFormat.INT8X127:
        out = out.view(torch.int8)
    _note("prob", np.int8 if p_format is PFormat.INT8X127 else np.uint8)
    return ProbMatrix(values=to_host(out, numpy_in), denom_scale=scale)
