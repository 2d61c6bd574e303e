"""Symmetric INT8 quantisation on the GPU (reference quantize.py).

Same types and signatures as the reference: ``QuantGranularity``,
``QuantizedMatrix``, ``quantize_symmetric``, ``dequantize``.  The arithmetic
runs in csrc/quantize.cu: a grid-wide max|x| (exact, float-bit atomics) and an
IEEE f32 quantise pass, ``scale = max(1e-12f, amax) / 127f``,
``q = clip(round_half_away(x / scale), -127, 127)`` (quantize.py:104-123).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import engine as E
from ._tensors import is_torch, to_device, to_host

EPS = 1e-12
PER_TENSOR = "per_tensor"
PER_ROW_GROUP = "per_row_group"
PER_COL_GROUP = "per_col_group"


@dataclass(frozen=True)
class QuantGranularity:
    """One scale for the whole matrix, or one per ``group_size`` consecutive
    rows / columns (quantize.py:26-57)."""

    kind: str = PER_TENSOR
    group_size: int | None = None

    @classmethod
    def per_tensor(cls):
        return cls(PER_TENSOR, None)

    @classmethod
    def per_row_group(cls, group_size):
        return cls(PER_ROW_GROUP, int(group_size))

    @classmethod
    def per_col_group(cls, group_size):
        return cls(PER_COL_GROUP, int(group_size))

    def num_groups(self, shape):
        rows, cols = shape
        if self.kind == PER_TENSOR:
            return 1
        if self.group_size is None or self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        extent = rows if self.kind == PER_ROW_GROUP else cols
        if extent % self.group_size:
            raise ValueError(f"group_size {self.group_size} does not divide dimension {extent}")
        return extent // self.group_size


@dataclass(frozen=True)
class QuantizedMatrix:
    """int8 ``values`` with positive ``scales`` (X ~ scale(g) * values in group g).

    ``values``/``scales`` are numpy arrays when the input was numpy and CUDA
    tensors when it was a torch tensor.
    """

    values: object
    scales: object
    granularity: QuantGranularity

    @property
    def shape(self):
        return tuple(self.values.shape)

    def scale_grid(self):
        """Scales broadcast to the matrix shape (quantize.py:74-89)."""
        rows, cols = self.shape
        g = self.granularity
        s = self.scales
        if is_torch(s):
            if g.kind == PER_TENSOR:
                return s.reshape(1, 1).expand(rows, cols)
            if g.kind == PER_ROW_GROUP:
                return s.repeat_interleave(g.group_size).reshape(rows, 1).expand(rows, cols)
            return s.repeat_interleave(g.group_size).reshape(1, cols).expand(rows, cols)
        s = np.asarray(s)
        if g.kind == PER_TENSOR:
            return np.broadcast_to(s.reshape(1, 1), (rows, cols))
        if g.kind == PER_ROW_GROUP:
            return np.broadcast_to(np.repeat(s, g.group_size)[:, None], (rows, cols))
        return np.broadcast_to(np.repeat(s, g.group_size)[None, :], (rows, cols))


def _quantize_dev(x: torch.Tensor, granularity: QuantGranularity):
    """x: f32 [R, C] CUDA.  Returns (int8 [R, C], f32 scales [G]) on device."""
    R, C = x.shape
    kind = granularity.kind
    try:
        G = granularity.num_groups((R, C))
        bad_gran = None
    except ValueError as e:  # the reference checks finiteness first (quantize.py:109-111)
        G, bad_gran = 1, e
    ws = E.Workspace(G, x.device)
    if kind == PER_COL_GROUP and bad_gran is None:
        _lib.check(_lib.load().ia_quant_amax_cols(E._p(x), R, C, granularity.group_size,
                                                   E._p(ws.amax), E._p(ws.err), E._stream()),
                   "amax")
    elif kind == PER_ROW_GROUP and bad_gran is None:
        gs = granularity.group_size
        E.amax_rows(x, R // gs, gs, C, ws.amax, ws.err)
    else:
        E.amax_rows(x, 1, R, C, ws.amax, ws.err)
    E.raise_if_nonfinite(ws.err)
    if bad_gran is not None:
        raise bad_gran
    E.scales_from_amax(ws.amax, ws.scales)
    pitch = (C + 3) // 4 * 4
    out = torch.empty((R, pitch), dtype=torch.int8, device=x.device)
    if kind == PER_COL_GROUP:
        E.quantize_rows(x, 1, R, C, ws.scales, out, pitch, mode=_lib.IA_QMODE_COLS,
                        col_group=granularity.group_size)
    elif kind == PER_ROW_GROUP:
        gs = granularity.group_size
        E.quantize_rows(x, R // gs, gs, C, ws.scales, out, pitch)
    else:
        E.quantize_rows(x, 1, R, C, ws.scales, out, pitch)
    values = out if pitch == C else out[:, :C].contiguous()
    return values, ws.scales


def quantize_symmetric(x, granularity=QuantGranularity.per_tensor()):
    """Quantise a real matrix to int8 with symmetric per-group scales (GPU)."""
    numpy_in = not is_torch(x)
    ndim = x.dim() if is_torch(x) else np.ndim(x)
    if ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={ndim}")
    xt = to_device(x, np.float32)
    if xt.numel() == 0:
        raise ValueError("zero-size matrix cannot be quantized")
    values, scales = _quantize_dev(xt, granularity)
    return QuantizedMatrix(values=to_host(values, numpy_in), scales=to_host(scales, numpy_in),
                           granularity=granularity)


def dequantize(q: QuantizedMatrix):
    """scale(g) * value elementwise in f32 (quantize.py:126-128), on the GPU."""
    numpy_in = not is_torch(q.values)
    v = to_device(q.values, np.int8)
    s = to_device(q.scales, np.float32)
    R, C = v.shape
    g = q.granularity
    out = torch.empty((R, C), dtype=torch.float32, device=v.device)
    if g.kind == PER_COL_GROUP:
        mode, group = _lib.IA_QMODE_COLS, g.group_size
    elif g.kind == PER_ROW_GROUP:
        mode, group = _lib.IA_QMODE_ROWS, g.group_size
    else:
        mode, group = _lib.IA_QMODE_ROWS, R
    _lib.check(_lib.load().ia_dequantize(E._p(v), R, C, mode, group, E._p(s), E._p(out),
                                         E._stream()), "dequantize")
    return to_host(out, numpy_in)
