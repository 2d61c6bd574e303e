"""Batched multi-head / GQA / causal / variable-length entry point.

The reference API is single-head ("multi-head batching is a loop
over independent heads at the CLI layer").  ``int_attention_batched`` is that
loop done on the device: one launch sequence covers every (b, h) unit, and each
unit's output is bit-identical to ``int_attention(q[b, h], k[b, h // g],
v[b, h // g], AttentionConfig(mask=...))`` on the unit's valid rows
(SURVEY.md §3.5, §8d).
"""
from __future__ import annotations

import numpy as np
import torch

from . import engine as E
from ._tensors import is_torch, to_device, to_host
from .gemm import MAX_SEQ_LEN
from .pipeline import AttentionConfig


def int_attention_batched(q, k, v, *, causal=False, seq_lens=None, mask=None,
                          scale_granularity="head", cfg=None, out=None, debug=False,
                          check_finite=True):
    """Fused IntAttention over all (b, h) units.

    q: [B, H, L, d] f32; k, v: [B, Hkv, L, d] f32 with H % Hkv == 0.
    causal: key j > query i excluded.  seq_lens: [B] valid lengths (rows at or
    beyond are padding: excluded as keys, +0.0 output as queries).  mask:
    optional bool [L, L] (True = excluded) shared by all units.
    scale_granularity: "head" (one scale per (b, head) slab over its valid rows)
    or "tensor" (one global scale per Q/K/V tensor).
    cfg: AttentionConfig for b, c and p_format (granularity/mask/threads unused).
    Returns out [B, H, L, d] f32 (numpy in -> numpy out), plus a dict of stage
    tensors (quantised operands, int32 logits, u8 P, int32 acc) with debug=True.
    """
    cfg = cfg or AttentionConfig()
    if scale_granularity not in ("head", "tensor"):
        raise ValueError("scale_granularity must be 'head' or 'tensor'")
    qs = tuple(q.shape)
    ks = tuple(k.shape)
    if len(qs) != 4 or len(ks) != 4 or tuple(v.shape) != ks:
        raise ValueError(f"expected q [B,H,L,d] and k, v [B,Hkv,L,d], got {qs}, {ks}, {tuple(v.shape)}")
    B, H, L, d = qs
    if ks[0] != B or ks[2] != L or ks[3] != d or ks[1] < 1 or H % ks[1]:
        raise ValueError(f"k/v shape {ks} incompatible with q {qs}")
    if L > MAX_SEQ_LEN:
        raise ValueError(f"sequence length exceeds {MAX_SEQ_LEN}")
    if min(B, H, L, d) < 1:
        raise ValueError("empty attention problem")
    numpy_in = not is_torch(q)
    qt, kt, vt = (to_device(x, np.float32) for x in (q, k, v))
    sl = None
    if seq_lens is not None:
        sl_h = np.asarray(seq_lens.cpu() if is_torch(seq_lens) else seq_lens).astype(np.int64)
        if sl_h.shape != (B,) or (sl_h < 0).any() or (sl_h > L).any():
            raise ValueError(f"seq_lens must be [B] with values in [0, {L}]")
        sl = torch.as_tensor(sl_h.astype(np.int32)).to(qt.device)
    mt = None
    if mask is not None:
        mt = to_device(mask).to(torch.bool)
        if tuple(mt.shape) != (L, L):
            raise ValueError(f"mask must be {L}x{L}, got {tuple(mt.shape)}")
    o = None if out is None else out
    res = E.attention(qt, kt, vt, causal=causal, seq_lens=sl, mask=mt,
                      scale_granularity=scale_granularity, b=cfg.b, c=cfg.c,
                      p_scale=cfg.p_format.value, out=o, debug=debug,
                      check_finite=check_finite)
    if debug:
        res, dbg = res
        return to_host(res, numpy_in), dbg
    return to_host(res, numpy_in)
