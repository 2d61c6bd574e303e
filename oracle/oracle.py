"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` arm may import this module -- as the checker, never as
the thing measured or shipped.  The product package never imports it.

The heavy lifting is in intattn_oracle.c (a plain-C restatement of the
reference path, see its header).  ``build_lut`` is restated here in numpy
because the reference builds its table with numpy's f64 ``exp``
(softmax.py:88-102); using the same exp keeps the table bytes identical.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

P_UINT8X255 = 255
P_INT8X127 = 127


def build() -> str:
    """Compile liboracle.so in place (gcc; see Makefile)."""
    src = os.path.join(_HERE, "intattn_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.ia_or_amax.restype = ctypes.c_float
        L.ia_or_amax.argtypes = [P, i64, P]
        L.ia_or_scale.restype = ctypes.c_float
        L.ia_or_scale.argtypes = [ctypes.c_float]
        L.ia_or_quantize.argtypes = [P, i64, ctypes.c_float, P]
        L.ia_or_c_int.restype = i64
        L.ia_or_c_int.argtypes = [ctypes.c_double, i64, ctypes.c_float, ctypes.c_float]
        L.ia_or_matmul_s8.argtypes = [P, P, i64, i64, i64, P]
        L.ia_or_gemm_pv.argtypes = [P, P, i64, i64, i64, P]
        L.ia_or_index_softmax.argtypes = [P, i64, i64, i64, P, ctypes.c_int,
                                          ctypes.c_int, P, P]
        L.ia_or_attention_batched.restype = ctypes.c_int
        L.ia_or_attention_batched.argtypes = [
            P, P, P, i64, i64, i64, i64, i64, P, ctypes.c_int, P, ctypes.c_int,
            ctypes.c_double, P, ctypes.c_int, ctypes.c_int, i64, ctypes.c_int,
            P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# Host-side constants (numpy, as the reference computes them)
# --------------------------------------------------------------------------

def build_lut(b: int = 5, c: float = 6.6) -> np.ndarray:
    """lut[i] = round_half_away(255*exp(-c*i/(2^b-1))) in f64, lut[last] = 0
    (softmax.py:88-102; rounding.py:12-21)."""
    n = 1 << b
    x = 255.0 * np.exp(-c * np.arange(n, dtype=np.float64) / (n - 1))
    e = np.copysign(np.floor(np.abs(x) + 0.5), x).astype(np.uint8)
    e[n - 1] = 0
    return e


def index_table(c_int: int, n_entries: int) -> np.ndarray:
    """itab[delta] = (2*delta*k + c)//(2c) (softmax.py:124-128)."""
    k = n_entries - 1
    delta = np.arange(c_int, dtype=np.int64)
    return ((2 * delta * k + c_int) // (2 * c_int)).astype(np.uint8)


# --------------------------------------------------------------------------
# Stage functions (small sizes; used by per-stage parity tests)
# --------------------------------------------------------------------------

def quantize_tensor(x: np.ndarray):
    """Per-tensor quantise_symmetric: returns (int8 values, f32 scale)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    bad = ctypes.c_int(0)
    amax = lib().ia_or_amax(_p(x), x.size, ctypes.byref(bad))
    if bad.value:
        raise ValueError("input contains non-finite elements")
    s = np.float32(lib().ia_or_scale(amax))
    out = np.empty(x.shape, np.int8)
    lib().ia_or_quantize(_p(x), x.size, s, _p(out))
    return out, s


def quantize_groups(x: np.ndarray, n_groups: int):
    """Row-major contiguous groups (per-row-group / per-head): (values, scales)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    flat = x.reshape(n_groups, -1)
    out = np.empty(flat.shape, np.int8)
    scales = np.empty(n_groups, np.float32)
    for g in range(n_groups):
        bad = ctypes.c_int(0)
        amax = lib().ia_or_amax(_p(flat[g]), flat.shape[1], ctypes.byref(bad))
        if bad.value:
            raise ValueError("input contains non-finite elements")
        scales[g] = lib().ia_or_scale(amax)
        lib().ia_or_quantize(_p(flat[g]), flat.shape[1], scales[g], _p(out[g]))
    return out.reshape(x.shape), scales


def c_int(c: float, d: int, s_q: float, s_k: float) -> int:
    return int(lib().ia_or_c_int(float(c), int(d), float(s_q), float(s_k)))


def matmul_s8(a: np.ndarray, b_t: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.int8)
    b_t = np.ascontiguousarray(b_t, np.int8)
    out = np.empty((a.shape[0], b_t.shape[0]), np.int32)
    lib().ia_or_matmul_s8(_p(a), _p(b_t), a.shape[0], b_t.shape[0], a.shape[1], _p(out))
    return out


def gemm_pv(p: np.ndarray, v: np.ndarray) -> np.ndarray:
    p = np.ascontiguousarray(p).view(np.uint8)
    v = np.ascontiguousarray(v, np.int8)
    out = np.empty((p.shape[0], v.shape[1]), np.int32)
    lib().ia_or_gemm_pv(_p(p), _p(v), p.shape[0], p.shape[1], v.shape[1], _p(out))
    return out


def index_softmax(logits: np.ndarray, ci: int, lut: np.ndarray, mask=None,
                  p_scale: int = P_UINT8X255) -> np.ndarray:
    logits = np.ascontiguousarray(logits, np.int32)
    lut = np.ascontiguousarray(lut, np.uint8)
    m8 = None if mask is None else np.ascontiguousarray(mask).astype(np.uint8)
    out = np.empty(logits.shape, np.uint8)
    lib().ia_or_index_softmax(_p(logits), logits.shape[0], logits.shape[1], int(ci),
                              _p(lut), lut.size, int(p_scale), _p(m8), _p(out))
    return out


def int_attention(q, k, v, b=5, c=6.6, mask=None, p_scale=P_UINT8X255):
    """Single-head reference pipeline (pipeline.py:202-256) -> f32 [L, d]."""
    q = np.ascontiguousarray(q, np.float32)
    out, _ = attention_batched(q[None, None], np.asarray(k, np.float32)[None, None],
                               np.asarray(v, np.float32)[None, None], mask=mask,
                               b=b, c=c, p_scale=p_scale)
    return out[0, 0]


def attention_batched(q, k, v, *, causal=False, seq_lens=None, mask=None,
                      scale_granularity="head", b=5, c=6.6, p_scale=P_UINT8X255,
                      row_stride=1, threads=0, lut=None, scales=None):
    """Batched oracle (see ia_or_attention_batched).  Returns (out, info)."""
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    B, H, L, d = q.shape
    Hkv = k.shape[1]
    lut = build_lut(b, c) if lut is None else np.ascontiguousarray(lut, np.uint8)
    sl = None if seq_lens is None else np.ascontiguousarray(seq_lens, np.int32)
    m8 = None if mask is None else np.ascontiguousarray(mask).astype(np.uint8)
    out = np.zeros(q.shape, np.float32)
    qs = np.empty(B * H, np.float32)
    ks = np.empty(B * Hkv, np.float32)
    vs = np.empty(B * Hkv, np.float32)
    ci = np.empty(B * H, np.int64)
    mode = {"head": 0, "tensor": 1}[scale_granularity]
    if scales is not None:  # given global scales (sharded launcher)
        mode = 2
        qs[0], ks[0], vs[0] = (np.float32(s) for s in scales)
    st = lib().ia_or_attention_batched(
        _p(q), _p(k), _p(v), B, H, Hkv, L, d, _p(sl), int(bool(causal)), _p(m8),
        mode, float(c), _p(lut), lut.size, int(p_scale), int(row_stride),
        int(threads), _p(out), _p(qs), _p(ks), _p(vs), _p(ci))
    if st == 1:
        raise ValueError("input contains non-finite elements")
    if st != 0:
        raise ValueError(f"oracle rejected arguments (status {st})")
    return out, {"q_scales": qs, "k_scales": ks, "v_scales": vs, "c_int": ci}


def index_softmax_grouped(logits: np.ndarray, groups: np.ndarray, c_ints, lut: np.ndarray,
                          mask=None, p_scale=P_UINT8X255) -> np.ndarray:
    """Grouped-key IndexSoftmax, default per-group-max mode (softmax.py:309-399):
    per group g a row max over the row's unmasked columns of g and the clip
    threshold c_ints[g]; e = lut[(2k min(m_g - a, c_g) + c_g) // (2c_g)], masked
    e = 0; shared row normalisation (2 scale e + s) // max(2s, 1)
    (softmax.py:300-306).  Plain int64 numpy; returns u8 (i8 bytes for 127)."""
    v = np.asarray(logits).astype(np.int64)
    groups = np.asarray(groups).astype(np.int64)
    lut = np.asarray(lut).astype(np.int64)
    k = len(lut) - 1
    m8 = None if mask is None else np.asarray(mask, bool)
    e = np.zeros(v.shape, np.int64)
    for g, ci in enumerate(c_ints):
        cols = np.flatnonzero(groups == g)
        if cols.size == 0:
            continue
        sub = v[:, cols]
        work = np.where(m8[:, cols], -(1 << 62), sub) if m8 is not None else sub
        m = work.max(axis=1)
        dl = np.minimum(np.maximum(m[:, None] - sub, 0), ci)
        e[:, cols] = lut[(2 * dl * k + ci) // (2 * ci)]
    if m8 is not None:
        e[m8] = 0
    s = e.sum(axis=1)
    out = (e * (2 * p_scale) + s[:, None]) // np.maximum(2 * s, 1)[:, None]
    return out.astype(np.uint8)


def c_int_from_alpha(c: float, alpha: float) -> int:
    """max(1, min(round_half_away(c / alpha), 2^52)) in f64 (softmax.py:105-108)."""
    r = float(c) / float(alpha)
    ci = int(np.copysign(np.floor(abs(r) + 0.5), r))
    return max(1, min(ci, 1 << 52))


def quant_only_attention(q, k, v, mask=None, p_scale=P_UINT8X255):
    """The reference's quant-only comparator (pipeline.py:259-296, f32 numpy as the
    reference computes it): int8 QK^T, real = f32(logits) * f32(alpha), stable f32
    softmax (masked -> -inf, fully masked row -> 0; pipeline.py:119-127), requantise
    floor(p * scale + 0.5) (pipeline.py:130-140), int8 P.V, out = f32(acc) * f32(s_v /
    scale).  Returns (out, phat)."""
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    d = q.shape[1]
    qq, sq = quantize_tensor(q)
    kq, sk = quantize_tensor(k)
    vq, sv = quantize_tensor(v)
    logits = qq.astype(np.int64) @ kq.astype(np.int64).T
    alpha = np.float32(float(sq) * float(sk) / np.sqrt(d))
    real = logits.astype(np.int32).astype(np.float32) * alpha
    if mask is not None:
        real = np.where(np.asarray(mask, bool), np.float32(-np.inf), real)
    m = real.max(axis=1, keepdims=True)
    m = np.where(np.isfinite(m), m, np.float32(0))
    e = np.exp(real - m)
    s = e.sum(axis=1, keepdims=True)
    p = e / np.where(s == 0, np.float32(1), s)
    phat = (p * np.float32(p_scale) + np.float32(0.5)).astype(np.uint8)
    acc = phat.astype(np.int64) @ vq.astype(np.int64)
    out = acc.astype(np.float32) * np.float32(float(sv) / p_scale)
    return out, phat


def attention_grouped_batched(q, k, v, k_group_size, *, causal=False, mask=None, b=5, c=6.6,
                              p_scale=P_UINT8X255):
    """Grouped-K pipeline (pipeline.py:229-246) per (b, head) unit, batched: Q and V
    quantised per (b, head), K per (b, KV head, group of k_group_size keys)
    (quantize.py:104-123 with per_row_group), int32 logits, the grouped IndexSoftmax
    (softmax.py:309-399, default per-group max) and the exact P.V + rescale
    (pipeline.py:248-252).  Plain composition of the oracle's stage functions."""
    q = np.ascontiguousarray(q, np.float32)
    B, H, L, d = q.shape
    Hkv = k.shape[1]
    g = H // Hkv
    G = L // k_group_size
    lut = build_lut(b, c)
    m = None
    if causal:
        m = np.triu(np.ones((L, L), bool), 1)
    if mask is not None:
        m = np.asarray(mask, bool) if m is None else (m | np.asarray(mask, bool))
    groups = (np.arange(L) // k_group_size).astype(np.int64)
    out = np.zeros(q.shape, np.float32)
    for bb in range(B):
        for h in range(H):
            qh, sq = quantize_tensor(q[bb, h])
            kh, sk = quantize_groups(k[bb, h // g], G)
            vh, sv = quantize_tensor(v[bb, h // g])
            logits = matmul_s8(qh, kh)
            cis = [c_int_from_alpha(c, float(sq) * float(s) / math.sqrt(d)) for s in sk]
            prob = index_softmax_grouped(logits, groups, cis, lut, m, p_scale)
            acc = gemm_pv(prob, vh)
            out[bb, h] = acc.astype(np.float32) * np.float32(float(sv) / p_scale)
    return out
