"""Attention pipelines on the B200 (reference pipeline.py).

``int_attention`` is the drop-in for the reference's hot entry point
(pipeline.py:202-256): same signature, same validation and exceptions, same
f32 output bits.  Internally it runs the quantiser kernels and ONE fused
kernel per (b, h, 128-row query tile) (csrc/attention.cu); the int32 logits
and uint8 probabilities never touch HBM.

Stage timings come from CUDA events.  Because QK^T, IndexSoftmax, P.V and the
rescale are one kernel, ``StageTimings`` reports the quantiser in
``quantize_ns`` and the fused kernel in ``softmax_path_ns``; ``qk_gemm_ns``,
``pv_gemm_ns`` and ``dequantize_ns`` are 0 (fused away).  ``int_attention_staged``
runs the same computation as the reference's five separate stages (bit-identical
output) and reports every stage's time.
"""
from __future__ import annotations

import math
import statistics
from dataclasses import dataclass, field

import numpy as np
import torch

from . import engine as E
from . import softmax as _sm
from ._tensors import is_torch, to_device, to_host
from .gemm import MAX_SEQ_LEN, gemm_real  # noqa: F401  (re-export parity)
from .quantize import PER_COL_GROUP, PER_ROW_GROUP, PER_TENSOR, QuantGranularity
from .softmax import PFormat


@dataclass(frozen=True)
class AttentionConfig:
    """Pipeline knobs; (b, c) default to the recommended (5, 6.6) (pipeline.py:49-58).
    ``threads`` is accepted for compatibility and ignored by the GPU path."""

    b: int = 5
    c: float = 6.6
    p_format: PFormat = PFormat.UINT8X255
    granularity: QuantGranularity = field(default_factory=QuantGranularity.per_tensor)
    threads: int = 1
    mask: object = None


@dataclass(frozen=True)
class StageTimings:
    """Nanoseconds per stage (median over iters); 0 for fused-away stages."""

    quantize_ns: int
    qk_gemm_ns: int
    softmax_path_ns: int
    pv_gemm_ns: int
    dequantize_ns: int
    total_ns: int

    STAGES = ("quantize", "qk_gemm", "softmax_path", "pv_gemm", "dequantize")

    def stage_ns(self):
        return {"quantize": self.quantize_ns, "qk_gemm": self.qk_gemm_ns,
                "softmax_path": self.softmax_path_ns, "pv_gemm": self.pv_gemm_ns,
                "dequantize": self.dequantize_ns}


def _check_inputs(q, k, v):
    shapes = [tuple(x.shape) if is_torch(x) else np.shape(x) for x in (q, k, v)]
    if len(shapes[0]) != 2 or shapes[0] != shapes[1] or shapes[0] != shapes[2]:
        raise ValueError(
            f"q, k, v must share one L x d shape, got {shapes[0]}, {shapes[1]}, {shapes[2]}")
    if shapes[0][0] > MAX_SEQ_LEN:
        raise ValueError(f"sequence length exceeds {MAX_SEQ_LEN}")
    if shapes[0][0] < 1 or shapes[0][1] < 1:
        raise ValueError("q, k, v must have at least one row and column")
    return shapes[0]


def _check_mask(mask, n):
    if mask is None:
        return None
    shape = tuple(mask.shape) if is_torch(mask) else np.shape(mask)
    if shape != (n, n):
        raise ValueError(f"mask must be {n}x{n}, got {shape}")
    return mask


def _k_granularity(cfg):
    g = cfg.granularity
    if g.kind in (PER_TENSOR, PER_ROW_GROUP):
        return g
    raise ValueError(
        "pipelines support per-tensor or per-row-group key quantization; per-column groups "
        f"mix feature dimensions inside one dot product and have no single logit scale (got {g.kind})")


class _EventClock:
    """CUDA-event stage clock on the current stream."""

    def __init__(self):
        self.ev = {}

    def mark(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev[name] = e

    def ns(self, a, b):
        return int(self.ev[a].elapsed_time(self.ev[b]) * 1e6)


def _run_measured(once, warmup, iters, stage_pairs):
    if iters < 1:
        raise ValueError("iters must be >= 1")
    for _ in range(warmup):
        once(None)
    out, samples = None, []
    for _ in range(iters):
        clk = _EventClock()
        out = once(clk)
        torch.cuda.synchronize()
        samples.append({name: clk.ns(a, b) for name, (a, b) in stage_pairs.items()})
    med = {k: int(statistics.median(s[k] for s in samples)) for k in samples[0]}
    return out, StageTimings(
        quantize_ns=med.get("quantize", 0), qk_gemm_ns=med.get("qk_gemm", 0),
        softmax_path_ns=med.get("softmax_path", 0), pv_gemm_ns=med.get("pv_gemm", 0),
        dequantize_ns=med.get("dequantize", 0), total_ns=med["total"])


def int_attention(q, k, v, cfg=None, warmup=0, iters=1):
    """Fully integer attention on the GPU; returns (output, StageTimings).

    Output = (s_v / denom) * (P^ V^) in f32 with denom 255 (UINT8X255) or 127
    (INT8X127), bit-identical to the reference's CPU result.
    """
    cfg = cfg or AttentionConfig()
    n, d = _check_inputs(q, k, v)
    mask = _check_mask(cfg.mask, n)
    k_gran = _k_granularity(cfg)
    numpy_in = not is_torch(q)
    qt = to_device(q, np.float32)
    kt = to_device(k, np.float32)
    vt = to_device(v, np.float32)
    mt = to_device(mask).to(torch.bool) if mask is not None else None
    p_scale = cfg.p_format.value
    lut = _sm.build_lut(cfg.b, cfg.c)

    if k_gran.kind == PER_ROW_GROUP:
        k_gran.num_groups((n, d))  # group_size must divide L (quantize.py:46-56)
        if E.pad_head_dim(d) is not None and E.grouped_fusable(n, d, k_gran.group_size,
                                                               len(lut.entries)):
            return _int_attention_grouped_fused(qt, kt, vt, mt, cfg, k_gran, lut, numpy_in,
                                                warmup, iters)
        return _int_attention_grouped(qt, kt, vt, mt, cfg, k_gran, lut, numpy_in, warmup, iters)

    p_dt = np.int8 if cfg.p_format is PFormat.INT8X127 else np.uint8

    def once(clk):
        # the reference's per-call audit stream (softmax.py:279-298, pipeline.py:248):
        # int32 logits (the s32 TMEM accumulator of the QK^T MMA), u8 index map, u8 LUT,
        # u8 mask, u8 / s8 P^ (the P.V MMA's A operand, in shared memory)
        _sm._note("logits", np.int32)
        _sm._note("index_table", np.uint8)
        _sm._note("lut", lut.entries)
        if mt is not None:
            _sm._note("mask", np.uint8)
        _sm._note("prob", p_dt)
        _sm._note("pv_in", p_dt)
        return E.attention(qt[None, None], kt[None, None], vt[None, None], mask=mt,
                           b=cfg.b, c=cfg.c, p_scale=p_scale, lut=lut.entries, timer=clk)

    out, timings = _run_measured(
        once, warmup, iters,
        {"quantize": ("start", "quantized"), "softmax_path": ("quantized", "attention"),
         "total": ("start", "attention")})
    return to_host(out[0, 0], numpy_in), timings


def int_attention_staged(q, k, v, cfg=None, warmup=0, iters=1):
    """``int_attention`` run as the reference's five stages, each its own launch
    sequence, so ``StageTimings`` carries the full split the reference reports
    (pipeline.py:61-81, 143-191, 215-253): quantize (3x quantize_symmetric), qk_gemm
    (tcgen05 INT8 GEMM -> int32 logits in HBM), softmax_path (LUT, c_int and the
    IndexSoftmax row kernel -> u8 P^ in HBM), pv_gemm (tcgen05 GEMM -> int32) and
    dequantize (f32 rescale).  A debug / analysis mode: the logits and P^ round-trip
    through HBM here, which the fused ``int_attention`` never does.  The output is
    bit-identical to ``int_attention``; the per-stage times explain the fused one."""
    from .gemm import gemm_pv, gemm_qk, matmul_int8
    from .quantize import quantize_symmetric

    cfg = cfg or AttentionConfig()
    n, d = _check_inputs(q, k, v)
    mask = _check_mask(cfg.mask, n)
    k_gran = _k_granularity(cfg)
    numpy_in = not is_torch(q)
    qt, kt, vt = (to_device(x, np.float32) for x in (q, k, v))
    mt = to_device(mask).to(torch.bool) if mask is not None else None

    def once(clk):
        if clk:
            clk.mark("start")
        qh = quantize_symmetric(qt)
        kh = quantize_symmetric(kt, k_gran)
        vh = quantize_symmetric(vt)
        if clk:
            clk.mark("quantized")
        if k_gran.kind == PER_TENSOR:
            lm = gemm_qk(qh, kh)
            logits = lm.values
        else:
            logits = matmul_int8(qh.values, kh.values)
        if clk:
            clk.mark("qk")
        lut = _sm.build_lut(cfg.b, cfg.c)
        if k_gran.kind == PER_TENSOR:
            ci = _sm.compute_c_int(cfg.c, d, float(qh.scales[0]), float(kh.scales[0]))
            prob = _sm.index_softmax(logits, ci, lut, mask=mt, p_format=cfg.p_format)
        else:
            s_q = float(qh.scales[0])
            alphas = [s_q * float(sk) / math.sqrt(d) for sk in kh.scales.tolist()]
            groups = np.repeat(np.arange(len(alphas)), k_gran.group_size)
            prob = _sm.index_softmax_grouped(logits, groups, alphas, cfg.c, lut, mask=mt,
                                             p_format=cfg.p_format)
        if clk:
            clk.mark("softmax")
        _sm._note("pv_in", prob.values)
        acc = gemm_pv(prob.values, vh)
        if clk:
            clk.mark("pv")
        out = acc.to(torch.float32) * torch.tensor(
            np.float32(float(vh.scales[0]) / prob.denom_scale), device=qt.device)
        if clk:
            clk.mark("end")
        return out

    out, timings = _run_measured(
        once, warmup, iters,
        {"quantize": ("start", "quantized"), "qk_gemm": ("quantized", "qk"),
         "softmax_path": ("qk", "softmax"), "pv_gemm": ("softmax", "pv"),
         "dequantize": ("pv", "end"), "total": ("start", "end")})
    return to_host(out, numpy_in), timings


def _int_attention_grouped_fused(qt, kt, vt, mt, cfg, k_gran, lut, numpy_in, warmup, iters):
    """Per-row-group K scales (pipeline.py:229-246) in ONE fused launch: the grouped
    IndexSoftmax (softmax.py:309-399) runs between the two INT8 MMAs with a per-group
    row max and clip threshold; logits never reach HBM (csrc/attention.cu, gk_passes)."""
    p_dt = np.int8 if cfg.p_format is PFormat.INT8X127 else np.uint8

    def once(clk):
        # audit stream of the grouped path (softmax.py:394, :398, pipeline.py:248): the
        # u8 surrogates and P^ the grouped kernel builds on chip
        _sm._note("surrogates", np.uint8)
        _sm._note("prob", p_dt)
        _sm._note("pv_in", p_dt)
        return E.attention(qt[None, None], kt[None, None], vt[None, None], mask=mt, b=cfg.b,
                           c=cfg.c, p_scale=cfg.p_format.value, lut=lut.entries, timer=clk,
                           k_group_size=k_gran.group_size)

    out, timings = _run_measured(
        once, warmup, iters,
        {"quantize": ("start", "quantized"), "softmax_path": ("quantized", "attention"),
         "total": ("start", "attention")})
    return to_host(out[0, 0], numpy_in), timings


def _int_attention_grouped(qt, kt, vt, mt, cfg, k_gran, lut, numpy_in, warmup, iters):
    """Per-row-group K scales (pipeline.py:229-246) outside the fused kernel's domain
    (group sizes that are not a power of two in [8, 128], d > 128): stage kernels + the
    grouped IndexSoftmax row kernel."""
    from .gemm import gemm_pv, matmul_int8
    from .quantize import quantize_symmetric

    n, d = qt.shape

    def once(clk):
        if clk:
            clk.mark("start")
        qh = quantize_symmetric(qt)
        kh = quantize_symmetric(kt, k_gran)
        vh = quantize_symmetric(vt)
        if clk:
            clk.mark("quantized")
        logits = matmul_int8(qh.values, kh.values)
        if clk:
            clk.mark("qk")
        s_q = float(qh.scales[0])
        alphas = [s_q * float(sk) / math.sqrt(d) for sk in kh.scales.tolist()]
        groups = np.repeat(np.arange(len(alphas)), k_gran.group_size)
        prob = _sm.index_softmax_grouped(logits, groups, alphas, cfg.c, lut, mask=mt,
                                         p_format=cfg.p_format)
        if clk:
            clk.mark("softmax")
        _sm._note("pv_in", prob.values)
        acc = gemm_pv(prob.values, vh)
        if clk:
            clk.mark("pv")
        out_scale = torch.tensor(np.float32(float(vh.scales[0]) / prob.denom_scale),
                                 device=qt.device)
        out = acc.to(torch.float32) * out_scale
        if clk:
            clk.mark("end")
        return out

    out, timings = _run_measured(
        once, warmup, iters,
        {"quantize": ("start", "quantized"), "qk_gemm": ("quantized", "qk"),
         "softmax_path": ("qk", "softmax"), "pv_gemm": ("softmax", "pv"),
         "dequantize": ("pv", "end"), "total": ("start", "end")})
    return to_host(out, numpy_in), timings


def _stable_softmax(a, mask=None):
    """Row softmax with max subtraction; fully masked rows -> 0 (pipeline.py:119-127)."""
    if mask is not None:
        a = a.masked_fill(mask, float("-inf"))
    m = a.max(dim=1, keepdim=True).values
    m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    e = torch.exp(a - m)
    s = e.sum(dim=1, keepdim=True)
    return e / torch.where(s == 0, torch.ones_like(s), s)


def _quantize_probs(p, p_format):
    """floor(p * scale + 0.5) onto the 8-bit grid (pipeline.py:130-140)."""
    q = (p * p_format.value + 0.5).to(torch.uint8)
    return q.view(torch.int8) if p_format is PFormat.INT8X127 else q


def quant_only_attention(q, k, v, cfg=None, warmup=0, iters=1):
    """The paper's comparator: INT8 GEMMs with a dequantise -> f32 softmax ->
    requantise detour (pipeline.py:259-296).  Per-tensor K with d <= 256 runs the
    fused kernel's quant-only mode (MUFU exp2 between the same tcgen05 INT8
    MMAs); per-row-group K composes the library's tcgen05 GEMMs with a torch f32
    softmax.  Either way results match the reference to float tolerance, not bit
    for bit."""
    from .gemm import gemm_pv, matmul_int8
    from .quantize import quantize_symmetric

    cfg = cfg or AttentionConfig()
    n, d = _check_inputs(q, k, v)
    mask = _check_mask(cfg.mask, n)
    k_gran = _k_granularity(cfg)
    numpy_in = not is_torch(q)
    qt, kt, vt = (to_device(x, np.float32) for x in (q, k, v))
    mt = to_device(mask).to(torch.bool) if mask is not None else None

    if k_gran.kind == PER_TENSOR and E.pad_head_dim(d) is not None:
        # fused kernel, quant-only mode (IA_SOFTMAX_FLOAT): same quantiser and MMAs
        def fused(clk):
            return E.attention(qt[None, None], kt[None, None], vt[None, None], mask=mt,
                               p_scale=cfg.p_format.value, timer=clk, softmax="float")

        out, timings = _run_measured(
            fused, warmup, iters,
            {"quantize": ("start", "quantized"), "softmax_path": ("quantized", "attention"),
             "total": ("start", "attention")})
        return to_host(out[0, 0], numpy_in), timings

    def once(clk):
        if clk:
            clk.mark("start")
        qh = quantize_symmetric(qt)
        kh = quantize_symmetric(kt, k_gran)
        vh = quantize_symmetric(vt)
        if clk:
            clk.mark("quantized")
        logits = matmul_int8(qh.values, kh.values)
        if clk:
            clk.mark("qk")
        s_q = float(qh.scales[0])
        if k_gran.kind == PER_TENSOR:
            alpha = torch.tensor(np.float32(s_q * float(kh.scales[0]) / math.sqrt(d)),
                                 device=qt.device)
            real = logits.to(torch.float32) * alpha
        else:
            col = np.repeat(kh.scales.cpu().numpy().astype(np.float64) * (s_q / math.sqrt(d)),
                            k_gran.group_size).astype(np.float32)
            real = logits.to(torch.float32) * torch.as_tensor(col, device=qt.device)[None, :]
        phat = _quantize_probs(_stable_softmax(real, mt), cfg.p_format)
        if clk:
            clk.mark("softmax")
        acc = gemm_pv(phat, vh)
        if clk:
            clk.mark("pv")
        out = acc.to(torch.float32) * torch.tensor(
            np.float32(float(vh.scales[0]) / cfg.p_format.value), device=qt.device)
        if clk:
            clk.mark("end")
        return out

    out, timings = _run_measured(
        once, warmup, iters,
        {"quantize": ("start", "quantized"), "qk_gemm": ("quantized", "qk"),
         "softmax_path": ("qk", "softmax"), "pv_gemm": ("softmax", "pv"),
         "dequantize": ("pv", "end"), "total": ("start", "end")})
    return to_host(out, numpy_in), timings


def reference_attention(q, k, v, mask=None):
    """Exact scaled-dot-product attention, f64 inside, f32 out (pipeline.py:299-302)."""
    o, _ = reference_attention_timed(q, k, v, mask=mask)
    return o


def reference_attention_timed(q, k, v, mask=None, threads=1, warmup=0, iters=1):
    """reference_attention plus stage timings (f64 on the device; fidelity oracle)."""
    n, d = _check_inputs(q, k, v)
    mask = _check_mask(mask, n)
    numpy_in = not is_torch(q)
    qt, kt, vt = (to_device(x, np.float32) for x in (q, k, v))
    mt = to_device(mask).to(torch.bool) if mask is not None else None
    inv = 1.0 / math.sqrt(d)

    def once(clk):
        if clk:
            clk.mark("start")
        q64, k64, v64 = qt.double(), kt.double(), vt.double()
        if clk:
            clk.mark("quantized")
        a = (q64 @ k64.T) * inv
        if clk:
            clk.mark("qk")
        p = _stable_softmax(a, mt)
        if clk:
            clk.mark("softmax")
        o = p @ v64
        if clk:
            clk.mark("pv")
        out = o.to(torch.float32)
        if clk:
            clk.mark("end")
        return out

    out, timings = _run_measured(
        once, warmup, iters,
        {"quantize": ("start", "quantized"), "qk_gemm": ("quantized", "qk"),
         "softmax_path": ("qk", "softmax"), "pv_gemm": ("softmax", "pv"),
         "dequantize": ("pv", "end"), "total": ("start", "end")})
    return to_host(out, numpy_in), timings
