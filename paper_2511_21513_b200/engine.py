"""Device-side driver of the B200 IntAttention path.

Owns the stream-ordered launch sequence over the C ABI (include/intattn_b200.h):

    amax(Q), amax(K), amax(V) -> scales -> quantise Q, K (row layout, zero-padded
    head dim) and V (transposed V^T layout) -> per-(b, h) parameters (c_int,
    exact index magic numbers, output scale) -> fused attention kernel.

PyTorch supplies device memory, the current stream and host<->device copies;
every byte of arithmetic runs in the library's sm_100a kernels.  There is no
CPU fallback: without the library or an sm_100 device every entry raises.

Shapes follow the batched contract of SURVEY.md §8b: q [B, H, L, d],
k/v [B, Hkv, L, d] f32; query head h attends with KV head h // (H // Hkv).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

MAX_SEQ_LEN = 65536
FUSED_MAX_HEAD_DIM = 256


_checked_devices = set()


def require_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_21513_b200 requires an sm_100 CUDA device; "
                           "there is no CPU fallback")
    dev = torch.cuda.current_device()
    if dev not in _checked_devices:  # cudaGetDeviceProperties is slow: check once per device
        _lib.check(_lib.load().ia_device_check(dev), "device check")
        _checked_devices.add(dev)
    return torch.device("cuda", dev)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def pad_head_dim(d: int) -> int | None:
    for p in (32, 64, 128, 256):
        if d <= p:
            return p
    return None


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


@dataclass
class QuantOut:
    values: torch.Tensor   # int8, layout depends on caller
    scales: torch.Tensor   # f32 [n_slots]


class Workspace:
    """Per-call scratch: amax bit slots and team arrival counters (both zeroed)
    + the non-finite flag."""

    def __init__(self, n_slots: int, device):
        # zeroed by a memset node of the library (no framework fill kernel per call)
        self.buf = torch.empty(2 * n_slots + 1, dtype=torch.int32, device=device)
        _lib.check(_lib.load().ia_zero_async(_p(self.buf), self.buf.numel() * 4, _stream()),
                   "workspace zero")
        self.amax = self.buf[:n_slots]
        self.count = self.buf[n_slots:2 * n_slots]
        self.err = self.buf[2 * n_slots:]
        self.scales = torch.empty(n_slots, dtype=torch.float32, device=device)
        self._off = 0

    def take(self, n: int):
        a = self.amax[self._off:self._off + n]
        s = self.scales[self._off:self._off + n]
        self._off += n
        return a, s


def amax_rows(x, n_groups, rows_per_group, cols, amax, err, *, seq_lens=None, valid_div=1,
              slot_div=1):
    L = _lib.load()
    _lib.check(L.ia_quant_amax_rows(_p(x), n_groups, rows_per_group, cols, _p(seq_lens),
                                    valid_div, slot_div, _p(amax), _p(err), _stream()), "amax")


def scales_from_amax(amax, scales):
    _lib.check(_lib.load().ia_quant_scales(_p(amax), amax.numel(), _p(scales), _stream()),
               "scales")


def quantize_rows(x, n_groups, rows_per_group, cols, scales, out, out_pitch, *, seq_lens=None,
                  valid_div=1, slot_div=1, mode=_lib.IA_QMODE_ROWS, col_group=1):
    _lib.check(_lib.load().ia_quantize(_p(x), n_groups, rows_per_group, cols, _p(seq_lens),
                                       valid_div, mode, slot_div, col_group, _p(scales), _p(out),
                                       out_pitch, 0, 0, _stream()), "quantize")


def quantize_vt(x, n_groups, rows, cols, scales, out, out_pitch, group_stride, *, seq_lens=None,
                valid_div=1, slot_div=1):
    _lib.check(_lib.load().ia_quantize(_p(x), n_groups, rows, cols, _p(seq_lens), valid_div,
                                       _lib.IA_QMODE_ROWS, slot_div, 1, _p(scales), _p(out),
                                       out_pitch, 1, group_stride, _stream()), "quantize V^T")


def pack_mask(mask: torch.Tensor) -> torch.Tensor:
    """bool/u8 [L, L] (True = excluded) -> u32 bits [L, ceil(L/32)] on device."""
    L = mask.shape[0]
    m8 = mask.to(torch.uint8).contiguous()
    bits = torch.empty((L, (L + 31) // 32), dtype=torch.int32, device=mask.device)
    _lib.check(_lib.load().ia_mask_pack(_p(m8), L, _p(bits), _stream()), "mask pack")
    return bits


def raise_if_nonfinite(err: torch.Tensor):
    e = int(err.item())
    if e & 2:  # quant_heads_kernel: a team barrier timed out (never expected)
        raise RuntimeError("quantiser team barrier timed out; results discarded")
    if e != 0:
        raise ValueError("input contains non-finite elements")


def check_out(out, q, shape):
    """A caller-supplied ``out`` is written by the kernel through a raw pointer: it
    must be a contiguous f32 CUDA tensor of the result's shape on q's device."""
    if not isinstance(out, torch.Tensor):
        raise TypeError("out must be a torch.Tensor")
    if out.device != q.device:
        raise ValueError(f"out is on {out.device}, the inputs on {q.device}")
    if out.dtype != torch.float32:
        raise ValueError(f"out must be float32, got {out.dtype}")
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"out must have shape {tuple(shape)}, got {tuple(out.shape)}")
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")
    return out


@dataclass
class Prepared:
    """Quantised operands + per-head parameters, ready for the fused kernel."""
    qhat: torch.Tensor    # [B*H, L, d_pad] int8
    khat: torch.Tensor    # [B*Hkv, L, d_pad] int8
    vt: torch.Tensor      # [B*Hkv, d_pad, l_pad] int8
    q_scales: torch.Tensor
    k_scales: torch.Tensor
    v_scales: torch.Tensor
    params: torch.Tensor  # [B*H] ia_head_params (raw bytes)
    err: torch.Tensor
    d_pad: int
    l_pad: int


HEAD_PARAMS_BYTES = ctypes.sizeof(_lib.HeadParams)


def prepare(q, k, v, *, seq_lens=None, scale_granularity="head", b=5, c=6.6, p_scale=255,
            d_pad=None, scales=None, quant="fused") -> Prepared:
    """Quantise Q/K/V on device and compute per-(b, h) parameters.

    ``scales`` (optional): precomputed global (q, k, v) f32 scales as 1-element
    device tensors -- the sharded launcher's all-reduced amax; implies
    ``scale_granularity="tensor"`` and skips the amax kernels.
    ``quant``: "fused" (default) quantises per-head Q/K/V in one launch
    (ia_quant_heads) when the layout allows; "split" forces the amax +
    quantise kernels (bit-identical; kept for A/B checks).
    """
    B, H, Lq, d = q.shape
    Hkv = k.shape[1]
    dev = q.device
    if d_pad is None:
        d_pad = pad_head_dim(d)
    l_pad = _round_up(Lq, 16)
    per_head = scale_granularity == "head" and scales is None
    nq = B * H if per_head else 1
    nkv = B * Hkv if per_head else 1
    ws = Workspace(nq + 2 * nkv, dev)
    aq, sq = ws.take(nq)
    ak, sk = ws.take(nkv)
    av, sv = ws.take(nkv)
    sl = seq_lens
    qhat = torch.empty((B * H, Lq, d_pad), dtype=torch.int8, device=dev)
    khat = torch.empty((B * Hkv, Lq, d_pad), dtype=torch.int8, device=dev)
    vt = torch.empty((B * Hkv, d_pad, l_pad), dtype=torch.int8, device=dev)
    if quant == "fused" and per_head and d % 4 == 0 and d_pad <= 256 and d_pad % 16 == 0 and all(
            t.is_contiguous() and t.data_ptr() % 16 == 0 for t in (q, k, v)):
        # one launch: per-head amax + quantise of Q, K, V (f32 read from HBM once)
        _lib.check(_lib.load().ia_quant_heads(
            _p(q), _p(k), _p(v), B, H, Hkv, Lq, d, _p(sl), _p(qhat), _p(khat), _p(vt), d_pad,
            l_pad, _p(ws.amax), _p(ws.count), _p(ws.scales), _p(ws.err), _stream()),
            "quantize heads")
        return _finish_prepare(qhat, khat, vt, sq, sk, sv, ws, per_head, B, H, Hkv, d, b, c,
                               p_scale, d_pad, l_pad)
    if quant == "fused" and scales is None and not per_head and d % 4 == 0 and d_pad <= 256 \
            and d_pad % 16 == 0 and all(t.is_contiguous() and t.data_ptr() % 16 == 0
                                        for t in (q, k, v)):
        # per-tensor scales: one amax launch over Q, K, V + one quantise launch
        _lib.check(_lib.load().ia_quant_tensors(
            _p(q), _p(k), _p(v), B, H, Hkv, Lq, d, _p(sl), _p(qhat), _p(khat), _p(vt), d_pad,
            l_pad, _p(ws.amax), _p(ws.scales), _p(ws.err), _stream()), "quantize tensors")
        return _finish_prepare(qhat, khat, vt, sq, sk, sv, ws, per_head, B, H, Hkv, d, b, c,
                               p_scale, d_pad, l_pad)
    if scales is None:
        amax_rows(q, B * H, Lq, d, aq, ws.err, seq_lens=sl, valid_div=H,
                  slot_div=1 if per_head else B * H)
        amax_rows(k, B * Hkv, Lq, d, ak, ws.err, seq_lens=sl, valid_div=Hkv,
                  slot_div=1 if per_head else B * Hkv)
        amax_rows(v, B * Hkv, Lq, d, av, ws.err, seq_lens=sl, valid_div=Hkv,
                  slot_div=1 if per_head else B * Hkv)
        scales_from_amax(ws.amax, ws.scales)
    else:
        for dst, src in zip((sq, sk, sv), scales):
            dst.copy_(src.reshape(1))
    quantize_rows(q, B * H, Lq, d, sq, qhat, d_pad, seq_lens=sl, valid_div=H,
                  slot_div=1 if per_head else B * H)
    quantize_rows(k, B * Hkv, Lq, d, sk, khat, d_pad, seq_lens=sl, valid_div=Hkv,
                  slot_div=1 if per_head else B * Hkv)
    quantize_vt(v, B * Hkv, Lq, d, sv, vt, l_pad, d_pad * l_pad, seq_lens=sl, valid_div=Hkv,
                slot_div=1 if per_head else B * Hkv)
    return _finish_prepare(qhat, khat, vt, sq, sk, sv, ws, per_head, B, H, Hkv, d, b, c, p_scale,
                           d_pad, l_pad)


def prepare_grouped(q, k, v, k_group_size, *, b=5, c=6.6, p_scale=255, d_pad=None):
    """Grouped-K quantisation (pipeline.py:217-219 with a per_row_group K granularity,
    quantize.py:92-123): Q and V one scale per (b, head), K one scale per (b, KV head,
    group of ``k_group_size`` keys); plus the per-(query head, key group) index maps
    (ia_group_params_dev) the grouped fused kernel reads.  Returns (Prepared, gparams)."""
    B, H, Lq, d = q.shape
    Hkv = k.shape[1]
    dev = q.device
    gs = int(k_group_size)
    G = Lq // gs
    if d_pad is None:
        d_pad = pad_head_dim(d)
    l_pad = _round_up(Lq, 16)
    ws = Workspace(B * H + B * Hkv * G + B * Hkv, dev)
    aq, sq = ws.take(B * H)
    ak, sk = ws.take(B * Hkv * G)
    av, sv = ws.take(B * Hkv)
    amax_rows(q, B * H, Lq, d, aq, ws.err)
    amax_rows(k, B * Hkv * G, gs, d, ak, ws.err)
    amax_rows(v, B * Hkv, Lq, d, av, ws.err)
    scales_from_amax(ws.amax, ws.scales)
    qhat = torch.empty((B * H, Lq, d_pad), dtype=torch.int8, device=dev)
    khat = torch.empty((B * Hkv, Lq, d_pad), dtype=torch.int8, device=dev)
    vt = torch.empty((B * Hkv, d_pad, l_pad), dtype=torch.int8, device=dev)
    quantize_rows(q, B * H, Lq, d, sq, qhat, d_pad)
    quantize_rows(k, B * Hkv * G, gs, d, sk, khat, d_pad)
    quantize_vt(v, B * Hkv, Lq, d, sv, vt, l_pad, d_pad * l_pad)
    # per-(b, h) parameters: only out_scale = s_v / p_scale is read in grouped mode (the
    # K-side index maps are per group, below); sv stands in for the per-head K scale
    params = torch.empty((B * H, HEAD_PARAMS_BYTES), dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().ia_head_params_dev(_p(sq), _p(sv), _p(sv), 1, 1, B, H, Hkv, d,
                                              float(c), 1 << b, int(p_scale), _p(params),
                                              _stream()), "head params")
    gparams = torch.empty((B * H, G, _lib.GROUP_PARAMS_BYTES), dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().ia_group_params_dev(_p(sq), _p(sk), B, H, Hkv, G, d, float(c),
                                               1 << b, _p(gparams), _stream()), "group params")
    return Prepared(qhat, khat, vt, sq, sk, sv, params, ws.err, d_pad, l_pad), gparams


def grouped_fusable(L, d, k_group_size, nlut, seq_lens=None, scale_granularity="head"):
    """The grouped-K fused kernel's domain: power-of-two groups of 8..128 keys that
    tile L, d <= 128, LUTs of <= 64 entries, per-head Q/V, no per-batch lengths."""
    gs = int(k_group_size)
    return (8 <= gs <= 128 and gs & (gs - 1) == 0 and L % gs == 0 and d <= 128 and nlut <= 64
            and seq_lens is None and scale_granularity == "head")


def _finish_prepare(qhat, khat, vt, sq, sk, sv, ws, per_head, B, H, Hkv, d, b, c, p_scale, d_pad,
                    l_pad) -> Prepared:
    params = torch.empty((B * H, HEAD_PARAMS_BYTES), dtype=torch.uint8, device=qhat.device)
    _lib.check(_lib.load().ia_head_params_dev(_p(sq), _p(sk), _p(sv), int(per_head),
                                              int(per_head), B, H, Hkv, d, float(c), 1 << b,
                                              int(p_scale), _p(params), _stream()), "head params")
    return Prepared(qhat, khat, vt, sq, sk, sv, params, ws.err, d_pad, l_pad)


def attn_fused(prep: Prepared, shape, out, *, causal=False, seq_lens=None, mask_bits=None,
               lut=None, p_scale=255, debug=None, times=None, softmax_mode=_lib.IA_SOFTMAX_INDEX,
               kgroup=None, k_group_size=0):
    B, H, Hkv, Lq, d = shape
    a = _lib.AttnArgs()
    a.q, a.k, a.vt = prep.qhat.data_ptr(), prep.khat.data_ptr(), prep.vt.data_ptr()
    a.out = out.data_ptr()
    a.params = prep.params.data_ptr()
    a.seq_lens = None if seq_lens is None else seq_lens.data_ptr()
    a.mask_bits = None if mask_bits is None else mask_bits.data_ptr()
    a.B, a.H, a.Hkv, a.L, a.d, a.d_pad, a.l_pad = B, H, Hkv, Lq, d, prep.d_pad, prep.l_pad
    a.causal = int(bool(causal))
    a.nlut = len(lut)
    a.p_scale = int(p_scale)
    a.softmax_mode = int(softmax_mode)
    for i, x in enumerate(lut):
        a.lut[i] = int(x)
    if debug is not None:
        a.dbg_logits = debug["logits"].data_ptr()
        a.dbg_prob = debug["prob"].data_ptr()
        a.dbg_acc = debug["acc"].data_ptr()
    if times is not None:
        a.dbg_times = times.data_ptr()
    if kgroup is not None:
        a.kgroup_params = kgroup.data_ptr()
        a.k_group_size = int(k_group_size)
    _lib.check(_lib.load().ia_attn_fwd(ctypes.byref(a), _stream()), "attention")


def lut_bytes(b: int, c: float) -> np.ndarray:
    """ExpLut entries (softmax.py:88-102), computed on the host in f64 as the
    reference does: a per-call host constant, not device work."""
    n = 1 << b
    x = 255.0 * np.exp(-c * np.arange(n, dtype=np.float64) / (n - 1))
    e = np.copysign(np.floor(np.abs(x) + 0.5), x).astype(np.uint8)
    e[n - 1] = 0
    return e


def attention(q, k, v, *, causal=False, seq_lens=None, mask=None, scale_granularity="head",
              b=5, c=6.6, p_scale=255, lut=None, out=None, debug=False, check_finite=True,
              timer=None, scales=None, softmax="index", k_group_size=None):
    """Batched fused IntAttention on the current CUDA device.

    softmax="index" is IndexSoftmax (bit-exact with the reference); "float" runs
    the quant-only comparator (pipeline.py:259-296: dequantise -> f32 softmax ->
    requantise between the same INT8 MMAs) in the same fused kernel.

    q [B, H, L, d], k/v [B, Hkv, L, d]: f32 CUDA tensors (contiguous).
    seq_lens: int32 CUDA [B] or None.  mask: bool CUDA [L, L] (True = excluded)
    shared by every unit, or None.  Returns out [B, H, L, d] f32 (and, with
    debug=True, a dict with the quantised operands, int32 logits, u8 P and int32
    P.V accumulators for parity checks).
    """
    B, H, Lq, d = q.shape
    Hkv = k.shape[1]
    if lut is None:
        lut = lut_bytes(b, c)
    if out is None:
        out = torch.empty((B, H, Lq, d), dtype=torch.float32, device=q.device)
    else:
        check_out(out, q, (B, H, Lq, d))
    if timer is not None:
        timer.mark("start")
    d_pad = pad_head_dim(d)
    if d_pad is not None and _lib.load().ia_attn_supported(d_pad, len(lut)) != _lib.IA_OK:
        d_pad = None  # e.g. d_pad 256 with a 2^6+ entry LUT: shared memory too small
    if softmax not in ("index", "float"):
        raise ValueError("softmax must be 'index' or 'float'")
    if d_pad is None and softmax == "float":
        raise ValueError("the fused quant-only path needs head dim <= 256")
    if k_group_size is not None and (d_pad is None or softmax != "index" or scales is not None
                                     or not grouped_fusable(Lq, d, k_group_size, len(lut),
                                                            seq_lens, scale_granularity)):
        raise ValueError("grouped K in the fused kernel needs a power-of-two group of 8..128 "
                         "keys dividing L, d <= 128, a <= 64-entry LUT, per-head Q/V scales "
                         "and no seq_lens")
    if d_pad is None:
        if scales is not None:
            raise ValueError("precomputed scales need the fused path (head dim <= 256)")
        res = _attention_unfused(q, k, v, causal=causal, seq_lens=seq_lens, mask=mask,
                                 scale_granularity=scale_granularity, b=b, c=c,
                                 p_scale=p_scale, lut=lut, out=out, check_finite=check_finite)
        if timer is not None:
            timer.mark("quantized")
            timer.mark("attention")
        return (res, {}) if debug else res
    gparams = None
    if k_group_size is not None:
        # grouped K (per_row_group K scales; softmax.py:309-399, pipeline.py:229-246)
        prep, gparams = prepare_grouped(q, k, v, k_group_size, b=b, c=c, p_scale=p_scale,
                                        d_pad=d_pad)
    else:
        prep = prepare(q, k, v, seq_lens=seq_lens, scale_granularity=scale_granularity, b=b,
                       c=c, p_scale=p_scale, d_pad=d_pad, scales=scales)
    mbits = pack_mask(mask) if mask is not None else None
    if timer is not None:
        timer.mark("quantized")
    dbg = None
    if debug:
        dbg = {"logits": torch.zeros((B * H, Lq, Lq), dtype=torch.int32, device=q.device),
               "prob": torch.zeros((B * H, Lq, Lq), dtype=torch.uint8, device=q.device),
               "acc": torch.zeros((B * H, Lq, d_pad), dtype=torch.int32, device=q.device)}
    attn_fused(prep, (B, H, Hkv, Lq, d), out, causal=causal, seq_lens=seq_lens,
               mask_bits=mbits, lut=lut, p_scale=p_scale, debug=dbg,
               softmax_mode=_lib.IA_SOFTMAX_FLOAT if softmax == "float" else _lib.IA_SOFTMAX_INDEX,
               kgroup=gparams, k_group_size=k_group_size or 0)
    if timer is not None:
        timer.mark("attention")
    if isinstance(check_finite, list):  # deferred: the caller checks after its pipeline
        check_finite.append(prep.err)
    elif check_finite:
        raise_if_nonfinite(prep.err)
    if debug:
        dbg.update(qhat=prep.qhat, khat=prep.khat, vt=prep.vt, q_scales=prep.q_scales,
                   k_scales=prep.k_scales, v_scales=prep.v_scales, params=prep.params)
        return out, dbg
    return out


class AttentionGraph:
    """One ``attention`` call on fixed device tensors, captured once into a CUDA graph
    and replayed: the workspace fill, the quantiser, the parameter and the fused
    launches go to the GPU as one graph launch with no host work between them (for
    small problems -- C1, C2 -- the host-side launch sequence is a large part of a
    call).  ``replay()`` recomputes ``out`` from the current contents of q, k, v.
    The non-finite check is not part of the graph (``check()`` reads the flag)."""

    def __init__(self, q, k, v, out, **kw):
        kw = dict(kw, out=out, check_finite=[])
        attention(q, k, v, **kw)  # eager warm-up: validation, tensor maps, smem attributes
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        flags = []
        with torch.cuda.stream(side), torch.cuda.graph(self.graph, stream=side):
            attention(q, k, v, **dict(kw, check_finite=flags))
        torch.cuda.current_stream().wait_stream(side)
        self._flags = flags
        self.out = out

    def replay(self):
        self.graph.replay()
        return self.out

    def check(self):
        for f in self._flags:
            raise_if_nonfinite(f)


def gemm_i8(a, b_t, *, a_signed=True):
    """C = a @ b_t^T (int32) on tcgen05.  a [M, K] int8/uint8, b_t [N, K] int8 (CUDA)."""
    M, K = a.shape
    N = b_t.shape[0]
    kp = _round_up(K, 16)
    if kp != K or not a.is_contiguous():
        a = torch.nn.functional.pad(a.contiguous(), (0, kp - K))
    if kp != K or not b_t.is_contiguous():
        b_t = torch.nn.functional.pad(b_t.contiguous(), (0, kp - K))
    out = torch.empty((M, N), dtype=torch.int32, device=a.device)
    _lib.check(_lib.load().ia_gemm_i8(_p(a), kp, int(a_signed), _p(b_t), kp, M, N, K, _p(out),
                                      N, _stream()), "gemm_i8")
    return out


def index_softmax_dev(logits, c_int, lut, mask=None, p_scale=255, delta_bound=(1 << 32) - 1):
    rows, cols = logits.shape
    lut_t = torch.as_tensor(np.ascontiguousarray(lut, np.uint8)).to(logits.device)
    hp = _lib.softmax_params_host(c_int, delta_bound, len(lut))
    m8 = None if mask is None else mask.to(torch.uint8).contiguous()
    out = torch.empty((rows, cols), dtype=torch.uint8, device=logits.device)
    _lib.check(_lib.load().ia_index_softmax(_p(logits), rows, cols, ctypes.byref(hp), _p(lut_t),
                                            len(lut), int(p_scale), _p(m8), _p(out), _stream()),
               "index_softmax")
    return out


def index_softmax_grouped_dev(logits, groups, c_ints, lut, mask=None, p_scale=255,
                              delta_bound=(1 << 32) - 1):
    """Grouped-key IndexSoftmax kernel (ia_index_softmax_grouped); ``groups`` is an
    int array [cols], ``c_ints`` the per-group clip thresholds."""
    rows, cols = logits.shape
    dev = logits.device
    lut_t = torch.as_tensor(np.ascontiguousarray(lut, np.uint8)).to(dev)
    hps = (_lib.HeadParams * len(c_ints))()
    for i, ci in enumerate(c_ints):
        hps[i] = _lib.softmax_params_host(int(ci), delta_bound, len(lut))
    hp_t = torch.frombuffer(bytearray(bytes(hps)), dtype=torch.uint8).to(dev)
    g_t = torch.as_tensor(np.ascontiguousarray(groups, np.int32)).to(dev)
    m8 = None if mask is None else mask.to(torch.uint8).contiguous()
    out = torch.empty((rows, cols), dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().ia_index_softmax_grouped(
        _p(logits), rows, cols, _p(g_t), len(c_ints), _p(hp_t), _p(lut_t), len(lut), int(p_scale),
        _p(m8), _p(out), _stream()), "index_softmax_grouped")
    return out


def _attention_unfused(q, k, v, *, causal, seq_lens, mask, scale_granularity, b, c, p_scale,
                       lut, out, check_finite):
    """d > 256: per-unit stage kernels (tcgen05 GEMM -> row IndexSoftmax -> tcgen05 GEMM)."""
    B, H, Lq, d = q.shape
    Hkv = k.shape[1]
    g = H // Hkv
    per_head = scale_granularity == "head"
    dp = _round_up(d, 16)
    lp = _round_up(Lq, 16)
    nq = B * H if per_head else 1
    nkv = B * Hkv if per_head else 1
    ws = Workspace(nq + 2 * nkv, q.device)
    aq, sq = ws.take(nq)
    ak, sk = ws.take(nkv)
    av, sv = ws.take(nkv)
    amax_rows(q, B * H, Lq, d, aq, ws.err, seq_lens=seq_lens, valid_div=H,
              slot_div=1 if per_head else B * H)
    amax_rows(k, B * Hkv, Lq, d, ak, ws.err, seq_lens=seq_lens, valid_div=Hkv,
              slot_div=1 if per_head else B * Hkv)
    amax_rows(v, B * Hkv, Lq, d, av, ws.err, seq_lens=seq_lens, valid_div=Hkv,
              slot_div=1 if per_head else B * Hkv)
    scales_from_amax(ws.amax, ws.scales)
    qhat = torch.empty((B * H, Lq, dp), dtype=torch.int8, device=q.device)
    khat = torch.empty((B * Hkv, Lq, dp), dtype=torch.int8, device=q.device)
    vt = torch.empty((B * Hkv, dp, lp), dtype=torch.int8, device=q.device)
    quantize_rows(q, B * H, Lq, d, sq, qhat, dp, seq_lens=seq_lens, valid_div=H,
                  slot_div=1 if per_head else B * H)
    quantize_rows(k, B * Hkv, Lq, d, sk, khat, dp, seq_lens=seq_lens, valid_div=Hkv,
                  slot_div=1 if per_head else B * Hkv)
    quantize_vt(v, B * Hkv, Lq, d, sv, vt, lp, dp * lp, seq_lens=seq_lens, valid_div=Hkv,
                slot_div=1 if per_head else B * Hkv)
    if isinstance(check_finite, list):
        check_finite.append(ws.err)
    elif check_finite:
        raise_if_nonfinite(ws.err)
    sq_h, sk_h, sv_h = sq.cpu().numpy(), sk.cpu().numpy(), sv.cpu().numpy()
    lens = None if seq_lens is None else seq_lens.cpu().numpy()
    for bb in range(B):
        n = Lq if lens is None else int(lens[bb])
        for h in range(H):
            u, ku = bb * H + h, bb * Hkv + h // g
            qs = sq_h[u if per_head else 0]
            ks = sk_h[ku if per_head else 0]
            vs = sv_h[ku if per_head else 0]
            hp = _lib.head_params_host(c, d, 1 << b, p_scale, qs, ks, vs)
            o = out[bb, h]
            o.zero_()
            if n == 0:
                continue
            logits = gemm_i8(qhat[u, :n], khat[ku, :n])
            m = None
            if causal:
                m = torch.ones((n, n), dtype=torch.bool, device=q.device).triu_(1)
            if mask is not None:
                mm = mask[:n, :n]
                m = mm if m is None else (m | mm)
            prob = index_softmax_dev(logits, hp.c_int, lut, m, p_scale,
                                     delta_bound=2 * d * 127 * 127)
            acc = gemm_i8(prob, vt[ku, :, :n], a_signed=False)
            o[:n] = acc[:, :d].to(torch.float32) * torch.tensor(hp.out_scale, dtype=torch.float32,
                                                                  device=q.device)
    return out
