"""Batched multi-head / GQA / causal / variable-length entry point.

The reference API is single-head ("multi-head batching is a loop
over independent heads at the CLI layer").  ``int_attention_batched`` is that
loop done on the device: one launch sequence covers every (b, h) unit, and each
unit's output is bit-identical to ``int_attention(q[b, h], k[b, h // g],
v[b, h // g], AttentionConfig(mask=...))`` on the unit's valid rows
(SURVEY.md §3.5, §8d).
"""
from __future__ import annotations

import os
from collections import OrderedDict

import numpy as np
import torch

from . import _lib
from . import engine as E
from ._tensors import is_torch, to_device, to_host
from .gemm import MAX_SEQ_LEN
from .pipeline import AttentionConfig


def int_attention_batched(q, k, v, *, causal=False, seq_lens=None, mask=None,
                          scale_granularity="head", cfg=None, out=None, debug=False,
                          check_finite=True, softmax="index", k_group_size=None):
    """Fused IntAttention over all (b, h) units.

    q: [B, H, L, d] f32; k, v: [B, Hkv, L, d] f32 with H % Hkv == 0.
    causal: key j > query i excluded.  seq_lens: [B] valid lengths (rows at or
    beyond are padding: excluded as keys, +0.0 output as queries).  mask:
    optional bool [L, L] (True = excluded) shared by all units.
    scale_granularity: "head" (one scale per (b, head) slab over its valid rows)
    or "tensor" (one global scale per Q/K/V tensor).
    cfg: AttentionConfig for b, c and p_format (granularity/mask/threads unused).
    k_group_size: grouped K -- one K scale per (b, KV head, group of k_group_size keys)
    and the grouped IndexSoftmax (softmax.py:309-399; a power of two in [8, 128]
    dividing L, d <= 128), fused in one launch.
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
    host_in = all((not is_torch(x)) or x.device.type == "cpu" for x in (q, k, v))
    if (host_in and not debug and scale_granularity == "head" and B * ks[1] > 1
            and softmax == "index" and k_group_size is None):
        return _host_pipelined(q, k, v, causal=causal, seq_lens=seq_lens, mask=mask, cfg=cfg,
                               out=out, check_finite=check_finite, numpy_in=numpy_in)
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
    host_out = out is not None and is_torch(out) and out.device.type == "cpu"
    if out is not None and not is_torch(out):
        raise TypeError("out must be a torch.Tensor")
    if host_out and (out.dtype != torch.float32 or tuple(out.shape) != (B, H, L, d)
                     or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous float32 tensor of shape {(B, H, L, d)}")
    # a CUDA ``out`` is validated (device, dtype, shape, contiguity) by E.attention
    o = None if (out is None or host_out) else out
    res = E.attention(qt, kt, vt, causal=causal, seq_lens=sl, mask=mt,
                      scale_granularity=scale_granularity, b=cfg.b, c=cfg.c,
                      p_scale=cfg.p_format.value, out=o, debug=debug,
                      check_finite=check_finite, softmax=softmax, k_group_size=k_group_size)
    dbg = None
    if debug:
        res, dbg = res
    if host_out:
        out.copy_(res)
        res = out
        if numpy_in:
            res = out.numpy()
    else:
        res = to_host(res, numpy_in)
    return (res, dbg) if debug else res


def quant_only_attention_batched(q, k, v, *, causal=False, seq_lens=None, mask=None,
                                 scale_granularity="head", cfg=None, out=None, debug=False,
                                 check_finite=True):
    """The paper's comparator over all (b, h) units: the same INT8 QK^T / P.V MMAs
    with the dequantise -> f32 softmax -> requantise detour of
    quant_only_attention (pipeline.py:259-296) instead of IndexSoftmax, fused
    (two passes: online max / sum-of-exp, then P^ and P.V).  exp is MUFU ex2, so
    P^ matches the reference to float tolerance, not bit for bit."""
    return int_attention_batched(q, k, v, causal=causal, seq_lens=seq_lens, mask=mask,
                                 scale_granularity=scale_granularity, cfg=cfg, out=out,
                                 debug=debug, check_finite=check_finite, softmax="float")


def _pinned(x):
    """Host f32 tensor view of a numpy array / CPU tensor (pinned when it already is)."""
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32))) if not is_torch(x) \
        else x.to(torch.float32).contiguous()
    return t


# captured host-pipeline graphs (least recently used last); each holds its chunk buffers
_GRAPHS: "OrderedDict[tuple, tuple]" = OrderedDict()
_SEEN: "OrderedDict[tuple, None]" = OrderedDict()  # keys called once (eager), bounded
_NO_GRAPH: set = set()
_GRAPH_CACHE = 2
_GRAPH_ON = os.environ.get("IA_NO_GRAPH", "0") != "1"


def chunk_plan(B, H, Hkv, L, d):
    """Chunks of the host pipeline: ~8+ chunks of whole KV groups (at least one KV head
    each).  With one KV head per chunk and GQA, each group is sent as two sub-chunks
    (K, V + the first half of its query heads, then the second half reusing the K / V
    already on the device): halves the pipeline fill (first H2D) and drain (last
    kernel + D2H) at no extra PCIe bytes.  Returns (KV heads per chunk, chunks) with
    chunk = (b, kv j0, kv j1, q head lo, q head hi, sends K/V)."""
    G = H // Hkv
    unit_bytes = 4 * L * d * (G + 2)
    per = max(1, min(Hkv, (B * Hkv * unit_bytes // 8) // unit_bytes))
    chunks = []
    for b in range(B):
        for j in range(0, Hkv, per):
            j1 = min(j + per, Hkv)
            if j1 - j == 1 and G >= 2:
                chunks.append((b, j, j1, j * G, j * G + G // 2, True))
                chunks.append((b, j, j1, j * G + G // 2, j1 * G, False))
            else:
                chunks.append((b, j, j1, j * G, j1 * G, True))
    return per, chunks


def _host_pipelined(q, k, v, *, causal, seq_lens, mask, cfg, out, check_finite, numpy_in):
    """Host-resident inputs with per-head scales: stream the problem through the
    device in (batch, KV-head group) chunks -- split into two query-head halves
    sharing the group's K/V when a chunk is a single GQA group -- so the
    host->device copy of chunk i+1, the fused kernel on chunk i and the
    device->host copy of chunk i-1 overlap (three CUDA streams; three Q / O slots,
    two K / V buffers).  Per-head scales and per-unit outputs depend only on the
    unit's own data, so every chunk's result is bit-identical to the one-shot
    launch."""
    dev = E.require_device()
    qh, kh, vh = _pinned(q), _pinned(k), _pinned(v)
    B, H, L, d = qh.shape
    Hkv = kh.shape[1]
    G = H // Hkv
    sl_h = None
    if seq_lens is not None:
        sl_h = np.asarray(seq_lens.cpu() if is_torch(seq_lens) else seq_lens).astype(np.int64)
        if sl_h.shape != (B,) or (sl_h < 0).any() or (sl_h > L).any():
            raise ValueError(f"seq_lens must be [B] with values in [0, {L}]")
    mt = None
    if mask is not None:
        mt = to_device(mask).to(torch.bool)
        if tuple(mt.shape) != (L, L):
            raise ValueError(f"mask must be {L}x{L}, got {tuple(mt.shape)}")
    per, chunks = chunk_plan(B, H, Hkv, L, d)
    if out is not None:
        # host inputs -> host output: ``out`` must be a host f32 tensor of the result's
        # shape (a CUDA ``out`` would silently not receive the result)
        if not is_torch(out) or out.device.type != "cpu":
            raise ValueError("with host inputs, out must be a CPU torch.Tensor")
        if out.dtype != torch.float32 or tuple(out.shape) != (B, H, L, d) or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous float32 tensor of shape {(B, H, L, d)}")
        oh = out
    else:
        oh = torch.empty((B, H, L, d), dtype=torch.float32, pin_memory=True)
    # lengths on the device before any capture (a pageable copy cannot be captured);
    # a captured graph keeps them alive with its entry
    sl_d = None if sl_h is None else torch.as_tensor(sl_h.astype(np.int32)).to(dev)

    def enqueue():
        """Every copy and launch of the call, stream-ordered (no host sync): run
        eagerly, or captured once into a CUDA graph and replayed."""
        # Q / O buffers triple-buffered per chunk, K / V double-buffered per KV group (a
        # group's second half reads the K / V its first half brought in)
        NS = 3  # Q / O slots: chunk i+3's copy only waits for chunk i's kernel
        slots = [{"q": torch.empty((1, per * G, L, d), dtype=torch.float32, device=dev),
                  "o": torch.empty((1, per * G, L, d), dtype=torch.float32, device=dev)}
                 for _ in range(NS)]
        kvbuf = [{"k": torch.empty((1, per, L, d), dtype=torch.float32, device=dev),
                  "v": torch.empty((1, per, L, d), dtype=torch.float32, device=dev)}
                 for _ in range(2)]
        main = torch.cuda.current_stream()
        s_in, s_run, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        for s in (s_in, s_run, s_out):
            s.wait_stream(main)
        q_read = [None] * NS    # last compute that read the slot's Q
        kv_read = [None, None]  # last compute that read the K / V buffer
        drained = [None] * NS   # device->host copy that last read the slot's output
        errs = [] if check_finite else False
        # K / V buffer of every chunk (a new group starts at each chunk that sends K / V)
        kv_of, g = [], -1
        for c in chunks:
            g += 1 if c[5] else 0
            kv_of.append(g % 2)
        loaded = [None] * len(chunks)

        def h2d(i):
            b, j0, j1, qa, qb, send_kv = chunks[i]
            si, kb = i % NS, kvbuf[kv_of[i]]
            # rows at or beyond seq_lens[b] never influence a result (excluded from the
            # amax, masked as keys, written as +0.0 as queries), so only valid rows cross
            # PCIe: one contiguous block per head when the batch entry is padded
            n = L if sl_h is None else int(sl_h[b])

            def put(dst, src):
                if n == L:
                    dst.copy_(src, non_blocking=True)
                elif n:  # the first n rows of every head: one pitched copy
                    row = L * d * 4  # head stride of both [1, heads, L, d] views
                    _lib.check(_lib.load().ia_copy_rows_async(
                        dst.data_ptr(), row, src.data_ptr(), row, n * d * 4, src.shape[1],
                        torch.cuda.current_stream().cuda_stream), "copy_rows")

            with torch.cuda.stream(s_in):
                if send_kv:
                    if kv_read[kv_of[i]] is not None:
                        s_in.wait_event(kv_read[kv_of[i]])
                    put(kb["k"][:, :j1 - j0], kh[b:b + 1, j0:j1])
                    put(kb["v"][:, :j1 - j0], vh[b:b + 1, j0:j1])
                if q_read[si] is not None:
                    s_in.wait_event(q_read[si])
                put(slots[si]["q"][:, :qb - qa], qh[b:b + 1, qa:qb])
                loaded[i] = torch.cuda.Event()
                loaded[i].record(s_in)

        # enqueue order H2D(i+1), kernel(i), D2H(i): the host never holds back the next
        # chunk's copy behind this chunk's launch overhead
        h2d(0)
        for i, (b, j0, j1, qa, qb, send_kv) in enumerate(chunks):
            if i + 1 < len(chunks):
                h2d(i + 1)
            si = i % NS
            nkv, nq = j1 - j0, qb - qa
            qs, os_ = slots[si]["q"][:, :nq], slots[si]["o"][:, :nq]
            kb = kvbuf[kv_of[i]]
            ks_, vs = kb["k"][:, :nkv], kb["v"][:, :nkv]
            with torch.cuda.stream(s_run):
                s_run.wait_event(loaded[i])
                if drained[si] is not None:
                    s_run.wait_event(drained[si])
                E.attention(qs, ks_, vs, causal=causal,
                            seq_lens=None if sl_d is None else sl_d[b:b + 1], mask=mt,
                            scale_granularity="head", b=cfg.b, c=cfg.c,
                            p_scale=cfg.p_format.value, out=os_, check_finite=errs)
                done = torch.cuda.Event()
                done.record(s_run)
                q_read[si] = done
                kv_read[kv_of[i]] = done
            with torch.cuda.stream(s_out):
                s_out.wait_event(done)
                oh[b:b + 1, qa:qb].copy_(os_, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_out)
                drained[si] = ev
        # join the side streams back into the calling (or capturing) stream
        main.wait_stream(s_in)
        main.wait_stream(s_run)
        main.wait_stream(s_out)
        return torch.stack(errs).amax() if errs else None

    # Pinned host tensors (no mask): the whole call is one CUDA graph, captured on the
    # second call with the same buffers and shapes and replayed after that, so the
    # ~4 ms of per-chunk host work (Python, argument packing, tensor-map encoding)
    # leaves the call and a busy host cannot starve the copy / compute pipeline.
    key = None
    if (mask is None and _GRAPH_ON and all(t.is_pinned() for t in (qh, kh, vh, oh))):
        key = (dev.index, qh.data_ptr(), kh.data_ptr(), vh.data_ptr(), oh.data_ptr(),
               tuple(qh.shape), tuple(kh.shape), None if sl_h is None else tuple(sl_h.tolist()),
               bool(causal), cfg.b, cfg.c, cfg.p_format.value, bool(check_finite))
    if key in _NO_GRAPH:
        key = None
    ent = _GRAPHS.get(key) if key is not None else None
    if ent is None and key is not None and key in _SEEN:
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g):
                flag = enqueue()
        except RuntimeError:  # capture refused: stay on the eager stream-ordered path
            _NO_GRAPH.add(key)
            key = None
        else:
            ent = _GRAPHS[key] = (g, flag, sl_d)
            while len(_GRAPHS) > _GRAPH_CACHE:
                _GRAPHS.popitem(last=False)
    if ent is not None:
        _GRAPHS.move_to_end(key)
        g, flag, _ = ent
        g.replay()
        torch.cuda.current_stream().synchronize()
    else:
        if key is not None:
            _SEEN[key] = None
            while len(_SEEN) > 16:
                _SEEN.popitem(last=False)
        flag = enqueue()
        torch.cuda.current_stream().synchronize()
    if flag is not None:  # one host read for every chunk's non-finite flag
        E.raise_if_nonfinite(flag)
    return oh.numpy() if numpy_in else oh
