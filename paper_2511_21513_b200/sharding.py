"""(batch x KV-head) sharding of the IntAttention forward across GPUs.

Every (b, KV head) group -- its KV head plus the H/Hkv query heads that read it
-- is independent: row max, row sum and normalisation are per query row, so
there is no inter-GPU reduction in per-head scale mode.  The
reference has no multi-head loop at all (SPEC.md:344 leaves it to the caller);
this launcher is that loop spread over one process per GPU:

  * ``plan`` decides which groups each rank owns (contiguous KV-head groups, or
    LPT -- longest processing time first -- over causal / varlen costs, as
    config 5 needs);
  * ``pack`` gathers a rank's groups into contiguous [n, g, L, d] / [n, 1, L, d]
    blocks (on the device when the inputs are CUDA tensors);
  * each rank runs its groups through the fused kernel on its own GPU;
  * a collective runs only where the path has a real exchange: an
    all-reduce(MAX) of the three global amax values in ``scale_granularity=
    "tensor"`` mode, and the gather of the f32 outputs when the caller wants
    them on one device.  Under NCCL both run on the rank's CUDA device (NVLink);
    under gloo (CPU tests) on the host.

The per-rank compute is injectable (``compute=``) so the host logic -- plan,
pack, global-scale exchange, gather -- is testable on CPU with ``gloo``.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Group:
    """One independent unit of work: batch entry b, KV head kvh (and its query heads)."""

    b: int
    kvh: int
    cost: int


def group_costs(B, H, Hkv, L, lens=None, causal=False):
    g = H // Hkv
    out = []
    for b in range(B):
        n = L if lens is None else int(lens[b])
        pairs = n * (n + 1) // 2 if causal else n * n
        for kvh in range(Hkv):
            out.append(Group(b, kvh, g * pairs))
    return out


def plan(B, H, Hkv, L, world, *, lens=None, causal=False, policy="auto"):
    """Assign groups to ranks.  Returns a list (per rank) of Group lists.

    "contiguous": consecutive groups in (b, kvh) order, split so each rank's
    summed cost is as even as a contiguous cut allows (C3/C4: whole KV heads
    per GPU, so K^/V^ are never duplicated).  "lpt": sort by cost, give each
    to the currently least-loaded rank (C5's ragged lengths).  "auto": lpt
    when costs differ, contiguous otherwise.
    """
    groups = group_costs(B, H, Hkv, L, lens, causal)
    if world < 1:
        raise ValueError("world must be >= 1")
    if policy == "auto":
        policy = "lpt" if len({gr.cost for gr in groups}) > 1 else "contiguous"
    ranks = [[] for _ in range(world)]
    if policy == "contiguous":
        total = sum(gr.cost for gr in groups)
        acc, r = 0, 0
        for idx, gr in enumerate(groups):
            remaining = len(groups) - idx
            if r < world - 1 and ranks[r] and (acc >= total * (r + 1) / world or
                                               remaining <= world - 1 - r):
                r += 1
            ranks[r].append(gr)
            acc += gr.cost
    elif policy == "lpt":
        heap = [(0, r) for r in range(world)]
        for gr in sorted(groups, key=lambda x: (-x.cost, x.b, x.kvh)):
            load, r = heapq.heappop(heap)
            ranks[r].append(gr)
            heapq.heappush(heap, (load + gr.cost, r))
        for r in range(world):
            ranks[r].sort(key=lambda x: (x.b, x.kvh))
    else:
        raise ValueError(f"unknown policy {policy!r}")
    return ranks


def pack(q, k, v, groups, g, lens=None):
    """Gather the groups' slices into contiguous [n, g, L, d] / [n, 1, L, d] blocks
    (numpy in -> numpy out; torch in -> torch out on the same device) plus the
    per-group valid lengths (int32 numpy, or None)."""
    if not groups:
        return None, None, None, None
    stack = torch.stack if isinstance(q, torch.Tensor) else np.stack
    qs = stack([q[gr.b, gr.kvh * g:(gr.kvh + 1) * g] for gr in groups])
    ks = stack([k[gr.b, gr.kvh:gr.kvh + 1] for gr in groups])
    vs = stack([v[gr.b, gr.kvh:gr.kvh + 1] for gr in groups])
    sl = None if lens is None else np.asarray([lens[gr.b] for gr in groups], np.int32)
    return qs, ks, vs, sl


def collective_device(group=None) -> torch.device:
    """Where this process group's collectives run: the rank's CUDA device under
    NCCL (NVLink / NVSwitch), the host under gloo."""
    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _default_compute(qs, ks, vs, *, causal, seq_lens, scale_granularity, cfg, scales):
    """The rank's groups through the fused kernel.  CUDA tensors in -> CUDA tensor
    out (no host round trip); host arrays are copied to the device and the result
    copied back."""
    from . import engine as E
    dev = torch.device("cuda", torch.cuda.current_device())
    on_dev = isinstance(qs, torch.Tensor) and qs.is_cuda
    if on_dev:
        qt, kt, vt = (x.contiguous() for x in (qs, ks, vs))
    else:
        qt, kt, vt = (torch.as_tensor(np.ascontiguousarray(x)).to(dev) for x in (qs, ks, vs))
    sl = None if seq_lens is None else torch.as_tensor(seq_lens, dtype=torch.int32).to(dev)
    sc = None
    if scales is not None:
        sc = tuple(s.reshape(1).to(dev, torch.float32) if isinstance(s, torch.Tensor)
                   else torch.tensor([s], dtype=torch.float32, device=dev) for s in scales)
    out = E.attention(qt, kt, vt, causal=causal, seq_lens=sl, scale_granularity=scale_granularity,
                      b=cfg.b, c=cfg.c, p_scale=cfg.p_format.value, scales=sc)
    return out if on_dev else out.cpu().numpy()


def _local_amax_host(x, sl):
    """Exact max|x| over each packed group's valid rows (host arrays)."""
    best = np.float32(0)
    for u in range(x.shape[0]):
        rows = x[u] if sl is None else x[u, :, :int(sl[u])]
        a = np.abs(np.asarray(rows))
        if not np.isfinite(a).all():
            raise ValueError("input contains non-finite elements")
        if a.size:
            best = max(best, np.float32(a.max()))
    return best


def _local_amax_device(x, sl, amax_bits, err):
    """max|x| over the valid rows of every packed group with the library's amax
    kernel (float bits, exact) into the 1-element int32 slot ``amax_bits``."""
    from . import engine as E
    n, g, L, d = x.shape
    slt = None if sl is None else torch.as_tensor(sl, dtype=torch.int32).to(x.device)
    E.amax_rows(x.contiguous(), n * g, L, d, amax_bits, err, seq_lens=slt, valid_div=g,
                slot_div=n * g)


def global_scales(qs, ks, vs, sl, group=None, world=1, device_out=False):
    """Global per-tensor scales of a sharded batch: every rank contributes the amax
    of the rows it owns, all-reduce(MAX) of 3 values on the collective device, then
    s = max(amax, 1e-12) / 127 in f32 (quantize.py:113).

    CUDA inputs (NCCL): the amax kernel writes the float bits of the three local
    maxima (non-negative floats order as their int32 bits), NCCL all-reduces them
    with MAX and the library's scales kernel turns them into scales -- no host round
    trip; with ``device_out`` the three scales come back as 1-element f32 CUDA
    tensors (what ``engine.attention(scales=...)`` takes).  Host inputs (gloo):
    numpy amax, host all-reduce, numpy f32 scales."""
    cdev = collective_device(group)
    if isinstance(qs, torch.Tensor) and qs.is_cuda and cdev.type == "cuda" or (
            qs is None and cdev.type == "cuda"):
        from . import engine as E
        buf = torch.zeros(4, dtype=torch.int32, device=cdev)
        if qs is not None:
            for t, x in enumerate((qs, ks, vs)):
                _local_amax_device(x, sl, buf[t:t + 1], buf[3:])
            E.raise_if_nonfinite(buf[3:])
        amax = buf[:3]
        if world > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=group)
        sc = torch.empty(3, dtype=torch.float32, device=cdev)
        E.scales_from_amax(amax, sc)
        if device_out:
            return tuple(sc[t:t + 1] for t in range(3))
        return tuple(np.float32(x) for x in sc.cpu().numpy())
    if qs is None:
        local = torch.zeros(3, dtype=torch.float32)
    elif isinstance(qs, torch.Tensor) and qs.is_cuda:  # CUDA data under gloo
        from . import engine as E
        buf = torch.zeros(4, dtype=torch.int32, device=qs.device)
        for t, x in enumerate((qs, ks, vs)):
            _local_amax_device(x, sl, buf[t:t + 1], buf[3:])
        E.raise_if_nonfinite(buf[3:])
        local = buf[:3].view(torch.float32).cpu()
    else:
        local = torch.tensor([_local_amax_host(x, sl) for x in (qs, ks, vs)], dtype=torch.float32)
    local = local.to(cdev)
    if world > 1:
        dist.all_reduce(local, op=dist.ReduceOp.MAX, group=group)
    amax = local.cpu().numpy()
    return tuple(np.float32(np.maximum(a, np.float32(1e-12)) / np.float32(127)) for a in amax)


def gather_blocks(local_out, ranks, rank, shape, g, *, group=None, gather_to=0, like=None):
    """Gather every rank's packed [n_r, g, L, d] block into the full [B, H, L, d]
    output.  ``gather_to`` = a rank (dist.gather: only that rank receives, the
    NVLink traffic is (world - 1) blocks) or "all" (all_gather_into_tensor).  The
    full output is a CUDA tensor on the collective device under NCCL, else numpy
    (or a CPU tensor when ``like`` is a tensor); ranks that do not receive get None.
    """
    B, H, L, d = shape
    world = len(ranks)
    G = g
    cdev = collective_device(group)
    max_n = max(len(r) for r in ranks)
    blk = torch.zeros((max_n, G, L, d), dtype=torch.float32, device=cdev)
    if local_out is not None:
        src = local_out if isinstance(local_out, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(local_out))
        # device -> device stays stream-ordered; device -> host must be a blocking copy
        # (a non_blocking D2H returns before the bytes have landed)
        blk[:src.shape[0]].copy_(src, non_blocking=cdev.type == "cuda" and src.is_cuda)
    if world == 1:
        parts = [blk]
    elif gather_to == "all":
        big = torch.empty((world * max_n, G, L, d), dtype=torch.float32, device=cdev)
        dist.all_gather_into_tensor(big, blk, group=group) if cdev.type == "cuda" else \
            dist.all_gather(list(big.chunk(world)), blk, group=group)
        parts = list(big.chunk(world))
    else:
        recv = rank == gather_to
        parts = [torch.empty_like(blk) for _ in range(world)] if recv else None
        dist.gather(blk, parts, dst=gather_to, group=group)
        if not recv:
            return None
    # one indexed copy places every rank's groups: group (b, kvh) -> out[b, kvh*G:(kvh+1)*G]
    Hkv = H // G
    src = [r * max_n + u for r, grs in enumerate(ranks) for u in range(len(grs))]
    dst = [gr.b * Hkv + gr.kvh for grs in ranks for gr in grs]
    blocks = torch.cat(parts) if len(parts) > 1 else parts[0]
    if src != list(range(len(src))):  # ranks hold fewer than max_n groups: compact first
        blocks = blocks[torch.as_tensor(src, device=cdev)]
    out = torch.empty((B, H, L, d), dtype=torch.float32, device=cdev)
    out.view(B * Hkv, G, L, d).index_copy_(0, torch.as_tensor(dst, device=cdev),
                                            blocks[:len(src)])
    if cdev.type == "cuda" or isinstance(like, torch.Tensor):
        return out
    return out.numpy()


def sharded_attention(q, k, v, *, causal=False, seq_lens=None, scale_granularity="head",
                      cfg=None, group=None, gather_to=0, policy="auto", compute=None):
    """Run this rank's share of a batched IntAttention and (optionally) gather.

    Every rank passes the same full q [B,H,L,d], k/v [B,Hkv,L,d]: host arrays, or
    CUDA tensors on the rank's device (then packing, compute and collectives stay
    on the device).  Returns (out, groups): with ``gather_to`` a rank (default 0)
    or "all", ``out`` is the full [B,H,L,d] f32 result on the receiving rank(s)
    (a CUDA tensor under NCCL / for CUDA inputs, numpy for host inputs under gloo;
    None elsewhere); with ``gather_to=None`` it is this rank's packed [n, g, L, d]
    block.  ``groups`` lists this rank's (b, kvh) groups.
    """
    from .pipeline import AttentionConfig
    cfg = cfg or AttentionConfig()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, H, L, d = q.shape
    Hkv = k.shape[1]
    g = H // Hkv
    lens = None if seq_lens is None else np.asarray(
        seq_lens.cpu() if isinstance(seq_lens, torch.Tensor) else seq_lens, np.int64)
    ranks = plan(B, H, Hkv, L, world, lens=lens, causal=causal, policy=policy)
    mine = ranks[rank]
    qs, ks, vs, sl = pack(q, k, v, mine, g, lens)

    scales = None
    if scale_granularity == "tensor":
        scales = global_scales(qs, ks, vs, sl, group=group, world=world)

    fn = compute or _default_compute
    local_out = None
    if mine:
        local_out = fn(qs, ks, vs, causal=causal, seq_lens=sl, scale_granularity=scale_granularity,
                       cfg=cfg, scales=scales)
    if gather_to is None:
        return local_out, mine
    out = gather_blocks(local_out, ranks, rank, (B, H, L, d), g, group=group,
                        gather_to=gather_to, like=q)
    if out is not None and isinstance(q, torch.Tensor) and q.is_cuda and out.device != q.device:
        out = out.to(q.device)
    return out, mine
