"""(batch x KV-head) sharding of the IntAttention forward across GPUs.

Every (b, KV head) group -- its KV head plus the H/Hkv query heads that read it
-- is independent: row max, row sum and normalisation are per query row, so
there is no inter-GPU reduction in per-head scale mode.  The
launcher therefore

  * plans which groups each rank owns (contiguous KV-head groups, or LPT --
    longest processing time first -- over causal/varlen costs, as config 5
    needs),
  * runs each rank's groups with the fused kernel on its own GPU (one process
    per GPU, ``torch.distributed`` over NCCL),
  * uses a collective only where the path has a real exchange: an
    all-reduce(MAX) of the three global amax values in ``scale_granularity=
    "tensor"`` mode, and an optional gather of the f32 outputs.

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
    """Gather the groups' slices into contiguous [n, g, L, d] / [n, 1, L, d] arrays."""
    idx_b = [gr.b for gr in groups]
    qs = np.stack([q[gr.b, gr.kvh * g:(gr.kvh + 1) * g] for gr in groups]) if groups else None
    ks = np.stack([k[gr.b, gr.kvh:gr.kvh + 1] for gr in groups]) if groups else None
    vs = np.stack([v[gr.b, gr.kvh:gr.kvh + 1] for gr in groups]) if groups else None
    sl = None if lens is None else np.asarray([lens[b] for b in idx_b], np.int32)
    return qs, ks, vs, sl


def _default_compute(qs, ks, vs, *, causal, seq_lens, scale_granularity, cfg, scales):
    from . import engine as E
    dev = torch.device("cuda", torch.cuda.current_device())
    qt, kt, vt = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (qs, ks, vs))
    sl = None if seq_lens is None else torch.from_numpy(seq_lens).to(dev)
    sc = None if scales is None else tuple(torch.tensor([s], dtype=torch.float32, device=dev)
                                           for s in scales)
    out = E.attention(qt, kt, vt, causal=causal, seq_lens=sl, scale_granularity=scale_granularity,
                      b=cfg.b, c=cfg.c, p_scale=cfg.p_format.value, scales=sc)
    return out.cpu().numpy()


def _local_amax(x, lens_per_group=None):
    a = np.abs(x)
    if not np.isfinite(a).all():
        raise ValueError("input contains non-finite elements")
    return np.float32(a.max()) if a.size else np.float32(0)


def sharded_attention(q, k, v, *, causal=False, seq_lens=None, scale_granularity="head",
                      cfg=None, group=None, gather_to=0, policy="auto", compute=None,
                      amax_device=None):
    """Run this rank's share of a batched IntAttention and (optionally) gather.

    Every rank passes the same full host arrays q [B,H,L,d], k/v [B,Hkv,L,d].
    Returns (out, groups): ``out`` is the full [B,H,L,d] f32 result on rank
    ``gather_to`` (None elsewhere) when gather_to is not None, else this rank's
    packed [n, g, L, d] block; ``groups`` lists this rank's (b, kvh) groups.
    """
    from .pipeline import AttentionConfig
    cfg = cfg or AttentionConfig()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, H, L, d = q.shape
    Hkv = k.shape[1]
    g = H // Hkv
    lens = None if seq_lens is None else np.asarray(seq_lens, np.int64)
    ranks = plan(B, H, Hkv, L, world, lens=lens, causal=causal, policy=policy)
    mine = ranks[rank]
    qs, ks, vs, sl = pack(q, k, v, mine, g, lens)

    scales = None
    if scale_granularity == "tensor":
        # one global scale per tensor: every rank contributes the amax of the rows
        # it owns; all-reduce(MAX) of 3 floats
        local = np.zeros(3, np.float32)
        if mine:
            for t, x in enumerate((qs, ks, vs)):
                if sl is None:
                    local[t] = _local_amax(x)
                else:
                    local[t] = max((_local_amax(x[u, :, :sl[u]]) for u in range(len(mine))),
                                   default=np.float32(0))
        dev = amax_device or torch.device("cpu")
        tl = torch.from_numpy(local).to(dev)
        if world > 1:
            dist.all_reduce(tl, op=dist.ReduceOp.MAX, group=group)
        amax = tl.cpu().numpy()
        scales = tuple(np.float32(np.maximum(a, np.float32(1e-12)) / np.float32(127)) for a in amax)

    fn = compute or _default_compute
    local_out = None
    if mine:
        local_out = fn(qs, ks, vs, causal=causal, seq_lens=sl, scale_granularity=scale_granularity,
                       cfg=cfg, scales=scales)
    if gather_to is None:
        return local_out, mine

    # gather: pad every rank's block to the largest group count
    max_n = max(len(r) for r in ranks)
    buf = np.zeros((max_n, g, L, d), np.float32)
    if mine:
        buf[:len(mine)] = local_out
    dev = amax_device or torch.device("cpu")
    t = torch.from_numpy(buf).to(dev)
    if world > 1:
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
    else:
        parts = [t]
    if rank != gather_to:
        return None, mine
    out = np.zeros((B, H, L, d), np.float32)
    for r, grs in enumerate(ranks):
        blk = parts[r].cpu().numpy()
        for u, gr in enumerate(grs):
            out[gr.b, gr.kvh * g:(gr.kvh + 1) * g] = blk[u]
    return out, mine
