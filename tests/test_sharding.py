"""Multi-GPU sharding launcher: host logic on CPU with gloo (world_size 2).

The per-rank compute is the CPU oracle here (tests may use it as the
checker); on a GPU box the same code path runs the fused kernel per rank.
The gathered result must be bit-identical to the unsharded oracle run --
per-head units need no cross-rank reduction, and "tensor" scale mode must
reproduce the global scales through the all-reduce(MAX) of the local amax.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2511_21513_b200 import sharding
from paper_2511_21513_b200.pipeline import AttentionConfig


def oracle_compute(qs, ks, vs, *, causal, seq_lens, scale_granularity, cfg, scales):
    out, _ = O.attention_batched(qs, ks, vs, causal=causal, seq_lens=seq_lens,
                                 scale_granularity=scale_granularity, b=cfg.b, c=cfg.c,
                                 p_scale=cfg.p_format.value, scales=scales)
    return out


def make_case(kind, seed=0):
    rng = np.random.default_rng(seed)
    if kind == "gqa":
        B, H, Hkv, L, d = 1, 8, 2, 160, 32
        lens = None
    elif kind == "varlen":
        B, H, Hkv, L, d = 5, 2, 2, 140, 16
        lens = rng.integers(1, L + 1, size=B)
    else:  # tensor-scale, MHA
        B, H, Hkv, L, d = 3, 4, 4, 96, 16
        lens = None
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    v = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    if lens is not None:
        for b, n in enumerate(lens):
            q[b, :, n:] = k[b, :, n:] = v[b, :, n:] = 0
    return q, k, v, lens


def test_plan_covers_every_group_once():
    for policy in ("contiguous", "lpt", "auto"):
        for world in (1, 2, 3, 8):
            lens = np.array([7045, 5404, 4438, 2584, 2876, 826, 1089, 638])
            ranks = sharding.plan(8, 16, 16, 7968, world, lens=lens, causal=True, policy=policy)
            seen = [(g.b, g.kvh) for r in ranks for g in r]
            assert sorted(seen) == [(b, h) for b in range(8) for h in range(16)]
            assert len(ranks) == world


def test_plan_balance():
    # C4-like: 8 equal KV groups over 8 ranks -> one whole KV head per rank
    ranks = sharding.plan(1, 32, 8, 16384, 8, causal=True)
    assert [len(r) for r in ranks] == [1] * 8
    assert [r[0].kvh for r in ranks] == list(range(8))
    # C5-like ragged lengths: LPT keeps the max load within one unit of the mean
    lens = np.array([7045, 5404, 4438, 2584, 2876, 826, 1089, 638, 1858, 6758, 5500, 7522,
                     4380, 5171, 7968, 6115])
    ranks = sharding.plan(16, 16, 16, 7968, 8, lens=lens, causal=True, policy="lpt")
    loads = [sum(g.cost for g in r) for r in ranks]
    biggest = max(g.cost for r in ranks for g in r)
    assert max(loads) - min(loads) <= biggest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, scale, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v, lens = make_case(kind)
        out, mine = sharding.sharded_attention(
            q, k, v, causal=True, seq_lens=lens, scale_granularity=scale,
            cfg=AttentionConfig(), compute=oracle_compute, gather_to=0)
        result_q.put((rank, None if out is None else out.tobytes(), len(mine)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,scale", [("gqa", "head"), ("varlen", "head"),
                                        ("tensor", "tensor")])
def test_world2_gloo_bit_identical(kind, scale):
    ctx = mp.get_context("spawn")
    qres = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, scale, qres)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, blob, n = qres.get(timeout=180)
        res[r] = (blob, n)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q, k, v, lens = make_case(kind)
    want, _ = O.attention_batched(q, k, v, causal=True, seq_lens=lens, scale_granularity=scale)
    got = np.frombuffer(res[0][0], dtype=np.float32).reshape(want.shape)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert res[1][0] is None and res[0][1] + res[1][1] == q.shape[0] * k.shape[1]


def test_single_process_no_dist():
    q, k, v, lens = make_case("gqa")
    out, mine = sharding.sharded_attention(q, k, v, causal=True, compute=oracle_compute)
    want, _ = O.attention_batched(q, k, v, causal=True)
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("B,H,Hkv,L,d", [(1, 32, 8, 16384, 128), (16, 16, 16, 7968, 64),
                                         (64, 12, 12, 197, 64), (2, 4, 2, 300, 64),
                                         (3, 6, 2, 100, 32), (1, 3, 3, 50, 8)])
def test_host_chunk_plan_covers_every_unit_once(B, H, Hkv, L, d):
    """Host pipeline chunk plan: every (b, query head) is computed exactly once, with
    its own KV head's K / V sent by the chunk itself or by the previous chunk of the
    same group, and K / V sent exactly once per (b, KV head)."""
    from paper_2511_21513_b200.batched import chunk_plan
    G = H // Hkv
    per, chunks = chunk_plan(B, H, Hkv, L, d)
    seen_q, seen_kv = set(), set()
    last_kv = None
    for (b, j0, j1, qa, qb, send_kv) in chunks:
        assert j0 * G <= qa < qb <= j1 * G and j1 - j0 <= per
        if send_kv:
            for j in range(j0, j1):
                assert (b, j) not in seen_kv
                seen_kv.add((b, j))
            last_kv = (b, j0, j1)
        else:
            assert last_kv == (b, j0, j1)  # reuses the previous chunk's K / V
        for h in range(qa, qb):
            assert (b, h) not in seen_q
            seen_q.add((b, h))
    assert seen_q == {(b, h) for b in range(B) for h in range(H)}
    assert seen_kv == {(b, j) for b in range(B) for j in range(Hkv)}
