"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference measures on no public benchmark for this path;
these seeded numpy PCG64 recipes stand in for real activations.  They are
generated once on the host and the *identical* f32 tensors are fed to the GPU
path and to the CPU oracle.  Draw order is fixed: (lengths, C5 only) -> Q -> K
-> V -> outlier channels.

C1 equals ``intattn.cli.gen_inputs(128, 64, 0)`` byte for byte
(reference ``pkg/src/intattn/cli.py:88-94``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Workload:
    """One attention configuration over (batch, head) units.

    q: [B, H, L, d] f32; k, v: [B, Hkv, L, d] f32.  ``seq_lens`` (C5 only)
    gives the valid length per batch entry; rows at or beyond it are zero.
    ``scale_granularity`` is "head" (one scale per (b, head) slab) or "tensor"
    (one global scale per Q/K/V tensor).
    """

    name: str
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    causal: bool
    scale_granularity: str = "head"
    seq_lens: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def shape(self):
        B, H, L, d = self.q.shape
        return B, H, self.k.shape[1], L, d

    def lengths(self):
        B, H, Hkv, L, d = self.shape
        if self.seq_lens is None:
            return np.full(B, L, dtype=np.int64)
        return np.asarray(self.seq_lens, dtype=np.int64)

    def pairs(self):
        """Unmasked (query, key) pairs summed over all (b, h) units."""
        B, H, Hkv, L, d = self.shape
        lens = self.lengths()
        if self.causal:
            per_b = lens * (lens + 1) // 2
        else:
            per_b = lens * lens
        return int(per_b.sum()) * H

    def ops(self):
        """Algorithmic integer ops: 4*d per unmasked pair (QK^T + PV, 2 ops/MAC).

        SURVEY.md §8d: recompute passes and softmax ALU work are not counted.
        """
        return 4 * self.shape[4] * self.pairs()

    def ops_l2(self):
        """The reference CLI's convention 4*L^2*d per head (cli.py:148-150)."""
        B, H, Hkv, L, d = self.shape
        lens = self.lengths()
        return int((4 * d * lens * lens).sum()) * H

    def tokens(self):
        return int(self.lengths().sum())

    def min_bytes(self):
        """Algorithmic HBM minimum: f32 QKV read + int8 write+read + f32 O write."""
        nq = self.q.size
        nkv = self.k.size + self.v.size
        return 4 * (nq + nkv) + 2 * (nq + nkv) + 4 * nq


def _rope_neox(x: np.ndarray, base: float = 10000.0) -> np.ndarray:
    """NeoX rotate-half RoPE over positions 0..L-1, computed in f64, cast to f32."""
    L, d = x.shape[-2], x.shape[-1]
    half = d // 2
    inv = base ** (-np.arange(half, dtype=np.float64) * 2.0 / d)
    ang = np.arange(L, dtype=np.float64)[:, None] * inv[None, :]
    cos, sin = np.cos(ang), np.sin(ang)
    x64 = x.astype(np.float64)
    x1, x2 = x64[..., :half], x64[..., half:]
    out = np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], axis=-1)
    return out.astype(np.float32)


def _scale_channels(x: np.ndarray, channels: np.ndarray, factor: float) -> None:
    """Multiply hidden-dim channels (indices into the flattened H*d) in place, in f32."""
    B, H, L, d = x.shape
    f = np.float32(factor)
    for ch in channels:
        h, c = divmod(int(ch), d)
        x[:, h, :, c] *= f


def make_c1(seed: int = 0) -> Workload:
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((128, 64), dtype=np.float32)
    k = rng.standard_normal((128, 64), dtype=np.float32)
    v = rng.standard_normal((128, 64), dtype=np.float32)
    return Workload("C1", q[None, None], k[None, None], v[None, None], causal=False)


def make_c2(seed: int = 0, scale_granularity: str = "tensor") -> Workload:
    B, H, L, d = 64, 12, 197, 64
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, H, L, d), dtype=np.float32)
    v = rng.standard_normal((B, H, L, d), dtype=np.float32)
    ch = rng.choice(H * d, 15, replace=False)  # round(2% of 768)
    for x in (q, k, v):
        _scale_channels(x, ch, 8.0)
    return Workload("C2", q, k, v, causal=False, scale_granularity=scale_granularity,
                    meta={"outlier_channels": ch.tolist()})


def make_c3(seed: int = 0) -> Workload:
    B, H, L, d = 1, 32, 2048, 128
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, H, L, d), dtype=np.float32)
    v = rng.standard_normal((B, H, L, d), dtype=np.float32)
    q = _rope_neox(q)
    k = _rope_neox(k)
    return Workload("C3", q, k, v, causal=True)


def make_c4(seed: int = 0) -> Workload:
    B, H, Hkv, L, d = 1, 32, 8, 16384, 128
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    v = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    q_ch = rng.choice(H * d, 41, replace=False)     # 1% of 4096
    kv_ch = rng.choice(Hkv * d, 10, replace=False)  # 1% of 1024, shared by K and V
    _scale_channels(q, q_ch, 10.0)
    _scale_channels(k, kv_ch, 10.0)
    _scale_channels(v, kv_ch, 10.0)
    return Workload("C4", q, k, v, causal=True,
                    meta={"q_channels": q_ch.tolist(), "kv_channels": kv_ch.tolist()})


def make_c5(seed: int = 0) -> Workload:
    B, H, d = 16, 16, 64
    rng = np.random.default_rng(seed)
    lens = rng.integers(512, 8192, size=B, endpoint=True)
    L = int(lens.max())
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, H, L, d), dtype=np.float32)
    v = rng.standard_normal((B, H, L, d), dtype=np.float32)
    for b, n in enumerate(lens):
        q[b, :, n:] = 0
        k[b, :, n:] = 0
        v[b, :, n:] = 0
    return Workload("C5", q, k, v, causal=True, seq_lens=lens.astype(np.int32))


def make_tiny(seed: int = 0) -> Workload:
    """Not a BASELINE config: a seconds-sized GQA + varlen causal batch for the CPU
    (gloo) test of bench.py's multi-rank path."""
    B, H, Hkv, d = 3, 4, 2, 32
    rng = np.random.default_rng(seed)
    lens = rng.integers(40, 96, size=B, endpoint=True)
    L = int(lens.max())
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    v = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    for b, n in enumerate(lens):
        q[b, :, n:] = k[b, :, n:] = v[b, :, n:] = 0
    return Workload("tiny", q, k, v, causal=True, seq_lens=lens.astype(np.int32))


MAKERS = {"C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5,
          "tiny": make_tiny}


def make(name: str, seed: int = 0) -> Workload:
    return MAKERS[name](seed)
