"""One small pass over every fused-kernel mode (development tool): the three-pass path (5
key tiles, causal, GQA), the resident path with a ragged varlen batch, grouped K, the
quant-only mode and per-tensor scales, each checked bit for bit against the CPU oracle.
(compute-sanitizer is closed on this GPU pool, so small oracle-checked cases like these,
the kernels' own watchdogs and the argument validation are the memory-safety evidence.)"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2511_21513_b200 as ia
from oracle import oracle as O

rng = np.random.default_rng(7)


def mk(B, H, Hkv, L, d):
    return (rng.standard_normal((B, H, L, d), dtype=np.float32),
            rng.standard_normal((B, Hkv, L, d), dtype=np.float32),
            rng.standard_normal((B, Hkv, L, d), dtype=np.float32))


def eq(name, got, want):
    ok = np.array_equal(np.asarray(got).view(np.uint32), np.asarray(want).view(np.uint32))
    print(f"{name}: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
    return ok


ok = True
q, k, v = mk(1, 2, 1, 640, 128)                       # three passes, causal, GQA
ok &= eq("three-pass causal GQA", ia.int_attention_batched(q, k, v, causal=True),
         O.attention_batched(q, k, v, causal=True)[0])
q, k, v = mk(2, 2, 2, 200, 64)                        # resident, ragged, varlen
lens = np.array([200, 77], dtype=np.int32)
ok &= eq("resident varlen", ia.int_attention_batched(q, k, v, seq_lens=lens),
         O.attention_batched(q, k, v, seq_lens=lens)[0])
q, k, v = mk(1, 2, 1, 512, 64)                        # grouped K, two passes
ok &= eq("grouped K", ia.int_attention_batched(q, k, v, causal=True, k_group_size=32),
         O.attention_grouped_batched(q, k, v, 32, causal=True))
q, k, v = mk(1, 1, 1, 512, 128)                       # quant-only comparator (tolerance path)
got = ia.quant_only_attention_batched(q, k, v, causal=True)
print("quant-only finite:", bool(np.isfinite(np.asarray(got)).all()), flush=True)
q, k, v = mk(1, 2, 2, 300, 32)                        # per-tensor scales (two-launch quantiser)
ok &= eq("tensor scales", ia.int_attention_batched(q, k, v, scale_granularity="tensor"),
         O.attention_batched(q, k, v, scale_granularity="tensor")[0])
sys.exit(0 if ok else 1)
