"""Injected compute for the CPU (gloo) test of bench.py's N-rank path: the CPU
oracle stands in for the fused kernel (tests may use the oracle as the checker)."""
from oracle import oracle as O


def oracle_compute(qs, ks, vs, *, causal, seq_lens, scale_granularity, cfg, scales):
    out, _ = O.attention_batched(qs, ks, vs, causal=causal, seq_lens=seq_lens,
                                 scale_granularity=scale_granularity, b=cfg.b, c=cfg.c,
                                 p_scale=cfg.p_format.value, scales=scales)
    return out
