"""Per-call wall time (ms) of the host-in/host-out API on one config, pinned buffers
(IA_NO_GRAPH=1: the eager stream-ordered path instead of the captured graph)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2511_21513_b200 as ia  # noqa: E402
from paper_2511_21513_b200 import workloads  # noqa: E402

wl = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "C4")
qh, kh, vh = (torch.from_numpy(x).pin_memory() for x in (wl.q, wl.k, wl.v))
oh = torch.empty(wl.q.shape, dtype=torch.float32).pin_memory()
for _ in range(3):
    ia.int_attention_batched(qh, kh, vh, causal=wl.causal, seq_lens=wl.seq_lens, out=oh)
rows = []
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    t0 = time.perf_counter()
    ia.int_attention_batched(qh, kh, vh, causal=wl.causal, seq_lens=wl.seq_lens, out=oh)
    t1 = time.perf_counter()
    rows.append(1e3 * (t1 - t0))
print(" ".join(f"{w:.2f}" for w in rows))
