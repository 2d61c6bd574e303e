"""Device timeline of one host-in/host-out call (torch.profiler / CUPTI): busy time of
H2D copies, kernels and D2H copies, and the span (is the call PCIe-bound, and do the
two copy directions overlap?).   python tools/e2e_timeline.py [C5]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2511_21513_b200 as ia  # noqa: E402
from paper_2511_21513_b200 import workloads  # noqa: E402

wl = workloads.make(sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "-v" else "C5")
qh, kh, vh = (torch.from_numpy(x).pin_memory() for x in (wl.q, wl.k, wl.v))
oh = torch.empty(wl.q.shape, dtype=torch.float32).pin_memory()
for _ in range(3):
    ia.int_attention_batched(qh, kh, vh, causal=wl.causal, seq_lens=wl.seq_lens, out=oh)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ia.int_attention_batched(qh, kh, vh, causal=wl.causal, seq_lens=wl.seq_lens, out=oh)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]


def kind(e):
    n = e.name.lower()
    if "memcpy" in n and "htod" in n:
        return "h2d"
    if "memcpy" in n and "dtoh" in n:
        return "d2h"
    if "memcpy" in n or "memset" in n:
        return "other"
    return "kernel"


def union(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    return tot + (cur[1] - cur[0] if cur else 0.0)


spans = {}
for e in ev:
    spans.setdefault(kind(e), []).append((e.time_range.start, e.time_range.end))
t0 = min(a for v in spans.values() for a, _ in v)
t1 = max(b for v in spans.values() for _, b in v)
print(f"span {(t1 - t0) / 1e3:.2f} ms")
for k, v in spans.items():
    print(f"{k:7s} n={len(v):5d} busy {union(v) / 1e3:8.2f} ms  first {(min(a for a, _ in v) - t0) / 1e3:7.2f}  last end {(max(b for _, b in v) - t0) / 1e3:7.2f}")
both = union(spans.get("h2d", [])) + union(spans.get("d2h", [])) - union(spans.get("h2d", []) + spans.get("d2h", []))
print(f"h2d/d2h overlap {both / 1e3:.2f} ms")
if "-v" in sys.argv:  # every copy / kernel interval, ms from the first
    for e in sorted(ev, key=lambda e: e.time_range.start):
        print(f"{kind(e):7s} {(e.time_range.start - t0) / 1e3:7.3f} {(e.time_range.end - t0) / 1e3:7.3f}  {e.name[:50]}")
