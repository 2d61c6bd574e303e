"""SM clock, power and clock-event reasons sampled (NVML, ~5 ms) while the fused
kernel runs back to back for ~2 s on one config (development instrumentation).
    IA_XFLAGS=<bits> python tools/power_probe.py [C4]"""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2511_21513_b200 import engine as E  # noqa: E402
from paper_2511_21513_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
wl = workloads.make(name)
B, H, Hkv, L, d = wl.shape
dev = torch.device("cuda", 0)
q, k, v = (torch.from_numpy(x).to(dev) for x in (wl.q, wl.k, wl.v))
sl = None if wl.seq_lens is None else torch.from_numpy(wl.seq_lens).to(dev)
lut = E.lut_bytes(5, 6.6)
prep = E.prepare(q, k, v, seq_lens=sl, scale_granularity=wl.scale_granularity)
out = torch.empty_like(q)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1e3,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)


for _ in range(3):
    E.attn_fused(prep, (B, H, Hkv, L, d), out, causal=wl.causal, seq_lens=sl, lut=lut)
torch.cuda.synchronize()
th = threading.Thread(target=sampler)
th.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 0
t0 = time.time()
a.record()
while time.time() - t0 < 2.0:
    for _ in range(20):
        E.attn_fused(prep, (B, H, Hkv, L, d), out, causal=wl.causal, seq_lens=sl, lut=lut)
        n += 1
    torch.cuda.synchronize()
b.record()
torch.cuda.synchronize()
stop.set()
th.join()
ms = a.elapsed_time(b) / n
reasons = 0
for s in samples:
    reasons |= s[2]
print(f"{name} xflags={os.environ.get('IA_XFLAGS', '0')} ms/launch {ms:.4f}  sm_mhz median "
      f"{statistics.median(s[0] for s in samples)} min {min(s[0] for s in samples)}  power W median "
      f"{statistics.median(s[1] for s in samples):.0f} max {max(s[1] for s in samples):.0f}  reasons 0x{reasons:x}  samples {len(samples)}")
