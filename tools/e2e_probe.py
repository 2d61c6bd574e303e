"""Host<->device copy rates and the pipelined host-in/host-out call (development tool)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2511_21513_b200 as ia
from paper_2511_21513_b200 import workloads

wl = workloads.make("C4")
qh = torch.from_numpy(wl.q).pin_memory(); kh = torch.from_numpy(wl.k).pin_memory()
vh = torch.from_numpy(wl.v).pin_memory()
oh = torch.empty(wl.q.shape, dtype=torch.float32).pin_memory()
qd = torch.empty_like(qh, device="cuda")

def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n

h2d = t(lambda: qd.copy_(qh, non_blocking=True))
d2h = t(lambda: oh.copy_(qd, non_blocking=True))
print(f"H2D {qh.numel()*4/h2d/1e9:.1f} GB/s  D2H {qh.numel()*4/d2h/1e9:.1f} GB/s")
s2 = torch.cuda.Stream()
def both():
    qd.copy_(qh, non_blocking=True)
    with torch.cuda.stream(s2):
        oh.copy_(qd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
bt = t(both)
print(f"H2D+D2H concurrent 2x{qh.numel()*4/1e6:.0f} MB: {bt*1e3:.2f} ms")
call = t(lambda: ia.int_attention_batched(qh, kh, vh, causal=True, out=oh))
print(f"pipelined call {call*1e3:.2f} ms")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ia.int_attention_batched(qh, kh, vh, causal=True, out=oh)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
