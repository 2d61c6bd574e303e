"""Event timeline of CTAs 0 and 1000 of the fused kernel (development tool).
Run with IA_LIB=paper_2511_21513_b200/_lib/libintattn_b200_prof.so; writes
gpurun_out/trace_<cfg>.npz (raw entries) and prints per-event intervals."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2511_21513_b200 import engine as E, workloads

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
wl = workloads.make(name)
B, H, Hkv, L, d = wl.shape
dev = torch.device("cuda", 0)
q, k, v = (torch.from_numpy(x).to(dev) for x in (wl.q, wl.k, wl.v))
sl = None if wl.seq_lens is None else torch.from_numpy(wl.seq_lens).to(dev)
lut = E.lut_bytes(5, 6.6)
prep = E.prepare(q, k, v, seq_lens=sl, scale_granularity=wl.scale_granularity)
out = torch.empty_like(q)
grid = ((L + 127) // 128) * B * H
times = torch.zeros(grid * 16 + 32 * 2048, dtype=torch.int64, device=dev)
for it in range(3):
    times.zero_()
    E.attn_fused(prep, (B, H, Hkv, L, d), out, causal=wl.causal, seq_lens=sl, lut=lut, times=times)
torch.cuda.synchronize()
t = times.cpu().numpy()
tr = t[grid * 16:].reshape(2, 16, 2048)
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/trace_{name}.npz", tr=tr, slots=t[:grid * 16].reshape(grid, 16))
NAMES = {1: "Kprod got k_empty", 2: "QK got s_free", 3: "QK got k_full", 4: "QK committed",
         5: "Vprod got v_empty", 6: "PV got p_full", 7: "PV got v_full", 8: "WG s_full wake",
         9: "WG s_free arrive", 10: "WG p_free got", 11: "WG p_full arrive"}
for c in range(2):
    seg = tr[c]
    allc = seg[seg != 0] >> 16
    t0 = allc.min()
    print(f"== CTA {'0' if c == 0 else 1000}: span {allc.max() - t0} cycles")
    for s in range(16):
        e = seg[s][seg[s] != 0]
        if len(e) == 0:
            continue
        clk = (e >> 16) - t0
        ev = (e >> 12) & 0xF
        tile = e & 0xFFF
        for code in np.unique(ev):
            m = ev == code
            cc = clk[m]
            dd = np.diff(cc)
            print(f"  seg{s} {NAMES.get(int(code), code):20s} n={m.sum():4d} first {cc[0]:8d} last {cc[-1]:8d}"
                  f"  median step {np.median(dd) if len(dd) else 0:7.0f}")
