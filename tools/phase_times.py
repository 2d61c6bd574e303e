"""Per-CTA phase clocks of the fused kernel (development instrumentation)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # run with IA_LIB=paper_2511_21513_b200/_lib/libintattn_b200_prof.so
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
n_qt = (L + 127) // 128
times = torch.zeros((n_qt * B * H, 16), dtype=torch.int64, device=dev)
for it in range(3):
    times.zero_()
    E.attn_fused(prep, (B, H, Hkv, L, d), out, causal=wl.causal, seq_lens=sl, lut=lut, times=times)
torch.cuda.synchronize()
t = times.cpu().numpy()
ok = t[:, 5] > 0
t = t[ok]
nkt = t[:, 10].astype(float)
pro = t[:, 0] - t[:, 6]; p1 = t[:, 1] - t[:, 0]; p2 = t[:, 2] - t[:, 1]; p3 = t[:, 3] - t[:, 2]
ow = t[:, 4] - t[:, 3]; ep = t[:, 5] - t[:, 4]
tot = t[:, 5] - t[:, 6]
print(f"{name}: CTAs {len(t)}  mean n_kt {nkt.mean():.1f}")
for nm, x in [("prologue", pro), ("pass1", p1), ("pass2", p2), ("pass3", p3), ("o_wait", ow), ("epilogue", ep), ("total", tot)]:
    print(f"  {nm:9s} mean {x.mean():10.0f} cyc  per-tile {np.mean(x / np.maximum(nkt, 1)):8.1f}")
print(f"  PV issuer wait p_full per tile {np.mean(t[:, 11] / nkt):.1f}  v_full per tile {np.mean(t[:, 12] / nkt):.1f}  softmax(wg0) p_free per own tile {np.mean(t[:, 13] / (nkt / 3)):.1f}")
print(f"  softmax(wg0) s_full wait per own tile: pass1 {np.mean(t[:, 15] / (nkt / 3)):.1f}  passes2+3 {np.mean(t[:, 14] / (2 * nkt / 3)):.1f}")
print(f"  QK issuer wait s_free per tile {np.mean(t[:, 8] / (3 * nkt)):.1f}  k_full per tile {np.mean(t[:, 9] / (3 * nkt)):.1f}")
