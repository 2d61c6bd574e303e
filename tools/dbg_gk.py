import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_2511_21513_b200 import engine as E
rng = np.random.default_rng(0)
B, H, Hkv, L, d, gs = 1, 1, 1, 96, 32, 32
dev = torch.device("cuda", 0)
q, k, v = (torch.from_numpy(rng.standard_normal(s, dtype=np.float32)).to(dev) for s in [(B, H, L, d), (B, Hkv, L, d), (B, Hkv, L, d)])
prep, gp = E.prepare_grouped(q, k, v, gs)
torch.cuda.synchronize(); print("prepare ok", prep.k_scales.cpu().numpy(), gp.view(torch.int32).cpu().numpy().reshape(-1, 4))
out = torch.empty_like(q)
E.attn_fused(prep, (B, H, Hkv, L, d), out, lut=E.lut_bytes(5, 6.6), kgroup=gp, k_group_size=gs)
torch.cuda.synchronize(); print("attn ok", out.abs().max().item())
