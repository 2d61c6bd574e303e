"""Quick GPU sanity check with per-stage diagnostics (development tool)."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
import torch
import paper_2511_21513_b200 as ia
from oracle import oracle as O


def diff(name, got, want):
    got, want = np.asarray(got), np.asarray(want)
    if got.shape != want.shape:
        print(f"  {name}: SHAPE {got.shape} vs {want.shape}"); return False
    bad = np.argwhere(got != want)
    if bad.size == 0:
        print(f"  {name}: OK"); return True
    i = tuple(bad[0])
    print(f"  {name}: {len(bad)} diffs / {got.size}; first {i}: got {got[i]} want {want[i]}")
    return False


def run(L, d, causal=False, seed=0, scale=1.0):
    print(f"case L={L} d={d} causal={causal}", flush=True)
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((L, d), dtype=np.float32) * np.float32(scale)
    k = rng.standard_normal((L, d), dtype=np.float32) * np.float32(scale)
    v = rng.standard_normal((L, d), dtype=np.float32) * np.float32(scale)
    mask = np.triu(np.ones((L, L), bool), 1) if causal else None
    t0 = time.time()
    out, dbg = ia.int_attention_batched(q[None, None], k[None, None], v[None, None],
                                        causal=causal, debug=True)
    torch.cuda.synchronize()
    print(f"  gpu call {time.time()-t0:.3f}s")
    qh, sq = O.quantize_tensor(q); kh, sk = O.quantize_tensor(k); vh, sv = O.quantize_tensor(v)
    ok = diff("qhat", dbg["qhat"][0, :, :d].cpu().numpy(), qh)
    ok &= diff("khat", dbg["khat"][0, :, :d].cpu().numpy(), kh)
    vt = dbg["vt"][0, :d, :L].cpu().numpy()
    ok &= diff("vt", vt, vh.T)
    lg = O.matmul_s8(qh, kh)
    got_lg = dbg["logits"][0].cpu().numpy()
    keep = ~mask if causal else np.ones((L, L), bool)
    ok &= diff("logits", np.where(keep, got_lg, 0), np.where(keep, lg, 0))
    ci = O.c_int(6.6, d, sq, sk)
    pr = O.index_softmax(lg, ci, O.build_lut(), mask=mask)
    ok &= diff("prob", dbg["prob"][0].cpu().numpy(), pr)
    acc = O.gemm_pv(pr, vh)
    ok &= diff("acc", dbg["acc"][0, :, :d].cpu().numpy(), acc)
    want = O.int_attention(q, k, v, mask=mask)
    ok &= diff("out", out[0, 0].view(np.uint32), want.view(np.uint32))
    return ok


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    allok = True
    for args in [(128, 64), (128, 128), (197, 64), (256, 128, True), (384, 128), (600, 128, True),
                 (300, 64, True), (100, 32), (512, 256, True)]:
        try:
            allok &= run(*args)
        except Exception as e:
            print("  EXC", type(e).__name__, e); allok = False
            break
    print("ALL OK" if allok else "FAILURES")
