"""All five BASELINE configs on one GPU: device time (CUDA events), TOPS,
tokens/s, and bit-exact check of every (b, head) unit against the reference's
golden digests.  Writes one JSON line per config (profiles/ summary input).

    python tools/bench_all.py [--configs C1,C2,...] [--iters 10]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from cases import digest  # noqa: E402
from golden_io import configs  # noqa: E402
from paper_2511_21513_b200 import engine as E  # noqa: E402
from paper_2511_21513_b200 import workloads  # noqa: E402


def run(name, iters, softmax="index", k_group_size=None, graph=False):
    G = configs().get(name)
    wl = workloads.make("C2" if name == "C2h" else name)
    gran = "head" if name == "C2h" else wl.scale_granularity
    B, H, Hkv, L, d = wl.shape
    dev = torch.device("cuda", 0)
    q, k, v = (torch.from_numpy(x).to(dev) for x in (wl.q, wl.k, wl.v))
    sl = None if wl.seq_lens is None else torch.from_numpy(wl.seq_lens).to(dev)
    out = torch.empty_like(q)
    lut = E.lut_bytes(5, 6.6)

    class T:
        def __init__(self):
            self.ev = {}

        def mark(self, n):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.ev[n] = e

    E.attention(q, k, v, causal=wl.causal, seq_lens=sl, scale_granularity=gran, lut=lut, out=out, softmax=softmax,
                k_group_size=k_group_size)
    for _ in range(3):
        E.attention(q, k, v, causal=wl.causal, seq_lens=sl, scale_granularity=gran, lut=lut,
                    out=out, check_finite=False, softmax=softmax, k_group_size=k_group_size)
    ts = []
    for _ in range(iters):
        t = T()
        E.attention(q, k, v, causal=wl.causal, seq_lens=sl, scale_granularity=gran, lut=lut,
                    out=out, check_finite=False, timer=t, softmax=softmax, k_group_size=k_group_size)
        ts.append(t)
    torch.cuda.synchronize()
    tot = statistics.median(t.ev["start"].elapsed_time(t.ev["attention"]) for t in ts) / 1e3
    graph_ms = None
    if graph:  # the same call replayed from a CUDA graph (no host gaps between launches)
        G_ = E.AttentionGraph(q, k, v, out, causal=wl.causal, seq_lens=sl, scale_granularity=gran,
                              lut=lut, softmax=softmax, k_group_size=k_group_size)
        for _ in range(3):
            G_.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            G_.replay()
        e1.record()
        torch.cuda.synchronize()
        graph_ms = e0.elapsed_time(e1) / iters
        G_.check()
    att = statistics.median(t.ev["quantized"].elapsed_time(t.ev["attention"]) for t in ts) / 1e3
    qnt = statistics.median(t.ev["start"].elapsed_time(t.ev["quantized"]) for t in ts) / 1e3
    res = out.cpu().numpy()
    exact = None
    if G is not None and softmax == "index" and k_group_size is None:
        lens = wl.lengths()
        bad = 0
        u = 0
        for b in range(B):
            for h in range(H):
                n = int(lens[b])
                if digest(res[b, h, :n]) != G["unit_digests"][u] or res[b, h, n:].view(np.uint32).any():
                    bad += 1
                u += 1
        exact = bad == 0
    ops = wl.ops()
    # algorithmic quantiser bytes over VALID rows only (pad rows are never read)
    qbytes = 5 * int(wl.lengths().sum()) * (H + 2 * Hkv) * d
    return {"config": name, "softmax": softmax, "k_group_size": k_group_size, "shape": [B, H, Hkv, L, d], "causal": wl.causal, "scale": gran,
            "ms_total": tot * 1e3, "ms_quantize": qnt * 1e3, "ms_fused": att * 1e3,
            "ms_step_graph": graph_ms,
            "tops_total": ops / tot / 1e12, "tops_fused": ops / att / 1e12,
            "tokens_per_s": wl.tokens() / tot, "quantizer_gbs": qbytes / qnt / 1e9,
            "bit_exact_vs_reference": exact,
            "ref_cpu_seconds_survey": None if G is None else G.get("ref_seconds")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C2h,C3,C4,C5")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--softmax", default="index", choices=["index", "float", "both"],
                    help="float = the quant-only comparator mode of the fused kernel")
    ap.add_argument("--graph", action="store_true",
                    help="also time the step replayed from a CUDA graph")
    ap.add_argument("--k-group-size", type=int, default=None,
                    help="grouped K (per-row-group key scales) in the fused kernel")
    a = ap.parse_args()
    for name in a.configs.split(","):
        for sm in (("index", "float") if a.softmax == "both" else (a.softmax,)):
            print(json.dumps(run(name, a.iters, sm, a.k_group_size, a.graph)), flush=True)


if __name__ == "__main__":
    main()
