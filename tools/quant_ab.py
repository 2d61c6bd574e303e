"""Quantiser timing per config (CUDA events, median of --iters), for A/B runs of the
quant_heads launch forms:  IA_QH_SPLIT=0|1 IA_QH_KB=<keys> python tools/quant_ab.py"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_21513_b200 import engine as E  # noqa: E402
from paper_2511_21513_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C4,C5")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--scale", default="head", choices=["head", "tensor"])
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    for name in args.configs.split(","):
        wl = workloads.make(name)
        q, k, v = (torch.from_numpy(x).to(dev) for x in (wl.q, wl.k, wl.v))
        sl = None if wl.seq_lens is None else torch.from_numpy(wl.seq_lens).to(dev)
        for _ in range(3):
            E.prepare(q, k, v, seq_lens=sl, scale_granularity=args.scale)
        ts = []
        for _ in range(args.iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            E.prepare(q, k, v, seq_lens=sl, scale_granularity=args.scale)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(x.elapsed_time(y) for x, y in ts)
        print(json.dumps({"config": name, "ms_prepare": round(ms, 4),
                          "split": os.environ.get("IA_QH_SPLIT"), "kb": os.environ.get("IA_QH_KB"),
                          "waves": os.environ.get("IA_QH_WAVES"), "scale": args.scale}))


if __name__ == "__main__":
    main()
