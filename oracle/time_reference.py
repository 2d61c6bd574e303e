"""Time the LIVE reference (numpy / numba / OpenBLAS, imported read-only from
/root/reference) beside this repo's C port of it (oracle/intattn_oracle.c) on the
same host cores and the same C3 heads, at T = 1 and T = cpu_count threads
(the reference's own two settings, pipeline.py:194-199).  Runs in
the build container only (the reference does not travel to the GPU box); the
result, profiles/cpu_reference_vs_port.json, states the port / reference speed
ratio that qualifies bench.py's ``cpu_baseline`` (kind "port").

    python oracle/time_reference.py [--heads 4] [--workload C3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_ref_cache"))
sys.dont_write_bytecode = True
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import intattn as ref  # noqa: E402  (the reference)

from oracle import oracle as O  # noqa: E402
from paper_2511_21513_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--heads", type=int, default=4)
    a = ap.parse_args()
    wl = workloads.make(a.workload)
    B, H, Hkv, L, d = wl.shape
    g = H // Hkv
    heads = list(range(min(a.heads, H)))
    mask = np.triu(np.ones((L, L), bool), 1) if wl.causal else None
    ops = 4 * d * (L * (L + 1) // 2 if wl.causal else L * L) * len(heads)
    # warm the reference's numba JIT on a tiny call first
    t = np.zeros((8, 8), np.float32) + 1
    ref.int_attention(t, t, t)
    res = {"workload": a.workload, "heads": len(heads), "host_cores": os.cpu_count(),
           "ops": ops, "by_threads": {}}
    for threads in sorted({1, os.cpu_count() or 1}):
        # reference: its own int_attention per head, total_ns from its StageTimings
        ref_ns = 0
        outs = []
        for h in heads:
            o, tm = ref.int_attention(wl.q[0, h], wl.k[0, h // g], wl.v[0, h // g],
                                      ref.AttentionConfig(mask=mask, threads=threads))
            ref_ns += tm.total_ns
            outs.append(np.asarray(o))
        # port: the same heads through the C restatement (same inputs, same thread count)
        t0 = time.perf_counter()
        po, _ = O.attention_batched(wl.q[:, heads], wl.k[:, [h // g for h in heads]],
                                    wl.v[:, [h // g for h in heads]], causal=wl.causal,
                                    threads=threads)
        port_s = time.perf_counter() - t0
        same = all(np.array_equal(po[0, j].view(np.uint32), outs[j].view(np.uint32))
                   for j in range(len(heads)))
        res["by_threads"][str(threads)] = {
            "reference_s": ref_ns / 1e9, "reference_tops": ops / (ref_ns / 1e9) / 1e12,
            "port_s": port_s, "port_tops": ops / port_s / 1e12,
            "port_over_reference": (ref_ns / 1e9) / port_s, "outputs_bit_identical": same}
        print(threads, res["by_threads"][str(threads)], flush=True)
    out = os.path.join(ROOT, "profiles", "cpu_reference_vs_port.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
