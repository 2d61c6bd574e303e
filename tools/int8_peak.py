"""Pin the dense INT8 tensor-core roofline peak of this pool's B200 once.

cuBLASLt ``torch._int_mm`` (and, for reference, this library's own tcgen05
``gemm_i8``) at M = N = K = 8192:
  burst     -- best single launch after warm-up (a kernel timed alone),
  sustained -- mean over a ~3 s back-to-back loop (a kernel timed inside a long run),
with the SM clock sampled during the sustained loop.  bench.py divides by the
pinned ``burst_tops`` (the larger, i.e. conservative, denominator) and also
reports the fraction of ``sustained_tops``.

    python tools/int8_peak.py [--out profiles/int8_peak.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402


def measure(fn, flops):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        n = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 3.0:
            for _ in range(50):
                fn()
            n += 50
            torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        sus = e0.elapsed_time(e1) / 1e3 / n
    return flops / best / 1e12, flops / sus / 1e12, clk.summary()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "int8_peak.json"))
    a = ap.parse_args()
    from paper_2511_21513_b200 import engine as E
    n = 8192
    A = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    B = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    bt = B.t().contiguous().t()
    flops = 2 * n ** 3
    res = {}
    b, s, c = measure(lambda: torch._int_mm(A, bt), flops)
    res["cublaslt_int_mm"] = {"burst_tops": b, "sustained_tops": s, "clocks": c}
    b2, s2, c2 = measure(lambda: E.gemm_i8(A, B), flops)
    res["tcgen05_gemm_i8 (this library)"] = {"burst_tops": b2, "sustained_tops": s2, "clocks": c2}
    best = max(res.values(), key=lambda r: r["burst_tops"])
    out = {"burst_tops": best["burst_tops"], "sustained_tops": best["sustained_tops"],
           "shape": "M=N=K=8192 int8 x int8 -> int32", "device": torch.cuda.get_device_name(),
           "source": "tools/int8_peak.py: best of the measured dense INT8 GEMMs", "detail": res}
    print(json.dumps(out, indent=1))
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
