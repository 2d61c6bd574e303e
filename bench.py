#!/usr/bin/env python
"""Benchmark of the B200 IntAttention forward path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl ours|reference]

A step is one full pass of the hot path over one batch of the workload: device
quantisation of f32 Q/K/V + the fused IntAttention kernel (QK^T -> IndexSoftmax
-> P.V -> rescale).  Default workload: BASELINE config 4 (LLaMA-style causal GQA
prefill, B=1, Hq=32, Hkv=8, L=16384, d=128) -- the config the north star's
"fraction of INT8 tensor peak at L >= 4096" target is quoted on.  Inputs are
seeded synthetic tensors (paper_2511_21513_b200/workloads.py) and are larger
than L2 (402 MB f32), so no L2 flush is needed between steps.

Multi-GPU (torchrun): weak scaling -- every rank processes its own batch entry
of the workload (independent (b, head) units, no data-path collective); the
timed region is bracketed by barrier + synchronize and the max over ranks is
reported.  ``--impl reference`` times the CPU oracle port (oracle/, the
reference algorithm restated in C) on the host cores on a bounded row sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IntAttention TOPS & tokens/s per GPU, % of INT8 tensor peak; bit-exact vs oracle"
INT8_DATASHEET_TOPS = 4500.0


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return json.load(open(path)), "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "B200_PROFILING.md fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (NVML at
    ~2 ms intervals; nvidia-smi fallback)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []  # (sm_mhz, max_mhz, reason_bits)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        self._max = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:  # match the CUDA device to its NVML handle by PCI bus id
                import torch
                want = self._norm_bus(torch.cuda.get_device_properties(gpu_index).pci_bus_id)
                for j in range(pynvml.nvmlDeviceGetCount()):
                    hj = pynvml.nvmlDeviceGetHandleByIndex(j)
                    bid = pynvml.nvmlDeviceGetPciInfo(hj).busId
                    if self._norm_bus(bid.decode() if isinstance(bid, bytes) else bid) == want:
                        h = hj
                        break
            except Exception:
                h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self._nvml = (pynvml, h)
        except Exception:
            self._nvml = None

    @staticmethod
    def _norm_bus(s):
        dom, _, rest = str(s).strip().upper().partition(":")
        return f"{int(dom, 16):x}:{rest}" if rest else str(s).upper()

    def _sample(self):
        if self._nvml:
            nv, h = self._nvml
            try:
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            if self._max is None:
                self._max = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            return (nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), self._max, int(rs))
        r = subprocess.run(["nvidia-smi", "-i", str(self.gpu),
                            "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True, timeout=5)
        f = [x.strip() for x in r.stdout.strip().split(",")]
        return (float(f[0]), float(f[1]), 0)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"]}
        sm = [s[0] for s in self.samples]
        bits = 0
        for s in self.samples:
            bits |= s[2]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(n for b, n in self.REASONS.items() if bits & b),
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


# ----------------------------------------------------------------------------- CPU arms

def sample_stride(wl, target_s=12.0):
    """Row stride giving a ~target_s oracle run (the C port sustains ~20 GOPS per
    core on the GPU box's host: 0.32 TOPS on 16 threads for C4)."""
    est_gops = 20.0 * (os.cpu_count() or 8)
    full_s = wl.ops() / (est_gops * 1e9)
    stride = 1
    while full_s / stride > target_s and stride < wl.shape[3]:
        stride *= 2
    return stride


def sampled_ops(wl, stride):
    B, H, Hkv, L, d = wl.shape
    lens = wl.lengths()
    pairs = 0
    for b in range(B):
        n = int(lens[b])
        rows = np.arange(0, n, stride, dtype=np.int64)
        pairs += int((rows + 1).sum() if wl.causal else rows.size * n)
    return 4 * d * pairs * H, int(sum(len(range(0, int(n), stride)) for n in lens))


def cpu_oracle_step(wl, stride, threads):
    from oracle import oracle as O
    t0 = time.perf_counter()
    O.attention_batched(wl.q, wl.k, wl.v, causal=wl.causal, seq_lens=wl.seq_lens,
                        scale_granularity=wl.scale_granularity, row_stride=stride,
                        threads=threads)
    return time.perf_counter() - t0


def cpu_baseline(wl, steps=1, warmup=0, threads=0, target_s=12.0):
    from oracle import oracle as O
    O.build()
    stride = sample_stride(wl, target_s)
    ops, rows = sampled_ops(wl, stride)
    for _ in range(warmup):
        cpu_oracle_step(wl, stride, threads)
    ts = [cpu_oracle_step(wl, stride, threads) for _ in range(steps)]
    t = statistics.median(ts)
    cores = threads or os.cpu_count()
    return {"value": ops / t / 1e12, "unit": "TOPS", "cores": cores, "kind": "port",
            "sample": f"{wl.name}: every {stride}th query row of every (b, head) unit "
                      f"({rows} rows/head-slab set, {ops / 1e9:.1f} G algorithmic ops) incl. "
                      f"full-tensor quantisation; oracle/intattn_oracle.c, {cores} threads",
            "seconds_per_sample": t}, ts


def run_reference(args, wl_name):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    from paper_2511_21513_b200 import workloads
    wl = workloads.make(wl_name)
    # every step is a bounded sample; the whole --steps/--warmup run stays ~2.5 min
    target = max(0.25, min(12.0, 150.0 / (args.steps + args.warmup)))
    cb, ts = cpu_baseline(wl, steps=args.steps, warmup=args.warmup, target_s=target)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "TOPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(ts), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8/int32 (u8 P)",
            "data": "synthetic (seeded PCG64, SURVEY.md §8d recipe)",
            "config": {"workload": wl_name, "sample": cb["sample"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "TOPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- GPU arm

def int8_peak_tops(torch):
    """Dense INT8 tensor throughput measured here: cuBLASLt (torch._int_mm) and
    this library's own tcgen05 GEMM at 8192^3; the larger is the roofline peak."""
    from paper_2511_21513_b200 import engine as E
    n = 8192
    a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    res = {}

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        return 2 * n ** 3 / best / 1e12

    try:
        bt = b.t().contiguous().t()
        res["cublaslt_int_mm"] = timeit(lambda: torch._int_mm(a, bt))
    except Exception as e:  # pragma: no cover
        res["cublaslt_int_mm_error"] = str(e)[:120]
    try:
        res["tcgen05_gemm_i8"] = timeit(lambda: E.gemm_i8(a, b))
    except Exception as e:  # pragma: no cover
        res["tcgen05_gemm_i8_error"] = str(e)[:120]
    vals = [v for v in res.values() if isinstance(v, float)]
    return (max(vals) if vals else None), res


def run_gpu(args, wl_name):
    import torch
    import torch.distributed as dist
    from paper_2511_21513_b200 import engine as E
    from paper_2511_21513_b200 import workloads
    import paper_2511_21513_b200 as ia

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = workloads.make(wl_name, seed=rank)
    B, H, Hkv, L, d = wl.shape
    dev = torch.device("cuda", local)
    q = torch.from_numpy(wl.q).to(dev)
    k = torch.from_numpy(wl.k).to(dev)
    v = torch.from_numpy(wl.v).to(dev)
    sl = None if wl.seq_lens is None else torch.from_numpy(wl.seq_lens).to(dev)
    out = torch.empty_like(q)
    lut = E.lut_bytes(5, 6.6)
    gran = wl.scale_granularity

    class Ev:
        def __init__(self):
            self.ev = {}

        def mark(self, n):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.ev[n] = e

    def step(timer=None):
        E.attention(q, k, v, causal=wl.causal, seq_lens=sl, scale_granularity=gran, lut=lut,
                    out=out, check_finite=False, timer=timer)

    # correctness guard: one checked run (non-finite flag) before timing
    E.attention(q, k, v, causal=wl.causal, seq_lens=sl, scale_granularity=gran, lut=lut,
                out=out, check_finite=True)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    timers = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            tm = Ev()
            step(tm)
            timers.append(tm)
        t1.record()
        torch.cuda.synchronize()
    elapsed = t0.elapsed_time(t1) / 1e3
    attn_s = [tm.ev["quantized"].elapsed_time(tm.ev["attention"]) / 1e3 for tm in timers]
    quant_s = [tm.ev["start"].elapsed_time(tm.ev["quantized"]) / 1e3 for tm in timers]
    if world > 1:
        tt = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
        dist.barrier()

    # ---- end-to-end through the public API: pinned host f32 in, host f32 out
    qh = torch.from_numpy(wl.q).pin_memory()
    kh = torch.from_numpy(wl.k).pin_memory()
    vh = torch.from_numpy(wl.v).pin_memory()
    oh = torch.empty(wl.q.shape, dtype=torch.float32).pin_memory()

    def e2e_step():
        # host in -> host out: the API streams (batch, KV-group) chunks through the
        # device with the H2D / kernel / D2H of consecutive chunks overlapped
        o = ia.int_attention_batched(qh, kh, vh, causal=wl.causal, seq_lens=wl.seq_lens,
                                     scale_granularity=gran, out=oh)
        assert o.device.type == "cpu"  # result is on the host when the call returns

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # per-call wall times (each call returns with the result on the host); the median
    # keeps one host-side hiccup (page faults, scheduler) from setting the number
    # (30 calls: host-side PCIe / memory contention on a shared box comes in bursts of
    # several calls; a longer window keeps the median out of one burst)
    e_steps = max(3, min(args.steps, 30))
    e_ts = []
    import gc
    gc.collect()
    gc.disable()  # a collector pass inside a ~10 ms call would be measured as PCIe time
    try:
        for _ in range(e_steps):
            e0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            e_ts.append(time.perf_counter() - e0)
    finally:
        gc.enable()
    e2e_t = statistics.median(e_ts)
    if world > 1:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())

    # ---- the paper's comparator on the same inputs: quant-only mode of the fused
    # kernel (dequantise -> f32 softmax -> requantise between the same INT8 MMAs)
    qo_ms = None
    if rank == 0 and not args.no_comparator:
        def qo_step():
            E.attention(q, k, v, causal=wl.causal, seq_lens=sl, scale_granularity=gran, lut=lut,
                        out=out, check_finite=False, softmax="float")
        for _ in range(2):
            qo_step()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        n_qo = max(3, min(args.steps, 10))
        c0.record()
        for _ in range(n_qo):
            qo_step()
        c1.record()
        torch.cuda.synchronize()
        qo_ms = c0.elapsed_time(c1) / n_qo

    ops = wl.ops()
    tokens = wl.tokens()
    step_s = elapsed / args.steps
    value = world * ops / step_s / 1e12
    line = None
    if rank == 0:
        pk, pk_src = peaks()
        int8_peak, int8_detail = int8_peak_tops(torch)
        attn_avg = statistics.mean(attn_s)
        achieved = ops / attn_avg / 1e12
        peak_val = int8_peak if int8_peak else INT8_DATASHEET_TOPS
        traffic = None
        tpath = os.path.join(ROOT, "profiles", f"traffic_{wl_name}.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb, _ = cpu_baseline(wl, steps=1)
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int8 MMA / int32 accumulate / u8 P (f32 in/out)",
            "data": "synthetic (seeded PCG64 per rank, SURVEY.md §8d recipe)",
            "config": {"workload": wl_name, "B_per_gpu": B, "H": H, "Hkv": Hkv, "L": L, "d": d,
                       "causal": wl.causal, "scale_granularity": gran,
                       "parallelism": f"dp{world} over (batch x head) units",
                       "l2": "inputs (402 MB f32 for C4) exceed the 126 MB L2; no flush"},
            "tokens_per_s": world * tokens / step_s,
            "tops_per_gpu": value / world,
            "pct_int8_peak": 100.0 * (ops / step_s / 1e12) / peak_val,
            "ops_per_step": ops, "ops_convention": "4*d*unmasked pairs (SURVEY.md §8d)",
            "stage_ms": {"quantize": 1e3 * statistics.mean(quant_s),
                         "fused_attention": 1e3 * attn_avg},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_val,
                         "unit": "TOPS", "frac": achieved / peak_val, "traffic": traffic,
                         "peak_source": "max of measured dense INT8 GEMMs at 8192^3 "
                                        f"(this run): {json.dumps(int8_detail)}; datasheet "
                                        f"{INT8_DATASHEET_TOPS} TOPS",
                         "frac_of_datasheet": achieved / INT8_DATASHEET_TOPS,
                         "kernel": "attn_fwd_kernel<128,false> (one launch per step)"},
            "quantizer_roofline": {"bound": "hbm",
                                   "achieved_gbs": 5 * (wl.q.size + wl.k.size + wl.v.size) / statistics.mean(quant_s) / 1e9,
                                   "peak_gbs": pk["hbm_gbs"], "peak_source": pk_src},
            "e2e": {"value": world * ops / e2e_t / 1e12, "unit": "TOPS",
                    "h2d_bytes_per_step": 4 * (wl.q.size + wl.k.size + wl.v.size),
                    "d2h_bytes_per_step": 4 * wl.q.size,
                    "path": "int_attention_batched(pinned host f32 in, pinned host f32 out; "
                            "chunked H2D / kernel / D2H overlap inside the call)",
                    "timing": f"median wall time of {e_steps} calls",
                    "calls_ms": [round(1e3 * x, 3) for x in e_ts]},
            # per step: ia_quant_heads + head_params + attn_fwd (the workspace memset is torch's)
            "gpu_launches": 3 * args.steps,
            "clocks": clk.summary(),
        }
        if qo_ms is not None:
            line["comparator"] = {
                "pipeline": "quant_only (pipeline.py:259-296) as the fused kernel's "
                            "IA_SOFTMAX_FLOAT mode, same quantiser and MMAs",
                "ms_per_step": qo_ms, "tops": ops / (qo_ms / 1e3) / 1e12,
                "int_attention_speedup": qo_ms / (1e3 * step_s)}
        if cb is not None:
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-comparator", action="store_true",
                    help="skip timing the quant-only comparator mode")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, args.workload)
    return run_gpu(args, args.workload)


if __name__ == "__main__":
    sys.exit(main())
