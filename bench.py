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

Multi-GPU: ``--gpus N`` (N > 1) re-executes itself under torch.distributed.run
with one rank per GPU when it is not already running under torchrun.  The ONE
workload is then sharded (strong scaling): ``sharding.plan`` gives every rank
whole (batch, KV-head) groups -- C4 on 8 GPUs = 1 KV head + its 4 query heads
per GPU, C5 by LPT over L_b^2 costs -- and each rank quantises and attends its
groups on its own device with no data-path collective.  The timed region is
bracketed by barrier + synchronize and the max over ranks is reported; the
NCCL gather of the device outputs to rank 0 (and an all-gather) is timed
separately.  After timing, the full output is checked unit by unit against the
live reference's digests (tests/golden/configs.json): the line carries
``"parity": "bit-exact"`` and the run exits non-zero otherwise.

``--impl reference`` times the CPU oracle port (oracle/, the reference
algorithm restated in C) on the host cores on a bounded row sample.
"""
from __future__ import annotations

import argparse
import importlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(1, os.path.join(ROOT, "tests"))  # golden_io: the reference's digests

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

def sample_stride(wl, target_s=12.0, threads=0):
    """Row stride giving a ~target_s oracle run (the C port sustains ~20 GOPS per
    core on the GPU box's host: 0.32 TOPS on 16 threads for C4)."""
    est_gops = 20.0 * (threads or os.cpu_count() or 8)
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


def cpu_baseline_one(wl, steps, warmup, threads, target_s):
    stride = sample_stride(wl, target_s, threads)
    ops, rows = sampled_ops(wl, stride)
    for _ in range(warmup):
        cpu_oracle_step(wl, stride, threads)
    ts = [cpu_oracle_step(wl, stride, threads) for _ in range(steps)]
    t = statistics.median(ts)
    return {"value": ops / t / 1e12, "unit": "TOPS", "cores": threads, "kind": "port",
            "sample": f"{wl.name}: every {stride}th query row of every (b, head) unit "
                      f"({rows} rows/head-slab set, {ops / 1e9:.1f} G algorithmic ops) incl. "
                      f"full-tensor quantisation; oracle/intattn_oracle.c, {threads} threads",
            "seconds_per_sample": t}, ts


def cpu_baseline(wl, steps=1, warmup=0, threads=None, target_s=12.0):
    """The reference algorithm on the host cores at T = 1 and T = cpu_count (the
    reference's own two settings, pipeline.py:194-199); the faster
    is reported, both are kept in ``by_threads``."""
    from oracle import oracle as O
    O.build()
    counts = [threads] if threads else sorted({1, os.cpu_count() or 1})
    runs = {}
    for t in counts:
        # the single-thread leg samples ~1/4 of the wall time budget
        runs[t] = cpu_baseline_one(wl, steps, warmup, t, target_s if t > 1 else target_s / 4)
    best_t = max(runs, key=lambda t: runs[t][0]["value"])
    cb, ts = runs[best_t]
    cb = dict(cb)
    cb["by_threads"] = {str(t): round(r[0]["value"], 6) for t, r in runs.items()}
    return cb, ts


def run_reference(args, wl_name):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    from paper_2511_21513_b200 import workloads
    wl = workloads.make(wl_name)
    # every step is a bounded sample; the whole --steps/--warmup run stays ~2.5 min
    target = max(0.25, min(12.0, 150.0 / (args.steps + args.warmup)))
    cb, ts = cpu_baseline(wl, steps=args.steps, warmup=args.warmup,
                          threads=os.cpu_count() or 1, target_s=target)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "TOPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(ts), "higher_is_better": True,
            "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "int8/int32 (u8 P)",
            "data": "synthetic (seeded PCG64, SURVEY.md §8d recipe)",
            "config": {"workload": wl_name, "sample": cb["sample"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "TOPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- shared

def int8_peak():
    """The pinned dense INT8 roofline peak (profiles/int8_peak.json: cuBLASLt
    torch._int_mm at 8192^3, burst and sustained, measured once by
    tools/int8_peak.py on this pool's B200); the datasheet figure otherwise."""
    path = os.path.join(ROOT, "profiles", "int8_peak.json")
    if os.path.exists(path):
        pk = json.load(open(path))
        return float(pk["burst_tops"]), pk
    return INT8_DATASHEET_TOPS, {"source": "datasheet (profiles/int8_peak.json missing)"}


def parity_check(out_host, wl, wl_name, reference=None):
    """Digest every (b, head) unit of the timed path's output against the live
    reference's digests (tests/golden/configs.json), or -- for a workload with no
    golden -- against ``reference`` (the unsharded result).  Returns the JSON
    ``parity`` string and whether it passed."""
    if reference is not None:
        ok = np.array_equal(out_host.view(np.uint32), reference.view(np.uint32))
        return ("bit-exact (vs the unsharded computation)" if ok else
                "MISMATCH vs the unsharded computation"), ok
    try:
        from golden_io import unit_mismatches
        bad, n = unit_mismatches(out_host, wl, wl_name)
    except (KeyError, FileNotFoundError):
        return "unchecked (no golden digests for this workload)", True
    if bad:
        return f"MISMATCH: {len(bad)} of {n} units differ from the reference digests, first {bad[:4]}", False
    return "bit-exact", True


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn(args):
    """``--gpus N`` outside torchrun: re-execute this script with one rank per GPU
    (torch.distributed.run, rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _load_compute(spec):
    mod, _, fn = spec.partition(":")
    return getattr(importlib.import_module(mod), fn)


# ----------------------------------------------------------------------------- GPU arm, N = 1

def run_gpu(args, wl_name):
    import torch
    from paper_2511_21513_b200 import engine as E
    from paper_2511_21513_b200 import workloads
    import paper_2511_21513_b200 as ia

    torch.cuda.set_device(0)
    wl = workloads.make(wl_name)
    B, H, Hkv, L, d = wl.shape
    dev = torch.device("cuda", 0)
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
    timers = []
    with ClockSampler(0) as clk:
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
    # parity of the timed launch shape itself: the output of the last timed step
    parity, parity_ok = parity_check(out.cpu().numpy(), wl, wl_name)

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

    e2e_t, e_ts = _time_e2e(args, e2e_step, torch)
    e2e_parity, e2e_ok = parity_check(oh.numpy(), wl, wl_name)

    # ---- the paper's comparator on the same inputs: quant-only mode of the fused
    # kernel (dequantise -> f32 softmax -> requantise between the same INT8 MMAs)
    qo_ms = None
    if not args.no_comparator:
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
    value = ops / step_s / 1e12
    pk, pk_src = peaks()
    peak_val, peak_info = int8_peak()
    attn_avg = statistics.mean(attn_s)
    achieved = ops / attn_avg / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{wl_name}.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
    cb = None
    if not args.no_cpu_baseline:
        cb, _ = cpu_baseline(wl, steps=1)
    valid_elems = _valid_elems(wl)
    line = {
        "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int8 MMA / int32 accumulate / u8 P (f32 in/out)",
        "data": "synthetic (seeded PCG64, SURVEY.md §8d recipe)",
        "config": {"workload": wl_name, "B": B, "H": H, "Hkv": Hkv, "L": L, "d": d,
                   "causal": wl.causal, "scale_granularity": gran,
                   "parallelism": "1 GPU, all (batch x KV-head) groups in one launch",
                   "l2": "inputs (402 MB f32 for C4) exceed the 126 MB L2; no flush"},
        "parity": parity,
        "tokens_per_s": tokens / step_s,
        "tops_per_gpu": value,
        "pct_int8_peak": 100.0 * value / peak_val,
        "ops_per_step": ops, "ops_convention": "4*d*unmasked pairs (SURVEY.md §8d)",
        "stage_ms": {"quantize": 1e3 * statistics.mean(quant_s),
                     "fused_attention": 1e3 * attn_avg},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_val,
                     "unit": "TOPS", "frac": achieved / peak_val, "traffic": traffic,
                     "peak_source": peak_info,
                     "frac_of_sustained": (achieved / peak_info["sustained_tops"]
                                           if "sustained_tops" in peak_info else None),
                     "frac_of_datasheet": achieved / INT8_DATASHEET_TOPS,
                     "kernel": "attn_fwd_kernel<128,false> (one launch per step)"},
        "quantizer_roofline": {"bound": "hbm",
                               "achieved_gbs": 5 * valid_elems / statistics.mean(quant_s) / 1e9,
                               "bytes": "5 B per valid element (f32 read + int8 write)",
                               "peak_gbs": pk["hbm_gbs"], "peak_source": pk_src},
        "e2e": {"value": ops / e2e_t / 1e12, "unit": "TOPS",
                "h2d_bytes_per_step": 4 * (wl.q.size + wl.k.size + wl.v.size),
                "d2h_bytes_per_step": 4 * wl.q.size,
                "parity": e2e_parity,
                "path": "int_attention_batched(pinned host f32 in, pinned host f32 out; "
                        "chunked H2D / kernel / D2H overlap inside the call)",
                "timing": f"median wall time of {len(e_ts)} calls",
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
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                    "by_threads")}
    print(json.dumps(line))
    return 0 if (parity_ok and e2e_ok) else 1


def _valid_elems(wl):
    B, H, Hkv, L, d = wl.shape
    lens = wl.lengths()
    return int(lens.sum()) * (H + 2 * Hkv) * d


def _time_e2e(args, fn, torch, world=1, dist=None):
    for _ in range(max(1, args.warmup)):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # per-call wall times (each call returns with the result on the host); the median
    # keeps one host-side hiccup (page faults, scheduler) from setting the number
    e_steps = max(3, min(args.steps, 30))
    e_ts = []
    import gc
    gc.collect()
    gc.disable()  # a collector pass inside a ~10 ms call would be measured as PCIe time
    try:
        for _ in range(e_steps):
            e0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            e_ts.append(time.perf_counter() - e0)
    finally:
        gc.enable()
    return statistics.median(e_ts), e_ts


# ----------------------------------------------------------------------------- N ranks

def run_sharded(args, wl_name, compute=None):
    """One workload sharded over the ranks (strong scaling).  ``compute`` (a
    ``module:function`` spec, CPU tests only) replaces the device compute and
    switches the process group to gloo."""
    import torch
    import torch.distributed as dist
    from paper_2511_21513_b200 import sharding, workloads

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    cpu = compute is not None
    if cpu:
        dist.init_process_group("gloo")
        fn = _load_compute(compute)
        from paper_2511_21513_b200.pipeline import AttentionConfig
        cfg0 = AttentionConfig()
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = workloads.make(wl_name)  # the same problem on every rank (seed 0)
    B, H, Hkv, L, d = wl.shape
    g = H // Hkv
    gran = wl.scale_granularity
    lens = wl.seq_lens
    ranks = sharding.plan(B, H, Hkv, L, world, lens=lens, causal=wl.causal)
    mine = ranks[rank]
    qs, ks, vs, sl = sharding.pack(wl.q, wl.k, wl.v, mine, g, lens)
    my_ops = 0
    if mine:
        my_ops = sum(4 * d * gr.cost for gr in mine)

    if cpu:
        def step():
            sc = sharding.global_scales(qs, ks, vs, sl, world=world) if gran == "tensor" else None
            return fn(qs, ks, vs, causal=wl.causal, seq_lens=sl, scale_granularity=gran,
                      cfg=cfg0, scales=sc) if mine else None

        for _ in range(args.warmup):
            step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            local_out = step()
        elapsed = time.perf_counter() - t0
        tt = torch.tensor([elapsed], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
        g0 = time.perf_counter()
        full = sharding.gather_blocks(local_out, ranks, rank, (B, H, L, d), g, gather_to=0)
        gather_s = time.perf_counter() - g0
        clocks, fused_s, extra = None, None, {}
    else:
        from paper_2511_21513_b200 import engine as E
        import paper_2511_21513_b200 as ia
        dev = torch.device("cuda", local)
        lut = E.lut_bytes(5, 6.6)
        if mine:
            qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (qs, ks, vs))
            sl_d = None if sl is None else torch.from_numpy(sl).to(dev)
            out_d = torch.empty_like(qd)
        else:
            qd = kd = vd = sl_d = out_d = None

        def step(timer=None):
            sc = None
            if gran == "tensor":  # all-reduce(MAX) of the 3 local amax values (NCCL, on device)
                sc = sharding.global_scales(qd, kd, vd, sl, world=world, device_out=True)
            if mine:
                E.attention(qd, kd, vd, causal=wl.causal, seq_lens=sl_d,
                            scale_granularity="tensor" if sc else gran, lut=lut, out=out_d,
                            check_finite=False, timer=timer, scales=sc)
            elif timer is not None:
                for n in ("start", "quantized", "attention"):
                    timer.mark(n)
            return out_d

        if mine:
            E.attention(qd, kd, vd, causal=wl.causal, seq_lens=sl_d, scale_granularity=gran,
                        lut=lut, out=out_d, check_finite=True,
                        scales=None if gran != "tensor" else
                        sharding.global_scales(qd, kd, vd, sl, world=world, device_out=True))
        elif gran == "tensor":
            sharding.global_scales(None, None, None, None, world=world, device_out=True)
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()

        class Ev:
            def __init__(self):
                self.ev = {}

            def mark(self, n):
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                self.ev[n] = e

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
        fused_s = statistics.mean(tm.ev["quantized"].elapsed_time(tm.ev["attention"]) / 1e3
                                  for tm in timers)
        tt = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
        clocks = clk.summary()

        # the NCCL output exchange, timed on its own (device events, max over ranks):
        # gather to rank 0 (what the API does for gather_to=0) and an all-gather
        def timed(fn_, reps=3):
            best = None
            res = None
            for _ in range(reps):
                torch.cuda.synchronize()
                dist.barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                res = fn_()
                e1.record()
                torch.cuda.synchronize()
                x = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
                dist.all_reduce(x, op=dist.ReduceOp.MAX)
                best = float(x.item()) if best is None else min(best, float(x.item()))
            return best, res

        gather_s, full = timed(lambda: sharding.gather_blocks(out_d, ranks, rank, (B, H, L, d), g,
                                                               gather_to=0))
        all_gather_s, _ = timed(lambda: sharding.gather_blocks(out_d, ranks, rank, (B, H, L, d), g,
                                                                gather_to="all"))
        if full is not None:
            full = full.cpu().numpy()

        # end to end through the public API on each rank's host-resident share
        e2e_t = None
        if mine:
            qh, kh, vh = (torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (qs, ks, vs))
            oh = torch.empty(qh.shape, dtype=torch.float32).pin_memory()

            def e2e_step():
                ia.int_attention_batched(qh, kh, vh, causal=wl.causal, seq_lens=sl,
                                         scale_granularity=gran, out=oh)
        else:
            def e2e_step():
                pass
        if gran == "head":
            e2e_t, _ = _time_e2e(args, e2e_step, torch, world, dist)
            x = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            e2e_t = float(x.item())
        extra = {"all_gather_ms": 1e3 * all_gather_s, "e2e_s": e2e_t}

    seen = torch.tensor([1], dtype=torch.int64, device="cpu" if cpu else torch.device("cuda", local))
    dist.all_reduce(seen)
    rc = 0
    if rank == 0:
        reference = None
        if cpu:
            reference = fn(wl.q, wl.k, wl.v, causal=wl.causal, seq_lens=wl.seq_lens,
                           scale_granularity=gran, cfg=cfg0, scales=None)
        parity, ok = parity_check(full, wl, wl_name, reference=reference)
        rc = 0 if ok else 1
        ops = wl.ops()
        step_s = elapsed / args.steps
        value = ops / step_s / 1e12
        peak_val, peak_info = int8_peak()
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world,
            "ranks_seen": int(seen.item()),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int8 MMA / int32 accumulate / u8 P (f32 in/out)",
            "data": "synthetic (seeded PCG64, SURVEY.md §8d recipe)",
            "config": {"workload": wl_name, "B": B, "H": H, "Hkv": Hkv, "L": L, "d": d,
                       "causal": wl.causal, "scale_granularity": gran,
                       "parallelism": f"{world} ranks x (batch, KV-head) groups "
                                      f"({'lpt' if lens is not None else 'contiguous'} plan)",
                       "groups_per_rank": [len(r) for r in ranks],
                       "l2": "per-rank inputs are resident; no flush"},
            "parity": parity,
            "tokens_per_s": wl.tokens() / step_s,
            "tops_per_gpu": value / world,
            "ops_per_step": ops, "ops_convention": "4*d*unmasked pairs (SURVEY.md §8d)",
            "gather_ms": 1e3 * gather_s,
            "gather": "dist.gather of every rank's f32 output block to rank 0 "
                      f"({'gloo' if cpu else 'NCCL over NVLink'}), timed separately from the step",
        }
        if not cpu:
            line["all_gather_ms"] = extra["all_gather_ms"]
            line["stage_ms"] = {"fused_attention_rank0": 1e3 * fused_s}
            if my_ops and fused_s:
                line["roofline"] = {"bound": "tensor", "achieved": my_ops / fused_s / 1e12,
                                    "peak": peak_val, "unit": "TOPS",
                                    "frac": my_ops / fused_s / 1e12 / peak_val, "traffic": None,
                                    "peak_source": peak_info,
                                    "kernel": "attn_fwd_kernel<128,false> on rank 0's groups"}
            if extra["e2e_s"]:
                line["e2e"] = {"value": ops / extra["e2e_s"] / 1e12, "unit": "TOPS",
                               "h2d_bytes_per_step": 4 * (wl.q.size + wl.k.size + wl.v.size),
                               "d2h_bytes_per_step": 4 * wl.q.size,
                               "path": "int_attention_batched on each rank's pinned host share; "
                                       "max over ranks of the median call"}
            line["gpu_launches"] = 3 * args.steps
            line["clocks"] = clocks
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4", choices=["C1", "C2", "C3", "C4", "C5", "tiny"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-comparator", action="store_true",
                    help="skip timing the quant-only comparator mode")
    ap.add_argument("--sharded", action="store_true",
                    help="run the N-rank sharded path even at N = 1 (exercises the NCCL "
                         "launcher on a single GPU)")
    ap.add_argument("--compute", default=None,
                    help="module:function replacing the device compute of the N-rank path "
                         "(gloo; CPU tests of the launcher only)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.impl == "reference":
        return run_reference(args, args.workload)
    if _env_int("WORLD_SIZE", 1) > 1 or args.compute or args.sharded:
        return run_sharded(args, args.workload, compute=args.compute)
    return run_gpu(args, args.workload)


if __name__ == "__main__":
    sys.exit(main())
