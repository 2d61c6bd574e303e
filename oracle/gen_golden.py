"""Generate tests/golden/ from the LIVE reference (run in the build container).

The reference (/root/reference/pkg/src/intattn, pure Python + numba +
OpenBLAS) cannot travel to the GPU box, so this script imports it here and
commits its outputs as small fixtures:

  tests/golden/kats.json         SPEC.md example blocks / SURVEY.md §4 KATs
  tests/golden/stage_cases.json  per-stage digests + scalars for the seeded
                                 cases of tests/cases.py (quantised Q/K/V and
                                 scales, int32 logits, c_int, u8/i8 P, int32
                                 P.V, f32 output)
  tests/golden/stage_small.npz   full per-stage arrays for a few tiny cases
  tests/golden/configs.json      per-(b, head) scales, c_int and output
                                 digests for the five BASELINE configs
  tests/golden/errors.json       the exception class (or "ok") the reference raises for
                                 each call of tests/cases.py:error_cases()
  tests/golden/quant_only_cases.npz  quant_only_attention (pipeline.py:259-296)
                                 outputs and requantised P^ (float comparator)
  tests/golden/audit.json        the dataflow_audit (tag, dtype) stream of the calls in
                                 tests/cases.py:audit_cases()
  tests/golden/grouped_cases.npz index_softmax_grouped (softmax.py:309-399)
                                 inputs and outputs, incl. the grouped-K
                                 int_attention pipeline (pipeline.py:229-246)

Usage:  python oracle/gen_golden.py [--configs C1,C2,...] [--skip-stages] [--grouped-only]
The reference is imported read-only: bytecode writing is disabled and numba's
cache is redirected to a temp dir so nothing is written under /root/reference.
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

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import intattn as ia  # noqa: E402  (the reference)
from intattn import softmax as ref_sm  # noqa: E402

from cases import (audit_cases, case_inputs, case_list, digest, error_cases,  # noqa: E402
                   run_audit_case, run_error_case)
from paper_2511_21513_b200 import workloads  # noqa: E402


def f32hex(x) -> str:
    return float(np.float32(x)).hex()


def kats():
    out = {}
    q = ia.quantize_symmetric(np.array([[1.0, -2.0], [0.5, 2.54]], np.float32))
    out["quant_example"] = {"scale": f32hex(q.scales[0]), "values": q.values.tolist()}
    z = ia.quantize_symmetric(np.zeros((3, 4), np.float32))
    out["quant_zero"] = {"scale": f32hex(z.scales[0]), "values": z.values.tolist()}
    s = np.float32(0.01)
    e = ia.quantize_symmetric(np.array([[127 * s, -127 * s]], np.float32))
    out["quant_endpoints"] = {"values": e.values.tolist()}
    a = ia.QuantizedMatrix(np.array([[1, 2]], np.int8), np.array([0.05], np.float32),
                           ia.QuantGranularity.per_tensor())
    b = ia.QuantizedMatrix(np.array([[3, 4]], np.int8), np.array([0.04], np.float32),
                           ia.QuantGranularity.per_tensor())
    lm = ia.gemm_qk(a, b)
    out["gemm_qk"] = {"values": lm.values.tolist(), "alpha": float(lm.alpha).hex()}
    out["gemm_pv"] = {"values": ia.gemm_pv(np.array([[255]], np.uint8),
                                            np.array([[7, -3]], np.int8)).tolist()}
    out["c_int"] = {
        "6.6,128,0.05,0.04": ia.compute_c_int(6.6, 128, 0.05, 0.04).c_int,
        "6.6,1,6.6,1.0": ia.compute_c_int(6.6, 1, 6.6, 1.0).c_int,
        "6.6,4,100.0,100.0": ia.compute_c_int(6.6, 4, 100.0, 100.0).c_int,
    }
    out["lut"] = {f"{b},{c}": ia.build_lut(b, c).entries.tolist()
                  for b in range(2, 9) for c in (4.4, 5.5, 6.6, 7.7, 8.8)}
    lut = ia.build_lut(5, 6.6)
    sm = {}
    sm["uniform"] = ia.index_softmax(np.array([[100, 100], [100, 100]], np.int32), 37335, lut).values.tolist()
    sm["clip50"] = ia.index_softmax(np.array([[100, 40], [40, 100]], np.int32), 50, lut).values.tolist()
    sm["single"] = ia.index_softmax(np.array([[7]], np.int32), 5, lut).values.tolist()
    sm["masked"] = ia.index_softmax(np.array([[1, 2], [3, 4]], np.int32), 50, lut,
                                    mask=np.array([[False, True], [True, True]])).values.tolist()
    sm["int8x127"] = ia.index_softmax(np.array([[100, 100], [100, 40]], np.int32), 50, lut,
                                      p_format=ia.PFormat.INT8X127).values.tolist()
    out["index_softmax"] = sm
    out["index_table_50_32"] = ref_sm._index_table(50, 32).tolist()
    return out


def ref_stages(q, k, v, mask, b, c, p):
    """Reference per-stage outputs via its own primitives (pipeline.py:215-253)."""
    pf = ia.PFormat.UINT8X255 if p == 255 else ia.PFormat.INT8X127
    qh = ia.quantize_symmetric(q)
    kh = ia.quantize_symmetric(k)
    vh = ia.quantize_symmetric(v)
    lm = ia.gemm_qk(qh, kh)
    lut = ia.build_lut(b, c)
    ci = ia.compute_c_int(c, q.shape[1], qh.scales[0], kh.scales[0])
    prob = ia.index_softmax(lm, ci, lut, mask=mask, p_format=pf)
    acc = ia.gemm_pv(prob.values, vh)
    out = acc.astype(np.float32) * np.float32(float(vh.scales[0]) / prob.denom_scale)
    full, _ = ia.int_attention(q, k, v, ia.AttentionConfig(b=b, c=c, p_format=pf, mask=mask))
    assert np.array_equal(full.view(np.uint32), out.view(np.uint32))
    return dict(qh=qh.values, kh=kh.values, vh=vh.values, sq=qh.scales[0], sk=kh.scales[0],
                sv=vh.scales[0], logits=lm.values, alpha=lm.alpha, c_int=ci.c_int,
                lut=lut.entries, prob=prob.values, acc=acc, out=out)


def stage_cases():
    rows = []
    small = {}
    for i, case in enumerate(case_list()):
        q, k, v, mask = case_inputs(case)
        r = ref_stages(q, k, v, mask, case["b"], case["c"], case["p"])
        rows.append(dict(case=case,
                         sq=f32hex(r["sq"]), sk=f32hex(r["sk"]), sv=f32hex(r["sv"]),
                         alpha=float(r["alpha"]).hex(), c_int=int(r["c_int"]),
                         lut=r["lut"].tolist(),
                         digests={n: digest(r[n]) for n in
                                  ("qh", "kh", "vh", "logits", "prob", "acc", "out")}))
        if case["L"] <= 24 and len(small) < 8 * 13:
            for n in ("qh", "kh", "vh", "logits", "prob", "acc", "out"):
                small[f"{i}_{n}"] = r[n]
    with open(os.path.join(GOLD, "stage_cases.json"), "w") as f:
        json.dump(rows, f, indent=0)
    np.savez_compressed(os.path.join(GOLD, "stage_small.npz"), **small)
    print(f"stage cases: {len(rows)}, small arrays: {len(small)}")


def config_golden(name, threads):
    wl = workloads.make(name)
    B, H, Hkv, L, d = wl.shape
    g = H // Hkv
    lens = wl.lengths()
    cfg_kw = dict(threads=threads)
    unit_digest = []
    qs, ks, vs, cis = [], [], [], []
    t0 = time.time()
    if wl.scale_granularity == "tensor":
        # compose the reference's primitives with global scales
        qg = ia.quantize_symmetric(wl.q.reshape(-1, d))
        kg = ia.quantize_symmetric(wl.k.reshape(-1, d))
        vg = ia.quantize_symmetric(wl.v.reshape(-1, d))
        qv = qg.values.reshape(wl.q.shape)
        kv = kg.values.reshape(wl.k.shape)
        vv = vg.values.reshape(wl.v.shape)
        lut = ia.build_lut(5, 6.6)
        ci = ia.compute_c_int(6.6, d, qg.scales[0], kg.scales[0])
        PT = ia.QuantGranularity.per_tensor()
        for bb in range(B):
            for h in range(H):
                qm = ia.QuantizedMatrix(qv[bb, h], qg.scales, PT)
                km = ia.QuantizedMatrix(kv[bb, h // g], kg.scales, PT)
                lm = ia.gemm_qk(qm, km)
                prob = ia.index_softmax(lm, ci, lut)
                acc = ia.gemm_pv(prob.values, vv[bb, h // g])
                o = acc.astype(np.float32) * np.float32(float(vg.scales[0]) / 255)
                unit_digest.append(digest(o))
        qs = [f32hex(qg.scales[0])]
        ks = [f32hex(kg.scales[0])]
        vs = [f32hex(vg.scales[0])]
        cis = [int(ci.c_int)]
    else:
        for bb in range(B):
            n = int(lens[bb])
            mask = np.triu(np.ones((n, n), dtype=bool), 1) if wl.causal else None
            for h in range(H):
                qq = wl.q[bb, h, :n]
                kk = wl.k[bb, h // g, :n]
                vv = wl.v[bb, h // g, :n]
                o, _ = ia.int_attention(qq, kk, vv, ia.AttentionConfig(mask=mask, **cfg_kw))
                unit_digest.append(digest(o))
                qs.append(f32hex(ia.quantize_symmetric(qq).scales[0]))
                sk = ia.quantize_symmetric(kk).scales[0]
                ks.append(f32hex(sk))
                vs.append(f32hex(ia.quantize_symmetric(vv).scales[0]))
                cis.append(int(ia.compute_c_int(6.6, d, np.float32(float.fromhex(qs[-1])), sk).c_int))
            print(f"  {name} b={bb} done ({time.time() - t0:.1f}s)", flush=True)
    return dict(name=name, shape=[B, H, Hkv, L, d], causal=wl.causal,
                scale_granularity=wl.scale_granularity,
                seq_lens=None if wl.seq_lens is None else [int(x) for x in wl.seq_lens],
                unit_digests=unit_digest, q_scales=qs, k_scales=ks, v_scales=vs,
                c_int=cis, ref_seconds=time.time() - t0, ref_threads=threads)


def grouped_cases():
    """Grouped-key IndexSoftmax straight from the reference: random int32 logits,
    contiguous and scattered column groups, masks, both P formats; plus the
    per-row-group-K int_attention pipeline end to end."""
    rng = np.random.default_rng(2511)
    out = {}
    lut = ref_sm.build_lut(5, 6.6)
    n_sm = 0
    for L, ng, contiguous, mask_kind, pf in [
            (64, 4, True, None, 255), (96, 3, False, None, 255), (80, 5, True, "causal", 255),
            (72, 2, False, "random", 127), (48, 1, True, None, 255), (128, 8, True, "causal", 127),
            (33, 6, False, "rowdead", 255)]:
        logits = rng.integers(-200000, 200000, size=(L, L)).astype(np.int32)
        if contiguous:
            groups = np.repeat(np.arange(ng), (L + ng - 1) // ng)[:L]
        else:
            groups = rng.integers(0, ng, size=L)
            groups[:ng] = np.arange(ng)
        alphas = (rng.uniform(0.2, 30.0, size=ng) / 1000.0).tolist()
        mask = None
        if mask_kind == "causal":
            mask = np.triu(np.ones((L, L), bool), 1)
        elif mask_kind == "random":
            mask = rng.random((L, L)) < 0.3
        elif mask_kind == "rowdead":
            mask = rng.random((L, L)) < 0.2
            mask[5, :] = True
        fmt = ref_sm.PFormat.UINT8X255 if pf == 255 else ref_sm.PFormat.INT8X127
        prob = ref_sm.index_softmax_grouped(ref_sm.np.asarray(logits), groups, alphas, 6.6, lut,
                                            mask=mask, p_format=fmt)
        key = f"sm{n_sm}"
        out[key + "_logits"] = logits
        out[key + "_groups"] = groups.astype(np.int32)
        out[key + "_alphas"] = np.array(alphas, np.float64)
        out[key + "_mask"] = np.zeros((0, 0), bool) if mask is None else mask
        out[key + "_pf"] = np.array(pf)
        out[key + "_prob"] = np.asarray(prob.values).view(np.uint8)
        n_sm += 1
    out["n_sm"] = np.array(n_sm)
    n_pipe = 0
    for L, d, gs, causal in [(96, 32, 32, False), (128, 64, 16, True), (70, 20, 7, False)]:
        q = rng.standard_normal((L, d), dtype=np.float32)
        k = rng.standard_normal((L, d), dtype=np.float32) * rng.uniform(0.5, 4.0, size=(L, 1)).astype(np.float32)
        v = rng.standard_normal((L, d), dtype=np.float32)
        mask = np.triu(np.ones((L, L), bool), 1) if causal else None
        cfg = ia.AttentionConfig(granularity=ia.QuantGranularity.per_row_group(gs), mask=mask)
        o, _ = ia.int_attention(q, k, v, cfg)
        key = f"pipe{n_pipe}"
        out[key + "_q"], out[key + "_k"], out[key + "_v"] = q, k, v
        out[key + "_gs"] = np.array(gs)
        out[key + "_causal"] = np.array(int(causal))
        out[key + "_out"] = np.asarray(o, np.float32)
        n_pipe += 1
    out["n_pipe"] = np.array(n_pipe)
    np.savez_compressed(os.path.join(GOLD, "grouped_cases.npz"), **out)


def quant_only_cases():
    """The paper's comparator from the reference: output and the requantised P^
    (its private _stable_softmax / _quantize_probs, pipeline.py:119-140)."""
    from intattn import pipeline as ref_pipe
    import math
    rng = np.random.default_rng(259)
    out = {}
    n = 0
    for L, d, mask_kind, pf in [(128, 64, None, 255), (300, 128, "causal", 255),
                                (77, 32, "dead", 255), (200, 64, "causal", 127),
                                (513, 128, None, 255)]:
        q = rng.standard_normal((L, d), dtype=np.float32)
        k = rng.standard_normal((L, d), dtype=np.float32)
        v = rng.standard_normal((L, d), dtype=np.float32)
        mask = None
        if mask_kind == "causal":
            mask = np.triu(np.ones((L, L), bool), 1)
        elif mask_kind == "dead":
            mask = rng.random((L, L)) < 0.25
            mask[3, :] = True
        fmt = ia.PFormat.UINT8X255 if pf == 255 else ia.PFormat.INT8X127
        o, _ = ia.quant_only_attention(q, k, v, ia.AttentionConfig(mask=mask, p_format=fmt))
        qh = ia.quantize_symmetric(q)
        kh = ia.quantize_symmetric(k)
        logits = ia.matmul_int8(qh.values, kh.values)
        alpha = np.float32(float(qh.scales[0]) * float(kh.scales[0]) / math.sqrt(d))
        phat = ref_pipe._quantize_probs(ref_pipe._stable_softmax(logits.astype(np.float32) * alpha, mask), fmt)
        key = f"qo{n}"
        out[key + "_q"], out[key + "_k"], out[key + "_v"] = q, k, v
        out[key + "_mask"] = np.zeros((0, 0), bool) if mask is None else mask
        out[key + "_pf"] = np.array(pf)
        out[key + "_out"] = np.asarray(o, np.float32)
        out[key + "_phat"] = np.asarray(phat).view(np.uint8)
        out[key + "_sv"] = np.array(float(ia.quantize_symmetric(v).scales[0]), np.float32)
        n += 1
    out["n"] = np.array(n)
    np.savez_compressed(os.path.join(GOLD, "quant_only_cases.npz"), **out)


def errors():
    """Exception class per error case, straight from the reference."""
    res = {name: run_error_case(fn, ia) for name, fn in error_cases().items()}
    with open(os.path.join(GOLD, "errors.json"), "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)


def audits():
    """dataflow_audit tag stream ((tag, dtype) per note) of each audited call."""
    res = {name: run_audit_case(fn, ia) for name, fn in audit_cases().items()}
    with open(os.path.join(GOLD, "audit.json"), "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C2h,C3,C4,C5")
    ap.add_argument("--skip-stages", action="store_true")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--grouped-only", action="store_true")
    ap.add_argument("--audit-only", action="store_true")
    a = ap.parse_args()
    os.makedirs(GOLD, exist_ok=True)
    audits()
    if a.audit_only:
        return
    grouped_cases()
    quant_only_cases()
    errors()
    if a.grouped_only:
        return
    with open(os.path.join(GOLD, "kats.json"), "w") as f:
        json.dump(kats(), f, indent=1)
    if not a.skip_stages:
        stage_cases()
    path = os.path.join(GOLD, "configs.json")
    allc = json.load(open(path)) if os.path.exists(path) else {}
    for name in [x for x in a.configs.split(",") if x]:
        t0 = time.time()
        if name == "C2h":
            orig = workloads.make_c2
            workloads.MAKERS["C2"] = lambda seed=0: orig(seed, scale_granularity="head")
            r = config_golden("C2", 1)
            workloads.MAKERS["C2"] = orig
            r["name"] = "C2h"
        else:
            r = config_golden(name, 1 if name in ("C1", "C2") else a.threads)
        allc[name] = r
        with open(path, "w") as f:
            json.dump(allc, f, indent=0)
        print(f"{name}: {len(r['unit_digests'])} units in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
