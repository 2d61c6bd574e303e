"""Seeded per-stage parity cases shared by oracle/gen_golden.py and the tests.

Each case regenerates identical f32 inputs from its parameters (numpy PCG64),
so the committed fixtures (tests/golden/stage_cases.json) hold only the case
parameters plus digests / scalars of the reference's per-stage outputs.
Edge cases follow SURVEY.md §4 / Appendix A: L = 1, L not a tile multiple,
all-zero heads (c_int = 2^52 clamp), planted +-0.5 ties, causal and random
masks with a fully masked row, both P formats, and the (b, c) range.
"""
from __future__ import annotations

import hashlib

import numpy as np


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


def case_list():
    cases = []
    rng = np.random.default_rng(12345)
    dims = [1, 3, 16, 64, 128]
    scales = [1e-3, 1.0, 50.0]
    masks = ["none", "none", "causal", "random"]
    for i in range(60):
        cases.append(dict(
            seed=1000 + i,
            L=int(rng.integers(1, 161)),
            d=int(dims[i % len(dims)]),
            scale=float(scales[(i // 5) % 3]),
            mask=masks[i % len(masks)],
            b=5, c=6.6, p=255, special="none"))
    # fixed shapes that hit tile edges of the GPU kernels
    for j, (L, d) in enumerate([(128, 64), (129, 64), (197, 64), (256, 128),
                                (255, 128), (300, 32), (64, 96), (200, 80)]):
        cases.append(dict(seed=2000 + j, L=L, d=d, scale=1.0,
                          mask=["none", "causal"][j % 2], b=5, c=6.6, p=255,
                          special="none"))
    for j, (b, c, p) in enumerate([(2, 6.6, 255), (3, 6.6, 255), (4, 6.6, 255),
                                   (6, 6.6, 255), (7, 6.6, 255), (8, 6.6, 255),
                                   (5, 4.4, 255), (5, 8.8, 255), (5, 6.6, 127),
                                   (4, 5.5, 127), (8, 7.7, 127)]):
        cases.append(dict(seed=3000 + j, L=96 + 7 * j, d=64, scale=1.0,
                          mask=["none", "causal", "random"][j % 3], b=b, c=c, p=p,
                          special="none"))
    for j, sp in enumerate(["zero_q", "zero_k", "zero_all", "ties", "ties",
                            "one_hot", "L1", "L1", "big_d", "masked_rows"]):
        cases.append(dict(seed=4000 + j, L=[40, 33, 17, 64, 128, 50, 1, 1, 32, 90][j],
                          d=[64, 16, 8, 32, 64, 128, 64, 1, 300, 64][j], scale=1.0,
                          mask=["none", "causal", "none", "none", "random", "none",
                                "none", "none", "causal", "random"][j],
                          b=5, c=6.6, p=[255, 255, 255, 255, 127, 255, 255, 255, 255, 255][j],
                          special=sp))
    return cases


def case_inputs(case):
    """(q, k, v, mask|None) f32 [L, d] for a case dict."""
    rng = np.random.default_rng(case["seed"])
    L, d = case["L"], case["d"]
    s = np.float32(case["scale"])
    q = rng.standard_normal((L, d), dtype=np.float32) * s
    k = rng.standard_normal((L, d), dtype=np.float32) * s
    v = rng.standard_normal((L, d), dtype=np.float32) * s
    sp = case["special"]
    if sp in ("zero_q", "zero_all"):
        q[:] = 0
    if sp in ("zero_k", "zero_all"):
        k[:] = 0
    if sp == "zero_all":
        v[:] = 0
    if sp == "ties":
        # amax = 127 -> scale = 1.0 exactly; plant halves so x/scale ties at .5
        for x in (q, k, v):
            x[:] = np.round(rng.uniform(-120, 120, size=x.shape)).astype(np.float32)
            x += np.where(rng.random(x.shape) < 0.5, np.float32(0.5), np.float32(-0.5))
            x.flat[0] = np.float32(127.0)
    if sp == "one_hot":
        q[:] = 0
        q[np.arange(L), np.arange(L) % d] = 3.0
    mask = None
    if case["mask"] == "causal":
        mask = np.triu(np.ones((L, L), dtype=bool), 1)
    elif case["mask"] == "random":
        mask = rng.random((L, L)) < 0.3
        if L > 2:
            mask[L // 2, :] = True       # one fully masked row
    if sp == "masked_rows" and L > 4:
        mask[::7, :] = True
    return q, k, v, mask


def error_cases():
    """Calls that the reference rejects (or accepts) -- the same lambda runs against the
    reference package (oracle/gen_golden.py records the exception class it raises into
    tests/golden/errors.json) and against this package (tests/test_gpu_errors.py).
    ``m`` is the package module."""
    f32 = np.float32
    z = lambda *s: np.zeros(s, f32)  # noqa: E731
    i8 = lambda *s: np.zeros(s, np.int8)  # noqa: E731
    i32 = lambda *s: np.zeros(s, np.int32)  # noqa: E731

    def lut(m):
        return m.build_lut(5, 6.6)

    return {
        "quantize_nan": lambda m: m.quantize_symmetric(np.array([[np.nan, 1.0]], f32)),
        "quantize_inf": lambda m: m.quantize_symmetric(np.array([[np.inf]], f32)),
        "quantize_ok": lambda m: m.quantize_symmetric(np.array([[1.0, -2.0]], f32)),
        "quantize_3d": lambda m: m.quantize_symmetric(z(2, 2, 2)),
        "matmul_not_int8": lambda m: m.matmul_int8(z(2, 2), i8(2, 2)),
        "matmul_k_mismatch": lambda m: m.matmul_int8(i8(2, 3), i8(2, 4)),
        "matmul_ok": lambda m: m.matmul_int8(i8(2, 3), i8(4, 3)),
        "gemm_qk_not_quantized": lambda m: m.gemm_qk(i8(2, 2), i8(2, 2)),
        "gemm_qk_row_groups": lambda m: m.gemm_qk(
            m.quantize_symmetric(np.ones((4, 2), f32)),
            m.quantize_symmetric(np.ones((4, 2), f32), m.QuantGranularity.per_row_group(2))),
        "gemm_pv_bad_p": lambda m: m.gemm_pv(i32(2, 2), i8(2, 3)),
        "gemm_pv_mismatch": lambda m: m.gemm_pv(np.zeros((2, 2), np.uint8), i8(3, 3)),
        "gemm_pv_not_square": lambda m: m.gemm_pv(np.zeros((2, 3), np.uint8), i8(3, 3)),
        "build_lut_b1": lambda m: m.build_lut(1, 6.6),
        "build_lut_b9": lambda m: m.build_lut(9, 6.6),
        "build_lut_c0": lambda m: m.build_lut(5, 0.0),
        "compute_c_int_bad_d": lambda m: m.compute_c_int(6.6, 0, 0.05, 0.04),
        "compute_c_int_bad_scale": lambda m: m.compute_c_int(6.6, 64, 0.0, 0.04),
        "softmax_not_square": lambda m: m.index_softmax(i32(2, 3), 10, lut(m)),
        "softmax_not_int32": lambda m: m.index_softmax(z(2, 2), 10, lut(m)),
        "softmax_c_zero": lambda m: m.index_softmax(i32(2, 2), 0, lut(m)),
        "softmax_lut_type": lambda m: m.index_softmax(i32(2, 2), 10, [255, 0]),
        "softmax_mask_shape": lambda m: m.index_softmax(i32(2, 2), 10, lut(m),
                                                        mask=np.zeros((3, 3), bool)),
        "softmax_ok": lambda m: m.index_softmax(np.array([[100, 40], [40, 100]], np.int32), 50,
                                                lut(m)),
        "grouped_groups_shape": lambda m: m.index_softmax_grouped(i32(3, 3), np.zeros(2, np.int64),
                                                                  [0.01], 6.6, lut(m)),
        "grouped_alpha_nonpositive": lambda m: m.index_softmax_grouped(
            i32(3, 3), np.zeros(3, np.int64), [0.0], 6.6, lut(m)),
        "grouped_group_out_of_range": lambda m: m.index_softmax_grouped(
            i32(3, 3), np.array([0, 1, 2]), [0.01, 0.02], 6.6, lut(m)),
        "grouped_no_alphas": lambda m: m.index_softmax_grouped(i32(3, 3), np.zeros(3, np.int64),
                                                               [], 6.6, lut(m)),
        "attention_shape_mismatch": lambda m: m.int_attention(z(4, 8), z(4, 8), z(5, 8)),
        "attention_1d": lambda m: m.int_attention(z(4), z(4), z(4)),
        "attention_mask_shape": lambda m: m.int_attention(z(4, 8), z(4, 8), z(4, 8),
                                                          m.AttentionConfig(mask=np.zeros((3, 3), bool))),
        "attention_col_groups": lambda m: m.int_attention(
            z(4, 8), z(4, 8), z(4, 8),
            m.AttentionConfig(granularity=m.QuantGranularity.per_col_group(4))),
        "attention_nan": lambda m: m.int_attention(np.full((4, 8), np.nan, f32), z(4, 8), z(4, 8)),
        "attention_ok": lambda m: m.int_attention(np.ones((4, 8), f32), np.ones((4, 8), f32),
                                                  np.ones((4, 8), f32)),
        "quant_only_shape_mismatch": lambda m: m.quant_only_attention(z(4, 8), z(4, 9), z(4, 8)),
        "quant_only_ok": lambda m: m.quant_only_attention(np.ones((4, 8), f32), np.ones((4, 8), f32),
                                                          np.ones((4, 8), f32)),
        "granularity_bad_group": lambda m: m.QuantGranularity.per_row_group(0),
        "dequantize_ok": lambda m: m.dequantize(m.quantize_symmetric(np.ones((2, 2), f32))),
    }


def run_error_case(fn, m):
    """Class name of the exception the call raises, or 'ok'."""
    try:
        fn(m)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__
    return "ok"


def audit_cases():
    """Calls whose ``dataflow_audit`` tag stream is pinned against the reference
    (softmax.py:207-228; notes at softmax.py:279-298, :394-398, pipeline.py:248).
    name -> fn(m) running the call on module ``m`` (the reference ``intattn`` or
    ``paper_2511_21513_b200``); the harness wraps it in ``m.dataflow_audit``."""
    rng = np.random.default_rng(777)
    L, d = 48, 32
    q, k, v = (rng.standard_normal((L, d), dtype=np.float32) for _ in range(3))
    causal = np.triu(np.ones((L, L), bool), 1)
    logits = rng.integers(-5000, 5000, size=(L, L), dtype=np.int32)

    def attn(**kw):
        def fn(m):
            cfg = m.AttentionConfig(**{key: (val(m) if callable(val) else val)
                                       for key, val in kw.items() if key not in ("warmup", "iters")})
            m.int_attention(q, k, v, cfg, warmup=kw.get("warmup", 0), iters=kw.get("iters", 1))
        return fn

    def isoft(mask=None, p127=False):
        def fn(m):
            fmt = m.PFormat.INT8X127 if p127 else m.PFormat.UINT8X255
            m.index_softmax(logits, m.ClipThreshold(c_int=4000), m.build_lut(5, 6.6), mask=mask,
                            p_format=fmt)
        return fn

    def grouped(m):
        groups = np.repeat(np.arange(3), L // 3)
        m.index_softmax_grouped(logits, groups, [0.002, 0.001, 0.004], 6.6, m.build_lut(5, 6.6),
                                mask=causal)

    def qonly(m):
        m.quant_only_attention(q, k, v)

    return {
        "int_attention": attn(),
        "int_attention_warmup1_iters2": attn(warmup=1, iters=2),
        "int_attention_causal_mask": attn(mask=causal),
        "int_attention_int8x127": attn(p_format=lambda m: m.PFormat.INT8X127),
        "int_attention_row_group_k": attn(granularity=lambda m: m.QuantGranularity.per_row_group(16)),
        "index_softmax": isoft(),
        "index_softmax_mask_int8x127": isoft(mask=causal, p127=True),
        "index_softmax_grouped": grouped,
        "quant_only_attention": qonly,
    }


def run_audit_case(fn, m):
    sink = []
    with m.dataflow_audit(sink):
        fn(m)
    return [[tag, np.dtype(dt).str] for tag, dt in sink]
