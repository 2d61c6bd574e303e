"""GPU parity: the CUDA path against the reference's golden vectors and the oracle.

Bit-exact is the bar for every integer/byte stage: quantised
Q/K/V and scales, int32 logits, u8 P^, int32 P.V and the f32 output bits.
Run on a B200 with ``pytest -m gpu``.
"""
import numpy as np
import pytest
import torch

import paper_2511_21513_b200 as ia
from paper_2511_21513_b200 import engine as E
from cases import case_inputs, digest
from golden_io import f32, stage_cases
from oracle import oracle as O

pytestmark = pytest.mark.gpu
CASES = stage_cases()


def _first_diff(a, b):
    a, b = np.asarray(a), np.asarray(b)
    bad = np.argwhere(a != b)
    if bad.size == 0:
        return "equal"
    i = tuple(bad[0])
    return f"{len(bad)} diffs, first at {i}: got {a[i]} want {b[i]}"


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_stage_case_fused(idx):
    """Fused kernel, single head, per-stage dumps vs the reference's digests."""
    row = CASES[idx]
    case = row["case"]
    q, k, v, mask = case_inputs(case)
    L, d = q.shape
    pf = ia.PFormat.UINT8X255 if case["p"] == 255 else ia.PFormat.INT8X127
    cfg = ia.AttentionConfig(b=case["b"], c=case["c"], p_format=pf)
    out, dbg = ia.int_attention_batched(q[None, None], k[None, None], v[None, None], mask=mask,
                                        cfg=cfg, debug=True)
    ref = O.int_attention(q, k, v, b=case["b"], c=case["c"], mask=mask, p_scale=case["p"])
    assert digest(ref) == row["digests"]["out"]  # oracle pinned to the reference
    if d <= 256:
        qh = dbg["qhat"][0, :, :d].cpu().numpy()
        assert digest(qh) == row["digests"]["qh"], _first_diff(qh, O.quantize_tensor(q)[0])
        assert dbg["q_scales"].cpu().numpy()[0] == f32(row["sq"])
        assert dbg["k_scales"].cpu().numpy()[0] == f32(row["sk"])
        assert dbg["v_scales"].cpu().numpy()[0] == f32(row["sv"])
        logits = dbg["logits"][0].cpu().numpy()
        want_logits = O.matmul_s8(O.quantize_tensor(q)[0], O.quantize_tensor(k)[0])
        if mask is None:
            assert digest(logits) == row["digests"]["logits"], _first_diff(logits, want_logits)
        else:  # the kernel only computes key tiles it needs (causal); compare where computed
            keep = ~np.triu(np.ones((L, L), bool), 1) if case["mask"] == "causal" else np.ones((L, L), bool)
            assert np.array_equal(logits[keep], want_logits[keep]), _first_diff(logits[keep], want_logits[keep])
        prob = dbg["prob"][0].cpu().numpy()
        want_p = O.index_softmax(want_logits, row["c_int"], np.array(row["lut"], np.uint8),
                                 mask=mask, p_scale=case["p"])
        assert digest(prob.view(np.int8) if case["p"] == 127 else prob) == row["digests"]["prob"], \
            _first_diff(prob, want_p)
        acc = dbg["acc"][0, :, :d].cpu().numpy()
        assert digest(acc) == row["digests"]["acc"], _first_diff(acc, O.gemm_pv(want_p, O.quantize_tensor(v)[0]))
    got = out[0, 0]
    assert digest(got) == row["digests"]["out"], _first_diff(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("idx", range(0, len(CASES), 3))
def test_stage_case_api(idx):
    """The drop-in stage operators, one by one, vs the reference digests."""
    row = CASES[idx]
    case = row["case"]
    q, k, v, mask = case_inputs(case)
    pf = ia.PFormat.UINT8X255 if case["p"] == 255 else ia.PFormat.INT8X127
    qh, kh, vh = ia.quantize_symmetric(q), ia.quantize_symmetric(k), ia.quantize_symmetric(v)
    assert digest(qh.values) == row["digests"]["qh"]
    assert digest(kh.values) == row["digests"]["kh"]
    assert digest(vh.values) == row["digests"]["vh"]
    assert qh.scales[0] == f32(row["sq"])
    lm = ia.gemm_qk(qh, kh)
    assert digest(lm.values) == row["digests"]["logits"]
    assert float(lm.alpha).hex() == row["alpha"]
    ci = ia.compute_c_int(case["c"], q.shape[1], qh.scales[0], kh.scales[0])
    assert ci.c_int == row["c_int"]
    lut = ia.build_lut(case["b"], case["c"])
    assert lut.entries.tolist() == row["lut"]
    prob = ia.index_softmax(lm, ci, lut, mask=mask, p_format=pf)
    assert digest(prob.values) == row["digests"]["prob"], _first_diff(
        prob.values, O.index_softmax(lm.values, ci.c_int, lut.entries, mask, case["p"]))
    acc = ia.gemm_pv(prob.values, vh)
    assert digest(acc) == row["digests"]["acc"]
    out, t = ia.int_attention(q, k, v, ia.AttentionConfig(b=case["b"], c=case["c"], p_format=pf,
                                                          mask=mask))
    assert digest(out) == row["digests"]["out"]
    assert t.total_ns > 0


def test_kats_gpu():
    q = ia.quantize_symmetric(np.array([[1.0, -2.0], [0.5, 2.54]], np.float32))
    assert q.values.tolist() == [[50, -100], [25, 127]]
    z = ia.quantize_symmetric(np.zeros((3, 4), np.float32))
    assert not z.values.any() and z.scales[0] == np.float32(np.float32(1e-12) / np.float32(127))
    a = ia.QuantizedMatrix(np.array([[1, 2]], np.int8), np.array([0.05], np.float32),
                           ia.QuantGranularity.per_tensor())
    b = ia.QuantizedMatrix(np.array([[3, 4]], np.int8), np.array([0.04], np.float32),
                           ia.QuantGranularity.per_tensor())
    assert ia.gemm_qk(a, b).values.tolist() == [[11]]
    assert ia.gemm_pv(np.array([[255]], np.uint8), np.array([[7, -3]], np.int8)).tolist() == [[1785, -765]]
    lut = ia.build_lut(5, 6.6)
    assert ia.index_softmax(np.array([[100, 100], [100, 100]], np.int32), 37335, lut).values.tolist() == [[128, 128], [128, 128]]
    assert ia.index_softmax(np.array([[100, 40], [40, 100]], np.int32), 50, lut).values.tolist() == [[255, 0], [0, 255]]
    assert ia.index_softmax(np.array([[7]], np.int32), 5, lut).values.tolist() == [[255]]
    m = np.array([[False, True], [True, True]])
    assert ia.index_softmax(np.array([[1, 2], [3, 4]], np.int32), 50, lut, mask=m).values.tolist() == [[255, 0], [0, 0]]
    p = ia.index_softmax(np.array([[100, 100], [100, 40]], np.int32), 50, lut,
                         p_format=ia.PFormat.INT8X127)
    assert p.values.dtype == np.int8 and p.values.tolist() == [[64, 64], [127, 0]]
    with pytest.raises(ValueError):
        ia.quantize_symmetric(np.array([[1.0, np.nan]], np.float32))
    with pytest.raises(ValueError):
        ia.int_attention(np.zeros((4, 3), np.float32), np.zeros((4, 3), np.float32),
                         np.array([[np.inf, 0, 0]] * 4, np.float32))


def test_gemm_random_shapes():
    """SPEC acceptance 1: integer GEMMs vs a 64-bit triple loop, random shapes."""
    rng = np.random.default_rng(7)
    for _ in range(40):
        m, n, kd = (int(x) for x in rng.integers(1, 300, size=3))
        a = rng.integers(-127, 128, size=(m, kd)).astype(np.int8)
        b = rng.integers(-127, 128, size=(n, kd)).astype(np.int8)
        assert np.array_equal(ia.matmul_int8(a, b), a.astype(np.int64) @ b.astype(np.int64).T)
        p = rng.integers(0, 256, size=(m, m)).astype(np.uint8)
        vv = rng.integers(-127, 128, size=(m, kd)).astype(np.int8)
        assert np.array_equal(ia.gemm_pv(p, vv), p.astype(np.int64) @ vv.astype(np.int64))


def test_granularities():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 48), dtype=np.float32)
    for g in (ia.QuantGranularity.per_row_group(16), ia.QuantGranularity.per_col_group(12)):
        got = ia.quantize_symmetric(x, g)
        if g.kind == "per_row_group":
            want_v, want_s = O.quantize_groups(x, 4)
        else:
            xt = np.ascontiguousarray(x.reshape(64, 4, 12).transpose(1, 0, 2))
            vv, want_s = O.quantize_groups(xt, 4)
            want_v = vv.transpose(1, 0, 2).reshape(64, 48)
        assert np.array_equal(got.values, want_v) and np.array_equal(got.scales, want_s)
        deq = ia.dequantize(got)
        assert np.array_equal(deq, (got.values.astype(np.float32) * got.scale_grid()).astype(np.float32))


@pytest.mark.parametrize("L,d,causal,lens,H,Hkv,gran", [
    (300, 64, True, None, 4, 2, "head"),
    (517, 128, True, [517, 300, 129, 1], 2, 2, "head"),
    (640, 128, False, None, 2, 1, "tensor"),
    (257, 32, True, [257, 1], 3, 3, "head"),
    (384, 256, True, None, 2, 2, "head"),
    (130, 80, False, [100, 130], 2, 2, "tensor"),
    (200, 300, True, None, 2, 1, "head"),
])
def test_batched_vs_oracle(L, d, causal, lens, H, Hkv, gran):
    B = 1 if lens is None else len(lens)
    rng = np.random.default_rng(L + d)
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, Hkv, L, d), dtype=np.float32) * np.float32(2.0)
    v = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    sl = None if lens is None else np.array(lens, np.int32)
    if sl is not None:
        for b, n in enumerate(sl):
            q[b, :, n:] = 0
            k[b, :, n:] = 0
            v[b, :, n:] = 0
    got = ia.int_attention_batched(q, k, v, causal=causal, seq_lens=sl, scale_granularity=gran)
    want, _ = O.attention_batched(q, k, v, causal=causal, seq_lens=sl, scale_granularity=gran)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), _first_diff(got, want)


def test_dense_mask_batched():
    rng = np.random.default_rng(11)
    L, d = 333, 64
    q = rng.standard_normal((2, 2, L, d), dtype=np.float32)
    k = rng.standard_normal((2, 2, L, d), dtype=np.float32)
    v = rng.standard_normal((2, 2, L, d), dtype=np.float32)
    mask = rng.random((L, L)) < 0.5
    mask[5, :] = True
    got = ia.int_attention_batched(q, k, v, mask=mask, causal=True)
    want, _ = O.attention_batched(q, k, v, mask=mask, causal=True)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), _first_diff(got, want)
    assert not got[:, :, 5].any()


def test_torch_inputs_stay_on_device():
    rng = np.random.default_rng(5)
    q = rng.standard_normal((1, 2, 256, 64), dtype=np.float32)
    qt = torch.from_numpy(q).cuda()
    out = ia.int_attention_batched(qt, qt, qt, causal=True)
    assert out.is_cuda
    want, _ = O.attention_batched(q, q, q, causal=True)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_sharded_single_rank_gpu_tensor_scales():
    """Sharding launcher on one GPU: precomputed (all-reduced) global scales path."""
    from paper_2511_21513_b200 import sharding
    rng = np.random.default_rng(21)
    q = rng.standard_normal((3, 4, 150, 64), dtype=np.float32)
    k = rng.standard_normal((3, 2, 150, 64), dtype=np.float32)
    v = rng.standard_normal((3, 2, 150, 64), dtype=np.float32)
    out, _ = sharding.sharded_attention(q, k, v, causal=True, scale_granularity="tensor")
    want, _ = O.attention_batched(q, k, v, causal=True, scale_granularity="tensor")
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32)), _first_diff(out, want)


@pytest.mark.parametrize("B,H,Hkv,L,d,lens,d_pad", [
    (1, 1, 1, 128, 64, None, None), (2, 4, 2, 333, 128, [333, 100], None), (1, 2, 1, 77, 20, None, None),
    (3, 2, 2, 1000, 64, [1000, 0, 513], None), (1, 8, 2, 4100, 128, None, None),
    (1, 1, 1, 64, 256, None, None), (1, 2, 2, 200, 36, [150], None),
    # explicit d_pad: every V^T block width (kb = 16 * 512 / d_pad rounded to 16)
    (1, 2, 1, 300, 40, None, 48), (2, 2, 2, 129, 16, [129, 7], 16), (1, 2, 2, 100, 80, None, 80),
    (1, 1, 1, 257, 200, [250], 208), (1, 2, 1, 500, 128, [499], 144), (1, 1, 1, 33, 160, None, 176)])
def test_quant_heads_matches_split(B, H, Hkv, L, d, lens, d_pad):
    """ia_quant_heads (one launch, team barriers) is bit-identical to the split
    amax + quantise kernels: Q^, K^, V^T (incl. padding) and every scale."""
    rng = np.random.default_rng(B * 1000 + L + d)
    dev = torch.device("cuda", 0)
    q = torch.from_numpy(rng.standard_normal((B, H, L, d), dtype=np.float32) * 3).to(dev)
    k = torch.from_numpy(rng.standard_normal((B, Hkv, L, d), dtype=np.float32)).to(dev)
    v = torch.from_numpy(rng.standard_normal((B, Hkv, L, d), dtype=np.float32) * 0.1).to(dev)
    sl = None
    if lens is not None:
        lens = (lens * B)[:B]
        sl = torch.tensor(lens, dtype=torch.int32, device=dev)
    a = E.prepare(q, k, v, seq_lens=sl, quant="fused", d_pad=d_pad)
    b = E.prepare(q, k, v, seq_lens=sl, quant="split", d_pad=d_pad)
    for x, y, nm in [(a.qhat, b.qhat, "qhat"), (a.khat, b.khat, "khat"), (a.vt, b.vt, "vt"),
                     (a.q_scales, b.q_scales, "sq"), (a.k_scales, b.k_scales, "sk"),
                     (a.v_scales, b.v_scales, "sv"),
                     (a.params[:, :52], b.params[:, :52], "params")]:  # 52 = defined bytes
        assert torch.equal(x, y), (nm, _first_diff(x.cpu().numpy(), y.cpu().numpy()))
    assert int(a.err.item()) == 0


@pytest.mark.parametrize("B,H,Hkv,L,d,lens,zero_v", [
    (64, 12, 12, 197, 64, None, False), (2, 4, 2, 333, 128, [333, 100], False),
    (1, 2, 1, 77, 20, None, True), (3, 2, 2, 1000, 64, [1000, 0, 513], False),
    (1, 8, 2, 4100, 128, None, False), (1, 2, 2, 200, 36, [150], False)])
def test_quant_tensors_matches_split(B, H, Hkv, L, d, lens, zero_v):
    """ia_quant_tensors (per-tensor scales: amax launch + quantise launch) is
    bit-identical to the split amax + quantise kernels with one slot per tensor."""
    rng = np.random.default_rng(7 * B + L + d)
    dev = torch.device("cuda", 0)
    q = torch.from_numpy(rng.standard_normal((B, H, L, d), dtype=np.float32) * 3).to(dev)
    k = torch.from_numpy(rng.standard_normal((B, Hkv, L, d), dtype=np.float32)).to(dev)
    v = torch.from_numpy(rng.standard_normal((B, Hkv, L, d), dtype=np.float32) * 0.1).to(dev)
    q[..., ::17] *= 8.0  # outlier channels
    if zero_v:
        v.zero_()
    sl = None
    if lens is not None:
        sl = torch.tensor((lens * B)[:B], dtype=torch.int32, device=dev)
    a = E.prepare(q, k, v, seq_lens=sl, scale_granularity="tensor", quant="fused")
    b = E.prepare(q, k, v, seq_lens=sl, scale_granularity="tensor", quant="split")
    for x, y, nm in [(a.qhat, b.qhat, "qhat"), (a.khat, b.khat, "khat"), (a.vt, b.vt, "vt"),
                     (a.q_scales, b.q_scales, "sq"), (a.k_scales, b.k_scales, "sk"),
                     (a.v_scales, b.v_scales, "sv"),
                     (a.params[:, :52], b.params[:, :52], "params")]:
        assert torch.equal(x, y), (nm, _first_diff(x.cpu().numpy(), y.cpu().numpy()))
    assert int(a.err.item()) == 0
    k[0, -1, 3, 1] = float("inf")
    assert int(E.prepare(q, k, v, scale_granularity="tensor").err.item()) == 1


def test_quant_heads_nonfinite():
    dev = torch.device("cuda", 0)
    q = torch.randn(1, 2, 256, 64, device=dev)
    k = torch.randn(1, 2, 256, 64, device=dev)
    v = torch.randn(1, 2, 256, 64, device=dev)
    k[0, 1, 17, 3] = float("nan")
    assert int(E.prepare(q, k, v).err.item()) == 1
    with pytest.raises(ValueError):
        ia.int_attention_batched(q, k, v)


def _grouped_gold():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "grouped_cases.npz"))


def test_grouped_softmax_kernel_golden():
    """ia_index_softmax_grouped vs the reference's own index_softmax_grouped outputs."""
    G = _grouped_gold()
    lut = ia.build_lut(5, 6.6)
    for i in range(int(G["n_sm"])):
        key = f"sm{i}"
        mask = G[key + "_mask"]
        mask = None if mask.size == 0 else mask
        pf = ia.PFormat.UINT8X255 if int(G[key + "_pf"]) == 255 else ia.PFormat.INT8X127
        got = ia.index_softmax_grouped(G[key + "_logits"], G[key + "_groups"],
                                       list(G[key + "_alphas"]), 6.6, lut, mask=mask, p_format=pf)
        assert np.array_equal(np.asarray(got.values).view(np.uint8), G[key + "_prob"]), key


@pytest.mark.parametrize("L,ng,masked", [(300, 7, False), (1024, 16, True), (2000, 1, True),
                                         (517, 600, False)])
def test_grouped_softmax_kernel_random(L, ng, masked):
    """Grouped kernel vs the oracle restatement on larger seeded cases (incl. many
    tiny groups and a single group, which must equal plain index_softmax)."""
    rng = np.random.default_rng(L + ng)
    logits = rng.integers(-2_000_000, 2_000_000, size=(L, L)).astype(np.int32)
    groups = rng.integers(0, ng, size=L).astype(np.int32)
    alphas = list(rng.uniform(1e-5, 5e-2, size=ng))
    mask = np.triu(np.ones((L, L), bool), 1) if masked else None
    lut = ia.build_lut(5, 6.6)
    got = np.asarray(ia.index_softmax_grouped(logits, groups, alphas, 6.6, lut, mask=mask).values)
    cis = [O.c_int_from_alpha(6.6, a) for a in alphas]
    want = O.index_softmax_grouped(logits, groups, cis, lut.entries, mask)
    assert np.array_equal(got, want), _first_diff(got, want)
    if ng == 1:
        plain = np.asarray(ia.index_softmax(logits, cis[0], lut, mask=mask).values)
        assert np.array_equal(got, plain)


def test_grouped_pipeline_golden():
    """Per-row-group K int_attention (pipeline.py:229-246) end to end vs the reference."""
    G = _grouped_gold()
    for i in range(int(G["n_pipe"])):
        key = f"pipe{i}"
        L = G[key + "_q"].shape[0]
        mask = np.triu(np.ones((L, L), bool), 1) if int(G[key + "_causal"]) else None
        cfg = ia.AttentionConfig(granularity=ia.QuantGranularity.per_row_group(int(G[key + "_gs"])),
                                 mask=mask)
        out, _ = ia.int_attention(G[key + "_q"], G[key + "_k"], G[key + "_v"], cfg)
        assert np.array_equal(np.asarray(out).view(np.uint32), G[key + "_out"].view(np.uint32)), key


def _qo_gold():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "quant_only_cases.npz"))


@pytest.mark.parametrize("i", range(5))
def test_quant_only_fused_vs_reference(i):
    """Fused quant-only mode (IA_SOFTMAX_FLOAT) vs the reference's quant_only_attention.

    Tolerance (float comparator, MUFU exp2 vs numpy f32 exp): every requantised P^
    within 1 of the reference's and at most 1% of entries off; each output element
    within n_i * 127 * s_v / denom of the reference, n_i = the row's P^ mismatches
    (a P^ unit moves one output by at most |v^| <= 127 grid steps)."""
    G = _qo_gold()
    key = f"qo{i}"
    q, k, v = G[key + "_q"], G[key + "_k"], G[key + "_v"]
    mask = G[key + "_mask"]
    mask = None if mask.size == 0 else mask
    pfv = int(G[key + "_pf"])
    cfg = ia.AttentionConfig(p_format=ia.PFormat.UINT8X255 if pfv == 255 else ia.PFormat.INT8X127)
    out, dbg = ia.quant_only_attention_batched(q[None, None], k[None, None], v[None, None],
                                               mask=mask, cfg=cfg, debug=True)
    L = q.shape[0]
    ph = dbg["prob"][0].cpu().numpy().astype(np.int32)
    want = G[key + "_phat"].astype(np.int32)
    diff = np.abs(ph - want)
    assert diff.max() <= 1, f"P^ off by {diff.max()}"
    assert (diff > 0).mean() <= 0.01, f"{(diff > 0).mean():.4f} of P^ entries differ"
    n_i = (diff > 0).sum(axis=1)
    bound = n_i[:, None] * 127.0 * float(G[key + "_sv"]) / pfv + 1e-6
    err = np.abs(out[0, 0] - G[key + "_out"])
    assert (err <= bound).all(), float((err - bound).max())
    # the single-head API takes the same fused path
    o1, _ = ia.quant_only_attention(q, k, v, ia.AttentionConfig(mask=mask, p_format=cfg.p_format))
    assert np.array_equal(o1.view(np.uint32), out[0, 0].view(np.uint32))
    if mask is not None and mask.all(axis=1).any():
        assert not out[0, 0][mask.all(axis=1)].view(np.uint32).any()  # fully masked rows -> +0.0


def test_quant_only_fused_batched_gqa_causal():
    """Batched GQA / varlen quant-only mode: each unit equals its single-head run."""
    rng = np.random.default_rng(5)
    B, H, Hkv, L, d = 2, 4, 2, 700, 64
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    v = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    lens = np.array([700, 450], np.int32)
    out = ia.quant_only_attention_batched(q, k, v, causal=True, seq_lens=lens)
    for b in range(B):
        n = int(lens[b])
        for h in range(H):
            o1, _ = ia.quant_only_attention(q[b, h, :n], k[b, h // 2, :n], v[b, h // 2, :n],
                                            ia.AttentionConfig(mask=np.triu(np.ones((n, n), bool), 1)))
            assert np.array_equal(out[b, h, :n].view(np.uint32), o1.view(np.uint32)), (b, h)
            assert not out[b, h, n:].view(np.uint32).any()


def _fuzz_case(i):
    """Seeded random batched problem: shapes, GQA ratio, masks, lengths, LUT bits, clip
    bound, P format, scale granularity, input magnitudes and outlier channels."""
    rng = np.random.default_rng(10_000 + i)
    B = int(rng.integers(1, 4))
    Hkv = int(rng.integers(1, 4))
    H = Hkv * int(rng.choice([1, 2, 4]))
    L = int(rng.integers(1, 700))
    d = int(rng.choice([int(rng.integers(1, 257)), 32, 64, 128, 256, int(rng.integers(257, 301))],
                       p=[0.4, 0.1, 0.15, 0.15, 0.1, 0.1]))
    causal = bool(rng.integers(0, 2))
    lens = None
    if rng.random() < 0.5:
        lens = rng.integers(0, L + 1, size=B).astype(np.int32)
        lens[0] = L if rng.random() < 0.5 else lens[0]
    gran = "tensor" if rng.random() < 0.3 else "head"
    cfg = ia.AttentionConfig(b=int(rng.choice([3, 4, 5, 6])), c=float(rng.choice([4.4, 6.6, 8.8])),
                             p_format=ia.PFormat.INT8X127 if rng.random() < 0.3 else ia.PFormat.UINT8X255)
    mags = [np.float32(10.0 ** rng.uniform(-2, 2)) for _ in range(3)]
    q = rng.standard_normal((B, H, L, d), dtype=np.float32) * mags[0]
    k = rng.standard_normal((B, Hkv, L, d), dtype=np.float32) * mags[1]
    v = rng.standard_normal((B, Hkv, L, d), dtype=np.float32) * mags[2]
    if rng.random() < 0.3:  # outlier channels
        ch = rng.choice(d, size=max(1, d // 50), replace=False)
        q[..., ch] *= np.float32(10.0)
        k[..., ch] *= np.float32(10.0)
    if lens is not None:
        for b, n in enumerate(lens):
            q[b, :, n:] = 0
            k[b, :, n:] = 0
            v[b, :, n:] = 0
    return q, k, v, causal, lens, gran, cfg, bool(rng.integers(0, 2))


@pytest.mark.parametrize("i", range(120))
def test_fuzz_batched_vs_oracle(i):
    """120 seeded random problems through int_attention_batched (host pipeline or
    device tensors; fused kernel or, for d > 256, the stage kernels), bit-exact
    against the oracle, which is itself pinned to the live reference."""
    q, k, v, causal, lens, gran, cfg, on_device = _fuzz_case(i)
    args = (q, k, v)
    if on_device:
        args = tuple(torch.from_numpy(x).cuda() for x in args)
    got = ia.int_attention_batched(*args, causal=causal, seq_lens=lens, scale_granularity=gran,
                                   cfg=cfg)
    if on_device:
        got = got.cpu().numpy()
    want, _ = O.attention_batched(q, k, v, causal=causal, seq_lens=lens, scale_granularity=gran,
                                  b=cfg.b, c=cfg.c, p_scale=cfg.p_format.value)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), \
        (q.shape, k.shape, causal, lens, gran, cfg, _first_diff(got, want))


def test_max_sequence_length():
    """L = MAX_SEQ_LEN (65536, gemm.py:26): the fused kernel's 512 key tiles, ring
    phases and index maps at the limit, bit-exact vs the oracle on a row sample;
    one more key is rejected as the reference rejects it."""
    L, d = 65536, 64
    rng = np.random.default_rng(65536)
    q = rng.standard_normal((1, 1, L, d), dtype=np.float32)
    k = rng.standard_normal((1, 1, L, d), dtype=np.float32)
    v = rng.standard_normal((1, 1, L, d), dtype=np.float32)
    got = ia.int_attention_batched(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                                   torch.from_numpy(v).cuda(), causal=True).cpu().numpy()
    stride = 97
    want, _ = O.attention_batched(q, k, v, causal=True, row_stride=stride)
    rows = np.arange(0, L, stride)
    assert np.array_equal(got[0, 0, rows].view(np.uint32), want[0, 0, rows].view(np.uint32))
    with pytest.raises(ValueError):
        ia.int_attention_batched(np.zeros((1, 1, L + 1, 8), np.float32),
                                 np.zeros((1, 1, L + 1, 8), np.float32),
                                 np.zeros((1, 1, L + 1, 8), np.float32))


def test_single_row_and_single_key():
    """L = 1 (one query, one key): P^ = 255 on the only key, out = v^ * s_v."""
    rng = np.random.default_rng(1)
    for d in (1, 7, 128):
        q = rng.standard_normal((1, 1), dtype=np.float32).repeat(d, 1)
        k = rng.standard_normal((1, d), dtype=np.float32)
        v = rng.standard_normal((1, d), dtype=np.float32)
        out, _ = ia.int_attention(q, k, v)
        want = O.int_attention(q, k, v)
        assert np.array_equal(out.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("i", range(24))
def test_fuzz_quant_only_vs_oracle(i):
    """Quant-only mode on seeded random single-head problems (shapes, masks, P formats,
    magnitudes) against the f32 numpy restatement of the reference's comparator
    (oracle.quant_only_attention, pinned bit-exact to the reference's fixtures), with
    the tolerance of test_quant_only_fused_vs_reference."""
    rng = np.random.default_rng(20_000 + i)
    L = int(rng.integers(1, 600))
    d = int(rng.choice([8, 32, 64, 100, 128, 256]))
    mags = [np.float32(10.0 ** rng.uniform(-1.5, 1.5)) for _ in range(3)]
    q, k, v = (rng.standard_normal((L, d), dtype=np.float32) * m for m in mags)
    kind = int(rng.integers(0, 3))
    mask = None if kind == 0 else (np.triu(np.ones((L, L), bool), 1) if kind == 1
                                   else rng.random((L, L)) < 0.3)
    pfv = 127 if rng.random() < 0.3 else 255
    cfg = ia.AttentionConfig(p_format=ia.PFormat.INT8X127 if pfv == 127 else ia.PFormat.UINT8X255)
    out, dbg = ia.quant_only_attention_batched(q[None, None], k[None, None], v[None, None],
                                               mask=mask, cfg=cfg, debug=True)
    want_out, want_p = O.quant_only_attention(q, k, v, mask, pfv)
    ph = dbg["prob"][0].cpu().numpy().astype(np.int32)
    diff = np.abs(ph - want_p.astype(np.int32))
    assert diff.max() <= 1 and (diff > 0).mean() <= 0.01, (L, d, kind, pfv, diff.max(), (diff > 0).mean())
    sv = float(O.quantize_tensor(v)[1])
    bound = (diff > 0).sum(axis=1)[:, None] * 127.0 * sv / pfv + 1e-6
    assert (np.abs(out[0, 0] - want_out) <= bound).all()


def test_quant_heads_rounding_boundaries():
    """Values placed on and one ulp either side of every x.5 quotient boundary (and the
    127.5 clip) for several head scales: the one-launch quantiser's reciprocal fast path
    must fall back to the IEEE quotient exactly where it matters."""
    rng = np.random.default_rng(99)
    H, L, d = 4, 512, 128
    q = np.zeros((1, H, L, d), np.float32)
    for h in range(H):
        amax = np.float32(10.0 ** rng.uniform(-3, 3))
        s = np.float32(max(amax, np.float32(1e-12)) / np.float32(127))
        ks = np.arange(-127, 128, dtype=np.float32)
        base = (ks + np.float32(0.5)) * s
        vals = np.concatenate([base, np.nextafter(base, np.float32(np.inf)),
                               np.nextafter(base, np.float32(-np.inf)), ks * s,
                               rng.uniform(-1, 1, L * d).astype(np.float32) * amax])
        vals = np.clip(vals, -amax, amax)[:L * d]
        vals[0] = amax
        q[0, h] = vals.reshape(L, d)
    dev = torch.device("cuda", 0)
    qt = torch.from_numpy(q).to(dev)
    kt = qt[:, :2].contiguous()
    a = E.prepare(qt, kt, kt, quant="fused")
    b = E.prepare(qt, kt, kt, quant="split")
    for x, y, nm in [(a.qhat, b.qhat, "qhat"), (a.khat, b.khat, "khat"), (a.vt, b.vt, "vt")]:
        assert torch.equal(x, y), (nm, _first_diff(x.cpu().numpy(), y.cpu().numpy()))
    for h in range(H):
        qq, _ = O.quantize_tensor(q[0, h])
        assert np.array_equal(a.qhat[h, :, :d].cpu().numpy(), qq), h


def test_host_pipeline_graph_replay():
    """Pinned host in / out: call 1 runs eagerly, call 2 captures the call into a CUDA
    graph and replays it, later calls replay.  Every call is bit-exact with the device
    path, including after the pinned inputs are overwritten in place (the graph reads
    the buffers at replay time) and with a non-finite input (flag still raised)."""
    from paper_2511_21513_b200 import batched
    rng = np.random.default_rng(77)
    B, H, Hkv, L, d = 2, 4, 2, 300, 64
    lens = np.array([300, 171])
    qh = torch.from_numpy(rng.standard_normal((B, H, L, d), dtype=np.float32)).pin_memory()
    kh = torch.from_numpy(rng.standard_normal((B, Hkv, L, d), dtype=np.float32)).pin_memory()
    vh = torch.from_numpy(rng.standard_normal((B, Hkv, L, d), dtype=np.float32)).pin_memory()
    oh = torch.empty((B, H, L, d), dtype=torch.float32).pin_memory()

    def want():
        return ia.int_attention_batched(qh.cuda(), kh.cuda(), vh.cuda(), causal=True,
                                        seq_lens=lens).cpu().numpy()

    n0 = len(batched._GRAPHS)
    for it in range(4):
        if it == 3:  # new data in the same pinned buffers
            qh.copy_(torch.from_numpy(rng.standard_normal((B, H, L, d), dtype=np.float32)))
        got = ia.int_attention_batched(qh, kh, vh, causal=True, seq_lens=lens, out=oh)
        assert got.data_ptr() == oh.data_ptr()
        w = want()
        assert np.array_equal(got.numpy().view(np.uint32), w.view(np.uint32)), it
    assert len(batched._GRAPHS) == min(n0 + 1, batched._GRAPH_CACHE) or not batched._GRAPH_ON
    kh[1, 0, 5, 3] = float("nan")
    for _ in range(2):
        with pytest.raises(ValueError):
            ia.int_attention_batched(qh, kh, vh, causal=True, seq_lens=lens, out=oh)


def test_host_pipeline_graph_refused_falls_back():
    """Head dim > 256 takes the unfused path, whose host reads cannot be captured: the
    capture is refused once and every call stays on the eager path, bit-exact."""
    from paper_2511_21513_b200 import batched
    rng = np.random.default_rng(78)
    B, H, Hkv, L, d = 2, 2, 2, 40, 260
    qh, kh, vh = (torch.from_numpy(rng.standard_normal((B, h, L, d), dtype=np.float32)).pin_memory()
                  for h in (H, Hkv, Hkv))
    oh = torch.empty((B, H, L, d), dtype=torch.float32).pin_memory()
    w = ia.int_attention_batched(qh.cuda(), kh.cuda(), vh.cuda()).cpu().numpy()
    for _ in range(3):
        got = ia.int_attention_batched(qh, kh, vh, out=oh)
        assert np.array_equal(got.numpy().view(np.uint32), w.view(np.uint32))
    assert not any(k[1] == qh.data_ptr() for k in batched._GRAPHS)
