"""Pin the CPU oracle (oracle/intattn_oracle.c) to the reference's own outputs.

The vectors were produced by importing the reference in the build container
(oracle/gen_golden.py); nothing here reads /root/reference at run time.
"""
import os

import numpy as np
import pytest

from cases import case_inputs, digest
from golden_io import configs, f32, kats, stage_cases, stage_small
from oracle import oracle as O
from paper_2511_21513_b200 import workloads


def test_kat_quantize():
    K = kats()
    v, s = O.quantize_tensor(np.array([[1.0, -2.0], [0.5, 2.54]], np.float32))
    assert s == f32(K["quant_example"]["scale"])
    assert v.tolist() == K["quant_example"]["values"] == [[50, -100], [25, 127]]
    v, s = O.quantize_tensor(np.zeros((3, 4), np.float32))
    assert s == f32(K["quant_zero"]["scale"]) and not v.any()
    s1 = np.float32(0.01)
    v, _ = O.quantize_tensor(np.array([[127 * s1, -127 * s1]], np.float32))
    assert v.tolist() == K["quant_endpoints"]["values"] == [[127, -127]]
    with pytest.raises(ValueError):
        O.quantize_tensor(np.array([[1.0, np.inf]], np.float32))


def test_kat_gemms_cint_lut():
    K = kats()
    assert O.matmul_s8(np.array([[1, 2]], np.int8), np.array([[3, 4]], np.int8)).tolist() == K["gemm_qk"]["values"]
    assert O.gemm_pv(np.array([[255]], np.uint8), np.array([[7, -3]], np.int8)).tolist() == K["gemm_pv"]["values"]
    for key, want in K["c_int"].items():
        c, d, sq, sk = key.split(",")
        assert O.c_int(float(c), int(d), np.float32(float(sq)), np.float32(float(sk))) == want
    assert K["c_int"]["6.6,128,0.05,0.04"] == 37335
    for key, want in K["lut"].items():
        b, c = key.split(",")
        assert O.build_lut(int(b), float(c)).tolist() == want
    assert O.index_table(50, 32).tolist() == K["index_table_50_32"]


def test_kat_index_softmax():
    K = kats()["index_softmax"]
    lut = O.build_lut(5, 6.6)
    assert O.index_softmax(np.array([[100, 100], [100, 100]]), 37335, lut).tolist() == K["uniform"] == [[128, 128], [128, 128]]
    assert O.index_softmax(np.array([[100, 40], [40, 100]]), 50, lut).tolist() == K["clip50"] == [[255, 0], [0, 255]]
    assert O.index_softmax(np.array([[7]]), 5, lut).tolist() == K["single"] == [[255]]
    m = np.array([[False, True], [True, True]])
    assert O.index_softmax(np.array([[1, 2], [3, 4]]), 50, lut, mask=m).tolist() == K["masked"] == [[255, 0], [0, 0]]
    got = O.index_softmax(np.array([[100, 100], [100, 40]]), 50, lut, p_scale=127).view(np.int8)
    assert got.tolist() == K["int8x127"] == [[64, 64], [127, 0]]


def _oracle_stages(q, k, v, mask, b, c, p):
    qh, sq = O.quantize_tensor(q)
    kh, sk = O.quantize_tensor(k)
    vh, sv = O.quantize_tensor(v)
    logits = O.matmul_s8(qh, kh)
    ci = O.c_int(c, q.shape[1], sq, sk)
    lut = O.build_lut(b, c)
    prob = O.index_softmax(logits, ci, lut, mask=mask, p_scale=p)
    if p == 127:
        prob = prob.view(np.int8)
    acc = O.gemm_pv(prob, vh)
    out = acc.astype(np.float32) * np.float32(float(sv) / p)
    return dict(qh=qh, kh=kh, vh=vh, sq=sq, sk=sk, sv=sv, logits=logits, c_int=ci,
                lut=lut, prob=prob, acc=acc, out=out)


@pytest.mark.parametrize("idx", range(len(stage_cases())))
def test_stage_case(idx):
    row = stage_cases()[idx]
    case = row["case"]
    q, k, v, mask = case_inputs(case)
    r = _oracle_stages(q, k, v, mask, case["b"], case["c"], case["p"])
    assert r["sq"] == f32(row["sq"]) and r["sk"] == f32(row["sk"]) and r["sv"] == f32(row["sv"])
    assert r["c_int"] == row["c_int"]
    assert r["lut"].tolist() == row["lut"]
    for n, want in row["digests"].items():
        assert digest(r[n]) == want, f"stage {n} differs in case {case}"
    # the batched oracle on the same single head must agree with the stages
    out, info = O.attention_batched(q[None, None], k[None, None], v[None, None], mask=mask,
                                    b=case["b"], c=case["c"], p_scale=case["p"])
    assert digest(out[0, 0]) == row["digests"]["out"]
    assert info["c_int"][0] == row["c_int"]


def test_stage_small_arrays():
    small = stage_small()
    rows = stage_cases()
    seen = 0
    for key in small:
        i, name = key.split("_", 1)
        row = rows[int(i)]
        assert digest(small[key]) == row["digests"][name]
        seen += 1
    assert seen > 0


def _check_config(name, row_stride=1):
    G = configs()[name]
    wl = workloads.make("C2" if name == "C2h" else name)
    gran = "head" if name == "C2h" else wl.scale_granularity
    out, info = O.attention_batched(wl.q, wl.k, wl.v, causal=wl.causal, seq_lens=wl.seq_lens,
                                    scale_granularity=gran, row_stride=row_stride)
    B, H, Hkv, L, d = wl.shape
    lens = wl.lengths()
    if gran == "tensor":
        assert info["q_scales"][0] == f32(G["q_scales"][0])
        assert info["k_scales"][0] == f32(G["k_scales"][0])
        assert info["v_scales"][0] == f32(G["v_scales"][0])
        assert int(info["c_int"][0]) == G["c_int"][0]
    else:
        qs = np.array([f32(h) for h in G["q_scales"]])
        assert np.array_equal(info["q_scales"], qs)
        assert info["c_int"].tolist() == G["c_int"]
    if row_stride == 1:
        u = 0
        for b in range(B):
            for h in range(H):
                n = int(lens[b])
                assert digest(out[b, h, :n]) == G["unit_digests"][u], (name, b, h)
                assert not out[b, h, n:].any()
                u += 1


@pytest.mark.parametrize("name", ["C1", "C2", "C2h", "C3"])
def test_configs_bit_exact(name):
    _check_config(name)


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_configs_scales(name):
    if name not in configs():
        pytest.skip("golden for this config not generated")
    _check_config(name, row_stride=1 << 20)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C4", "C5"])
def test_configs_bit_exact_long(name):
    if name not in configs():
        pytest.skip("golden for this config not generated")
    _check_config(name)


def _grouped():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "grouped_cases.npz"))


def test_oracle_grouped_softmax_matches_reference():
    """The numpy restatement of index_softmax_grouped equals the reference's
    own outputs (tests/golden/grouped_cases.npz, oracle/gen_golden.py)."""
    G = _grouped()
    lut = O.build_lut(5, 6.6)
    for i in range(int(G["n_sm"])):
        key = f"sm{i}"
        mask = G[key + "_mask"]
        mask = None if mask.size == 0 else mask
        cis = [O.c_int_from_alpha(6.6, a) for a in G[key + "_alphas"]]
        got = O.index_softmax_grouped(G[key + "_logits"], G[key + "_groups"], cis, lut, mask,
                                      int(G[key + "_pf"]))
        assert np.array_equal(got, G[key + "_prob"]), key


def test_oracle_quant_only_matches_reference():
    """The numpy restatement of quant_only_attention reproduces the reference's own
    outputs and requantised P^ (tests/golden/quant_only_cases.npz) exactly: same f32
    numpy operations."""
    import os
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "quant_only_cases.npz"))
    for i in range(int(G["n"])):
        key = f"qo{i}"
        mask = G[key + "_mask"]
        mask = None if mask.size == 0 else mask
        out, phat = O.quant_only_attention(G[key + "_q"], G[key + "_k"], G[key + "_v"], mask,
                                           int(G[key + "_pf"]))
        assert np.array_equal(phat, G[key + "_phat"]), key
        assert np.array_equal(out.view(np.uint32), G[key + "_out"].view(np.uint32)), key


def test_oracle_grouped_pipeline_vs_reference():
    """The grouped-K oracle composition (oracle.attention_grouped_batched) reproduces the
    reference's per-row-group K int_attention (pipeline.py:229-246) bit for bit on the
    committed fixtures (gs 32, 16 and 7; causal and not)."""
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "grouped_cases.npz"))
    for i in range(int(G["n_pipe"])):
        key = f"pipe{i}"
        q, k, v = G[key + "_q"], G[key + "_k"], G[key + "_v"]
        out = O.attention_grouped_batched(q[None, None], k[None, None], v[None, None],
                                          int(G[key + "_gs"]), causal=bool(int(G[key + "_causal"])))
        assert np.array_equal(out[0, 0].view(np.uint32), G[key + "_out"].view(np.uint32)), key
