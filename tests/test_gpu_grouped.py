"""Grouped-K IndexSoftmax inside the fused kernel (reference
softmax.py:309-399 default per-group-max mode, pipeline.py:229-246): one launch,
per-(head, key group) clip thresholds and row maxima, no int32 logits in HBM.
Checked bit for bit against the oracle composition (pinned to the reference's own
grouped pipeline outputs in test_oracle_golden.py) and the reference fixtures."""
import numpy as np
import pytest
import torch

import paper_2511_21513_b200 as ia
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _inputs(B, H, Hkv, L, d, seed, kscale=True):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, H, L, d), dtype=np.float32)
    k = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    if kscale:  # per-row K magnitudes vary, so the groups get different scales
        k *= rng.uniform(0.3, 6.0, size=(B, Hkv, L, 1)).astype(np.float32)
    v = rng.standard_normal((B, Hkv, L, d), dtype=np.float32)
    return q, k, v


@pytest.mark.parametrize("B,H,Hkv,L,d,gs,causal", [
    (1, 1, 1, 96, 32, 32, False),     # one resident tile, groups inside a half
    (1, 2, 1, 256, 64, 16, True),     # 2 tiles, GQA
    (2, 4, 2, 384, 128, 128, False),  # a group = a whole tile (both halves)
    (1, 2, 2, 1024, 64, 8, True),     # many groups, non-resident (8 tiles)
    (1, 1, 1, 200, 128, 8, True),     # ragged last tile
    (1, 2, 1, 576, 128, 64, True),    # ragged last tile, 64-key groups
])
def test_grouped_fused_vs_oracle(B, H, Hkv, L, d, gs, causal):
    q, k, v = _inputs(B, H, Hkv, L, d, seed=B * 7 + L + gs)
    got = ia.int_attention_batched(q, k, v, causal=causal, k_group_size=gs)
    want = O.attention_grouped_batched(q, k, v, gs, causal=causal)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_grouped_fused_mask_and_int8x127():
    rng = np.random.default_rng(5)
    L, d, gs = 320, 64, 32
    q, k, v = _inputs(1, 2, 1, L, d, seed=11)
    mask = rng.random((L, L)) < 0.3
    mask[7, :] = True  # a fully masked row -> zeros
    cfg = ia.AttentionConfig(p_format=ia.PFormat.INT8X127)
    got = ia.int_attention_batched(q, k, v, mask=mask, cfg=cfg, k_group_size=gs)
    want = O.attention_grouped_batched(q, k, v, gs, mask=mask, p_scale=127)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert not got[0, :, 7].any()


def test_grouped_fused_int_attention_api_matches_reference_fixtures():
    """ia.int_attention with per_row_group(gs) K takes the fused path for gs in
    {16, 32} (the reference's own fixtures) and the stage path for gs = 7."""
    import os
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "grouped_cases.npz"))
    for i in range(int(G["n_pipe"])):
        key = f"pipe{i}"
        L = G[key + "_q"].shape[0]
        gs = int(G[key + "_gs"])
        mask = np.triu(np.ones((L, L), bool), 1) if int(G[key + "_causal"]) else None
        cfg = ia.AttentionConfig(granularity=ia.QuantGranularity.per_row_group(gs), mask=mask)
        out, t = ia.int_attention(G[key + "_q"], G[key + "_k"], G[key + "_v"], cfg)
        assert np.array_equal(np.asarray(out).view(np.uint32), G[key + "_out"].view(np.uint32)), key
        if gs in (16, 32):  # fused: no separate QK^T / P.V stages
            assert t.qk_gemm_ns == 0 and t.pv_gemm_ns == 0


@pytest.mark.parametrize("scale", [0.25, 0.05, 0.004])
@pytest.mark.parametrize("masked", [False, True])
def test_grouped_fused_integer_form_groups(scale, masked):
    """Small operand scales make c_int large: groups whose c_eff (2k + 1) >= 2^23 leave the
    float index form for the magic-number form (and, smaller still, the c_eff sentinel);
    with per-row K magnitudes spread over 20x the two forms mix inside one head, sharing
    the reversed row table."""
    L, d, gs = 576, 64, 16
    q, k, v = _inputs(1, 2, 1, L, d, seed=21)
    q *= np.float32(scale)
    k *= np.float32(scale)
    mask = None
    if masked:
        mask = np.random.default_rng(9).random((L, L)) < 0.25
    got = ia.int_attention_batched(q, k, v, causal=not masked, mask=mask, k_group_size=gs)
    want = O.attention_grouped_batched(q, k, v, gs, causal=not masked, mask=mask)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_grouped_fused_c3_shape():
    """C3-shaped (L = 2048, d = 128, causal) with 64-key K groups, 4 heads."""
    q, k, v = _inputs(1, 4, 2, 2048, 128, seed=3)
    got = ia.int_attention_batched(q, k, v, causal=True, k_group_size=64)
    want = O.attention_grouped_batched(q, k, v, 64, causal=True)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_grouped_fused_rejects_outside_domain():
    q, k, v = _inputs(1, 1, 1, 96, 32, seed=1)
    for gs in (7, 256, 12):
        with pytest.raises(ValueError):
            ia.int_attention_batched(q, k, v, k_group_size=gs)
    with pytest.raises(ValueError):
        ia.int_attention_batched(q, k, v, k_group_size=32, seq_lens=[96])
