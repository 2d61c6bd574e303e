"""int_attention_staged: the reference's five stages as separate launches
(pipeline.py:215-253), giving the full StageTimings split (quantize / qk_gemm /
softmax_path / pv_gemm / dequantize, pipeline.py:61-81) -- bit-identical to the
fused int_attention and to the oracle."""
import numpy as np
import pytest

import paper_2511_21513_b200 as ia
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,d,masked,p127,gs", [(200, 64, False, False, None),
                                                (333, 128, True, True, None),
                                                (256, 64, True, False, 16),
                                                (70, 20, False, False, 7)])
def test_staged_matches_fused_and_splits_every_stage(L, d, masked, p127, gs):
    rng = np.random.default_rng(L + d)
    q, k, v = (rng.standard_normal((L, d), dtype=np.float32) for _ in range(3))
    mask = np.triu(np.ones((L, L), bool), 1) if masked else None
    kw = {}
    if gs:
        kw["granularity"] = ia.QuantGranularity.per_row_group(gs)
    cfg = ia.AttentionConfig(mask=mask, p_format=ia.PFormat.INT8X127 if p127 else ia.PFormat.UINT8X255,
                             **kw)
    fused, tf = ia.int_attention(q, k, v, cfg)
    staged, ts = ia.int_attention_staged(q, k, v, cfg, warmup=1, iters=3)
    assert np.array_equal(np.asarray(staged).view(np.uint32), np.asarray(fused).view(np.uint32))
    if gs is None:
        want = O.int_attention(q, k, v, mask=mask, p_scale=127 if p127 else 255)
        assert np.array_equal(np.asarray(staged).view(np.uint32), want.view(np.uint32))
    for f in ("quantize_ns", "qk_gemm_ns", "softmax_path_ns", "pv_gemm_ns", "dequantize_ns"):
        assert getattr(ts, f) > 0, f
    assert ts.total_ns >= ts.qk_gemm_ns + ts.pv_gemm_ns
