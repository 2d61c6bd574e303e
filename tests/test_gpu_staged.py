"""int_attention_staged: the reference's five stages as separate launches
(pipeline.py:215-253), giving the full StageTimings split (quantize / qk_gemm /
softmax_path / pv_gemm / dequantize, pipeline.py:61-81) -- bit-identical to the
fused int_attention and to the oracle."""
import numpy as np
import pytest
import torch

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


@pytest.mark.parametrize("M,N,K,ldc_pad,c_off", [
    (300, 260, 96, 0, 0),    # whole-line vector stores with ragged last column block
    (257, 131, 64, 0, 0),    # N % 4 != 0: scalar epilogue
    (128, 256, 128, 3, 0),   # row pitch not a multiple of 4 ints: scalar epilogue
    (200, 192, 160, 4, 1),   # C not 16-byte aligned: scalar epilogue
    (513, 384, 32, 4, 4),    # aligned offset view: vector stores into a strided C
])
def test_gemm_i8_epilogue_forms_through_c_abi(M, N, K, ldc_pad, c_off):
    """ia_gemm_i8 writes whole 128-byte lines with 16-byte stores when C and its row pitch
    allow it and falls back to scalar stores otherwise; both forms are exact (gemm.py:45-59)
    and never touch C outside [M, N] (checked with a guard pattern)."""
    import ctypes

    from paper_2511_21513_b200 import _lib
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N)
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, generator=g).to(dev)
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, generator=g).to(dev)
    kp = (K + 15) // 16 * 16
    a_p = torch.zeros((M, kp), dtype=torch.int8, device=dev)
    b_p = torch.zeros((N, kp), dtype=torch.int8, device=dev)
    a_p[:, :K] = a
    b_p[:, :K] = b
    ldc = N + ldc_pad
    guard = 0x5A5A5A5A
    buf = torch.full((c_off + M * ldc + 8,), guard, dtype=torch.int32, device=dev)
    c_ptr = buf.data_ptr() + 4 * c_off
    L = _lib.load()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.ia_gemm_i8(ctypes.c_void_p(a_p.data_ptr()), kp, 1, ctypes.c_void_p(b_p.data_ptr()),
                            kp, M, N, K, ctypes.c_void_p(c_ptr), ldc, st), "gemm")
    torch.cuda.synchronize()
    c = buf[c_off:c_off + M * ldc].view(M, ldc)
    want = (a.cpu().to(torch.int64) @ b.cpu().to(torch.int64).T).to(torch.int32)
    assert torch.equal(c[:, :N].cpu(), want)
    if ldc_pad:
        assert bool((c[:, N:] == guard).all())
    assert bool((buf[:c_off] == guard).all()) and bool((buf[c_off + M * ldc:] == guard).all())
