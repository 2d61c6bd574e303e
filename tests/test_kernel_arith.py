"""CPU checks of the integer-exactness arguments the fused kernel relies on
(float32 arithmetic emulated with numpy's IEEE round-to-nearest operations)."""
import numpy as np


def _rowtab_entry_kernel(num, two_s):
    """attention.cu, per-row table: q = trunc(f32(num) * rcp_rn(f32(2S))), then one
    remainder correction."""
    rden = np.float32(1.0) / two_s.astype(np.float32)
    q = np.trunc(num.astype(np.float32) * rden).astype(np.int64)
    r = num.astype(np.int64) - q * two_s.astype(np.int64)
    return q + np.where(r < 0, -1, np.where(r >= two_s.astype(np.int64), 1, 0))


def test_rowtab_division_exact():
    """(2 * p_scale * lut[t] + S) // (2S) for every LUT value, both P formats and S
    over its whole range (1 .. 255 * 65536: every key of a 65536-key row at lut 255)."""
    rng = np.random.default_rng(0)
    s = np.concatenate([np.arange(1, 20001), rng.integers(1, 255 * 65536 + 1, 200_000),
                        255 * 65536 - np.arange(2000), 2 ** np.arange(25)[2 ** np.arange(25) <= 255 * 65536]])
    s = s.astype(np.int64)
    lt = np.arange(1, 256, dtype=np.int64)
    for p_scale in (255, 127):
        num = (2 * p_scale * lt[None, :] + s[:, None])
        two_s = np.broadcast_to(2 * s[:, None], num.shape)
        got = _rowtab_entry_kernel(num, two_s)
        assert np.array_equal(got, num // two_s)
