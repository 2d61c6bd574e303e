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


def _float_ratio_parts(r):
    """f32 r > 0 as R * 2^-E with R a 24-bit integer."""
    mant, exp = np.frexp(np.float64(r))  # r = mant * 2^exp, mant in [0.5, 1)
    R = int(mant * (1 << 24))
    assert np.float64(R) * 2.0 ** (int(exp) - 24) == np.float64(r)
    return R, 24 - int(exp)


def test_float_index_map_exact():
    """params.cuh float form of idx = (2k*delta' + c) // (2c): with u = c - delta' =
    max(a - (m - c), 0) the kernel reads the integer u as the f32 denormal u * 2^-149 and
    takes j = RN(u * r + A) (pass 2) or RZ(u * 512 r + 256 + A) >> 9 (pass 3) from one FMA,
    idx = k - j.  Both are checked here in exact integer arithmetic for EVERY u in [0, c]
    with the ratio the library itself computes (ia_head_params.fratio)."""
    from paper_2511_21513_b200 import _lib

    rng = np.random.default_rng(7)
    for b in (2, 3, 5, 6):
        nlut = 1 << b
        k = nlut - 1
        cmax = ((1 << 23) - 1) // (2 * k + 1)          # largest c_eff with c (2k + 1) < 2^23
        c_values = [1, 2, 3, 7, 31, 62, 587, 660, 5233, 37474, 48161, 54498, cmax, cmax - 1, cmax + 1,
                    cmax + 2, 1 << 22, (1 << 23) - 1, 1 << 23]
        c_values += [int(x) for x in rng.integers(1, cmax + 1, size=8)]
        c_values += [k * (1 << j) for j in range(0, 14)]  # k / c exactly representable
        for c in c_values:
            hp = _lib.softmax_params_host(c, 2 * 256 * 127 * 127, nlut)
            c_eff = int(hp.c_eff)
            r = np.float32(hp.fratio)
            if not (hp.use32 and c_eff * (2 * k + 1) < (1 << 23)):
                assert r == 0, (b, c)
                continue
            assert r > 0 and np.float64(r) * c_eff < k   # strictly below k / c_eff ...
            above = np.nextafter(r, np.float32(np.inf))
            assert np.float64(above) * c_eff >= k         # ... and the largest such f32
            R, E = _float_ratio_parts(r)
            u = np.arange(0, c_eff + 1, dtype=np.int64)   # every clipped distance, reversed
            delta = c_eff - u
            want = (2 * k * delta + c_eff) // (2 * c_eff)
            prod = u * R  # < 2^47
            q, rem = prod >> E, prod & ((1 << E) - 1)
            half = 1 << (E - 1)
            rn = q + ((rem > half) | ((rem == half) & (q & 1 == 1)))
            assert np.array_equal(k - rn, want), (b, c, "RN form")
            rz = ((prod.astype(np.uint64) << np.uint64(9)) + (np.uint64(256) << np.uint64(E))) >> np.uint64(E)
            assert np.array_equal(k - (rz >> np.uint64(9)).astype(np.int64), want), (b, c, "RZ form")
