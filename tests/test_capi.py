"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and its host-side parameter math (c_int, the exact
magic-number index map) is right.  The product path must refuse to run
without a device (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

from golden_io import f32, stage_cases
from oracle import oracle as O
from paper_2511_21513_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "intattn_b200.h")


def header_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ia_\w+)\s*\(", txt, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.load()
    declared = header_functions()
    assert len(declared) >= 16
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/intattn_b200.h but not exported"
    assert sorted(_lib.EXPORTS) == declared
    assert L.ia_abi_version() == 5


def test_status_strings():
    L = _lib.load()
    for code in range(8):
        assert L.ia_status_string(code)
    assert L.ia_status_string(4).decode() == "input contains non-finite elements"


def test_no_device_raises():
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    L = _lib.load()
    assert L.ia_device_check(0) == _lib.IA_ERR_NO_DEVICE
    import paper_2511_21513_b200 as ia
    x = np.ones((4, 8), np.float32)
    with pytest.raises(RuntimeError):
        ia.int_attention(x, x, x)
    with pytest.raises(RuntimeError):
        ia.quantize_symmetric(x)


def test_quant_entry_points_validate_before_device_work():
    """ia_quant_heads / ia_quant_tensors reject null pointers, bad shapes and
    misaligned operands with IA_ERR_INVALID_ARGUMENT before any CUDA call."""
    L = _lib.load()
    buf = (ctypes.c_uint8 * 4096)()
    p = ctypes.addressof(buf)
    p = (p + 15) & ~15
    bad = _lib.IA_ERR_INVALID_ARGUMENT
    # B, H, Hkv, L, d, d_pad, l_pad
    good = (1, 2, 1, 16, 8, 16, 16)
    cases = [((1, 2, 1, 16, 8, 16, 16), True),    # null operand
             ((1, 3, 2, 16, 8, 16, 16), False),   # H % Hkv
             ((1, 2, 1, 16, 6, 16, 16), False),   # d % 4
             ((1, 2, 1, 16, 8, 8, 16), False),    # d_pad < d
             ((1, 2, 1, 17, 8, 16, 16), False)]   # l_pad < L
    for (B, H, Hkv, Lq, d, dp, lp), null in cases:
        ptrs = [p] * 6
        if null:
            ptrs[1] = None
        q, k, v, qh, kh, vt = ptrs
        assert L.ia_quant_heads(q, k, v, B, H, Hkv, Lq, d, None, qh, kh, vt, dp, lp,
                                p, p, p, p, None) == bad
        assert L.ia_quant_tensors(q, k, v, B, H, Hkv, Lq, d, None, qh, kh, vt, dp, lp,
                                  p, p, p, None) == bad
    B, H, Hkv, Lq, d, dp, lp = good
    assert L.ia_quant_tensors(p + 4, p, p, B, H, Hkv, Lq, d, None, p, p, p, dp, lp,
                              p, p, p, None) == bad  # misaligned
    assert L.ia_quant_heads(p, p, p, B, H, Hkv, Lq, d, None, p, p, p, dp, lp,
                            p, None, p, p, None) == bad  # per-head needs counters
    assert L.ia_last_error()


@pytest.mark.parametrize("idx", range(0, len(stage_cases()), 7))
def test_c_int_matches_reference(idx):
    row = stage_cases()[idx]
    case = row["case"]
    d = case["d"]
    p = case["p"]
    hp = _lib.head_params_host(case["c"], d, 1 << case["b"], p, f32(row["sq"]), f32(row["sk"]),
                               f32(row["sv"]))
    assert hp.c_int == row["c_int"]
    assert hp.out_scale == np.float32(float(f32(row["sv"])) / p)


def _check_map(hp, k, deltas):
    """Device index map (softmax.py:144-153 via params.cuh) vs exact integer division."""
    c_eff = hp.c_eff
    dp = np.minimum(deltas.astype(np.int64), c_eff)
    n = (2 * k * dp + c_eff).astype(np.uint64)
    want = n // np.uint64(2 * c_eff)
    if hp.use32:
        assert int(n.max()) < (1 << 31)
        q = (n * np.uint64(hp.magic)) >> np.uint64(32)
        got_shf = q >> np.uint64(hp.shift)
        got_mul = (q * np.uint64(1 << (32 - hp.shift))) >> np.uint64(32)
        assert np.array_equal(got_shf, want)
        assert np.array_equal(got_mul, want)
    if hp.magic9:  # pass-3 row-table address form: umulhi(n, magic9) & ~511 == idx * 512
        assert hp.use32 and int(n.max()) <= (2 * k + 1) * c_eff
        q9 = (n * np.uint64(hp.magic9)) >> np.uint64(32)
        assert np.array_equal(q9 & np.uint64(0xFFFFFE00), want * np.uint64(512))
        # ... and for the UNCLIPPED n of rows whose largest index fits the kernel's
        # zero-extended row table (idx <= NT9 = 55 for <= 32-entry LUTs)
        nt9 = (56 if k + 1 <= 32 else k + 1) - 1
        top = (2 * c_eff * (nt9 + 1) - 1 - c_eff) // (2 * k)  # largest delta with idx <= NT9
        step = max(1, top // 2_000_000)
        du = np.unique(np.concatenate([np.arange(0, top + 1, step, dtype=np.int64),
                                       np.arange(max(0, top - 5000), top + 1, dtype=np.int64)]))
        nu = (2 * k * du + c_eff).astype(np.uint64)
        wu = nu // np.uint64(2 * c_eff)
        assert int(wu.max()) <= nt9
        qu = (nu * np.uint64(hp.magic9)) >> np.uint64(32)
        assert np.array_equal(qu & np.uint64(0xFFFFFE00), wu * np.uint64(512))


@pytest.mark.parametrize("b", [2, 5, 8])
@pytest.mark.parametrize("d", [1, 64, 128, 256])
def test_magic_index_map_exhaustive(b, d):
    """Exhaustive over every reachable clipped distance for a spread of c_int."""
    k = (1 << b) - 1
    rng = np.random.default_rng(b * 1000 + d)
    c_values = [1, 2, 3, 50, 614, 716, 37335, 45302, 63190, 1 << 20, 1 << 40, 1 << 52]
    c_values += [int(x) for x in rng.integers(1, 200000, size=6)]
    dbound = 2 * d * 127 * 127
    for ci in c_values:
        hp = _lib.softmax_params_host(ci, dbound, 1 << b)
        c_eff = hp.c_eff
        assert c_eff == min(ci, 2 * k * dbound + 1)
        top = min(c_eff, dbound)
        if top <= 3_000_000:
            deltas = np.arange(0, top + 1, dtype=np.int64)
        else:
            deltas = np.unique(np.concatenate([rng.integers(0, top + 1, 2_000_000),
                                               np.arange(0, 1000), np.arange(top - 1000, top + 1)]))
        _check_map(hp, k, deltas)
        if hp.unc32:  # the same magic is exact without the clip, up to delta = dbound
            un = np.unique(np.concatenate([rng.integers(0, dbound + 1, 400000),
                                           np.arange(max(0, dbound - 2000), dbound + 1)]))
            n_u = (2 * k * un + c_eff).astype(np.uint64)
            assert int(n_u.max()) < (1 << 31)
            got = ((n_u * np.uint64(hp.magic)) >> np.uint64(32)) >> np.uint64(hp.shift)
            assert np.array_equal(got, n_u // np.uint64(2 * c_eff))
        # the reference's branchy form (delta >= c_int -> k) agrees on the full range
        big = np.unique(np.concatenate([deltas[::97], rng.integers(0, dbound + 1, 20000)]))
        ref = np.where(big >= ci, k, (2 * big * k + ci) // (2 * ci))
        dp = np.minimum(big, c_eff)
        mine = (2 * k * dp + c_eff) // (2 * c_eff)
        assert np.array_equal(ref, mine)


def test_use32_holds_for_baseline_configs():
    """The BASELINE configs (b = 5, d <= 128) always take the exact 32-bit path."""
    for ci in (614, 716, 5359, 37335, 48161, 58043, 63190, 1 << 52):
        for d in (64, 128):
            hp = _lib.softmax_params_host(ci, 2 * d * 127 * 127, 32)
            assert hp.use32 == 1 and hp.unc32 == 1


# The reference package's public names (intattn/__init__.py:56-92, its __all__).
REFERENCE_API = (
    "AttentionConfig", "ClipThreshold", "ElementKindMismatchError", "ExpLut", "FidelityReport",
    "LogitMatrix", "MalformedHeaderError", "MAX_HEAD_DIM", "MAX_SEQ_LEN", "PFormat",
    "ProbMatrix", "QuantGranularity", "QuantizedMatrix", "StageTimings", "TensorIOError",
    "TruncatedPayloadError", "build_lut", "compare", "compute_c_int", "dataflow_audit",
    "dequantize", "gemm_pv", "gemm_qk", "gemm_real", "index_softmax",
    "index_softmax_grouped", "int_attention", "load_tensor", "matmul_int8", "quant_only_attention",
    "quantize_symmetric", "reference_attention", "reference_attention_timed", "round_half_away", "save_tensor",
)


def test_exports_every_reference_name():
    """The drop-in exports each of the reference's 35 public names."""
    import paper_2511_21513_b200 as ia
    missing = [n for n in REFERENCE_API if not hasattr(ia, n)]
    assert not missing, missing
    assert len(REFERENCE_API) == 35
