"""ctypes binding of the C ABI in include/intattn_b200.h.

The library is built in-tree (paper_2511_21513_b200/_lib/libintattn_b200.so,
see csrc/Makefile).  There is no CPU fallback: if the library or an sm_100
device is missing, every operator raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("IA_LIB") or os.path.join(_HERE, "_lib", "libintattn_b200.so")
CSRC = os.path.join(_HERE, "csrc")

IA_OK = 0
IA_ERR_INVALID_ARGUMENT = 1
IA_ERR_SEQ_LEN = 2
IA_ERR_HEAD_DIM = 3
IA_ERR_NONFINITE = 4
IA_ERR_CUDA = 5
IA_ERR_NO_DEVICE = 6
IA_ERR_LUT = 7

IA_QMODE_ROWS = 0
IA_QMODE_COLS = 1

# Every symbol include/intattn_b200.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "ia_abi_version", "ia_status_string", "ia_last_error", "ia_device_check",
    "ia_quant_amax_rows", "ia_quant_amax_cols", "ia_quant_scales", "ia_quantize",
    "ia_dequantize", "ia_quant_heads", "ia_quant_tensors", "ia_head_params_host", "ia_softmax_params_host", "ia_head_params_dev",
    "ia_mask_pack", "ia_attn_fwd", "ia_attn_supported", "ia_index_softmax", "ia_index_softmax_grouped",
    "ia_gemm_i8", "ia_copy_rows_async", "ia_group_params_dev", "ia_zero_async",
)


class HeadParams(ctypes.Structure):
    _fields_ = [("c_int", ctypes.c_int64), ("c_eff", ctypes.c_int64),
                ("magic", ctypes.c_uint32), ("shift", ctypes.c_int32),
                ("use32", ctypes.c_int32), ("out_scale", ctypes.c_float),
                ("s_q", ctypes.c_float), ("s_k", ctypes.c_float), ("s_v", ctypes.c_float),
                ("unc32", ctypes.c_int32), ("magic9", ctypes.c_uint32),
                ("fratio", ctypes.c_float)]


class AttnArgs(ctypes.Structure):
    _fields_ = [("q", ctypes.c_void_p), ("k", ctypes.c_void_p), ("vt", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("params", ctypes.c_void_p),
                ("seq_lens", ctypes.c_void_p), ("mask_bits", ctypes.c_void_p),
                ("B", ctypes.c_int64), ("H", ctypes.c_int64), ("Hkv", ctypes.c_int64),
                ("L", ctypes.c_int64), ("d", ctypes.c_int64), ("d_pad", ctypes.c_int64),
                ("l_pad", ctypes.c_int64), ("causal", ctypes.c_int32),
                ("nlut", ctypes.c_int32), ("p_scale", ctypes.c_int32),
                ("lut", ctypes.c_uint8 * 256), ("dbg_logits", ctypes.c_void_p),
                ("dbg_prob", ctypes.c_void_p), ("dbg_acc", ctypes.c_void_p),
                ("dbg_times", ctypes.c_void_p), ("softmax_mode", ctypes.c_int32),
                ("kgroup_params", ctypes.c_void_p), ("k_group_size", ctypes.c_int32)]

GROUP_PARAMS_BYTES = 16  # ia_group_params {c_eff, magic, shift, use32}

IA_SOFTMAX_INDEX = 0
IA_SOFTMAX_FLOAT = 1


_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the CUDA library in-tree with nvcc (sm_100a)."""
    if force or not os.path.exists(SO_PATH):
        subprocess.run(["make", "-s", "-C", CSRC] + (["-B"] if force else []), check=True)
    else:
        subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return SO_PATH


def load():
    """Load (once) and return the ctypes handle; raises if the library is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SO_PATH):
            raise RuntimeError(
                f"CUDA extension not built: {SO_PATH} is missing "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        L = ctypes.CDLL(SO_PATH)
        P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        sig = {
            "ia_abi_version": ([], i32),
            "ia_status_string": ([i32], ctypes.c_char_p),
            "ia_last_error": ([], ctypes.c_char_p),
            "ia_device_check": ([i32], i32),
            "ia_quant_amax_rows": ([P, i64, i64, i64, P, i64, i64, P, P, P], i32),
            "ia_quant_amax_cols": ([P, i64, i64, i64, P, P, P], i32),
            "ia_quant_scales": ([P, i64, P, P], i32),
            "ia_quant_heads": ([P, P, P, i64, i64, i64, i64, i64, P, P, P, P, i64, i64, P, P, P,
                                P, P], i32),
            "ia_quant_tensors": ([P, P, P, i64, i64, i64, i64, i64, P, P, P, P, i64, i64, P, P,
                                  P, P], i32),
            "ia_quantize": ([P, i64, i64, i64, P, i64, i32, i64, i64, P, P, i64, i32, i64, P], i32),
            "ia_dequantize": ([P, i64, i64, i32, i64, P, P, P], i32),
            "ia_head_params_host": ([ctypes.c_double, i64, i32, i32, ctypes.c_float,
                                     ctypes.c_float, ctypes.c_float, ctypes.POINTER(HeadParams)], i32),
            "ia_softmax_params_host": ([i64, i64, i32, ctypes.POINTER(HeadParams)], i32),
            "ia_head_params_dev": ([P, P, P, i32, i32, i64, i64, i64, i64, ctypes.c_double,
                                    i32, i32, P, P], i32),
            "ia_mask_pack": ([P, i64, P, P], i32),
            "ia_attn_fwd": ([ctypes.POINTER(AttnArgs), P], i32),
            "ia_attn_supported": ([i64, i32], i32),
            "ia_index_softmax": ([P, i64, i64, ctypes.POINTER(HeadParams), P, i32, i32, P, P, P], i32),
            "ia_index_softmax_grouped": ([P, i64, i64, P, i32, P, P, i32, i32, P, P, P], i32),
            "ia_gemm_i8": ([P, i64, i32, P, i64, i64, i64, i64, P, i64, P], i32),
            "ia_copy_rows_async": ([P, i64, P, i64, i64, i64, P], i32),
            "ia_group_params_dev": ([P, P, i64, i64, i64, i64, i64, ctypes.c_double, i32, P, P],
                                    i32),
            "ia_zero_async": ([P, i64, P], i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return _lib


def check(status: int, what: str = "") -> None:
    """Map an ia_status to the reference's exception types."""
    if status == IA_OK:
        return
    L = load()
    detail = L.ia_last_error().decode(errors="replace")
    msg = f"{what}: {detail}" if what else detail
    if status in (IA_ERR_INVALID_ARGUMENT, IA_ERR_SEQ_LEN, IA_ERR_HEAD_DIM, IA_ERR_NONFINITE,
                  IA_ERR_LUT):
        raise ValueError(msg)
    raise RuntimeError(msg)


def head_params_host(c, d, nlut, p_scale, s_q, s_k, s_v) -> HeadParams:
    hp = HeadParams()
    check(load().ia_head_params_host(float(c), int(d), int(nlut), int(p_scale), float(s_q),
                                     float(s_k), float(s_v), ctypes.byref(hp)), "head params")
    return hp


def softmax_params_host(c_int, delta_bound, nlut) -> HeadParams:
    hp = HeadParams()
    check(load().ia_softmax_params_host(int(c_int), int(delta_bound), int(nlut),
                                        ctypes.byref(hp)), "softmax params")
    return hp
