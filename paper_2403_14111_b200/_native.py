"""ctypes binding of the in-tree CUDA library ``libhc_b200.so`` (include/hc.h).

There is no CPU fallback: if the library is missing, ``lib()`` raises.  The
library itself loads without a GPU (static cudart); compute calls need a
B200 and fail with ``HC_ECUDA`` otherwise.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HC_LIB_PATH") or os.path.join(HERE, "libhc_b200.so")
CSRC = os.path.join(HERE, "csrc")

HC_EPARAM, HC_ECUDA, HC_EDEPTH, HC_ELEVEL, HC_EENCODE = -1, -2, -3, -4, -5
NCOUNTS = 8

_lib = None

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
I = C.c_int
I64 = C.c_int64
U64 = C.c_uint64
D = C.c_double
DP = C.POINTER(C.c_double)
U64P = C.POINTER(C.c_uint64)
I64P = C.POINTER(C.c_int64)
IP = C.POINTER(C.c_int)
REDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.c_int)

# name -> (restype, argtypes); mirrors include/hc.h one to one
SIGNATURES = {
    "hc_last_error": (C.c_char_p, []),
    "hc_ctx_create": (I, [I, I, IP, I, IP, I, I, I, D, U64, I, PP]),
    "hc_ctx_destroy": (I, [P]),
    "hc_ctx_info": (I, [P, U64P, DP]),
    "hc_set_grid_rows": (I, [P, I]),
    "hc_set_auto_bootstrap": (I, [P, I]),
    "hc_set_streams": (I, [P, I]),
    "hc_set_hoist": (I, [P, I]),
    "hc_ct_upload_async": (I, [P, U64P, I, PP]),
    "hc_ct_download_async": (I, [P, U64P]),
    "hc_ctx_counts": (I, [P, I64P, I]),
    "hc_ctx_nonce": (I, [P, U64P, U64P]),
    "hc_sync": (I, [P]),
    "hc_keygen": (I, [P, I]),
    "hc_key_download": (I, [P, I, U64P]),
    "hc_galois_rot": (U64, [P, I64]),
    "hc_ct_free": (I, [P]),
    "hc_ct_level": (I, [P]),
    "hc_ct_download": (I, [P, U64P]),
    "hc_ct_upload": (I, [P, U64P, I, PP]),
    "hc_ct_device_ptr": (I, [P, C.POINTER(U64P)]),
    "hc_pt_free": (I, [P]),
    "hc_encode_pt": (I, [P, DP, DP, I, PP]),
    "hc_pt_download": (I, [P, U64P]),
    "hc_encode_coef": (I, [P, DP, DP, D, I64P]),
    "hc_encrypt": (I, [P, DP, DP, I, U64, PP]),
    "hc_decrypt": (I, [P, P, DP, DP]),
    "hc_op_add": (I, [P, P, P, I, PP]),
    "hc_op_add_scalar": (I, [P, P, D, D, I, PP]),
    "hc_op_add_plain": (I, [P, P, DP, DP, C.c_char_p, I, PP]),
    "hc_op_mult": (I, [P, P, P, PP]),
    "hc_op_mult_scalar": (I, [P, P, D, D, PP]),
    "hc_op_mult_plain": (I, [P, P, DP, DP, C.c_char_p, PP]),
    "hc_op_lrot": (I, [P, P, I64, PP]),
    "hc_op_lrot_hoisted": (I, [P, P, C.POINTER(C.c_int64), I, PP]),
    "hc_op_ladder": (I, [P, P, C.c_int64, I, PP]),
    "hc_op_mult_sum": (I, [P, PP, PP, I, PP]),
    "hc_op_conj": (I, [P, P, PP]),
    "hc_op_mul_i": (I, [P, P, PP]),
    "hc_op_bootstrap": (I, [P, P, PP]),
    "hc_rescale": (I, [P, P, PP]),
    "hc_level_adjust": (I, [P, P, I, PP]),
    "hc_diag_abt": (I, [P, PP, I, I, PP, I, D, PP, I64P]),
    "hc_diag_atb": (I, [P, PP, I, PP, I, I, D, PP, I64P, REDUCE_FN, P]),
    "hc_softmax": (I, [P, PP, I, I, I, DP, PP, I64P]),
    "hc_approx": (I, [P, I, PP, PP, I, I, I, DP, PP, I64P]),
    "hc_col_major_abt": (I, [P, PP, I, I, PP, I, D, PP, I64P]),
    "hc_row_major_atb": (I, [P, PP, I, PP, I, I, D, PP, I64P]),
    "hc_mod_reduce": (I, [P, P]),
    "hc_set_shard": (I, [P, I, I]),
    "hc_set_app_level": (I, [P, I]),
    "hc_set_bootstrap": (I, [P, I]),
    "hc_bootstrap_ct": (I, [P, P, PP]),
    "hc_set_pass_shard": (I, [P, I, I, REDUCE_FN, P]),
    "hc_ctx_model_bytes": (I, [P, DP, I]),
    "hc_ctx_stream": (I, [P, PP]),
    "hc_timer_begin": (I, [P]),
    "hc_timer_end": (I, [P, C.POINTER(C.c_float)]),
    "hc_launch_count": (I64, [P]),
    "hc_bench_keyswitch": (I, [P, P, I, I, C.POINTER(C.c_float)]),
    "hc_bench_keyswitch_batch": (I, [P, P, I, I, I, C.POINTER(C.c_float)]),
    "hc_bench_ladder": (I, [P, P, I, I, C.c_int64, I, I, C.POINTER(C.c_float)]),
    "hc_bench_ntt": (I, [P, I, I, I, C.POINTER(C.c_float)]),
    "hc_prof_begin": (I, [P]),
    "hc_prof_end": (I, [P, C.c_char_p, I]),
}


def build(force: bool = False) -> str:
    """Compile the CUDA library in-tree for sm_100a (nvcc; no GPU needed)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-j8", "-C", CSRC])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA library {LIB_PATH} is not built; run `make -C {CSRC}` or "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc == 0:
        return
    from . import errors as E
    msg = lib().hc_last_error().decode(errors="replace")
    if rc == HC_EDEPTH:
        raise E.DepthExhausted(msg)
    if rc == HC_ELEVEL:
        raise E.ShapeMismatch(msg)
    if rc == HC_EENCODE:
        raise OverflowError(msg)
    if rc == HC_EPARAM:
        raise ValueError(msg)
    raise RuntimeError(f"hc error {rc}: {msg}")
