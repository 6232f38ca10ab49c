"""ctypes mirror of include/frsvt.h (layouts must match the header exactly)."""
import ctypes
import os

FRSVT_LMAX = 128
FRSVT_F32, FRSVT_F64 = 0, 1

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfrsvt.so")

# every entry point include/frsvt.h declares (checked by tests/test_abi.py)
SYMBOLS = [
    "frsvt_batched_apply", "frsvt_batched_apply_f64", "frsvt_loopback_create", "frsvt_loopback_destroy", "frsvt_get_unique_id", "frsvt_create", "frsvt_destroy", "frsvt_status_string",
    "frsvt_apply", "frsvt_apply_weighted", "rpca_alm_step", "frsvt_set_omega",
    "frsvt_draw_omega", "frsvt_get_carry", "frsvt_set_carry", "frsvt_reset_carry",
    "frsvt_set_call_index", "frsvt_set_adaptive_rank", "frsvt_get_info", "rpca_get_mu", "rpca_set_mu",
    "frsvt_kernel_launches", "frsvt_profile", "frsvt_profile_read", "frsvt_debug_pass",
    "frsvt_debug_small_svd", "frsvt_debug_pass_timed", "frsvt_debug_chol", "frsvt_debug_chol_inv",
]


class FrsvtConfig(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("m_local", ctypes.c_int64), ("n", ctypes.c_int64),
                ("m_global", ctypes.c_int64), ("row0", ctypes.c_int64), ("l", ctypes.c_int32),
                ("q", ctypes.c_int32), ("range_propagation", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nccl_id", ctypes.POINTER(ctypes.c_ubyte)), ("options", ctypes.c_uint32),
                ("group", ctypes.c_void_p)]

FRSVT_OPT_FUSED_SKETCH = 1
FRSVT_OPT_TF32_OMEGA = 2


class FrsvtInfo(ctypes.Structure):
    _fields_ = [("s", ctypes.c_int32), ("r", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("sweeps", ctypes.c_int32), ("calls", ctypes.c_int64),
                ("sigma", ctypes.c_double * FRSVT_LMAX), ("d", ctypes.c_double * FRSVT_LMAX),
                ("mu", ctypes.c_double), ("l_next", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("varsigma", ctypes.c_double)]


class RpcaState(ctypes.Structure):
    _fields_ = [("D", ctypes.c_void_p), ("E", ctypes.c_void_p), ("A", ctypes.c_void_p),
                ("L", ctypes.c_void_p), ("ld", ctypes.c_int64), ("lambda_", ctypes.c_double),
                ("rho", ctypes.c_double), ("mu_max_factor", ctypes.c_double),
                ("norm2_D", ctypes.c_double), ("mu0", ctypes.c_double), ("iter", ctypes.c_int32),
                ("keep", ctypes.c_int32), ("transfer", ctypes.c_int32)]


def load_library(path=LIB_PATH):
    if not os.path.exists(path):
        raise ImportError("libfrsvt.so is not built (%s); run `python paper_1509_00296_b200/build.py` "
                          "or __graft_entry__.build()" % path)
    lib = ctypes.CDLL(path)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    sig = {
        "frsvt_batched_apply": (i32, [i32, i64, i64, i32, i32, vp, i64, i64, vp, i64, i32, dbl, vp, vp, vp, i64, i64,
                                      vp, vp, vp]),
        "frsvt_batched_apply_f64": (i32, [i32, i64, i64, i32, i32, vp, i64, i64, vp, i64, i32, dbl, vp, vp, vp, i64,
                                          i64, vp, vp, vp]),
        "frsvt_loopback_create": (i32, [i32, P(vp)]),
        "frsvt_loopback_destroy": (None, [vp]),
        "frsvt_get_unique_id": (i32, [P(ctypes.c_ubyte)]),
        "frsvt_create": (i32, [P(FrsvtConfig), vp, P(vp)]),
        "frsvt_destroy": (None, [vp]),
        "frsvt_status_string": (ctypes.c_char_p, [i32]),
        "frsvt_apply": (i32, [vp, vp, i64, dbl, vp, i64, P(FrsvtInfo)]),
        "frsvt_apply_weighted": (i32, [vp, vp, i64, i32, P(dbl), dbl, dbl, vp, i64, P(FrsvtInfo)]),
        "rpca_alm_step": (i32, [vp, P(RpcaState), i32, P(dbl)]),
        "frsvt_set_omega": (i32, [vp, vp, i64]),
        "frsvt_draw_omega": (i32, [vp, i64, vp, i64]),
        "frsvt_get_carry": (i32, [vp, vp, i64, P(i32)]),
        "frsvt_set_carry": (i32, [vp, vp, i64, i32]),
        "frsvt_reset_carry": (i32, [vp]),
        "frsvt_set_call_index": (i32, [vp, i64]),
        "frsvt_set_adaptive_rank": (i32, [vp, i32, i32, i32, i32]),
        "frsvt_get_info": (i32, [vp, P(FrsvtInfo)]),
        "rpca_get_mu": (i32, [vp, P(dbl)]),
        "rpca_set_mu": (i32, [vp, dbl, dbl]),
        "frsvt_kernel_launches": (i64, [vp]),
        "frsvt_profile": (i32, [vp, i32]),
        "frsvt_debug_pass": (i32, [vp, i32, i32, vp, i64, vp, vp]),
        "frsvt_profile_read": (i32, [vp, i32, P(dbl), P(i64), P(dbl)]),
        "frsvt_debug_small_svd": (i32, [vp, i32, vp, vp, vp, vp, P(i32), i32, P(dbl)]),
        "frsvt_debug_pass_timed": (i32, [vp, i32, i32, vp, i64, vp, vp, i32, P(dbl)]),
        "frsvt_debug_chol": (i32, [vp, vp, vp, P(i32), vp]),
        "frsvt_debug_chol_inv": (i32, [vp, vp, i32, vp, P(i32), vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib, path


def status_string(lib, st):
    s = lib.frsvt_status_string(int(st))
    return s.decode() if s else "unknown"
