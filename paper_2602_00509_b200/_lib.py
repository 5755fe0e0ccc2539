"""ctypes binding of include/probe.h — argument marshalling only.

Every step of the hot path runs in libprobe.so (sm_100a CUDA).  If the library
is missing or cannot be loaded this module raises: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libprobe.so")

PROBE_NSYM = 9
PROBE_NBUF = 10
BUF_RECV, BUF_Y, BUF_REP_W13, BUF_REP_W2, BUF_BOARD, BUF_SIGNAL, BUF_META, BUF_COMB, BUF_PRE, BUF_SCRATCH = range(10)

STATUS = {0: "PROBE_OK", 1: "PROBE_EINVAL", 2: "PROBE_ESHAPE", 3: "PROBE_EBUDGET", 4: "PROBE_ECAPACITY",
          5: "PROBE_ECUDA", 6: "PROBE_ECOMM", 7: "PROBE_ESTATE"}

# every exported symbol declared in include/probe.h
EXPORTS = ["probe_workspace", "probe_init", "probe_moe_forward", "probe_predict", "probe_plan",
           "probe_prefetch", "probe_debug_layout", "probe_debug_prefetch", "probe_debug_flags", "probe_window", "probe_test_gemm", "probe_check", "probe_last_error",
           "probe_finalize", "probe_launch_count", "probe_profile", "probe_profile_read", "probe_bench_gemm",
           "probe_ipc_export", "probe_ipc_import", "probe_ipc_close", "probe_set_option",
           "probe_history_update", "probe_distill_grad", "probe_distill_apply", "probe_predict_prepare"]
OPT_EP_EMULATION, OPT_UNFUSED_TOPK, OPT_FUSED_EPILOGUE_TOPK, OPT_AUX_SMS, OPT_PAIR_GEMM = 1, 2, 3, 4, 5
OPT_AUX_START, OPT_PRED_MAXREG, OPT_L2_HINTS, OPT_PRED_PAIR = 8, 9, 10, 11
DTYPES = {"bf16": 0, "fp32": 1}      # probe_config.dtype (PROBE_BF16, PROBE_FP32)
PROBE_NPHASE = 13
PHASES = ["gate", "select", "counts", "layout", "dispatch", "expand", "wait", "gemm1", "gemm2", "combine", "reduce",
          "total", "predispatch"]


class probe_config(C.Structure):
    _fields_ = [("ep_size", C.c_int32), ("rank_begin", C.c_int32), ("local_ranks", C.c_int32),
                ("num_experts", C.c_int32), ("top_k", C.c_int32), ("hidden", C.c_int32), ("ffn", C.c_int32),
                ("res_hidden", C.c_int32), ("max_tokens", C.c_int32), ("recv_capacity", C.c_int32),
                ("replica_budget", C.c_int32), ("kmax", C.c_int32), ("n_sat", C.c_int32), ("dtype", C.c_int32),
                ("dedup_wire", C.c_int32), ("predispatch", C.c_int32), ("fuse_gate_predictor", C.c_int32),
                ("alpha_ps", C.c_int64), ("beta_ps", C.c_int64), ("bw_bytes_per_us", C.c_int64),
                ("expert_bytes", C.c_int64)]


class ProbeError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if path == LIB_PATH and os.environ.get("PROBE_LIB_PATH"):   # A/B of two builds (tools only)
        path = os.environ["PROBE_LIB_PATH"]
    elif path == LIB_PATH:
        from . import build as _build
        try:
            if _build.stale():
                _build.build()
        except Exception as e:  # no nvcc: fall through to the existence check (no CPU fallback)
            if not os.path.exists(path):
                raise ImportError(f"libprobe.so missing and build failed: {e}") from e
    if not os.path.exists(path):
        raise ImportError(f"libprobe.so not built at {path} (run paper_2602_00509_b200/build.py); "
                          "there is no CPU fallback")
    lib = C.CDLL(path)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "probe_workspace": (i32, [C.POINTER(probe_config), C.POINTER(C.c_uint64)]),
        "probe_init": (i32, [C.POINTER(probe_config), C.POINTER(C.c_uint64), vp, C.POINTER(vp)]),
        "probe_moe_forward": (i32, [vp, i32, vp, i32, vp, vp, vp, vp, i32, vp, i32, vp, vp, vp]),
        "probe_predict": (i32, [vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp]),
        "probe_predict_prepare": (i32, [vp, i32, vp, vp]),
        "probe_plan": (i32, [vp, i32, vp, vp, vp, vp, vp, vp]),
        "probe_prefetch": (i32, [vp, i32, vp, vp, i32, vp]),
        "probe_debug_layout": (i32, [vp, vp, vp, vp, vp, vp, vp]),
        "probe_debug_prefetch": (i32, [vp, vp, vp]),
        "probe_debug_flags": (i32, [vp, vp, vp]),
        "probe_window": (i32, [vp, i64, i64, vp, vp]),
        "probe_test_gemm": (i32, [vp, i64, vp, i64, i32, i32, C.POINTER(C.c_int32), i32, i32, vp, vp]),
        "probe_bench_gemm": (i32, [vp, i64, vp, i64, i32, i32, C.POINTER(C.c_int32), i32, i32, i32, i32,
                                   C.POINTER(C.c_float), vp, vp]),
        "probe_ipc_export": (i32, [vp, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)]),
        "probe_ipc_import": (i32, [C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_uint64)]),
        "probe_ipc_close": (i32, [C.c_uint64]),
        "probe_set_option": (i32, [vp, i32, i64]),
        "probe_history_update": (i32, [vp, i32, i32, vp, vp]),
        "probe_distill_grad": (i32, [vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp]),
        "probe_distill_apply": (i32, [vp, vp, vp, vp, i64, C.c_float, vp]),
        "probe_check": (i32, [vp]),
        "probe_last_error": (C.c_char_p, [vp]),
        "probe_finalize": (i32, [vp]),
        "probe_launch_count": (i64, [vp]),
        "probe_profile": (i32, [vp, i32]),
        "probe_profile_read": (i32, [vp, vp, C.POINTER(C.c_int32)]),
    }
    for name, (res, args) in sig.items():
        if path != LIB_PATH and not hasattr(lib, name):     # an older build under A/B (tools only)
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(fn: str, status: int, ctx=None):
    if status != 0:
        msg = load().probe_last_error(ctx)
        raise ProbeError(fn, status, msg.decode() if msg else "")
