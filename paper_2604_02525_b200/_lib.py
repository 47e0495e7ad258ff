"""ctypes loader for libadahop.so (the C ABI declared in include/adahop.h).

Argument marshalling only. There is no CPU fallback: if the shared library is missing
or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ADAHOP_LIB selects another in-tree build of the same ABI (kernel experiments)
LIB_PATH = os.environ.get("ADAHOP_LIB") or os.path.join(_HERE, "libadahop.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libadahop.so not found at {LIB_PATH}; build it with "
        "`python paper_2604_02525_b200/build.py` (no CPU fallback exists)")

lib = C.CDLL(LIB_PATH)


class Params(C.Structure):
    """adahop_params_t (include/adahop.h)."""
    _fields_ = [("had_block", C.c_int32), ("oe_k", C.c_int32), ("foid_probe", C.c_int32),
                ("level", C.c_int32), ("tau", C.c_float), ("eps", C.c_float)]

    def __init__(self, had_block=32, oe_k=64, foid_probe=64, level=1, tau=2.0, eps=1e-8):
        super().__init__(had_block, oe_k, foid_probe, level, tau, eps)


P = C.c_void_p
I32, I64, SZ, F64 = C.c_int32, C.c_int64, C.c_size_t, C.c_double
PP = C.POINTER(Params)

# name -> (restype, argtypes). Every symbol declared in include/adahop.h.
SIGNATURES = {
    "adahop_default_params": (None, [PP]),
    "adahop_abi_version": (I32, []),
    "adahop_status_string": (C.c_char_p, [I32]),
    "adahop_strategy_for_pair": (I32, [I32, I32, I32]),
    "adahop_majority_vote": (I32, [C.POINTER(I32), I32]),
    "adahop_classify_cv": (I32, [F64, F64, PP]),
    "adahop_layer_strategies": (I32, [I32, I32, I32, I32, C.POINTER(I32), C.POINTER(I32)]),
    "adahop_stats_workspace_bytes": (SZ, [I64, I64]),
    "adahop_stats": (I32, [P, I32, I64, I64, I64, P, P, P, SZ, P]),
    "adahop_classify": (I32, [P, I64, P, I64, I64, PP, P, P, P]),
    "adahop_classify_sums": (I32, [P, I64, I64, PP, P, P]),
    "adahop_calibrate_workspace_bytes": (SZ, [I64, I64]),
    "adahop_calibrate": (I32, [P, I32, I64, I64, I64, PP, P, SZ, P, P, P]),
    "adahop_calibrate_batch_workspace_bytes": (SZ, [I32, P, P]),
    "adahop_calibrate_batch": (I32, [I32, P, I32, P, P, P, PP, P, SZ, P, P, P]),
    "adahop_calibrate_batch_outliers": (I32, [I32, P, P, P, SZ, C.c_double, P, P]),
    "adahop_gemm_workspace_bytes": (SZ, [I64, I64, I64, I32, PP]),
    "adahop_gemm": (I32, [P, I32, I64, P, I32, I64, P, I32, I64, I64, I64, I64, I32, PP, P, SZ, P]),
    "adahop_workspace_bytes": (SZ, [I32, I64, I64, I64, I32, PP]),
    "adahop_linear_fwd": (I32, [P, P, P, I32, I64, I64, I64, I32, PP, P, SZ, P]),
    "adahop_linear_dgrad": (I32, [P, P, P, I32, I64, I64, I64, I32, PP, P, SZ, P]),
    "adahop_linear_wgrad": (I32, [P, P, P, I32, I64, I64, I64, I32, PP, P, SZ, P]),
    "adahop_layer_workspace_bytes": (SZ, [I64, I64, I64, C.POINTER(I32), PP]),
    "adahop_linear_layer": (I32, [P, P, P, P, P, P, I32, I32, I64, I64, I64, C.POINTER(I32), PP, P, SZ, P]),
    "adahop_linear_ctx_bytes": (SZ, [I64, I64, I64, C.POINTER(I32), PP]),
    "adahop_linear_split_workspace_bytes": (SZ, [I64, I64, I64, C.POINTER(I32), PP]),
    "adahop_linear_backward_needs_x": (I32, [C.POINTER(I32), PP]),
    "adahop_linear_forward": (I32, [P, P, P, I32, I64, I64, I64, C.POINTER(I32), PP, P, SZ, P, SZ, P]),
    "adahop_linear_backward": (I32, [P, P, P, P, P, I32, I32, I64, I64, I64, C.POINTER(I32), PP, P, SZ, P, SZ, P]),
    "adahop_debug_iht_quant": (I32, [P, I32, I64, I64, I64, I32, P, I32, P, P, P, P, SZ, P]),
    "adahop_debug_quant_dual": (I32, [P, I32, I64, I64, I64, P, I32, P, I32, P, P, P, P, P, P, P, SZ, P]),
    "adahop_debug_workspace_bytes": (SZ, [I64, I64]),
    "adahop_debug_foid": (I32, [P, I32, I64, I64, I64, I32, I32, I32, P, P, P, SZ, P]),
    "adahop_debug_gemm_mxf4": (I32, [P, P, P, P, P, I32, I64, I64, I64, I64, P, SZ, P]),
    "adahop_debug_gemm_workspace_bytes": (SZ, [I64, I64, I64]),
    "adahop_debug_sf_bytes": (SZ, [I64, I64]),
    "adahop_debug_gemm_mxf4_tcsf": (I32, [P, P, P, P, P, I32, I64, I64, I64, I64, P]),
    "adahop_debug_e2m1": (I32, [P, I64, P, P, P]),
    "adahop_debug_e2m1_exhaustive": (I32, [C.c_uint64, C.c_uint64, P, P, P]),
    "adahop_last_launch_count": (I32, []),
    "adahop_set_stage_events": (None, [P]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class AdahopError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = lib.adahop_status_string(status).decode()
        super().__init__(f"{fn} failed: {msg} (status {status})")
        self.status = status


def check(fn: str, status: int) -> None:
    if status != 0:
        raise AdahopError(fn, status)
