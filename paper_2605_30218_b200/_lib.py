"""ctypes binding of libmargingate.so (include/mg.h + include/mg_debug.h).

Argument marshalling only: every step of the decode path runs in the CUDA
kernels of the shared library.  There is no CPU fallback: if the library is
missing, `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# MG_LIB_PATH: another in-tree build of the same library (A/B timing scripts only)
LIB_PATH = os.environ.get("MG_LIB_PATH") or os.path.join(_HERE, "lib", "libmargingate.so")
_lock = threading.Lock()
_lib = None

MG_OK, MG_ERR_INVALID, MG_ERR_CAPACITY, MG_ERR_CUDA, MG_ERR_STATE, MG_ERR_NUMERIC = range(6)
STATUS = {0: "MG_OK", 1: "MG_ERR_INVALID", 2: "MG_ERR_CAPACITY", 3: "MG_ERR_CUDA", 4: "MG_ERR_STATE",
          5: "MG_ERR_NUMERIC"}


class MgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class MgConfig(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32), ("n_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32), ("qkv_bias", C.c_int32),
                ("rms_eps", C.c_float), ("rope_theta", C.c_float), ("weight_seed", C.c_uint64),
                ("max_batch", C.c_int32), ("max_slots", C.c_int32), ("max_seq", C.c_int32),
                ("page_size", C.c_int32), ("verify_chunk", C.c_int32)]


class MgSizes(C.Structure):
    _fields_ = [("weights", C.c_size_t), ("kv_fast", C.c_size_t), ("kv_shadow", C.c_size_t),
                ("workspace", C.c_size_t)]


class MgBuffers(C.Structure):
    _fields_ = [("weights", C.c_void_p), ("kv_fast", C.c_void_p), ("kv_shadow", C.c_void_p),
                ("workspace", C.c_void_p)]


class MgStats(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("rows", C.c_uint64), ("protected_rows", C.c_uint64),
                ("triggers", C.c_uint64), ("verified", C.c_uint64), ("repairs", C.c_uint64),
                ("verifier_launches", C.c_uint64), ("catchup_tokens", C.c_uint64), ("window_rows", C.c_uint64),
                ("rollbacks", C.c_uint64), ("rolled_back_tokens", C.c_uint64), ("error_flags", C.c_uint32)]


# every symbol declared in include/mg.h and include/mg_debug.h
PUBLIC_SYMBOLS = ["mg_query_sizes", "mg_init", "mg_prefill", "mg_decode_step", "mg_stats", "mg_release",
                  "mg_destroy", "mg_last_error", "mg_set_policy", "mg_verify_window"]
DEBUG_SYMBOLS = ["mgd_gen_tensor", "mgd_rmsnorm", "mgd_gemm", "mgd_qkv_epilogue", "mgd_attention",
                 "mgd_attention_streams", "mgd_residual", "mgd_swiglu", "mgd_top2", "mgd_gate", "mgd_read_column", "mgd_cache_digest", "mgd_last_step",
                 "mgd_capture_logits", "mgd_weight", "mgd_schedule", "mgd_launch_count", "mgd_set_timing",
                 "mgd_timing", "mgd_capture_verifier_logits", "mgd_set_inject",
                 "mgd_force_schedule", "mgd_gemm_top2", "mgd_launch_floor"]

_vp, _i32, _u32, _i64, _u64, _f32 = C.c_void_p, C.c_int32, C.c_uint32, C.c_int64, C.c_uint64, C.c_float
_P = C.POINTER

_SIGS = {
    "mg_query_sizes": [_P(MgConfig), _P(MgSizes)],
    "mg_init": [_P(MgConfig), _P(MgBuffers), _vp, _P(_vp)],
    "mg_prefill": [_vp, _i32, _P(_i32), _i32, _P(_i32)],
    "mg_decode_step": [_vp, _P(_i32), _i32, _P(C.c_uint8), _f32, _vp, _vp, _vp],
    "mg_stats": [_vp, _P(MgStats)],
    "mg_set_policy": [_vp, _i32, _i32, _i32],
    "mgd_set_inject": [_vp, _f32, _u64],
    "mgd_gemm_top2": [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "mgd_force_schedule": [_vp, _i32],
    "mg_verify_window": [_vp, _vp, _i32, _vp, _vp, _vp],
    "mg_release": [_vp, _i32],
    "mg_destroy": [_vp],
    "mg_last_error": [_vp],
    "mgd_gen_tensor": [_u64, _u32, _i64, _i32, _i32, _vp, _vp],
    "mgd_rmsnorm": [_vp, _vp, _i32, _i32, _f32, _vp, _vp],
    "mgd_gemm": [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp],
    "mgd_qkv_epilogue": [_vp, _i32, _vp, _vp, _i32, _i32, _i32, _i32, _f32, _i32, _vp, _vp, _vp, _vp],
    "mgd_attention": [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp],
    "mgd_attention_streams": [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp],
    "mgd_launch_floor": [_i32, _i32, _vp, _vp],
    "mgd_residual": [_vp, _vp, _i32, _i32, _i32, _vp, _vp],
    "mgd_swiglu": [_vp, _i32, _i32, _i32, _vp, _vp],
    "mgd_top2": [_vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "mgd_gate": [_vp, _vp, _i32, _f32, _vp, _vp, _vp, _vp],
    "mgd_read_column": [_vp, _i32, _i32, _i32, _vp],
    "mgd_cache_digest": [_vp, _i32, _i32, _i32, _P(_u64)],
    "mgd_last_step": [_vp] + [_vp] * 9,
    "mgd_capture_logits": [_vp, _vp],
    "mgd_weight": [_vp, _i32, _i32, _vp, _P(_i64)],
    "mgd_schedule": [_vp, _i32, _i32, _i32, _P(_i32)],
    "mgd_launch_count": [_vp, _P(_u64)],
    "mgd_set_timing": [_vp, _i32],
    "mgd_timing": [_vp, _P(C.c_double)],
    "mgd_capture_verifier_logits": [_vp, _vp],
}


def lib():
    """Load libmargingate.so (built in-tree by `make` / __graft_entry__.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} missing: run `make` (or __graft_entry__.build()); "
                                   "there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = C.c_char_p if name == "mg_last_error" else (None if name == "mg_destroy" else C.c_int)
            _lib = L
    return _lib


def check(status: int, ctx=None, what: str = ""):
    if status != MG_OK:
        msg = lib().mg_last_error(ctx)
        raise MgError(status, f"{what}: {msg.decode() if msg else ''}")
