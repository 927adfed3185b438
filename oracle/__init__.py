"""CPU oracle for the MarginGate decode hot path (arxiv 2605.30218).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2605_30218_b200``) never imports it and
shares no code with it.

This module is argument marshalling (ctypes + numpy) around
``oracle/mg_oracle.c``; all arithmetic lives in the C file, each function of
which cites the PAPER.md passage it follows.  bf16 values travel as uint16 bit
patterns.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "mg_oracle.c")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
          "-Wall", "-Wno-unused-function"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, IEEE fp32)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "mg_oracle.h"))):
        tmp = _SO + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class Cfg(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ff", C.c_int32),
                ("vocab", C.c_int32), ("qkv_bias", C.c_int32), ("rms_eps", C.c_float),
                ("rope_theta", C.c_float), ("weight_seed", C.c_uint64)]


class Sched(C.Structure):
    _fields_ = [("split_qkv", C.c_int32), ("split_o", C.c_int32), ("split_gu", C.c_int32),
                ("split_down", C.c_int32), ("split_lm", C.c_int32), ("attn_chunk", C.c_int32),
                ("attn_splits", C.c_int32), ("noise_amp", C.c_float), ("noise_seed", C.c_uint64)]


def _P(t):
    return C.POINTER(t)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            u16p, i32p, f32p, u8p, u64p = _P(C.c_uint16), _P(C.c_int32), _P(C.c_float), _P(C.c_uint8), _P(C.c_uint64)
            sig = {
                "or_f32_to_bf16": (C.c_uint16, [C.c_float]),
                "or_bf16_to_f32": (C.c_float, [C.c_uint16]),
                "or_dot_bf16": (C.c_float, [u16p, u16p, C.c_int32, C.c_int32]),
                "or_splitmix64": (C.c_uint64, [C.c_uint64]),
                "or_tensor_id": (C.c_uint32, [_P(Cfg), C.c_int32, C.c_int32]),
                "or_gen_tensor": (None, [C.c_uint64, C.c_uint32, C.c_int64, C.c_int32, C.c_int32, u16p]),
                "or_rmsnorm": (None, [u16p, u16p, C.c_int32, C.c_int32, C.c_float, u16p]),
                "or_gemm": (None, [u16p, u16p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, f32p]),
                "or_rope_table": (None, [C.c_int32, C.c_float, C.c_int32, f32p, f32p]),
                "or_qkv_epilogue": (None, [f32p, u16p, i32p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_float, u16p, u16p, u16p]),
                "or_attention": (None, [u16p, u16p, u16p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, C.c_int32, u16p]),
                "or_residual": (None, [u16p, f32p, C.c_int64, u16p]),
                "or_swiglu": (None, [f32p, f32p, C.c_int64, u16p]),
                "or_top2": (None, [f32p, C.c_int32, C.c_int32, f32p, i32p, f32p, i32p, f32p, i32p]),
                "or_gate": (C.c_int32, [f32p, u8p, C.c_int32, C.c_float, i32p]),
                "or_model_create": (C.c_void_p, [_P(Cfg)]),
                "or_model_free": (None, [C.c_void_p]),
                "or_model_tensor": (u16p, [C.c_void_p, C.c_int32, C.c_int32, _P(C.c_int64)]),
                "or_state_create": (C.c_void_p, [C.c_void_p, C.c_int32, C.c_int32]),
                "or_state_free": (None, [C.c_void_p]),
                "or_prefill": (C.c_int32, [C.c_void_p, C.c_int32, i32p, C.c_int32, _P(Sched), f32p]),
                "or_step": (C.c_int32, [C.c_void_p, i32p, C.c_int32, u8p, C.c_float, _P(Sched), _P(Sched),
                                        u8p, i32p, u8p, i32p, f32p, f32p, f32p, u8p, i32p, f32p, u8p, i32p,
                                        f32p]),
                "or_state_pos": (C.c_int32, [C.c_void_p, C.c_int32]),
                "or_state_shadow_len": (C.c_int32, [C.c_void_p, C.c_int32]),
                "or_state_token": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32]),
                "or_state_column": (None, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, u16p]),
                "or_state_digest": (C.c_uint64, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32]),
                "or_state_stats": (None, [C.c_void_p, u64p]),
                "or_state_set_repair_mode": (None, [C.c_void_p, C.c_int32]),
                "or_verify_window": (C.c_int32, [C.c_void_p, i32p, C.c_int32, _P(Sched), i32p, i32p, i32p]),
                "or_state_window_stats": (None, [C.c_void_p, u64p]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _ptr(a: np.ndarray | None, ct):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle needs C-contiguous arrays"
    return a.ctypes.data_as(_P(ct))


def u16(a):
    return _ptr(a, C.c_uint16)


def i32(a):
    return _ptr(a, C.c_int32)


def f32(a):
    return _ptr(a, C.c_float)


def u8(a):
    return _ptr(a, C.c_uint8)


# ----------------------------------------------------------------- numerics
def f32_to_bf16(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    f = lib().or_f32_to_bf16
    return np.fromiter((f(float(v)) for v in x.ravel()), dtype=np.uint16, count=x.size).reshape(x.shape)


def bf16_to_f32(h) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint16)
    return (h.astype(np.uint32) << 16).view(np.float32)


def dot_bf16(a, b, splits=1) -> float:
    a = np.ascontiguousarray(a, dtype=np.uint16)
    b = np.ascontiguousarray(b, dtype=np.uint16)
    return float(lib().or_dot_bf16(u16(a), u16(b), a.size, splits))


def make_cfg(shape: dict) -> Cfg:
    return Cfg(shape["n_layers"], shape["d_model"], shape["n_heads"], shape["n_kv_heads"], shape["head_dim"],
               shape["d_ff"], shape["vocab"], int(shape.get("qkv_bias", 0)), shape["rms_eps"],
               shape["rope_theta"], shape["weight_seed"])


def make_sched(split_qkv=1, split_o=1, split_gu=1, split_down=1, split_lm=1, attn_chunk=0, attn_splits=1,
               noise_amp=0.0, noise_seed=0) -> Sched:
    return Sched(split_qkv, split_o, split_gu, split_down, split_lm, attn_chunk, attn_splits, noise_amp,
                 noise_seed)


def gen_tensor(seed: int, tensor_id: int, n: int, kind: int, fan_in: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint16)
    lib().or_gen_tensor(seed, tensor_id, n, kind, fan_in, u16(out))
    return out


def tensor_id(shape: dict, layer: int, which: int) -> int:
    cfg = make_cfg(shape)
    return int(lib().or_tensor_id(C.byref(cfg), layer, which))


# ----------------------------------------------------------------- op level
def rmsnorm(x, w, eps):
    x = np.ascontiguousarray(x, dtype=np.uint16)
    w = np.ascontiguousarray(w, dtype=np.uint16)
    T, d = x.shape
    out = np.empty_like(x)
    lib().or_rmsnorm(u16(x), u16(w), T, d, eps, u16(out))
    return out


def gemm(x, W, splits=1):
    x = np.ascontiguousarray(x, dtype=np.uint16)
    W = np.ascontiguousarray(W, dtype=np.uint16)
    T, K = x.shape
    N = W.shape[0]
    out = np.empty((T, N), dtype=np.float32)
    lib().or_gemm(u16(x), u16(W), T, N, K, splits, f32(out))
    return out


def rope_table(hd, theta, pos):
    c = np.empty(hd // 2, np.float32)
    s = np.empty(hd // 2, np.float32)
    lib().or_rope_table(hd, theta, pos, f32(c), f32(s))
    return c, s


def qkv_epilogue(acc, bias, pos, H, KV, hd, theta):
    acc = np.ascontiguousarray(acc, dtype=np.float32)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    T = acc.shape[0]
    q = np.empty((T, H * hd), np.uint16)
    k = np.empty((T, KV * hd), np.uint16)
    v = np.empty((T, KV * hd), np.uint16)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.uint16)
    lib().or_qkv_epilogue(f32(acc), u16(b), i32(pos), T, H, KV, hd, theta, u16(q), u16(k), u16(v))
    return q, k, v


def attention(q, K, V, n_keys, chunk=0, splits=1):
    """q [H, hd]; K, V [KV, key_stride, hd] -> o [H*hd] (bf16 bits)."""
    q = np.ascontiguousarray(q, dtype=np.uint16)
    K = np.ascontiguousarray(K, dtype=np.uint16)
    V = np.ascontiguousarray(V, dtype=np.uint16)
    H, hd = q.shape
    KVh, stride, _ = K.shape
    o = np.empty(H * hd, np.uint16)
    lib().or_attention(u16(q), u16(K), u16(V), H, KVh, hd, n_keys, stride, chunk, splits, u16(o))
    return o


def residual(x, acc):
    x = np.ascontiguousarray(x, dtype=np.uint16)
    acc = np.ascontiguousarray(acc, dtype=np.float32)
    out = np.empty_like(x)
    lib().or_residual(u16(x), f32(acc), x.size, u16(out))
    return out


def swiglu(g, u):
    g = np.ascontiguousarray(g, dtype=np.float32)
    u = np.ascontiguousarray(u, dtype=np.float32)
    out = np.empty(g.shape, np.uint16)
    lib().or_swiglu(f32(g), f32(u), g.size, u16(out))
    return out


def top2(logits):
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    if logits.ndim == 1:
        logits = logits[None]
    T, V = logits.shape
    v1 = np.empty(T, np.float32); v2 = np.empty(T, np.float32); g = np.empty(T, np.float32)
    i1 = np.empty(T, np.int32); i2 = np.empty(T, np.int32)
    nan = C.c_int32(0)
    lib().or_top2(f32(logits), T, V, f32(v1), i32(i1), f32(v2), i32(i2), f32(g), C.byref(nan))
    return dict(v1=v1, i1=i1, v2=v2, i2=i2, g=g, nan=bool(nan.value))


def gate(g, prot, tau):
    g = np.ascontiguousarray(g, dtype=np.float32)
    prot = np.ascontiguousarray(prot, dtype=np.uint8)
    rows = np.empty(g.size, np.int32)
    n = lib().or_gate(f32(g), u8(prot), g.size, float(tau), i32(rows))
    return rows[:n].copy()


# ----------------------------------------------------------------- model + policy
class Model:
    """Oracle decoder with weights from the documented counter PRNG."""

    def __init__(self, shape: dict):
        self.shape = dict(shape)
        self.cfg = make_cfg(shape)
        self._h = lib().or_model_create(C.byref(self.cfg))

    def tensor(self, layer: int, which: int) -> np.ndarray:
        n = C.c_int64(0)
        p = lib().or_model_tensor(self._h, layer, which, C.byref(n))
        if n.value == 0:
            return np.empty(0, np.uint16)
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy()

    def close(self):
        if self._h:
            lib().or_model_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class State:
    """Per-row fast cache + shadow (deterministic) cache + committed history."""

    def __init__(self, model: Model, n_rows: int, max_seq: int):
        self.model = model
        self.n_rows, self.max_seq = n_rows, max_seq
        self._h = lib().or_state_create(model._h, n_rows, max_seq)

    def prefill(self, row: int, prompt, det: Sched, want_logits: bool = False):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        lg = np.empty(self.model.shape["vocab"], np.float32) if want_logits else None
        y0 = int(lib().or_prefill(self._h, row, i32(p), p.size, C.byref(det), f32(lg)))
        return (y0, lg) if want_logits else y0

    def step(self, rows, prot, tau, fast: Sched, det: Sched, forced_trig=None, forced_out=None,
             forced_kind=None, want_logits=False):
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        B = rows.size
        prot = np.ascontiguousarray(prot, dtype=np.uint8)
        ft = None if forced_trig is None else np.ascontiguousarray(forced_trig, dtype=np.uint8)
        fo = None if forced_out is None else np.ascontiguousarray(forced_out, dtype=np.int32)
        fk = None if forced_kind is None else np.ascontiguousarray(forced_kind, dtype=np.uint8)
        r = dict(f_tok=np.empty(B, np.int32), g=np.empty(B, np.float32), fv1=np.empty(B, np.float32),
                 fv2=np.empty(B, np.float32), trig=np.empty(B, np.uint8), v_tok=np.empty(B, np.int32),
                 v_g=np.empty(B, np.float32), kind=np.empty(B, np.uint8), out=np.empty(B, np.int32))
        logits = np.empty((B, self.model.shape["vocab"]), np.float32) if want_logits else None
        n = lib().or_step(self._h, i32(rows), B, u8(prot), float(tau), C.byref(fast), C.byref(det), u8(ft), i32(fo),
                          u8(fk), i32(r["f_tok"]), f32(r["g"]), f32(r["fv1"]), f32(r["fv2"]), u8(r["trig"]),
                          i32(r["v_tok"]), f32(r["v_g"]), u8(r["kind"]), i32(r["out"]), f32(logits))
        r["n_trig"] = int(n)
        if want_logits:
            r["logits"] = logits
        return r

    def pos(self, row):
        return int(lib().or_state_pos(self._h, row))

    def shadow_len(self, row):
        return int(lib().or_state_shadow_len(self._h, row))

    def token(self, row, q):
        return int(lib().or_state_token(self._h, row, q))

    def column(self, which, row, pos):
        s = self.model.shape
        out = np.empty((s["n_layers"], 2, s["n_kv_heads"], s["head_dim"]), np.uint16)
        lib().or_state_column(self._h, which, row, pos, u16(out))
        return out

    def digest(self, which, skip_row=-1, skip_pos=-1):
        return int(lib().or_state_digest(self._h, which, skip_row, skip_pos))

    def stats(self):
        out = np.zeros(9, np.uint64)
        lib().or_state_stats(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        keys = ["steps", "rows", "protected_rows", "triggers", "verified", "repairs", "verifier_launches",
                "catchup_tokens", "nan"]
        return {k: int(v) for k, v in zip(keys, out)}

    def set_repair_mode(self, mode: int):
        """0 column repair, 1 token-only ablation."""
        lib().or_state_set_repair_mode(self._h, int(mode))

    def verify_window(self, rows, det: Sched):
        """LLM-42-style windowed verify + rollback.
        Returns (new_pos, last_tok, rolled_back) per row."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        n = rows.size
        npos, last, rb = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.int32)
        lib().or_verify_window(self._h, i32(rows), n, C.byref(det), i32(npos), i32(last), i32(rb))
        return npos, last, rb

    def window_stats(self):
        out = np.zeros(3, np.uint64)
        lib().or_state_window_stats(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return {k: int(v) for k, v in zip(["window_rows", "rollbacks", "rolled_back_tokens"], out)}

    def close(self):
        if self._h:
            lib().or_state_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fast_sched(B: int, noise_amp: float = 0.0, noise_seed: int = 0) -> Sched:
    """The ORACLE's own batch-shaped reduction plan, SPEC.md:93 ("C =
    min(batch_size, 8)"): every dot product split in C chunks and attention
    keys cut in C equal chunks.  This is how the oracle exhibits the
    phenomenon of PAPER.md:35; it is not the GPU's schedule."""
    c = max(1, min(int(B), 8))
    return make_sched(c, c, c, c, c, 0, c, noise_amp, noise_seed)


def det_sched() -> Sched:
    """The oracle verifier's pinned plan: plain left-to-right sums, one
    attention chunk ("fixed deterministic kernels/settings")."""
    return make_sched(1, 1, 1, 1, 1, 0, 1)


def reference_decode(model: Model, prompt, n_tokens: int, max_seq: int | None = None):
    """Deterministic batch-invariant reference trajectory:
    greedy decode of the prompt alone with the pinned schedule, i.e. the
    tau=+inf run at batch 1."""
    prompt = list(prompt)
    st = State(model, 1, max_seq or (len(prompt) + n_tokens + 1))
    det = det_sched()
    toks = [st.prefill(0, prompt, det)]
    for _ in range(n_tokens - 1):
        r = st.step([0], [1], float("inf"), det, det)
        toks.append(int(r["out"][0]))
    st.close()
    return toks
