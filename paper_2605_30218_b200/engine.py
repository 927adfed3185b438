"""Python front end of the MarginGate decode engine (include/mg.h).

torch is used only to allocate the device buffers the C ABI asks for and to
hand over the CUDA stream; every step of the path runs in libmargingate.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import MgBuffers, MgConfig, MgSizes, MgStats, check, lib

KIND_FAST, KIND_VERIFIED, KIND_REPAIR = 0, 1, 2
FAST_BATCH_SHAPED, FAST_BATCH_INVARIANT = 0, 1   # mg_fast_schedule
REPAIR_COLUMN, REPAIR_TOKEN_ONLY = 0, 1         # mg_repair_action
VERIFY_SYNC, VERIFY_PIPELINED = 0, 1            # mg_verify_mode
KIND_TENTATIVE, KIND_REPLACE = 3, 4             # pipelined-mode kinds


def make_config(shape: dict, max_batch: int, max_slots: int, max_seq: int, page_size: int = 64,
                verify_chunk: int = 0) -> MgConfig:
    return MgConfig(shape["n_layers"], shape["d_model"], shape["n_heads"], shape["n_kv_heads"], shape["head_dim"],
                    shape["d_ff"], shape["vocab"], int(shape.get("qkv_bias", 0)), shape["rms_eps"],
                    shape["rope_theta"], shape["weight_seed"], max_batch, max_slots, max_seq, page_size,
                    verify_chunk)


def query_sizes(cfg: MgConfig) -> dict:
    s = MgSizes()
    check(lib().mg_query_sizes(C.byref(cfg), C.byref(s)), None, "mg_query_sizes")
    return {"weights": s.weights, "kv_fast": s.kv_fast, "kv_shadow": s.kv_shadow, "workspace": s.workspace}


class Engine:
    """One MarginGate context on the current CUDA device."""

    def __init__(self, shape: dict, max_batch: int, max_slots: int | None = None, max_seq: int = 1024,
                 page_size: int = 64, verify_chunk: int = 0, stream=None):
        import torch
        self.torch = torch
        self.shape = dict(shape)
        self.max_batch = max_batch
        self.max_slots = max_slots or max_batch
        self.cfg = make_config(shape, max_batch, self.max_slots, max_seq, page_size, verify_chunk)
        self.sizes = query_sizes(self.cfg)
        dev = torch.device("cuda", torch.cuda.current_device())
        self._bufs = {k: torch.empty(max(v, 256), dtype=torch.uint8, device=dev) for k, v in self.sizes.items()}
        self.stream = stream or torch.cuda.current_stream()
        bufs = MgBuffers(*(self._bufs[k].data_ptr() for k in ("weights", "kv_fast", "kv_shadow", "workspace")))
        ctx = C.c_void_p()
        st = lib().mg_init(C.byref(self.cfg), C.byref(bufs), C.c_void_p(self.stream.cuda_stream), C.byref(ctx))
        check(st, None, "mg_init")
        self.ctx = ctx
        self.V = shape["vocab"]

    # ------------------------------------------------------------ product API
    def prefill(self, slot: int, prompt) -> int:
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        out = C.c_int32(0)
        check(lib().mg_prefill(self.ctx, slot, p.ctypes.data_as(C.POINTER(C.c_int32)), p.size, C.byref(out)),
              self.ctx, "mg_prefill")
        return int(out.value)

    def step(self, slots, protected, tau: float, tokens_out, kind_out=None, margin_out=None):
        """Enqueue one decode step; outputs are torch CUDA tensors (int32, uint8, float32)."""
        s = np.ascontiguousarray(slots, dtype=np.int32)
        pp = None
        if protected is not None:
            pa = np.ascontiguousarray(protected, dtype=np.uint8)
            pp = pa.ctypes.data_as(C.POINTER(C.c_uint8))
        st = lib().mg_decode_step(self.ctx, s.ctypes.data_as(C.POINTER(C.c_int32)), s.size, pp, float(tau),
                                  C.c_void_p(tokens_out.data_ptr()),
                                  C.c_void_p(kind_out.data_ptr()) if kind_out is not None else None,
                                  C.c_void_p(margin_out.data_ptr()) if margin_out is not None else None)
        check(st, self.ctx, "mg_decode_step")

    def stats(self) -> dict:
        s = MgStats()
        st = lib().mg_stats(self.ctx, C.byref(s))
        if st not in (_lib.MG_OK, _lib.MG_ERR_NUMERIC):
            check(st, self.ctx, "mg_stats")
        d = {k: int(getattr(s, k)) for k, _ in MgStats._fields_}
        d["nan"] = st == _lib.MG_ERR_NUMERIC
        return d

    def set_policy(self, fast_schedule: int | None = None, repair_action: int | None = None,
                   verify_mode: int | None = None):
        """mg_set_policy: fast_schedule 0 batch-shaped (default) / 1 batch-invariant
        (PAPER.md:227 global baseline); repair_action 0 column /
        1 token-only ablation; verify_mode 0 sync / 1 pipelined
        (include/mg.h MG_VERIFY_PIPELINED: kinds 3 tentative, 4 replace).
        None keeps the current value."""
        cur = getattr(self, "_policy", (0, 0, 0))
        new = tuple(int(v) if v is not None else c for v, c in zip((fast_schedule, repair_action, verify_mode), cur))
        check(lib().mg_set_policy(self.ctx, *new), self.ctx, "mg_set_policy")
        self._policy = new

    def verify_window(self, slots):
        """mg_verify_window (LLM-42-style verify + rollback, PAPER.md:227, 251,
        255).  Returns (pos, last_token, rolled_back) numpy arrays per slot."""
        s = np.ascontiguousarray(slots, dtype=np.int32)
        n = s.size
        pos, last, rb = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.int32)
        check(lib().mg_verify_window(self.ctx, s.ctypes.data, n, pos.ctypes.data, last.ctypes.data, rb.ctypes.data),
              self.ctx, "mg_verify_window")
        return pos, last, rb

    def release(self, slot: int):
        check(lib().mg_release(self.ctx, slot), self.ctx, "mg_release")

    def close(self):
        if getattr(self, "ctx", None):
            lib().mg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ debug hooks
    def read_column(self, which: int, slot: int, pos: int) -> np.ndarray:
        sh = self.shape
        out = np.empty((sh["n_layers"], 2, sh["n_kv_heads"], sh["head_dim"]), np.uint16)
        check(lib().mgd_read_column(self.ctx, which, slot, pos, out.ctypes.data), self.ctx, "mgd_read_column")
        return out

    def digest(self, which: int, skip_slot: int = -1, skip_pos: int = -1) -> int:
        h = C.c_uint64(0)
        check(lib().mgd_cache_digest(self.ctx, which, skip_slot, skip_pos, C.byref(h)), self.ctx, "digest")
        return int(h.value)

    def last_step(self, B: int) -> dict:
        r = dict(f_tok=np.empty(B, np.int32), g=np.empty(B, np.float32), v1=np.empty(B, np.float32),
                 v2=np.empty(B, np.float32), trig=np.empty(B, np.uint8), v_tok=np.empty(B, np.int32),
                 v_g=np.empty(B, np.float32), kind=np.empty(B, np.uint8), out=np.empty(B, np.int32))
        check(lib().mgd_last_step(self.ctx, *(r[k].ctypes.data for k in ("f_tok", "g", "v1", "v2", "trig", "v_tok",
                                                                           "v_g", "kind", "out"))),
              self.ctx, "mgd_last_step")
        return r

    def set_inject(self, amp: float, seed: int = 0):
        """Test-only SPEC.md:76-84 logit noise on the fast rows (mg_debug.h)."""
        check(lib().mgd_set_inject(self.ctx, float(amp), int(seed)), self.ctx, "mgd_set_inject")

    def force_schedule(self, B_as_if: int):
        """Test-only: fast attention splits of batch size B_as_if (0: off)."""
        check(lib().mgd_force_schedule(self.ctx, int(B_as_if)), self.ctx, "mgd_force_schedule")

    def capture_logits(self, buf):
        check(lib().mgd_capture_logits(self.ctx, C.c_void_p(buf.data_ptr()) if buf is not None else None),
              self.ctx, "capture")

    def capture_verifier_logits(self, buf):
        """Debug: verifier fp32 logits of the gated rows of the next steps into
        buf [max_batch, vocab] (rank order, include/mg_debug.h); None stops."""
        check(lib().mgd_capture_verifier_logits(self.ctx, C.c_void_p(buf.data_ptr()) if buf is not None else None),
              self.ctx, "capture_verifier_logits")

    def weight(self, layer: int, which: int):
        n = C.c_int64(0)
        check(lib().mgd_weight(self.ctx, layer, which, None, C.byref(n)), self.ctx, "mgd_weight")
        t = self.torch.empty(max(n.value, 1), dtype=self.torch.int16, device="cuda")
        check(lib().mgd_weight(self.ctx, layer, which, C.c_void_p(t.data_ptr()), C.byref(n)), self.ctx, "mgd_weight")
        return t[: n.value].cpu().numpy().view(np.uint16)

    def schedule(self, T: int, det: bool, max_ctx: int) -> dict:
        o = (C.c_int32 * 8)()
        check(lib().mgd_schedule(self.ctx, T, int(det), max_ctx, o), self.ctx, "mgd_schedule")
        keys = ["split_qkv", "split_o", "split_gu", "split_down", "split_lm", "attn_chunk", "impl", "mma_n"]
        return dict(zip(keys, list(o)))

    def launches(self) -> int:
        n = C.c_uint64(0)
        check(lib().mgd_launch_count(self.ctx, C.byref(n)), self.ctx, "launch count")
        return int(n.value)

    def set_timing(self, on: bool):
        check(lib().mgd_set_timing(self.ctx, int(on)), self.ctx, "set_timing")

    def timing(self) -> dict:
        o = (C.c_double * 8)()
        check(lib().mgd_timing(self.ctx, o), self.ctx, "timing")
        return dict(gemm_ms=o[0], gemm_launches=int(o[1]), gemm_bytes=o[2], attn_ms=o[3], attn_launches=int(o[4]),
                    step_ms=o[5], steps=int(o[6]))
