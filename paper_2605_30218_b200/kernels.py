"""Op-level calls into libmargingate.so (include/mg_debug.h) on torch CUDA tensors.

Used by the parity tests to hold each hot-path kernel against the oracle on
identical inputs.  bf16 tensors travel as torch.int16 holding the bit
patterns (numpy uint16 on the host side).  Marshalling only.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib


def _t():
    import torch
    return torch


def to_dev_u16(a: np.ndarray):
    torch = _t()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint16).view(np.int16)).cuda()


def to_host_u16(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return C.c_void_p(_t().cuda.current_stream().cuda_stream)


def _sync():
    _t().cuda.synchronize()


def gen_tensor(seed, tid, n, kind, fan_in):
    torch = _t()
    out = torch.empty(n, dtype=torch.int16, device="cuda")
    check(lib().mgd_gen_tensor(seed, tid, n, kind, fan_in, _p(out), _stream()), None, "gen")
    _sync()
    return to_host_u16(out)


def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    torch = _t()
    T, d = x.shape
    xd, wd = to_dev_u16(x), to_dev_u16(w)
    out = torch.empty_like(xd)
    check(lib().mgd_rmsnorm(_p(xd), _p(wd), T, d, eps, _p(out), _stream()), None, "rmsnorm")
    _sync()
    return to_host_u16(out)


def streamk_counts(N: int, K: int, G: int) -> list[int]:
    """Pieces per 128-feature tile of the stream-K partition (include/mg_debug.h)."""
    KB, n_m = K // 64, N // 128
    W = n_m * KB
    owner = lambda w: ((w + 1) * G - 1) // W
    return [owner((m + 1) * KB - 1) - owner(m * KB) + 1 for m in range(n_m)]


def gemm(x: np.ndarray, W: np.ndarray, splits=1, impl=0, mma_n=0, tile_n=0, x_dev=None, w_dev=None):
    """Returns the fp32 partials [slots, T, N] (splits < 0: stream-K pieces,
    tile m's pieces in slots 0..streamk_counts()[m]-1, k order)."""
    torch = _t()
    T, K = x.shape
    N = W.shape[0]
    xd = x_dev if x_dev is not None else to_dev_u16(x)
    wd = w_dev if w_dev is not None else to_dev_u16(W)
    slots = splits if splits > 0 else max(streamk_counts(N, K, -splits))
    out = torch.full((slots, T, N), float("nan"), dtype=torch.float32, device="cuda")
    check(lib().mgd_gemm(_p(xd), _p(wd), T, N, K, splits, impl, mma_n, tile_n, _p(out), _stream()), None, "gemm")
    _sync()
    return out.cpu().numpy()


def qkv_epilogue(part: np.ndarray, bias, pos, H, KV, hd, theta):
    torch = _t()
    S, T, N = part.shape
    pd = torch.from_numpy(np.ascontiguousarray(part, dtype=np.float32)).cuda()
    bd = to_dev_u16(bias) if bias is not None else None
    posd = torch.from_numpy(np.ascontiguousarray(pos, dtype=np.int32)).cuda()
    q = torch.empty((T, H * hd), dtype=torch.int16, device="cuda")
    k = torch.empty((T, KV * hd), dtype=torch.int16, device="cuda")
    v = torch.empty((T, KV * hd), dtype=torch.int16, device="cuda")
    check(lib().mgd_qkv_epilogue(_p(pd), S, _p(bd), _p(posd), T, H, KV, hd, theta, int(np.max(pos)) + 1, _p(q), _p(k),
                                 _p(v), _stream()), None, "qkv")
    _sync()
    return to_host_u16(q), to_host_u16(k), to_host_u16(v)


def attention(q: np.ndarray, K: np.ndarray, V: np.ndarray, n_keys, split_keys: int, streams: int = 4):
    """q [T, H, hd]; K, V [T, KV, key_stride, hd] -> o [T, H*hd] (streamed form,
    splits of split_keys keys, `streams` key streams per split; include/mg_debug.h)."""
    torch = _t()
    T, H, hd = q.shape
    _, KVh, stride, _ = K.shape
    qd, kd, vd = to_dev_u16(q), to_dev_u16(K), to_dev_u16(V)
    nk = torch.from_numpy(np.ascontiguousarray(n_keys, dtype=np.int32)).cuda()
    o = torch.empty((T, H * hd), dtype=torch.int16, device="cuda")
    check(lib().mgd_attention_streams(_p(qd), _p(kd), _p(vd), _p(nk), T, H, KVh, hd, stride, split_keys, streams,
                                      _p(o), _stream()), None, "attention")
    _sync()
    return to_host_u16(o)


def residual(x: np.ndarray, part: np.ndarray):
    torch = _t()
    S, T, N = part.shape
    xd = to_dev_u16(x)
    pd = torch.from_numpy(np.ascontiguousarray(part, dtype=np.float32)).cuda()
    out = torch.empty_like(xd)
    check(lib().mgd_residual(_p(xd), _p(pd), S, T, N, _p(out), _stream()), None, "residual")
    _sync()
    return to_host_u16(out)


def swiglu(part: np.ndarray, F: int):
    torch = _t()
    S, T, N2 = part.shape
    pd = torch.from_numpy(np.ascontiguousarray(part, dtype=np.float32)).cuda()
    out = torch.empty((T, F), dtype=torch.int16, device="cuda")
    check(lib().mgd_swiglu(_p(pd), S, T, F, _p(out), _stream()), None, "swiglu")
    _sync()
    return to_host_u16(out)


def top2(logits: np.ndarray):
    torch = _t()
    T, V = logits.shape
    ld = torch.from_numpy(np.ascontiguousarray(logits, dtype=np.float32)).cuda()
    f = lambda dt: torch.empty(T, dtype=dt, device="cuda")
    v1, v2, g = f(torch.float32), f(torch.float32), f(torch.float32)
    i1, i2 = f(torch.int32), f(torch.int32)
    nan = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(lib().mgd_top2(_p(ld), T, V, _p(v1), _p(i1), _p(v2), _p(i2), _p(g), _p(nan), _stream()), None, "top2")
    _sync()
    return dict(v1=v1.cpu().numpy(), i1=i1.cpu().numpy(), v2=v2.cpu().numpy(), i2=i2.cpu().numpy(),
                g=g.cpu().numpy(), nan=bool(nan.item()))


def gemm_top2(x: np.ndarray, W: np.ndarray, tile_n=0):
    """LM head with the fused top-2 epilogue (include/mg_debug.h mgd_gemm_top2)."""
    torch = _t()
    T, K = x.shape
    N = W.shape[0]
    xd, wd = to_dev_u16(x), to_dev_u16(W)
    f = lambda dt: torch.empty(T, dtype=dt, device="cuda")
    v1, v2, g = f(torch.float32), f(torch.float32), f(torch.float32)
    i1, i2 = f(torch.int32), f(torch.int32)
    nan = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(lib().mgd_gemm_top2(_p(xd), _p(wd), T, N, K, tile_n, _p(v1), _p(i1), _p(v2), _p(i2), _p(g), _p(nan),
                              _stream()), None, "gemm_top2")
    _sync()
    return dict(v1=v1.cpu().numpy(), i1=i1.cpu().numpy(), v2=v2.cpu().numpy(), i2=i2.cpu().numpy(),
                g=g.cpu().numpy(), nan=bool(nan.item()))


def gate(g: np.ndarray, prot: np.ndarray, tau: float):
    torch = _t()
    B = g.size
    gd = torch.from_numpy(np.ascontiguousarray(g, dtype=np.float32)).cuda()
    pd = torch.from_numpy(np.ascontiguousarray(prot, dtype=np.uint8)).cuda()
    trig = torch.empty(B, dtype=torch.uint8, device="cuda")
    rows = torch.empty(B, dtype=torch.int32, device="cuda")
    cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    check(lib().mgd_gate(_p(gd), _p(pd), B, float(tau), _p(trig), _p(rows), _p(cnt), _stream()), None, "gate")
    _sync()
    n = int(cnt.item())
    return trig.cpu().numpy(), rows.cpu().numpy()[:n]
