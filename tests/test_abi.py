"""The C-ABI library loads and exports every symbol include/*.h declares; the
host-side argument checks work without a GPU (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

from paper_2605_30218_b200 import _lib, inputs
from paper_2605_30218_b200.engine import make_config, query_sizes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mgd?_[a-z_0-9]+)\s*\(", txt)) - {"mg_status"})


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _declared("mg.h") + _declared("mg_debug.h")
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_lib.PUBLIC_SYMBOLS) == _declared("mg.h")
    assert sorted(_lib.DEBUG_SYMBOLS) == _declared("mg_debug.h")


def test_library_is_sm100a():
    """The fatbin carries sm_100a SASS with tcgen05 MMAs and TMA loads."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True,
                                       text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out


@pytest.mark.parametrize("name", ["tiny", "llama8b", "qwen14b", "dsr1_7b"])
def test_query_sizes(name):
    shp = inputs.shape(name)
    cfg = make_config(shp, 64, 64, 1024)
    s = query_sizes(cfg)
    # weights: the bf16 parameter count of the model (+ alignment)
    L, d, H, KV, hd, F, V = (shp[k] for k in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "d_ff",
                                              "vocab"))
    n = V * d * 2 + d + L * (2 * d + (H + 2 * KV) * hd * d + d * H * hd + 3 * F * d)
    if shp["qkv_bias"]:
        n += L * (H + 2 * KV) * hd
    assert n * 2 <= s["weights"] <= n * 2 + 256 * (16 * L + 8)
    assert s["kv_fast"] == s["kv_shadow"] >= L * 2 * KV * hd * 2 * 64 * 1024


def test_invalid_configs_rejected():
    shp = dict(inputs.shape("tiny"))
    for bad in [dict(head_dim=96), dict(d_model=200), dict(vocab=4000), dict(n_kv_heads=3)]:
        s = dict(shp, **bad)
        with pytest.raises(_lib.MgError) as e:
            query_sizes(make_config(s, 8, 8, 64))
        assert e.value.status == _lib.MG_ERR_INVALID
    with pytest.raises(_lib.MgError):
        query_sizes(make_config(shp, 0, 8, 64))
    with pytest.raises(_lib.MgError):
        query_sizes(make_config(shp, 8, 8, 64, page_size=48))


def test_init_rejects_null_buffers():
    shp = inputs.shape("tiny")
    cfg = make_config(shp, 8, 8, 64)
    bufs = _lib.MgBuffers(None, None, None, None)
    ctx = C.c_void_p()
    st = _lib.lib().mg_init(C.byref(cfg), C.byref(bufs), None, C.byref(ctx))
    assert st == _lib.MG_ERR_INVALID and not ctx.value
    assert b"null" in _lib.lib().mg_last_error(None)


def test_null_ctx_calls_are_invalid():
    L = _lib.lib()
    assert L.mg_stats(None, None) == _lib.MG_ERR_INVALID
    assert L.mg_release(None, 0) == _lib.MG_ERR_INVALID
    assert L.mg_decode_step(None, None, 1, None, 0.0, None, None, None) == _lib.MG_ERR_INVALID
    L.mg_destroy(None)  # no-op


def test_graft_entry_imports():
    """The driver's entry module parses and exposes build() / smoke()."""
    import importlib
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    m = importlib.import_module("__graft_entry__")
    assert callable(m.build) and callable(m.smoke)
