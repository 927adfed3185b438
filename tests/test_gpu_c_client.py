"""The C ABI used from plain C (examples/mg_decode.c): caller-owned cudaMalloc
buffers, mg_init / mg_prefill / mg_decode_step / mg_stats / mg_destroy, no
Python or torch in the process.  The program checks its own results (tau=inf:
the protected request identical alone vs in a batch of 8; stats invariants)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_client_runs():
    exe = os.path.join(ROOT, "examples", "mg_decode")
    if not os.path.exists(exe):
        subprocess.check_call(["make", "-C", ROOT, "examples/mg_decode"])
    r = subprocess.run([exe, "16"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok: protected request identical alone vs in a batch of 8" in r.stdout
