"""A short decode of the tiny config in every verify mode, for
compute-sanitizer (memcheck / racecheck / synccheck) -- diagnostic only.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py
Runs: prefill of 4 ragged prompts; 8 synchronous steps at tau = 0.3 with real
triggers (the whole-step CUDA graph with conditional nodes from the second
step on), then at tau = inf; 6 fused and 6 pipelined steps; a window verify;
multi-split attention (verify_chunk 16, contexts > 64 keys); the small-grid
(4, 4) attention rings (these grids have < 1 CTA per SM); and the fast path's
2-stream attention CTAs through mgd_attention_streams (hd 128 and 64, one
and several splits)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30218_b200 import inputs  # noqa: E402
from paper_2605_30218_b200.engine import Engine  # noqa: E402

shp = inputs.shape("tiny")
B = 4
prompts = inputs.prompts(B, inputs.ragged_lengths(B, 60, 90, seed=3), shp["vocab"], seed=77)
out = torch.empty(B, dtype=torch.int32, device="cuda")
kind = torch.empty(B, dtype=torch.uint8, device="cuda")
for mode in (0, 2, 1):
    eng = Engine(shp, max_batch=B, max_seq=160, page_size=16, verify_chunk=16)
    eng.set_policy(verify_mode=mode)
    for i, p in enumerate(prompts):
        eng.prefill(i, p)
    prot = [1, 0, 1, 1]
    for t in range(8):
        eng.step(list(range(B)), prot, 0.3 if t < 5 else float("inf"), out, kind)
    eng.verify_window(list(range(B)))
    st = eng.stats()
    torch.cuda.synchronize()
    print("mode", mode, st)
    eng.close()
import numpy as np  # noqa: E402

from paper_2605_30218_b200 import kernels as K  # noqa: E402

rng = np.random.default_rng(5)
for H, KVh, hd, sk, nk in ((32, 8, 128, 512, (1, 37, 700)), (4, 4, 64, 64, (5, 130, 300))):
    T, stride = len(nk), max(nk)
    kv = rng.standard_normal((T, KVh, stride, hd)).astype(np.float32)
    k16 = (kv.view(np.uint32) >> 16).astype(np.uint16)
    q16 = (rng.standard_normal((T, H, hd)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    K.attention(q16, k16, k16, np.array(nk, np.int32), sk, streams=2)
torch.cuda.synchronize()
print("SANITIZE RUN OK")
