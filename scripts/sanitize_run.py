"""A short decode of the tiny config in every verify mode, for
compute-sanitizer (memcheck / racecheck / synccheck) -- diagnostic only.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py
Runs: prefill of 4 ragged prompts; 8 synchronous steps at tau = 0.3 with real
triggers (the whole-step CUDA graph with conditional nodes from the second
step on), then at tau = inf; 6 fused and 6 pipelined steps; a window verify;
multi-split attention (verify_chunk 16, contexts > 64 keys)."""
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
print("SANITIZE RUN OK")
