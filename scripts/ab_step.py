"""A/B timing of the fast decode step (tau = 0) -- diagnostic only.

usage: [MG_LIB_PATH=...] python scripts/ab_step.py [model] [B] [ctx] [steps] [reps] [tau]
Prints the median ms/step over `reps` runs of `steps` back-to-back steps
(CUDA events on the engine stream), same prompts every time.
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30218_b200 import inputs  # noqa: E402
from paper_2605_30218_b200.engine import Engine  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "llama8b"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 384
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 16
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
tau = float(sys.argv[6]) if len(sys.argv) > 6 else 0.0
shp = inputs.shape(model)
eng = Engine(shp, max_batch=B, max_seq=ctx + reps * (steps + 4) + 16, page_size=64)
for i, p in enumerate(inputs.prompts(B, ctx, shp["vocab"])):
    eng.prefill(i, p)
out = torch.empty(B, dtype=torch.int32, device="cuda")
rows = list(range(B))
ms = []
for r in range(reps):
    for _ in range(4):
        eng.step(rows, None, tau, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    for _ in range(steps):
        eng.step(rows, None, tau, out)
    b.record(eng.stream)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b) / steps)
print(f"{os.environ.get('MG_LIB_PATH', 'current')}: {statistics.median(ms):.4f} ms/step  "
      f"({B / statistics.median(ms) * 1e3:.0f} tok/s)  all {[round(m, 4) for m in ms]}")
