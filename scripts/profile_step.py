"""One MarginGate decode step under a profiler window (cudaProfilerStart/Stop).

usage: ncu --profile-from-start off ... python scripts/profile_step.py [model] [B] [tau] [ctx]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30218_b200 import inputs  # noqa: E402
from paper_2605_30218_b200.engine import Engine  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "llama8b"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
tau = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 384
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
shp = inputs.shape(model)
eng = Engine(shp, max_batch=B, max_seq=ctx + 16, page_size=64)
for i, p in enumerate(inputs.prompts(B, ctx, shp["vocab"])):
    eng.prefill(i, p)
out = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    eng.step(list(range(B)), None, tau, out)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(steps):
    eng.step(list(range(B)), None, tau, out)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done", out[:4].tolist())
