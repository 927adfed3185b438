"""Per-phase timeline of one layer-chain launch (diagnostic only).

usage: python scripts/chain_trace.py [model] [B] [ctx] [layer]
Columns per phase: first stage landed / last MMA / partials out / barrier-1
passed / op done / barrier-2 passed (B producer of the next phase), each as
median and max over CTAs, in us from the earliest CTA entry.
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
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 384
layer = int(sys.argv[4]) if len(sys.argv) > 4 else 10
shp = inputs.shape(model)
eng = Engine(shp, max_batch=B, max_seq=ctx + 64, page_size=64)
for i, p in enumerate(inputs.prompts(B, ctx, shp["vocab"])):
    eng.prefill(i, p)
eng.chain_trace(layer)
out = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(5):
    eng.step(list(range(B)), None, 0.0, out)
torch.cuda.synchronize()
tr = eng.chain_trace(layer, read=True)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
names = ["first-stage", "last-mma", "partials-out", "barrier1", "op-done", "barrier2(B)"]
print(f"{len(tr)} CTAs; entry spread {(tr[:, 0].max() - t0) / 1e3:.2f} us")
for p in range(4):
    cols = tr[:, 1 + p * 6: 1 + p * 6 + 6]
    if not (cols > 0).any():
        continue
    cells = []
    for e in range(6):
        v = cols[:, e]
        v = v[v > 0]
        if len(v) == 0:
            cells.append(f"{names[e]} -")
            continue
        d = (v - t0) / 1e3
        cells.append(f"{names[e]} {np.median(d):7.2f}/{d.max():7.2f}")
    print(f"phase {p}: " + " | ".join(cells))
