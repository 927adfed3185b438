"""Kernel timeline of pipelined decode steps via torch.profiler (CUPTI) -- diagnostic only.

usage: python scripts/timeline.py [model] [B] [ctx] [tau] [steps] [passes] > summary
Prints per kernel class: count, mean duration, and the mean gap between the
end of the previous kernel and the start of this one (the pipeline bubble).
passes = 2 (tau = inf, every row protected: a fast forward then a verifier
forward per step) labels the GEMMs and attention kernels F / V by forward.
"""
import collections
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30218_b200 import inputs  # noqa: E402
from paper_2605_30218_b200.engine import Engine  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "llama8b"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 384
tau = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
passes = int(sys.argv[6]) if len(sys.argv) > 6 else 1
shp = inputs.shape(model)
eng = Engine(shp, max_batch=B, max_seq=ctx + 64, page_size=64)
for i, p in enumerate(inputs.prompts(B, ctx, shp["vocab"])):
    eng.prefill(i, p)
out = torch.empty(B, dtype=torch.int32, device="cuda")
rows = list(range(B))
for _ in range(6):
    eng.step(rows, None, tau, out)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        eng.step(rows, None, tau, out)
    torch.cuda.synchronize()
fn = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(fn)
ev = json.load(open(fn))["traceEvents"]
ks = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
print(f"{len(ks)} kernels in {steps} steps; span {(ks[-1]['ts'] + ks[-1]['dur'] - ks[0]['ts']) / steps:.1f} us/step")
# critical-path accounting: each kernel is charged end(k) - end(k-1), the time
# it added to the stream (PDL lets a kernel START before its predecessor ends,
# so start-based durations overlap)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
prev_end = None
# GEMMs are labelled by their place in the step: 4 per layer (qkv, o, gate/up,
# down), then the LM head; a step starts at its k_embed
gi, gname = 0, ("qkv", "o", "gu", "down")
nl = shp["n_layers"]
ne = -1
for e in ks:
    n = e["name"].split("(")[0].replace("void ", "")[:34]
    if "k_embed" in n:
        gi = 0
        ne += 1
    tag = ("F", "V")[ne % 2] + " " if passes == 2 else ""
    if "k_gemm_tc" in n:
        n = f"{tag}{n[:26]} {gname[gi % 4] if gi < 4 * nl else 'lm'}"
        gi += 1
    elif "k_attn" in n:
        n = f"{tag}{n}"
    end = e["ts"] + e["dur"]
    a = agg[n]
    a[0] += 1
    a[1] += e["dur"]
    if prev_end is not None:
        a[2] += end - prev_end
    prev_end = max(prev_end or 0, end)
for n, a in sorted(agg.items(), key=lambda x: -x[1][2]):
    print(f"{n:36s} n={a[0]:5d} start-to-end {a[1] / a[0]:8.2f} us  end-to-end {a[2] / a[0]:7.2f} us  "
          f"= {a[2] / steps:8.1f} us/step")
print(f"sum end-to-end {sum(a[2] for a in agg.values()) / steps:.1f} us/step")
