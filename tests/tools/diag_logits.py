"""Diagnostic: distribution of |GPU fast logits - oracle logits| per decode
step (teacher-forced), tiny config.  Prints one line per step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
from paper_2605_30218_b200 import inputs  # noqa: E402
from paper_2605_30218_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 6
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
shp = inputs.shape(name)
m = oracle.Model(shp)
prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 20, seed=5), shp["vocab"], seed=40)
eng = Engine(shp, max_batch=B, max_seq=96, page_size=16)
cap = torch.empty((B, shp["vocab"]), dtype=torch.float32, device="cuda")
eng.capture_logits(cap)
st = oracle.State(m, B, 96)
det = oracle.det_sched()
for i, p in enumerate(prompts):
    a = eng.prefill(i, p)
    b, lg = st.prefill(i, p, det, want_logits=True)
    print("prefill", i, a, b, "oracle margin", float(oracle.top2(lg)["g"][0]))
for i, p in enumerate(prompts):
    for q in range(len(p)):
        c_gpu = eng.read_column(1, i, q).astype(np.uint16)
        c_or = st.column(1, i, q)
        d = np.abs(oracle.bf16_to_f32(c_gpu).astype(np.float64) - oracle.bf16_to_f32(c_or))
        if q in (0, len(p) - 1):
            print(f"shadow col row {i} pos {q}: differing elems {(c_gpu != c_or).sum()}/{c_gpu.size} max {d.max():.3g}")
out = torch.empty(B, dtype=torch.int32, device="cuda")
for t in range(steps):
    eng.step(list(range(B)), None, 0.0, out)
    o = out.cpu().numpy()
    r = st.step(np.arange(B), np.zeros(B, np.uint8), 0.0, oracle.fast_sched(B), det, forced_out=o,
                forced_kind=np.zeros(B, np.uint8), want_logits=True)
    e = np.abs(cap.cpu().numpy().astype(np.float64) - r["logits"])
    mag = np.abs(r["logits"]).max()
    print(f"step {t}: max {e.max():.4g} p99.9 {np.quantile(e, 0.999):.3g} mean {e.mean():.3g} "
          f">1e-3 {(e > 1e-3).sum()} |l|max {mag:.3g} rows_max {np.round(e.max(1), 4).tolist()}")
