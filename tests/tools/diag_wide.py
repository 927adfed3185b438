"""Per-row logit error of the wide config at a given batch, GPU vs oracle (teacher-forced)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle
from paper_2605_30218_b200 import inputs, kernels as K
from paper_2605_30218_b200.engine import Engine
# op-level: stream-K GEMM at tile 32
rng = np.random.default_rng(0)
for T, tile, G in ((24, 32, 148), (24, 32, 0), (20, 32, 37), (40, 64, 148)):
    x = oracle.f32_to_bf16(rng.standard_normal((T, 1024)).astype(np.float32))
    W = oracle.f32_to_bf16((rng.standard_normal((768, 1024)) / 32).astype(np.float32))
    part = K.gemm(x, W, splits=-G if G else 1, impl=0, tile_n=tile)
    if G:
        cnt = K.streamk_counts(768, 1024, G)
        y = part[0].copy()
        for s in range(1, part.shape[0]):
            for m, cc in enumerate(cnt):
                if s < cc: y[:, 128*m:128*(m+1)] += part[s][:, 128*m:128*(m+1)]
    else:
        y = part[0]
    ref = oracle.gemm(x, W, 1)
    print("gemm T", T, "tile", tile, "G", G, "max err per row", np.round(np.abs(y - ref).max(1), 5).tolist())
shp = inputs.shape(sys.argv[1] if len(sys.argv) > 1 else "wide")
B = int(sys.argv[2]) if len(sys.argv) > 2 else 24
m = oracle.Model(shp)
prompts = inputs.prompts(B, inputs.ragged_lengths(B, 5, 12, seed=B), shp["vocab"], seed=600)
eng = Engine(shp, max_batch=B, max_seq=32, page_size=16)
cap = torch.empty((B, shp["vocab"]), dtype=torch.float32, device="cuda")
eng.capture_logits(cap)
st = oracle.State(m, B, 32)
det = oracle.det_sched()
y0 = [eng.prefill(i, p) for i, p in enumerate(prompts)]
y0o = [st.prefill(i, p, det) for i, p in enumerate(prompts)]
print("prefill agree", sum(a == b for a, b in zip(y0, y0o)), "/", B)
out = torch.empty(B, dtype=torch.int32, device="cuda")
eng.step(list(range(B)), None, 0.0, out)
o = out.cpu().numpy()
r = st.step(np.arange(B), np.zeros(B, np.uint8), 0.0, oracle.fast_sched(B), det, forced_out=o,
            forced_kind=np.zeros(B, np.uint8), want_logits=True)
e = np.abs(cap.cpu().numpy() - r["logits"])
print("row max err", np.round(e.max(1), 4).tolist())
print("schedule fast", eng.schedule(B, False, 32), "det", eng.schedule(B, True, 32))
