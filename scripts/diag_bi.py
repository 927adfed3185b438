"""Diagnostic: batch-invariant fast schedule (tau=0) vs the synchronous
always-on verifier (tau=inf): first divergence per row and the logit gap there."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_30218_b200 import inputs  # noqa: E402
from paper_2605_30218_b200.engine import Engine  # noqa: E402

name = sys.argv[1]
B, P, steps = 8, int(sys.argv[3]) if len(sys.argv) > 3 else 376, 40
for cap in [int(x) for x in sys.argv[2].split(",")]:
    shp = inputs.shape(name)
    eng = Engine(shp, max_batch=B, max_slots=B, max_seq=cap, page_size=64)
    prompts = inputs.prompts(B, P, shp["vocab"], seed=7)
    V = shp["vocab"]
    res = {}
    for mode, tau in (("bi", 0.0), ("ao", float("inf"))):
        eng.set_policy(fast_schedule=1 if mode == "bi" else 0)
        for i in range(B):
            try:
                eng.release(i)
            except Exception:
                pass
        cap_buf = torch.empty((B, V), dtype=torch.float32, device="cuda")
        if mode == "bi":
            eng.capture_logits(cap_buf)
        else:
            eng.capture_verifier_logits(cap_buf)
        seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        lg = []
        for _ in range(steps):
            eng.step(list(range(B)), None, tau, out)
            o = out.cpu().numpy()
            for b in range(B):
                seqs[b].append(int(o[b]))
            lg.append(cap_buf.cpu().numpy().copy())
        eng.capture_logits(None)
        eng.capture_verifier_logits(None)
        res[mode] = (seqs, lg)
    eng.set_policy(0)
    for b in range(B):
        a, r = res["bi"][0][b], res["ao"][0][b]
        d = next((i for i in range(len(a)) if a[i] != r[i]), None)
        t = 0 if d is None else d - 1
        diff = float(np.abs(res["bi"][1][t][b] - res["ao"][1][t][b]).max())
        print(f"{name} cap={cap} row {b}: first divergence {d}, max|dlogit| at step {t}: {diff:.3g}", flush=True)
    d0 = [float(np.abs(res["bi"][1][0][b] - res["ao"][1][0][b]).max()) for b in range(B)]
    print(f"{name} cap={cap} step0 max|dlogit| per row: {d0}", flush=True)
    eng.close()
