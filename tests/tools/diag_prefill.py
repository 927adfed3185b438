"""Diagnostic: per-position / per-layer differences of the prefill shadow
columns, GPU vs oracle (tiny config)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle
from paper_2605_30218_b200 import inputs
from paper_2605_30218_b200.engine import Engine
shp = inputs.shape(sys.argv[1] if len(sys.argv) > 1 else "tiny")
m = oracle.Model(shp)
B = 6
prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 20, seed=5), shp["vocab"], seed=40)
eng = Engine(shp, max_batch=B, max_seq=96, page_size=16)
st = oracle.State(m, B, 96)
det = oracle.det_sched()
for i, p in enumerate(prompts):
    eng.prefill(i, p); st.prefill(i, p, det)
for i in (0, 5, 1):
    p = prompts[i]
    line = []
    for q in range(len(p)):
        a = eng.read_column(1, i, q).astype(np.uint16); b = st.column(1, i, q)
        line.append("/".join(str(int((a[l, kv] != b[l, kv]).sum())) for l in range(shp["n_layers"]) for kv in range(2)))
    print("row", i, "len", len(p), " ".join(line))
