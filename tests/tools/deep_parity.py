"""Full-depth oracle parity past 512 keys (diagnostic; the result is committed
to profiles/r02_deep_parity_llama8b.json).

Llama-3.1-8B shape (32 layers, full vocabulary) at batch 64 with prompts of
513-560 tokens: the fast attention takes one split per (token, kv head)
while the verifier pins 512-key splits, so the two GPU plans differ.  One
sampled row (the shortest prompt) is recomputed by the CPU oracle,
teacher-forced on the GPU's committed tokens, twice (the oracle's batch-shaped
plan A and its pinned plan D), for `steps` decode steps at tau = +inf; the
GPU's fast logits are compared with A and its verifier logits with D within
max(2e-2, 2 x the pooled |A - D| spread), tokens exactly
outside the PAPER.md:203 band.  The oracle needs ~30 minutes of 16-core CPU
time per plan at this depth, so this runs outside the pytest suite.

usage: python tests/tools/deep_parity.py [steps] > profiles/r02_deep_parity_llama8b.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as orc  # noqa: E402
from paper_2605_30218_b200 import inputs  # noqa: E402
from paper_2605_30218_b200.engine import Engine  # noqa: E402

TOL = 2e-2
INF = float("inf")


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    shp = inputs.shape("llama8b")
    B, V = 64, shp["vocab"]
    lengths = inputs.ragged_lengths(B, 513, 560, seed=99)
    prompts = inputs.prompts(B, lengths, V, seed=6000)
    row = int(np.argmin(lengths))
    eng = Engine(shp, max_batch=B, max_slots=B, max_seq=max(lengths) + steps + 4, page_size=64)
    capf = torch.empty((B, V), dtype=torch.float32, device="cuda")
    capv = torch.empty((B, V), dtype=torch.float32, device="cuda")
    eng.capture_logits(capf)
    eng.capture_verifier_logits(capv)
    first = [eng.prefill(i, p) for i, p in enumerate(prompts)]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    toks, fl, vl, vt, vg = [first[row]], [], [], [], []
    for _ in range(steps):
        eng.step(list(range(B)), None, INF, out)          # every row protected: verifier rank == row
        torch.cuda.synchronize()
        r = eng.last_step(B)
        toks.append(int(out[row].item()))
        fl.append(capf[row].cpu().numpy().copy())
        vl.append(capv[row].cpu().numpy().copy())
        vt.append(int(r["v_tok"][row]))
        vg.append(float(r["v_g"][row]))
    sched = eng.schedule(B, False, max(lengths) + steps + 4)
    eng.close()
    del capf, capv
    torch.cuda.empty_cache()

    t0 = time.time()
    m = orc.Model(shp)
    det = orc.det_sched()
    plen = len(prompts[row])
    A = orc.State(m, 1, plen + steps + 2)
    D = orc.State(m, 1, plen + steps + 2)
    ya, la = A.prefill(0, prompts[row], det, want_logits=True)
    D.prefill(0, prompts[row], det)
    res = {"model": "llama8b (32 layers, vocab 128256)", "batch": B, "row": row, "prompt_len": plen,
           "gpu_fast_attention_plan": sched, "verifier_split_keys": 512,
           "first_token_equal": ya == first[row], "first_token_margin": float(orc.top2(la)["g"][0]), "steps": []}
    if ya != first[row]:
        res["note"] = "first token inside the argmax band: the trajectories differ, no teacher forcing possible"
        print(json.dumps(res))
        return
    ras, rds = [], []
    for t in range(steps):
        kw = dict(forced_trig=[1], forced_out=[toks[t + 1]], want_logits=True)
        ras.append(A.step([0], [1], INF, orc.fast_sched(B), det, **kw))
        rds.append(D.step([0], [1], INF, det, det, **kw))
    noise = np.concatenate([np.abs(a["logits"][0] - d["logits"][0]) for a, d in zip(ras, rds)])
    q_tol = max(TOL, 2 * float(np.quantile(noise, 0.999)))
    m_tol = max(TOL, 2 * float(noise.max()))
    ok = True
    for t in range(steps):
        ef = np.abs(fl[t] - ras[t]["logits"][0])
        ev = np.abs(vl[t] - rds[t]["logits"][0])
        st = {"ctx": plen + t + 1,
              "fast_vs_oracle": {"p999": float(np.quantile(ef, 0.999)), "max": float(ef.max())},
              "verifier_vs_oracle": {"p999": float(np.quantile(ev, 0.999)), "max": float(ev.max())},
              "oracle_spread": {"p999": float(np.quantile(np.abs(ras[t]["logits"][0] - rds[t]["logits"][0]), 0.999)),
                                "max": float(np.abs(ras[t]["logits"][0] - rds[t]["logits"][0]).max())},
              "fast_token": {"gpu": int(np.argmax(fl[t])), "oracle": int(ras[t]["f_tok"][0]),
                             "oracle_margin": float(ras[t]["g"][0])},
              "verifier_token": {"gpu": vt[t], "oracle": int(rds[t]["v_tok"][0]), "oracle_margin": float(rds[t]["v_g"][0])}}
        within = (st["fast_vs_oracle"]["p999"] <= q_tol and st["fast_vs_oracle"]["max"] <= m_tol and
                  st["verifier_vs_oracle"]["p999"] <= q_tol and st["verifier_vs_oracle"]["max"] <= m_tol)
        fast_tok_ok = st["fast_token"]["gpu"] == st["fast_token"]["oracle"] or \
            st["fast_token"]["oracle_margin"] <= 2 * m_tol
        ver_tok_ok = vt[t] == st["verifier_token"]["oracle"] or st["verifier_token"]["oracle_margin"] <= 2 * m_tol
        st["within_bound"] = bool(within)
        st["tokens_ok_outside_band"] = bool(fast_tok_ok and ver_tok_ok)
        ok = ok and within and fast_tok_ok and ver_tok_ok
        res["steps"].append(st)
    res["bound"] = {"p999": q_tol, "max": m_tol, "rule": "max(2e-2, 2 x pooled oracle A-D spread), DESIGN.md 9"}
    res["pass"] = bool(ok)
    res["oracle_seconds"] = round(time.time() - t0, 1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
