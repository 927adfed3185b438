"""GPU parity of the SURVEY 8(f) NEXT rows through the C ABI.

* NEXT-2 windowed verify + rollback (mg_verify_window; PAPER.md:227, 251,
  255): the verified output equals the GPU's own tau=inf run bit for bit
  (both are the deterministic path over the same prefix) and the oracle's
  window verifier, teacher-forced on the GPU's unverified tokens, rolls back
  at the same positions to the same tokens (exact wherever the argmax bound
  of PAPER.md:203 makes the verifier token unique).
* NEXT-4 global batch-invariant fast schedule: tau=0 decode is
  bit-identical across batch sizes and equals the tau=inf run.
* NEXT-3 repair-action ablation: token-only repair keeps the
  BF16 column; under reading A1 tau=inf still emits the reference.
* Pipelined verification (MG_VERIFY_PIPELINED, include/mg.h): the gated rows'
  verifier rides on the next step's weight pass; the committed sequences are
  bit-identical to the synchronous mode's (a row's fast path does not depend
  on the other rows), with and without the long-catch-up fallback.
"""
import numpy as np
import pytest

from paper_2605_30218_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = 2e-2
BAND = 2 * TOL
INF = float("inf")


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


@pytest.fixture(scope="module")
def tiny(orc):
    shp = inputs.shape("tiny")
    return shp, orc.Model(shp)


def _engine(shape, B, max_seq=128, page_size=16, verify_chunk=0):
    from paper_2605_30218_b200.engine import Engine
    return Engine(shape, max_batch=B, max_slots=B, max_seq=max_seq, page_size=page_size, verify_chunk=verify_chunk)


def _decode(torch, eng, prompts, steps, tau, prot=None):
    B = len(prompts)
    seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    for _ in range(steps - 1):
        eng.step(list(range(B)), prot, tau, out)
        o = out.cpu().numpy()
        for b in range(B):
            seqs[b].append(int(o[b]))
    return seqs


def _windowed(torch, eng, prompts, K, target, trace=None):
    """tau=0 steps in windows of K + mg_verify_window on every row until each
    row holds `target` verified tokens.  trace: list receiving, per window,
    (unverified sequences before the verify, verify results)."""
    B = len(prompts)
    P = [len(p) for p in prompts]
    seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    while min(len(s) for s in seqs) < target:
        for _ in range(K):
            eng.step(list(range(B)), None, 0.0, out)
            o = out.cpu().numpy()
            for b in range(B):
                seqs[b].append(int(o[b]))
        before = [list(s) for s in seqs]
        pos, last, rb = eng.verify_window(list(range(B)))
        for b in range(B):
            n = pos[b] - P[b] + 1
            assert rb[b] == len(seqs[b]) - n
            seqs[b] = seqs[b][:n]
            seqs[b][-1] = int(last[b])
        if trace is not None:
            trace.append((before, (pos.copy(), last.copy(), rb.copy())))
    return seqs


def _det_margin(orc, m, prefix):
    """Oracle reference margin of the next token after `prefix`."""
    st = orc.State(m, 1, len(prefix) + 2)
    _, lg = st.prefill(0, prefix, orc.det_sched(), want_logits=True)
    st.close()
    return float(orc.top2(lg)["g"][0])


@pytest.mark.parametrize("K", [1, 5, 16])
def test_window_verify_equals_tau_inf(torch, tiny, K):
    shp, _ = tiny
    B, target = 6, 40
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=12), shp["vocab"], seed=300)
    ref = _decode(torch, _engine(shp, B), prompts, target, INF)
    eng = _engine(shp, B)
    win = _windowed(torch, eng, prompts, K, target)
    for b in range(B):
        assert win[b][:target] == ref[b], (K, b)
    st = eng.stats()
    assert st["window_rows"] > 0 and st["rollbacks"] <= st["window_rows"]
    assert st["triggers"] == 0  # windows only: the per-step gate never ran
    eng.close()


def test_window_rollback_matches_oracle(orc, torch, tiny):
    """Oracle window verifier teacher-forced on the GPU's unverified tokens:
    same rollback position, token and count per row (exact outside the
    argmax-ambiguity band of the oracle reference margin)."""
    shp, m = tiny
    B, K = 6, 12
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=13), shp["vocab"], seed=310)
    eng = _engine(shp, B)
    trace = []
    _windowed(torch, eng, prompts, K, 3 * K, trace)
    eng.close()
    det = orc.det_sched()
    st = orc.State(m, B, 160)
    for i, p in enumerate(prompts):
        st.prefill(i, p, det)
    checked = 0
    stop = False
    for before, (pos, last, rb) in trace:
        if stop:
            break
        # teacher-force the oracle's fast cache + history with the GPU's unverified tokens
        P0 = [st.pos(b) for b in range(B)]
        for k in range(K):
            forced = np.array([before[b][P0[b] - len(prompts[b]) + 1 + k] for b in range(B)], np.int32)
            st.step(np.arange(B), np.zeros(B, np.uint8), 0.0, orc.fast_sched(B), det,
                    forced_trig=np.zeros(B, np.uint8), forced_out=forced, forced_kind=np.zeros(B, np.uint8))
        opos, olast, orb = st.verify_window(np.arange(B), det)
        for b in range(B):
            if (opos[b], olast[b], orb[b]) == (pos[b], last[b], rb[b]):
                checked += 1
                continue
            # allowed only where the reference token at the first differing point is ambiguous
            q = min(opos[b], pos[b])
            prefix = list(prompts[b]) + before[b][:q - len(prompts[b]) + 1]
            assert _det_margin(orc, m, prefix[:q]) <= BAND, (b, opos[b], pos[b])
            stop = True   # the trajectories legitimately part here: the comparison ends
            break
    assert checked >= B
    st.close()


def test_batch_invariant_fast_schedule(torch, tiny):
    """mg_set_policy(MG_FAST_BATCH_INVARIANT): pure BF16 decode (tau=0, no
    verifier) is bit-identical at batch 1 and 8 and equals the tau=inf run --
    the global-intervention baseline of PAPER.md:227."""
    shp, _ = tiny
    prompts = inputs.prompts(8, inputs.ragged_lengths(8, 8, 23, seed=21), shp["vocab"], seed=330)
    steps = 32
    ref = _decode(torch, _engine(shp, 8), prompts, steps, INF)
    for B in (1, 8):
        got = []
        for i0 in range(0, 8, B):
            eng = _engine(shp, B)
            eng.set_policy(fast_schedule=1)
            got += _decode(torch, eng, prompts[i0:i0 + B], steps, 0.0)
            assert eng.stats()["triggers"] == 0
            eng.close()
        assert got == ref, B


def test_token_only_repair_gpu(torch, tiny):
    """PAPER.md:317 ablation on the GPU: with token-only repair the emitted
    tokens at tau=inf are still the reference (reading A1); with column
    repair every repaired fast column equals the verifier's shadow column,
    with token-only repair none is written (the columns are the BF16 path's)."""
    shp, _ = tiny
    B, steps = 8, 40
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=31), shp["vocab"], seed=340)
    runs = {}
    for mode in (0, 1):
        eng = _engine(shp, B)
        eng.set_policy(repair_action=mode)
        seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        repaired = []
        for _ in range(steps - 1):
            pos = [len(prompts[b]) + len(seqs[b]) - 1 for b in range(B)]
            eng.step(list(range(B)), None, INF, out)
            r = eng.last_step(B)
            o = out.cpu().numpy()
            for b in range(B):
                seqs[b].append(int(o[b]))
                if r["kind"][b] == 2:
                    repaired.append((b, pos[b]))
        same = [np.array_equal(eng.read_column(0, b, p), eng.read_column(1, b, p)) for b, p in repaired]
        runs[mode] = (seqs, repaired, same, eng.stats())
        eng.close()
    assert runs[0][0] == runs[1][0]
    assert all(runs[0][2])                      # column repair: fast column p == verifier column p
    assert runs[0][3]["repairs"] == len(runs[0][1])


def test_policy_and_window_errors(torch, tiny):
    from paper_2605_30218_b200 import _lib
    shp, _ = tiny
    eng = _engine(shp, 2)
    L = _lib.lib()
    assert L.mg_set_policy(eng.ctx, 2, 0, 0) == _lib.MG_ERR_INVALID
    assert L.mg_set_policy(eng.ctx, 0, 7, 0) == _lib.MG_ERR_INVALID
    assert L.mg_set_policy(eng.ctx, 0, 0, 5) == _lib.MG_ERR_INVALID
    s = np.array([0], np.int32)
    assert L.mg_verify_window(eng.ctx, s.ctypes.data, 1, None, None, None) == _lib.MG_ERR_INVALID  # inactive
    eng.prefill(0, [1, 2, 3])
    s2 = np.array([0, 0], np.int32)
    assert L.mg_verify_window(eng.ctx, s2.ctypes.data, 2, None, None, None) == _lib.MG_ERR_INVALID  # duplicate
    assert L.mg_verify_window(eng.ctx, s.ctypes.data, 0, None, None, None) == _lib.MG_ERR_INVALID
    # nothing unverified: a no-op that reports the current position
    pos, last, rb = eng.verify_window([0])
    assert pos[0] == 3 and rb[0] == 0
    eng.close()


def _pipelined(torch, eng, prompts, steps, tau, prot=None, recs=None):
    """Pipelined decode: kinds 0/1/3 append, kind 4 replaces the slot's last
    token (include/mg.h).  Ends with mg_verify_window to resolve the last
    tentative tokens."""
    from paper_2605_30218_b200.engine import VERIFY_PIPELINED
    B = len(prompts)
    eng.set_policy(verify_mode=VERIFY_PIPELINED)
    seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    kind = torch.empty(B, dtype=torch.uint8, device="cuda")
    for _ in range(steps - 1):
        eng.step(list(range(B)), prot, tau, out, kind)
        o, k = out.cpu().numpy(), kind.cpu().numpy()
        if recs is not None:
            recs.append(k.copy())
        for b in range(B):
            if k[b] == 4:
                seqs[b][-1] = int(o[b])
            else:
                seqs[b].append(int(o[b]))
    pos, last, rb = eng.verify_window(list(range(B)))
    for b in range(B):
        n = int(pos[b]) - len(prompts[b]) + 1
        del seqs[b][n:]
        seqs[b][-1] = int(last[b])
    return seqs


@pytest.mark.parametrize("tau,prot_mode,vc", [(INF, "all", 0), (0.3, "half", 0), (0.3, "all", 16), (INF, "all", 16)])
def test_pipelined_equals_sync(torch, tiny, tau, prot_mode, vc):
    shp, _ = tiny
    B, steps = 6, 40
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=41), shp["vocab"], seed=350)
    prot = inputs.protected_mask(B, prot_mode)
    ref = _decode(torch, _engine(shp, B, verify_chunk=vc), prompts, steps, tau, prot)
    eng = _engine(shp, B, verify_chunk=vc)
    recs = []
    got = _pipelined(torch, eng, prompts, steps, tau, prot, recs)
    st = eng.stats()
    for b in range(B):
        n = min(len(got[b]), len(ref[b]))
        assert n >= steps // 2
        assert got[b][:n] == ref[b][:n], b
    kinds = np.array(recs)
    assert (kinds == 4).sum() == st["repairs"]
    assert st["triggers"] >= st["verified"] + st["repairs"]
    if tau == INF:
        assert (kinds == 3).all() or ((kinds == 3) | (kinds == 4)).all()
    eng.close()


def test_pipelined_errors(torch, tiny):
    from paper_2605_30218_b200 import _lib
    shp, _ = tiny
    eng = _engine(shp, 2)
    eng.set_policy(verify_mode=1)
    for i in range(2):
        eng.prefill(i, [3 + i, 4, 5, 6])
    out = torch.empty(2, dtype=torch.int32, device="cuda")
    eng.step([0, 1], None, INF, out)          # both rows tentative now
    from paper_2605_30218_b200._lib import MgError
    with pytest.raises(MgError):
        eng.step([0], None, INF, out)         # slot 1 pending but missing
    L = _lib.lib()
    assert L.mg_set_policy(eng.ctx, 0, 0, 0) == _lib.MG_ERR_STATE
    eng.verify_window([0, 1])
    assert L.mg_set_policy(eng.ctx, 0, 0, 0) == _lib.MG_OK
    eng.close()


@pytest.mark.parametrize("tau,prot_mode,vc", [(INF, "all", 0), (0.3, "half", 0), (0.3, "all", 16), (0.0, "all", 0)])
def test_fused_equals_sync(torch, tiny, tau, prot_mode, vc):
    """MG_VERIFY_FUSED (include/mg.h): the verifier rides on the same step's
    weight pass; tokens, kinds and the gate/repair counters are identical to
    the synchronous mode at every step (with the long-catch-up fallback at
    verify_chunk 16)."""
    shp, _ = tiny
    B, steps = 6, 32
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=43), shp["vocab"], seed=360)
    prot = inputs.protected_mask(B, prot_mode)
    runs = []
    for mode in (0, 2):
        eng = _engine(shp, B, verify_chunk=vc)
        eng.set_policy(verify_mode=mode)
        seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        kind = torch.empty(B, dtype=torch.uint8, device="cuda")
        kinds = []
        for _ in range(steps - 1):
            eng.step(list(range(B)), prot, tau, out, kind)
            o = out.cpu().numpy()
            kinds.append(kind.cpu().numpy().copy())
            for b in range(B):
                seqs[b].append(int(o[b]))
        st = eng.stats()
        runs.append((seqs, np.array(kinds), {k: st[k] for k in ("triggers", "verified", "repairs", "protected_rows")}))
        eng.close()
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
    assert runs[0][2] == runs[1][2]


def test_injected_noise_matches_oracle(orc, torch, tiny):
    """mgd_set_inject (SURVEY 8(b) test-only export): the GPU adds
    the oracle's documented perturbation bit for bit, so with real forced
    flips the GPU's per-step margins, fast tokens and gate decisions replay
    through the oracle (teacher-forced on the GPU's committed tokens and kinds)
    within the logit tolerance; repairs fire; at batch 1 the noise is zero."""
    shp, m = tiny
    B, steps, amp, seed, tau = 4, 12, 0.5, 9, 0.3
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 20, seed=8), shp["vocab"], seed=370)
    prot = inputs.protected_mask(B, "all")
    eng = _engine(shp, B)
    eng.set_inject(amp, seed)
    first = [eng.prefill(i, p) for i, p in enumerate(prompts)]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    kind = torch.empty(B, dtype=torch.uint8, device="cuda")
    det = orc.det_sched()
    st = orc.State(m, B, 64)
    if [st.prefill(i, p, det) for i, p in enumerate(prompts)] != first:
        pytest.skip("prefill token inside the ambiguity band")
    fs = orc.fast_sched(B, noise_amp=amp, noise_seed=seed)
    rep = checked = kinds_checked = 0
    for _ in range(steps):
        eng.step(list(range(B)), prot, tau, out, kind)
        r = eng.last_step(B)
        o = out.cpu().numpy()
        # teacher-forced on the GPU's committed tokens and gate decisions (so
        # both sides verify the same rows); the oracle takes its OWN verifier
        # token and commit kind (nothing else is forced)
        ro = st.step(np.arange(B), prot, tau, fs, det, forced_trig=r["trig"], forced_out=o)
        for b in range(B):
            assert abs(float(r["g"][b]) - float(ro["g"][b])) <= BAND, (b, r["g"][b], ro["g"][b])
            f_unique = ro["g"][b] > BAND
            if f_unique:
                assert r["f_tok"][b] == ro["f_tok"][b]
                checked += 1
            if abs(float(ro["g"][b]) - tau) > BAND:
                assert bool(r["trig"][b]) == bool(ro["g"][b] < tau)
            if r["trig"][b] and ro["v_g"][b] > BAND:         # the verifier token is unique
                assert int(r["v_tok"][b]) == int(ro["v_tok"][b]), b
                if f_unique:
                    assert int(r["kind"][b]) == int(ro["kind"][b]), b
                    kinds_checked += 1
        rep += int((r["kind"] == 2).sum())
    assert rep > 0 and checked > B * steps // 2 and kinds_checked > 0
    eng.close()
    st.close()
    # batch 1: the perturbation is exactly zero
    seqs = []
    for a in (0.0, amp):
        e1 = _engine(shp, 1)
        e1.set_inject(a, seed)
        seqs.append(_decode(torch, e1, prompts[:1], 10, 0.0)[0])
        e1.close()
    assert seqs[0] == seqs[1]


def test_force_schedule_reproduces_batch_shape(torch, tiny):
    """mgd_force_schedule: a row decoded alone with the attention splits of
    batch 8 gives bit-identical fast logits to the same row inside a batch of
    8 (the GEMMs are column-invariant), i.e. a controlled batch-shape flip
    source without changing the batch."""
    shp, _ = tiny
    V = shp["vocab"]
    prompts = inputs.prompts(8, inputs.ragged_lengths(8, 8, 23, seed=51), shp["vocab"], seed=380)
    caps = []
    for B, force in ((8, 0), (1, 8)):
        eng = _engine(shp, B, max_seq=4096)   # capacity large enough that batch 1 and 8 split differently
        assert eng.schedule(1, False, 4096)["attn_chunk"] != eng.schedule(8, False, 4096)["attn_chunk"]
        eng.force_schedule(force)
        cap = torch.empty((B, V), dtype=torch.float32, device="cuda")
        eng.capture_logits(cap)
        for i, p in enumerate(prompts[:B]):
            eng.prefill(i, p)
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        lg = []
        for _ in range(4):
            eng.step(list(range(B)), None, 0.0, out)
            lg.append(cap[0].cpu().numpy().copy())
        caps.append(lg)
        eng.close()
    for a, b in zip(*caps):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("B,mode", [(6, 0), (6, 2), (1, 0)])
def test_fused_lm_top2_equals_logits_path(torch, tiny, B, mode):
    """The LM head's fused top-2 epilogue (per-tile top-2 in the tcgen05 GEMM
    epilogue, then a merge over the tiles) gives bit-identical (v1, i1, v2, i2,
    g) to the fp32-logits + top-2 kernels (MG_LM_UNFUSED=1), for the fast rows
    and the verifier rows: the top-2 under (value desc, id asc) is exact, so
    the merge order cannot matter."""
    import os
    shp, _ = tiny
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=61), shp["vocab"], seed=390)
    recs = []
    for unfused in ("1", "0"):
        os.environ["MG_LM_UNFUSED"] = unfused
        try:
            eng = _engine(shp, B)
        finally:
            del os.environ["MG_LM_UNFUSED"]
        eng.set_policy(verify_mode=mode)
        for i, p in enumerate(prompts):
            eng.prefill(i, p)
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        rr = []
        for _ in range(8):
            eng.step(list(range(B)), None, INF, out)
            r = eng.last_step(B)
            rr.append((r["f_tok"].copy(), r["g"].copy(), r["v1"].copy(), r["v2"].copy(), r["v_tok"].copy(),
                       r["v_g"].copy(), out.cpu().numpy().copy()))
        recs.append(rr)
        eng.close()
    for a, b in zip(*recs):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_slot_churn_tau_inf_is_reference(torch, tiny, mode):
    """Continuous batching: requests leave (mg_release) and new ones are
    prefilled into the freed slots while the others keep decoding; at tau=inf
    every request's committed sequence equals its own batch-1 reference in
    the synchronous, pipelined and fused verify modes (the verifier depends
    only on the request's prefix)."""
    shp, _ = tiny
    S, B, steps = 8, 5, 36
    reqs = inputs.prompts(12, inputs.ragged_lengths(12, 6, 20, seed=71), shp["vocab"], seed=400)
    eng = _engine(shp, S)
    eng.set_policy(verify_mode=mode)
    out = torch.empty(S, dtype=torch.int32, device="cuda")
    kind = torch.empty(S, dtype=torch.uint8, device="cuda")
    live, done, nxt = {}, {}, 0          # slot -> (request, sequence)
    for s in range(B):
        live[s] = (nxt, [eng.prefill(s, reqs[nxt])])
        nxt += 1
    for step in range(steps):
        slots = sorted(live)
        eng.step(slots, None, INF, out[:len(slots)], kind[:len(slots)])
        o, k = out.cpu().numpy(), kind.cpu().numpy()
        for j, s in enumerate(slots):
            seq = live[s][1]
            if mode == 1 and k[j] == 4:
                seq[-1] = int(o[j])
            else:
                seq.append(int(o[j]))
        if step % 6 == 5 and nxt < len(reqs):      # one request leaves, a new one joins a free slot
            s = slots[step // 6 % len(slots)]
            r, seq = live.pop(s)
            pos, last, _ = eng.verify_window([s])   # resolve a tentative token (pipelined) before leaving
            n = int(pos[0]) - len(reqs[r]) + 1
            done[r] = seq[:n - 1] + [int(last[0])]
            eng.release(s)
            free = [x for x in range(S) if x not in live and x != s]
            live[free[0]] = (nxt, [eng.prefill(free[0], reqs[nxt])])
            nxt += 1
    slots = sorted(live)
    pos, last, _ = eng.verify_window(slots)
    for j, s in enumerate(slots):
        r, seq = live[s]
        n = int(pos[j]) - len(reqs[r]) + 1
        done[r] = seq[:n - 1] + [int(last[j])]
    eng.close()
    for r, seq in done.items():
        e1 = _engine(shp, 1)
        ref = _decode(torch, e1, [reqs[r]], len(seq), INF)[0]
        e1.close()
        assert seq == ref, (mode, r)


@pytest.mark.parametrize("mode", [1, 2])
def test_changing_protection_mask_matches_sync(torch, tiny, mode):
    """Per-step protection masks that change (a row unprotected for a few steps
    then protected again, so its shadow cache catches up several positions in
    one launch): the fused and pipelined modes commit the synchronous mode's
    tokens (tau = 0.3, real triggers)."""
    shp, _ = tiny
    B, steps, tau = 6, 30, 0.3
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=91), shp["vocab"], seed=410)
    rng = np.random.default_rng(5)
    masks = [(rng.random(B) < 0.5).astype(np.uint8) for _ in range(steps - 1)]
    runs = []
    for m in (0, mode):
        eng = _engine(shp, B)
        eng.set_policy(verify_mode=m)
        seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        kind = torch.empty(B, dtype=torch.uint8, device="cuda")
        for t in range(steps - 1):
            eng.step(list(range(B)), masks[t], tau, out, kind)
            o, k = out.cpu().numpy(), kind.cpu().numpy()
            for b in range(B):
                if m == 1 and k[b] == 4:
                    seqs[b][-1] = int(o[b])
                else:
                    seqs[b].append(int(o[b]))
        if m == 1:
            pos, last, _ = eng.verify_window(list(range(B)))
            for b in range(B):
                n = int(pos[b]) - len(prompts[b]) + 1
                del seqs[b][n:]
                seqs[b][-1] = int(last[b])
        runs.append(seqs)
        eng.close()
    for b in range(B):
        n = min(len(runs[0][b]), len(runs[1][b]))
        assert n >= steps // 2 and runs[0][b][:n] == runs[1][b][:n], b
    if mode == 2:
        assert runs[0] == runs[1]


def test_pipelined_prefill_while_pending(torch, tiny):
    """a prefill into a never-used slot while other slots hold
    pending tentative tokens (no mg_verify_window in between) overwrites the
    device catch-up list the pipelined mode reuses; the next step must rebuild
    it.  At tau=inf every request's resolved sequence equals its batch-1
    reference and no false kind-4 replacement appears."""
    from paper_2605_30218_b200.engine import VERIFY_PIPELINED
    shp, _ = tiny
    S, steps = 6, 18
    reqs = inputs.prompts(S, inputs.ragged_lengths(S, 6, 20, seed=73), shp["vocab"], seed=420)
    eng = _engine(shp, S)
    eng.set_policy(verify_mode=VERIFY_PIPELINED)
    out = torch.empty(S, dtype=torch.int32, device="cuda")
    kind = torch.empty(S, dtype=torch.uint8, device="cuda")
    seqs = {s: [eng.prefill(s, reqs[s])] for s in range(4)}
    for step in range(steps):
        if step in (5, 11):                       # join while slots 0..3 (and later 4) are pending
            s = 4 if step == 5 else 5
            seqs[s] = [eng.prefill(s, reqs[s])]
        slots = sorted(seqs)
        eng.step(slots, None, INF, out[:len(slots)], kind[:len(slots)])
        o, k = out.cpu().numpy(), kind.cpu().numpy()
        for j, s in enumerate(slots):
            if k[j] == 4:
                seqs[s][-1] = int(o[j])
            else:
                seqs[s].append(int(o[j]))
    slots = sorted(seqs)
    pos, last, _ = eng.verify_window(slots)
    st = eng.stats()
    eng.close()
    for j, s in enumerate(slots):
        n = int(pos[j]) - len(reqs[s]) + 1
        seq = seqs[s][:n - 1] + [int(last[j])]
        e1 = _engine(shp, 1)
        ref = _decode(torch, e1, [reqs[s]], len(seq), INF)[0]
        e1.close()
        assert seq == ref, s
    # tau = inf: every decision of a protected row triggers (r_verify = 1)
    assert st["triggers"] == st["protected_rows"]
