"""End-to-end parity of the CUDA decode engine (C ABI) against the oracle, and
the GPU path's own determinism (SURVEY 8(c) parity protocol steps 2-4).

Tolerance (BASELINE north_star): |delta logit| <= 2e-2.  Discrete outputs
are compared exactly wherever the paper's argmax bound makes them unique
(PAPER.md:203): tokens where the oracle margin g > 2 * 2e-2, gate decisions
where |g - tau| > 2 * 2e-2.  The verifier must be bit-identical to itself
across batch sizes (100% sequence-level determinism).
"""
import math

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


def _engine(shape, B, max_seq=96, page_size=16, verify_chunk=0, slots=None):
    from paper_2605_30218_b200.engine import Engine
    return Engine(shape, max_batch=B, max_slots=slots or B, max_seq=max_seq, page_size=page_size,
                  verify_chunk=verify_chunk)


def _decode(torch, eng, prompts, steps, tau, prot=None, record=False):
    B = len(prompts)
    seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    kind = torch.empty(B, dtype=torch.uint8, device="cuda")
    marg = torch.empty(B, dtype=torch.float32, device="cuda")
    recs = []
    for _ in range(steps - 1):
        eng.step(list(range(B)), prot, tau, out, kind, marg)
        o = out.cpu().numpy()
        for b in range(B):
            seqs[b].append(int(o[b]))
        if record:
            r = eng.last_step(B)
            r["kind_out"] = kind.cpu().numpy()
            r["margin_out"] = marg.cpu().numpy()
            recs.append(r)
    return seqs, recs


def _oracle_reference(orc, m, prompt, n):
    """Reference decode (tau=inf at batch 1) with the det margin of every emission."""
    st = orc.State(m, 1, len(prompt) + n + 2)
    det = orc.det_sched()
    y0, lg = st.prefill(0, prompt, det, want_logits=True)
    toks, gs = [y0], [float(orc.top2(lg)["g"][0])]
    for _ in range(n - 1):
        r = st.step([0], [1], INF, det, det)
        toks.append(int(r["out"][0]))
        gs.append(float(r["v_g"][0]))
    st.close()
    return toks, gs


def _check_logit_err(e, noise):
    """|delta logit| within max(2e-2, 2 x the oracle's own
    schedule-to-schedule noise) -- at p99.9 against the noise's p99.9 and at
    the max against its max.  `noise` = |oracle(batch-shaped plan) -
    oracle(pinned plan)| on the same teacher-forced prefixes: two valid fp32
    summation orders of the same model; the GPU's order is a third, so its
    distance to either is bounded by about twice their spread (bf16
    activation roundings turn reorder differences into occasional 1-ulp flips
    that propagate).  Callers pool e and noise over every sampled row and step
    of the test: the tail of the flip distribution is estimated from all of
    them, not from one step's sample.  A wrong index or dropped term gives
    O(1) errors."""
    q_tol = max(TOL, 2 * float(np.quantile(noise, 0.999)))
    m_tol = max(TOL, 2 * float(noise.max()))
    assert np.quantile(e, 0.999) <= q_tol, (float(np.quantile(e, 0.999)), q_tol)
    assert e.max() <= m_tol, (float(e.max()), m_tol)
    return m_tol


def _agree_until_band(gpu, ora, margins):
    """Tokens must match while the oracle margin is outside the ambiguity
    band; the first allowed mismatch ends the comparison (the trajectories
    then decode different continuations).  Returns #compared tokens."""
    for t, (a, b) in enumerate(zip(gpu, ora)):
        if a != b:
            assert margins[t] <= BAND, f"token {t}: gpu {a} != oracle {b} at margin {margins[t]}"
            return t
    return len(gpu)


@pytest.fixture(scope="module")
def tiny(orc):
    shp = inputs.shape("tiny")
    return shp, orc.Model(shp)


@pytest.fixture(scope="module")
def tiny_gqa(orc):
    shp = inputs.shape("tiny_gqa")
    return shp, orc.Model(shp)


@pytest.mark.parametrize("which", ["tiny", "tiny_gqa"])
def test_weights_bit_exact(orc, torch, tiny, tiny_gqa, which):
    shp, m = tiny if which == "tiny" else tiny_gqa
    eng = _engine(shp, 2)
    for layer, ws in [(-1, range(3))] + [(l, range(12)) for l in range(shp["n_layers"])]:
        for w in ws:
            assert np.array_equal(eng.weight(layer, w), m.tensor(layer, w)), (layer, w)
    eng.close()


@pytest.mark.parametrize("which", ["tiny", "tiny_gqa"])
def test_tau_inf_reference_and_batch_invariance(orc, torch, tiny, tiny_gqa, which):
    """tau=+inf (always-on verification) on the GPU: every row's sequence is
    bit-identical at batch 1, 3 and 8 (whatever shares the batch), and equals
    the oracle's deterministic reference outside the argmax-ambiguity band."""
    shp, m = tiny if which == "tiny" else tiny_gqa
    prompts = inputs.prompts(8, inputs.ragged_lengths(8, 8, 23), shp["vocab"])
    steps = 32
    runs = {}
    for B in (1, 3, 8):
        got = []
        for i0 in range(0, 8, B):
            group = prompts[i0:i0 + B]
            eng = _engine(shp, len(group))
            s, _ = _decode(torch, eng, group, steps, INF)
            st = eng.stats()
            assert st["triggers"] == st["protected_rows"] == len(group) * (steps - 1)   # r_verify = 1
            eng.close()
            got += s
        runs[B] = got[:8]
    assert runs[1] == runs[3] == runs[8]
    compared = 0
    for i, p in enumerate(prompts):
        toks, gs = _oracle_reference(orc, m, p, steps)
        compared += _agree_until_band(runs[1][i], toks, gs)
    assert compared >= 0.6 * 8 * steps   # most tokens are outside the band on random-init logits


def test_fast_logits_teacher_forced(orc, torch, tiny):
    """tau=0 (pure BF16 batched, r_verify=0): the fast logits the GPU
    captures stay within 2e-2 of the oracle's, teacher-forced on the GPU's
    tokens; the fast argmax agrees outside the band."""
    shp, m = tiny
    B, steps = 6, 12
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 20, seed=5), shp["vocab"], seed=40)
    eng = _engine(shp, B)
    cap = torch.empty((B, shp["vocab"]), dtype=torch.float32, device="cuda")
    eng.capture_logits(cap)
    st = orc.State(m, B, 64)
    sd = orc.State(m, B, 64)            # the same prefix under the pinned plan (self-noise)
    det = orc.det_sched()
    y0 = [eng.prefill(i, p) for i, p in enumerate(prompts)]
    y0o = [st.prefill(i, p, det) for i, p in enumerate(prompts)]
    for i, p in enumerate(prompts):
        sd.prefill(i, p, det)
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    for i in range(B):
        if y0[i] != y0o[i]:
            pytest.skip("prefill token inside the ambiguity band")
    errs, noises = [], []
    for _ in range(steps):
        eng.step(list(range(B)), None, 0.0, out)
        o = out.cpu().numpy()
        lg = cap.cpu().numpy()
        kw = dict(forced_out=o, forced_kind=np.zeros(B, np.uint8), want_logits=True)
        r = st.step(np.arange(B), np.zeros(B, np.uint8), 0.0, orc.fast_sched(B), det, **kw)
        rd = sd.step(np.arange(B), np.zeros(B, np.uint8), 0.0, det, det, **kw)
        e = np.abs(lg - r["logits"])
        errs.append(e)
        noises.append(np.abs(r["logits"] - rd["logits"]))
        for b in range(B):
            if r["g"][b] > 2 * e[b].max():      # argmax bound, per row
                assert o[b] == r["f_tok"][b]
    _check_logit_err(np.concatenate(errs), np.concatenate(noises))
    s = eng.stats()
    assert s["triggers"] == 0 and s["repairs"] == 0 and s["steps"] == steps
    eng.close()


def test_controller_replay_and_stats(orc, torch, tiny):
    """The GPU's per-step (g, f_tok, v_tok, prot, tau) replayed through the
    oracle's gate give exactly the GPU's trigger set; kinds and emitted tokens
    follow the commit rule; counters add up."""
    shp, m = tiny
    B, steps = 8, 24
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=9), shp["vocab"], seed=70)
    prot = inputs.protected_mask(B, "half")
    eng = _engine(shp, B)
    seqs, recs = _decode(torch, eng, prompts, steps, 0.3, prot=prot, record=True)
    n_trig = n_ver = n_rep = 0
    for r in recs:
        rows = orc.gate(r["g"], prot, 0.3)
        assert np.array_equal(np.nonzero(r["trig"])[0], rows)
        for b in range(B):
            k = int(r["kind"][b])
            assert k == int(r["kind_out"][b])
            assert r["margin_out"][b] == r["g"][b]
            if not r["trig"][b]:
                assert k == 0 and r["out"][b] == r["f_tok"][b]
            elif r["v_tok"][b] == r["f_tok"][b]:
                assert k == 1 and r["out"][b] == r["f_tok"][b]
            else:
                assert k == 2 and r["out"][b] == r["v_tok"][b]
        n_trig += int(r["trig"].sum())
        n_ver += int((r["kind"] == 1).sum())
        n_rep += int((r["kind"] == 2).sum())
    s = eng.stats()
    assert s["steps"] == steps - 1 and s["rows"] == B * (steps - 1)
    assert s["protected_rows"] == int(prot.sum()) * (steps - 1)
    assert (s["triggers"], s["verified"], s["repairs"]) == (n_trig, n_ver, n_rep)
    assert n_trig > 0
    eng.close()


def test_protected_row_deterministic_alone_vs_batched(torch, tiny):
    """The paper's protocol: the protected request gives the
    same sequence decoded alone and inside a batch, at a finite threshold,
    as long as the gate covers every flip; at tau=inf this holds by
    construction and must be exact."""
    shp, _ = tiny
    target = inputs.prompts(1, 12, shp["vocab"], seed=321)[0]
    alone, _ = _decode(torch, _engine(shp, 1), [target], 40, INF, prot=[1])
    for B in (2, 5, 8):
        others = inputs.prompts(B - 1, inputs.ragged_lengths(B - 1, 8, 23, seed=B), shp["vocab"], seed=1000 + B)
        prot = np.zeros(B, np.uint8)
        prot[B // 2] = 1
        batch = others[:B // 2] + [target] + others[B // 2:]
        seqs, _ = _decode(torch, _engine(shp, B), batch, 40, INF, prot=prot)
        assert seqs[B // 2] == alone[0]


def test_catchup_chunking_invariance_gpu(torch, tiny):
    """Verifier results do not depend on how the lazy catch-up is chunked
    (verify_chunk 16 vs 512) or how often it fires: shadow columns bit-equal."""
    shp, _ = tiny
    prompt = inputs.prompts(1, 40, shp["vocab"], seed=5)[0]
    cols = []
    for vc, tau in ((16, INF), (512, INF), (16, 1e-30)):
        eng = _engine(shp, 1, verify_chunk=vc)
        _decode(torch, eng, [prompt], 20, tau)
        if tau != INF:  # lazily catch up everything now
            out = torch.empty(1, dtype=torch.int32, device="cuda")
            eng.step([0], [1], INF, out)
        cols.append([eng.read_column(1, 0, q) for q in range(40 + 18)])
        eng.close()
    for q in range(40 + 18):
        assert np.array_equal(cols[0][q], cols[1][q]) and np.array_equal(cols[0][q], cols[2][q]), q


def test_repair_locality_gpu(torch, tiny):
    """Only column p of the stepped row changes in the fast cache; a repaired
    column equals the verifier's shadow column bit for bit."""
    shp, _ = tiny
    prompts = inputs.prompts(3, 10, shp["vocab"], seed=17)
    eng = _engine(shp, 3)
    for i, p in enumerate(prompts):
        eng.prefill(i, p)
    out = torch.empty(3, dtype=torch.int32, device="cuda")
    kind = torch.empty(3, dtype=torch.uint8, device="cuda")
    kinds = []
    for t in range(16):
        before = eng.digest(0)
        eng.step([0], [1], INF, out, kind)        # row 0 alone: only (0, p) may change
        p = 10 + t
        assert eng.digest(0, 0, p) == before
        k = int(kind[0].item())
        kinds.append(k)
        if k == 2:
            assert np.array_equal(eng.read_column(0, 0, p), eng.read_column(1, 0, p))
    assert set(kinds) <= {1, 2}
    eng.close()


def test_api_errors(torch, tiny):
    from paper_2605_30218_b200 import _lib
    shp, _ = tiny
    eng = _engine(shp, 2, max_seq=24, slots=3)
    out = torch.empty(2, dtype=torch.int32, device="cuda")
    with pytest.raises(_lib.MgError) as e:
        eng.step([0], None, 0.0, out)                  # inactive slot
    assert e.value.status == _lib.MG_ERR_INVALID
    eng.prefill(0, [1, 2, 3])
    eng.prefill(1, [4, 5])
    with pytest.raises(_lib.MgError) as e:
        eng.prefill(1, [4, 5])                         # already active
    assert e.value.status == _lib.MG_ERR_STATE
    for bad in (dict(slots=[0, 0]), dict(tau=-1.0), dict(tau=float("nan")), dict(slots=[0, 1, 2])):
        with pytest.raises(_lib.MgError) as e:
            eng.step(bad.get("slots", [0, 1]), None, bad.get("tau", 0.0), out)
        assert e.value.status == _lib.MG_ERR_INVALID
    with pytest.raises(_lib.MgError) as e:
        eng.prefill(2, [9999999])
    assert e.value.status == _lib.MG_ERR_INVALID
    with pytest.raises(_lib.MgError) as e:
        eng.prefill(2, list(range(30)))
    assert e.value.status == _lib.MG_ERR_CAPACITY
    # run slot 1 to max_seq: capacity error, no state change
    n = 0
    while True:
        try:
            eng.step([1], None, 0.0, out)
            n += 1
        except _lib.MgError as e2:
            assert e2.status == _lib.MG_ERR_CAPACITY
            break
    assert n == 24 - 2
    eng.release(1)
    eng.prefill(1, [7, 7])                             # slot reusable after release
    eng.step([0, 1], None, INF, out)
    eng.close()


@pytest.mark.slow
def test_wide_shallow_parity(orc, torch):
    """8B widths (d 4096, d_ff 14336, GQA 32/8, hd 128), 2 layers, full
    128256 vocabulary: tau=0 fast logits within 2e-2 teacher-forced at batch
    4 and 24 (tcgen05 token tiles 16 and 32), and the tau=inf sequence equals
    the oracle reference outside the band."""
    shp = inputs.shape("wide")
    m = orc.Model(shp)
    for B in (4, 24):
        prompts = inputs.prompts(B, inputs.ragged_lengths(B, 5, 12, seed=B), shp["vocab"], seed=600)
        eng = _engine(shp, B, max_seq=32)
        cap = torch.empty((B, shp["vocab"]), dtype=torch.float32, device="cuda")
        eng.capture_logits(cap)
        st = orc.State(m, B, 32)
        sd = orc.State(m, B, 32)        # pinned plan on the same prefix (self-noise)
        det = orc.det_sched()
        y0 = [eng.prefill(i, p) for i, p in enumerate(prompts)]
        pre = [st.prefill(i, p, det, want_logits=True) for i, p in enumerate(prompts)]
        for i, p in enumerate(prompts):
            sd.prefill(i, p, det)
        # a first token may differ only inside the argmax-ambiguity band; such a
        # row then consumes a different input token and is left out below
        same = np.array([a == b for a, (b, _) in zip(y0, pre)])
        for i in np.nonzero(~same)[0]:
            assert float(orc.top2(pre[i][1])["g"][0]) <= BAND, i
        assert same.sum() >= B - 2
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        errs, noises = [], []
        for _ in range(3):
            eng.step(list(range(B)), None, 0.0, out)
            o = out.cpu().numpy()
            kw = dict(forced_out=o, forced_kind=np.zeros(B, np.uint8), want_logits=True)
            r = st.step(np.arange(B), np.zeros(B, np.uint8), 0.0, orc.fast_sched(B), det, **kw)
            rd = sd.step(np.arange(B), np.zeros(B, np.uint8), 0.0, det, det, **kw)
            errs.append(np.abs(cap.cpu().numpy() - r["logits"])[same])
            noises.append(np.abs(r["logits"] - rd["logits"])[same])
        _check_logit_err(np.concatenate(errs), np.concatenate(noises))
        eng.close()
        st.close()
        sd.close()
    p = inputs.prompts(1, 9, shp["vocab"], seed=777)[0]
    eng = _engine(shp, 1, max_seq=32)
    seqs, _ = _decode(torch, eng, [p], 6, INF)
    toks, gs = _oracle_reference(orc, m, p, 6)
    assert _agree_until_band(seqs[0], toks, gs) >= 1
    eng.close()


@pytest.mark.parametrize("which,B", [("tiny", 6), ("wide", 4)])
def test_fast_path_equals_verifier_when_splits_agree(torch, which, B):
    """the fast GEMMs use the verifier's weight-shape-fixed
    stream-K partition and a token column's tcgen05 result does not depend on
    the MMA width, so whenever the attention splits also agree (here: short
    contexts, one split per token on both paths) the fast logits equal the
    verifier's logits bit for bit (tau=inf, all rows protected: verifier rank
    k = row k)."""
    shp = inputs.shape(which)
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 5, 12, seed=3), shp["vocab"], seed=900)
    eng = _engine(shp, B, max_seq=32)
    capf = torch.empty((B, shp["vocab"]), dtype=torch.float32, device="cuda")
    capv = torch.empty((B, shp["vocab"]), dtype=torch.float32, device="cuda")
    for i, p in enumerate(prompts):
        eng.prefill(i, p)
    eng.capture_logits(capf)
    eng.capture_verifier_logits(capv)
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    for _ in range(4):
        eng.step(list(range(B)), None, INF, out)
        assert torch.equal(capf, capv)
    st = eng.stats()
    assert st["repairs"] == 0 and st["triggers"] == st["protected_rows"] == 4 * B
    eng.close()


def test_sync_graph_dispatch_equals_eager(torch, tiny):
    """MG_VERIFY_SYNC runs each step as one CUDA graph whose verifier sits
    behind device-side conditions (WHILE over the catch-up chunks, SWITCH on
    the chunk size, IF on the LM head; include/mg.h): the committed tokens,
    kinds and counters equal the eager form's (the debug path with one host
    readback of the gate), with real triggers, changing protection masks and
    multi-token catch-ups (verify_chunk 16: several loop iterations) and a
    threshold that changes every step (uploaded with the batch, not baked
    into the graph)."""
    shp, _ = tiny
    B, steps = 6, 30
    prompts = inputs.prompts(B, inputs.ragged_lengths(B, 8, 23, seed=93), shp["vocab"], seed=430)
    rng = np.random.default_rng(7)
    masks = [(rng.random(B) < (0.15 if t % 7 else 0.9)).astype(np.uint8) for t in range(steps)]
    taus = [(0.3, 0.1, INF, 0.6)[t % 4] for t in range(steps)]   # a per-step threshold (read on the device)
    runs = []
    for eager in (True, False):
        eng = _engine(shp, B, verify_chunk=16)
        if eager:   # a logit capture forces the eager form
            cap = torch.empty((B, shp["vocab"]), dtype=torch.float32, device="cuda")
            eng.capture_logits(cap)
        seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        kind = torch.empty(B, dtype=torch.uint8, device="cuda")
        kinds = []
        for t in range(steps):
            eng.step(list(range(B)), masks[t], taus[t], out, kind)
            o = out.cpu().numpy()
            kinds.append(kind.cpu().numpy().copy())
            for b in range(B):
                seqs[b].append(int(o[b]))
        st = eng.stats()
        cols = [eng.read_column(1, 0, q) for q in range(len(prompts[0]), len(prompts[0]) + 8)]
        runs.append((seqs, np.array(kinds), st, cols))
        eng.close()
    (s0, k0, st0, c0), (s1, k1, st1, c1) = runs
    assert s0 == s1 and np.array_equal(k0, k1)
    for k in ("steps", "rows", "protected_rows", "triggers", "verified", "repairs", "verifier_launches",
              "catchup_tokens"):
        assert st0[k] == st1[k], k
    assert st0["triggers"] > 0 and st0["catchup_tokens"] > st0["verifier_launches"]
    assert all(np.array_equal(a, b) for a, b in zip(c0, c1))   # shadow columns: bit-identical


def test_sync_step_does_not_wait_on_device(torch, tiny):
    """mg_decode_step in the synchronous verify mode never synchronises the
    stream: with the device busy in a long spin kernel,
    a step with real triggers is enqueued and returns while the spin still
    runs; its results then match the same step taken after a drain."""
    shp, _ = tiny
    B, tau = 4, INF
    prompts = inputs.prompts(B, 12, shp["vocab"], seed=440)
    eng = _engine(shp, B)
    for i, p in enumerate(prompts):
        eng.prefill(i, p)
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    for _ in range(3):                          # first use eager, second builds the step graph
        eng.step(list(range(B)), None, tau, out)
    torch.cuda.synchronize()
    with torch.cuda.stream(eng.stream):
        torch.cuda._sleep(400_000_000)          # ~0.2 s of device time
    eng.step(list(range(B)), None, tau, out)
    busy = not eng.stream.query()
    torch.cuda.synchronize()
    assert busy, "the step waited for the device"
    st = eng.stats()
    assert st["triggers"] == st["protected_rows"] == 4 * B
    eng.close()
