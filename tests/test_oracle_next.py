"""Pins for the oracle's SURVEY 8(f) NEXT rows.

* NEXT-2: LLM-42-style windowed verification with rollback (PAPER.md:227
  "keeps the default path but verifies every token", "verifier
  setting K=64", "restart-from-rollback").  Pinned by the
  closed-form end point -- whatever the window K and the batch, the verified
  output is the deterministic reference decode (the tau=inf run)
  -- and by the rollback arithmetic: the first rollback lands exactly on the
  first divergence of the unverified BF16 trajectory from the reference
  ("first divergence").
* NEXT-3 repair-action ablation: token-only repair emits the
  verifier token but leaves the BF16 column; column repair copies it.
"""
import numpy as np
import pytest

from paper_2605_30218_b200 import inputs, metrics


@pytest.fixture(scope="module")
def tiny(orc):
    shp = inputs.shape("tiny")
    m = orc.Model(shp)
    yield shp, m
    m.close()


def _seq(st, row, P):
    return [st.token(row, q) for q in range(P, st.pos(row) + 1)]


def _windowed(orc, m, prompts, K, target, noise=0.3):
    """Fast (tau=0) steps in windows of K, each followed by verify_window on
    every row, until every row holds `target` verified tokens."""
    B = len(prompts)
    st = orc.State(m, B, max(len(p) for p in prompts) + target + 4 * K + 8)
    det = orc.det_sched()
    fs = orc.fast_sched(B, noise_amp=noise, noise_seed=77)
    for i, p in enumerate(prompts):
        st.prefill(i, p, det)
    rolled = 0
    while min(st.pos(i) - len(prompts[i]) + 1 for i in range(B)) < target:
        for _ in range(K):
            st.step(np.arange(B), np.zeros(B, np.uint8), 0.0, fs, det)
        npos, last, rb = st.verify_window(np.arange(B), det)
        for i in range(B):
            assert st.shadow_len(i) == st.pos(i) == npos[i]
            assert st.token(i, npos[i]) == last[i]
        rolled += int(rb.sum())
    return st, rolled


@pytest.mark.parametrize("K", [1, 3, 8])
def test_window_verify_equals_reference(orc, tiny, K):
    """Every verified token equals the deterministic reference decode for any
    window size and batch size (LLM-42's guarantee), with
    injected perturbations that really flip tokens."""
    shp, m = tiny
    target = 10
    prompts = inputs.prompts(5, inputs.ragged_lengths(5, 8, 19), shp["vocab"])
    refs = [orc.reference_decode(m, p, target) for p in prompts]
    any_roll = 0
    for B in (1, 5):
        st, rolled = _windowed(orc, m, prompts[:B], K, target)
        for i in range(B):
            assert _seq(st, i, len(prompts[i]))[:target] == refs[i], (K, B, i)
        ws = st.window_stats()
        assert ws["rolled_back_tokens"] == rolled and ws["rollbacks"] <= ws["window_rows"]
        any_roll += ws["rollbacks"]
        st.close()
    assert any_roll > 0  # the noise forced rollbacks


def test_first_rollback_is_first_divergence(orc, tiny):
    """The first window's rollback position equals the first divergence of
    the unverified BF16 trajectory from the reference, the
    replaced token is the reference token there, and the discarded count is
    K - d (metrics.first_divergence is itself pinned in test_metrics)."""
    shp, m = tiny
    K, B = 12, 4
    prompts = inputs.prompts(B, 9, shp["vocab"], seed=808)
    det = orc.det_sched()
    fs = orc.fast_sched(B, noise_amp=0.6, noise_seed=5)
    # unverified BF16 trajectory
    st = orc.State(m, B, 40)
    seqs = [[st.prefill(i, p, det)] for i, p in enumerate(prompts)]
    for _ in range(K):
        r = st.step(np.arange(B), np.zeros(B, np.uint8), 0.0, fs, det)
        for b in range(B):
            seqs[b].append(int(r["out"][b]))
    npos, last, rb = st.verify_window(np.arange(B), det)
    seen = 0
    for i in range(B):
        ref = orc.reference_decode(m, prompts[i], K + 1)
        d = metrics.first_divergence(seqs[i], ref)
        if d is None:
            assert npos[i] == 9 + K and rb[i] == 0
        else:
            seen += 1
            assert npos[i] == 9 + d and last[i] == ref[d] and rb[i] == K - d
    assert seen > 0
    st.close()


def test_window_shadow_columns_match_per_step_catchup(orc, tiny):
    """The window verifier writes the same shadow columns as the per-step
    verifier over the same committed tokens (catch-up chunking invariance,
    SURVEY 8(c) A23)."""
    shp, m = tiny
    prompt = inputs.prompts(1, 10, shp["vocab"], seed=71)[0]
    det = orc.det_sched()
    a = orc.State(m, 1, 32)
    a.prefill(0, prompt, det)
    for _ in range(6):
        a.step([0], [1], float("inf"), det, det)
    b = orc.State(m, 1, 32)
    b.prefill(0, prompt, det)
    for _ in range(6):
        b.step([0], [0], 0.0, det, det)      # det fast schedule: never diverges
    npos, last, rb = b.verify_window([0], det)
    assert rb[0] == 0 and npos[0] == a.pos(0) == 16
    # a's shadow covers 0..15 (through the last verified step), b's 0..15
    for q in range(16):
        assert np.array_equal(a.column(1, 0, q), b.column(1, 0, q)), q
    a.close()
    b.close()


def test_token_only_repair_leaves_bf16_column(orc, tiny):
    """PAPER.md:317 ablation: token-only emits the verifier token but keeps the
    tentative BF16 K/V column -- the fast cache after a token-only repair is
    the cache of the same run with a verified (no-write) commit, while column
    repair makes column p equal the verifier's."""
    shp, m = tiny
    prompts = inputs.prompts(2, 12, shp["vocab"], seed=45)
    det = orc.det_sched()
    fs = orc.fast_sched(2, 0.8, 3)
    states = {}
    for mode, k in (("verified", 1), ("column", 2), ("token", 2)):
        st = orc.State(m, 2, 32)
        if mode == "token":
            st.set_repair_mode(1)
        for i, p in enumerate(prompts):
            st.prefill(i, p, det)
        for t in range(4):
            st.step([0, 1], [1, 1], 0.0, fs, det, forced_trig=[1, 1], forced_out=[5 + t, 9 + t],
                    forced_kind=[k if t == 2 else 1, 1])
        states[mode] = st
    p = 12 + 2
    v, c, t = states["verified"], states["column"], states["token"]
    assert t.digest(0) == v.digest(0)                       # no fast-cache write at all
    assert c.digest(0, 0, p) == v.digest(0, 0, p)           # column repair: only (0, p) differs
    assert np.array_equal(c.column(0, 0, p), c.column(1, 0, p))
    assert np.array_equal(t.column(0, 0, p), v.column(0, 0, p))  # the BF16 path's own column
    assert t.token(0, p + 1) == c.token(0, p + 1) == 7      # the emitted token is the same
    for s in states.values():
        s.close()


def test_token_only_repair_keeps_tau_inf_reference(orc, tiny):
    """Under reading A1 the verifier reads only its shadow cache, so at
    tau=inf (every token verified) the token-only ablation still emits the
    reference; the ablation changes only what the BF16 path sees next."""
    shp, m = tiny
    prompts = inputs.prompts(3, inputs.ragged_lengths(3, 8, 14, seed=2), shp["vocab"], seed=17)
    steps = 8
    refs = [orc.reference_decode(m, p, steps) for p in prompts]
    st = orc.State(m, 3, 40)
    st.set_repair_mode(1)
    det = orc.det_sched()
    seqs = [[st.prefill(i, p, det)] for i, p in enumerate(prompts)]
    for _ in range(steps - 1):
        r = st.step(np.arange(3), np.ones(3, np.uint8), float("inf"), orc.fast_sched(3, 0.5, 8), det)
        for b in range(3):
            seqs[b].append(int(r["out"][b]))
    assert seqs == refs
    assert st.stats()["repairs"] > 0
    st.close()
