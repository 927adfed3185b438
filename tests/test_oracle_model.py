"""Pins for the oracle's decoder forward and MarginGate policy loop.

The forward is pinned by an independent fp64 numpy implementation of the
same decoder (library matmuls, exact exp) with bf16 rounding at the
DESIGN.md 3.3 points; the policy loop by the paper's special cases
(tau=0 -> BF16, tau=inf -> always-on verification = reference,
PAPER.md:215), by brute-force batch invariance of the
verifier over every batch size 1..8 on the tiny model (BASELINE.json
north_star), by repair locality and by the commit-record
invariants.
"""
import math

import numpy as np
import pytest

from paper_2605_30218_b200 import inputs


def _rne(x64: np.ndarray) -> np.ndarray:
    """fp64 -> fp32 -> bf16 (RNE) -> fp64; vectorised, independent of the oracle."""
    x32 = np.asarray(x64, dtype=np.float32)
    u = x32.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _np_forward(model, shape, tokens):
    """Textbook pre-norm Llama/Qwen decoder in fp64 over a whole sequence
    (causal), bf16 at the documented rounding points.  Returns fp64 logits
    for every position."""
    f = lambda a: (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    L, d, H, KV, hd, F, V = (shape[k] for k in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim",
                                                 "d_ff", "vocab"))
    eps, theta = shape["rms_eps"], shape["rope_theta"]
    T = len(tokens)
    E = f(model.tensor(-1, 0)).reshape(V, d)
    x = E[tokens]

    def norm(x, w):
        return _rne(x / np.sqrt((x * x).mean(-1, keepdims=True) + eps) * w)

    j = np.arange(hd // 2)
    ang = np.arange(T)[:, None] * theta ** (-2.0 * j / hd)
    cos, sin = np.cos(ang), np.sin(ang)

    def rope(a):  # a [T, heads, hd]
        lo, hi = a[..., :hd // 2], a[..., hd // 2:]
        c, s = cos[:, None, :], sin[:, None, :]
        return np.concatenate([lo * c - hi * s, hi * c + lo * s], -1)

    for l in range(L):
        W = lambda w, *sh: f(model.tensor(l, w)).reshape(*sh)
        xn = norm(x, W(0, d))
        q = xn @ W(1, H * hd, d).T
        k = xn @ W(2, KV * hd, d).T
        v = xn @ W(3, KV * hd, d).T
        if shape.get("qkv_bias"):
            q, k, v = q + W(9, H * hd), k + W(10, KV * hd), v + W(11, KV * hd)
        q = _rne(rope(q.reshape(T, H, hd)))
        k = _rne(rope(k.reshape(T, KV, hd)))
        v = _rne(v.reshape(T, KV, hd))
        att = np.zeros((T, H, hd))
        G = H // KV
        for h in range(H):
            s = q[:, h] @ k[:, h // G].T / math.sqrt(hd)
            s = np.where(np.tril(np.ones((T, T), bool)), s, -np.inf)
            p = np.exp(s - s.max(1, keepdims=True))
            p /= p.sum(1, keepdims=True)
            att[:, h] = p @ v[:, h // G]
        att = _rne(att.reshape(T, H * hd))
        x = _rne(x + att @ W(4, d, H * hd).T)
        xn = norm(x, W(5, d))
        g = xn @ W(6, F, d).T
        u = xn @ W(7, F, d).T
        a = _rne(g / (1 + np.exp(-g)) * u)
        x = _rne(x + a @ W(8, d, F).T)
    xf = norm(x, f(model.tensor(-1, 1)))
    return xf @ f(model.tensor(-1, 2)).reshape(V, d).T


@pytest.fixture(scope="module")
def tiny(orc):
    shp = inputs.shape("tiny")
    m = orc.Model(shp)
    yield shp, m
    m.close()


@pytest.fixture(scope="module")
def tiny_gqa(orc):
    shp = inputs.shape("tiny_gqa")
    m = orc.Model(shp)
    yield shp, m
    m.close()


def test_tensor_ids_follow_documented_layout(orc, tiny):
    """DESIGN.md 3.1 tensor-id table, evaluated independently."""
    shp, m = tiny
    L, d, H, hd, F = shp["n_layers"], shp["d_model"], shp["n_heads"], shp["head_dim"], shp["d_ff"]
    seed = shp["weight_seed"]
    assert np.array_equal(m.tensor(-1, 0), orc.gen_tensor(seed, 0, shp["vocab"] * d, 1, 0))
    assert np.array_equal(m.tensor(-1, 1), orc.gen_tensor(seed, 1 + 16 * L, d, 2, 0))
    assert np.array_equal(m.tensor(-1, 2), orc.gen_tensor(seed, 2 + 16 * L, shp["vocab"] * d, 0, d))
    assert np.array_equal(m.tensor(1, 1), orc.gen_tensor(seed, 1 + 16 + 1, H * hd * d, 0, d))
    assert np.array_equal(m.tensor(1, 8), orc.gen_tensor(seed, 1 + 16 + 8, d * F, 0, F))
    assert np.array_equal(m.tensor(0, 5), orc.gen_tensor(seed, 1 + 5, d, 2, 0))


@pytest.mark.parametrize("which", ["tiny", "tiny_gqa"])
def test_forward_matches_fp64_decoder(orc, tiny, tiny_gqa, which):
    """Oracle decode logits vs an independent fp64 decoder (bf16 roundings at
    the same points).  A dropped residual, wrong RoPE pair, wrong GQA head or
    transposed weight gives O(1) errors; rounding-order effects stay << 0.05."""
    shp, m = tiny if which == "tiny" else tiny_gqa
    prompt = inputs.prompts(1, 13, shp["vocab"], seed=101)[0]
    st = orc.State(m, 1, 32)
    det = orc.det_sched()
    y0 = st.prefill(0, prompt, det)
    toks = [y0]
    logits = []
    for _ in range(3):
        r = st.step([0], [0], 0.0, det, det, want_logits=True)
        logits.append(r["logits"][0])
        toks.append(int(r["out"][0]))
    ref = _np_forward(m, shp, prompt + toks[:-1])
    ref_last = ref[len(prompt) - 1:]
    assert int(np.argmax(ref_last[0])) == y0 or np.sort(ref_last[0])[-1] - np.sort(ref_last[0])[-2] < 0.1
    for t in range(3):
        err = np.abs(logits[t] - ref_last[t + 1]).max()
        assert err < 0.05, (t, err)
    st.close()


def _run(orc, m, prompts, B, tau, prot_mode="all", steps=12, noise=0.0, fast=None):
    st = orc.State(m, len(prompts), max(len(p) for p in prompts) + steps + 2)
    det = orc.det_sched()
    fs = fast or orc.fast_sched(B, noise_amp=noise, noise_seed=77)
    seqs = [[st.prefill(i, p, det)] for i, p in enumerate(prompts)]
    prot = inputs.protected_mask(B, prot_mode)
    recs = []
    for _ in range(steps - 1):
        r = st.step(np.arange(B), prot, tau, fs, det)
        recs.append(r)
        for b in range(B):
            seqs[b].append(int(r["out"][b]))
    stats = st.stats()
    return st, seqs, recs, stats


def test_tau_inf_is_reference_at_every_batch_size(orc, tiny):
    """tau=+inf == LLM-42-style always-on verification (r_verify = 1,
    PAPER.md:215): every protected row's sequence equals the deterministic
    batch-invariant reference decode, at every batch size 1..8, with the
    batch-shaped fast schedule and injected perturbations that force real
    flips and repairs."""
    shp, m = tiny
    prompts = inputs.prompts(8, inputs.ragged_lengths(8, 8, 23), shp["vocab"])
    steps = 10
    refs = [orc.reference_decode(m, p, steps) for p in prompts]
    total_rep = 0
    for B in range(1, 9):
        st, seqs, recs, stats = _run(orc, m, prompts[:B], B, float("inf"), steps=steps, noise=0.3)
        for b in range(B):
            assert seqs[b] == refs[b], (B, b)
        assert stats["triggers"] == stats["protected_rows"] == B * (steps - 1)     # r_verify = 1
        total_rep += stats["repairs"]
        st.close()
    assert total_rep > 0  # the noise really flipped tokens and repairs fired


def test_tau_zero_is_plain_bf16_batched(orc, tiny):
    """tau=0 never fires (g >= 0, strict <): kinds all fast, r_verify = 0,
    outputs == the fast-path argmax, shadow cache untouched after prefill."""
    shp, m = tiny
    prompts = inputs.prompts(4, 9, shp["vocab"], seed=33)
    st, seqs, recs, stats = _run(orc, m, prompts, 4, 0.0, steps=8, noise=0.3)
    assert stats["triggers"] == 0 and stats["verified"] == 0 and stats["repairs"] == 0
    for r in recs:
        assert np.all(r["kind"] == 0) and np.array_equal(r["out"], r["f_tok"])
    for i in range(4):
        assert st.shadow_len(i) == 9
    st.close()


def test_verifier_batch_composition_brute_force(orc, tiny):
    """The verifier's committed sequence for a protected request is the same
    whichever other requests share the batch and wherever it sits in it:
    protected request 0 placed at every slot of batches of size 1..6 with
    different co-batched prompts (BASELINE.json north_star)."""
    shp, m = tiny
    target = inputs.prompts(1, 11, shp["vocab"], seed=500)[0]
    steps = 8
    ref = orc.reference_decode(m, target, steps)
    for B in range(1, 7):
        for slot in range(B):
            others = inputs.prompts(B, inputs.ragged_lengths(B, 8, 20, seed=B * 10 + slot), shp["vocab"],
                                    seed=900 + 31 * B + slot)
            ps = others[:slot] + [target] + others[slot + 1:]
            prot = np.zeros(B, np.uint8)
            prot[slot] = 1
            st = orc.State(m, B, 40)
            det = orc.det_sched()
            seqs = [[st.prefill(i, p, det)] for i, p in enumerate(ps)]
            for _ in range(steps - 1):
                r = st.step(np.arange(B), prot, float("inf"), orc.fast_sched(B, 0.3, 5), det)
                for b in range(B):
                    seqs[b].append(int(r["out"][b]))
            assert seqs[slot] == ref, (B, slot)
            st.close()


def test_catchup_chunking_invariance(orc, tiny):
    """Shadow columns are bit-identical however the lazy catch-up is chunked
    (SURVEY 8(c) A23): teacher-forced identical tokens, verifier fired every
    step vs every third step vs only at the end."""
    shp, m = tiny
    prompt = inputs.prompts(1, 10, shp["vocab"], seed=71)[0]
    steps = 9
    toks = orc.reference_decode(m, prompt, steps + 1)
    cols = []
    for every in (1, 3, steps):
        st = orc.State(m, 1, 32)
        det = orc.det_sched()
        st.prefill(0, prompt, det)
        for t in range(steps):
            fire = (t + 1) % every == 0
            st.step([0], [1], 0.0, orc.fast_sched(1), det, forced_trig=[int(fire)], forced_out=[toks[t + 1]],
                    forced_kind=[1 if fire else 0])
        assert st.shadow_len(0) == 10 + steps
        cols.append([st.column(1, 0, q) for q in range(10 + steps)])
        st.close()
    for q in range(10 + steps):
        assert np.array_equal(cols[0][q], cols[1][q]) and np.array_equal(cols[0][q], cols[2][q])


def test_repair_touches_exactly_one_column(orc, tiny):
    """the step appends column p and a repair overwrites that
    single column (all layers, K and V) with the verifier's; every other
    column of the fast cache is unchanged."""
    shp, m = tiny
    prompts = inputs.prompts(2, 12, shp["vocab"], seed=44)
    S = 40
    st = orc.State(m, 2, S)
    det = orc.det_sched()
    for i, p in enumerate(prompts):
        st.prefill(i, p, det)
    snap = lambda: {(r, q): st.column(0, r, q) for r in range(2) for q in range(S)}
    seen = {0: 0, 1: 0, 2: 0}
    for _ in range(20):
        p0, p1 = st.pos(0), st.pos(1)
        before = snap()
        r = st.step([0, 1], [1, 1], 0.6, orc.fast_sched(2, 0.8, 9), det)
        after = snap()
        changed = {k for k in before if not np.array_equal(before[k], after[k])}
        assert changed <= {(0, p0), (1, p1)}
        for b, (rr, q) in enumerate(((0, p0), (1, p1))):
            k = int(r["kind"][b])
            seen[k] += 1
            if k == 2:
                assert np.array_equal(st.column(0, rr, q), st.column(1, rr, q))
    assert seen[2] > 0 and seen[1] + seen[0] > 0
    st.close()


def test_repair_locality_digest(orc, tiny):
    """Locality by construction: teacher-force the same tokens with kind
    verified vs kind repair; the fast caches then differ only at (row, p)."""
    shp, m = tiny
    prompt = inputs.prompts(2, 12, shp["vocab"], seed=45)
    states = []
    for k in (1, 2):
        st = orc.State(m, 2, 32)
        det = orc.det_sched()
        for i, p in enumerate(prompt):
            st.prefill(i, p, det)
        for t in range(4):
            st.step([0, 1], [1, 1], 0.0, orc.fast_sched(2, 0.8, 3), det, forced_trig=[1, 1],
                    forced_out=[5 + t, 9 + t], forced_kind=[k if t == 2 else 1, 1])
        states.append(st)
    p = 12 + 2
    a, b = states
    assert a.digest(0, 0, p) == b.digest(0, 0, p)
    assert np.array_equal(b.column(0, 0, p), b.column(1, 0, p))
    assert a.digest(1) == b.digest(1)
    for s in states:
        s.close()


def test_commit_records_and_stats(orc, tiny):
    """fast => (not protected or g >= tau) and out == f_tok;
    verified => g < tau and out == f_tok == v_tok; repair => g < tau and
    out == v_tok != f_tok; 0 <= r_repair <= r_verify <= 1."""
    shp, m = tiny
    prompts = inputs.prompts(6, inputs.ragged_lengths(6, 8, 16, seed=4), shp["vocab"], seed=61)
    tau = 0.4
    st, seqs, recs, stats = _run(orc, m, prompts, 6, tau, prot_mode="half", steps=14, noise=0.5)
    prot = inputs.protected_mask(6, "half")
    nt = 0
    for r in recs:
        for b in range(6):
            k, g = int(r["kind"][b]), float(r["g"][b])
            if k == 0:
                assert (not prot[b]) or g >= tau
                assert r["out"][b] == r["f_tok"][b]
            elif k == 1:
                assert prot[b] and g < tau and r["out"][b] == r["f_tok"][b] == r["v_tok"][b]
            else:
                assert prot[b] and g < tau and r["out"][b] == r["v_tok"][b] != r["f_tok"][b]
            nt += int(r["trig"][b])
    assert stats["triggers"] == nt
    assert 0 <= stats["repairs"] <= stats["triggers"] <= stats["protected_rows"]
    assert stats["verified"] + stats["repairs"] == stats["triggers"]
    assert stats["rows"] == 6 * 13 and stats["protected_rows"] == int(prot.sum()) * 13
    st.close()


def test_injected_noise_zero_at_batch_one(orc, tiny):
    """the injected perturbation is exactly zero at batch 1."""
    shp, m = tiny
    p = inputs.prompts(1, 9, shp["vocab"], seed=3)[0]
    outs = []
    for amp in (0.0, 5.0):
        st = orc.State(m, 1, 20)
        st.prefill(0, p, orc.det_sched())
        r = st.step([0], [0], 0.0, orc.fast_sched(1, amp, 1), orc.det_sched(), want_logits=True)
        outs.append(r["logits"])
        st.close()
    assert np.array_equal(outs[0], outs[1])
