"""Pins for the oracle's numeric primitives.

Every check compares the oracle against something other than itself: values
printed in SPEC/PAPER, closed forms, fp64 brute force within a textbook error
bound, or an independently written bit-level routine.
"""
import math

import numpy as np
import pytest


# ----------------------------------------------------------------- bf16
def _ref_bf16_bits(x32: np.ndarray) -> np.ndarray:
    """Independent RNE: choose between the two bf16 neighbours by exact
    fp64 distance, ties to the even mantissa.  Finite inputs only."""
    u = x32.view(np.uint32)
    lo = (u & np.uint32(0xFFFF0000))
    hi = lo + np.uint32(0x10000)             # next bf16 away from zero (same sign)
    xf = x32.astype(np.float64)
    flo = lo.view(np.float32).astype(np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        fhi = hi.view(np.float32).astype(np.float64)
        # the 'hi' neighbour of the largest finite magnitude is +-inf: its
        # distance is taken as the distance to 2^128 (IEEE overflow rule)
        over = np.isinf(fhi)
        fhi_d = np.where(over, np.sign(xf) * 2.0 ** 128, fhi)
    dlo = np.abs(xf - flo)
    dhi = np.abs(fhi_d - xf)
    lo_even = ((lo >> np.uint32(16)) & np.uint32(1)) == 0
    pick_hi = (dhi < dlo) | ((dhi == dlo) & ~lo_even)
    return np.where(pick_hi, hi >> np.uint32(16), lo >> np.uint32(16)).astype(np.uint16)


def _oracle_bf16(orc, x32):
    import ctypes as C
    f = orc.lib().or_f32_to_bf16
    return np.array([f(C.c_float(float(v))) for v in x32], dtype=np.uint16)


def test_bf16_spec_values(orc):
    # 1.0 -> 1.0; 1.00390625 (tie) -> 1.0 (even); 3.14159 -> 3.140625
    got = orc.bf16_to_f32(orc.f32_to_bf16([1.0, 1.00390625, 3.14159]))
    assert got.tolist() == [1.0, 1.0, 3.140625]


def test_bf16_structured_sweep(orc):
    """Every sign/exponent/mantissa top half x a set of low halves covering
    exact, tie, just-below/above-tie and sticky cases (all rounding paths)."""
    tops = np.arange(0, 1 << 16, dtype=np.uint32)
    lows = np.array([0, 1, 0x7FFF, 0x8000, 0x8001, 0xFFFF, 0x4000, 0xC000, 0x1234, 0xBEEF], np.uint32)
    u = (tops[:, None] << 16 | lows[None, :]).ravel()
    finite = (u & 0x7F800000) != 0x7F800000
    x = u[finite].view(np.float32)
    # oracle over the array through the C function, vectorised via a chunked loop
    import ctypes as C
    lib = orc.lib()
    got = np.empty(x.size, np.uint16)
    xs = x.tolist()
    f = lib.or_f32_to_bf16
    for i, v in enumerate(xs):
        got[i] = f(v)
    ref = _ref_bf16_bits(x)
    assert np.array_equal(got, ref)


def test_bf16_random_and_idempotent(orc):
    rng = np.random.default_rng(0)
    u = rng.integers(0, 1 << 32, size=200_000, dtype=np.uint64).astype(np.uint32)
    u = u[(u & 0x7F800000) != 0x7F800000]
    x = u.view(np.float32)
    got = _oracle_bf16(orc, x)
    assert np.array_equal(got, _ref_bf16_bits(x))
    back = orc.bf16_to_f32(got)
    assert np.array_equal(_oracle_bf16(orc, back), got)  # round(round(x)) == round(x)


def test_bf16_exhaustive(orc, tmp_path):
    """All 2^32 fp32 bit patterns (test plan item 1) through the
    oracle's conversion against tests/bf16_exhaustive.c, which rounds by exact
    fp64 distance to the two bf16 neighbours (not the oracle's add-and-
    truncate); a C loop over liboracle.so, ~5 s on 8 cores."""
    import os
    import subprocess
    lib = orc.lib()._name
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bf16_exhaustive.c")
    exe = str(tmp_path / "bf16_exhaustive")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-Wall", src, lib,
                           "-Wl,-rpath," + os.path.dirname(lib), "-lm", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "checked 4294967296 mismatches 0" in out.stdout, out.stdout


def test_bf16_specials(orc):
    b = _oracle_bf16(orc, np.array([np.inf, -np.inf, np.nan, 3.4e38, -3.4e38], np.float32))
    f = orc.bf16_to_f32(b)
    assert f[0] == np.inf and f[1] == -np.inf and np.isnan(f[2])
    assert f[3] == np.inf and f[4] == -np.inf  # above max bf16 -> rounds to inf


# ----------------------------------------------------------------- PRNG + weights
def test_splitmix64_published_vectors(orc):
    # SplitMix64 seeded with 0 emits 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4,
    # 0x06c45d188009454f (Steele, Lea, Flood 2014 / Vigna's splitmix64.c);
    # our counter form is mix(x + golden), so x = k*golden gives output k+1.
    g = 0x9E3779B97F4A7C15
    lib = orc.lib()
    assert lib.or_splitmix64(0) == 0xE220A8397B1DCDAF
    assert lib.or_splitmix64(g) == 0x6E789E6AA1B965F4
    assert lib.or_splitmix64((2 * g) % (1 << 64)) == 0x06C45D188009454F


def test_weight_generator_distribution(orc):
    """Projection weights ~ U(-sqrt(3/fan_in), sqrt(3/fan_in)): mean 0,
    variance 1/fan_in; gains in [7/8, 9/8]; deterministic per (seed, id)."""
    n, fan = 1 << 20, 4096
    w = orc.bf16_to_f32(orc.gen_tensor(42, 5, n, 0, fan)).astype(np.float64)
    assert abs(w.mean()) < 4 * math.sqrt(1 / fan / n)
    assert abs(w.var() * fan - 1.0) < 0.01
    assert np.abs(w).max() <= math.sqrt(3 / fan) * (1 + 2 ** -8)
    g = orc.bf16_to_f32(orc.gen_tensor(42, 6, 65536, 2, 0))
    assert g.min() >= 0.875 and g.max() <= 1.125 and abs(g.mean() - 1) < 0.002
    assert np.array_equal(orc.gen_tensor(42, 5, 1000, 0, fan), orc.gen_tensor(42, 5, 1000, 0, fan))
    assert not np.array_equal(orc.gen_tensor(42, 5, 1000, 0, fan), orc.gen_tensor(42, 6, 1000, 0, fan))
    assert not np.array_equal(orc.gen_tensor(42, 5, 1000, 0, fan), orc.gen_tensor(43, 5, 1000, 0, fan))


def test_weight_generator_first_values_from_spec(orc):
    """The documented recipe evaluated by hand for element 0
    of tensor 0 (embedding, sigma=1): splitmix64(42) -> top 24 bits."""
    r = orc.lib().or_splitmix64(42)
    u = (r >> 40) - (1 << 23)
    c = np.float32(math.sqrt(3.0) / 8388608.0)
    want = np.float32(np.float32(u) * c)
    got = orc.bf16_to_f32(orc.gen_tensor(42, 0, 1, 1, 0))[0]
    assert got == orc.bf16_to_f32(orc.f32_to_bf16([want]))[0]
    assert abs(float(got) - float(want)) <= abs(float(want)) * 2 ** -8


# ----------------------------------------------------------------- dot / gemm
def _rand_bf16(orc, rng, shape, scale=1.0):
    return orc.f32_to_bf16((rng.standard_normal(shape) * scale).astype(np.float32))


def test_dot_exact_on_integers(orc):
    """Small integers: every partial sum is exact in fp32, so any chunking
    equals the exact integer dot product."""
    rng = np.random.default_rng(1)
    a = rng.integers(-8, 9, 1000).astype(np.float32)
    b = rng.integers(-8, 9, 1000).astype(np.float32)
    A, Bb = orc.f32_to_bf16(a), orc.f32_to_bf16(b)
    exact = float(np.dot(a.astype(np.int64), b.astype(np.int64)))
    for S in (1, 2, 3, 7, 8, 1000, 5000):
        assert orc.dot_bf16(A, Bb, S) == exact


def test_dot_reduction_order_matters(orc):
    """[b, 1, -b, 1] . ones with b = 2^25 (fp32 ulp 4 there):
    sequential ((b+1)-b)+1 = 0+1 = 1; two chunks (b+1) + (-b+1) = b + (-b)
    = 0 -- both ones absorbed.  Different plans, different results (the
    mechanism of PAPER.md:35)."""
    b = 2.0 ** 25
    a = orc.f32_to_bf16(np.array([b, 1.0, -b, 1.0], np.float32))
    ones = orc.f32_to_bf16(np.ones(4, np.float32))
    assert orc.dot_bf16(a, ones, 1) == 1.0
    assert orc.dot_bf16(a, ones, 2) == 0.0


@pytest.mark.parametrize("K", [256, 4096, 14336])
def test_dot_within_fp32_bound(orc, K):
    """|fp32 chunked dot - exact| <= K * 2^-24 * sum|a_i b_i| (textbook
    recursive-summation bound; products of bf16 are exact in fp32)."""
    rng = np.random.default_rng(K)
    for S in (1, 3, 8):
        a = _rand_bf16(orc, rng, K)
        b = _rand_bf16(orc, rng, K)
        af, bf = orc.bf16_to_f32(a).astype(np.float64), orc.bf16_to_f32(b).astype(np.float64)
        exact = float(np.dot(af, bf))
        bound = K * 2 ** -24 * float(np.abs(af * bf).sum())
        assert abs(orc.dot_bf16(a, b, S) - exact) <= bound


def test_gemm_matches_fp64_and_layout(orc):
    """y = x W^T: a transposed or mis-indexed operand fails the fp64 check."""
    rng = np.random.default_rng(2)
    T, N, K = 5, 37, 200
    x = _rand_bf16(orc, rng, (T, K))
    W = _rand_bf16(orc, rng, (N, K))
    xf, Wf = orc.bf16_to_f32(x).astype(np.float64), orc.bf16_to_f32(W).astype(np.float64)
    ref = xf @ Wf.T
    bound = K * 2 ** -24 * (np.abs(xf) @ np.abs(Wf).T)
    for S in (1, 4):
        y = orc.gemm(x, W, S)
        assert np.all(np.abs(y - ref) <= bound)


# ----------------------------------------------------------------- rmsnorm / rope / swiglu / residual
def test_rmsnorm_fp64(orc):
    rng = np.random.default_rng(3)
    T, d = 4, 256
    x = _rand_bf16(orc, rng, (T, d), 3.0)
    w = orc.f32_to_bf16((1 + 0.1 * rng.standard_normal(d)).astype(np.float32))
    y = orc.bf16_to_f32(orc.rmsnorm(x, w, 1e-5)).astype(np.float64)
    xf, wf = orc.bf16_to_f32(x).astype(np.float64), orc.bf16_to_f32(w).astype(np.float64)
    ref = xf / np.sqrt((xf ** 2).mean(1, keepdims=True) + 1e-5) * wf
    assert np.all(np.abs(y - ref) <= np.abs(ref) * 2 ** -7 + 1e-30)  # <= 1 bf16 ulp (+fp32 slack)
    # scale invariance of the normalised vector (before the gain): x and 2x
    y2 = orc.rmsnorm(orc.f32_to_bf16(2 * orc.bf16_to_f32(x)), w, 0.0)
    assert np.array_equal(y2, orc.rmsnorm(x, w, 0.0))


def test_rope_identity_at_zero_and_rotation(orc):
    c, s = orc.rope_table(128, 500000.0, 0)
    assert np.all(c == 1.0) and np.all(s == 0.0)
    rng = np.random.default_rng(4)
    H, KV, hd = 4, 2, 64
    N = (H + 2 * KV) * hd
    acc = rng.standard_normal((3, N)).astype(np.float32)
    pos = np.array([0, 5, 1000], np.int32)
    q, k, v = orc.qkv_epilogue(acc, None, pos, H, KV, hd, 10000.0)
    qf = orc.bf16_to_f32(q).astype(np.float64).reshape(3, H, hd)
    # position 0: identity (up to bf16 rounding of the accumulator)
    assert np.array_equal(q[0], orc.f32_to_bf16(acc[0, :H * hd]))
    # fp64 complex rotation reference: z = (a + i b) * exp(i * pos * theta^(-2j/hd))
    a = acc[:, :H * hd].astype(np.float64).reshape(3, H, hd)
    j = np.arange(hd // 2)
    ang = pos[:, None].astype(np.float64) * 10000.0 ** (-2.0 * j / hd)
    z = (a[..., :hd // 2] + 1j * a[..., hd // 2:]) * np.exp(1j * ang)[:, None, :]
    ref = np.concatenate([z.real, z.imag], -1)
    assert np.all(np.abs(qf - ref) <= np.abs(ref) * 2 ** -7 + 2e-6 * np.abs(a).max())
    # pair norms preserved
    nq = qf[..., :hd // 2] ** 2 + qf[..., hd // 2:] ** 2
    na = a[..., :hd // 2] ** 2 + a[..., hd // 2:] ** 2
    assert np.allclose(nq, na, rtol=2 ** -6, atol=1e-6)
    # v untouched (bf16 of the accumulator)
    assert np.array_equal(v, orc.f32_to_bf16(acc[:, (H + KV) * hd:]))


def test_qkv_bias_added(orc):
    rng = np.random.default_rng(5)
    H, KV, hd = 2, 1, 64
    N = (H + 2 * KV) * hd
    acc = np.zeros((1, N), np.float32)
    bias = orc.f32_to_bf16(rng.standard_normal(N).astype(np.float32))
    q, k, v = orc.qkv_epilogue(acc, bias, np.array([0], np.int32), H, KV, hd, 10000.0)
    assert np.array_equal(np.concatenate([q[0], k[0], v[0]]), bias)


def test_swiglu_and_residual_fp64(orc):
    rng = np.random.default_rng(6)
    g = (rng.standard_normal(5000) * 4).astype(np.float32)
    u = rng.standard_normal(5000).astype(np.float32)
    a = orc.bf16_to_f32(orc.swiglu(g, u)).astype(np.float64)
    gd = g.astype(np.float64)
    ref = gd / (1 + np.exp(-gd)) * u
    assert np.all(np.abs(a - ref) <= np.abs(ref) * 2 ** -7 + 1e-30)
    assert orc.bf16_to_f32(orc.swiglu(np.zeros(1, np.float32), np.ones(1, np.float32)))[0] == 0.0
    x = _rand_bf16(orc, rng, 5000)
    r = orc.bf16_to_f32(orc.residual(x, u)).astype(np.float64)
    refr = orc.bf16_to_f32(x).astype(np.float64) + u
    assert np.all(np.abs(r - refr) <= np.abs(refr) * 2 ** -8 + 1e-30)


# ----------------------------------------------------------------- attention
def _attn_fp64(q, K, V, n):
    H, hd = q.shape
    KVh = K.shape[0]
    G = H // KVh
    out = np.zeros((H, hd))
    for h in range(H):
        kk, vv = K[h // G, :n], V[h // G, :n]
        s = kk @ q[h] / math.sqrt(hd)
        p = np.exp(s - s.max())
        p /= p.sum()
        out[h] = p @ vv
    return out


# chunk < 0: the streamed form (4 round-robin block streams per split of -chunk keys)
@pytest.mark.parametrize("n,chunk,splits", [(1, 0, 1), (37, 0, 1), (37, 16, 1), (200, 0, 7), (200, 64, 1),
                                            (1, -64, 1), (37, -64, 1), (200, -64, 1), (250, -512, 1),
                                            (77, -16, 1)])
def test_attention_fp64(orc, n, chunk, splits):
    rng = np.random.default_rng(n + abs(chunk) + splits)
    H, KVh, hd, stride = 8, 2, 64, 256
    q = _rand_bf16(orc, rng, (H, hd))
    K = _rand_bf16(orc, rng, (KVh, stride, hd))
    V = _rand_bf16(orc, rng, (KVh, stride, hd))
    o = orc.bf16_to_f32(orc.attention(q, K, V, n, chunk, splits)).astype(np.float64).reshape(H, hd)
    f = lambda a: orc.bf16_to_f32(a).astype(np.float64)
    ref = _attn_fp64(f(q), f(K), f(V), n)
    assert np.all(np.abs(o - ref) <= np.abs(ref) * 2 ** -7 + 1e-5 * np.abs(f(V)).max())


@pytest.mark.parametrize("chunk", [0, -64, -16])
def test_attention_special_cases(orc, chunk):
    rng = np.random.default_rng(9)
    H, KVh, hd = 4, 4, 64
    q = _rand_bf16(orc, rng, (H, hd))
    K = _rand_bf16(orc, rng, (KVh, 8, hd))
    V = _rand_bf16(orc, rng, (KVh, 8, hd))
    # one key: softmax weight exactly 1 -> o == v
    o = orc.attention(q, K, V, 1, chunk).reshape(H, hd)
    assert np.array_equal(o, V[:, 0, :])
    # identical keys: uniform weights -> o == mean of the values (fp64, 1 ulp)
    K2 = np.repeat(K[:, :1, :], 8, axis=1)
    o2 = orc.bf16_to_f32(orc.attention(q, K2, V, 8, chunk)).reshape(H, hd).astype(np.float64)
    ref = orc.bf16_to_f32(V).astype(np.float64).mean(1)
    assert np.all(np.abs(o2 - ref) <= np.abs(ref) * 2 ** -7 + 1e-6)


# ----------------------------------------------------------------- top-2 / gate
def test_top2_spec_values(orc):
    r = orc.top2(np.array([3.5, 1.25, 0.0], np.float32))
    assert r["g"][0] == 2.25 and r["i1"][0] == 0 and r["i2"][0] == 1
    r = orc.top2(np.array([2.0, 2.0, 1.0], np.float32))
    assert r["g"][0] == 0.0 and r["i1"][0] == 0 and r["i2"][0] == 1


def test_top2_brute_force_with_ties_and_nan(orc):
    rng = np.random.default_rng(10)
    T, V = 300, 97
    L = rng.integers(-5, 6, (T, V)).astype(np.float32) * 0.5   # many ties
    L[::7, 3] = np.nan
    r = orc.top2(L)
    for t in range(T):
        vals = np.where(np.isnan(L[t]), -np.inf, L[t])
        order = np.lexsort((np.arange(V), -vals))          # value desc, id asc
        assert r["i1"][t] == order[0] and r["i2"][t] == order[1]
        assert r["g"][t] == np.float32(vals[order[0]] - vals[order[1]])
    assert r["nan"]


def test_margin_is_cluster_count_test(orc):
    """N(D) > 1  <=>  g <= D with N(D) = |{j : l_j >= l(1) - D}|
    (the paper's >= makes the boundary inclusive; the gate uses strict <).
    SPEC.md:383 example: [5.0, 4.9, 4.4, 1.0] -> N(0.25)=2, N(1.0)=3."""
    ex = np.array([5.0, 4.9, 4.4, 1.0], np.float32)
    N = lambda l, D: int((l >= l.max() - np.float32(D)).sum())
    assert N(ex, 0.25) == 2 and N(ex, 1.0) == 3
    rng = np.random.default_rng(12)
    L = rng.standard_normal((500, 64)).astype(np.float32)
    g = orc.top2(L)["g"]
    for D in (0.05, 0.1, 0.5):
        for t in range(500):
            assert (N(L[t], D) > 1) == (g[t] <= np.float32(D))


def test_gate_special_cases_and_monotone(orc):
    rng = np.random.default_rng(13)
    g = np.abs(rng.standard_normal(64)).astype(np.float32)
    g[5] = 0.0
    prot = (rng.random(64) < 0.6).astype(np.uint8)
    assert orc.gate(g, prot, 0.0).size == 0                           # tau=0: r_verify = 0
    allp = orc.gate(g, prot, float("inf"))
    assert np.array_equal(allp, np.nonzero(prot)[0])                 # tau=inf: every protected row
    prev = set()
    for tau in np.sort(np.concatenate([g, [0.3, 1.0, 5.0]])):
        cur = set(orc.gate(g, prot, float(tau)).tolist())
        assert prev <= cur                                           # monotone in tau
        prev = cur
    # strict inequality at g == tau
    t = float(g[np.nonzero(prot)[0][0]])
    row = int(np.nonzero(prot)[0][0])
    assert row not in orc.gate(g, prot, t).tolist()
    assert row in orc.gate(g, prot, np.nextafter(np.float32(t), np.float32(np.inf))).tolist()
    # ascending order
    r = orc.gate(g, np.ones(64, np.uint8), 10.0)
    assert np.all(np.diff(r) > 0)


def test_gate_non_finite_margins(orc):
    """DESIGN.md A4/A7: tau=+inf is always-on for EVERY protected row, also one
    whose margin is +inf (second logit -inf) -- r_verify = 1;
    a row whose logits are all NaN (ranked -inf, A7) has margin -inf - -inf =
    NaN and fires for any tau > 0; tau = 0 never fires (pure BF16)."""
    L = np.zeros((4, 8), np.float32)
    L[0, 3] = 1.0                       # ordinary row: g = 1
    L[1, :] = -np.inf
    L[1, 2] = 0.5                       # second logit -inf: g = +inf
    L[2, :] = np.nan                    # all NaN: v1 = v2 = -inf, g = NaN
    L[3, 5] = 2.0                       # g = 2
    g = orc.top2(L)["g"]
    assert g[0] == 1.0 and np.isposinf(g[1]) and np.isnan(g[2]) and g[3] == 2.0
    prot = np.array([1, 1, 1, 0], np.uint8)
    assert orc.gate(g, prot, float("inf")).tolist() == [0, 1, 2]     # always-on: every protected row
    assert orc.gate(g, prot, 1.5).tolist() == [0, 2]                 # NaN margin fires, +inf does not
    assert orc.gate(g, prot, 0.0).tolist() == []                     # tau = 0: pure BF16
