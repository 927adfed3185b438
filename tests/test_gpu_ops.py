"""Per-kernel parity: each CUDA kernel of the hot path vs the oracle on
identical seeded inputs (SURVEY 8(c) parity protocol, step 1).

Tolerances (BASELINE north_star / DESIGN.md 6):
  * fp32 GEMM accumulators: |gpu - oracle| <= 1e-5 * sum|x_k w_k|
  * bf16 outputs: equal or 1 ulp apart (2 ulp where a libm-vs-CUDA expf enters)
  * weights, top-2, gate, QKV epilogue, residual: bit-exact
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2605_30218_b200 import kernels
    return kernels


def _bf(orc, a):
    return orc.bf16_to_f32(a).astype(np.float64)


def _rand(orc, rng, shape, scale=1.0):
    return orc.f32_to_bf16((rng.standard_normal(shape) * scale).astype(np.float32))


def _ulps(orc, a, b):
    """|a - b| in units of bf16 ulp of max(|a|,|b|) (bit patterns)."""
    fa, fb = _bf(orc, a), _bf(orc, b)
    mag = np.maximum(np.abs(fa), np.abs(fb))
    ulp = np.where(mag > 0, 2.0 ** (np.floor(np.log2(np.maximum(mag, 1e-38))) - 7), 2.0 ** -133)
    return np.abs(fa - fb) / ulp


# ------------------------------------------------------------------ K0
@pytest.mark.parametrize("kind,fan", [(0, 4096), (0, 14336), (1, 0), (2, 0), (3, 0)])
def test_weight_generator_bit_exact(orc, K, kind, fan):
    n = 1 << 18
    for tid in (0, 7, 513):
        assert np.array_equal(K.gen_tensor(42, tid, n, kind, fan), orc.gen_tensor(42, tid, n, kind, fan))


# ------------------------------------------------------------------ a2
@pytest.mark.parametrize("T,d", [(1, 256), (7, 4096), (3, 5120), (2, 3584)])
def test_rmsnorm(orc, K, T, d):
    rng = np.random.default_rng(T * d)
    x = _rand(orc, rng, (T, d), 3.0)
    w = orc.f32_to_bf16((1 + 0.1 * rng.standard_normal(d)).astype(np.float32))
    got = K.rmsnorm(x, w, 1e-5)
    ref = orc.rmsnorm(x, w, 1e-5)
    assert _ulps(orc, got, ref).max() <= 1.0


# ------------------------------------------------------------------ GEMM
def _sum_pieces(part, counts=None):
    """Sum the fp32 partial slots in k order (per 128-feature tile for stream-K)."""
    y = part[0].astype(np.float32).copy()
    for s in range(1, part.shape[0]):
        if counts is None:
            y = (y + part[s]).astype(np.float32)
        else:
            for m, c in enumerate(counts):
                if s < c:
                    sl = slice(128 * m, 128 * (m + 1))
                    y[:, sl] = (y[:, sl] + part[s][:, sl]).astype(np.float32)
    return y


def _check_gemm(orc, x, W, part, counts=None):
    xf, Wf = _bf(orc, x), _bf(orc, W)
    y = _sum_pieces(part, counts)
    ref = orc.gemm(x, W, 1).astype(np.float64)
    scale = np.abs(xf) @ np.abs(Wf).T
    err = np.abs(y - ref)
    assert np.all(np.isfinite(y))
    assert np.all(err <= 1e-5 * scale + 1e-30), float((err / (scale + 1e-30)).max())


@pytest.mark.parametrize("T,N,K_,splits,mma_n,tile_n", [
    (1, 128, 64, 1, 0, 16), (5, 256, 256, 1, 0, 16), (16, 384, 512, 2, 16, 16), (17, 256, 256, 1, 0, 32),
    (48, 128, 1024, 3, 16, 64), (64, 512, 4096, 7, 0, 64), (64, 512, 4096, 7, 16, 64), (100, 256, 768, 1, 16, 128),
    (256, 128, 256, 1, 0, 256), (300, 256, 512, 2, 16, 256), (96, 128, 14336, 16, 0, 128), (3, 128, 192, 3, 0, 16),
    (65, 256, 1024, 1, 0, 80), (80, 384, 4096, 5, 16, 80), (170, 128, 512, 2, 0, 80)])
def test_gemm_tcgen05(orc, K, T, N, K_, splits, mma_n, tile_n):
    rng = np.random.default_rng(T * 131 + N + K_)
    x = _rand(orc, rng, (T, K_))
    W = _rand(orc, rng, (N, K_), 1 / np.sqrt(K_))
    part = K.gemm(x, W, splits=splits, impl=0, mma_n=mma_n, tile_n=tile_n)
    assert part.shape == (splits, T, N)
    _check_gemm(orc, x, W, part)
    # each split is the dot product over its own contiguous range of 64-wide k-blocks
    KB = K_ // 64
    for s in range(splits):
        lo = (s * (KB // splits) + min(s, KB % splits)) * 64
        hi = ((s + 1) * (KB // splits) + min(s + 1, KB % splits)) * 64
        sub = orc.gemm(np.ascontiguousarray(x[:, lo:hi]), np.ascontiguousarray(W[:, lo:hi]), 1)
        sc = np.abs(_bf(orc, x[:, lo:hi])) @ np.abs(_bf(orc, W[:, lo:hi])).T
        assert np.all(np.abs(part[s] - sub) <= 1e-5 * sc + 1e-30)


@pytest.mark.parametrize("T,N,K_,G,mma_n,tile_n", [
    (1, 128, 256, 3, 16, 16), (16, 6144, 4096, 148, 16, 16), (64, 4096, 4096, 148, 0, 64),
    (64, 4096, 14336, 148, 16, 64), (33, 1024, 1024, 7, 16, 64), (300, 768, 256, 5, 16, 256),
    (8, 28672 // 8, 4096, 148, 0, 16), (128, 1024, 640, 29, 0, 128)])
def test_gemm_tcgen05_streamk(orc, K, T, N, K_, G, mma_n, tile_n):
    """Stream-K partition (the engine's schedule): tile m's pieces, summed in
    k order, equal the full dot product within the fp32 tolerance; every
    piece is the dot product over exactly its k-block range."""
    rng = np.random.default_rng(T + N + G)
    x = _rand(orc, rng, (T, K_))
    W = _rand(orc, rng, (N, K_), 1 / np.sqrt(K_))
    part = K.gemm(x, W, splits=-G, impl=0, mma_n=mma_n, tile_n=tile_n)
    counts = K.streamk_counts(N, K_, G)
    _check_gemm(orc, x, W, part, counts)
    KB, n_m = K_ // 64, N // 128
    Wk = n_m * KB
    for m in (0, n_m // 2, n_m - 1):
        w0 = m * KB
        first = ((w0 + 1) * G - 1) // Wk
        for p in range(counts[m]):
            i = first + p
            lo = max(i * Wk // G, w0) - w0
            hi = min((i + 1) * Wk // G, w0 + KB) - w0
            sl = slice(128 * m, 128 * (m + 1))
            sub = orc.gemm(np.ascontiguousarray(x[:, 64 * lo:64 * hi]),
                           np.ascontiguousarray(W[sl, 64 * lo:64 * hi]), 1)
            sc = np.abs(_bf(orc, x[:, 64 * lo:64 * hi])) @ np.abs(_bf(orc, W[sl, 64 * lo:64 * hi])).T
            assert np.all(np.abs(part[p][:, sl] - sub) <= 1e-5 * sc + 1e-30), (m, p)


def test_gemm_column_invariance(orc, K):
    """Verifier GEMM (fixed split): a token's output is bit-identical whatever
    other tokens share the launch, wherever its column sits, for any T, tile
    width and MMA instruction width (16 columns or the whole tile) --
    BASELINE north_star: bit-identical at batch 1..B."""
    rng = np.random.default_rng(77)
    N, K_ = 256, 2048
    W = _rand(orc, rng, (N, K_), 1 / np.sqrt(K_))
    target = _rand(orc, rng, (1, K_))
    for splits in (4, -5):  # uniform split-K and the engine's stream-K partition
        ref = K.gemm(target, W, splits=splits, impl=0, mma_n=16, tile_n=16)[:, 0]
        for T in (2, 15, 16, 33, 64, 130, 256, 300):
            others = _rand(orc, rng, (T, K_), 3.0)
            for col in sorted(c for c in {0, 1, 15, T // 2, T - 1} if c < T):
                x = others.copy()
                x[col] = target[0]
                for tile in (16, 32, 64, 80, 128, 256):
                    for mma in sorted({16, tile}):
                        part = K.gemm(x, W, splits=splits, impl=0, mma_n=mma, tile_n=tile)
                        ok = np.isnan(ref) == np.isnan(part[:, col])
                        assert ok.all() and np.array_equal(np.nan_to_num(part[:, col]), np.nan_to_num(ref)), \
                            (T, col, tile, mma)


# ------------------------------------------------------------------ a3 epilogue
@pytest.mark.parametrize("H,KV,hd,bias,S", [(4, 4, 64, False, 1), (32, 8, 128, False, 3), (28, 4, 128, True, 2)])
def test_qkv_epilogue_bit_exact(orc, K, H, KV, hd, bias, S):
    rng = np.random.default_rng(H + KV + S)
    T = 5
    N = (H + 2 * KV) * hd
    part = rng.standard_normal((S, T, N)).astype(np.float32)
    b = orc.f32_to_bf16((0.02 * rng.standard_normal(N)).astype(np.float32)) if bias else None
    pos = np.array([0, 1, 17, 640, 4000], np.int32)
    theta = 1e6 if bias else 5e5
    q, k, v = K.qkv_epilogue(part, b, pos, H, KV, hd, theta)
    acc = part[0]
    for s in range(1, S):
        acc = (acc + part[s]).astype(np.float32)            # splits summed left to right
    rq, rk, rv = orc.qkv_epilogue(acc, b, pos, H, KV, hd, theta)
    assert np.array_equal(q, rq) and np.array_equal(k, rk) and np.array_equal(v, rv)


# ------------------------------------------------------------------ a4
# split_keys: 64 / 128 -> many splits (last-CTA combine); 512 -> 1-2 splits;
# 4096 with 2600 keys -> one split of 163 blocks (> 32 per warp: the
# page-coordinate batches of the ring refill)
@pytest.mark.parametrize("H,KV,hd,sk,stride,nk", [
    (4, 4, 64, 64, 700, (1, 37, 513, 700)), (4, 2, 64, 128, 700, (1, 37, 513, 700)),
    (32, 8, 128, 512, 700, (1, 37, 513, 700)), (40, 8, 128, 64, 700, (1, 37, 513, 700)),
    (28, 4, 128, 128, 700, (1, 37, 513, 700)), (32, 8, 128, 64, 700, (16, 64, 65, 700)),
    (64, 4, 128, 128, 700, (1, 37, 513, 700)), (32, 8, 128, 4096, 2600, (2100, 2600)),
    (8, 8, 64, 4096, 2600, (17, 2600))])
def test_attention(orc, K, H, KV, hd, sk, stride, nk):
    rng = np.random.default_rng(H * hd + sk + stride)
    n_keys = np.array(nk, np.int32)
    T = len(nk)
    q = _rand(orc, rng, (T, H, hd))
    Kc = _rand(orc, rng, (T, KV, stride, hd))
    Vc = _rand(orc, rng, (T, KV, stride, hd))
    o = K.attention(q, Kc, Vc, n_keys, sk)
    vmax = float(np.abs(_bf(orc, Vc)).max())
    for t in range(T):
        n = int(n_keys[t])
        # (1) the PLAIN definition: softmax(q K^T / sqrt(hd)) V
        # in the oracle's chunked form -- one chunk, and 512-key chunks (the
        # verifier's split size) -- each pinned to fp64 in
        # tests/test_oracle_numerics.py.  Derived bound: the kernel and the
        # oracle compute the same exact value in two fp32 orders; the kernel's
        # probabilities enter the PV product as bf16 hi + lo (>= 16 significant
        # bits, relative error <= 2^-16) and each fp32 sum over n keys adds <= n
        # 2^-24 relative, so before the final bf16 rounding the two differ by
        # eps = (2^-15 + n 2^-23) relative to sum_j p_j |v_j| <= vmax -- far
        # below half a bf16 ulp (2^-9): the rounded outputs are equal or 1 ulp
        # apart, except outputs that cancel to ~0, bounded by eps * vmax.
        eps = (2.0 ** -15 + n * 2.0 ** -23) * vmax
        for chunk in (0, 512):
            plain = orc.attention(q[t], Kc[t], Vc[t], n, chunk, 1)
            d = np.abs(_bf(orc, o[t]) - _bf(orc, plain))
            ok = (_ulps(orc, o[t], plain) <= 1.0) | (d <= eps)
            assert ok.all(), (t, chunk, float(_ulps(orc, o[t], plain).max()), float(d.max()), eps)
        # (2) the streamed form of DESIGN.md 3.2 (the kernel's own summation
        # order): the same bound
        ref = orc.attention(q[t], Kc[t], Vc[t], n, -sk, 1)
        ok = (_ulps(orc, o[t], ref) <= 1.0) | (np.abs(_bf(orc, o[t]) - _bf(orc, ref)) <= eps)
        assert ok.all(), t


@pytest.mark.parametrize("H,KV,hd,sk,stride,nk", [
    (32, 8, 128, 4096, 700, (1, 17, 513, 700)), (32, 8, 128, 512, 1300, (600, 1300)),
    (28, 4, 128, 128, 700, (1, 37, 513, 700)), (4, 4, 64, 64, 700, (1, 37, 513, 700))])
def test_attention_two_streams(orc, K, H, KV, hd, sk, stride, nk):
    """The fast path's 2-stream CTAs (grids above one wave of 4-warp CTAs):
    16-key blocks dealt round-robin to 2 warps instead of 4 -- another fp32
    order of the same sums, so test_attention's derived bound against the
    PLAIN chunked definition applies unchanged (one chunk and 512-key chunks)."""
    rng = np.random.default_rng(H * hd + sk + stride + 2)
    n_keys = np.array(nk, np.int32)
    T = len(nk)
    q = _rand(orc, rng, (T, H, hd))
    Kc = _rand(orc, rng, (T, KV, stride, hd))
    Vc = _rand(orc, rng, (T, KV, stride, hd))
    o = K.attention(q, Kc, Vc, n_keys, sk, streams=2)
    vmax = float(np.abs(_bf(orc, Vc)).max())
    for t in range(T):
        n = int(n_keys[t])
        eps = (2.0 ** -15 + n * 2.0 ** -23) * vmax
        for chunk in (0, 512):
            plain = orc.attention(q[t], Kc[t], Vc[t], n, chunk, 1)
            d = np.abs(_bf(orc, o[t]) - _bf(orc, plain))
            ok = (_ulps(orc, o[t], plain) <= 1.0) | (d <= eps)
            assert ok.all(), (t, chunk, float(_ulps(orc, o[t], plain).max()), float(d.max()), eps)


# ------------------------------------------------------------------ a5-a7 epilogues
def test_residual_bit_exact(orc, K):
    rng = np.random.default_rng(5)
    T, N, S = 3, 4096, 4
    x = _rand(orc, rng, (T, N), 4.0)
    part = rng.standard_normal((S, T, N)).astype(np.float32)
    got = K.residual(x, part)
    acc = part[0]
    for s in range(1, S):
        acc = (acc + part[s]).astype(np.float32)
    assert np.array_equal(got, orc.residual(x, acc))


def test_swiglu(orc, K):
    rng = np.random.default_rng(6)
    T, F, S = 3, 1024, 2
    part = (4 * rng.standard_normal((S, T, 2 * F))).astype(np.float32)
    got = K.swiglu(part, F)
    acc = (part[0] + part[1]).astype(np.float32)
    # interleaved-by-64 physical layout: row r of tile r//128 is gate if r%128 < 64
    j = np.arange(F)
    gcol = (j // 64) * 128 + j % 64
    ref = orc.swiglu(acc[:, gcol], acc[:, gcol + 64])
    assert _ulps(orc, got, ref).max() <= 1.0


# ------------------------------------------------------------------ a8, a9
def test_top2_bit_exact(orc, K):
    rng = np.random.default_rng(8)
    T, V = 9, 128256
    L = rng.standard_normal((T, V)).astype(np.float32)
    L[1, 5] = L[1, 77] = 50.0            # duplicated max -> g = 0, lowest id first
    L[2, 1000:1010] = 9.0                # ties
    L[3] = 0.0                           # all equal
    L[4, 3] = np.nan                     # NaN ranks as -inf, flag set
    got = K.top2(L)
    ref = orc.top2(L)
    for k in ("v1", "i1", "v2", "i2", "g"):
        assert np.array_equal(got[k], ref[k]), k
    assert got["nan"] and ref["nan"]
    assert got["i1"][1] == 5 and got["i2"][1] == 77 and got["g"][1] == 0.0
    assert got["i1"][3] == 0 and got["i2"][3] == 1


def test_gate_exact(orc, K):
    rng = np.random.default_rng(9)
    for B in (1, 7, 64, 256):
        g = np.abs(rng.standard_normal(B)).astype(np.float32)
        if B > 4:                           # non-finite margins (A4/A7)
            g[1], g[3] = np.inf, np.nan
        prot = (rng.random(B) < 0.7).astype(np.uint8)
        for tau in (0.0, 0.3, float(g[0]), 1.0, float("inf")):
            trig, rows = K.gate(g, prot, tau)
            ref = orc.gate(g, prot, tau)
            assert np.array_equal(rows, ref)
            assert np.array_equal(np.nonzero(trig)[0], ref)


@pytest.mark.parametrize("T,tile", [(5, 16), (64, 64), (70, 80)])
def test_fused_lm_top2_epilogue(orc, K, T, tile):
    """The LM head's fused top-2 epilogue (mgd_gemm_top2) equals the oracle's
    top-2 (value desc, id asc; NaN as -inf + flag) applied
    to the same tcgen05 GEMM's fp32 logits -- bit for bit, including a tie
    between two rows in different 128-row tiles (lowest id wins, g = 0) and a
    NaN weight row."""
    rng = np.random.default_rng(T * 7 + tile)
    N, K_ = 640, 256
    x = _rand(orc, rng, (T, K_))
    W = _rand(orc, rng, (N, K_), 1 / np.sqrt(K_))
    xf = (x.astype(np.uint32) << 16).view(np.float32)
    row = np.where(xf[0] >= 0, 0x3F00, 0xBF00).astype(np.uint16)   # +-0.5: row . x[0] = 0.5 sum|x0| (maximal)
    W[130] = row
    W[600] = row                                                    # exact tie across tiles 1 and 4
    W[7, 3] = 0x7FC0                                                # NaN weight -> NaN logit in every token
    got = K.gemm_top2(x, W, tile_n=tile)
    logits = K.gemm(x, W, splits=1, impl=0, tile_n=tile)[0]
    ref = orc.top2(logits)
    for k in ("v1", "i1", "v2", "i2", "g"):
        assert np.array_equal(got[k], ref[k]), k
    assert got["nan"] and ref["nan"]
    assert got["i1"][0] == 130 and got["i2"][0] == 600 and got["g"][0] == 0.0
