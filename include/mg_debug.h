/*
 * include/mg_debug.h -- TEST-ONLY op-level entry points of libmargingate.so.
 *
 * Not part of the product ABI.  They launch exactly the kernels the engine
 * launches (same code, same schedules) on caller-provided device buffers, so
 * the parity tests can compare each hot-path kernel with the oracle on
 * identical inputs (SURVEY 8(c) "Parity protocol" step 1), plus hooks to read
 * engine state.  All pointers are DEVICE pointers unless suffixed _host; all
 * work is enqueued on `stream` (cudaStream_t, NULL = default) and the call
 * returns after enqueueing (no synchronisation).  bf16 tensors are uint16_t
 * bit patterns, row-major.  Return: MG_OK or MG_ERR_INVALID / MG_ERR_CUDA.
 */
#ifndef MG_DEBUG_H
#define MG_DEBUG_H

#include "mg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* K0: DESIGN.md 3.1 generator for ONE logical tensor (kind 0..3) into out[n]. */
mg_status mgd_gen_tensor(uint64_t seed, uint32_t tensor_id, int64_t n, int32_t kind, int32_t fan_in,
                         uint16_t* out, void* stream);

/* a2: out[T][d] = bf16((x*inv)*w), inv = 1/sqrtf(sum x^2/d + eps), fixed tree. */
mg_status mgd_rmsnorm(const uint16_t* x, const uint16_t* w, int32_t T, int32_t d, float eps, uint16_t* out,
                      void* stream);

/* GEMM partials: out[s][t][n] = sum_{k in piece s of n's tile} x[t][k] * W[n][k].
 * impl must be 0 (tcgen05, TMA + TMEM; other values: MG_ERR_INVALID).
 * splits > 0: uniform split-K count over 64-wide k-blocks (piece s = split s);
 * splits < 0: stream-K over G = -splits virtual CTAs: CTA i owns k-blocks
 * [i W / G, (i+1) W / G) of the W = (N/128)(K/64) tile-major k-blocks, and
 * the pieces of tile m are numbered in k order (tcgen05 only);
 * mma_n = tcgen05 instruction N
 * (16 = the verifier's pinned slot groups, 0 = whole tile); tile_n = tokens
 * per CTA (16, 32, 64, 128 or 256; 0 = auto).  N % 128 == 0, K % 64 == 0.
 * W is row-major [N][K] here; the call tiles it into the engine's layout. */
mg_status mgd_gemm(const uint16_t* x, const uint16_t* W, int32_t T, int32_t N, int32_t K, int32_t splits,
                   int32_t impl, int32_t mma_n, int32_t tile_n, float* out, void* stream);

/* QKV epilogue: acc = sum_s part[s][t][:] (+bias) -> RoPE(q,k) -> q[T][H*hd],
 * k[T][KV*hd], v[T][KV*hd] (dense outputs, not the paged cache). */
/* LM head with the FUSED top-1/top-2 epilogue (the engine's path):
 * tcgen05 GEMM of x [T][K] by W [N][K] (row-major bf16; N % 128 == 0) whose
 * epilogue writes one top-2 set per (token, 128-row tile), then the tile merge;
 * outputs per token v1, i1, v2, i2, g = v1 - v2 (device), *nan_flag |= 1 on a
 * NaN product sum (ranked -inf).  tile_n 0: the engine's choice. */
mg_status mgd_gemm_top2(const uint16_t* x, const uint16_t* W, int32_t T, int32_t N, int32_t K, int32_t tile_n,
                        float* v1, int32_t* i1, float* v2, int32_t* i2, float* g, int32_t* nan_flag, void* stream);
mg_status mgd_qkv_epilogue(const float* part, int32_t splits, const uint16_t* bias, const int32_t* pos,
                           int32_t T, int32_t H, int32_t KV, int32_t hd, float theta, int32_t max_pos,
                           uint16_t* q, uint16_t* k, uint16_t* v, void* stream);

/* Decode attention over a dense per-token K/V (the streamed form of
 * DESIGN.md 3.3 = oracle or_attention with chunk = -split_keys):
 * q[T][H*hd]; K,V [T][KV][key_stride][hd]; n_keys[T] (1..key_stride); keys
 * cut in splits of split_keys (a multiple of 64), each streamed as 4
 * round-robin 16-key block streams, splits combined in order -> o[T][H*hd].
 * H/KV <= 16.  Blocking; MG_ERR_INVALID on bad sizes. */
mg_status mgd_attention(const uint16_t* q, const uint16_t* K, const uint16_t* V, const int32_t* n_keys, int32_t T,
                        int32_t H, int32_t KV, int32_t hd, int32_t key_stride, int32_t split_keys, uint16_t* o,
                        void* stream);
/* The same with `streams` (2 or 4) round-robin key streams per split: the
 * fast path runs 2 streams when its grid exceeds one wave of 4-warp CTAs
 * (DESIGN.md 7); 4 = mgd_attention. */
mg_status mgd_attention_streams(const uint16_t* q, const uint16_t* K, const uint16_t* V, const int32_t* n_keys,
                                int32_t T, int32_t H, int32_t KV, int32_t hd, int32_t key_stride, int32_t split_keys,
                                int32_t streams, uint16_t* o, void* stream);

/* Measurement floor of bench.py's per-launch roofline timing: an empty kernel
 * with the GEMM's launch shape (one CTA per SM x 192 threads, smem_bytes of
 * dynamic shared memory) bracketed by two CUDA events on `stream`, `reps`
 * times; *us_out = the mean bracketed time in microseconds.  Blocking. */
mg_status mgd_launch_floor(int32_t smem_bytes, int32_t reps, void* stream, float* us_out);

/* out[t][i] = bf16(x[t][i] + sum_s part[s][t][i]) */
mg_status mgd_residual(const uint16_t* x, const float* part, int32_t splits, int32_t T, int32_t N, uint16_t* out,
                       void* stream);

/* a[t][j] = bf16(silu(g) * u), g/u from the interleaved-by-64 gate/up layout
 * of part[s][t][2*F] (physical row r: tile r/128, gate if r%128 < 64). */
mg_status mgd_swiglu(const float* part, int32_t splits, int32_t T, int32_t F, uint16_t* out, void* stream);

/* Top-2 under (value desc, id asc): v1,i1,v2,i2,g per row of logits[T][V];
 * *nan_flag (device int) |= 1 on NaN. */
mg_status mgd_top2(const float* logits, int32_t T, int32_t V, float* v1, int32_t* i1, float* v2, int32_t* i2,
                   float* g, int32_t* nan_flag, void* stream);

/* Gate: trig[b] = prot[b] && g[b] < tau; rows[0..n) ascending; n -> *count. */
mg_status mgd_gate(const float* g, const uint8_t* prot, int32_t B, float tau, uint8_t* trig, int32_t* rows,
                   int32_t* count, void* stream);

/* ---- controlled perturbations (SURVEY 8(b) test-only exports) ---- */
/* SPEC.md:76-84 injected logit noise on the FAST rows' logits (never the
 * verifier's): l[v] += amp * (u * 2^-23) with u = (splitmix64(seed ^ B<<56 ^
 * slot<<44 ^ pos<<20 ^ v) >> 40) - 2^23 -- the formula of the oracle's
 * fast_sched(noise_amp, noise_seed), bit-exact; exactly zero at batch 1.
 * amp = 0 turns it off.  While on, the step runs without CUDA graphs. */
mg_status mgd_set_inject(mg_ctx* ctx, float amp, uint64_t seed);
/* Fast path with the attention split schedule of batch size B_as_if (0: the
 * real batch) -- controlled batch-shape flips without changing the batch. */
mg_status mgd_force_schedule(mg_ctx* ctx, int32_t B_as_if);

/* ---- engine introspection (synchronise; host outputs) ---- */
/* Fast (which=0) or shadow (which=1) column (slot, pos) -> out [L][2][KV][hd] */
mg_status mgd_read_column(mg_ctx* ctx, int32_t which, int32_t slot, int32_t pos, uint16_t* out_host);
/* FNV-1a digest of a whole cache (all active slots, all written positions),
 * excluding (skip_slot, skip_pos) if skip_slot >= 0. */
mg_status mgd_cache_digest(mg_ctx* ctx, int32_t which, int32_t skip_slot, int32_t skip_pos, uint64_t* out_host);
/* Per-row debug record of the LAST decode step: f_tok, g, v1, v2, trig,
 * v_tok (-1), v_g, kind, out (each [B]). */
mg_status mgd_last_step(mg_ctx* ctx, int32_t* f_tok, float* g, float* v1, float* v2, uint8_t* trig,
                        int32_t* v_tok, float* v_g, uint8_t* kind, int32_t* out);
/* Capture the fp32 fast logits [B][V] of subsequent steps into dev_buf (NULL: off). */
mg_status mgd_capture_logits(mg_ctx* ctx, float* dev_buf);

/* From the next step on, after each verifier LM head copy the fp32 logits of
 * the verifier's rows into dev_buf[k][vocab], k = the row's rank among the
 * rows the verifier ran on (ascending batch index): in MG_VERIFY_SYNC and
 * MG_VERIFY_FUSED every protected row of a step whose verifier ran, in
 * MG_VERIFY_PIPELINED the pending rows; nullptr stops.  Disables CUDA graphs
 * while set.  For the tau calibration (eps_pert). */
mg_status mgd_capture_verifier_logits(mg_ctx* ctx, float* dev_buf);
/* Copy the weight tensor (layer, which) as the ORACLE's logical layout
 * (DESIGN.md 3.1 ids) to out_dev. */
mg_status mgd_weight(mg_ctx* ctx, int32_t layer, int32_t which, uint16_t* out_dev, int64_t* n_host);
/* Schedule in force for a T-token launch: writes splits of qkv,o,gu,down,lm,
 * attention chunk, gemm impl, mma_n (8 ints) for det (det=1) or fast (det=0). */
mg_status mgd_schedule(mg_ctx* ctx, int32_t T, int32_t det, int32_t max_ctx, int32_t* out8_host);
/* Kernel launches enqueued by this context since init (the bench's
 * gpu_launches claim). */
mg_status mgd_launch_count(mg_ctx* ctx, uint64_t* out_host);
/* Per-kernel-class event timing of subsequent steps (1 on / 0 off); read back
 * average ms per launch of the GEMM class and the whole step. */
mg_status mgd_set_timing(mg_ctx* ctx, int32_t on);
mg_status mgd_timing(mg_ctx* ctx, double* out8_host);

#ifdef __cplusplus
}
#endif
#endif
