/*
 * oracle/mg_oracle.h -- CPU ORACLE for the MarginGate decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path (paper_2605_30218_b200/csrc, include/mg.h); the two only agree on
 * the DOCUMENTED specification in DESIGN.md section 3 (weight generator,
 * rounding points, schedules-as-data).
 *
 * Paper: arxiv 2605.30218 "MarginGate", /root/reference/PAPER.md.
 *   margin          g = l(1) - l(2)                          PAPER.md:197-201 (S3.1)
 *   trigger         g < tau  (strict)                        PAPER.md:201 (S3.1)
 *   commit / repair fast | verified | repair, one column     PAPER.md:208 (S3.2)
 *   verifier        deterministic in (weights, prefix)       PAPER.md:210 (S3.2)
 *   accounting      r_verify, r_repair                       PAPER.md:215 (S3.3)
 *   protected rows  per-request policy                       PAPER.md:217 (S3.3)
 *   batch variance  "serving shape changes the reduction plan" PAPER.md:35 (S2.1)
 *
 * Parity-pin status of every function is listed in DESIGN.md section 4.
 */
#ifndef MG_ORACLE_H
#define MG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab, qkv_bias;
  float rms_eps, rope_theta;
  uint64_t weight_seed;
} or_cfg;

/* A reduction schedule, as DATA (SPEC numerics
 * "chunked_dot").  split_* = number of contiguous K-chunks of a dot
 * product (remainder to the leading chunks), each chunk summed left to
 * right in fp32, chunk partials summed left to right.  Attention keys
 * 0..q are cut either into attn_chunk-sized chunks (attn_chunk > 0), into
 * attn_splits equal chunks (attn_chunk == 0), or streamed in splits of
 * -attn_chunk keys (attn_chunk < 0: or_attention's streamed form).
 * noise_amp > 0 adds SPEC's test-only injected logit perturbation
 * (SPEC.md:76-84), exactly 0 at batch 1. */
typedef struct {
  int32_t split_qkv, split_o, split_gu, split_down, split_lm;
  int32_t attn_chunk, attn_splits;
  float noise_amp;
  uint64_t noise_seed;
} or_sched;

/* ---- numerics primitives ---- */
uint16_t or_f32_to_bf16(float x);
float    or_bf16_to_f32(uint16_t h);
float    or_dot_bf16(const uint16_t* a, const uint16_t* b, int32_t n, int32_t splits);
uint64_t or_splitmix64(uint64_t x);

/* ---- weight generator ---- */
uint32_t or_tensor_id(const or_cfg* c, int32_t layer, int32_t which);
void     or_gen_tensor(uint64_t seed, uint32_t tensor_id, int64_t n, int32_t kind,
                       int32_t fan_in, uint16_t* out);

/* ---- op-level reference functions (row-major, bf16 as uint16 bits) ---- */
void or_rmsnorm(const uint16_t* x, const uint16_t* w, int32_t T, int32_t d, float eps, uint16_t* out);
void or_gemm(const uint16_t* x, const uint16_t* W, int32_t T, int32_t N, int32_t K, int32_t splits,
             float* out /* [T][N] */);
void or_rope_table(int32_t head_dim, float theta, int32_t pos, float* cos_out, float* sin_out);
void or_qkv_epilogue(const float* acc /* [T][(H+2KV)*hd] */, const uint16_t* bias /* nullable */,
                     const int32_t* pos, int32_t T, int32_t H, int32_t KV, int32_t hd, float theta,
                     uint16_t* q /* [T][H*hd] */, uint16_t* k /* [T][KV*hd] */, uint16_t* v);
void or_attention(const uint16_t* q /* [H][hd] */, const uint16_t* K /* [KV][n][hd] */,
                  const uint16_t* V, int32_t H, int32_t KV, int32_t hd, int32_t n_keys,
                  int32_t key_stride /* >= n_keys */, int32_t chunk, int32_t splits, uint16_t* o /* [H*hd] */);
/* chunk < 0 selects the streamed form (or_attention_stream) with
 * split_keys = -chunk; see DESIGN.md 3.3 / A14. */
void or_residual(const uint16_t* x, const float* acc, int64_t n, uint16_t* out);
void or_swiglu(const float* g, const float* u, int64_t n, uint16_t* out);
/* top-2 under the total order (value desc, id asc); NaN ranks as -inf and
 * sets *nan_flag.  Returns nothing; writes v1,i1,v2,i2,g per row. */
void or_top2(const float* logits, int32_t T, int32_t V, float* v1, int32_t* i1, float* v2,
             int32_t* i2, float* g, int32_t* nan_flag);
/* gate: rows_out[0..n) = ascending b with prot[b] && g[b] < tau.  Returns n. */
int32_t or_gate(const float* g, const uint8_t* prot, int32_t B, float tau, int32_t* rows_out);

/* ---- model + policy ---- */
typedef struct or_model or_model;
typedef struct or_state or_state;

or_model* or_model_create(const or_cfg* cfg);   /* generates all weights */
void      or_model_free(or_model* m);
const uint16_t* or_model_tensor(const or_model* m, int32_t layer, int32_t which, int64_t* n_out);

or_state* or_state_create(const or_model* m, int32_t n_rows, int32_t max_seq);
void      or_state_free(or_state* s);

/* deterministic prefill of `row`: fills the shadow cache
 * with the det schedule, copies it into the fast cache, returns y0. */
int32_t or_prefill(or_state* s, int32_t row, const int32_t* prompt, int32_t len, const or_sched* det,
                   float* logits_out /* nullable [V]: logits at position len-1 */);

/* One MarginGate decode step over rows[0..B) (SURVEY 8(c)
 * step 3).  Outputs per batch position b (all nullable except out_tok):
 *   f_tok, g (fast top-2 margin), fv1/fv2 (fast top-2 values), trig,
 *   v_tok (-1 if not verified), v_g (verifier margin), kind (0 fast,
 *   1 verified, 2 repair), out_tok, fast_logits [B][V].
 * Teacher forcing: if forced_trig != NULL the gate decision is taken
 * from it; if forced_out != NULL the committed token is taken from it and
 * kind==2 (repair) copies the shadow column iff forced_kind says so.
 * Returns the number of triggered rows. */
int32_t or_step(or_state* s, const int32_t* rows, int32_t B, const uint8_t* prot, float tau,
                const or_sched* fast, const or_sched* det,
                const uint8_t* forced_trig, const int32_t* forced_out, const uint8_t* forced_kind,
                int32_t* f_tok, float* g, float* fv1, float* fv2, uint8_t* trig,
                int32_t* v_tok, float* v_g, uint8_t* kind, int32_t* out_tok, float* fast_logits);

/* state introspection (locality digests, parity) */
int32_t  or_state_pos(const or_state* s, int32_t row);
int32_t  or_state_shadow_len(const or_state* s, int32_t row);
int32_t  or_state_token(const or_state* s, int32_t row, int32_t q);
/* copy column (row, pos) of cache (0 fast, 1 shadow) -> out [L][2][KV][hd] */
void     or_state_column(const or_state* s, int32_t which, int32_t row, int32_t pos, uint16_t* out);
/* FNV-1a 64 digest of a cache excluding (skip_row, skip_pos) (skip_row<0: none) */
uint64_t or_state_digest(const or_state* s, int32_t which, int32_t skip_row, int32_t skip_pos);
/* stats: [steps, rows, protected_rows, triggers, verified, repairs, verifier_launches, catchup_tokens, nan] */
void     or_state_stats(const or_state* s, uint64_t* out9);

/* Repair-action ablation: 0 = copy the verifier column on a
 * repair (default), 1 = token-only (leave the BF16 column). */
void     or_state_set_repair_mode(or_state* s, int32_t mode);

/* LLM-42-style windowed verification with rollback over every token
 * committed since the row's last verification (
 * SURVEY 8(f) NEXT-2).  See mg_oracle.c for the exact order.  Returns the
 * number of discarded tokens. */
int32_t  or_verify_window(or_state* s, const int32_t* rows, int32_t n, const or_sched* det,
                          int32_t* new_pos, int32_t* last_tok, int32_t* rolled_back);
/* [window verifies (rows), rollbacks, rolled-back tokens] */
void     or_state_window_stats(const or_state* s, uint64_t* out3);

#ifdef __cplusplus
}
#endif
#endif
