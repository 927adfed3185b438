/*
 * include/mg.h -- C ABI of the B200-native MarginGate decode engine.
 *
 * Paper: arxiv 2605.30218 "MarginGate".  One call
 * of mg_decode_step is one MarginGate decode step (PAPER.md:185-217,
 * Fig. fig:margingate_arch):
 *   BF16 batched fast forward that tentatively appends the K/V column
 *    -> fused top-1/top-2 margin g = l(1) - l(2)
 *    -> gate  protected && g < tau
 *   -> deterministic verifier on the gated rows ->
 *   fast / verified / repair commit of the single current column
 *    -> r_verify / r_repair accounting.
 *
 * Conventions:
 *  - Every entry point returns mg_status; nothing throws or aborts across the
 *    ABI.  MG_ERR_INVALID and MG_ERR_CAPACITY leave the context unchanged.
 *    MG_ERR_CUDA is sticky: the context is dead, only mg_destroy is legal.
 *  - Ownership: the caller allocates the four device buffers reported by
 *    mg_query_sizes (e.g. with torch) and keeps them alive until mg_destroy.
 *    The context owns host metadata, CUDA events and tensor maps.
 *  - Synchrony: all work is ordered on the stream given to mg_init.
 *    mg_decode_step returns once the step is enqueued and never waits on the
 *    device: in MG_VERIFY_SYNC the step is one CUDA graph whose verifier runs
 *    behind device-side conditions (graph conditional nodes: WHILE over the
 *    catch-up chunks, SWITCH on the chunk size, IF on the verifier's LM head)
 *    set by the gate kernel.  Exceptions, all debug or first-use: the first
 *    step of a new (batch, protected-count) shape and steps with logit
 *    captures / timing / injected noise (include/mg_debug.h) run the same
 *    kernels eagerly and read the gate back once.  The slots, the mask and
 *    the threshold travel in the step's single H2D copy and the graph reads
 *    them from device memory, so a per-step threshold costs nothing extra.
 *    Device outputs are valid after stream completion.  mg_stats,
 *    mg_prefill and mg_verify_window synchronise.
 *  - Host arrays: the slots and the protection mask of a step are HOST
 *    arrays (SURVEY 8(b) lists device pointers): the host owns the page
 *    allocator and the capacity checks (MG_ERR_CAPACITY before any state
 *    change), which need the slots without a device round trip; the mask
 *    travels with the slots in the step's single H2D copy.
 *  - Threading: one context = one host thread.  Not thread-safe.
 *  - Arrays whose name ends in _host are host memory, _dev device memory.
 */
#ifndef MG_H
#define MG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MG_OK = 0,
  MG_ERR_INVALID = 1,   /* bad argument; no state change                       */
  MG_ERR_CAPACITY = 2,  /* position would reach max_seq / pages exhausted      */
  MG_ERR_CUDA = 3,      /* CUDA error; sticky, context unusable                */
  MG_ERR_STATE = 4,     /* call not legal in this state (e.g. slot inactive)   */
  MG_ERR_NUMERIC = 5    /* a logit was NaN (reported by mg_stats)              */
} mg_status;

typedef struct mg_ctx mg_ctx; /* opaque */

/* Model shape + capacity.  Shapes of the named models: SURVEY.md 2.3
 * [public cfg]; init of weights: DESIGN.md 3.1 (counter PRNG, weight_seed). */
typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab, qkv_bias;
  float rms_eps, rope_theta;
  uint64_t weight_seed;
  int32_t max_batch;   /* rows per decode step, 1..256                         */
  int32_t max_slots;   /* concurrent requests                                  */
  int32_t max_seq;     /* positions per request (prompt + decode)              */
  int32_t page_size;   /* K/V page size in tokens (16, 32 or 64)               */
  int32_t verify_chunk;/* max tokens per verifier/prefill launch (0: 512)       */
} mg_config;

/* Bytes of each caller-owned device buffer (256-byte aligned). */
typedef struct {
  size_t weights, kv_fast, kv_shadow, workspace;
} mg_sizes;

typedef struct {
  void *weights, *kv_fast, *kv_shadow, *workspace;
} mg_buffers;

/* Device-side counters, summed over all steps since mg_init.
 * r_verify = triggers / protected_rows, r_repair = repairs / protected_rows
 * (PAPER.md:215).  protected_rows counts the gate decisions of protected rows
 * (in MG_VERIFY_PIPELINED a kind-4 replacement step makes none: its fast
 * output is dropped), so r_verify = 1 at tau = +inf in every verify mode.
 * verifier_launches / catchup_tokens count the verifier's work: in
 * MG_VERIFY_SYNC every protected row is caught up when the verifier runs, in
 * MG_VERIFY_FUSED on every step (speculative); tentative tokens resolved by
 * mg_verify_window count as window_rows, not as verified / repairs. */
typedef struct {
  uint64_t steps, rows, protected_rows, triggers, verified, repairs, verifier_launches, catchup_tokens;
  /* windowed verification (mg_verify_window): rows verified, rows rolled
   * back, committed tokens discarded by rollbacks */
  uint64_t window_rows, rollbacks, rolled_back_tokens;
  uint32_t error_flags; /* bit0: NaN logit seen */
} mg_stats_t;

/* Fast-path schedule (mg_set_policy).
 *   MG_FAST_BATCH_SHAPED     the performance-chosen plan sched_fast(B) whose
 *                            attention splits depend on the batch -- the
 *                            paper's source of batch variance;
 *                            default.
 *   MG_FAST_BATCH_INVARIANT  every row runs the verifier's pinned schedule:
 *                            the "global intervention" baseline of PAPER.md:227
 *                            (Batch-Invariant Ops). */
typedef enum { MG_FAST_BATCH_SHAPED = 0, MG_FAST_BATCH_INVARIANT = 1 } mg_fast_schedule;
/* Repair action on a verifier disagreement (mg_set_policy).
 *   MG_REPAIR_COLUMN      emit the verifier token AND copy the verifier's K/V
 *                         column p into the fast cache; default.
 *   MG_REPAIR_TOKEN_ONLY  emit the verifier token, keep the tentative BF16
 *                         column: the ablation of PAPER.md:317. */
typedef enum { MG_REPAIR_COLUMN = 0, MG_REPAIR_TOKEN_ONLY = 1 } mg_repair_action;
/* When the verifier runs (mg_set_policy).
 *   MG_VERIFY_SYNC       the gated rows of a step are verified inside the same
 *                        mg_decode_step, before it commits;
 *                        every row's token is final when emitted; default.
 *                        The verifier runs only when some protected row's gate
 *                        fires; when it runs it catches up the
 *                        shadow cache of EVERY protected row of the batch
 *                        (its weight pass is paid anyway; results do not
 *                        depend on the chunking, A23) and computes
 *                        the LM head of every protected row -- only the fired
 *                        rows commit the verifier token.
 *   MG_VERIFY_PIPELINED  a gated row's token is emitted TENTATIVELY (kind 3)
 *                        and verified in the slot's next step, whose forward
 *                        carries the verifier's catch-up tokens as extra GEMM
 *                        columns of the same weight pass (the native-runtime
 *                        lever of PAPER.md:393; SURVEY 7 "hard parts").  If the
 *                        verifier disagrees, that next step emits kind 4: the
 *                        verifier token REPLACES the slot's last emitted token,
 *                        its K/V column is repaired and the slot
 *                        does not advance.  The committed sequences equal the
 *                        MG_VERIFY_SYNC ones (the fast path of a row does not
 *                        depend on the other rows).  A slot with a pending token
 *                        must be in the next batch (else MG_ERR_STATE) or be
 *                        resolved with mg_verify_window.
 *   MG_VERIFY_FUSED      the synchronous semantics (same committed tokens,
 *                        kinds and step) at the pipelined cost: every
 *                        protected row's verifier token for the CURRENT step
 *                        is computed speculatively inside the step's own
 *                        weight pass (catch-up tokens as extra GEMM columns),
 *                        and the gate prot && g < tau only selects whose
 *                        verifier token is used.  r_verify counts the gated
 *                        rows as before; verifier_launches / catchup_tokens
 *                        count the speculative work (every protected row). */
typedef enum { MG_VERIFY_SYNC = 0, MG_VERIFY_PIPELINED = 1, MG_VERIFY_FUSED = 2 } mg_verify_mode;

/* Sizes the four buffers for `cfg`.  MG_ERR_INVALID on unsupported shapes
 * (d_model % 64, d_ff % 64, (H+2KV)*hd % 128, vocab % 128, head_dim in
 * {64,128}, H % KV). */
mg_status mg_query_sizes(const mg_config* cfg, mg_sizes* out);

/* Creates a context on the current CUDA device, generates the weights into
 * bufs->weights and captures nothing else.  `cuda_stream` is
 * a cudaStream_t (NULL = legacy default stream). */
mg_status mg_init(const mg_config* cfg, const mg_buffers* bufs, void* cuda_stream, mg_ctx** out);

/* Deterministic prefill of request `slot`: runs the pinned
 * verifier schedule over prompt_host[0..len) into the shadow cache, copies the
 * columns into the fast cache and writes the first token (argmax, not gated)
 * to *first_token_host.  Synchronises.  The slot becomes active.
 * MG_ERR_STATE if the slot is already active; MG_ERR_CAPACITY if len+1 >
 * max_seq or pages run out; MG_ERR_INVALID for len < 1 or token ids out of
 * range. */
mg_status mg_prefill(mg_ctx* ctx, int32_t slot, const int32_t* prompt_host, int32_t len,
                     int32_t* first_token_host);

/* One MarginGate decode step over `batch` active, distinct slots.
 *   slots_host[b]          request of row b
 *   protected_host[b]      1 = the row is gated; NULL = all rows
 *   threshold              tau >= 0; 0 = pure BF16 (r_verify = 0), +INFINITY =
 *                          always-on verification (r_verify = 1)
 *   tokens_out_dev[b]      committed token (int32)
 *   kind_out_dev[b]        nullable: 0 fast, 1 verified, 2 repair; MG_VERIFY_PIPELINED:
 *                          0 final, 1 final (the previous tentative token was
 *                          verified), 3 tentative, 4 the token REPLACES the
 *                          slot's previous (tentative) token, no new token
 *   margin_out_dev[b]      nullable: fp32 margin g of the fast logits
 * Each row consumes its last committed token at position p and commits exactly
 * one token.  MG_ERR_INVALID: batch not in [1, max_batch], inactive or
 * duplicate slot, tau NaN or < 0.  MG_ERR_CAPACITY: a row's position p has
 * reached max_seq (columns are 0 .. max_seq - 1) or pages run out. */
mg_status mg_decode_step(mg_ctx* ctx, const int32_t* slots_host, int32_t batch, const uint8_t* protected_host,
                         float threshold, int32_t* tokens_out_dev, uint8_t* kind_out_dev, float* margin_out_dev);

/* Selects the fast-path schedule, the repair action and the verify mode for
 * later steps (values of mg_fast_schedule / mg_repair_action /
 * mg_verify_mode).  MG_ERR_INVALID for unknown values, MG_ERR_STATE when the
 * verify mode changes while tentative tokens are pending (no state change). */
mg_status mg_set_policy(mg_ctx* ctx, int32_t fast_schedule, int32_t repair_action, int32_t verify_mode);

/* LLM-42-style windowed verification with rollback ("keeps the
 * default path but verifies every token", "verifier setting
 * K=64", "restart-from-rollback").  For each
 * of the n active, distinct slots in slots_host, every token committed since
 * the slot's last verification (positions shadow_len+1 .. p) is checked in
 * order against the deterministic verifier run over the committed prefix
 * (the pinned schedule, shadow cache, reading A1).  At the first disagreement
 * at position m the slot ROLLS BACK: the verifier token replaces the token at
 * m, the tokens after m are discarded, and the next decode step consumes
 * position m.  Outputs (host, nullable, n entries): pos_host = the position
 * of the slot's last committed token after the call, last_token_host = that
 * token, rolled_back_host = tokens discarded.  Synchronises.  Cost: one
 * verifier forward over all unverified tokens of the n slots (chunks of
 * verify_chunk tokens) with the LM head on every one.  MG_ERR_INVALID for
 * n not in [1, max_batch] or an inactive / duplicate slot. */
mg_status mg_verify_window(mg_ctx* ctx, const int32_t* slots_host, int32_t n, int32_t* pos_host,
                           int32_t* last_token_host, int32_t* rolled_back_host);

/* Synchronises the stream and copies the counters; returns MG_ERR_NUMERIC if
 * a NaN logit was seen (counters still written). */
mg_status mg_stats(mg_ctx* ctx, mg_stats_t* out_host);

/* Frees the slot's pages; the slot may be prefilled again. */
mg_status mg_release(mg_ctx* ctx, int32_t slot);

void mg_destroy(mg_ctx* ctx);

/* Last error message of this context (or of the last failed mg_init when
 * ctx == NULL).  Valid until the next call on the context. */
const char* mg_last_error(const mg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
