// control.h -- argument blocks of the gate / commit kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mg {

struct GateArgs {
  const float* g;          // [B] fast margins
  const uint8_t* prot;     // [B] or nullptr (all protected)
  float tau;
  const int32_t* slots;    // [B]
  int B;
  const int32_t* pos;      // [max_slots]
  const int32_t* shadow_len;
  const int32_t* hist;
  int hist_stride;
  uint8_t* trig;           // [B]
  int32_t* rank;           // [B] index among gated rows, -1 if not gated
  int32_t* ctrl;           // [2 + B]: n_gated, M, rows...
  int32_t* last;           // [B] catch-up list index of each gated row's last token
  int32_t* cu_slot;        // catch-up list
  int32_t* cu_pos;
  int32_t* cu_tok;
  int32_t* cu_nk;
  // pipelined verification (MG_VERIFY_PIPELINED): when pend != nullptr the
  // rows to verify are the slots with pend[slot] = 1 (their tentative token
  // sits at position pos - 1) instead of prot && g < tau
  const uint8_t* pend;     // [max_slots] or nullptr
  int32_t* rank_slot;      // [max_slots] rank of each listed slot (nullable)
  // fused same-step verification (MG_VERIFY_FUSED): list every protected row
  // (p = pos) before the fast forward, independent of the margin
  int32_t list_protected;
  // synchronous verification with opportunistic eager catch-up
  // (MG_VERIFY_SYNC): the trigger prot && g < tau decides WHETHER the verifier
  // runs this step; when it runs it catches up EVERY protected row of the
  // batch (the list is the protected rows, ascending; trig[] marks them),
  // since its weight pass is paid anyway (A23: the verifier's
  // results do not depend on the chunking).  ran[0] = rows whose gate fired;
  // ctrl[1] = catch-up tokens if ran[0] > 0, else 0.
  int32_t eager;
  int32_t* ran;
  // device-side dispatch (CUDA-graph conditional nodes): the loop over the
  // catch-up chunks (WHILE) and the verifier's LM head (IF) run only when the
  // gate fired; handles are 0 outside a graph.  vctl[0] (chunk cursor) is reset.
  unsigned long long h_loop, h_lm;
  int32_t* vctl;
  unsigned long long* stats;  // [12] += 1 when the LM-head IF body runs (launch accounting)
  const float* tau_d;         // nullable: the step's threshold in device memory (overrides tau)
};
cudaError_t launch_gate(const GateArgs& a, cudaStream_t st);

struct ColCopy {
  const uint16_t* src;
  uint16_t* dst;
  const int32_t* pt;
  int32_t max_pages, page_size, n_pages, L, kv, hd;
};
cudaError_t launch_copy_cols(const ColCopy& c, int slot, int p0, int p1, cudaStream_t st);

struct CommitArgs {
  int B;
  const int32_t* slots;
  const uint8_t* prot;
  int gate_ran;
  const uint8_t* trig;
  const int32_t* rank;
  const int32_t* ctrl;
  const int32_t* f_tok;
  const float* g;
  const int32_t* v_tok;    // [n_gated]
  const float* v_g;
  int32_t* pos;
  int32_t* shadow_len;
  int32_t* hist;
  int hist_stride;
  ColCopy copy;            // shadow -> fast
  int repair_copy;         // 1: copy the verifier column on a repair; 0: token-only
  // MG_VERIFY_FUSED: trig[b] marks the rows whose verifier ran speculatively
  // (every protected row); the gate prot && g < spec_tau decides which of them
  // commit the verifier's result; all of them have their shadow cache caught up
  int spec;
  float spec_tau;
  // MG_VERIFY_SYNC (eager catch-up): the listed rows were verified only if
  // ran[0] > 0 (nullable: always)
  const int32_t* ran;
  const float* tau_d;      // nullable: spec_tau in device memory (overrides spec_tau)
  int32_t* tokens_out;
  uint8_t* kind_out;
  float* margin_out;
  unsigned long long* stats;
  // debug record of the step (nullable)
  int32_t* dbg_vtok;
  float* dbg_vg;
  uint8_t* dbg_kind;
  uint8_t* dbg_trig;
  int32_t* dbg_out;
};
cudaError_t launch_commit(const CommitArgs& a, cudaStream_t st);

// one iteration of the synchronous verifier's chunk loop (device-side
// dispatch): picks the smallest chunk size >= the remaining catch-up tokens
// (the largest if none), writes the chunk's token list (entries past the end
// are no-ops: slot -1, 0 keys), advances the cursor and sets the SWITCH
// (chunk size) and WHILE (more chunks) conditions
struct VChunkArgs {
  const int32_t* ctrl;     // [1] = catch-up tokens M
  int32_t* vctl;           // [0] cursor, [1] base of this chunk
  const int32_t *cu_slot, *cu_pos, *cu_tok, *cu_nk;
  int32_t *v_slot, *v_pos, *v_tok, *v_nk;
  int32_t n_sizes;
  int32_t sizes[8];        // ascending
  unsigned long long h_loop, h_case;
  unsigned long long* stats;  // [11] += 1 per iteration
};
cudaError_t launch_vchunk(const VChunkArgs& a, cudaStream_t st);
// copy a step's committed tokens / kinds / margins from the engine's buffers
// (where a whole-step CUDA graph writes them) to the caller's (kind, margin nullable)
cudaError_t launch_emit(const int32_t* tok, const uint8_t* kind, const float* marg, int B, int32_t* tok_out,
                        uint8_t* kind_out, float* marg_out, cudaStream_t st);
// rows r < ctrl[0] whose last catch-up token lies in this chunk
// (last[r] - vctl[1] in [0, T)): xgn[r] = xn[last[r] - vctl[1]]
cudaError_t launch_gather_last(const uint16_t* xn, const int32_t* last, const int32_t* ctrl, const int32_t* vctl,
                               int T, int n_max, int d, uint16_t* xgn, cudaStream_t st);

// windowed verification (LLM-42 style)
struct WindowArgs {
  int n;
  const int32_t* slots;    // [n]
  const int32_t* off;      // [n] catch-up list offset of each row
  int32_t* pos;            // [max_slots]
  int32_t* shadow_len;
  int32_t* hist;
  int hist_stride;
  int32_t* cu_slot;        // catch-up list (k_window_list writes it)
  int32_t* cu_pos;
  int32_t* cu_tok;
  int32_t* cu_nk;
  const int32_t* v_tok;    // [M] verifier argmax of every catch-up token
  int32_t* res;            // [3n]: new pos, last token, rolled-back count
  unsigned long long* stats;
  uint8_t* pend;           // [max_slots] pipelined-verification flags, cleared (nullable)
};
cudaError_t launch_window_list(const WindowArgs& a, cudaStream_t st);
cudaError_t launch_window_commit(const WindowArgs& a, cudaStream_t st);

// pipelined verification: commit of one step (include/mg.h, MG_VERIFY_PIPELINED)
struct FusedCommitArgs {
  int B;
  const int32_t* slots;
  const uint8_t* prot;     // [B] or nullptr
  float tau;
  int gate_on;             // any protected row && tau > 0
  int had_pend;            // this step verified the pending slots (v_tok valid)
  uint8_t* pend;           // [max_slots]
  const int32_t* rank_slot;
  const int32_t* f_tok;
  const float* g;
  const int32_t* v_tok;    // [n_pend] by rank
  const float* v_g;
  int32_t* pos;
  int32_t* shadow_len;
  int32_t* hist;
  int hist_stride;
  ColCopy copy;            // shadow -> fast
  int repair_copy;
  int32_t* tokens_out;
  uint8_t* kind_out;
  float* margin_out;
  unsigned long long* stats;
  int32_t n_pend, M;       // verifier accounting of this step
  int32_t* dbg_vtok;
  float* dbg_vg;
  uint8_t* dbg_kind;
  uint8_t* dbg_trig;
  int32_t* dbg_out;
};
cudaError_t launch_commit_fused(const FusedCommitArgs& a, cudaStream_t st);
// mixed token list: rows [0,B) the fast rows (slot, pos, hist[pos], pos+1),
// rows [B, B+M) a copy of the catch-up list cu_*[0, M)
cudaError_t launch_prepare_mixed(const int32_t* slots, int B, const int32_t* pos, const int32_t* hist, int hist_stride,
                                 const int32_t* cu_slot, const int32_t* cu_pos, const int32_t* cu_tok,
                                 const int32_t* cu_nk, int M, const int32_t* ctrl /* [1] = real M */,
                                 int32_t* m_slot, int32_t* m_pos, int32_t* m_tok, int32_t* m_nk, cudaStream_t st);
// LM-head input rows: dst[i] = src[i] for i < B, dst[B + r] = src[B + last[min(r, ctrl[0]-1)]] for r < n
cudaError_t launch_lm_rows(const uint16_t* src, int B, const int32_t* last, const int32_t* ctrl, int n, int d,
                           uint16_t* dst, cudaStream_t st);

// test-only SPEC.md:76-84 logit perturbation of the fast rows (mgd_set_inject)
cudaError_t launch_inject(float* logits, int B, int V, float amp, unsigned long long seed, const int32_t* slot,
                          const int32_t* pos, cudaStream_t st);

cudaError_t launch_prepare(const int32_t* slots, int B, const int32_t* pos, const int32_t* hist, int hist_stride,
                           int32_t* f_slot, int32_t* f_pos, int32_t* f_tok, int32_t* f_nk, cudaStream_t st);
cudaError_t launch_prefill_done(int32_t* hist, int hist_stride, int32_t* pos, int32_t* shadow_len, int slot, int len,
                                const int32_t* tok, cudaStream_t st);
cudaError_t launch_gather_rows_sub(const uint16_t* src, const int32_t* rows, int sub, int n, int d, uint16_t* dst,
                                   cudaStream_t st);

}  // namespace mg
