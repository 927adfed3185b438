// engine.h -- the per-context state of libmargingate (internal).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mg.h"
#include "control.h"
#include "kernels.h"

namespace mg {

struct OpSched {
  int impl;    // 0 tcgen05, 1 CUDA-core
  int splits;  // uniform split-K over 64-wide k-blocks (G == 0)
  int G;       // stream-K virtual CTAs per token tile (0 = uniform split-K)
  int N, K;    // weight shape (for the partial layout)
  PartSpec ps() const { return PartSpec{splits, G, K / 64, N / 128}; }
  int tile_n;  // tokens per CTA (tcgen05)
  int mma_n;   // tcgen05 instruction N
};
struct Sched {
  OpSched qkv, o, gu, down, lm;
  int attn_sk, attn_ns;  // attention: keys per split, grid splits
};

struct Weight {
  uint16_t* ptr = nullptr;
  int N = 0, K = 0;
  CUtensorMap map;
};

struct LayerW {
  uint16_t *attn_norm, *mlp_norm, *bqkv;
  Weight qkv, o, gu, down;
};

struct Timing {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  // pairs: (start idx, stop idx, class)  class 0 gemm, 1 attention, 2 step
  std::vector<std::tuple<size_t, size_t, int, double>> rec;  // double = algorithmic bytes
};

}  // namespace mg

struct mg_ctx {
  mg_config cfg{};
  mg_buffers buf{};
  cudaStream_t st = nullptr;
  std::string err;
  bool dead = false;
  int dev = 0;

  // derived shape
  int L, d, H, KV, hd, F, V, NQ, NK, NQKV;
  int Tv;     // verifier / prefill chunk (tokens)
  int Tmax;   // activation rows
  int PS, max_pages, n_pages;
  int nb_top2;

  // weights
  uint16_t *embed, *final_norm;
  mg::Weight lm;
  std::vector<mg::LayerW> layers;

  // caches
  uint16_t *kv_fast, *kv_shadow;

  // workspace
  uint16_t *x, *xn, *q, *att, *a, *xg, *xgn;
  float *part, *logits, *attn_acc, *attn_ml, *top2_part;
  float* t2tiles = nullptr;  // fused LM-head top-2: per-(token, 128-row tile) sets [Tlm][V/128][4]
  int32_t* attn_cnt;                     // [Tmax][KV] chunk-arrival counters
  int fast_sk_override = 0;  // MG_FAST_SK (measurement)
  int verify_mode = 0;       // mg_verify_mode (mg_set_policy)
  uint8_t* pend_d = nullptr;  // [max_slots] pipelined verification: tentative token pending
  int32_t* rank_slot_d = nullptr;
  int32_t *mx_slot, *mx_pos, *mx_tok, *mx_nk;  // mixed token list [Tmax]
  uint16_t* xlm = nullptr;   // LM-head input rows [2 * max_batch][d]
  int32_t* fpin = nullptr;   // pinned readback of a pipelined step: ctrl | last | pos | shadow | pend
  cudaEvent_t fev = nullptr;
  bool f_sync = false;       // a pipelined step's readback is in flight
  bool pend_dirty = false;   // pending set changed outside a step (mg_verify_window / mg_release)
  std::vector<char> pend_h;
  int fast_mode = 0;         // mg_fast_schedule (mg_set_policy)
  bool lm_unfused = false;   // MG_LM_UNFUSED=1: fp32 logits + separate top-2 (A/B measurement)
  float inj_amp = 0.f;       // test-only logit perturbation (mgd_set_inject)
  unsigned long long inj_seed = 0;
  int force_B = 0;           // test-only: fast attention splits of another batch size (mgd_force_schedule)
  int repair_mode = 0;       // mg_repair_action
  int det_sk = 512;          // verifier attention keys per split (A14; MG_DET_SK for measurement)
  CUtensorMap attn_qmap, kv_map[2];      // TMA maps: q [Tmax][H][hd]; pools (fast, shadow)
  float *rope_cos, *rope_sin;
  size_t part_elems;
  // device state
  int32_t *pos_d, *shadow_d, *hist_d, *pt_d;
  unsigned long long* stats_d;
  int32_t* nan_d;
  // batch / step buffers
  int32_t *slots_d, *f_slot, *f_pos, *f_tok, *f_nk, *f_i2;
  uint8_t* prot_d;
  // a step's host inputs, one H2D copy into batch_d: [slots: max_batch][prot
  // bytes: ceil(max_batch/4) words][tau][3 pad][page-table updates: 2 per row]
  int32_t* batch_d = nullptr;
  float* tau_d = nullptr;
  int32_t* ptu_d = nullptr;
  int batch_pw = 0;
  float *f_g, *f_v1, *f_v2;
  uint8_t* trig_d;
  int32_t *rank_d, *ctrl_d, *last_d;
  int32_t *cu_slot, *cu_pos, *cu_tok, *cu_nk;
  int32_t *v_tok, *v_i2;
  int32_t *w_tok, *w_res;  // window verify: argmax per catch-up token [B*max_seq]; results [3B]
  float *v_g, *v_v1, *v_v2;
  int32_t* staging_d;  // uploads: [slots | prot bytes | pt updates]
  // debug record
  int32_t *dbg_vtok, *dbg_out;
  float* dbg_vg;
  uint8_t *dbg_kind, *dbg_trig;
  float* capture = nullptr;    // fast logits [B][V] of the next steps (mgd_capture_logits)
  float* capture_v = nullptr;  // verifier logits [gated rank][V] (mgd_capture_verifier_logits)
  int last_B = 0;

  // host mirrors
  std::vector<int> pos_h, shadow_h;
  std::vector<char> active;
  std::vector<std::vector<int>> pages;
  std::vector<int> free_pages;
  int32_t* pinned = nullptr;  // 2 staging regions + ctrl
  size_t pinned_words = 0, stage_words = 0;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  int stage_idx = 0;

  std::map<std::tuple<const void*, int, int, int>, CUtensorMap> xmaps;
  unsigned long long launches = 0;   // kernels enqueued (conditional bodies: mgd_launch_count adds them)
  mg::Timing timing;

  // CUDA graphs of the launch sequences (fast step per (B, attention chunks);
  // verifier chunks per (T, chunks, offsets)); captured on the second use
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int seen = 0;
    unsigned long long launches = 0;
  };
  std::map<std::tuple<int, int, int, int, int, int>, GraphEntry> graphs;
  bool use_graphs = true;
  cudaStream_t cap_st = nullptr;  // private capture stream
  cudaStream_t cap_st2 = nullptr; // capture of conditional-node bodies

  // synchronous verification, device-side dispatch (engine.cu decode_sync)
  int32_t *vx_slot = nullptr, *vx_pos = nullptr, *vx_tok = nullptr, *vx_nk = nullptr;  // chunk list [Tmax]
  int32_t* vctl_d = nullptr;  // [4] chunk cursor
  int32_t* ran_d = nullptr;   // [1] rows whose gate fired this step
  int32_t* o_tok_d = nullptr; // a whole-step graph's outputs [max_batch] (then copied to the caller's)
  uint8_t* o_kind_d = nullptr;
  float* o_marg_d = nullptr;
  int32_t* spin = nullptr;    // pinned readback of the eager (debug) path: ctrl | last | ran
  bool shadow_stale = false;  // shadow_h not refreshed since a graph-dispatched sync step
  unsigned long long cond_body_launches = 0, cond_lm_launches = 0;  // kernels per loop iteration / LM body
};
