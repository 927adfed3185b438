// control.cu -- margin, gate, verifier bookkeeping and commit
// (SURVEY 8(a) rows a8 (top-2), a9, a10 bookkeeping, a11).
//
// k_top2_partial / k_top2_final: top-1/top-2 of fp32 logits under the total
// order (value desc, id asc) -- exact, so any merge order gives the same
// (v1,i1,v2,i2); g = v1 - v2 is one IEEE subtraction.
// k_gate: trig = prot && g < tau, ballot/popc
// compaction in ascending row order, catch-up token list of every gated row
// (positions shadow_len..p, A1).
// k_commit: fast / verified / repair: a repair copies the
// verifier's column p of every layer (K and V) from the shadow cache into
// the fast cache and emits the verifier token; nothing else is written.
#include <climits>

#include "common.cuh"
#include "control.h"
#include "kernels.h"

namespace mg {

int top2_blocks(int V) {
  int nb = (V + 8191) / 8192;
  return nb < 1 ? 1 : (nb > 64 ? 64 : nb);
}

// grid (T, nb), 256 threads; block b scans [b*V/nb, (b+1)*V/nb)
__global__ void __launch_bounds__(256) k_top2_partial(const float* __restrict__ logits, int V, int nb,
                                                      float* __restrict__ part, int32_t* __restrict__ nan_flag) {
  griddep();
  __shared__ Top2 sm[8];
  const int t = blockIdx.x, b = blockIdx.y;
  const int lo = chunk_start(V, nb, b), hi = chunk_start(V, nb, b + 1);
  const float* l = logits + (size_t)t * V;
  Top2 r{-INFINITY, INT_MAX, -INFINITY, INT_MAX};
  bool nan = false;
  for (int j = lo + threadIdx.x; j < hi; j += 256) {
    float v = l[j];
    if (v != v) { nan = true; v = -INFINITY; }
    t2_push(r, v, j);
  }
  if (nan) atomicOr(nan_flag, 1);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) r = t2_merge(r, t2_shfl(r, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    Top2 a = sm[0];
    for (int w = 1; w < 8; ++w) a = t2_merge(a, sm[w]);
    float* p = part + ((size_t)t * nb + b) * 4;
    p[0] = a.v1; p[1] = __int_as_float(a.i1); p[2] = a.v2; p[3] = __int_as_float(a.i2);
  }
}

__global__ void k_top2_final(const float* __restrict__ part, int nb, float* v1, int32_t* i1, float* v2,
                             int32_t* i2, float* g) {
  griddep();
  const int t = blockIdx.x;
  if (threadIdx.x != 0) return;
  const float* p = part + (size_t)t * nb * 4;
  Top2 a{p[0], __float_as_int(p[1]), p[2], __float_as_int(p[3])};
  for (int b = 1; b < nb; ++b) {
    const float* q = p + b * 4;
    a = t2_merge(a, Top2{q[0], __float_as_int(q[1]), q[2], __float_as_int(q[3])});
  }
  if (v1) v1[t] = a.v1;
  if (i1) i1[t] = a.i1;
  if (v2) v2[t] = a.v2;
  if (i2) i2[t] = a.i2;
  if (g) g[t] = __fsub_rn(a.v1, a.v2);
}

cudaError_t launch_top2(const float* logits, int T, int V, float* part, int nb, float* v1, int32_t* i1, float* v2,
                        int32_t* i2, float* g, int32_t* nan_flag, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  dim3 g1(T, nb);
  cudaError_t e = launch_k(k_top2_partial, g1, dim3(256), 0, st, logits, V, nb, part, nan_flag);
  if (e != cudaSuccess) return e;
  return launch_k(k_top2_final, dim3(T), dim3(32), 0, st, (const float*)part, nb, v1, i1, v2, i2, g);
}

// merge of the per-tile top-2 sets written by the LM head's fused epilogue:
// CTA per token, 256 threads, strided merge then warp and CTA trees
__global__ void __launch_bounds__(256) k_top2_tiles(const float* __restrict__ t2, int nt, float* v1, int32_t* i1,
                                                    float* v2, int32_t* i2, float* g) {
  griddep();
  __shared__ Top2 sm[8];
  const int t = blockIdx.x;
  const float4* p = reinterpret_cast<const float4*>(t2) + (size_t)t * nt;
  Top2 r{-INFINITY, INT_MAX, -INFINITY, INT_MAX};
  for (int j = threadIdx.x; j < nt; j += 256) {
    const float4 q = p[j];
    r = t2_merge(r, Top2{q.x, __float_as_int(q.y), q.z, __float_as_int(q.w)});
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) r = t2_merge(r, t2_shfl(r, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    Top2 a = sm[0];
    for (int w = 1; w < 8; ++w) a = t2_merge(a, sm[w]);
    if (v1) v1[t] = a.v1;
    if (i1) i1[t] = a.i1;
    if (v2) v2[t] = a.v2;
    if (i2) i2[t] = a.i2;
    if (g) g[t] = __fsub_rn(a.v1, a.v2);
  }
}

cudaError_t launch_top2_tiles(const float* t2, int T, int nt, float* v1, int32_t* i1, float* v2, int32_t* i2,
                              float* g, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  return launch_k(k_top2_tiles, dim3(T), dim3(256), 0, st, t2, nt, v1, i1, v2, i2, g);
}

// ------------------------------------------------------------------ gate
// The trigger g < tau, strict, with DESIGN.md A4/A7 for the
// non-finite cases: tau = +inf fires for every margin (always-on, r_verify = 1,
// PAPER.md:215), a NaN margin (all logits NaN) fires for any tau > 0.
MG_DEV bool gate_fires(float g, float tau) { return tau > 0.f && (g < tau || isinf(tau) || g != g); }

// Single CTA of 1024 threads (B <= 1024).  Row b = thread b.
__global__ void __launch_bounds__(1024) k_gate(GateArgs a) {
  griddep();
  __shared__ int wsum[32], wgap[32];
  __shared__ int s_fired;
  const int b = threadIdx.x, warp = b >> 5, lane = b & 31;
  const bool valid = b < a.B;
  int slot = 0, p = 0, s0 = 0;
  bool tr = false;
  if (b == 0) s_fired = 0;
  __syncthreads();
  if (valid) {
    slot = a.slots[b];
    p = a.pos[slot];
    s0 = a.shadow_len[slot];
    if (a.pend) {  // pipelined verification: the tentative token sits at position p (= pos - 1 here)
      tr = a.pend[slot] != 0;
      p -= 1;
    } else if (a.list_protected) {  // fused verification: every protected row, before its margin exists
      tr = a.prot ? a.prot[b] != 0 : true;
    } else if (a.eager) {  // synchronous: list every protected row, count the rows whose gate fires
      tr = a.prot ? a.prot[b] != 0 : true;
      if (tr && gate_fires(a.g[b], a.tau_d ? *a.tau_d : a.tau)) atomicAdd(&s_fired, 1);  // strict <
    } else {
      const bool prot = a.prot ? a.prot[b] != 0 : true;
      tr = prot && gate_fires(a.g[b], a.tau_d ? *a.tau_d : a.tau);  // strict <
    }
  }
  const int gap = tr ? (p - s0 + 1) : 0;
  // exclusive scans of trig flags and gaps (ascending row order)
  const unsigned bal = __ballot_sync(0xffffffffu, tr);
  int rank_in_warp = __popc(bal & ((1u << lane) - 1u));
  int g_incl = gap;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, g_incl, off);
    if (lane >= off) g_incl += v;
  }
  if (lane == 31) { wsum[warp] = __popc(bal); wgap[warp] = g_incl; }
  __syncthreads();
  if (b == 0) {
    int acc = 0, accg = 0;
    for (int w = 0; w < 32; ++w) {
      const int c = wsum[w], cg = wgap[w];
      wsum[w] = acc; wgap[w] = accg;
      acc += c; accg += cg;
    }
    if (a.eager && s_fired == 0) accg = 0;  // nothing fired: no verifier this step
    a.ctrl[0] = acc;   // number of listed rows
    a.ctrl[1] = accg;  // catch-up tokens M
    if (a.eager) {
      a.ran[0] = s_fired;
      if (a.vctl) a.vctl[0] = 0;
      if (a.h_loop) cudaGraphSetConditional(a.h_loop, accg > 0 ? 1u : 0u);
      if (a.h_lm) cudaGraphSetConditional(a.h_lm, s_fired > 0 ? 1u : 0u);
      if (a.h_lm && a.stats && s_fired > 0) atomicAdd(&a.stats[12], 1ull);
    }
  }
  __syncthreads();
  if (!valid) return;
  a.trig[b] = tr ? 1 : 0;
  if (!tr) { a.rank[b] = -1; return; }
  const int r = wsum[warp] + rank_in_warp;
  const int off = wgap[warp] + g_incl - gap;
  a.rank[b] = r;
  if (a.rank_slot) a.rank_slot[slot] = r;
  a.ctrl[2 + r] = b;
  a.last[r] = off + gap - 1;
  const int32_t* h = a.hist + (size_t)slot * a.hist_stride;
  for (int q = s0; q <= p; ++q) {
    const int e = off + (q - s0);
    a.cu_slot[e] = slot;
    a.cu_pos[e] = q;
    a.cu_tok[e] = h[q];
    a.cu_nk[e] = q + 1;
  }
}

cudaError_t launch_gate(const GateArgs& a, cudaStream_t st) {
  if (a.B > 1024) return cudaErrorInvalidValue;
  return launch_k(k_gate, dim3(1), dim3(1024), 0, st, a);
}

// ------------------------------------------------------------------ prepare
// fast-path token list: slot, position p = pos[slot], input token hist[slot][p]
__global__ void k_prepare(const int32_t* __restrict__ slots, int B, const int32_t* __restrict__ pos,
                          const int32_t* __restrict__ hist, int hist_stride, int32_t* f_slot, int32_t* f_pos,
                          int32_t* f_tok, int32_t* f_nk) {
  griddep();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int s = slots[b], p = pos[s];
  f_slot[b] = s;
  f_pos[b] = p;
  f_tok[b] = hist[(size_t)s * hist_stride + p];
  f_nk[b] = p + 1;
}

cudaError_t launch_prepare(const int32_t* slots, int B, const int32_t* pos, const int32_t* hist, int hist_stride,
                           int32_t* f_slot, int32_t* f_pos, int32_t* f_tok, int32_t* f_nk, cudaStream_t st) {
  return launch_k(k_prepare, dim3((B + 127) / 128), dim3(128), 0, st, slots, B, pos, hist, hist_stride, f_slot, f_pos,
                  f_tok, f_nk);
}

// ------------------------------------------------------------------ column copy
// copy columns [p0, p1) of `slot`, all layers, K and V, src pool -> dst pool
__device__ __forceinline__ void copy_cols(const ColCopy& c, int slot, int p0, int p1, int tid, int nth) {
  const int vec_per_col = c.hd / 8;
  const int per_pos = c.L * 2 * c.kv * vec_per_col;
  const int total = (p1 - p0) * per_pos;
  for (int e = tid; e < total; e += nth) {
    const int q = p0 + e / per_pos;
    int r = e % per_pos;
    const int v8 = r % vec_per_col; r /= vec_per_col;
    const int kh = r % c.kv; r /= c.kv;
    const int kvsel = r % 2;
    const int l = r / 2;
    const int page = c.pt[(size_t)slot * c.max_pages + q / c.page_size];
    const size_t off = ((((size_t)l * c.n_pages + page) * 2 + kvsel) * c.kv + kh) * (size_t)c.page_size * c.hd +
                       (size_t)(q % c.page_size) * c.hd + (size_t)v8 * 8;
    *reinterpret_cast<uint4*>(c.dst + off) = *reinterpret_cast<const uint4*>(c.src + off);
  }
}

__global__ void k_copy_cols(ColCopy c, int slot, int p0, int p1) {
  griddep();
  copy_cols(c, slot, p0, p1, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

cudaError_t launch_copy_cols(const ColCopy& c, int slot, int p0, int p1, cudaStream_t st) {
  if (p1 <= p0) return cudaSuccess;
  const int total = (p1 - p0) * c.L * 2 * c.kv * (c.hd / 8);
  int blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  return launch_k(k_copy_cols, dim3(blocks), dim3(256), 0, st, c, slot, p0, p1);
}

// ------------------------------------------------------------------ commit
__global__ void __launch_bounds__(256) k_commit(CommitArgs a) {
  griddep();
  const int b = blockIdx.x;
  const int slot = a.slots[b];
  const int p = a.pos[slot];
  const bool listed = a.gate_ran && a.trig[b] && (!a.ran || a.ran[0] > 0);
  const bool tr = listed && (!a.spec || gate_fires(a.g[b], a.tau_d ? *a.tau_d : a.spec_tau));  // the gate
  const int f = a.f_tok[b];
  const int v = tr ? a.v_tok[a.rank[b]] : -1;
  const int kind = !tr ? 0 : (v == f ? 1 : 2);
  if (kind == 2 && a.repair_copy) copy_cols(a.copy, slot, p, p + 1, threadIdx.x, blockDim.x);  // single-column repair
  if (threadIdx.x == 0) {
    const int out = kind == 2 ? v : f;
    a.tokens_out[b] = out;
    if (a.kind_out) a.kind_out[b] = (uint8_t)kind;
    if (a.margin_out) a.margin_out[b] = a.g[b];
    a.hist[(size_t)slot * a.hist_stride + p + 1] = out;
    a.pos[slot] = p + 1;
    if (listed) a.shadow_len[slot] = p + 1;
    if (a.dbg_vtok) {
      a.dbg_vtok[b] = v;
      a.dbg_vg[b] = tr ? a.v_g[a.rank[b]] : 0.f;
      a.dbg_kind[b] = (uint8_t)kind;
      a.dbg_trig[b] = tr ? 1 : 0;
      a.dbg_out[b] = out;
    }
    const bool prot = a.prot ? a.prot[b] != 0 : true;
    unsigned long long* s = a.stats;
    atomicAdd(&s[1], 1ull);
    if (prot) atomicAdd(&s[2], 1ull);
    if (tr) atomicAdd(&s[3], 1ull);
    if (kind == 1) atomicAdd(&s[4], 1ull);
    if (kind == 2) atomicAdd(&s[5], 1ull);
    if (b == 0) {
      atomicAdd(&s[0], 1ull);
      if (a.gate_ran && a.ctrl[0] > 0 && (!a.ran || a.ran[0] > 0)) {
        atomicAdd(&s[6], 1ull);
        atomicAdd(&s[7], (unsigned long long)a.ctrl[1]);
      }
    }
  }
}

cudaError_t launch_commit(const CommitArgs& a, cudaStream_t st) {
  return launch_k(k_commit, dim3(a.B), dim3(256), 0, st, a);
}

// ------------------------------------------------------------------ device-side verifier dispatch
__global__ void k_vchunk(VChunkArgs a) {
  griddep();
  __shared__ int s_n, s_base, s_tc;
  if (threadIdx.x == 0) {
    const int M = a.ctrl[1], c0 = a.vctl[0], rem = M - c0;
    int k = a.n_sizes - 1;
    for (int i = 0; i < a.n_sizes; ++i)
      if (a.sizes[i] >= rem) { k = i; break; }
    const int tc = a.sizes[k];
    s_n = rem < tc ? rem : tc;
    s_base = c0;
    s_tc = tc;
    a.vctl[1] = c0;
    a.vctl[0] = c0 + tc;
    if (a.stats) atomicAdd(&a.stats[11], 1ull);
    if (a.h_case) cudaGraphSetConditional(a.h_case, (unsigned)k);
    if (a.h_loop) cudaGraphSetConditional(a.h_loop, c0 + tc < M ? 1u : 0u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s_tc; i += blockDim.x) {
    if (i < s_n) {
      const int e = s_base + i;
      a.v_slot[i] = a.cu_slot[e];
      a.v_pos[i] = a.cu_pos[e];
      a.v_tok[i] = a.cu_tok[e];
      a.v_nk[i] = a.cu_nk[e];
    } else {  // no-op entry: no cache write (slot -1), no keys, a valid embedding row
      a.v_slot[i] = -1;
      a.v_pos[i] = 0;
      a.v_tok[i] = 0;
      a.v_nk[i] = 0;
    }
  }
}

cudaError_t launch_vchunk(const VChunkArgs& a, cudaStream_t st) {
  if (a.n_sizes < 1 || a.n_sizes > 8) return cudaErrorInvalidValue;
  return launch_k(k_vchunk, dim3(1), dim3(512), 0, st, a);
}

__global__ void k_emit(const int32_t* __restrict__ tok, const uint8_t* __restrict__ kind,
                       const float* __restrict__ marg, int B, int32_t* tok_out, uint8_t* kind_out, float* marg_out) {
  griddep();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  tok_out[b] = tok[b];
  if (kind_out) kind_out[b] = kind[b];
  if (marg_out) marg_out[b] = marg[b];
}

cudaError_t launch_emit(const int32_t* tok, const uint8_t* kind, const float* marg, int B, int32_t* tok_out,
                        uint8_t* kind_out, float* marg_out, cudaStream_t st) {
  return launch_k(k_emit, dim3((B + 255) / 256), dim3(256), 0, st, tok, kind, marg, B, tok_out, kind_out, marg_out);
}

__global__ void k_gather_last(const uint16_t* __restrict__ xn, const int32_t* __restrict__ last,
                              const int32_t* __restrict__ ctrl, const int32_t* __restrict__ vctl, int T, int d,
                              uint16_t* __restrict__ xgn) {
  griddep();
  const int r = blockIdx.x;
  if (r >= ctrl[0]) return;
  const int l = last[r] - vctl[1];
  if (l < 0 || l >= T) return;
  const uint4* s = reinterpret_cast<const uint4*>(xn + (size_t)l * d);
  uint4* o = reinterpret_cast<uint4*>(xgn + (size_t)r * d);
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) o[j] = s[j];
}

cudaError_t launch_gather_last(const uint16_t* xn, const int32_t* last, const int32_t* ctrl, const int32_t* vctl,
                               int T, int n_max, int d, uint16_t* xgn, cudaStream_t st) {
  if (n_max <= 0) return cudaSuccess;
  return launch_k(k_gather_last, dim3(n_max), dim3(128), 0, st, xn, last, ctrl, vctl, T, d, xgn);
}

// ------------------------------------------------------------------ window verify
// LLM-42-style windowed verification (include/mg.h
// mg_verify_window).  Row i's unverified tokens are the inputs at positions
// shadow_len .. p-1; the verifier's argmax at q predicts position q+1.
// k_window_list: catch-up list entries off[i] + (q - shadow_len).  CTA per row.
__global__ void k_window_list(WindowArgs a) {
  griddep();
  const int i = blockIdx.x;
  const int slot = a.slots[i], s0 = a.shadow_len[slot], p = a.pos[slot];
  const int32_t* h = a.hist + (size_t)slot * a.hist_stride;
  for (int q = s0 + threadIdx.x; q < p; q += blockDim.x) {
    const int e = a.off[i] + (q - s0);
    a.cu_slot[e] = slot;
    a.cu_pos[e] = q;
    a.cu_tok[e] = h[q];
    a.cu_nk[e] = q + 1;
  }
}

cudaError_t launch_window_list(const WindowArgs& a, cudaStream_t st) {
  return launch_k(k_window_list, dim3(a.n), dim3(128), 0, st, a);
}

// k_window_commit: first disagreement m -> hist[m] = verifier token,
// pos = shadow_len = m (rollback); else shadow_len = p.  CTA (one warp) per row;
// the first mismatch is the minimum mismatching q over a warp-strided scan.
__global__ void k_window_commit(WindowArgs a) {
  griddep();
  const int i = blockIdx.x, lane = threadIdx.x;
  const int slot = a.slots[i], s0 = a.shadow_len[slot], p = a.pos[slot];
  int32_t* h = a.hist + (size_t)slot * a.hist_stride;
  int first = INT_MAX;
  for (int q = s0 + lane; q < p; q += 32)
    if (a.v_tok[a.off[i] + (q - s0)] != h[q + 1]) { first = q; break; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  if (lane != 0) return;
  int np = p, rb = 0;
  if (first != INT_MAX) {
    np = first + 1;
    rb = p - np;
    h[np] = a.v_tok[a.off[i] + (first - s0)];
    a.pos[slot] = np;
  }
  a.shadow_len[slot] = np;
  if (a.pend) a.pend[slot] = 0;
  a.res[3 * i] = np;
  a.res[3 * i + 1] = h[np];
  a.res[3 * i + 2] = rb;
  unsigned long long* s = a.stats;
  atomicAdd(&s[8], 1ull);
  atomicAdd(&s[7], (unsigned long long)(p - s0));
  if (first != INT_MAX) {
    atomicAdd(&s[9], 1ull);
    atomicAdd(&s[10], (unsigned long long)rb);
  }
}

cudaError_t launch_window_commit(const WindowArgs& a, cudaStream_t st) {
  return launch_k(k_window_commit, dim3(a.n), dim3(32), 0, st, a);
}

// ------------------------------------------------------------------ pipelined verification
// (include/mg.h MG_VERIFY_PIPELINED).  The rows gated at step t are verified
// inside step t+1's forward (their catch-up tokens are extra GEMM columns --
// the tcgen05 GEMM's per-column result is independent of the other columns,
// and a separate pinned-split attention launch over the
// shadow cache).  Row b of step t+1, slot s, tentative token y at position p:
//   pending and v == y: verified (shadow_len = p); the step's fast output stands
//   pending and v != y: repair -- hist[p] = v, shadow column p-1 -> fast cache
//                       (PAPER.md:208), the row does not advance (its fast
//                       output was computed from y and is dropped), kind 4
//   then (not repaired): commit f_tok at p+1; gated = prot && g < tau ->
//                        pending (kind 3), else kind 0 (1 if a pending token
//                        was just verified)
__global__ void __launch_bounds__(256) k_commit_fused(FusedCommitArgs a) {
  griddep();
  const int b = blockIdx.x;
  const int slot = a.slots[b];
  const int p = a.pos[slot];
  int32_t* h = a.hist + (size_t)slot * a.hist_stride;
  const bool pend = a.had_pend && a.pend[slot];
  const int v = pend ? a.v_tok[a.rank_slot[slot]] : -1;
  const bool rep = pend && v != h[p];
  if (rep && a.repair_copy) copy_cols(a.copy, slot, p - 1, p, threadIdx.x, blockDim.x);
  if (threadIdx.x != 0) return;
  const bool prot = a.prot ? a.prot[b] != 0 : true;
  unsigned long long* s = a.stats;
  atomicAdd(&s[1], 1ull);
  // a replacement step (kind 4) drops the row's fast output: no gate decision,
  // so it is not a protected row of r_verify's denominator (r_verify = 1 at
  // tau = +inf, as in the synchronous mode)
  if (prot && !rep) atomicAdd(&s[2], 1ull);
  if (pend) atomicAdd(&s[rep ? 5 : 4], 1ull);
  if (b == 0) {
    atomicAdd(&s[0], 1ull);
    if (a.had_pend && a.n_pend > 0) {
      atomicAdd(&s[6], 1ull);
      atomicAdd(&s[7], (unsigned long long)a.M);
    }
  }
  int kind, out;
  bool gated = false;
  if (pend) a.shadow_len[slot] = p;  // shadow columns 0..p-1 are final
  if (rep) {
    h[p] = v;
    a.pend[slot] = 0;
    kind = 4;
    out = v;
  } else {
    out = a.f_tok[b];
    gated = a.gate_on && prot && gate_fires(a.g[b], a.tau);  // strict <
    h[p + 1] = out;
    a.pos[slot] = p + 1;
    a.pend[slot] = gated ? 1 : 0;
    kind = gated ? 3 : (pend ? 1 : 0);
    if (gated) atomicAdd(&s[3], 1ull);
  }
  a.tokens_out[b] = out;
  if (a.kind_out) a.kind_out[b] = (uint8_t)kind;
  if (a.margin_out) a.margin_out[b] = a.g[b];
  if (a.dbg_vtok) {
    a.dbg_vtok[b] = v;
    a.dbg_vg[b] = pend ? a.v_g[a.rank_slot[slot]] : 0.f;
    a.dbg_kind[b] = (uint8_t)kind;
    a.dbg_trig[b] = gated ? 1 : 0;
    a.dbg_out[b] = out;
  }
}

cudaError_t launch_commit_fused(const FusedCommitArgs& a, cudaStream_t st) {
  return launch_k(k_commit_fused, dim3(a.B), dim3(256), 0, st, a);
}

// M = the bucketed catch-up length of the launch; the real one is ctrl[1]
// (written by the pending-list gate of the previous step).  Padding rows
// repeat the last real entry: they recompute the same shadow column from the
// same inputs (identical values), so the padding changes nothing but keeps
// the number of distinct CUDA graphs small.
__global__ void k_prepare_mixed(const int32_t* __restrict__ slots, int B, const int32_t* __restrict__ pos,
                                const int32_t* __restrict__ hist, int hist_stride, const int32_t* cu_slot,
                                const int32_t* cu_pos, const int32_t* cu_tok, const int32_t* cu_nk, int M,
                                const int32_t* __restrict__ ctrl, int32_t* m_slot, int32_t* m_pos, int32_t* m_tok,
                                int32_t* m_nk) {
  griddep();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B) {
    const int s = slots[i], p = pos[s];
    m_slot[i] = s;
    m_pos[i] = p;
    m_tok[i] = hist[(size_t)s * hist_stride + p];
    m_nk[i] = p + 1;
  } else if (i < B + M) {
    const int e = min(i - B, ctrl[1] - 1);
    m_slot[i] = cu_slot[e];
    m_pos[i] = cu_pos[e];
    m_tok[i] = cu_tok[e];
    m_nk[i] = cu_nk[e];
  }
}

cudaError_t launch_prepare_mixed(const int32_t* slots, int B, const int32_t* pos, const int32_t* hist, int hist_stride,
                                 const int32_t* cu_slot, const int32_t* cu_pos, const int32_t* cu_tok,
                                 const int32_t* cu_nk, int M, const int32_t* ctrl, int32_t* m_slot, int32_t* m_pos,
                                 int32_t* m_tok, int32_t* m_nk, cudaStream_t st) {
  return launch_k(k_prepare_mixed, dim3((B + M + 127) / 128), dim3(128), 0, st, slots, B, pos, hist, hist_stride,
                  cu_slot, cu_pos, cu_tok, cu_nk, M, ctrl, m_slot, m_pos, m_tok, m_nk);
}

// one CTA per output row, 16-byte copies; verifier rows past the real count
// ctrl[0] (bucket padding) repeat the last real one
__global__ void k_lm_rows(const uint16_t* __restrict__ src, int B, const int32_t* __restrict__ last,
                          const int32_t* __restrict__ ctrl, int d, uint16_t* __restrict__ dst) {
  griddep();
  const int i = blockIdx.x;
  const int r = i < B ? i : B + last[min(i - B, ctrl[0] - 1)];
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)r * d);
  uint4* o = reinterpret_cast<uint4*>(dst + (size_t)i * d);
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) o[j] = s[j];
}

cudaError_t launch_lm_rows(const uint16_t* src, int B, const int32_t* last, const int32_t* ctrl, int n, int d,
                           uint16_t* dst, cudaStream_t st) {
  return launch_k(k_lm_rows, dim3(B + n), dim3(128), 0, st, src, B, last, ctrl, d, dst);
}

// ------------------------------------------------------------------ test-only perturbation
// SPEC.md:76-84 injected logit noise (mgd_set_inject; never on by default):
// l[v] += amp * (u * 2^-23), u = (splitmix64(seed ^ B<<56 ^ slot<<44 ^ pos<<20 ^ v) >> 40) - 2^23,
// exactly zero at batch 1 -- the documented formula the oracle applies too.
__device__ __forceinline__ uint64_t inj_mix(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_inject(float* logits, int B, int V, float amp, unsigned long long seed, const int32_t* slot,
                         const int32_t* pos) {
  griddep();
  const int b = blockIdx.y;
  const uint64_t key = seed ^ ((uint64_t)B << 56) ^ ((uint64_t)slot[b] << 44) ^ ((uint64_t)pos[b] << 20);
  float* l = logits + (size_t)b * V;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    const int u = (int)(inj_mix(key ^ (uint64_t)v) >> 40) - 8388608;
    l[v] = __fadd_rn(l[v], __fmul_rn(amp, __fmul_rn((float)u, 1.1920928955078125e-07f)));
  }
}

cudaError_t launch_inject(float* logits, int B, int V, float amp, unsigned long long seed, const int32_t* slot,
                          const int32_t* pos, cudaStream_t st) {
  if (B <= 1 || !(amp > 0.f)) return cudaSuccess;
  return launch_k(k_inject, dim3(16, B), dim3(256), 0, st, logits, B, V, amp, seed, slot, pos);
}

// prefill bookkeeping: hist[slot][len] = token, pos = shadow_len = len
__global__ void k_prefill_done(int32_t* hist, int hist_stride, int32_t* pos, int32_t* shadow_len, int slot, int len,
                               const int32_t* tok) {
  griddep();
  hist[(size_t)slot * hist_stride + len] = tok[0];
  pos[slot] = len;
  shadow_len[slot] = len;
}

cudaError_t launch_prefill_done(int32_t* hist, int hist_stride, int32_t* pos, int32_t* shadow_len, int slot, int len,
                                const int32_t* tok, cudaStream_t st) {
  return launch_k(k_prefill_done, dim3(1), dim3(1), 0, st, hist, hist_stride, pos, shadow_len, slot, len, tok);
}

}  // namespace mg
