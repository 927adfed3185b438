// gemm_tc.cuh -- pieces shared by the tcgen05 weight-streaming kernels
// (k_gemm_tc in gemm.cu, scripts/gemm_*.cu microbenchmarks):
// the smem/pipeline configuration, the stream-K piece iterator and the
// per-stage MMA issue.
#pragma once
#include "common.cuh"
#include "kernels.h"

#ifndef MG_GEMM_SMEM_KB
#define MG_GEMM_SMEM_KB 192  // smem ring budget per CTA
#endif
#ifndef MG_GEMM_NS_MAX
#define MG_GEMM_NS_MAX 8
#endif
#ifndef MG_GEMM_KS
#define MG_GEMM_KS 2
#endif

namespace mg {

template <int TN>
struct GemmTcCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int KS = MG_GEMM_KS;      // 64-wide k-blocks per pipeline stage
  static constexpr int A_BOX = BM * BK * 2;  // one TMA box (16 KB, contiguous in HBM)
  static constexpr int B_BOX = TN * BK * 2;
  static constexpr int A_BYTES = KS * A_BOX;
  static constexpr int B_BYTES = KS * B_BOX;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // the 80-token tile (a batch of 64 plus the fused verifier's columns) gets
  // 208 KB so it keeps 4 stages (128 KB of weights in flight) like the 64 tile
  static constexpr int NS0 = ((TN == 80 ? 208 : MG_GEMM_SMEM_KB) * 1024) / STAGE;
  static constexpr int NS = NS0 > MG_GEMM_NS_MAX ? MG_GEMM_NS_MAX : NS0;
  static constexpr int ACC_COLS = TN < 32 ? 32 : (TN + 31) / 32 * 32;  // accumulator columns (32-aligned)
  static constexpr int TMEM_COLS = 2 * ACC_COLS <= 64 ? 64 : (2 * ACC_COLS <= 128 ? 128 : (2 * ACC_COLS <= 256 ? 256 : 512));
  static constexpr int THREADS = 192;
  static constexpr int SMEM = 1024 + NS * STAGE + (2 * NS + 4) * 8 + 16;
  static_assert(NS >= 2, "pipeline needs two stages");
};

struct GemmArgs {
  int N, K, T, splits;
  int n_m, n_t, units;
  int G;    // > 0: stream-K over G virtual CTAs per token tile; 0: uniform split-K
  int dbg;  // microbenchmark knobs (0 in the product): 1 skip MMAs, 2 skip stores, 1024 trace CTA 0
  float* out;
  // fused top-1/top-2 epilogue (LM head, "computes only the top
  // two values"): instead of the fp32 logits, each 128-row tile writes, per
  // token, its top-2 (v1, i1, v2, i2) to t2[t][n_m][4]; NaN ranks as -inf and
  // sets *nan_flag.  Requires a single piece per tile (G == 0, splits == 1).
  float* t2;
  int32_t* nan_flag;
};

// A piece = one contiguous k-block range of one 128-feature tile for one
// token tile; its fp32 partial goes to out[slot].  Every role of the CTA
// walks the same piece sequence.
struct Piece {
  int mt, kb0, kb1, slot, tt;
};
struct PieceIter {
  int KB, n_m, n_t, S, G, units;
  long long W, w, w1;
  int v, i, tt, u;
  __device__ explicit PieceIter(const GemmArgs& g, int KB_) {
    KB = KB_; n_m = g.n_m; n_t = g.n_t; S = g.splits; G = g.G; units = g.units;
    W = (long long)n_m * KB;
    u = blockIdx.x;
    v = (int)blockIdx.x - (int)gridDim.x;
    w = w1 = 0;
    i = tt = 0;
  }
  __device__ bool next(Piece& p) {
    if (G == 0) {
      if (u >= units) return false;
      p.tt = u % n_t;
      const int r = u / n_t;
      p.slot = r % S;
      p.mt = r / S;
      p.kb0 = chunk_start(KB, S, p.slot);
      p.kb1 = chunk_start(KB, S, p.slot + 1);
      u += gridDim.x;
      return true;
    }
    while (w >= w1) {
      v += gridDim.x;
      if (v >= G * n_t) return false;
      tt = v / G;
      i = v % G;
      w = (long long)i * W / G;
      w1 = (long long)(i + 1) * W / G;
    }
    p.tt = tt;
    p.mt = (int)(w / KB);
    p.kb0 = (int)(w % KB);
    p.kb1 = (int)min((long long)KB, p.kb0 + (w1 - w));
    p.slot = i - streamk_owner((long long)p.mt * KB, W, G);
    w += p.kb1 - p.kb0;
    return true;
  }
};

// Issue the MMAs of one pipeline stage (lane 0 of the MMA warp): nk k-blocks of
// A (128 x 64 weight boxes) x B (TN tokens x 64) into the accumulator dacc.
template <int TN, bool MMA16>
MG_DEV void issue_stage(uint64_t a_st, uint64_t b_st, int nk, uint32_t dacc, bool first) {
  using C = GemmTcCfg<TN>;
  constexpr int MN = MMA16 ? 16 : TN;  // instruction N
  constexpr int NG = TN / MN;          // instructions per k-step
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(MN >> 3) << 17) | ((128u >> 4) << 24);
#pragma unroll
  for (int i = 0; i < C::KS; ++i) {
    if (i < nk) {
#pragma unroll
      for (int kk = 0; kk < C::BK / 16; ++kk) {
        const uint64_t ad = a_st + (uint64_t)((i * C::A_BOX + kk * 32) >> 4);
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
          const uint64_t bd = b_st + (uint64_t)((i * C::B_BOX + gi * MN * 128 + kk * 32) >> 4);
          tc_mma_bf16(dacc + (uint32_t)(gi * MN), ad, bd, idesc, (!first || i > 0 || kk > 0) ? 1u : 0u);
        }
      }
    }
  }
}

}  // namespace mg
