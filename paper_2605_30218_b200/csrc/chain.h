// chain.h -- the persistent layer chain (chain.cu): several weight-streaming
// GEMM phases and their epilogues in ONE kernel, so the HBM weight stream does
// not drain at every op boundary.
#pragma once
#include "epilogue.cuh"
#include "kernels.h"

namespace mg {

enum ChainOp : int32_t {
  CH_NONE = 0,
  CH_RESNORM = 1,  // x <- bf16(x + sum part); xn <- RMSNorm(x) * w      (a5 / a7 + a2)
  CH_SWIGLU = 2,   // a <- bf16(silu(g) * u) from the [gate;up] partials  (a6)
  CH_QKV = 3,      // bias + RoPE, q out, k/v appended to the cache       (a3)
};

struct ChainPhase {
  CUtensorMap mw;  // weights: 4-D tiled map (make_tmap_w_tiled)
  const uint16_t* wbase;  // the same weights (tiled: k-block (mt, kb) at (mt * K/64 + kb) * 16 KB)
  CUtensorMap mx;  // activations [rows][K]: 2-D map, box = tile_n rows (make_tmap_2d)
  int32_t N, K, G;  // G: stream-K virtual CTAs (a function of the weight shape)
  float* part;      // [slots][T][N] fp32 partials (slot = k order)
  int32_t op;       // ChainOp applied after this GEMM, by every CTA
  uint16_t* x;      // CH_RESNORM: residual stream [T][N] (in/out)
  const uint16_t* w;  // CH_RESNORM: norm gains [N]
  uint16_t* xn;     // CH_RESNORM: normed output [T][N]
  float eps;
  uint16_t* a;      // CH_SWIGLU: [T][N/2]
  QkvArgs qkv;      // CH_QKV
};

constexpr int kChainMax = 4;
struct ChainArgs {
  ChainPhase ph[kChainMax];
  int32_t n_ph;
  int32_t T;
  uint32_t* sync;   // [2 * kChainMax + 1] grid-barrier counters + epoch (zero at init, never reset)
  int32_t* err;     // set to 1 when a grid barrier times out (the step is then garbage)
  unsigned long long* trace;  // diagnostics (nullptr in the product): per CTA [1 + kChainMax * 6] globaltimer stamps
  int32_t pf_kblocks;  // L2 run-ahead of each CTA's weight stream, in 16 KB k-blocks (0: off)
};
constexpr int kChainTraceWords = 1 + kChainMax * 6;

// tile_n / mma_n as for launch_gemm_tc (mma_n 16 = the verifier's slot groups).
// Grid = one CTA per SM (all CTAs must be co-resident: grid barriers).
cudaError_t launch_chain(const ChainArgs& a, int tile_n, int mma_n, cudaStream_t st);
int chain_grid();

}  // namespace mg
