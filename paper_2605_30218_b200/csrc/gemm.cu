// gemm.cu -- weight-streaming GEMM partials for the decode path (SURVEY 8(a)
// rows a3, a5-a8): out[s][t][n] = sum_{k in piece s} x[t][k] * W[n][k].
//
// k_gemm_tc: persistent, warp-specialised tcgen05 "swap-AB" kernel.
//   Work piece = (128 output features, a contiguous range of 64-wide
//   k-blocks, one tile of <= TN tokens); pieces come from a stream-K
//   partition over G virtual CTAs (or a uniform split-K), so every SM streams
//   the same number of weight bytes.
//   warp 0     TMA producer: weight boxes (128 x 64, tiled layout = one
//              contiguous 16 KB each, 128B swizzle) are the MMA M operand, the
//              TN tokens x 64 the N operand; KS k-blocks per stage behind one
//              mbarrier, NS stages, a ring that never drains between pieces;
//   warp 1     tcgen05.mma (M128 x N x K16, bf16 -> fp32) into one of two TMEM
//              accumulators (double buffered), issued by one lane of a
//              warp-uniform loop with precomputed descriptors (the issue
//              loop, not HBM, was the measured bottleneck of a per-lane loop);
//   warps 2-5  epilogue: tcgen05.ld the accumulator, write the piece's fp32
//              partial, release the TMEM buffer.
//   PDL: before griddepcontrol.wait the producer already streams the first
//   stages' weights (weights never depend on the previous kernel).
// The split-K reduction and the op's epilogue (bias/RoPE/append, residual,
// SwiGLU, top-2) run in the consumer kernels in k order, so results are
// run-to-run deterministic (no float atomics).
//
// Batch invariance (BASELINE north_star, A14): the partition is a
// function of the weight shape only, and a token column's fp32 result does
// not depend on the instruction width N, its slot or the other columns
// (tests/test_gpu_ops.py::test_gemm_column_invariance: N = 16..256), so the
// verifier runs the same full-width MMAs as the fast path.  MMA16 (16-column
// instructions per slot group) remains as an option.
//
// (A CUDA-core GEMV for T <= 8 tokens measured 1.6-2.4x slower per step at
// B = 2 / 4 than this kernel's 16-token tile and was removed in round 2.)
#include "common.cuh"
#include <climits>

#include "gemm_tc.cuh"
#include "kernels.h"

#ifndef MG_EPI_STORE
#define MG_EPI_STORE 1  // 1: partials via a shared-memory transpose and float4 stores; 0: scalar stores
#endif
#ifndef MG_PART_EVICT_LAST
#define MG_PART_EVICT_LAST 1  // fp32 partial stores with an L2 evict_last hint
#endif
#ifndef MG_EPI_WAIT
#define MG_EPI_WAIT mbar_wait  // accumulator-ready wait of the epilogue poller
#endif

namespace mg {

int g_pdl = 1;
int g_gemm_dbg = 0;  // microbenchmark knobs (scripts/gemm_bench.cu); always 0 in the library

template <int TN, bool MMA16>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapX, GemmArgs g) {
  using C = GemmTcCfg<TN>;
  constexpr int KS = C::KS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::NS * C::A_BYTES;
  uint64_t* full = (uint64_t*)(sB + C::NS * C::B_BYTES);
  uint64_t* empty = full + C::NS;
  uint64_t* tfull = empty + C::NS;  // [2]
  uint64_t* tempty = tfull + 2;     // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = g.K / C::BK;
  long long* trace = ((g.dbg & 1024) && blockIdx.x == 0) ? reinterpret_cast<long long*>(g.out) : nullptr;
  // dbg 2048: per-CTA globaltimer stamps [entry, first stage landed, last MMA issued, exit]
  long long* ctr = (g.dbg & 2048) ? reinterpret_cast<long long*>(g.out) + blockIdx.x * 4 : nullptr;
  if (ctr && threadIdx.x == 0) ctr[0] = (long long)globaltimer();

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mapW);
    tma_prefetch_desc(&mapX);
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);  // one arrival per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 2) tc_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  Piece pc;
  if (warp == 0) {
    // ---- TMA producer: warp-uniform loop, lane 0 issues
    const uint64_t pol = policy_evict_first();  // weights are streamed once
    int it = 0;                                  // stage counter of this CTA
    int pre = 0;                                 // stages whose weights went out before griddepcontrol.wait
    {
      PieceIter first(g, KB);
      if (first.next(pc)) {
        for (int kb = pc.kb0; kb < pc.kb1 && pre < C::NS; kb += KS, ++pre) {
          const int nk = min(KS, pc.kb1 - kb);
          if (lane == 0) {
            mbar_expect_tx(&full[pre], (uint32_t)nk * (C::A_BOX + C::B_BOX));
            for (int i = 0; i < nk; ++i)
              tma_load_4d_hint(sA + pre * C::A_BYTES + i * C::A_BOX, &mapW, &full[pre], 0, 0, kb + i, pc.mt, pol);
          }
        }
      }
    }
    griddep_wait();
    PieceIter pi(g, KB);
    while (pi.next(pc)) {
      for (int kb = pc.kb0; kb < pc.kb1; kb += KS, ++it) {
        const int st = it % C::NS;
        const uint32_t ph = (uint32_t)(it / C::NS) & 1u;
        const int nk = min(KS, pc.kb1 - kb);
        if (it >= pre) mbar_spin(&empty[st], ph ^ 1u);
        if (lane == 0) {
          if (it >= pre) {
            mbar_expect_tx(&full[st], (uint32_t)nk * (C::A_BOX + C::B_BOX));
            for (int i = 0; i < nk; ++i)
              tma_load_4d_hint(sA + st * C::A_BYTES + i * C::A_BOX, &mapW, &full[st], 0, 0, kb + i, pc.mt, pol);
          }
          if (g.dbg & 4) {  // microbenchmark: no activation loads (their expected bytes completed by hand)
            asm volatile("mbarrier.complete_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[st])),
                         "r"((uint32_t)nk * C::B_BOX)
                         : "memory");
          } else {
            for (int i = 0; i < nk; ++i)
              tma_load_2d(sB + st * C::B_BYTES + i * C::B_BOX, &mapX, &full[st], (kb + i) * C::BK, pc.tt * TN);
          }
          if (trace && it < 256) trace[it * 4 + 0] = clock64();
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: warp-uniform loop, lane 0 issues tcgen05.mma / commit
    const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA));
    const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sB));
    const bool do_mma = !(g.dbg & 1);
    int it = 0, j = 0;
    PieceIter pi(g, KB);
    for (; pi.next(pc); ++j) {
      const int buf = j & 1;
      mbar_spin(&tempty[buf], ((uint32_t)(j >> 1) & 1u) ^ 1u);  // epilogue drained this accumulator
      tc_fence_after();
      const uint32_t dacc = tmem + (uint32_t)(buf * C::ACC_COLS);
      for (int kb = pc.kb0; kb < pc.kb1; kb += KS, ++it) {
        const int st = it % C::NS;
        const int nk = min(KS, pc.kb1 - kb);
        mbar_spin(&full[st], (uint32_t)(it / C::NS) & 1u);
        tc_fence_after();
        if (lane == 0) {
          if (trace && it < 256) trace[it * 4 + 1] = clock64();
          if (ctr && it == 0) ctr[1] = (long long)globaltimer();
          // descriptor of (stage st, box i, k-step kk) = base + byte offset / 16
          const uint64_t a_st = a_desc0 + (uint64_t)((st * C::A_BYTES) >> 4);
          const uint64_t b_st = b_desc0 + (uint64_t)((st * C::B_BYTES) >> 4);
          if (do_mma) issue_stage<TN, MMA16>(a_st, b_st, nk, dacc, kb == pc.kb0);
          tc_commit(&empty[st]);  // frees the smem stage when these MMAs retire
          if (trace && it < 256) trace[it * 4 + 2] = clock64();
        }
        __syncwarp();
      }
      if (lane == 0) tc_commit(&tfull[buf]);  // accumulator complete
      __syncwarp();
    }
    if (ctr && lane == 0) ctr[2] = (long long)globaltimer();
  } else {  // ---- epilogue warps 2..5: TMEM lanes 32*(warp%4) ..
    __shared__ Top2 s_t2[4][16];         // fused top-2: per-warp results of one 16-token chunk
    __shared__ __align__(16) float s_val[4][16 * 33];  // per-warp [token][row] transposes (top-2 padded; stores dense)
    griddep_wait();
    const int q = warp & 3;
#if MG_PART_EVICT_LAST
    const uint64_t pol_part = policy_evict_last();
#endif
    int j = 0;
    PieceIter pi(g, KB);
    for (; pi.next(pc); ++j) {
      const int buf = j & 1;
      // one thread polls the mbarrier; the other 127 sleep in a named barrier
      if (warp == 2 && lane == 0) MG_EPI_WAIT(&tfull[buf], (uint32_t)(j >> 1) & 1u);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc_fence_after();
      const int n = pc.mt * C::BM + q * 32 + lane;
      float* o = g.out + (size_t)pc.slot * (size_t)g.T * (size_t)g.N;
      const int t0 = pc.tt * TN;
#pragma unroll 1
      for (int c0 = 0; c0 < TN; c0 += 16) {
        if (t0 + c0 >= g.T) break;
        uint32_t r[16];
        tc_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * C::ACC_COLS + c0), r);
        tc_wait_ld();
        if (g.t2) {
          // fused top-2 over this tile's 128 rows for each of the 16 tokens:
          // each warp transposes its 32 rows x 16 tokens through shared memory,
          // lane (token i, half h) scans 16 rows, one shuffle merges the halves;
          // then the 4 warps merge through s_t2
          bool nan = false;
          float* sv = s_val[q];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float v = __uint_as_float(r[i]);
            if (v != v) { nan = true; v = -INFINITY; }
            sv[i * 33 + lane] = v;
          }
          if (nan) atomicOr(g.nan_flag, 1);
          __syncwarp();
          {
            const int i = lane & 15, h = lane >> 4;
            const int id0 = pc.mt * C::BM + q * 32 + h * 16;
            Top2 tt{-INFINITY, INT_MAX, -INFINITY, INT_MAX};
#pragma unroll
            for (int rr = 0; rr < 16; ++rr) t2_push(tt, sv[i * 33 + h * 16 + rr], id0 + rr);
            tt = t2_merge(tt, t2_shfl(tt, 16));
            if (lane < 16) s_t2[q][i] = tt;
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (q == 0 && lane < 16 && t0 + c0 + lane < g.T) {
            Top2 a = s_t2[0][lane];
#pragma unroll
            for (int w = 1; w < 4; ++w) a = t2_merge(a, s_t2[w][lane]);
            float* dst = g.t2 + ((size_t)(t0 + c0 + lane) * g.n_m + pc.mt) * 4;
            *reinterpret_cast<float4*>(dst) = make_float4(a.v1, __int_as_float(a.i1), a.v2, __int_as_float(a.i2));
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          continue;
        }
        if (!(g.dbg & 2)) {
#if MG_EPI_STORE == 1
          // transpose the warp's 32 rows x 16 tokens through shared memory and
          // write each token's 32 consecutive features as float4s: 4 store
          // instructions of 4 full 128-byte lines each instead of 16 scalar ones
          float* sv = s_val[q];
#pragma unroll
          for (int i = 0; i < 16; ++i) sv[i * 32 + lane] = __uint_as_float(r[i]);
          __syncwarp();
          const int n0 = pc.mt * C::BM + q * 32;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int idx = k * 32 + lane, i = idx >> 3, p4 = (idx & 7) * 4;
            const int t = t0 + c0 + i;
            if (t < g.T) {
#if MG_PART_EVICT_LAST
              // the partials are re-read from L2 by the next kernel: keep them
              // there while the weight stream (evict_first) flows past
              st_v4_hint(o + (size_t)t * g.N + n0 + p4, *reinterpret_cast<const float4*>(sv + i * 32 + p4), pol_part);
#else
              *reinterpret_cast<float4*>(o + (size_t)t * g.N + n0 + p4) = *reinterpret_cast<const float4*>(sv + i * 32 + p4);
#endif
            }
          }
          __syncwarp();
#else
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int t = t0 + c0 + i;
            if (t < g.T) o[(size_t)t * g.N + n] = __uint_as_float(r[i]);
          }
#endif
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  griddep_launch();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tc_dealloc(tmem, C::TMEM_COLS);
  }
  if (ctr && threadIdx.x == 0) ctr[3] = (long long)globaltimer();
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool get_encode() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  return true;
}

bool make_tmap_2d(CUtensorMap* m, const void* base, int inner_k, int rows, int box_rows) {
  if (!get_encode()) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner_k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)inner_k * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D bf16 tensor [d2][d1][d0] (d0 innermost, d0 % 64 == 0): box 64 x box1 x 1,
// 128B swizzle -- attention's Q tiles and K/V blocks
bool make_tmap_3d(CUtensorMap* m, const void* base, int d0, int64_t d1, int64_t d2, int box1) {
  if (!get_encode() || d0 % 64 || d1 < 1 || d2 < 1 || d2 > INT32_MAX || d1 > INT32_MAX) return false;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)d0 * 2, (cuuint64_t)d0 * 2 * (cuuint64_t)d1};
  cuuint32_t box[3] = {64, (cuuint32_t)box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// weights in the tiled layout [N/128][K/64][128][64]: 4-D map, box = one
// contiguous 16 KB tile, coordinates (0, 0, k-block, m-tile)
bool make_tmap_w_tiled(CUtensorMap* m, const void* base, int K, int N) {
  if (!get_encode()) return false;
  const cuuint64_t KB = (cuuint64_t)K / 64;
  cuuint64_t dims[4] = {64, 128, KB, (cuuint64_t)N / 128};
  cuuint64_t strides[3] = {128, 128 * 128, 128 * 128 * KB};
  cuuint32_t box[4] = {64, 128, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || g_num_sms <= 0)
      g_num_sms = 148;
  }
  return g_num_sms;
}

template <int TN, bool MMA16>
static cudaError_t launch_tc_t(const CUtensorMap& mw, const CUtensorMap& mx, int N, int K, int T, int splits, int G,
                               float* out, cudaStream_t st, float* t2, int32_t* nan_flag) {
  using C = GemmTcCfg<TN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(k_gemm_tc<TN, MMA16>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  GemmArgs g;
  g.N = N; g.K = K; g.T = T; g.splits = G > 0 ? 1 : splits;
  g.n_m = N / 128; g.n_t = (T + TN - 1) / TN; g.units = g.n_m * g.splits * g.n_t;
  g.G = G;
  g.dbg = g_gemm_dbg;
  g.out = out;
  g.t2 = t2;
  g.nan_flag = nan_flag;
  if (t2 && (G != 0 || g.splits != 1 || !nan_flag)) return cudaErrorInvalidValue;
  const int work = G > 0 ? G * g.n_t : g.units;
  const int grid = work < num_sms() ? work : num_sms();
  return launch_k(k_gemm_tc<TN, MMA16>, dim3(grid), dim3(C::THREADS), C::SMEM, st, mw, mx, g);
}

template <int TN>
static cudaError_t launch_tc_m(const CUtensorMap& mw, const CUtensorMap& mx, int N, int K, int T, int splits, int G,
                               int mma_n, float* out, cudaStream_t st, float* t2, int32_t* nan_flag) {
  if (mma_n == 16 && TN > 16) return launch_tc_t<TN, true>(mw, mx, N, K, T, splits, G, out, st, t2, nan_flag);
  return launch_tc_t<TN, false>(mw, mx, N, K, T, splits, G, out, st, t2, nan_flag);
}

cudaError_t launch_gemm_tc(const CUtensorMap& mw, const CUtensorMap& mx, int N, int K, int T, int splits, int G,
                           int tile_n, int mma_n, float* out, cudaStream_t st, float* t2, int32_t* nan_flag) {
  if (mma_n != 16) mma_n = tile_n;
  switch (tile_n) {
    case 16: return launch_tc_m<16>(mw, mx, N, K, T, splits, G, mma_n, out, st, t2, nan_flag);
    case 32: return launch_tc_m<32>(mw, mx, N, K, T, splits, G, mma_n, out, st, t2, nan_flag);
    case 64: return launch_tc_m<64>(mw, mx, N, K, T, splits, G, mma_n, out, st, t2, nan_flag);
    case 80: return launch_tc_m<80>(mw, mx, N, K, T, splits, G, mma_n, out, st, t2, nan_flag);
    case 128: return launch_tc_m<128>(mw, mx, N, K, T, splits, G, mma_n, out, st, t2, nan_flag);
    case 256: return launch_tc_m<256>(mw, mx, N, K, T, splits, G, mma_n, out, st, t2, nan_flag);
    default: return cudaErrorInvalidValue;
  }
}

int part_slots(const PartSpec& p, int N) {
  int mx = 1;
  for (int n = 0; n < N; n += 128) {
    const int c = part_count(p, n);
    mx = c > mx ? c : mx;
  }
  return mx;
}

int gemm_tile_n(int T) {
  if (T <= 16) return 16;
  if (T <= 32) return 32;
  if (T <= 64) return 64;
  if (T <= 80) return 80;  // e.g. a batch of 64 plus the fused verifier's columns: 4 stages, not the 128 tile's 3
  if (T <= 128) return 128;
  return 256;
}

}  // namespace mg
