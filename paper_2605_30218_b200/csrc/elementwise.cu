// elementwise.cu -- the CUDA-core kernels of the decode path that are not
// GEMMs (SURVEY 8(a) rows a1, a2 and the GEMM epilogues of a3, a5-a7), plus
// the K0 weight generator.  Every rounding point follows DESIGN.md 3.3:
// IEEE fp32 with explicit __fmul_rn/__fadd_rn/__fdiv_rn/__fsqrt_rn (no FMA
// contraction of the epilogue math), bf16 by round-to-nearest-even.
// All kernels are per-token: a token's output never depends on which other
// tokens share the launch (the verifier's batch invariance).  All are
// launched with PDL (griddep() first), so the next GEMM's weight prefetch
// overlaps them.
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace mg {

// ------------------------------------------------------------------ K0
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_gen(GenSpec g, float c, float offset, uint16_t* __restrict__ dst) {
  const uint64_t key = g.seed ^ ((uint64_t)g.tid << 40);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = splitmix64(key ^ (uint64_t)i);
    const int32_t u = (int32_t)(r >> 40) - 8388608;
    const float v = __fadd_rn(offset, __fmul_rn((float)u, c));
    int64_t o = i;
    if (g.remap || g.tiled || g.row_off) {
      const int64_t row = i / g.row_len, col = i % g.row_len;
      int64_t prow = row;
      if (g.remap)  // [gate; up] rows interleaved by 64 inside each 128-row tile
        prow = (row / 64) * 128 + (g.remap == 2 ? 64 : 0) + row % 64;
      prow += g.row_off;
      o = g.tiled ? (int64_t)tiled_offset(prow, col, g.row_len) : prow * g.row_len + col;
    }
    dst[o] = f2bf(v);
  }
}

cudaError_t launch_gen(const GenSpec& g, uint16_t* dst, cudaStream_t st) {
  float c, offset = 0.f;
  switch (g.kind) {
    case 0: c = (float)(sqrt(3.0 / (double)g.fan_in) / 8388608.0); break;
    case 1: c = (float)(sqrt(3.0) / 8388608.0); break;
    case 2: c = (float)(0.125 / 8388608.0); offset = 1.0f; break;
    default: c = (float)(0.02 * sqrt(3.0) / 8388608.0); break;
  }
  int64_t blocks = (g.n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  k_gen<<<(unsigned)blocks, 256, 0, st>>>(g, c, offset, dst);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a1: embed
__global__ void k_embed(const uint16_t* __restrict__ E, const int32_t* __restrict__ tok, int d,
                        uint16_t* __restrict__ x) {
  griddep();
  const int t = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(E + (size_t)tok[t] * d);
  uint4* dst = reinterpret_cast<uint4*>(x + (size_t)t * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) dst[i] = __ldg(src + i);
}

cudaError_t launch_embed(const uint16_t* E, const int32_t* tok, int T, int d, uint16_t* x, cudaStream_t st) {
  return launch_k(k_embed, dim3(T), dim3(128), 0, st, E, tok, d, x);
}

// ------------------------------------------------------------------ a2: RMSNorm
// One CTA (256 threads) per token.  Fixed reduction tree: thread i sums the
// squares of the 8-element vectors i, i+256, ... in order; xor-shuffle tree
// inside the warp; warp partials summed 0..7 by thread 0.  Same tree at every
// T and in the fused residual variant below (bit-identical results).
__device__ __forceinline__ float block_inv_rms(float ss, int d, float eps, float* red, float* s_inv) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) s = __fadd_rn(s, red[i]);
    const float mean = __fdiv_rn(s, (float)d);
    *s_inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(mean, eps)));
  }
  __syncthreads();
  return *s_inv;
}

__global__ void __launch_bounds__(256) k_rmsnorm(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int d,
                                                 float eps, uint16_t* __restrict__ out) {
  __shared__ float red[8];
  __shared__ float s_inv;
  griddep();
  const int t = blockIdx.x;
  const uint4* xv = reinterpret_cast<const uint4*>(x + (size_t)t * d);
  const int nv = d / 8;
  float ss = 0.f;
  for (int i = threadIdx.x; i < nv; i += 256) ss = ss8(xv[i], ss);
  const float inv = block_inv_rms(ss, d, eps, red, &s_inv);
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  uint4* ov = reinterpret_cast<uint4*>(out + (size_t)t * d);
  for (int i = threadIdx.x; i < nv; i += 256) ov[i] = norm8(xv[i], __ldg(wv + i), inv);
}

cudaError_t launch_rmsnorm(const uint16_t* x, const uint16_t* w, int T, int d, float eps, uint16_t* out,
                           cudaStream_t st) {
  return launch_k(k_rmsnorm, dim3(T), dim3(256), 0, st, x, w, d, eps, out);
}

// ------------------------------------------------------------------ a5/a7 (+a2): residual + RMSNorm
// x <- bf16(x + sum_s part[s]) (splits summed in order), then xn <- RMSNorm(x)
// with the same fixed tree as k_rmsnorm.  One CTA per token.
constexpr int kResThreads = 512;
constexpr int kResMaxV = 2;  // 8-feature vectors per thread: d <= 2 * 512 * 8

// PDL: the residual row (last written >= 2 kernels earlier) and the gains do
// not depend on the immediately preceding kernel, so they are loaded before
// griddepcontrol.wait; only the GEMM partials are read after it.
__global__ void __launch_bounds__(kResThreads) k_residual_norm(uint16_t* __restrict__ x, const float* __restrict__ part,
                                                               PartSpec ps, int T, int d,
                                                               const uint16_t* __restrict__ w, float eps,
                                                               uint16_t* __restrict__ xn) {
  __shared__ float red[kResThreads / 32];
  __shared__ float s_inv;
  const int t = blockIdx.x;
  const size_t stride = (size_t)T * d;
  uint4* xv = reinterpret_cast<uint4*>(x + (size_t)t * d);
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  const int nv = d / 8;
  uint4 hr[kResMaxV], wr[kResMaxV];
#pragma unroll
  for (int j = 0; j < kResMaxV; ++j) {
    const int i = threadIdx.x + j * kResThreads;
    if (i < nv) {
      hr[j] = __ldcg(xv + i);
      if (xn) wr[j] = __ldg(wv + i);
    }
  }
  griddep();
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kResMaxV; ++j) {
    const int i = threadIdx.x + j * kResThreads;
    if (i < nv) {
      float acc[8];
      sum8_pieces(part, part_count(ps, i * 8), stride, (size_t)t * d + (size_t)i * 8, acc);  // one 128-feature tile
      hr[j] = residual8(hr[j], acc);
      xv[i] = hr[j];
      ss = ss8(hr[j], ss);
    }
  }
  const float inv = block_inv_rms(ss, d, eps, red, &s_inv);
  if (!xn) return;
  uint4* ov = reinterpret_cast<uint4*>(xn + (size_t)t * d);
#pragma unroll
  for (int j = 0; j < kResMaxV; ++j) {
    const int i = threadIdx.x + j * kResThreads;
    if (i < nv) ov[i] = norm8(hr[j], wr[j], inv);
  }
}

cudaError_t launch_residual_norm(uint16_t* x, const float* part, PartSpec ps, int T, int d, const uint16_t* w,
                                 float eps, uint16_t* xn, cudaStream_t st) {
  if (d % 8 || d > kResMaxV * kResThreads * 8) return cudaErrorInvalidValue;
  return launch_k(k_residual_norm, dim3(T), dim3(kResThreads), 0, st, x, part, ps, T, d, w, eps, xn);
}

// ------------------------------------------------------------------ a3 epilogue
// grid (T, H + 2KV), block hd/2: thread i owns the rotate-half pair (i, i+hd/2).
// PDL: positions, bias, RoPE factors and the cache slot do not depend on the
// preceding kernel (the QKV GEMM) -- gathered before griddepcontrol.wait.
__global__ void k_epi_qkv(const float* __restrict__ part, PartSpec ps, QkvArgs a) {
  const QkvPair r = qkv_prep(a, blockIdx.x, blockIdx.y, threadIdx.x);
  griddep();
  qkv_finish(a, r, part, ps, blockIdx.y, threadIdx.x);
}

cudaError_t launch_epi_qkv(const float* part, PartSpec ps, const uint16_t* bias, const int32_t* pos, int T, int H,
                           int KV, int hd, const float* rope_cos, const float* rope_sin, uint16_t* q,
                           const CacheView* cache, const int32_t* slot, uint16_t* k_out, uint16_t* v_out,
                           cudaStream_t st, int part_T) {
  QkvArgs a{};
  a.part_T = part_T;
  a.bias = bias; a.pos = pos; a.T = T; a.H = H; a.KV = KV; a.hd = hd; a.rcos = rope_cos; a.rsin = rope_sin;
  a.q = q; a.paged = cache != nullptr; a.slot = slot; a.kd = k_out; a.vd = v_out;
  if (cache) a.cache = *cache;
  return launch_k(k_epi_qkv, dim3(T, H + 2 * KV), dim3(hd / 2), 0, st, part, ps, a);
}

// ------------------------------------------------------------------ residual (op-level tests)
__global__ void k_epi_residual(const uint16_t* __restrict__ x, const float* __restrict__ part, PartSpec ps, size_t n,
                               int N, uint16_t* __restrict__ out) {
  griddep();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float a = sum_splits(part, part_count(ps, (int)(i % N)), n, i);
    out[i] = f2bf(__fadd_rn(bf2f(x[i]), a));
  }
}

cudaError_t launch_epi_residual(const uint16_t* x, const float* part, PartSpec ps, int T, int N, uint16_t* out,
                                cudaStream_t st) {
  const size_t n = (size_t)T * N;
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_k(k_epi_residual, dim3((unsigned)blocks), dim3(256), 0, st, x, part, ps, n, N, out);
}

// ------------------------------------------------------------------ a6: SwiGLU
// thread per 4 consecutive outputs (epilogue.cuh swiglu4)
// The kernel is L2-latency bound: its time is the number of rounds of partial
// loads.  With the slot count of the op's partition known at launch (<= 2 for
// the stream-K gate/up GEMMs of the model shapes), the light SMAX = 2 form
// keeps the registers low enough that every item's loads are in flight in one
// wave of threads.
template <int SMAX>
__global__ void k_epi_swiglu(const float* __restrict__ part, PartSpec ps, int T, int F, uint16_t* __restrict__ out) {
  griddep();
  const size_t n4 = (size_t)T * F / 4;
  for (size_t e4 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e4 < n4; e4 += (size_t)gridDim.x * blockDim.x)
    swiglu4_s<SMAX>(part, ps, T, F, e4 * 4, out);
}

// two items per thread, every load of both issued before any arithmetic, for
// partitions with <= 2 slots per output (one round of L2 latency per thread)
__global__ void __launch_bounds__(256) k_epi_swiglu2(const float* __restrict__ part, PartSpec ps, int T, int F,
                                                     uint16_t* __restrict__ out) {
  griddep();
  const size_t n4 = (size_t)T * F / 4;
  const size_t stride = (size_t)T * 2 * F;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  float4 v[2][4];
  size_t e[2];
  int S[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const size_t e4 = i0 + k * nth;
    e[k] = e4 * 4;
    S[k] = 0;
    if (e4 < n4) {
      const int t = (int)e[k] / F, j = (int)e[k] % F;
      const int col = (j / 64) * 128 + (j % 64);
      S[k] = part_count(ps, col);
      const float* p0 = part + (size_t)t * 2 * F + (size_t)col;
      v[k][0] = __ldcg(reinterpret_cast<const float4*>(p0));
      v[k][1] = __ldcg(reinterpret_cast<const float4*>(p0 + 64));
      if (S[k] > 1) {
        v[k][2] = __ldcg(reinterpret_cast<const float4*>(p0 + stride));
        v[k][3] = __ldcg(reinterpret_cast<const float4*>(p0 + stride + 64));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (S[k] == 0) continue;
    float4 g = v[k][0], u = v[k][1];
    if (S[k] > 1) {
      g.x = __fadd_rn(g.x, v[k][2].x); g.y = __fadd_rn(g.y, v[k][2].y); g.z = __fadd_rn(g.z, v[k][2].z); g.w = __fadd_rn(g.w, v[k][2].w);
      u.x = __fadd_rn(u.x, v[k][3].x); u.y = __fadd_rn(u.y, v[k][3].y); u.z = __fadd_rn(u.z, v[k][3].z); u.w = __fadd_rn(u.w, v[k][3].w);
    }
    const float gg[4] = {g.x, g.y, g.z, g.w}, uu[4] = {u.x, u.y, u.z, u.w};
    float a[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = __fmul_rn(__fdiv_rn(gg[q], __fadd_rn(1.0f, expf(-gg[q]))), uu[q]);
    *reinterpret_cast<uint2*>(out + e[k]) = make_uint2(pack_bf2(a[0], a[1]), pack_bf2(a[2], a[3]));
  }
}

#ifndef MG_SWIGLU_LIGHT
#define MG_SWIGLU_LIGHT 2
#endif
cudaError_t launch_epi_swiglu(const float* part, PartSpec ps, int T, int F, uint16_t* out, cudaStream_t st) {
  if ((long long)T * 2 * F >= (1LL << 31)) return cudaErrorInvalidValue;
  const size_t n4 = (size_t)T * F / 4;
  size_t blocks = (n4 + 255) / 256;
  if (MG_SWIGLU_LIGHT == 2 && part_slots(ps, 2 * F) <= 2) {
    const size_t b2 = (n4 + 511) / 512;
    return launch_k(k_epi_swiglu2, dim3((unsigned)b2), dim3(256), 0, st, part, ps, T, F, out);
  }
  if (MG_SWIGLU_LIGHT && part_slots(ps, 2 * F) <= 2) {
    if (blocks > (size_t)num_sms() * 64) blocks = (size_t)num_sms() * 64;
    return launch_k(k_epi_swiglu<2>, dim3((unsigned)blocks), dim3(256), 0, st, part, ps, T, F, out);
  }
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_k(k_epi_swiglu<4>, dim3((unsigned)blocks), dim3(256), 0, st, part, ps, T, F, out);
}

// ------------------------------------------------------------------ row gather
__global__ void k_gather_rows(const uint16_t* __restrict__ src, const int32_t* __restrict__ rows, int sub, int d,
                              uint16_t* __restrict__ dst) {
  griddep();
  const int i = blockIdx.x;
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)(rows[i] - sub) * d);
  uint4* o = reinterpret_cast<uint4*>(dst + (size_t)i * d);
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) o[j] = s[j];
}

cudaError_t launch_gather_rows(const uint16_t* src, const int32_t* rows, int n, int d, uint16_t* dst,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_k(k_gather_rows, dim3(n), dim3(128), 0, st, src, rows, 0, d, dst);
}

cudaError_t launch_gather_rows_sub(const uint16_t* src, const int32_t* rows, int sub, int n, int d, uint16_t* dst,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_k(k_gather_rows, dim3(n), dim3(128), 0, st, src, rows, sub, d, dst);
}

}  // namespace mg
