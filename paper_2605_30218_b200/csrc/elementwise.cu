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

__device__ __forceinline__ uint4 norm8(uint4 v, uint4 g, float inv) {
  const uint32_t u[4] = {v.x, v.y, v.z, v.w}, gw[4] = {g.x, g.y, g.z, g.w};
  uint32_t r[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    r[j] = pack_bf2(__fmul_rn(__fmul_rn(lo_bf(u[j]), inv), lo_bf(gw[j])),
                    __fmul_rn(__fmul_rn(hi_bf(u[j]), inv), hi_bf(gw[j])));
  return make_uint4(r[0], r[1], r[2], r[3]);
}

__device__ __forceinline__ float ss8(uint4 v, float ss) {
  const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float a = lo_bf(u[j]), b = hi_bf(u[j]);
    ss = fmaf(a, a, ss);  // bf16^2 is exact in fp32: fma == mul+add
    ss = fmaf(b, b, ss);
  }
  return ss;
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
// sum of the S partial slots of one output, in slot (= k) order; the first 8
// loads are issued together (predicated), the adds stay in order
__device__ __forceinline__ float sum_splits(const float* __restrict__ part, int S, size_t stride, size_t idx) {
  float v[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = s < S ? part[(size_t)s * stride + idx] : 0.f;
  float a = v[0];
#pragma unroll
  for (int s = 1; s < 8; ++s)
    if (s < S) a = __fadd_rn(a, v[s]);
  for (int s = 8; s < S; ++s) a = __fadd_rn(a, part[(size_t)s * stride + idx]);
  return a;
}

// 8 consecutive fp32 partial sums (one 8-feature vector), pieces added in order;
// the loads of up to 8 pieces are issued together
__device__ __forceinline__ void sum8_pieces(const float* __restrict__ part, int S, size_t stride, size_t idx,
                                            float* out) {
  float4 lo[8], hi[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    if (s < S) {
      lo[s] = *reinterpret_cast<const float4*>(part + (size_t)s * stride + idx);
      hi[s] = *reinterpret_cast<const float4*>(part + (size_t)s * stride + idx + 4);
    }
  }
  float a[8] = {lo[0].x, lo[0].y, lo[0].z, lo[0].w, hi[0].x, hi[0].y, hi[0].z, hi[0].w};
#pragma unroll
  for (int s = 1; s < 8; ++s) {
    if (s < S) {
      a[0] = __fadd_rn(a[0], lo[s].x); a[1] = __fadd_rn(a[1], lo[s].y);
      a[2] = __fadd_rn(a[2], lo[s].z); a[3] = __fadd_rn(a[3], lo[s].w);
      a[4] = __fadd_rn(a[4], hi[s].x); a[5] = __fadd_rn(a[5], hi[s].y);
      a[6] = __fadd_rn(a[6], hi[s].z); a[7] = __fadd_rn(a[7], hi[s].w);
    }
  }
  for (int s = 8; s < S; ++s)
    for (int k = 0; k < 8; ++k) a[k] = __fadd_rn(a[k], part[(size_t)s * stride + idx + k]);
#pragma unroll
  for (int k = 0; k < 8; ++k) out[k] = a[k];
}

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
      const uint32_t u[4] = {hr[j].x, hr[j].y, hr[j].z, hr[j].w};
      float acc[8];
      sum8_pieces(part, part_count(ps, i * 8), stride, (size_t)t * d + (size_t)i * 8, acc);  // one 128-feature tile
      uint32_t r[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        r[q] = pack_bf2(__fadd_rn(lo_bf(u[q]), acc[2 * q]), __fadd_rn(hi_bf(u[q]), acc[2 * q + 1]));
      hr[j] = make_uint4(r[0], r[1], r[2], r[3]);
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
__device__ __forceinline__ uint16_t* cache_ptr(const CacheView& c, int slot, int pos, int kvsel, int head) {
  const int page = c.pt[(size_t)slot * c.max_pages + pos / c.page_size];
  return c.pool + ((((size_t)c.layer * c.n_pages + page) * 2 + kvsel) * c.kv + head) * (size_t)c.page_size * c.hd +
         (size_t)(pos % c.page_size) * c.hd;
}

// grid (T, H + 2KV), block hd/2: thread i owns the rotate-half pair (i, i+hd/2)
__global__ void k_epi_qkv(const float* __restrict__ part, PartSpec ps, const uint16_t* __restrict__ bias,
                          const int32_t* __restrict__ pos, int T, int H, int KV, int hd,
                          const float* __restrict__ rcos, const float* __restrict__ rsin, uint16_t* __restrict__ q,
                          CacheView cache, bool paged, const int32_t* __restrict__ slot, uint16_t* __restrict__ kd,
                          uint16_t* __restrict__ vd) {
  // PDL: positions, bias, RoPE factors and the cache slot do not depend on
  // the preceding kernel (the QKV GEMM) -- gathered before griddepcontrol.wait
  const int t = blockIdx.x, h = blockIdx.y, i = threadIdx.x, h2 = hd / 2;
  const int NQKV = (H + 2 * KV) * hd;
  const size_t stride = (size_t)T * NQKV;
  const int f1 = h * hd + i, f2 = f1 + h2;
  const int p = pos[t];
  float ba = 0.f, bb = 0.f, c = 1.f, sn = 0.f;
  if (bias) {
    ba = bf2f(bias[f1]);
    bb = bf2f(bias[f2]);
  }
  if (h < H + KV) {
    c = rcos[(size_t)p * h2 + i];
    sn = rsin[(size_t)p * h2 + i];
  }
  uint16_t* dst;
  if (h < H) {
    dst = q + (size_t)t * H * hd + h * hd;
  } else {
    const int kvsel = h < H + KV ? 0 : 1;
    const int kh = h - H - kvsel * KV;
    dst = paged ? cache_ptr(cache, slot[t], p, kvsel, kh)  // tentative append of column p
                : (kvsel ? vd : kd) + (size_t)t * KV * hd + kh * hd;
  }
  griddep();
  float a = sum_splits(part, part_count(ps, f1), stride, (size_t)t * NQKV + f1);
  float b = sum_splits(part, part_count(ps, f2), stride, (size_t)t * NQKV + f2);
  if (bias) {
    a = __fadd_rn(a, ba);
    b = __fadd_rn(b, bb);
  }
  uint16_t oa, ob;
  if (h < H + KV) {  // RoPE on q and k
    oa = f2bf(__fsub_rn(__fmul_rn(a, c), __fmul_rn(b, sn)));
    ob = f2bf(__fadd_rn(__fmul_rn(b, c), __fmul_rn(a, sn)));
  } else {
    oa = f2bf(a);
    ob = f2bf(b);
  }
  dst[i] = oa;
  dst[i + h2] = ob;
}

cudaError_t launch_epi_qkv(const float* part, PartSpec ps, const uint16_t* bias, const int32_t* pos, int T, int H,
                           int KV, int hd, const float* rope_cos, const float* rope_sin, uint16_t* q,
                           const CacheView* cache, const int32_t* slot, uint16_t* k_out, uint16_t* v_out,
                           cudaStream_t st) {
  CacheView cv{};
  if (cache) cv = *cache;
  const bool paged = cache != nullptr;
  return launch_k(k_epi_qkv, dim3(T, H + 2 * KV), dim3(hd / 2), 0, st, part, ps, bias, pos, T, H, KV, hd, rope_cos,
                  rope_sin, q, cv, paged, slot, k_out, v_out);
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
// thread per 4 consecutive outputs (same 64-block, so gate/up columns are
// contiguous float4s)
__global__ void k_epi_swiglu(const float* __restrict__ part, PartSpec ps, int T, int F, uint16_t* __restrict__ out) {
  griddep();
  const size_t n4 = (size_t)T * F / 4, stride = (size_t)T * 2 * F;
  for (size_t e4 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e4 < n4; e4 += (size_t)gridDim.x * blockDim.x) {
    const size_t e = e4 * 4;
    const size_t t = e / F;
    const int j = (int)(e % F);
    const int col = (j / 64) * 128 + (j % 64);  // gate column; up = col + 64 (same 128-feature tile)
    const int S = part_count(ps, col);
    const size_t gcol = t * 2 * F + (size_t)col;
    float4 g = *reinterpret_cast<const float4*>(part + gcol);
    float4 u = *reinterpret_cast<const float4*>(part + gcol + 64);
    for (int s = 1; s < S; ++s) {
      const float4 g2 = *reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol);
      const float4 u2 = *reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol + 64);
      g.x = __fadd_rn(g.x, g2.x); g.y = __fadd_rn(g.y, g2.y); g.z = __fadd_rn(g.z, g2.z); g.w = __fadd_rn(g.w, g2.w);
      u.x = __fadd_rn(u.x, u2.x); u.y = __fadd_rn(u.y, u2.y); u.z = __fadd_rn(u.z, u2.z); u.w = __fadd_rn(u.w, u2.w);
    }
    const float gg[4] = {g.x, g.y, g.z, g.w}, uu[4] = {u.x, u.y, u.z, u.w};
    float a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float den = __fadd_rn(1.0f, expf(-gg[k]));
      a[k] = __fmul_rn(__fdiv_rn(gg[k], den), uu[k]);
    }
    *reinterpret_cast<uint2*>(out + e) = make_uint2(pack_bf2(a[0], a[1]), pack_bf2(a[2], a[3]));
  }
}

cudaError_t launch_epi_swiglu(const float* part, PartSpec ps, int T, int F, uint16_t* out, cudaStream_t st) {
  const size_t n4 = (size_t)T * F / 4;
  size_t blocks = (n4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_k(k_epi_swiglu, dim3((unsigned)blocks), dim3(256), 0, st, part, ps, T, F, out);
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
