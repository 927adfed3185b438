// elementwise.cu -- the CUDA-core kernels of the decode path that are not
// GEMMs (SURVEY 8(a) rows a1, a2 and the GEMM epilogues of a3, a5-a7), plus
// the K0 weight generator.  Every rounding point follows DESIGN.md 3.3:
// IEEE fp32 with explicit __fmul_rn/__fadd_rn/__fdiv_rn/__fsqrt_rn (no FMA
// contraction of the epilogue math), bf16 by round-to-nearest-even.
// All kernels are per-token: a token's output never depends on which other
// tokens share the launch (the verifier's batch invariance).
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
    if (g.remap) {  // [gate; up] rows interleaved by 64 inside each 128-row tile
      const int64_t row = i / g.row_len, col = i % g.row_len;
      const int64_t prow = (row / 64) * 128 + (g.remap == 2 ? 64 : 0) + row % 64;
      o = prow * g.row_len + col;
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
  const int t = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(E + (size_t)tok[t] * d);
  uint4* dst = reinterpret_cast<uint4*>(x + (size_t)t * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) dst[i] = __ldg(src + i);
}

cudaError_t launch_embed(const uint16_t* E, const int32_t* tok, int T, int d, uint16_t* x, cudaStream_t st) {
  k_embed<<<T, 128, 0, st>>>(E, tok, d, x);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a2: RMSNorm
// One CTA (256 threads) per token.  Fixed reduction tree: thread i sums the
// 8-element vectors i, i+256, ... in order; xor-shuffle tree inside the warp;
// warp partials summed 0..7 by thread 0.  Same tree at every T.
__global__ void __launch_bounds__(256) k_rmsnorm(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int d,
                                                 float eps, uint16_t* __restrict__ out) {
  __shared__ float red[8];
  __shared__ float s_inv;
  const int t = blockIdx.x;
  const uint4* xv = reinterpret_cast<const uint4*>(x + (size_t)t * d);
  const int nv = d / 8;
  float ss = 0.f;
  for (int i = threadIdx.x; i < nv; i += 256) {
    const uint4 v = xv[i];
    const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float a = lo_bf(u[j]), b = hi_bf(u[j]);
      ss = fmaf(a, a, ss);  // bf16^2 is exact in fp32: fma == mul+add
      ss = fmaf(b, b, ss);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = red[0];
    for (int i = 1; i < 8; ++i) s = __fadd_rn(s, red[i]);
    const float mean = __fdiv_rn(s, (float)d);
    s_inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(mean, eps)));
  }
  __syncthreads();
  const float inv = s_inv;
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  uint4* ov = reinterpret_cast<uint4*>(out + (size_t)t * d);
  for (int i = threadIdx.x; i < nv; i += 256) {
    const uint4 v = xv[i], g = __ldg(wv + i);
    const uint32_t u[4] = {v.x, v.y, v.z, v.w}, gw[4] = {g.x, g.y, g.z, g.w};
    uint32_t r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      r[j] = pack_bf2(__fmul_rn(__fmul_rn(lo_bf(u[j]), inv), lo_bf(gw[j])),
                      __fmul_rn(__fmul_rn(hi_bf(u[j]), inv), hi_bf(gw[j])));
    ov[i] = make_uint4(r[0], r[1], r[2], r[3]);
  }
}

cudaError_t launch_rmsnorm(const uint16_t* x, const uint16_t* w, int T, int d, float eps, uint16_t* out,
                           cudaStream_t st) {
  k_rmsnorm<<<T, 256, 0, st>>>(x, w, d, eps, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a3 epilogue
__device__ __forceinline__ float sum_splits(const float* __restrict__ part, int S, size_t stride, size_t idx) {
  float a = part[idx];
  for (int s = 1; s < S; ++s) a = __fadd_rn(a, part[(size_t)s * stride + idx]);
  return a;
}

__device__ __forceinline__ uint16_t* cache_ptr(const CacheView& c, int slot, int pos, int kvsel, int head) {
  const int page = c.pt[(size_t)slot * c.max_pages + pos / c.page_size];
  return c.pool + ((((size_t)c.layer * c.n_pages + page) * 2 + kvsel) * c.kv + head) * (size_t)c.page_size * c.hd +
         (size_t)(pos % c.page_size) * c.hd;
}

// grid (T, H + 2KV), block hd/2: thread i owns the rotate-half pair (i, i+hd/2)
__global__ void k_epi_qkv(const float* __restrict__ part, int S, const uint16_t* __restrict__ bias,
                          const int32_t* __restrict__ pos, int T, int H, int KV, int hd,
                          const float* __restrict__ rcos, const float* __restrict__ rsin, uint16_t* __restrict__ q,
                          CacheView cache, bool paged, const int32_t* __restrict__ slot, uint16_t* __restrict__ kd,
                          uint16_t* __restrict__ vd) {
  const int t = blockIdx.x, h = blockIdx.y, i = threadIdx.x, h2 = hd / 2;
  const int NQKV = (H + 2 * KV) * hd;
  const size_t stride = (size_t)T * NQKV;
  const int f1 = h * hd + i, f2 = f1 + h2;
  float a = sum_splits(part, S, stride, (size_t)t * NQKV + f1);
  float b = sum_splits(part, S, stride, (size_t)t * NQKV + f2);
  if (bias) {
    a = __fadd_rn(a, bf2f(bias[f1]));
    b = __fadd_rn(b, bf2f(bias[f2]));
  }
  const int p = pos[t];
  uint16_t oa, ob;
  if (h < H + KV) {  // RoPE on q and k
    const float c = rcos[(size_t)p * h2 + i], s = rsin[(size_t)p * h2 + i];
    oa = f2bf(__fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s)));
    ob = f2bf(__fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s)));
  } else {
    oa = f2bf(a);
    ob = f2bf(b);
  }
  if (h < H) {
    q[(size_t)t * H * hd + h * hd + i] = oa;
    q[(size_t)t * H * hd + h * hd + i + h2] = ob;
    return;
  }
  const int kvsel = h < H + KV ? 0 : 1;
  const int kh = h - H - kvsel * KV;
  uint16_t* dst;
  if (paged) {
    dst = cache_ptr(cache, slot[t], p, kvsel, kh);  // tentative append of column p
  } else {
    dst = (kvsel ? vd : kd) + (size_t)t * KV * hd + kh * hd;
  }
  dst[i] = oa;
  dst[i + h2] = ob;
}

cudaError_t launch_epi_qkv(const float* part, int S, const uint16_t* bias, const int32_t* pos, int T, int H, int KV,
                           int hd, const float* rope_cos, const float* rope_sin, uint16_t* q,
                           const CacheView* cache, const int32_t* slot, uint16_t* k_out, uint16_t* v_out,
                           cudaStream_t st) {
  CacheView cv{};
  if (cache) cv = *cache;
  dim3 grid(T, H + 2 * KV);
  k_epi_qkv<<<grid, hd / 2, 0, st>>>(part, S, bias, pos, T, H, KV, hd, rope_cos, rope_sin, q, cv, cache != nullptr,
                                     slot, k_out, v_out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a5/a7: residual
__global__ void k_epi_residual(const uint16_t* __restrict__ x, const float* __restrict__ part, int S, size_t n,
                               uint16_t* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float a = sum_splits(part, S, n, i);
    out[i] = f2bf(__fadd_rn(bf2f(x[i]), a));
  }
}

cudaError_t launch_epi_residual(const uint16_t* x, const float* part, int S, int T, int N, uint16_t* out,
                                cudaStream_t st) {
  const size_t n = (size_t)T * N;
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_epi_residual<<<(unsigned)blocks, 256, 0, st>>>(x, part, S, n, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a6: SwiGLU
__global__ void k_epi_swiglu(const float* __restrict__ part, int S, int T, int F, uint16_t* __restrict__ out) {
  const size_t n = (size_t)T * F, stride = (size_t)T * 2 * F;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const size_t t = e / F;
    const int j = (int)(e % F);
    const size_t gcol = (size_t)(j / 64) * 128 + (j % 64);
    const float g = sum_splits(part, S, stride, t * 2 * F + gcol);
    const float u = sum_splits(part, S, stride, t * 2 * F + gcol + 64);
    const float den = __fadd_rn(1.0f, expf(-g));
    out[e] = f2bf(__fmul_rn(__fdiv_rn(g, den), u));
  }
}

cudaError_t launch_epi_swiglu(const float* part, int S, int T, int F, uint16_t* out, cudaStream_t st) {
  const size_t n = (size_t)T * F;
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_epi_swiglu<<<(unsigned)blocks, 256, 0, st>>>(part, S, T, F, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ row gather
__global__ void k_gather_rows(const uint16_t* __restrict__ src, const int32_t* __restrict__ rows, int sub, int d,
                              uint16_t* __restrict__ dst) {
  const int i = blockIdx.x;
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)(rows[i] - sub) * d);
  uint4* o = reinterpret_cast<uint4*>(dst + (size_t)i * d);
  for (int j = threadIdx.x; j < d / 8; j += blockDim.x) o[j] = s[j];
}

cudaError_t launch_gather_rows(const uint16_t* src, const int32_t* rows, int n, int d, uint16_t* dst,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_gather_rows<<<n, 128, 0, st>>>(src, rows, 0, d, dst);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows_sub(const uint16_t* src, const int32_t* rows, int sub, int n, int d, uint16_t* dst,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_gather_rows<<<n, 128, 0, st>>>(src, rows, sub, d, dst);
  return cudaGetLastError();
}

}  // namespace mg
