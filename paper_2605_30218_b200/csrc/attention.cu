// attention.cu -- paged GQA decode attention.
//
// k_attn_partial: one CTA per (token, kv head, key chunk).  The chunk's keys
// [c*chunk, min((c+1)*chunk, n_keys)) are read from the paged cache (or a
// dense buffer in the op-level tests); the G = H/KV query heads that share
// the kv head are processed together so each K/V byte is read once per
// token.  Scores: warp w takes keys lo+w, lo+w+4, ...; each lane holds
// hd/32 dims, fp32 dot + fixed xor-shuffle tree, times fp32(1/sqrt(hd)).
// Softmax partial per head: m = max, e = expf(s - m), l = fixed-tree sum;
// acc[d] = sum_j e_j v_j[d] over the chunk's keys in order.
// k_attn_combine: chunks combined in chunk order with weights expf(m_c - m*),
// o = bf16(acc / l).
//
// Schedules: the fast path picks `chunk` from (batch, context) to fill the
// 148 SMs (the serving shape changes the reduction plan); the
// verifier always uses a fixed chunk (A14), so a query's result
// depends only on its own keys.
#include "common.cuh"
#include "kernels.h"

namespace mg {

constexpr int kAttnThreads = 128;
constexpr int kAttnCMax = 512;  // max keys per chunk
constexpr int kAttnGMax = 8;    // max query heads per kv head

__global__ void __launch_bounds__(kAttnThreads) k_attn_partial(AttnArgs a) {
  __shared__ float qs[kAttnGMax][128];
  __shared__ float sc[kAttnGMax][kAttnCMax];
  __shared__ float red[4][kAttnGMax];
  __shared__ float s_m[kAttnGMax], s_l[kAttnGMax];
  __shared__ float accx[kAttnGMax][64];

  const int t = blockIdx.x, kvh = blockIdx.y, c = blockIdx.z;
  const int H = a.H, hd = a.hd, G = a.H / a.KV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.n_keys[t];
  const int lo = c * a.chunk;
  const size_t po = ((size_t)t * H + (size_t)kvh * G) * a.n_chunks + c;  // head g: po + g*n_chunks
  if (lo >= n) {
    if (threadIdx.x < G) {
      a.part_ml[(po + (size_t)threadIdx.x * a.n_chunks) * 2 + 0] = -INFINITY;
      a.part_ml[(po + (size_t)threadIdx.x * a.n_chunks) * 2 + 1] = 0.f;
    }
    return;
  }
  const int hi = min(n, lo + a.chunk);
  const int len = hi - lo;

  for (int e = threadIdx.x; e < G * hd; e += kAttnThreads)
    qs[e / hd][e % hd] = bf2f(a.q[(size_t)t * H * hd + (size_t)kvh * G * hd + e]);

  // K/V row pointer of key j
  int slot = 0;
  if (a.paged) slot = a.slot[t];
  auto krow = [&](int j, int kvsel) -> const uint16_t* {
    if (a.paged) {
      const CacheView& cv = a.cache;
      const int page = cv.pt[(size_t)slot * cv.max_pages + j / cv.page_size];
      return cv.pool + ((((size_t)cv.layer * cv.n_pages + page) * 2 + kvsel) * cv.kv + kvh) *
                           (size_t)cv.page_size * hd +
             (size_t)(j % cv.page_size) * hd;
    }
    const uint16_t* base = kvsel ? a.Vd : a.Kd;
    return base + (((size_t)t * a.KV + kvh) * a.key_stride + j) * hd;
  };
  __syncthreads();

  const float scale = (float)(1.0 / sqrt((double)hd));
  // ---- scores
  if (hd == 128) {
    for (int j = lo + warp; j < hi; j += 4) {
      const uint2 kv = *reinterpret_cast<const uint2*>(krow(j, 0) + lane * 4);
      const float k0 = lo_bf(kv.x), k1 = hi_bf(kv.x), k2 = lo_bf(kv.y), k3 = hi_bf(kv.y);
      for (int g = 0; g < G; ++g) {
        const float* qg = &qs[g][lane * 4];
        float p = qg[0] * k0;
        p = fmaf(qg[1], k1, p);
        p = fmaf(qg[2], k2, p);
        p = fmaf(qg[3], k3, p);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) p = __fadd_rn(p, __shfl_xor_sync(0xffffffffu, p, off));
        if (lane == 0) sc[g][j - lo] = __fmul_rn(p, scale);
      }
    }
  } else {  // hd == 64
    for (int j = lo + warp; j < hi; j += 4) {
      const uint32_t kv = *reinterpret_cast<const uint32_t*>(krow(j, 0) + lane * 2);
      const float k0 = lo_bf(kv), k1 = hi_bf(kv);
      for (int g = 0; g < G; ++g) {
        float p = qs[g][lane * 2] * k0;
        p = fmaf(qs[g][lane * 2 + 1], k1, p);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) p = __fadd_rn(p, __shfl_xor_sync(0xffffffffu, p, off));
        if (lane == 0) sc[g][j - lo] = __fmul_rn(p, scale);
      }
    }
  }
  __syncthreads();

  // ---- softmax partial per head (fixed trees)
  for (int g = 0; g < G; ++g) {
    float m = -INFINITY;
    for (int j = threadIdx.x; j < len; j += kAttnThreads) m = fmaxf(m, sc[g][j]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (lane == 0) red[warp][g] = m;
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int g = threadIdx.x;
    s_m[g] = fmaxf(fmaxf(red[0][g], red[1][g]), fmaxf(red[2][g], red[3][g]));
  }
  __syncthreads();
  for (int g = 0; g < G; ++g) {
    const float m = s_m[g];
    float l = 0.f;
    for (int j = threadIdx.x; j < len; j += kAttnThreads) {
      const float e = expf(__fsub_rn(sc[g][j], m));
      sc[g][j] = e;
      l = __fadd_rn(l, e);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l = __fadd_rn(l, __shfl_xor_sync(0xffffffffu, l, off));
    if (lane == 0) red[warp][g] = l;
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int g = threadIdx.x;
    s_l[g] = __fadd_rn(__fadd_rn(red[0][g], red[1][g]), __fadd_rn(red[2][g], red[3][g]));
  }
  // ---- P.V: thread (kg, d) sums keys lo+kg, lo+kg+KG, ... in order
  const int KG = kAttnThreads / hd;  // 1 (hd 128) or 2 (hd 64)
  const int kg = threadIdx.x / hd, d = threadIdx.x % hd;
  float acc[kAttnGMax];
#pragma unroll
  for (int g = 0; g < kAttnGMax; ++g) acc[g] = 0.f;
  for (int j = lo + kg; j < hi; j += KG) {
    const float v = bf2f(krow(j, 1)[d]);
#pragma unroll
    for (int g = 0; g < kAttnGMax; ++g)
      if (g < G) acc[g] = fmaf(sc[g][j - lo], v, acc[g]);
  }
  if (KG == 2) {
    __syncthreads();
    if (kg == 1)
      for (int g = 0; g < G; ++g) accx[g][d] = acc[g];
    __syncthreads();
    if (kg == 1) return;
    for (int g = 0; g < G; ++g) acc[g] = __fadd_rn(acc[g], accx[g][d]);
  } else {
    __syncthreads();
  }
  for (int g = 0; g < G; ++g) {
    const size_t o = po + (size_t)g * a.n_chunks;
    a.part_acc[o * hd + d] = acc[g];
    if (d == 0) {
      a.part_ml[o * 2 + 0] = s_m[g];
      a.part_ml[o * 2 + 1] = s_l[g];
    }
  }
}

// grid (T, H), block hd
__global__ void k_attn_combine(const float* __restrict__ part_acc, const float* __restrict__ part_ml,
                               const int32_t* __restrict__ n_keys, int H, int hd, int chunk, int n_chunks,
                               uint16_t* __restrict__ out) {
  const int t = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const int nch = (n_keys[t] + chunk - 1) / chunk;
  const size_t base = ((size_t)t * H + h) * n_chunks;
  float ms = -INFINITY;
  for (int c = 0; c < nch; ++c) ms = fmaxf(ms, part_ml[(base + c) * 2]);
  float L = 0.f, acc = 0.f;
  for (int c = 0; c < nch; ++c) {
    const float w = expf(__fsub_rn(part_ml[(base + c) * 2], ms));
    L = __fadd_rn(L, __fmul_rn(part_ml[(base + c) * 2 + 1], w));
    acc = __fadd_rn(acc, __fmul_rn(part_acc[(base + c) * hd + d], w));
  }
  out[(size_t)t * H * hd + (size_t)h * hd + d] = f2bf(__fdiv_rn(acc, L));
}

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t st) {
  if (a.hd != 64 && a.hd != 128) return cudaErrorInvalidValue;
  if (a.H / a.KV > kAttnGMax || a.chunk > kAttnCMax || a.chunk < 1) return cudaErrorInvalidValue;
  dim3 g1(a.T, a.KV, a.n_chunks);
  k_attn_partial<<<g1, kAttnThreads, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 g2(a.T, a.H);
  k_attn_combine<<<g2, a.hd, 0, st>>>(a.part_acc, a.part_ml, a.n_keys, a.H, a.hd, a.chunk, a.n_chunks, a.out);
  return cudaGetLastError();
}

}  // namespace mg
