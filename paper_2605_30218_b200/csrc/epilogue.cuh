// epilogue.cuh -- device-side GEMM epilogue math shared by the standalone
// elementwise kernels (elementwise.cu), the attention kernel's fused QKV
// epilogue and the GEMM's fused prologue (gemm.cu): split-K partial sums in k
// order, the RMSNorm pieces, SwiGLU and the QKV bias + RoPE + cache append.  Every rounding point follows DESIGN.md
// 3.3 (explicit __fadd_rn/__fmul_rn/__fdiv_rn, bf16 round-to-nearest-even).
// Partials are read with ld.global.cg (L2): other CTAs wrote them, so no L1
// line may be trusted.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace mg {

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

// sum of the S partial slots of one output, in slot (= k) order; the first 8
// loads are issued together (predicated), the adds stay in order
__device__ __forceinline__ float sum_splits(const float* __restrict__ part, int S, size_t stride, size_t idx) {
  float v[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = s < S ? __ldcg(part + (size_t)s * stride + idx) : 0.f;
  float a = v[0];
#pragma unroll
  for (int s = 1; s < 8; ++s)
    if (s < S) a = __fadd_rn(a, v[s]);
  for (int s = 8; s < S; ++s) a = __fadd_rn(a, __ldcg(part + (size_t)s * stride + idx));
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
      lo[s] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + idx));
      hi[s] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + idx + 4));
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
    for (int k = 0; k < 8; ++k) a[k] = __fadd_rn(a[k], __ldcg(part + (size_t)s * stride + idx + k));
#pragma unroll
  for (int k = 0; k < 8; ++k) out[k] = a[k];
}

// x (bf16 vector) + 8 partial sums -> bf16 residual vector
__device__ __forceinline__ uint4 residual8(uint4 x, const float* acc) {
  const uint32_t u[4] = {x.x, x.y, x.z, x.w};
  uint32_t r[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    r[q] = pack_bf2(__fadd_rn(lo_bf(u[q]), acc[2 * q]), __fadd_rn(hi_bf(u[q]), acc[2 * q + 1]));
  return make_uint4(r[0], r[1], r[2], r[3]);
}

__device__ __forceinline__ uint16_t* cache_ptr(const CacheView& c, int slot, int pos, int kvsel, int head) {
  const int page = c.pt[(size_t)slot * c.max_pages + pos / c.page_size];
  return c.pool + ((((size_t)c.layer * c.n_pages + page) * 2 + kvsel) * c.kv + head) * (size_t)c.page_size * c.hd +
         (size_t)(pos % c.page_size) * c.hd;
}

// ---- SwiGLU: 4 consecutive outputs e..e+3 of a [T][F] (same 64-block, so the
// gate/up columns are contiguous float4s in the 64-interleaved [gate;up] tile)
// SMAX: slots whose loads are issued together (more slots are added in a
// loop, still in slot order); the kernel picks the smallest SMAX covering the
// op's partition so the thread stays light enough for one wave of threads.
template <int SMAX>
__device__ __forceinline__ void swiglu4_s(const float* __restrict__ part, const PartSpec& ps, int T, int F, size_t e,
                                          uint16_t* __restrict__ out) {
  const size_t stride = (size_t)T * 2 * F;
  const int t = (int)e / F;
  const int j = (int)e % F;
  const int col = (j / 64) * 128 + (j % 64);
  const int S = part_count(ps, col);
  const size_t gcol = (size_t)t * 2 * F + (size_t)col;
  float4 gs[SMAX], us[SMAX];
#pragma unroll
  for (int s = 0; s < SMAX; ++s)
    if (s < S) {
      gs[s] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol));
      us[s] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol + 64));
    }
  float4 g = gs[0], u = us[0];
#pragma unroll
  for (int s = 1; s < SMAX; ++s)
    if (s < S) {
      g.x = __fadd_rn(g.x, gs[s].x); g.y = __fadd_rn(g.y, gs[s].y); g.z = __fadd_rn(g.z, gs[s].z); g.w = __fadd_rn(g.w, gs[s].w);
      u.x = __fadd_rn(u.x, us[s].x); u.y = __fadd_rn(u.y, us[s].y); u.z = __fadd_rn(u.z, us[s].z); u.w = __fadd_rn(u.w, us[s].w);
    }
  for (int s = SMAX; s < S; ++s) {
    const float4 g2 = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol));
    const float4 u2 = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol + 64));
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

__device__ __forceinline__ void swiglu4(const float* __restrict__ part, const PartSpec& ps, int T, int F, size_t e,
                                        uint16_t* __restrict__ out) {
  const size_t stride = (size_t)T * 2 * F;
  const int t = (int)e / F;  // T * 2F < 2^31 (launchers check)
  const int j = (int)e % F;
  const int col = (j / 64) * 128 + (j % 64);  // gate column; up = col + 64 (same 128-feature tile)
  const int S = part_count(ps, col);
  const size_t gcol = (size_t)t * 2 * F + (size_t)col;
  // the first 4 slots' loads are issued together (predicated); adds in slot order
  float4 gs[4], us[4];
#pragma unroll
  for (int s = 0; s < 4; ++s)
    if (s < S) {
      gs[s] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol));
      us[s] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol + 64));
    }
  float4 g = gs[0], u = us[0];
#pragma unroll
  for (int s = 1; s < 4; ++s)
    if (s < S) {
      g.x = __fadd_rn(g.x, gs[s].x); g.y = __fadd_rn(g.y, gs[s].y); g.z = __fadd_rn(g.z, gs[s].z); g.w = __fadd_rn(g.w, gs[s].w);
      u.x = __fadd_rn(u.x, us[s].x); u.y = __fadd_rn(u.y, us[s].y); u.z = __fadd_rn(u.z, us[s].z); u.w = __fadd_rn(u.w, us[s].w);
    }
  for (int s = 4; s < S; ++s) {
    const float4 g2 = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol));
    const float4 u2 = __ldcg(reinterpret_cast<const float4*>(part + (size_t)s * stride + gcol + 64));
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

// ---- QKV epilogue for the rotate-half pair (i, i + hd/2) of head h of token t
// (heads 0..H-1 = q, H..H+KV-1 = k, then v): bias, RoPE on q and k, bf16, and
// q written or k/v appended at column pos[t] of the cache.
// prep() gathers what does not depend on the QKV GEMM (PDL pre-wait part).
struct QkvArgs {
  const uint16_t* bias;  // nullable
  const int32_t* pos;
  int T, H, KV, hd;
  int part_T;            // rows of the partial buffer (slot stride); 0 = T
  const float* rcos;
  const float* rsin;
  uint16_t* q;
  CacheView cache;
  int32_t paged;
  const int32_t* slot;
  uint16_t* kd;  // dense k/v [T][KV*hd] when !paged
  uint16_t* vd;
};
struct QkvPair {
  float ba, bb, c, sn;
  uint16_t* dst;
  int f1, f2;
  size_t row;
};
__device__ __forceinline__ QkvPair qkv_prep(const QkvArgs& a, int t, int h, int i) {
  QkvPair r;
  const int h2 = a.hd / 2;
  const int NQKV = (a.H + 2 * a.KV) * a.hd;
  r.f1 = h * a.hd + i;
  r.f2 = r.f1 + h2;
  r.row = (size_t)t * NQKV;
  const int p = a.pos[t];
  r.ba = r.bb = 0.f;
  r.c = 1.f;
  r.sn = 0.f;
  if (a.bias) {
    r.ba = bf2f(a.bias[r.f1]);
    r.bb = bf2f(a.bias[r.f2]);
  }
  if (h < a.H + a.KV) {
    r.c = a.rcos[(size_t)p * h2 + i];
    r.sn = a.rsin[(size_t)p * h2 + i];
  }
  if (h < a.H) {
    r.dst = a.q + (size_t)t * a.H * a.hd + h * a.hd;
  } else {
    const int kvsel = h < a.H + a.KV ? 0 : 1;
    const int kh = h - a.H - kvsel * a.KV;
    if (a.paged && a.slot[t] < 0) {
      r.dst = nullptr;  // a no-op entry of a padded verifier chunk: nothing to append
    } else {
      r.dst = a.paged ? cache_ptr(a.cache, a.slot[t], p, kvsel, kh)  // tentative append of column p
                      : (kvsel ? a.vd : a.kd) + (size_t)t * a.KV * a.hd + kh * a.hd;
    }
  }
  return r;
}
__device__ __forceinline__ void qkv_finish(const QkvArgs& a, const QkvPair& r, const float* part, const PartSpec& ps,
                                           int h, int i) {
  if (!r.dst) return;
  const size_t stride = (size_t)(a.part_T ? a.part_T : a.T) * (a.H + 2 * a.KV) * a.hd;
  float x = sum_splits(part, part_count(ps, r.f1), stride, r.row + r.f1);
  float y = sum_splits(part, part_count(ps, r.f2), stride, r.row + r.f2);
  if (a.bias) {
    x = __fadd_rn(x, r.ba);
    y = __fadd_rn(y, r.bb);
  }
  uint16_t oa, ob;
  if (h < a.H + a.KV) {  // RoPE on q and k
    oa = f2bf(__fsub_rn(__fmul_rn(x, r.c), __fmul_rn(y, r.sn)));
    ob = f2bf(__fadd_rn(__fmul_rn(y, r.c), __fmul_rn(x, r.sn)));
  } else {
    oa = f2bf(x);
    ob = f2bf(y);
  }
  r.dst[i] = oa;
  r.dst[i + a.hd / 2] = ob;
}

}  // namespace mg
