// attention.cu -- paged GQA decode attention.
//
// k_attn_chunk<HD, NB>: one CTA (4 warps) per (token, kv head, key chunk of
// 64*NB keys).  The G = H/KV query heads sharing the kv head form the 16-row
// M side of mma.sync.m16n8k16 tiles (rows >= G are zero), so every K/V byte
// of the chunk is read from HBM once per token.  Keys come in 16-key blocks
// (a block never crosses a KV page); warp w owns blocks w, w+4, ...  At kernel
// start every warp issues ALL its K and V rows as 256-byte cp.async.bulk
// copies (one mbarrier for K, one for V; rows padded to HD*2+16 bytes so the
// ldmatrix reads are bank-conflict free), so one HBM round trip per CTA is
// exposed and the V stream overlaps the score phase.  The chunk follows
// DESIGN.md 3.3 exactly, in two passes:
//   pass 1  s_j = (q . k_j) * fp32(1/sqrt(hd))  (bf16 x bf16 products, fp32 acc)
//   softmax m = max_j s_j, e_j = expf(s_j - m), l = sum_j e_j (fixed trees)
//   pass 2  acc = sum_j e_j v_j  with e split as bf16 hi + bf16 lo (16+ bit
//           mantissa) so the probabilities are not rounded to bf16
// then the 4 warps' partial sums are added in warp order.
// k_attn_combine: chunks combined in chunk order with weights
// expf(m_c - m*), o = bf16(acc / l).
//
// Schedules: the fast path uses 64-key chunks (most CTAs, best at every batch
// size measured); the verifier uses pinned 128-key chunks (A14), so
// a query's result depends only on its own keys: the block/warp structure is
// a function of the chunk bounds alone.
#include "common.cuh"
#include "kernels.h"

namespace mg {

constexpr int kAtThreads = 128;

template <int HD, int NB>
struct AtCfg {
  static constexpr int ROWB = HD * 2 + 16;
  static constexpr int BLKB = 16 * ROWB;
  static constexpr int CH = 64 * NB;                  // keys per chunk
  static constexpr int S_BYTES = 16 * CH * 4;
  static constexpr int KV_BYTES = 2 * 4 * NB * BLKB;  // [K|V][warp][NB] blocks
  static constexpr int X_BYTES = 4 * 16 * HD * 4;     // cross-warp sums, aliases the K/V region
  static_assert(X_BYTES <= KV_BYTES, "reduction scratch must fit in the K/V region");
  static constexpr int SMEM = S_BYTES + KV_BYTES + 4 * 16 * 4 + 32 * 4 + 8 * 8;
};

MG_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
MG_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
MG_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
MG_DEV void mma_bf16(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int HD, int NB>
__global__ void __launch_bounds__(kAtThreads) k_attn_chunk(AttnArgs a) {
  using C = AtCfg<HD, NB>;
  extern __shared__ __align__(16) uint8_t sm[];
  float* S = reinterpret_cast<float*>(sm);                                // [16][CH]
  uint8_t* kvr = sm + C::S_BYTES;                                         // K/V blocks
  float* red = reinterpret_cast<float*>(sm + C::S_BYTES + C::KV_BYTES);  // [4][16]
  float* s_ml = red + 4 * 16;                                             // m[16], l[16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_ml + 32);                // [K 4][V 4]

  const int t = blockIdx.x, kvh = blockIdx.y, c = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.H, G = a.H / a.KV;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  griddep();
  const int n = a.n_keys[t];
  const int lo = c * C::CH;
  const size_t po = ((size_t)t * H + (size_t)kvh * G) * a.n_chunks + c;
  if (lo >= n) {
    if (threadIdx.x < G) {
      a.part_ml[(po + (size_t)threadIdx.x * a.n_chunks) * 2 + 0] = -INFINITY;
      a.part_ml[(po + (size_t)threadIdx.x * a.n_chunks) * 2 + 1] = 0.f;
    }
    return;
  }
  const int hi = min(n, lo + C::CH);
  const int len = hi - lo;
  const int nblk = (len + 15) >> 4;
  const int nbw = nblk > warp ? min(NB, (nblk - warp + 3) >> 2) : 0;  // blocks of this warp

  // ---- issue every K and V row of this warp's blocks (one round trip)
  {
    const int slot = a.paged ? a.slot[t] : 0;
    auto krow = [&](int j, int kvsel) -> const uint16_t* {
      if (a.paged) {
        const CacheView& cv = a.cache;
        const int page = cv.pt[(size_t)slot * cv.max_pages + j / cv.page_size];
        return cv.pool + ((((size_t)cv.layer * cv.n_pages + page) * 2 + kvsel) * cv.kv + kvh) *
                             (size_t)cv.page_size * HD +
               (size_t)(j % cv.page_size) * HD;
      }
      const uint16_t* base = kvsel ? a.Vd : a.Kd;
      return base + (((size_t)t * a.KV + kvh) * a.key_stride + j) * HD;
    };
    int valid_rows = 0;
    for (int j = 0; j < nbw; ++j) valid_rows += min(16, hi - (lo + 16 * (warp + 4 * j)));
    if (lane == 0) {
      mbar_expect_tx(&bars[warp], (uint32_t)valid_rows * HD * 2);
      mbar_expect_tx(&bars[4 + warp], (uint32_t)valid_rows * HD * 2);
    }
    __syncwarp();
    for (int e = lane; e < nbw * 32; e += 32) {
      const int j = e >> 5, kvsel = (e >> 4) & 1, r = e & 15;
      const int key = lo + 16 * (warp + 4 * j) + r;
      uint8_t* dst = kvr + ((size_t)(kvsel * 4 + warp) * NB + j) * C::BLKB + r * C::ROWB;
      if (key < hi) {
        bulk_g2s(dst, krow(key, kvsel), HD * 2, &bars[kvsel * 4 + warp]);
      } else {
        for (int q = 0; q < HD / 8; ++q) reinterpret_cast<uint4*>(dst)[q] = make_uint4(0, 0, 0, 0);
      }
    }
  }

  // ---- Q fragments (A operand, rows = query heads of this kv head, zero-padded)
  const int r0 = lane >> 2, r1 = r0 + 8, cc = 2 * (lane & 3);
  const uint16_t* qp = a.q + (size_t)t * H * HD + (size_t)kvh * G * HD;
  uint32_t qf[HD / 16][4];
#pragma unroll
  for (int ks = 0; ks < HD / 16; ++ks) {
    const int k0 = ks * 16 + cc;
    qf[ks][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(qp + r0 * HD + k0) : 0u;
    qf[ks][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(qp + r1 * HD + k0) : 0u;
    qf[ks][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(qp + r0 * HD + k0 + 8) : 0u;
    qf[ks][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(qp + r1 * HD + k0 + 8) : 0u;
  }
  const float scale = (float)(1.0 / sqrt((double)HD));

  // ---- pass 1: scores
  __syncwarp();
  mbar_wait(&bars[warp], 0);
  for (int j = 0; j < nbw; ++j) {
    const uint32_t kb = smem_u32(kvr + ((size_t)warp * NB + j) * C::BLKB);
    const int b = warp + 4 * j;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kg = 0; kg < HD / 32; ++kg) {
        uint32_t b0, b1, b2, b3;
        const int mi = lane >> 3, rr = lane & 7;
        ldsm_x4(kb + (8 * nt + rr) * C::ROWB + (32 * kg + 8 * mi) * 2, b0, b1, b2, b3);
        mma_bf16(sacc, qf[2 * kg], b0, b1);
        mma_bf16(sacc, qf[2 * kg + 1], b2, b3);
      }
      const int j0 = 16 * b + 8 * nt + cc;  // key index within the chunk
      const bool v0 = lo + j0 < hi, v1 = lo + j0 + 1 < hi;
      S[r0 * C::CH + j0] = v0 ? __fmul_rn(sacc[0], scale) : -INFINITY;
      S[r0 * C::CH + j0 + 1] = v1 ? __fmul_rn(sacc[1], scale) : -INFINITY;
      S[r1 * C::CH + j0] = v0 ? __fmul_rn(sacc[2], scale) : -INFINITY;
      S[r1 * C::CH + j0 + 1] = v1 ? __fmul_rn(sacc[3], scale) : -INFINITY;
    }
  }
  __syncthreads();

  // ---- softmax over the chunk: query head g is owned by warp g % 4, lane l
  // takes keys l, l+32, ... (fixed trees, no CTA-wide barrier per head)
  for (int g = warp; g < G; g += 4) {
    float* sg = S + g * C::CH;
    float m = -INFINITY;
    for (int j = lane; j < len; j += 32) m = fmaxf(m, sg[j]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float l = 0.f;
    for (int j = lane; j < C::CH; j += 32) {
      const float e = j < len ? expf(__fsub_rn(sg[j], m)) : 0.f;
      sg[j] = e;
      l = __fadd_rn(l, e);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l = __fadd_rn(l, __shfl_xor_sync(0xffffffffu, l, off));
    if (lane == 0) {
      s_ml[g] = m;
      s_ml[16 + g] = l;
    }
  }
  __syncthreads();

  // ---- pass 2: acc = sum_j e_j v_j  (e = hi + lo, two bf16 MMAs).  Warp w owns
  // head dims [w*HD/4, (w+1)*HD/4) and sums ALL the chunk's key blocks in order,
  // so no cross-warp reduction is needed.
  constexpr int NT = HD / 32;  // 8-dim n-tiles per warp
  float acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
  for (int w = 0; w < 4; ++w) mbar_wait(&bars[4 + w], 0);  // every warp's V rows landed
  const int d0 = warp * (HD / 4);
  for (int b = 0; b < nblk; ++b) {
    const uint32_t vb = smem_u32(kvr + ((size_t)(4 + (b & 3)) * NB + (b >> 2)) * C::BLKB);
    const int j0 = 16 * b;
    uint32_t ph[4], pl[4];
    {
      const float* s0 = S + r0 * C::CH + j0 + cc;
      const float* s1 = S + r1 * C::CH + j0 + cc;
      const bool g0 = r0 < G, g1 = r1 < G;  // rows >= G are padding: P = 0
      const float e[8] = {g0 ? s0[0] : 0.f, g0 ? s0[1] : 0.f, g1 ? s1[0] : 0.f, g1 ? s1[1] : 0.f,
                          g0 ? s0[8] : 0.f, g0 ? s0[9] : 0.f, g1 ? s1[8] : 0.f, g1 ? s1[9] : 0.f};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t h = pack_bf2(e[2 * q], e[2 * q + 1]);
        ph[q] = h;
        pl[q] = pack_bf2(__fsub_rn(e[2 * q], lo_bf(h)), __fsub_rn(e[2 * q + 1], hi_bf(h)));
      }
    }
#pragma unroll
    for (int n2 = 0; n2 < NT / 2; ++n2) {
      uint32_t b0, b1, b2, b3;
      const int mi = lane >> 3, rr = lane & 7;
      ldsm_x4_t(vb + ((mi & 1) * 8 + rr) * C::ROWB + (d0 + 16 * n2 + 8 * (mi >> 1)) * 2, b0, b1, b2, b3);
      mma_bf16(acc[2 * n2], ph, b0, b1);
      mma_bf16(acc[2 * n2], pl, b0, b1);
      mma_bf16(acc[2 * n2 + 1], ph, b2, b3);
      mma_bf16(acc[2 * n2 + 1], pl, b2, b3);
    }
  }
  // ---- write the chunk partials (rows < G)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int d = d0 + 8 * nt + cc;
    if (r0 < G) {
      float* o = a.part_acc + (po + (size_t)r0 * a.n_chunks) * HD + d;
      *reinterpret_cast<float2*>(o) = make_float2(acc[nt][0], acc[nt][1]);
    }
    if (r1 < G) {
      float* o = a.part_acc + (po + (size_t)r1 * a.n_chunks) * HD + d;
      *reinterpret_cast<float2*>(o) = make_float2(acc[nt][2], acc[nt][3]);
    }
  }
  if (threadIdx.x < G) {
    const size_t o = po + (size_t)threadIdx.x * a.n_chunks;
    a.part_ml[o * 2 + 0] = s_ml[threadIdx.x];
    a.part_ml[o * 2 + 1] = s_ml[16 + threadIdx.x];
  }
}

// grid (T, H), block hd
__global__ void k_attn_combine(const float* __restrict__ part_acc, const float* __restrict__ part_ml,
                               const int32_t* __restrict__ n_keys, int H, int hd, int chunk, int n_chunks,
                               uint16_t* __restrict__ out) {
  griddep();
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

template <int HD, int NB>
static cudaError_t launch_attn_t(const AttnArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_chunk<HD, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AtCfg<HD, NB>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_k(k_attn_chunk<HD, NB>, dim3(a.T, a.KV, a.n_chunks), dim3(kAtThreads), AtCfg<HD, NB>::SMEM, st, a);
}

int attn_max_chunk() { return 256; }

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t st) {
  if (a.H / a.KV > 16 || a.H % a.KV) return cudaErrorInvalidValue;
  cudaError_t e;
  if (a.hd == 128) {
    if (a.chunk == 64) e = launch_attn_t<128, 1>(a, st);
    else if (a.chunk == 128) e = launch_attn_t<128, 2>(a, st);
    else if (a.chunk == 256) e = launch_attn_t<128, 4>(a, st);
    else return cudaErrorInvalidValue;
  } else if (a.hd == 64) {
    if (a.chunk == 64) e = launch_attn_t<64, 1>(a, st);
    else if (a.chunk == 128) e = launch_attn_t<64, 2>(a, st);
    else if (a.chunk == 256) e = launch_attn_t<64, 4>(a, st);
    else return cudaErrorInvalidValue;
  } else {
    return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return launch_k(k_attn_combine, dim3(a.T, a.H), dim3(a.hd), 0, st, (const float*)a.part_acc,
                  (const float*)a.part_ml, a.n_keys, a.H, a.hd, a.chunk, a.n_chunks, a.out);
}

}  // namespace mg
