// attention.cu -- paged GQA decode attention.
//
// k_attn<HD, R>: one CTA (4 warps) per (token, kv head, key split).  The
// G = H/KV query heads sharing the kv head form the 16-row M side of
// mma.sync.m16n8k16 tiles (rows >= G are don't-care: an MMA output row depends
// only on its own A row), so every K/V byte is read from HBM once per token.
//
// Arithmetic = the streamed form of DESIGN.md 3.3 (oracle or_attention with
// chunk = -split_keys): the split's 16-key blocks are dealt round-robin to the
// 4 warps (block b -> warp b mod 4; a block never crosses a KV page).  Each
// warp streams its blocks with a running (m, l, acc) per query head:
//   s_j = (q . k_j) * fp32(1/sqrt(hd))              QK^T on the tensor cores
//   m' = max(m, max_j s_j), alpha = expf(m - m'),   row max by quad shuffles
//   e_j = expf(s_j - m'), l = l*alpha + sum_j e_j, acc = acc*alpha + sum_j e_j v_j
// with e_j fed to the PV MMA as bf16 hi + bf16 lo (16+ bit mantissa) straight
// from the score registers (the m16n8 C layout of two key tiles IS the m16k16
// A layout), so scores and probabilities never touch shared memory.  The 4
// warps are then combined in warp order with weights expf(m_w - max m); a
// token with one split writes o = bf16(acc / l); otherwise each split writes
// (acc, m, l) and the LAST CTA of the (token, kv head) to arrive (atomic
// counter, reset by it) combines the splits in split order.  Every choice is
// a function of (n_keys, split_keys) alone, so with a pinned split_keys (the
// verifier) a query's result does not depend on the batch.
//
// Data movement: TMA only.  Each warp owns a ring of RK K blocks and one of RV
// V blocks (box 64 dims x 16 keys, 128B swizzle -> conflict-free ldmatrix);
// its lane 0 refills a K stage right after QK^T has read it and a V stage
// right after PV; warp 0 loads the Q tile once.  On the fast path (prewait) the first blocks, which hold
// only keys of earlier steps, are requested before griddepcontrol.wait, so
// their latency overlaps the tail of the QKV epilogue.  Page-table lookups for 32 blocks at a time are done by the
// 32 lanes in parallel and shuffled to lane 0 at issue time.
#include <cstdlib>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace mg {


// Per warp: a ring of RK K blocks and a separate ring of RV V blocks, each
// with its own mbarriers, so the K block of step i + RK is requested as soon as
// QK^T of step i has read its stage (it streams while softmax and PV run) and
// the V block of step i + RV as soon as PV of step i is done.
template <int HD, int RK, int RV, int NW = 4>
struct AtCfg {
  static constexpr int HALVES = HD / 64;
  static constexpr int BLK = HALVES * 2048;        // one 16-row tile: HALVES x [16][128 B] swizzled
  static constexpr int WRING = (RK + RV) * BLK;    // one warp's K ring then V ring
  static constexpr int XST = HD + 8;               // cross-warp scratch row stride (floats)
  static constexpr int RING = NW * WRING;
  static constexpr int XG = NW * 16 * XST * 4;     // [warp][16][XST] fp32, aliases the rings
  static constexpr int Q_OFF = 0;
  static constexpr int RING_OFF = BLK;
  static constexpr int ML_OFF = RING_OFF + (RING > XG ? RING : XG);  // m, l: [warp][16] each
  static constexpr int KVN_OFF = ML_OFF + 2 * 64 * 4;                // fused QKV: new K and V rows [2][HD] bf16
  static constexpr int NBAR = 1 + NW * (RK + RV);                    // Q, then [warp][RK K | RV V]
  static constexpr int BAR_OFF = KVN_OFF + 2 * HD * 2;
  static constexpr int SMEM = BAR_OFF + NBAR * 8 + 8 + 1024;         // + flag + alignment slack
};

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
// byte offset of the 16-byte chunk holding (row r, column col) of a TMA tile
// stored as HD/64 halves of [16 rows][128 B] with the 128B swizzle
MG_DEV uint32_t swz(int r, int col) {
  return (uint32_t)((col >> 6) * 2048 + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) << 4));
}
// hi/lo bf16 pair of two fp32 probabilities: hi = bf16(e), lo = bf16(e - hi)
MG_DEV void split_pair(float e0, float e1, uint32_t& hi, uint32_t& lo) {
  hi = pack_bf2(e0, e1);
  lo = pack_bf2(__fsub_rn(e0, lo_bf(hi)), __fsub_rn(e1, hi_bf(hi)));
}

template <int HD, int RK, int RV, int NW>
__global__ void __launch_bounds__(NW * 32, 16 / NW) k_attn(const __grid_constant__ AttnArgs a) {
  using C = AtCfg<HD, RK, RV, NW>;
  constexpr int kAtThreads = NW * 32;  // NW streams (warps) per CTA
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  float* s_m = reinterpret_cast<float*>(sm + C::ML_OFF);  // [warp][16]
  float* s_l = s_m + 64;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  int* s_flag = reinterpret_cast<int*>(bars + C::NBAR);

  const int t = blockIdx.x, kvh = blockIdx.y, sp = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.H, G = a.H / a.KV;
  // token group: the second one (t >= T1) is the verifier's in a mixed launch
  const bool g1 = a.T1 > 0 && t >= a.T1;
  const CacheView& cview = g1 ? a.cache1 : a.cache;
  const CUtensorMap* kmp = g1 ? &a.kvmap1 : &a.kmap;
  const CUtensorMap* vmp = g1 ? &a.kvmap1 : &a.vmap;
  const int split_keys = g1 ? a.split_keys1 : a.split_keys;
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NBAR; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (!a.prewait) griddep();
  const int n = a.n_keys[t];
  const int lo = sp * split_keys;
  if (lo >= n) return;
  const int hi = min(n, lo + split_keys);
  const int nblk = (hi - lo + 15) >> 4;
  const int nbw = nblk > warp ? (nblk - warp + NW - 1) / NW : 0;  // blocks of this warp
  const int n_sp = (n + split_keys - 1) / split_keys;
  uint8_t* kring = sm + C::RING_OFF + warp * C::WRING;
  uint8_t* vring = kring + RK * C::BLK;
  uint64_t* kfull = bars + 1 + warp * (RK + RV);
  uint64_t* vfull = kfull + RK;

  // ---- TMA issue: Q tile (warp 0), then the first RK K / RV V blocks of each warp.
  // Lane j caches the page coordinates of block (32*batch + j); the K and V
  // streams advance at different times and keep one cache each.
  int k_sl = 0, k_row = 0, v_sl = 0, v_row = 0;
  auto coords = [&](int base, int& o_sl, int& o_row) {
    const int i = base + lane;
    if (i < nbw) {
      const int key0 = lo + 16 * (warp + NW * i);
      if (a.paged) {
        const CacheView& cv = cview;
        const int page = cv.pt[(size_t)a.slot[t] * cv.max_pages + key0 / cv.page_size];
        o_sl = (cv.layer * cv.n_pages + page) * 2 * a.KV + kvh;
        o_row = key0 % cv.page_size;
      } else {
        o_sl = t * a.KV + kvh;
        o_row = key0;
      }
    }
  };
  const int vsl = a.paged ? a.KV : 0;  // V slab offset inside the pool map
  auto issue_k = [&](int i) {          // warp-wide (shuffles); lane 0 issues
    const int sl = __shfl_sync(0xffffffffu, k_sl, i & 31), row = __shfl_sync(0xffffffffu, k_row, i & 31);
    if (lane == 0) {
      const int s = i % RK;
      mbar_expect_tx(&kfull[s], C::BLK);
#pragma unroll
      for (int h = 0; h < C::HALVES; ++h)
        tma_load_3d(kring + s * C::BLK + h * 2048, kmp, &kfull[s], 64 * h, row, sl);
    }
  };
  auto issue_v = [&](int i) {
    const int sl = __shfl_sync(0xffffffffu, v_sl, i & 31), row = __shfl_sync(0xffffffffu, v_row, i & 31);
    if (lane == 0) {
      const int s = i % RV;
      mbar_expect_tx(&vfull[s], C::BLK);
#pragma unroll
      for (int h = 0; h < C::HALVES; ++h)
        tma_load_3d(vring + s * C::BLK + h * 2048, vmp, &vfull[s], 64 * h, row, sl + vsl);
    }
  };
  coords(0, k_sl, k_row);
  v_sl = k_sl;
  v_row = k_row;
  int ik = 0, iv = 0;  // blocks issued per stream
  uint16_t* kvn = reinterpret_cast<uint16_t*>(sm + C::KVN_OFF);
  const bool has_new = a.fuse_qkv && sp == n_sp - 1;  // this CTA holds key n - 1

  // fused QKV epilogue (the same arithmetic as k_epi_qkv): q rows
  // of the G heads into the swizzled Q tile; the new K/V column (RoPE on K) into
  // kvn and appended to the cache at position p = n - 1.  Items
  // (one rotation pair each) are taken QI per thread per round; everything that
  // does not depend on the QKV GEMM (position, bias, RoPE factors, the cache
  // address) is loaded first -- on the fast path before griddepcontrol.wait --
  // and the partial-slot loads of all QI items are issued together after it,
  // so a round costs one L2 round trip instead of one per item and operand.
  constexpr int h2 = HD / 2, QI = RK + RV > 2 ? 2 : 3;  // 2 keeps the deeper-ring variants spill-free
  struct QItem {
    int f1, g, i;  // feature of the pair's first half; q head in group (isq) or 0 = K, 1 = V; pair index
    bool isq, live;
    float ba, bb, c, sn;
    uint16_t* dst;
  };
  const int nq = G * h2, nitems = (a.fuse_qkv && !(a.dbg & 1)) ? nq + (has_new ? 2 * h2 : 0) : 0;
  int p = 0;
  QItem qi[QI];
  auto prep = [&](int base) {
#pragma unroll
    for (int j = 0; j < QI; ++j) {
      QItem& it = qi[j];
      const int w = base + j * kAtThreads + threadIdx.x;
      it.live = w < nitems;
      if (!it.live) continue;
      it.isq = w < nq;
      it.g = it.isq ? w / h2 : (w - nq) / h2;
      it.i = (it.isq ? w : w - nq) % h2;
      const int h = it.isq ? kvh * G + it.g : H + it.g * a.KV + kvh;
      it.f1 = h * HD + it.i;
      it.ba = a.bias ? bf2f(a.bias[it.f1]) : 0.f;
      it.bb = a.bias ? bf2f(a.bias[it.f1 + h2]) : 0.f;
      if (it.isq || it.g == 0) {
        it.c = a.rcos[(size_t)p * h2 + it.i];
        it.sn = a.rsin[(size_t)p * h2 + it.i];
      }
      it.dst = it.isq ? nullptr : cache_ptr(cview, a.slot[t], p, it.g, kvh);
    }
  };
  if (nitems) p = a.pos[t];
  if (a.prewait) {
    // PDL: blocks whose keys all precede this step's appended column (n - 1)
    // were written by earlier steps -- fetched before griddepcontrol.wait
    auto early = [&](int i) { return lo + 16 * (warp + NW * i) + 16 <= n - 1; };
    for (; ik < RK && ik < nbw && early(ik); ++ik) issue_k(ik);
    for (; iv < RV && iv < nbw && early(iv); ++iv) issue_v(iv);
    if (nitems) prep(0);
    griddep();
  } else if (nitems) {
    prep(0);
  }
  for (; ik < RK && ik < nbw; ++ik) issue_k(ik);  // the remaining first blocks (after the wait)
  for (; iv < RV && iv < nbw; ++iv) issue_v(iv);
  if (!a.fuse_qkv) {
    if (warp == 0 && lane == 0) {
      mbar_expect_tx(&bars[0], C::BLK);
#pragma unroll
      for (int h = 0; h < C::HALVES; ++h)
        tma_load_3d(sm + C::Q_OFF + h * 2048, &a.qmap, &bars[0], 64 * h, kvh * G, t + a.q_row0);
    }
  } else {
    const int NQKV = (H + 2 * a.KV) * HD;
    const size_t stride = (size_t)(a.part_T ? a.part_T : a.T) * NQKV, row = (size_t)t * NQKV;
    for (int base = 0; base < nitems; base += QI * kAtThreads) {
      if (base) prep(base);
      // all slot loads of the round first (<= 8 per operand, predicated), then
      // the sums in slot (= k) order -- sum_splits' arithmetic
      float vx[QI][8], vy[QI][8];
      int S[QI];
#pragma unroll
      for (int j = 0; j < QI; ++j) {
        S[j] = qi[j].live ? part_count(a.qkv_ps, qi[j].f1) : 0;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          vx[j][s] = s < S[j] ? __ldcg(a.qkv_part + (size_t)s * stride + row + qi[j].f1) : 0.f;
          vy[j][s] = s < S[j] ? __ldcg(a.qkv_part + (size_t)s * stride + row + qi[j].f1 + h2) : 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < QI; ++j) {
        const QItem& it = qi[j];
        if (!it.live) continue;
        float x = vx[j][0], y = vy[j][0];
#pragma unroll
        for (int s = 1; s < 8; ++s)
          if (s < S[j]) {
            x = __fadd_rn(x, vx[j][s]);
            y = __fadd_rn(y, vy[j][s]);
          }
        for (int s = 8; s < S[j]; ++s) {
          x = __fadd_rn(x, __ldcg(a.qkv_part + (size_t)s * stride + row + it.f1));
          y = __fadd_rn(y, __ldcg(a.qkv_part + (size_t)s * stride + row + it.f1 + h2));
        }
        if (a.bias) {
          x = __fadd_rn(x, it.ba);
          y = __fadd_rn(y, it.bb);
        }
        uint16_t oa, ob;
        if (it.isq || it.g == 0) {  // RoPE on q and k
          oa = f2bf(__fsub_rn(__fmul_rn(x, it.c), __fmul_rn(y, it.sn)));
          ob = f2bf(__fadd_rn(__fmul_rn(y, it.c), __fmul_rn(x, it.sn)));
        } else {
          oa = f2bf(x);
          ob = f2bf(y);
        }
        const int i = it.i;
        if (it.isq) {
          uint8_t* qt = sm + C::Q_OFF;
          *reinterpret_cast<uint16_t*>(qt + swz(it.g, i) + (i & 7) * 2) = oa;
          *reinterpret_cast<uint16_t*>(qt + swz(it.g, i + h2) + ((i + h2) & 7) * 2) = ob;
        } else {
          kvn[it.g * HD + i] = oa;
          kvn[it.g * HD + i + h2] = ob;
          it.dst[i] = oa;
          it.dst[i + h2] = ob;
        }
      }
    }
    __syncthreads();
  }

  const int rr = lane & 7, mi = lane >> 3;
  const int r0 = lane >> 2, r1 = r0 + 8, cc = 2 * (lane & 3);
  // ---- Q tile (A operand; rows >= G are other heads / zero fill, ignored).
  // Its fragments are re-read from shared memory per block (ldmatrix) rather
  // than held in registers, which keeps the kernel at 4 CTAs per SM.
  if (!a.fuse_qkv) mbar_wait(&bars[0], 0);
  const uint32_t qa = smem_u32(sm + C::Q_OFF);
  const float scale = (float)(1.0 / sqrt((double)HD));

  // ---- stream this warp's blocks
  constexpr int NT = HD / 8;  // 8-dim n-tiles of the output
  float acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows r0, r1 (l: this lane's keys)
  for (int i = 0; i < nbw; ++i) {
    uint8_t* kst = kring + (i % RK) * C::BLK;
    uint8_t* vst = vring + (i % RV) * C::BLK;
    const uint32_t kb = smem_u32(kst), vb = smem_u32(vst);
    const int valid = min(16, hi - (lo + 16 * (warp + NW * i)));
    const bool new_blk = has_new && lo + 16 * (warp + NW * i) + 16 >= n;  // holds key n - 1
    const int rr_new = n - 1 - (lo + 16 * (warp + NW * i));
    mbar_wait(&kfull[i % RK], (uint32_t)((i / RK) & 1));
    if (a.dbg & 2) {  // microbenchmark: stream only
      __syncwarp();
      if (i + RK < nbw) {
        if (((i + RK) & 31) == 0) coords(i + RK, k_sl, k_row);
        issue_k(i + RK);
      }
      mbar_wait(&vfull[i % RV], (uint32_t)((i / RV) & 1));
      __syncwarp();
      if (i + RV < nbw) {
        if (((i + RV) & 31) == 0) coords(i + RV, v_sl, v_row);
        issue_v(i + RV);
      }
      continue;
    }
    if (new_blk) {  // patch the new K row
      for (int e = lane; e < HD / 8; e += 32)
        *reinterpret_cast<uint4*>(kst + swz(rr_new, e * 8)) = *reinterpret_cast<const uint4*>(kvn + e * 8);
      __syncwarp();
    }
    // scores: two 8-key tiles
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kg = 0; kg < HD / 32; ++kg) {
      uint32_t q0[4], q1[4];
      ldsm_x4(qa + swz((mi & 1) * 8 + rr, 32 * kg + 8 * (mi >> 1)), q0[0], q0[1], q0[2], q0[3]);
      ldsm_x4(qa + swz((mi & 1) * 8 + rr, 32 * kg + 16 + 8 * (mi >> 1)), q1[0], q1[1], q1[2], q1[3]);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kb + swz(8 * nt + rr, 32 * kg + 8 * mi), b0, b1, b2, b3);
        mma_bf16(sc[nt], q0, b0, b1);
        mma_bf16(sc[nt], q1, b2, b3);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        sc[nt][q] = 8 * nt + cc + (q & 1) < valid ? __fmul_rn(sc[nt][q], scale) : -INFINITY;
    float b0m = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
    float b1m = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
    b0m = fmaxf(b0m, __shfl_xor_sync(0xffffffffu, b0m, 1));
    b1m = fmaxf(b1m, __shfl_xor_sync(0xffffffffu, b1m, 1));
    b0m = fmaxf(b0m, __shfl_xor_sync(0xffffffffu, b0m, 2));
    b1m = fmaxf(b1m, __shfl_xor_sync(0xffffffffu, b1m, 2));
    const float n0 = fmaxf(m0, b0m), n1 = fmaxf(m1, b1m);
    const float al0 = expf(__fsub_rn(m0, n0)), al1 = expf(__fsub_rn(m1, n1));
    m0 = n0;
    m1 = n1;
    float e[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      e[nt][0] = expf(__fsub_rn(sc[nt][0], n0));
      e[nt][1] = expf(__fsub_rn(sc[nt][1], n0));
      e[nt][2] = expf(__fsub_rn(sc[nt][2], n1));
      e[nt][3] = expf(__fsub_rn(sc[nt][3], n1));
    }
    l0 = __fadd_rn(__fmul_rn(l0, al0), __fadd_rn(__fadd_rn(e[0][0], e[0][1]), __fadd_rn(e[1][0], e[1][1])));
    l1 = __fadd_rn(__fmul_rn(l1, al1), __fadd_rn(__fadd_rn(e[0][2], e[0][3]), __fadd_rn(e[1][2], e[1][3])));
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      acc[nt][0] = __fmul_rn(acc[nt][0], al0);
      acc[nt][1] = __fmul_rn(acc[nt][1], al0);
      acc[nt][2] = __fmul_rn(acc[nt][2], al1);
      acc[nt][3] = __fmul_rn(acc[nt][3], al1);
    }
    // the K stage is consumed: stream the K block RK steps ahead during softmax + PV
    if (i + RK < nbw) {
      __syncwarp();
      fence_proxy_async();
      if (((i + RK) & 31) == 0) coords(i + RK, k_sl, k_row);
      issue_k(i + RK);
    }
    mbar_wait(&vfull[i % RV], (uint32_t)((i / RV) & 1));
    if (valid < 16) {  // the split's last block: zero V rows past the end (P is 0 there)
      for (int e = lane; e < (16 - valid) * C::HALVES * 8; e += 32) {
        const int row = valid + e / (C::HALVES * 8), rem = e % (C::HALVES * 8);
        reinterpret_cast<uint4*>(vst + (rem >> 3) * 2048 + row * 128)[rem & 7] = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
    }
    if (new_blk) {  // patch the new V row
      for (int e = lane; e < HD / 8; e += 32)
        *reinterpret_cast<uint4*>(vst + swz(rr_new, e * 8)) = *reinterpret_cast<const uint4*>(kvn + HD + e * 8);
      __syncwarp();
    }
    uint32_t ph[4], pl[4];
    split_pair(e[0][0], e[0][1], ph[0], pl[0]);  // row r0, keys cc, cc+1
    split_pair(e[0][2], e[0][3], ph[1], pl[1]);  // row r1, keys cc, cc+1
    split_pair(e[1][0], e[1][1], ph[2], pl[2]);  // row r0, keys 8+cc
    split_pair(e[1][2], e[1][3], ph[3], pl[3]);  // row r1, keys 8+cc
#pragma unroll
    for (int n2 = 0; n2 < NT / 2; ++n2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(vb + swz((mi & 1) * 8 + rr, 16 * n2 + 8 * (mi >> 1)), b0, b1, b2, b3);
      mma_bf16(acc[2 * n2], ph, b0, b1);
      mma_bf16(acc[2 * n2], pl, b0, b1);
      mma_bf16(acc[2 * n2 + 1], ph, b2, b3);
      mma_bf16(acc[2 * n2 + 1], pl, b2, b3);
    }
    if (i + RV < nbw) {  // refill the V stage just consumed
      __syncwarp();
      fence_proxy_async();
      if (((i + RV) & 31) == 0) coords(i + RV, v_sl, v_row);
      issue_v(i + RV);
    }
  }
  // lane partial sums -> row sums (fixed butterfly, the same in all 4 lanes)
  l0 = __fadd_rn(l0, __shfl_xor_sync(0xffffffffu, l0, 1));
  l1 = __fadd_rn(l1, __shfl_xor_sync(0xffffffffu, l1, 1));
  l0 = __fadd_rn(l0, __shfl_xor_sync(0xffffffffu, l0, 2));
  l1 = __fadd_rn(l1, __shfl_xor_sync(0xffffffffu, l1, 2));

  // ---- combine the 4 warps (streams) in warp order
  if (a.dbg & 4) return;
  __syncthreads();  // every ring consumed: the scratch may alias them
  float* X = reinterpret_cast<float*>(sm + C::RING_OFF);
  if ((lane & 3) == 0) {
    s_m[warp * 16 + r0] = m0;
    s_m[warp * 16 + r1] = m1;
    s_l[warp * 16 + r0] = l0;
    s_l[warp * 16 + r1] = l1;
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int d = 8 * nt + cc;
    if (r0 < G) *reinterpret_cast<float2*>(X + (warp * 16 + r0) * C::XST + d) = make_float2(acc[nt][0], acc[nt][1]);
    if (r1 < G) *reinterpret_cast<float2*>(X + (warp * 16 + r1) * C::XST + d) = make_float2(acc[nt][2], acc[nt][3]);
  }
  __syncthreads();
  const size_t obase = ((size_t)t * H + (size_t)kvh * G) * HD;
  const size_t pbase = ((size_t)t * H + (size_t)kvh * G) * a.n_splits + sp;  // + g * n_splits
  for (int e = threadIdx.x; e < G * HD; e += kAtThreads) {
    const int g = e / HD, d = e % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w * 16 + g]);
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float wt = expf(__fsub_rn(s_m[w * 16 + g], M));
      L = __fadd_rn(L, __fmul_rn(s_l[w * 16 + g], wt));
      A = __fadd_rn(A, __fmul_rn(X[(w * 16 + g) * C::XST + d], wt));
    }
    if (n_sp == 1) {
      a.out[obase + (size_t)g * HD + d] = f2bf(__fdiv_rn(A, L));
    } else {
      const size_t p = pbase + (size_t)g * a.n_splits;
      a.part_acc[p * HD + d] = A;
      if (d == 0) {
        a.part_ml[p * 2 + 0] = M;
        a.part_ml[p * 2 + 1] = L;
      }
    }
  }
  if (n_sp == 1) return;

  // ---- several splits: the last CTA to arrive combines them in split order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* cnt = a.counter + (size_t)t * a.KV + kvh;
    const int last = atomicAdd(cnt, 1) == n_sp - 1;
    if (last) *cnt = 0;
    *s_flag = last;
  }
  __syncthreads();
  if (!*s_flag) return;
  __threadfence();
  for (int e = threadIdx.x; e < G * HD; e += kAtThreads) {
    const int g = e / HD, d = e % HD;
    const size_t base = ((size_t)t * H + (size_t)kvh * G + g) * a.n_splits;
    float M = -INFINITY;
    for (int k = 0; k < n_sp; ++k) M = fmaxf(M, __ldcg(a.part_ml + (base + k) * 2));
    float L = 0.f;
    for (int k = 0; k < n_sp; ++k)
      L = __fadd_rn(L, __fmul_rn(__ldcg(a.part_ml + (base + k) * 2 + 1),
                                 expf(__fsub_rn(__ldcg(a.part_ml + (base + k) * 2), M))));
    float A = 0.f;
    for (int k = 0; k < n_sp; ++k)
      A = __fadd_rn(A, __fmul_rn(__ldcg(a.part_acc + (base + k) * HD + d),
                                 expf(__fsub_rn(__ldcg(a.part_ml + (base + k) * 2), M))));
    a.out[obase + (size_t)g * HD + d] = f2bf(__fdiv_rn(A, L));
  }
}

template <int HD, int RK, int RV, int NW = 4>
static cudaError_t launch_attn_t(const AttnArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn<HD, RK, RV, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AtCfg<HD, RK, RV, NW>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_k(k_attn<HD, RK, RV, NW>, dim3(a.T, a.KV, a.n_splits), dim3(NW * 32), AtCfg<HD, RK, RV, NW>::SMEM,
                  st, a);
}

// ring depths (RK, RV): (4, 4) when the grid has at most one CTA per SM (small
// batches and the verifier's few rows: a warp's blocks are in flight together;
// 1% faster steps at B = 1 / 8, profiles/r02_ab_attn_deep_ring.txt), (2, 2)
// while it fits ~3 CTAs per SM, else (1, 1) (4 CTAs per SM, 40 KB each at hd
// 128).  (2, 1) -- the K stream two blocks ahead at 55 KB per CTA, still 4 per
// SM -- measured the same step time at B = 64 / 8 (llama8b, ctx 384: 4.34 vs
// 4.33 ms, 3.48 vs 3.49 ms), so the smaller footprint stays the default.
// MG_ATTN_RING=11|21|22|44|66 forces a ring, MG_ATTN_DEEP=0|44|66 sets the
// small-grid one (measurement only).  Ring depth changes timing only.
static int g_attn_ring = 0, g_attn_deep = 44, g_attn_nw2 = 1;

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t st) {
  if (a.H % a.KV || a.H / a.KV > 16 || !a.counter || a.split_keys < 64 || a.split_keys % 64 || a.n_splits < 1)
    return cudaErrorInvalidValue;
  if (a.T1 > 0 && a.T1 < a.T && (a.split_keys1 < 64 || a.split_keys1 % 64)) return cudaErrorInvalidValue;
  if (a.streams != 0 && a.streams != 2 && a.streams != 4) return cudaErrorInvalidValue;
  if (!g_attn_ring) {
    const char* s = getenv("MG_ATTN_RING");
    const int v = s ? atoi(s) : 0;
    g_attn_ring = (v == 11 || v == 21 || v == 22 || v == 44 || v == 66) ? v : -1;
    const char* d = getenv("MG_ATTN_DEEP");  // ring of grids with <= one CTA per SM (44 / 66; 0 = the 22 rule)
    if (d) g_attn_deep = atoi(d);
    const char* n2 = getenv("MG_ATTN_NW2");  // 0: always 4 streams (measurement)
    if (n2) g_attn_nw2 = atoi(n2);
  }
  const long ctas = (long)a.T * a.KV * a.n_splits;
  const int R = g_attn_ring > 0 ? g_attn_ring
                                : (ctas <= num_sms() && g_attn_deep ? g_attn_deep : (ctas <= 3L * num_sms() ? 22 : 11));
  // The fast path (one token group, batch-shaped arithmetic anyway) with more
  // CTAs than one wave of 4-warp CTAs holds runs 2-warp CTAs (2 key streams, 8
  // CTAs per SM), which keeps it in one wave: 1-1.5% faster steps at B = 96 /
  // 128 (profiles/r02_ab_attn_two_streams.txt).  The verifier (pinned
  // arithmetic, A14) and mixed launches always take 4 streams.
  if (a.streams == 2 || (a.streams == 0 && g_attn_nw2 && a.prewait && (a.T1 == 0 || a.T1 >= a.T) &&
                         ctas > 4L * num_sms() && g_attn_ring <= 0)) {
    if (a.hd == 128) return launch_attn_t<128, 1, 1, 2>(a, st);
    if (a.hd == 64) return launch_attn_t<64, 1, 1, 2>(a, st);
  }
  if (a.hd == 128) {
    switch (R) {
      case 66: return launch_attn_t<128, 6, 6>(a, st);
      case 44: return launch_attn_t<128, 4, 4>(a, st);
      case 22: return launch_attn_t<128, 2, 2>(a, st);
      case 21: return launch_attn_t<128, 2, 1>(a, st);
      default: return launch_attn_t<128, 1, 1>(a, st);
    }
  }
  if (a.hd == 64) {
    switch (R) {
      case 66: return launch_attn_t<64, 6, 6>(a, st);
      case 44: return launch_attn_t<64, 4, 4>(a, st);
      case 22: return launch_attn_t<64, 2, 2>(a, st);
      case 21: return launch_attn_t<64, 2, 1>(a, st);
      default: return launch_attn_t<64, 1, 1>(a, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace mg
