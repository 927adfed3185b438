// chain.cu -- persistent layer chain: up to four weight-streaming GEMM phases
// and their epilogues in ONE kernel (SURVEY 8(a) rows a3, a5, a6, a7 with the
// a2 norms).  Per decode layer the engine runs
//     [O-proj -> residual+RMSNorm -> gate/up -> SwiGLU -> down -> residual+RMSNorm
//      -> next layer's QKV -> bias/RoPE/append]  then attention,
// instead of eight separate kernels.  Measured motivation (scripts/rdsize.cu,
// scripts/timeline.py): every kernel boundary drains the HBM weight stream
// for ~3-5 us; here the weights of the next phase keep streaming while the
// current phase's epilogue runs.
//
// Roles (one CTA per SM, 16 warps):
//   warp 0   A producer: TMA of the weight boxes of EVERY phase, in phase
//            order, gated only by free ring slots (weights never depend on
//            the activations, so the ring is refilled across phase changes);
//   warp 6   B producer: TMA of the activation tiles; phase p waits for the
//            grid barrier "op p-1 done" (phase 0: griddepcontrol.wait);
//   warp 1   tcgen05.mma issue (lane 0), as in k_gemm_tc;
//   warps 2-5 epilogue: TMEM -> fp32 partials of each piece; after the last
//            piece of phase p: grid barrier "partials of p written", then the
//            op of phase p, then grid barrier "op p done";
//   warps 7-11 op helpers: join warps 2-5 for every phase op (288 threads per
//            CTA: the ops are L2-latency bound and need the parallelism).
// Grid barriers are monotone counters (never reset): each launch reads the
// epoch E, barrier k completes at (E+1) * gridDim.x arrivals, and CTA 0 bumps
// E once every CTA has passed the last barrier.  All CTAs are co-resident
// (grid = #SMs, 1 CTA/SM) and the dependent kernel is released only at the
// very end, so a barrier can never wait on a CTA that cannot be scheduled.
// A barrier that does not complete within 2 s sets *err and releases (the
// step is reported as failed instead of hanging the GPU).
//
// Arithmetic is the same as the separate kernels' except the RMSNorm tree
// (128 threads per row: thread i sums vectors i, i+128, ... in order, xor
// tree in the warp, 4 warp partials in order) -- fixed per row, so the
// verifier stays batch invariant.
#include "chain.h"
#include "common.cuh"
#include "epilogue.cuh"
#include "gemm_tc.cuh"
#include "kernels.h"

namespace mg {

#ifndef MG_CHAIN_WARPS
#define MG_CHAIN_WARPS 12
#endif
constexpr int kChainThreads = 32 * MG_CHAIN_WARPS;
constexpr int kOpThreads = kChainThreads - 96;  // warps 2-5 and 7.. (the epilogue warps + the op helpers)

MG_DEV uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// wait until *p reaches target (wrap-safe); false (and *err = 1) after 2 s
MG_DEV bool wait_count(const uint32_t* p, uint32_t target, int32_t* err) {
  if ((int32_t)(ld_acquire(p) - target) >= 0) return true;
  const uint64_t t0 = globaltimer();
  while ((int32_t)(ld_acquire(p) - target) < 0) {
    __nanosleep(40);
    if (globaltimer() - t0 > 2000000000ull) {
      atomicExch(err, 1);
      return false;
    }
  }
  return true;
}
MG_DEV void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
MG_DEV void op_bar() { asm volatile("bar.sync 2, %0;" ::"n"(kOpThreads) : "memory"); }

template <int TN>
struct ChainCfg {
  using G = GemmTcCfg<TN>;
  static constexpr int NS = G::NS;
  // 1 KB alignment slack, the ring, then fullA/fullB/empty[NS], tfull/tempty[2], tmem slot, norm scratch
  static constexpr int SMEM_FIXED = 1024 + NS * G::STAGE + (3 * NS + 4) * 8 + 192;  // + 8 B per token
};

// ---- phase ops, run by the 288 op threads of every CTA (otid 0..287).  They
// are L2-latency bound; one output group per thread per round, all its slot
// loads issued together.
// The op-side fields of a phase, copied out of the kernel parameters into
// registers once per op (a dynamically indexed __grid_constant__ access is an
// indexed constant load -- measured as the top stall of the op loops).
struct OpDesc {
  float* part;
  int N, K, G, op;
  uint16_t* x;
  const uint16_t* w;
  uint16_t* xn;
  float eps;
  uint16_t* a;
  QkvArgs qkv;
};
MG_DEV OpDesc op_desc(const ChainPhase& ph) {
  OpDesc d;
  d.part = ph.part; d.N = ph.N; d.K = ph.K; d.G = ph.G; d.op = ph.op;
  d.x = ph.x; d.w = ph.w; d.xn = ph.xn; d.eps = ph.eps; d.a = ph.a; d.qkv = ph.qkv;
  return d;
}

// 8 consecutive partial sums, slots added in k order, 4 slots' loads in flight
MG_DEV void sum8_slots4(const float* __restrict__ part, int S, size_t stride, size_t idx, float* a) {
  for (int s0 = 0; s0 < S; s0 += 4) {
    float4 lo[4], hi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (s0 + u < S) {
        lo[u] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)(s0 + u) * stride + idx));
        hi[u] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)(s0 + u) * stride + idx + 4));
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (s0 + u < S) {
        const float v[8] = {lo[u].x, lo[u].y, lo[u].z, lo[u].w, hi[u].x, hi[u].y, hi[u].z, hi[u].w};
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = (s0 + u == 0) ? v[k] : __fadd_rn(a[k], v[k]);
      }
  }
}

MG_DEV void op_resnorm(const OpDesc& ph, int T, const PartSpec& ps, int otid, float* red, float* s_inv) {
  const int d = ph.N, nv = d / 8;
  const size_t stride = (size_t)T * d;
  const uint4* wv = reinterpret_cast<const uint4*>(ph.w);
  for (int r = blockIdx.x; r < T; r += gridDim.x) {
    uint4* xv = reinterpret_cast<uint4*>(ph.x + (size_t)r * d);
    float ss = 0.f;
    for (int i = otid; i < nv; i += kOpThreads) {
      float acc[8];
      const uint4 x0 = __ldcg(xv + i);
      sum8_slots4(ph.part, part_count(ps, i * 8), stride, (size_t)r * d + (size_t)i * 8, acc);
      const uint4 h = residual8(x0, acc);
      xv[i] = h;
      ss = ss8(h, ss);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, off));
    if ((otid & 31) == 0) red[otid >> 5] = ss;
    op_bar();
    if (otid == 0) {
      float s = red[0];
      for (int w = 1; w < kOpThreads / 32; ++w) s = __fadd_rn(s, red[w]);
      *s_inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(s, (float)d), ph.eps)));
    }
    op_bar();
    const float inv = *s_inv;
    uint4* ov = reinterpret_cast<uint4*>(ph.xn + (size_t)r * d);
    for (int i = otid; i < nv; i += kOpThreads) ov[i] = norm8(__ldcg(xv + i), __ldg(wv + i), inv);
    op_bar();  // red / s_inv reused by the next row
  }
}

MG_DEV void op_swiglu(const OpDesc& ph, int T, const PartSpec& ps, int otid) {
  const int F = ph.N / 2;
  const int n4 = T * F / 4;
  const int gs = gridDim.x * kOpThreads;
  for (int e4 = blockIdx.x * kOpThreads + otid; e4 < n4; e4 += gs) swiglu4(ph.part, ps, T, F, (size_t)e4 * 4, ph.a);
}

// tok_pos / tok_page: the tokens' positions and the KV page of that position,
// staged in shared memory at kernel start
MG_DEV void op_qkv(const OpDesc& ph, int T, const PartSpec& ps, int otid, const int* tok_pos,
                   const int* tok_page) {
  const QkvArgs& q = ph.qkv;
  const int h2 = q.hd / 2, nh = q.H + 2 * q.KV;
  const int n = T * nh * h2;
  for (int w = blockIdx.x * kOpThreads + otid; w < n; w += gridDim.x * kOpThreads) {
    const int t = w / (nh * h2), rem = w % (nh * h2);
    const int h = rem / h2, i = rem % h2;
    const QkvPair r = qkv_prep_staged(q, t, h, i, tok_pos[t], tok_page[t]);
    qkv_finish(q, r, ph.part, ps, h, i);
  }
}

MG_DEV void run_op(const OpDesc& ph, int T, int otid, float* red, float* s_inv, const int* tok_pos,
                   const int* tok_page) {
  const PartSpec ps{1, ph.G, ph.K / 64, ph.N / 128};
  if (ph.op == CH_RESNORM) op_resnorm(ph, T, ps, otid, red, s_inv);
  else if (ph.op == CH_SWIGLU) op_swiglu(ph, T, ps, otid);
  else if (ph.op == CH_QKV) op_qkv(ph, T, ps, otid, tok_pos, tok_page);
  __threadfence();
  fence_proxy_async_global();  // the next phase reads these outputs with TMA
}

template <int TN, bool MMA16>
__global__ void __launch_bounds__(kChainThreads, 1) k_chain(const __grid_constant__ ChainArgs a) {
  using C = GemmTcCfg<TN>;
  constexpr int KS = C::KS, NS = C::NS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + NS * C::A_BYTES;
  uint64_t* fullA = (uint64_t*)(smem + NS * C::STAGE);  // barriers after the ring
  uint64_t* fullB = fullA + NS;
  uint64_t* empty = fullB + NS;
  uint64_t* tfull = empty + NS;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  float* red = (float*)(tmem_slot + 2);  // [kOpThreads / 32] op-warp partials
  float* s_inv = red + 32;
  uint32_t* s_epoch = (uint32_t*)(s_inv + 1);
  int* tok_pos = (int*)(s_epoch + 4);  // [T] staged token positions (QKV ops), then [T] their KV pages
  int* tok_page = tok_pos + a.T;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.T;
  const int n_t = (T + TN - 1) / TN;
  uint32_t* epoch = a.sync + 2 * kChainMax;

  if (threadIdx.x == 0) {
    for (int p = 0; p < a.n_ph; ++p) tma_prefetch_desc(&a.ph[p].mw);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&fullA[i], 1);
      mbar_init(&fullB[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);  // one arrival per epilogue warp
    }
    fence_mbar_init();
    *s_epoch = *(volatile uint32_t*)epoch;
  }
  if (warp == 2) tc_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // per-token position and KV page of the QKV ops (written by earlier kernels)
  int qkv_ph = -1;
  for (int p = 0; p < a.n_ph; ++p)
    if (a.ph[p].op == CH_QKV) qkv_ph = p;
  if (qkv_ph >= 0 && threadIdx.x >= 224) {  // the op-helper warps
    const QkvArgs& q = a.ph[qkv_ph].qkv;
    for (int t = threadIdx.x - 224; t < a.T; t += kChainThreads - 224) {
      const int p = q.pos[t];
      tok_pos[t] = p;
      tok_page[t] = q.paged ? q.cache.pt[(size_t)q.slot[t] * q.cache.max_pages + p / q.cache.page_size] : 0;
    }
  }
  __syncthreads();
  const uint32_t tmem = *tmem_slot;
  const uint32_t target = (*s_epoch + 1u) * gridDim.x;
  // diagnostics: [0] entry, then per phase [first stage landed, last MMA, partials out,
  // barrier 1 passed, op done, (B producer) barrier 2 passed]
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * kChainTraceWords : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();

  Piece pc;
  if (warp == 0) {
    // ---- A producer: the weights of all phases, back to back (gated only by
    // free ring slots: the next phase's weights stream during this phase's op)
    const uint64_t pol = policy_evict_first();
    int it = 0;
    for (int p = 0; p < a.n_ph; ++p) {
      const ChainPhase& ph = a.ph[p];
      const int KB = ph.K / C::BK;
      PieceIter pi(KB, ph.N / 128, n_t, ph.G);
      while (pi.next(pc)) {
        for (int kb = pc.kb0; kb < pc.kb1; kb += KS, ++it) {
          const int st = it % NS;
          const int nk = min(KS, pc.kb1 - kb);
          mbar_spin(&empty[st], ((uint32_t)(it / NS) & 1u) ^ 1u);
          if (lane == 0) {
            mbar_expect_tx(&fullA[st], (uint32_t)nk * C::A_BOX);
            for (int i = 0; i < nk; ++i)
              tma_load_4d_hint(sA + st * C::A_BYTES + i * C::A_BOX, &ph.mw, &fullA[st], 0, 0, kb + i, pc.mt, pol);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 6) {
    // ---- B producer: activations, once the previous phase's op is done everywhere
    int it = 0;
    for (int p = 0; p < a.n_ph; ++p) {
      const ChainPhase& ph = a.ph[p];
      if (p == 0) {
        griddep_wait();
      } else if (lane == 0) {
        wait_count(&a.sync[2 * (p - 1) + 1], target, a.err);
        if (tr) tr[1 + (p - 1) * 6 + 5] = globaltimer();
      }
      __syncwarp();
      fence_proxy_async_global();
      const int KB = ph.K / C::BK;
      PieceIter pi(KB, ph.N / 128, n_t, ph.G);
      while (pi.next(pc)) {
        for (int kb = pc.kb0; kb < pc.kb1; kb += KS, ++it) {
          const int st = it % NS;
          const int nk = min(KS, pc.kb1 - kb);
          mbar_spin(&empty[st], ((uint32_t)(it / NS) & 1u) ^ 1u);
          if (lane == 0) {
            mbar_expect_tx(&fullB[st], (uint32_t)nk * C::B_BOX);
            for (int i = 0; i < nk; ++i)
              tma_load_2d(sB + st * C::B_BYTES + i * C::B_BOX, &ph.mx, &fullB[st], (kb + i) * C::BK, pc.tt * TN);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA));
    const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sB));
    int it = 0, j = 0;
    for (int p = 0; p < a.n_ph; ++p) {
      const ChainPhase& ph = a.ph[p];
      const int KB = ph.K / C::BK;
      PieceIter pi(KB, ph.N / 128, n_t, ph.G);
      bool pi_started = false;
      for (; pi.next(pc); ++j) {
        const int buf = j & 1;
        mbar_spin(&tempty[buf], ((uint32_t)(j >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(buf * C::ACC_COLS);
        for (int kb = pc.kb0; kb < pc.kb1; kb += KS, ++it) {
          const int st = it % NS;
          const uint32_t ph_ = (uint32_t)(it / NS) & 1u;
          mbar_spin(&fullA[st], ph_);
          mbar_spin(&fullB[st], ph_);
          tc_fence_after();
          if (tr && lane == 0 && kb == pc.kb0 && !pi_started) tr[1 + p * 6 + 0] = globaltimer();
          pi_started = true;
          if (lane == 0) {
            const uint64_t a_st = a_desc0 + (uint64_t)((st * C::A_BYTES) >> 4);
            const uint64_t b_st = b_desc0 + (uint64_t)((st * C::B_BYTES) >> 4);
            issue_stage<TN, MMA16>(a_st, b_st, min(KS, pc.kb1 - kb), dacc, kb == pc.kb0);
            tc_commit(&empty[st]);
          }
          __syncwarp();
        }
        if (lane == 0) tc_commit(&tfull[buf]);
        __syncwarp();
      }
      if (tr && lane == 0) tr[1 + p * 6 + 1] = globaltimer();
    }
  } else if (warp >= 2 && warp <= 5) {
    // ---- epilogue warps 2..5: partials, grid barrier, phase op, grid barrier
    griddep_wait();
    const int q = warp & 3;
    const int ltid = threadIdx.x - 64;
    int j = 0;
    for (int p = 0; p < a.n_ph; ++p) {
      const ChainPhase& ph = a.ph[p];
      const int KB = ph.K / C::BK;
      PieceIter pi(KB, ph.N / 128, n_t, ph.G);
      for (; pi.next(pc); ++j) {
        const int buf = j & 1;
        if (warp == 2 && lane == 0) mbar_wait(&tfull[buf], (uint32_t)(j >> 1) & 1u);
        epi_bar();
        tc_fence_after();
        const int n = pc.mt * C::BM + q * 32 + lane;
        const int N = ph.N;
        float* o = ph.part + (size_t)pc.slot * (size_t)T * (size_t)N;
        const int t0 = pc.tt * TN;
#pragma unroll 1
        for (int c0 = 0; c0 < TN; c0 += 16) {
          if (t0 + c0 >= T) break;
          uint32_t r[16];
          tc_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * C::ACC_COLS + c0), r);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int t = t0 + c0 + i;
            if (t < T) o[(size_t)t * N + n] = __uint_as_float(r[i]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      }
      // all of this CTA's partials of phase p are written
      __threadfence();
      epi_bar();
      if (ltid == 0) {
        if (tr) tr[1 + p * 6 + 2] = globaltimer();
        atomicAdd(&a.sync[2 * p], 1u);
        wait_count(&a.sync[2 * p], target, a.err);
        if (tr) tr[1 + p * 6 + 3] = globaltimer();
        if (p == a.n_ph - 1 && blockIdx.x == 0) atomicAdd(epoch, 1u);  // every CTA is past its epoch read
      }
      op_bar();  // releases the op helpers
      run_op(op_desc(ph), T, ltid, red, s_inv, tok_pos, tok_page);
      op_bar();
      if (ltid == 0) {
        if (tr) tr[1 + p * 6 + 4] = globaltimer();
        atomicAdd(&a.sync[2 * p + 1], 1u);
      }
    }
    // keep every counter of this epoch in step: arrive on the unused ones
    if (ltid == 0)
      for (int k = 2 * a.n_ph; k < 2 * kChainMax; ++k) atomicAdd(&a.sync[k], 1u);
  } else if (warp >= 7) {  // warps 7 .. MG_CHAIN_WARPS-1
    // ---- op helpers: one op per phase, between the epilogue's two op_bar()s
    const int otid = 128 + threadIdx.x - 224;
    for (int p = 0; p < a.n_ph; ++p) {
      op_bar();
      run_op(op_desc(a.ph[p]), T, otid, red, s_inv, tok_pos, tok_page);
      op_bar();
    }
  }
  tc_fence_before();
  __syncthreads();
  griddep_launch();
  if (warp == 2) {
    tc_fence_after();
    tc_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int TN, bool MMA16>
static cudaError_t launch_chain_t(const ChainArgs& a, cudaStream_t st) {
  using CC = ChainCfg<TN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_chain<TN, MMA16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const size_t smem = CC::SMEM_FIXED + (size_t)a.T * 8;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  return launch_k(k_chain<TN, MMA16>, dim3(chain_grid()), dim3(kChainThreads), smem, st, a);
}

template <int TN>
static cudaError_t launch_chain_m(const ChainArgs& a, int mma_n, cudaStream_t st) {
  if (mma_n == 16 && TN > 16) return launch_chain_t<TN, true>(a, st);
  return launch_chain_t<TN, false>(a, st);
}

int chain_grid() { return num_sms(); }

cudaError_t launch_chain(const ChainArgs& a, int tile_n, int mma_n, cudaStream_t st) {
  if (a.n_ph < 1 || a.n_ph > kChainMax || a.T < 1 || !a.sync || !a.err) return cudaErrorInvalidValue;
  for (int p = 0; p < a.n_ph; ++p) {
    const ChainPhase& ph = a.ph[p];
    if (ph.N % 128 || ph.K % 64 || ph.G < 1 || !ph.part) return cudaErrorInvalidValue;
    if (ph.op == CH_RESNORM && (!ph.x || !ph.w || !ph.xn))
      return cudaErrorInvalidValue;
    if (ph.op == CH_SWIGLU && (ph.N % 128 || !ph.a)) return cudaErrorInvalidValue;
    if (ph.op == CH_QKV && ph.qkv.T != a.T) return cudaErrorInvalidValue;
  }
  switch (tile_n) {
    case 16: return launch_chain_m<16>(a, mma_n, st);
    case 32: return launch_chain_m<32>(a, mma_n, st);
    case 64: return launch_chain_m<64>(a, mma_n, st);
    case 128: return launch_chain_m<128>(a, mma_n, st);
    case 256: return launch_chain_m<256>(a, mma_n, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mg
