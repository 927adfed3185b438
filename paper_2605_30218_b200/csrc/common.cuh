// common.cuh -- device helpers shared by the sm_100a kernels of libmargingate.
// bf16 is carried as uint16_t bit patterns; conversions use the hardware
// round-to-nearest-even cvt.  PTX wrappers for mbarrier,
// TMA (cp.async.bulk.tensor) and tcgen05 (alloc / mma / commit / ld).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define MG_DEV __device__ __forceinline__

namespace mg {

MG_DEV float bf2f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }
MG_DEV uint16_t f2bf(float f) {
  __nv_bfloat16 b = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&b);
}
MG_DEV float lo_bf(uint32_t w) { return __uint_as_float(w << 16); }
MG_DEV float hi_bf(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
MG_DEV uint32_t pack_bf2(float lo, float hi) { return (uint32_t)f2bf(lo) | ((uint32_t)f2bf(hi) << 16); }

// contiguous equal chunks, remainder to the leading chunks
__host__ __device__ __forceinline__ int chunk_start(int n, int S, int c) {
  int base = n / S, rem = n % S;
  return c * base + (c < rem ? c : rem);
}

MG_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
MG_DEV uint64_t globaltimer() {  // ns, comparable across SMs (diagnostics only)
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ split-K partial layout
// Stream-K partition of W = n_m * KB k-blocks over G virtual CTAs: CTA i owns
// [floor(i W / G), floor((i+1) W / G)).  owner(w) = CTA that owns k-block w.
__host__ __device__ __forceinline__ int streamk_owner(long long w, long long W, int G) {
  return (int)(((w + 1) * G - 1) / W);
}
// How many fp32 partial slots hold output feature n (slot p = k order):
// uniform split-K (G == 0): S; stream-K: pieces of n's 128-feature tile.
struct PartSpec {
  int S;   // uniform splits (G == 0)
  int G;   // stream-K virtual CTAs (0 = uniform)
  int KB;  // 64-wide k-blocks per tile
  int n_m; // 128-feature tiles
};
__host__ __device__ __forceinline__ int part_count(const PartSpec& p, int n) {
  if (p.G == 0) return p.S;
  const long long W = (long long)p.n_m * p.KB;
  const int m = n / 128;
  if (W * (p.G + 1) < 2147483647LL) {  // the same formula in 32-bit arithmetic (hot in the epilogues)
    const int w0 = m * p.KB, w1 = (m + 1) * p.KB - 1, Wi = (int)W;
    return ((w1 + 1) * p.G - 1) / Wi - ((w0 + 1) * p.G - 1) / Wi + 1;
  }
  return streamk_owner((long long)(m + 1) * p.KB - 1, W, p.G) - streamk_owner((long long)m * p.KB, W, p.G) + 1;
}

// ------------------------------------------------------------------ top-2
// top-1/top-2 under the total order (value desc, id asc): exact, so any merge
// order gives the same (v1, i1, v2, i2) (A6)
struct Top2 {
  float v1;
  int i1;
  float v2;
  int i2;
};

MG_DEV bool better(float a, int ia, float b, int ib) { return a > b || (a == b && ia < ib); }

MG_DEV void t2_push(Top2& t, float v, int i) {
  if (better(v, i, t.v1, t.i1)) {
    t.v2 = t.v1;
    t.i2 = t.i1;
    t.v1 = v;
    t.i1 = i;
  } else if (better(v, i, t.v2, t.i2)) {
    t.v2 = v;
    t.i2 = i;
  }
}
// merge two top-2 sets over disjoint index ranges
MG_DEV Top2 t2_merge(const Top2& a, const Top2& b) {
  Top2 r;
  if (better(a.v1, a.i1, b.v1, b.i1)) {
    r.v1 = a.v1; r.i1 = a.i1;
    if (better(a.v2, a.i2, b.v1, b.i1)) { r.v2 = a.v2; r.i2 = a.i2; } else { r.v2 = b.v1; r.i2 = b.i1; }
  } else {
    r.v1 = b.v1; r.i1 = b.i1;
    if (better(a.v1, a.i1, b.v2, b.i2)) { r.v2 = a.v1; r.i2 = a.i1; } else { r.v2 = b.v2; r.i2 = b.i2; }
  }
  return r;
}
MG_DEV Top2 t2_shfl(const Top2& t, int off) {
  Top2 o;
  o.v1 = __shfl_xor_sync(0xffffffffu, t.v1, off);
  o.i1 = __shfl_xor_sync(0xffffffffu, t.i1, off);
  o.v2 = __shfl_xor_sync(0xffffffffu, t.v2, off);
  o.i2 = __shfl_xor_sync(0xffffffffu, t.i2, off);
  return o;
}

// ------------------------------------------------------------------ PDL
// Programmatic dependent launch: every kernel waits for its prerequisite
// grid before touching data it produced, then lets the next grid launch
// (trigger only AFTER the wait, so at most one dependent grid is resident
// early).  Both are no-ops when the kernel was launched without PDL.
MG_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
MG_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
MG_DEV void griddep() {
  griddep_wait();
  griddep_launch();
}

// ------------------------------------------------------------------ mbarrier
MG_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
MG_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
MG_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// order this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) writes to the same buffer
MG_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// the same for global memory: generic-proxy stores before later TMA reads
MG_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
MG_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
MG_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// pure spin on test_wait (no suspension): for the single-thread TMA producer
// and MMA issuer, whose hand-off latency bounds the weight stream
MG_DEV void mbar_spin(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "SPIN_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra SPIN_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------ TMA
MG_DEV void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
MG_DEV void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
MG_DEV void tma_load_2d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
MG_DEV void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// bulk L2 prefetch of a contiguous global range (size a multiple of 16 B)
MG_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
MG_DEV void tma_load_4d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3,
                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
      : "memory");
}
MG_DEV void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
MG_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 16-byte global store with an L2 cache-policy hint
MG_DEV void st_v4_hint(float* dst, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
MG_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------------ tcgen05
MG_DEV void tc_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
MG_DEV void tc_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
MG_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
MG_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate)
MG_DEV void tc_mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on an mbarrier once all previously issued tcgen05 ops completed
MG_DEV void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
MG_DEV void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32b, 16 consecutive columns -> 16 regs per thread
MG_DEV void tc_ld_32x32b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, rows of
// 64 bf16 (128 B), 8-row core groups 1024 B apart (SBO), version 1 (sm_100).
MG_DEV uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;  // SBO
  d |= (uint64_t)1u << 46;            // descriptor version
  d |= (uint64_t)2u << 61;            // SWIZZLE_128B
  return d;
}
// instruction descriptor: D fp32, A/B bf16, both K-major, shape M x N
__host__ __device__ __forceinline__ uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace mg
