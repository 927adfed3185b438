// membw.cu -- HBM read-bandwidth microbenchmark on B200 (diagnostic only).
//   (1) LDG.128 streaming read with k loads in flight per thread
//   (2) TMA 2-D box streaming (one producer thread per CTA, NS stages of 16 KB)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membw scripts/membw.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void rd_ldg(const uint4* __restrict__ p, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (; i < n; i += stride) {
    uint4 v = __ldg(p + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS>
__global__ void __launch_bounds__(128, 1) rd_tma(const __grid_constant__ CUtensorMap m, int tiles_per_cta, int n_tiles,
                                                 uint4* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(buf + NS * 16384);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int t0 = blockIdx.x * tiles_per_cta;
  uint32_t acc = 0;
  for (int i = 0; i < tiles_per_cta + NS; ++i) {
    if (i >= NS) {  // consume tile i-NS
      int st = (i - NS) % NS;
      uint32_t ph = ((i - NS) / NS) & 1;
      asm volatile(
          "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
              s32(&full[st])),
          "r"(ph));
      acc ^= *(volatile uint32_t*)(buf + st * 16384);
    }
    if (i < tiles_per_cta) {
      int st = i % NS;
      int tile = (t0 + i) % n_tiles;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(s32(&full[st])));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              s32(buf + st * 16384)),
          "l"((uint64_t)&m), "r"(s32(&full[st])), "r"(0), "r"(tile * 128));
    }
  }
  if (acc == 0x12345678) sink[0].x = acc;
}

int main() {
  size_t bytes = (size_t)4 << 30;
  void* p;
  cudaMalloc(&p, bytes);
  cudaMemset(p, 1, bytes);
  uint4* sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int bpsm : {2, 4, 8, 16}) {
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(a);
      rd_ldg<<<148 * bpsm, 512>>>((const uint4*)p, bytes / 16, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("LDG.128 blocks/SM %2d x512 thr: %.0f GB/s\n", bpsm, bytes / ms / 1e6);
  }
  // TMA: tensor [rows][64] bf16 (128 B rows), box 64 x 128 rows = 16 KB contiguous
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t rows = bytes / 128;
  cuuint64_t dims[2] = {64, rows};
  cuuint64_t str[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int n_tiles = (int)(bytes / 16384);
  auto run = [&](auto kern, int ns, int ctas_per_sm) {
    int grid = 148 * ctas_per_sm;
    int tpc = n_tiles / grid;
    size_t smem = ns * 16384 + 1024 + 8 * ns;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(a);
      kern<<<grid, 128, smem>>>(m, tpc, n_tiles, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    cudaError_t e = cudaGetLastError();
    printf("TMA NS=%2d ctas/SM=%d: %.0f GB/s %s\n", ns, ctas_per_sm, (double)tpc * grid * 16384 / ms / 1e6,
           e ? cudaGetErrorString(e) : "");
  };
  run(rd_tma<4>, 4, 1);
  run(rd_tma<8>, 8, 1);
  run(rd_tma<12>, 12, 1);
  run(rd_tma<4>, 4, 2);
  run(rd_tma<6>, 6, 2);
  run(rd_tma<4>, 4, 3);
  return 0;
}
