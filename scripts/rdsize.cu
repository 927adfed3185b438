// rdsize.cu -- per-launch cost of a plain streaming read vs buffer size (diagnostic only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ab/rdsize scripts/rdsize.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void __launch_bounds__(512) rd(const uint4* __restrict__ p, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (; i < n; i += stride) {
    uint4 v = __ldcs(p + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

int main() {
  const size_t total = (size_t)4 << 30;
  uint8_t* buf;
  uint4* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 1, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double sizes_mb[] = {8, 16, 33.5, 50.3, 117.4, 234.9, 1050.0};
  for (double mb : sizes_mb) {
    const size_t bytes = ((size_t)(mb * 1e6) + 255) & ~(size_t)255;
    const int nbuf = (int)(total / bytes) < 20 ? (int)(total / bytes) : 20;
    for (int blocks : {148 * 2, 148 * 4}) {
      float best = 1e9f;
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r)
          rd<<<blocks, 512>>>((const uint4*)(buf + (size_t)(r % nbuf) * bytes), bytes / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms / 20 < best ? ms / 20 : best;
      }
      printf("%8.1f MB  blocks %4d: %8.2f us/launch  %6.0f GB/s\n", mb, blocks, best * 1e3, bytes / best / 1e6);
    }
  }
  return 0;
}
