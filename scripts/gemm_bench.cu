// gemm_bench.cu -- isolate k_gemm_tc throughput (diagnostic only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o scripts/gemm_bench scripts/gemm_bench.cu -lcuda
#include "../paper_2605_30218_b200/csrc/gemm.cu"

#include <stdio.h>

using namespace mg;

int main() {
  const int shapes[][2] = {{28672, 4096}, {128256, 4096}};
  uint16_t *W, *X;
  float* out;
  cudaMalloc(&W, (size_t)128256 * 4096 * 2);
  cudaMalloc(&X, (size_t)512 * 14336 * 2);
  cudaMalloc(&out, (size_t)64 << 20 << 2);
  cudaMemset(W, 0, (size_t)128256 * 4096 * 2);
  cudaMemset(X, 0, (size_t)512 * 14336 * 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& s : shapes) {
    const int N = s[0], K = s[1];
    CUtensorMap mw4, mw2;
    make_tmap_w_tiled(&mw4, W, K, N);
    make_tmap_2d(&mw2, W, 64, N * (K / 64), 128);
    for (int T : {16, 64}) {
      const int tile = gemm_tile_n(T);
      CUtensorMap mx;
      make_tmap_2d(&mx, X, K, 512, tile);
      const int G = (N / 128) * (K / 64) / 4 < 148 ? (N / 128) * (K / 64) / 4 : 148;
      for (int dbg : {0, 1}) {
        for (int pdl : {1}) {
          g_gemm_dbg = dbg;
          g_pdl = pdl;
          float best = 1e9f;
          for (int it = 0; it < 5; ++it) {
            cudaEventRecord(a);
            for (int r = 0; r < 10; ++r)
              launch_gemm_tc(mw4, mx, N, K, T, 1, N == 128256 ? 0 : G, tile, tile, out, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms / 10 < best ? ms / 10 : best;
          }
          const double bytes = (double)N * K * 2;
          printf("N=%6d K=%5d T=%3d dbg=%d pdl=%d: %8.2f us  %6.0f GB/s  %s\n", N, K, T, dbg, pdl, best * 1e3,
                 bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
  }
  return 0;
}
