// gemm_dbg.cu -- where a k_gemm_tc launch spends its time at 64 vs 128 tokens
// (diagnostic only): steady-state us/launch (20 back-to-back launches, PDL) of
// the llama8b layer GEMMs with the product kernel (dbg 0), without the
// epilogue's partial stores (dbg 2), without the MMAs (dbg 1), both (dbg 3),
// without the activation TMA loads (dbg 4) and without loads and stores (dbg 6).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o scripts/gemm_dbg scripts/gemm_dbg.cu -lcuda
#include "../paper_2605_30218_b200/csrc/gemm.cu"

#include <stdio.h>

#include <algorithm>

using namespace mg;

int main() {
  const int shapes[][2] = {{6144, 4096}, {4096, 4096}, {28672, 4096}, {4096, 14336}};
  const char* names[] = {"qkv", "o", "gu", "down"};
  uint16_t *W, *X;
  float* out;
  size_t wtot = 0;
  for (auto& s : shapes) wtot += (size_t)s[0] * s[1];
  cudaMalloc(&W, wtot * 2);
  cudaMalloc(&X, (size_t)256 * 14336 * 2);
  cudaMalloc(&out, (size_t)512 << 20);
  cudaMemset(W, 0, wtot * 2);
  cudaMemset(X, 0, (size_t)256 * 14336 * 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int T : {64, 128}) {
    const int tile = gemm_tile_n(T);
    size_t off = 0;
    for (int s = 0; s < 4; ++s) {
      const int N = shapes[s][0], K = shapes[s][1];
      CUtensorMap mw, mx;
      make_tmap_w_tiled(&mw, W + off, K, N);
      make_tmap_2d(&mx, X, K, 256, tile);
      off += (size_t)N * K;
      const int G = std::max(1, std::min((N / 128) * (K / 64) / 4, 148));
      printf("T=%3d %-5s", T, names[s]);
      for (int dbg : {0, 2, 1, 3, 4, 6}) {
        g_gemm_dbg = dbg;
        for (int i = 0; i < 5; ++i) launch_gemm_tc(mw, mx, N, K, T, 1, G, tile, tile, out, 0);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int i = 0; i < 20; ++i) launch_gemm_tc(mw, mx, N, K, T, 1, G, tile, tile, out, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("  dbg%d %7.2f us", dbg, ms * 1e3f / 20);
      }
      printf("   (%s)\n", cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
