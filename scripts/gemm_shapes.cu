// gemm_shapes.cu -- k_gemm_tc on the llama8b decode shapes (diagnostic only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o scripts/gemm_shapes scripts/gemm_shapes.cu -lcuda
// Prints, per shape at T tokens: steady-state us/launch (20 back-to-back
// launches with PDL), isolated us/launch, and a per-CTA timeline of one
// isolated launch (globaltimer: entry spread, first-stage latency, MMA end,
// exit) -- where a small GEMM's fixed cost goes.
#include "../paper_2605_30218_b200/csrc/gemm.cu"

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

using namespace mg;

#ifndef SK_MAX
#define SK_MAX 148
#endif
static int sk_G(int N, int K) {
  const int W = (N / 128) * (K / 64);
  return std::max(1, std::min(W / 4, SK_MAX));
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 64;
  const int shapes[][2] = {{6144, 4096}, {4096, 4096}, {28672, 4096}, {4096, 14336}, {128256, 4096}};
  const char* names[] = {"qkv", "o", "gu", "down", "lm"};
  uint16_t *W, *X;
  float* out;
  cudaMalloc(&W, (size_t)128256 * 4096 * 2);
  cudaMalloc(&X, (size_t)512 * 14336 * 2);
  cudaMalloc(&out, (size_t)256 << 20);
  cudaMemset(W, 0, (size_t)128256 * 4096 * 2);
  cudaMemset(X, 0, (size_t)512 * 14336 * 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int tile = gemm_tile_n(T);
  CUtensorMap mw[5], mx[5];
  size_t woff[5];
  size_t off = 0;
  for (int s = 0; s < 5; ++s) {
    const int N = shapes[s][0], K = shapes[s][1];
    woff[s] = s == 4 ? 0 : off;  // distinct weights for the 4 layer GEMMs (no L2 reuse)
    if (s < 4) off += (size_t)N * K;
    make_tmap_w_tiled(&mw[s], W + woff[s], K, N);
    make_tmap_2d(&mx[s], X, K, 512, tile);
  }
  auto launch = [&](int s, int G) {
    const int N = shapes[s][0], K = shapes[s][1];
    return launch_gemm_tc(mw[s], mx[s], N, K, T, 1, s == 4 ? 0 : G, tile, tile, out, 0);
  };
  for (int s = 0; s < 5; ++s) {
    const int N = shapes[s][0], K = shapes[s][1];
    const double bytes = (double)N * K * 2;
    for (int G : {sk_G(N, K)}) {
      if (s == 4 && G != sk_G(N, K)) continue;
      if (G > (N / 128) * (K / 64)) continue;
      g_gemm_dbg = 0;
      float best = 1e9f, iso = 1e9f;
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) launch(s, G);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms / 20);
        for (int r = 0; r < 5; ++r) {
          cudaEventRecord(a);
          launch(s, G);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms, a, b);
          iso = std::min(iso, ms);
        }
      }
      // per-CTA timeline of one isolated launch (stores skipped: out holds the stamps)
      g_gemm_dbg = 2048 | 2;
      cudaMemset(out, 0, 296 * 4 * 8);
      launch(s, G);
      cudaDeviceSynchronize();
      std::vector<long long> tr(296 * 4);
      cudaMemcpy(tr.data(), out, tr.size() * 8, cudaMemcpyDeviceToHost);
      int n = 0;
      long long t0 = 1LL << 62;
      for (int c = 0; c < 296; ++c)
        if (tr[c * 4]) { t0 = std::min(t0, tr[c * 4]); ++n; }
      std::vector<double> ent, first, mma, ex;
      for (int c = 0; c < 296; ++c)
        if (tr[c * 4]) {
          ent.push_back((tr[c * 4] - t0) * 1e-3);
          first.push_back((tr[c * 4 + 1] - tr[c * 4]) * 1e-3);
          mma.push_back((tr[c * 4 + 2] - t0) * 1e-3);
          ex.push_back((tr[c * 4 + 3] - t0) * 1e-3);
        }
      auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v.empty() ? 0.0 : v[v.size() / 2]; };
      auto mx_ = [](const std::vector<double>& v) { return v.empty() ? 0.0 : *std::max_element(v.begin(), v.end()); };
      printf("%-5s N=%6d K=%5d T=%d G=%3d: steady %7.2f us (%5.0f GB/s)  isolated %7.2f us | CTAs %d entry-spread "
             "%.2f first-stage med %.2f max %.2f | mma-end med %.2f max %.2f | exit med %.2f max %.2f us  %s\n",
             names[s], N, K, T, G, best * 1e3, bytes / best / 1e6, iso * 1e3, n, mx_(ent), med(first), mx_(first),
             med(mma), mx_(mma), med(ex), mx_(ex), cudaGetErrorString(cudaGetLastError()));
    }
  }
  // the engine's per-layer sequence, 32 layers back to back
  g_gemm_dbg = 0;
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(a);
    for (int l = 0; l < 32; ++l)
      for (int s = 0; s < 4; ++s) launch(s, sk_G(shapes[s][0], shapes[s][1]));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = 0;
    for (int s = 0; s < 4; ++s) bytes += 32.0 * shapes[s][0] * shapes[s][1] * 2;
    printf("layer sequence x32: %.3f ms  %.0f GB/s (weights only)\n", ms, bytes / ms / 1e6);
  }
  return 0;
}
