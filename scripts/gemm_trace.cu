// gemm_trace.cu -- per-stage timeline of CTA 0 of k_gemm_tc (diagnostic only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o scripts/gemm_trace scripts/gemm_trace.cu -lcuda
#include "../paper_2605_30218_b200/csrc/gemm.cu"

#include <stdio.h>

#include <vector>

using namespace mg;

int main() {
  const int N = 128256, K = 4096;
  uint16_t *W, *X;
  float* out;
  cudaMalloc(&W, (size_t)N * K * 2);
  cudaMalloc(&X, (size_t)512 * K * 2);
  cudaMalloc(&out, (size_t)64 << 22);
  cudaMemset(W, 0x11, (size_t)N * K * 2);
  cudaMemset(X, 0, (size_t)512 * K * 2);
  CUtensorMap mw, mx;
  make_tmap_w_tiled(&mw, W, K, N);
  const int T = 16, tile = 16;
  make_tmap_2d(&mx, X, K, 512, tile);
  using C = GemmTcCfg<16>;
  printf("KS=%d NS=%d stage=%d B\n", C::KS, C::NS, C::STAGE);
  for (int dbg : {1026, 1027}) {
    g_gemm_dbg = dbg;
    for (int r = 0; r < 3; ++r) launch_gemm_tc(mw, mx, N, K, T, 1, 0, tile, tile, out, 0);
    cudaDeviceSynchronize();
    std::vector<long long> tr(256 * 4);
    cudaMemcpy(tr.data(), out, tr.size() * 8, cudaMemcpyDeviceToHost);
    printf("dbg=%d %s\n", dbg, cudaGetErrorString(cudaGetLastError()));
    double lat = 0, mma = 0, rec = 0, inter = 0;
    int n = 0;
    for (int it = 16; it < 200; ++it) {
      const long long* a = &tr[it * 4];
      lat += a[1] - a[0];
      mma += a[2] - a[1];
      inter += tr[(it + 1) * 4 + 1] - a[1];
      rec += tr[(it + C::NS) * 4 + 0] - a[2];
      ++n;
      if (it < 24)
        printf("  it %3d  issue->arrive %6lld  arrive->commit %5lld  commit->reissue %6lld  inter-arrival %6lld\n",
               it, a[1] - a[0], a[2] - a[1], tr[(it + C::NS) * 4 + 0] - a[2], tr[(it + 1) * 4 + 1] - a[1]);
    }
    printf("  mean cycles: issue->arrive %.0f arrive->commit %.0f commit->reissue %.0f inter-arrival %.0f "
           "(-> %.1f GB/s/SM at 1.9 GHz)\n",
           lat / n, mma / n, rec / n, inter / n, C::KS * 16384.0 / (inter / n / 1.9));
  }
  return 0;
}
