// capi_debug.cu -- test-only op-level entry points (include/mg_debug.h).
// Each one launches exactly the kernel the engine launches for that step of
// the path, on caller buffers, so the parity tests can hold every kernel
// against the oracle on identical inputs.
#include <cmath>
#include <vector>

#include "../../include/mg_debug.h"
#include "control.h"
#include "kernels.h"

using namespace mg;

static mg_status st_of(cudaError_t e) { return e == cudaSuccess ? MG_OK : MG_ERR_CUDA; }

// ---------------------------------------------------------------- launch floor
namespace {
__global__ void k_null() {
  extern __shared__ unsigned char s_null[];
  if (threadIdx.x == 1023) s_null[0] = 0;  // never true: keeps the shared-memory reservation
}
}  // namespace

extern "C" {

mg_status mgd_gen_tensor(uint64_t seed, uint32_t tid, int64_t n, int32_t kind, int32_t fan_in, uint16_t* out,
                         void* stream) {
  if (!out || n < 0 || kind < 0 || kind > 3 || (kind == 0 && fan_in < 1)) return MG_ERR_INVALID;
  GenSpec g{seed, tid, n, kind, fan_in, 0, 0, 0, 0};
  return st_of(launch_gen(g, out, (cudaStream_t)stream));
}

mg_status mgd_rmsnorm(const uint16_t* x, const uint16_t* w, int32_t T, int32_t d, float eps, uint16_t* out,
                      void* stream) {
  if (!x || !w || !out || T < 1 || d % 8) return MG_ERR_INVALID;
  return st_of(launch_rmsnorm(x, w, T, d, eps, out, (cudaStream_t)stream));
}

mg_status mgd_gemm(const uint16_t* x, const uint16_t* W, int32_t T, int32_t N, int32_t K, int32_t splits,
                   int32_t impl, int32_t mma_n, int32_t tile_n, float* out, void* stream) {
  // splits < 0: stream-K over G = -splits virtual CTAs (tcgen05 only)
  const int G = splits < 0 ? -splits : 0;
  if (!x || !W || !out || T < 1 || N % 128 || K % 64 || splits == 0 || splits > K / 64 ||
      G > (N / 128) * (K / 64))
    return MG_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (impl != 0) return MG_ERR_INVALID;  // tcgen05 only (the CUDA-core GEMV was removed)
  if (tile_n <= 0) tile_n = gemm_tile_n(T);
  if (mma_n < 0 || mma_n > tile_n || (mma_n && tile_n % mma_n) || (mma_n && mma_n % 16)) return MG_ERR_INVALID;
  // the kernels read weights in the engine's tiled layout: tile W (row-major here)
  std::vector<uint16_t> rm((size_t)N * K), tl((size_t)N * K);
  cudaStreamSynchronize(st);
  if (cudaMemcpy(rm.data(), W, rm.size() * 2, cudaMemcpyDeviceToHost) != cudaSuccess) return MG_ERR_CUDA;
  for (size_t r = 0; r < (size_t)N; ++r)
    for (size_t k = 0; k < (size_t)K; ++k) tl[tiled_offset(r, k, K)] = rm[r * K + k];
  uint16_t* Wt = nullptr;
  if (cudaMalloc(&Wt, tl.size() * 2) != cudaSuccess) return MG_ERR_CUDA;
  cudaMemcpy(Wt, tl.data(), tl.size() * 2, cudaMemcpyHostToDevice);
  cudaError_t e;
  {
    CUtensorMap mw, mx;
    if (!make_tmap_w_tiled(&mw, Wt, K, N) || !make_tmap_2d(&mx, x, K, T, tile_n)) {
      cudaFree(Wt);
      return MG_ERR_CUDA;
    }
    e = launch_gemm_tc(mw, mx, N, K, T, G ? 1 : splits, G, tile_n, mma_n, out, st);
  }
  cudaStreamSynchronize(st);
  cudaFree(Wt);
  return st_of(e);
}

mg_status mgd_gemm_top2(const uint16_t* x, const uint16_t* W, int32_t T, int32_t N, int32_t K, int32_t tile_n,
                        float* v1, int32_t* i1, float* v2, int32_t* i2, float* g, int32_t* nan_flag, void* stream) {
  if (!x || !W || !v1 || !i1 || !v2 || !i2 || !g || !nan_flag || T < 1 || N % 128 || K % 64) return MG_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (tile_n <= 0) tile_n = gemm_tile_n(T);
  std::vector<uint16_t> rm((size_t)N * K), tl((size_t)N * K);
  cudaStreamSynchronize(st);
  if (cudaMemcpy(rm.data(), W, rm.size() * 2, cudaMemcpyDeviceToHost) != cudaSuccess) return MG_ERR_CUDA;
  for (size_t r = 0; r < (size_t)N; ++r)
    for (size_t k = 0; k < (size_t)K; ++k) tl[tiled_offset(r, k, K)] = rm[r * K + k];
  uint16_t* Wt = nullptr;
  float* t2 = nullptr;
  if (cudaMalloc(&Wt, tl.size() * 2) != cudaSuccess) return MG_ERR_CUDA;
  if (cudaMalloc(&t2, (size_t)T * (N / 128) * 16) != cudaSuccess) {
    cudaFree(Wt);
    return MG_ERR_CUDA;
  }
  cudaMemcpy(Wt, tl.data(), tl.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap mw, mx;
  cudaError_t e = cudaErrorInvalidValue;
  if (make_tmap_w_tiled(&mw, Wt, K, N) && make_tmap_2d(&mx, x, K, T, tile_n)) {
    e = launch_gemm_tc(mw, mx, N, K, T, 1, 0, tile_n, tile_n, nullptr, st, t2, nan_flag);
    if (e == cudaSuccess) e = launch_top2_tiles(t2, T, N / 128, v1, i1, v2, i2, g, st);
  }
  cudaStreamSynchronize(st);
  cudaFree(Wt);
  cudaFree(t2);
  return st_of(e);
}

mg_status mgd_qkv_epilogue(const float* part, int32_t splits, const uint16_t* bias, const int32_t* pos, int32_t T,
                           int32_t H, int32_t KV, int32_t hd, float theta, int32_t max_pos, uint16_t* q, uint16_t* k,
                           uint16_t* v, void* stream) {
  if (!part || !pos || !q || !k || !v || T < 1 || (hd != 64 && hd != 128) || max_pos < 1) return MG_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  // RoPE tables, computed like the engine's
  const int h2 = hd / 2;
  std::vector<float> cs((size_t)max_pos * h2), sn((size_t)max_pos * h2);
  for (int p = 0; p < max_pos; ++p)
    for (int i = 0; i < h2; ++i) {
      const double ang = (double)p * pow((double)theta, -(2.0 * (double)i) / (double)hd);
      cs[(size_t)p * h2 + i] = (float)cos(ang);
      sn[(size_t)p * h2 + i] = (float)sin(ang);
    }
  float *dc = nullptr, *ds = nullptr;
  if (cudaMalloc(&dc, cs.size() * 4) != cudaSuccess || cudaMalloc(&ds, sn.size() * 4) != cudaSuccess)
    return MG_ERR_CUDA;
  cudaMemcpy(dc, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice);
  const PartSpec ps{splits, 0, 1, (H + 2 * KV) * hd / 128};
  cudaError_t e = launch_epi_qkv(part, ps, bias, pos, T, H, KV, hd, dc, ds, q, nullptr, nullptr, k, v, st);
  cudaStreamSynchronize(st);
  cudaFree(dc);
  cudaFree(ds);
  return st_of(e);
}

mg_status mgd_launch_floor(int32_t smem_bytes, int32_t reps, void* stream, float* us_out) {
  if (!us_out || reps < 1 || smem_bytes < 0 || smem_bytes > 227 * 1024) return MG_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaFuncSetAttribute(k_null, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess)
    return MG_ERR_CUDA;
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return MG_ERR_CUDA;
  const int grid = num_sms();
  for (int i = 0; i < 5; ++i) k_null<<<grid, 192, smem_bytes, st>>>();
  double sum = 0.0;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a, st);
    k_null<<<grid, 192, smem_bytes, st>>>();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    sum += ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *us_out = (float)(1e3 * sum / reps);
  return st_of(cudaGetLastError());
}

mg_status mgd_attention(const uint16_t* q, const uint16_t* K, const uint16_t* V, const int32_t* n_keys, int32_t T,
                        int32_t H, int32_t KVh, int32_t hd, int32_t key_stride, int32_t split_keys, uint16_t* o,
                        void* stream) {
  return mgd_attention_streams(q, K, V, n_keys, T, H, KVh, hd, key_stride, split_keys, 4, o, stream);
}

mg_status mgd_attention_streams(const uint16_t* q, const uint16_t* K, const uint16_t* V, const int32_t* n_keys,
                                int32_t T, int32_t H, int32_t KVh, int32_t hd, int32_t key_stride, int32_t split_keys,
                                int32_t streams, uint16_t* o, void* stream) {
  if (!q || !K || !V || !n_keys || !o || T < 1 || split_keys < 64 || split_keys % 64 || key_stride < 1)
    return MG_ERR_INVALID;
  if (streams != 2 && streams != 4) return MG_ERR_INVALID;
  if (KVh < 1 || H % KVh || H / KVh > 16) return MG_ERR_INVALID;
  const int nsp = (key_stride + split_keys - 1) / split_keys;
  float *acc = nullptr, *ml = nullptr;
  int32_t* cnt = nullptr;
  if (cudaMalloc(&acc, (size_t)T * H * nsp * hd * 4) != cudaSuccess ||
      cudaMalloc(&ml, (size_t)T * H * nsp * 2 * 4) != cudaSuccess ||
      cudaMalloc(&cnt, (size_t)T * KVh * 4) != cudaSuccess)
    return MG_ERR_CUDA;
  cudaMemset(cnt, 0, (size_t)T * KVh * 4);
  AttnArgs a{};
  a.q = q; a.paged = 0; a.n_keys = n_keys; a.Kd = K; a.Vd = V; a.key_stride = key_stride;
  a.T = T; a.H = H; a.KV = KVh; a.hd = hd; a.split_keys = split_keys; a.n_splits = nsp;
  a.part_acc = acc; a.part_ml = ml; a.counter = cnt; a.out = o;
  a.streams = streams;
  cudaError_t e = cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  if (make_tmap_3d(&a.qmap, q, hd, H, T, 16) && make_tmap_3d(&a.kmap, K, hd, key_stride, (int64_t)T * KVh, 16) &&
      make_tmap_3d(&a.vmap, V, hd, key_stride, (int64_t)T * KVh, 16))
    e = launch_attention(a, st);
  cudaStreamSynchronize(st);
  cudaFree(acc);
  cudaFree(ml);
  cudaFree(cnt);
  return st_of(e);
}

mg_status mgd_residual(const uint16_t* x, const float* part, int32_t splits, int32_t T, int32_t N, uint16_t* out,
                       void* stream) {
  if (!x || !part || !out || T < 1 || N < 1 || splits < 1) return MG_ERR_INVALID;
  return st_of(launch_epi_residual(x, part, PartSpec{splits, 0, 1, 1}, T, N, out, (cudaStream_t)stream));
}

mg_status mgd_swiglu(const float* part, int32_t splits, int32_t T, int32_t F, uint16_t* out, void* stream) {
  if (!part || !out || T < 1 || F % 64 || splits < 1) return MG_ERR_INVALID;
  return st_of(launch_epi_swiglu(part, PartSpec{splits, 0, 1, 1}, T, F, out, (cudaStream_t)stream));
}

mg_status mgd_top2(const float* logits, int32_t T, int32_t V, float* v1, int32_t* i1, float* v2, int32_t* i2,
                   float* g, int32_t* nan_flag, void* stream) {
  if (!logits || T < 1 || V < 2 || !nan_flag) return MG_ERR_INVALID;
  const int nb = top2_blocks(V);
  float* part = nullptr;
  if (cudaMalloc(&part, (size_t)T * nb * 4 * 4) != cudaSuccess) return MG_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = launch_top2(logits, T, V, part, nb, v1, i1, v2, i2, g, nan_flag, st);
  cudaStreamSynchronize(st);
  cudaFree(part);
  return st_of(e);
}

mg_status mgd_gate(const float* g, const uint8_t* prot, int32_t B, float tau, uint8_t* trig, int32_t* rows,
                   int32_t* count, void* stream) {
  if (!g || !prot || !trig || !rows || !count || B < 1 || B > 1024) return MG_ERR_INVALID;
  // standalone gate: identity slots, no catch-up list (pos = shadow_len - 1 => gap 0 is not used)
  cudaStream_t st = (cudaStream_t)stream;
  int32_t *slots = nullptr, *zeros = nullptr, *ctrl = nullptr, *rank = nullptr, *last = nullptr, *cu = nullptr;
  std::vector<int32_t> h(B);
  for (int i = 0; i < B; ++i) h[i] = i;
  if (cudaMalloc(&slots, B * 4) || cudaMalloc(&zeros, B * 4 * 2) || cudaMalloc(&ctrl, (2 + B) * 4) ||
      cudaMalloc(&rank, B * 4) || cudaMalloc(&last, B * 4) || cudaMalloc(&cu, (size_t)B * 4 * 4))
    return MG_ERR_CUDA;
  cudaMemcpy(slots, h.data(), B * 4, cudaMemcpyHostToDevice);
  cudaMemset(zeros, 0, B * 4 * 2);
  GateArgs a{};
  a.g = g; a.prot = prot; a.tau = tau; a.slots = slots; a.B = B;
  a.pos = zeros; a.shadow_len = zeros; a.hist = zeros + B; a.hist_stride = 0;
  a.trig = trig; a.rank = rank; a.ctrl = ctrl; a.last = last;
  a.cu_slot = cu; a.cu_pos = cu + B; a.cu_tok = cu + 2 * B; a.cu_nk = cu + 3 * B;
  cudaError_t e = launch_gate(a, st);
  cudaStreamSynchronize(st);
  std::vector<int32_t> ch(2 + B);
  cudaMemcpy(ch.data(), ctrl, (2 + B) * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(count, ctrl, 4, cudaMemcpyDeviceToDevice);
  cudaMemcpy(rows, ctrl + 2, B * 4, cudaMemcpyDeviceToDevice);
  cudaFree(slots); cudaFree(zeros); cudaFree(ctrl); cudaFree(rank); cudaFree(last); cudaFree(cu);
  return st_of(e);
}

}  // extern "C"
