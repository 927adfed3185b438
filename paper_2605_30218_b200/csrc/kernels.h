// kernels.h -- host-side launchers of the sm_100a kernels (internal to
// libmargingate; the public ABI is include/mg.h).  Every launcher only
// enqueues on `st` and returns cudaGetLastError().
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mg {

// ---- weights (K0)
struct GenSpec {
  uint64_t seed;
  uint32_t tid;
  int64_t n;        // logical elements
  int32_t kind;     // 0 proj, 1 embed, 2 gain, 3 bias
  int32_t fan_in;
  int32_t row_len;  // logical row length (for remaps)
  int32_t remap;    // 0 identity, 1 gate rows of the 64-interleaved [gate;up], 2 up rows
};
cudaError_t launch_gen(const GenSpec& g, uint16_t* dst, cudaStream_t st);

// ---- GEMM (a3, a5-a8)
bool make_tmap_2d(CUtensorMap* m, const void* base, int inner_k, int rows, int box_rows);
cudaError_t launch_gemm_tc(const CUtensorMap& mw, const CUtensorMap& mx, int N, int K, int T, int splits,
                           int tile_n, int mma_n, float* out, cudaStream_t st);
cudaError_t launch_gemm_cc(const uint16_t* x, const uint16_t* W, int N, int K, int T, int splits, float* out,
                           cudaStream_t st);
int gemm_tile_n(int T);

// ---- elementwise (a1, a2, epilogues)
// token list entry for a launch: which request, which position, which token
struct TokRef {
  const int32_t* slot;  // [T]
  const int32_t* pos;   // [T]
  const int32_t* tok;   // [T]
};
// paged cache view of one layer
struct CacheView {
  uint16_t* pool;        // pool base of the whole cache
  const int32_t* pt;     // page table [max_slots][max_pages]
  int32_t max_pages, page_size, n_pages, layer, kv, hd;
};
cudaError_t launch_embed(const uint16_t* E, const int32_t* tok, int T, int d, uint16_t* x, cudaStream_t st);
cudaError_t launch_rmsnorm(const uint16_t* x, const uint16_t* w, int T, int d, float eps, uint16_t* out,
                           cudaStream_t st);
// qkv: part[S][T][NQKV] -> q[T][H*hd]; k, v appended to the cache at (slot, pos)
// (cache == nullptr: dense k_out/v_out [T][KV*hd] instead)
cudaError_t launch_epi_qkv(const float* part, int S, const uint16_t* bias, const int32_t* pos, int T, int H, int KV,
                           int hd, const float* rope_cos, const float* rope_sin, uint16_t* q,
                           const CacheView* cache, const int32_t* slot, uint16_t* k_out, uint16_t* v_out,
                           cudaStream_t st);
cudaError_t launch_epi_residual(const uint16_t* x, const float* part, int S, int T, int N, uint16_t* out,
                                cudaStream_t st);
cudaError_t launch_epi_swiglu(const float* part, int S, int T, int F, uint16_t* out, cudaStream_t st);
cudaError_t launch_gather_rows(const uint16_t* src, const int32_t* rows, int n, int d, uint16_t* dst,
                               cudaStream_t st);

// ---- attention (a4)
// Keys of token t: positions 0..n_keys(t)-1 of request slot(t) in the paged
// cache (or dense K/V [T][KV][key_stride][hd] when cache == nullptr).
struct AttnArgs {
  const uint16_t* q;      // [T][H*hd]
  CacheView cache;        // paged view (engine), valid when paged != 0
  int32_t paged;
  const int32_t* slot;    // [T] (paged)
  const int32_t* n_keys;  // [T]
  const uint16_t* Kd;     // dense (debug)
  const uint16_t* Vd;
  int32_t key_stride;
  int32_t T, H, KV, hd, chunk, n_chunks;
  float* part_acc;        // [T][H][n_chunks][hd]
  float* part_ml;         // [T][H][n_chunks][2]
  uint16_t* out;          // [T][H*hd]
};
cudaError_t launch_attention(const AttnArgs& a, cudaStream_t st);

// ---- top-2, gate, catch-up, commit (a8-a11)
cudaError_t launch_top2(const float* logits, int T, int V, float* part /*[T][nb][4]*/, int nb, float* v1, int32_t* i1,
                        float* v2, int32_t* i2, float* g, int32_t* nan_flag, cudaStream_t st);
int top2_blocks(int V);

}  // namespace mg
