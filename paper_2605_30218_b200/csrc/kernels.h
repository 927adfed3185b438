// kernels.h -- host-side launchers of the sm_100a kernels (internal to
// libmargingate; the public ABI is include/mg.h).  Every launcher only
// enqueues on `st` and returns cudaGetLastError().
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "common.cuh"

namespace mg {

// ---- launch helper: programmatic dependent launch (PDL) on every kernel of
// the decode path, so a kernel's prologue (barrier init, TMEM alloc, weight
// prefetch) overlaps the tail of its predecessor.
extern int g_pdl;  // 1 = launch with programmatic stream serialization
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// ---- weights (K0)
struct GenSpec {
  uint64_t seed;
  uint32_t tid;
  int64_t n;        // logical elements
  int32_t kind;     // 0 proj, 1 embed, 2 gain, 3 bias
  int32_t fan_in;
  int32_t row_len;  // logical row length K (for remaps / tiling)
  int32_t remap;    // 0 identity, 1 gate rows of the 64-interleaved [gate;up], 2 up rows
  int32_t row_off;  // physical row of logical row 0 (q|k|v inside the fused QKV matrix)
  int32_t tiled;    // 1: GEMM weight layout [N/128][K/64][128][64] (see tiled_offset)
};
// Physical offset of element (row, col) of a weight matrix with K columns in
// the tiled layout: 128 x 64 tiles, k-blocks of one 128-row tile contiguous,
// so every TMA box (and every stream-K range) is one contiguous HBM stream.
__host__ __device__ __forceinline__ size_t tiled_offset(size_t row, size_t col, int K) {
  const size_t KB = (size_t)K / 64;
  return (((row / 128) * KB + col / 64) * 128 + row % 128) * 64 + col % 64;
}
bool make_tmap_w_tiled(CUtensorMap* m, const void* base, int K, int N);
cudaError_t launch_gen(const GenSpec& g, uint16_t* dst, cudaStream_t st);

// ---- GEMM (a3, a5-a8)
bool make_tmap_2d(CUtensorMap* m, const void* base, int inner_k, int rows, int box_rows);
// splits: uniform split-K (G == 0) or ignored; G > 0: stream-K over G
// virtual CTAs per token tile (partial slots per tile: part_count()).
// tile_n in {16, 32, 64, 128, 256}; mma_n 16 (verifier slot groups) or tile_n
// t2 != nullptr: fused top-2 epilogue (GemmArgs::t2; LM head only: G == 0, splits == 1)
cudaError_t launch_gemm_tc(const CUtensorMap& mw, const CUtensorMap& mx, int N, int K, int T, int splits, int G,
                           int tile_n, int mma_n, float* out, cudaStream_t st, float* t2 = nullptr,
                           int32_t* nan_flag = nullptr);
// max partial slots of any tile for a GEMM shape (buffer sizing)
int part_slots(const PartSpec& p, int N);
int num_sms();
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
cudaError_t launch_epi_qkv(const float* part, PartSpec ps, const uint16_t* bias, const int32_t* pos, int T, int H,
                           int KV, int hd, const float* rope_cos, const float* rope_sin, uint16_t* q,
                           const CacheView* cache, const int32_t* slot, uint16_t* k_out, uint16_t* v_out,
                           cudaStream_t st, int part_T = 0 /* partial rows (slot stride); 0 = T */);
cudaError_t launch_epi_residual(const uint16_t* x, const float* part, PartSpec ps, int T, int N, uint16_t* out,
                                cudaStream_t st);
// x <- bf16(x + sum_s part[s]); xn <- RMSNorm(x, w) (xn nullable)
cudaError_t launch_residual_norm(uint16_t* x, const float* part, PartSpec ps, int T, int d, const uint16_t* w,
                                 float eps, uint16_t* xn, cudaStream_t st);
cudaError_t launch_epi_swiglu(const float* part, PartSpec ps, int T, int F, uint16_t* out, cudaStream_t st);
cudaError_t launch_gather_rows(const uint16_t* src, const int32_t* rows, int n, int d, uint16_t* dst,
                               cudaStream_t st);

// ---- attention (a4)
// Keys of token t: positions 0..n_keys(t)-1 of request slot(t) in the paged
// cache (or dense K/V [T][KV][key_stride][hd] when cache == nullptr).
// Q and K/V are read by TMA through 3-D maps (make_tmap_3d, box 64 x 16 x 1):
//   qmap  over q        [T'][H][hd]                     (T' >= T rows allocated)
//   kmap  paged: over the pool [L*n_pages*2*KV][PS][hd] (slab = ((l*n_pages+page)*2+kvsel)*KV+kvh)
//         dense: over Kd [T*KV][key_stride][hd];  vmap: the same pool (paged) or Vd
struct AttnArgs {
  CUtensorMap qmap, kmap, vmap;
  const uint16_t* q;      // [T][H*hd]
  CacheView cache;        // paged view (engine), valid when paged != 0
  int32_t paged;
  const int32_t* slot;    // [T] (paged)
  const int32_t* n_keys;  // [T]
  const uint16_t* Kd;     // dense (debug)
  const uint16_t* Vd;
  int32_t key_stride;
  int32_t T, H, KV, hd;
  int32_t split_keys;     // keys per split (multiple of 64); token t has ceil(n_keys/split_keys) splits
  int32_t n_splits;       // grid splits (>= the max over tokens)
  float* part_acc;        // [T][H][n_splits][hd]  split partials (tokens with > 1 split)
  float* part_ml;         // [T][H][n_splits][2]
  int32_t* counter;       // [T][KV] arrival counters, zero between launches
  uint16_t* out;          // [T][H*hd]
  int32_t prewait;        // 1: keys < n_keys-1 predate the previous kernel (fast path: one new column
                          //    per token) and may be read before griddepcontrol.wait
  // fused QKV epilogue (fast path, one new column per token): the CTA builds
  // the q rows of its G query heads from the QKV GEMM partials (bias, RoPE,
  // bf16) in shared memory, and the CTA holding key n-1 builds the new K/V
  // column, appends it to the cache at pos[t] and patches it into its tile
  int32_t fuse_qkv;
  const float* qkv_part;  // [slots][T][(H+2KV)*hd]
  PartSpec qkv_ps;
  const uint16_t* bias;   // nullable
  const int32_t* pos;     // [T] (= n_keys - 1)
  const float* rcos;      // RoPE tables [max_pos][hd/2]
  const float* rsin;
  // mixed launches (fast rows + verifier rows in one GEMM pass, engine.cu
  // forward_mixed): rows of the QKV partial buffer (0 = T) and the q-row
  // offset of this launch's token 0 in the Q tensor map
  int32_t part_T;
  int32_t q_row0;
  // second token group (mixed fast + verifier launch): tokens t >= T1 read and
  // append through cache1 / kvmap1 with split_keys1 (T1 == 0 or >= T: one group)
  int32_t T1;
  int32_t split_keys1;
  CacheView cache1;
  CUtensorMap kvmap1;
  // microbenchmark knobs (scripts/attn_dbg.cu; 0 in the library): 1 skip the
  // fused QKV epilogue's arithmetic, 2 skip QK^T / softmax / PV (stream only),
  // 4 skip the warp combine and the output stores
  int32_t dbg;
  int32_t streams;        // warps (key streams) per CTA: 0 = launch_attention's rule, 2 or 4 forced (tests)
};
bool make_tmap_3d(CUtensorMap* m, const void* base, int d0, int64_t d1, int64_t d2, int box1);
cudaError_t launch_attention(const AttnArgs& a, cudaStream_t st);

// ---- top-2, gate, catch-up, commit (a8-a11)
cudaError_t launch_top2(const float* logits, int T, int V, float* part /*[T][nb][4]*/, int nb, float* v1, int32_t* i1,
                        float* v2, int32_t* i2, float* g, int32_t* nan_flag, cudaStream_t st);
// merge of the fused LM-head epilogue's per-tile top-2 sets t2 [T][nt][4] -> v1, i1, v2, i2, g = v1 - v2
cudaError_t launch_top2_tiles(const float* t2, int T, int nt, float* v1, int32_t* i1, float* v2, int32_t* i2,
                              float* g, cudaStream_t st);
int top2_blocks(int V);

}  // namespace mg
