// attn_dbg.cu -- where a k_attn launch spends its time (diagnostic only):
// steady-state us/launch (20 back-to-back PDL launches, rotating over 4 layers
// of a paged Llama-8B-shaped cache so the K/V bytes come from HBM) of the fast
// path's launch (fused QKV epilogue, prewait, one split per (token, kv head))
// at batch B and context ctx, and with the microbenchmark knobs of AttnArgs.dbg:
// 1 no QKV-epilogue arithmetic, 2 no QK^T / softmax / PV, 4 no combine / stores.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o scripts/attn_dbg scripts/attn_dbg.cu -lcuda
#include "../paper_2605_30218_b200/csrc/gemm.cu"
#include "../paper_2605_30218_b200/csrc/attention.cu"

#include <stdio.h>
#include <stdlib.h>

#include <vector>

using namespace mg;

int main(int argc, char** argv) {
  const int H = 32, KV = 8, HD = 128, PS = 64, L = 4, NQKV = (H + 2 * KV) * HD;
  int Bs[] = {64, 128, 64, 32, 8};
  int ctxs[] = {384, 384, 620, 620, 620};
  int ncfg = 5;
  if (argc > 2) {  // one configuration: attn_dbg B ctx
    Bs[0] = atoi(argv[1]);
    ctxs[0] = atoi(argv[2]);
    ncfg = 1;
  }
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int c = 0; c < ncfg; ++c) {
    const int B = Bs[c], ctx = ctxs[c];
    const int max_pages = (ctx + 1 + PS - 1) / PS, n_pages = B * max_pages;
    const size_t slab = (size_t)PS * HD;  // one (page, K|V, kv head) slab
    const size_t pool_elems = (size_t)L * n_pages * 2 * KV * slab;
    uint16_t* pool;
    cudaMalloc(&pool, pool_elems * 2);
    cudaMemset(pool, 0, pool_elems * 2);
    std::vector<int32_t> hpt((size_t)B * max_pages), hslot(B), hn(B), hpos(B);
    for (int b = 0; b < B; ++b) {
      for (int j = 0; j < max_pages; ++j) hpt[(size_t)b * max_pages + j] = b * max_pages + j;
      hslot[b] = b;
      hn[b] = ctx;
      hpos[b] = ctx - 1;
    }
    int32_t *pt, *slot, *nk, *pos, *cnt;
    cudaMalloc(&pt, hpt.size() * 4);
    cudaMalloc(&slot, B * 4);
    cudaMalloc(&nk, B * 4);
    cudaMalloc(&pos, B * 4);
    cudaMalloc(&cnt, B * KV * 4);
    cudaMemcpy(pt, hpt.data(), hpt.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(slot, hslot.data(), B * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(nk, hn.data(), B * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(pos, hpos.data(), B * 4, cudaMemcpyHostToDevice);
    cudaMemset(cnt, 0, B * KV * 4);
    const int S = 4;  // QKV partial slots (stream-K over 148 virtual CTAs: 3-4 per tile)
    float *part, *rc, *rs, *pacc, *pml;
    uint16_t *q, *out;
    cudaMalloc(&part, (size_t)S * B * NQKV * 4);
    cudaMemset(part, 0, (size_t)S * B * NQKV * 4);
    cudaMalloc(&rc, (size_t)(ctx + 1) * HD / 2 * 4);
    cudaMalloc(&rs, (size_t)(ctx + 1) * HD / 2 * 4);
    cudaMemset(rc, 0, (size_t)(ctx + 1) * HD / 2 * 4);
    cudaMemset(rs, 0, (size_t)(ctx + 1) * HD / 2 * 4);
    cudaMalloc(&q, (size_t)B * H * HD * 2);
    cudaMemset(q, 0, (size_t)B * H * HD * 2);
    cudaMalloc(&out, (size_t)B * H * HD * 2);
    cudaMalloc(&pacc, (size_t)B * H * HD * 4);
    cudaMalloc(&pml, (size_t)B * H * 2 * 4);
    AttnArgs a{};
    const int64_t slabs = (int64_t)L * n_pages * 2 * KV;
    make_tmap_3d(&a.kmap, pool, HD, PS, slabs, 16);
    a.vmap = a.kmap;
    make_tmap_3d(&a.qmap, q, HD, H, B, 16);
    a.q = q;
    a.paged = 1;
    a.slot = slot;
    a.n_keys = nk;
    a.T = B; a.H = H; a.KV = KV; a.hd = HD;
    a.split_keys = (ctx + 63) / 64 * 64 + 64;
    a.n_splits = 1;
    a.part_acc = pacc; a.part_ml = pml; a.counter = cnt; a.out = out;
    a.prewait = 1;
    a.fuse_qkv = 1;
    a.qkv_part = part;
    a.qkv_ps = PartSpec{S, 0, 0, 0};
    a.pos = pos; a.rcos = rc; a.rsin = rs;
    printf("B=%3d ctx=%4d  KV bytes/launch %6.1f MB ", B, ctx, (double)B * ctx * KV * HD * 4 / 1e6);
    const int modes[] = {0, 1, 4, 2, 7, -1};
    for (int m : modes) {
      AttnArgs x = a;
      if (m < 0) {  // the unfused launch: Q tile by TMA from q, no epilogue
        x.fuse_qkv = 0;
        x.prewait = 0;
      } else {
        x.dbg = m;
      }
      auto run = [&](int n) {
        for (int i = 0; i < n; ++i) {
          x.cache = CacheView{pool, pt, max_pages, PS, n_pages, i % L, KV, HD};
          launch_attention(x, st);
        }
      };
      run(8);
      cudaEventRecord(e0, st);
      run(20);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1000 / 20;
      printf(" | %s %6.2f us %4.2f TB/s", m < 0 ? "unfused" : (m == 0 ? "dbg0" : (m == 1 ? "dbg1" : (m == 2 ? "dbg2" : (m == 4 ? "dbg4" : "dbg7")))),
             us, (double)B * ctx * KV * HD * 4 / (us * 1e6));
    }
    cudaError_t err = cudaGetLastError();
    printf("  (%s)\n", cudaGetErrorString(err));
    cudaFree(pool); cudaFree(pt); cudaFree(slot); cudaFree(nk); cudaFree(pos); cudaFree(cnt);
    cudaFree(part); cudaFree(rc); cudaFree(rs); cudaFree(q); cudaFree(out); cudaFree(pacc); cudaFree(pml);
  }
  return 0;
}
