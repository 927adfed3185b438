/*
 * examples/mg_decode.c -- a plain C client of the MarginGate C ABI
 * (include/mg.h): no Python, no torch.  The caller owns the device memory
 * (cudaMalloc), prefills a few requests, runs MarginGate decode steps
 * with one protected request, and checks the ABI's
 * contract on its own results:
 *   - tau = +inf (always-on verification): the protected
 *     request decoded inside a batch equals the same request decoded alone;
 *   - every step commits one token per row; kinds are 0/1/2;
 *   - mg_stats: 0 <= repairs <= triggers <= protected_rows.
 * Exit code 0 on success.  Build: make examples (gcc + libcudart).
 * usage: mg_decode [steps]
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mg.h"

#define CHECK(x)                                                                  \
  do {                                                                            \
    mg_status s_ = (x);                                                           \
    if (s_ != MG_OK) {                                                            \
      fprintf(stderr, "%s -> %d: %s\n", #x, (int)s_, mg_last_error(ctx));         \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static int run(int B, int steps, const int32_t prompts[][12], int32_t* seq_out /* [B][steps+1] */) {
  mg_ctx* ctx = NULL;
  /* BASELINE.json configs[0]: the tiny decoder (2 layers, d 256, 4 heads, vocab 4096) */
  mg_config cfg = {2, 256, 4, 4, 64, 1024, 4096, 0, 1e-5f, 10000.0f, 42, B, B, 64, 16, 0};
  mg_sizes sz;
  if (mg_query_sizes(&cfg, &sz) != MG_OK) return 1;
  mg_buffers buf;
  if (cudaMalloc(&buf.weights, sz.weights) || cudaMalloc(&buf.kv_fast, sz.kv_fast) ||
      cudaMalloc(&buf.kv_shadow, sz.kv_shadow) || cudaMalloc(&buf.workspace, sz.workspace))
    return 1;
  CHECK(mg_init(&cfg, &buf, NULL, &ctx));
  int32_t *tok_d = NULL;
  uint8_t *kind_d = NULL;
  if (cudaMalloc((void**)&tok_d, B * 4) || cudaMalloc((void**)&kind_d, B)) return 1;
  int32_t slots[8];
  uint8_t prot[8];
  for (int b = 0; b < B; ++b) {
    slots[b] = b;
    prot[b] = b == 0;  /* one protected request */
    CHECK(mg_prefill(ctx, b, prompts[b], 12, &seq_out[b * (steps + 1)]));
  }
  for (int t = 0; t < steps; ++t) {
    CHECK(mg_decode_step(ctx, slots, B, prot, INFINITY, tok_d, kind_d, NULL));
    int32_t tok[8];
    uint8_t kind[8];
    if (cudaMemcpy(tok, tok_d, B * 4, cudaMemcpyDeviceToHost) || cudaMemcpy(kind, kind_d, B, cudaMemcpyDeviceToHost))
      return 1;
    for (int b = 0; b < B; ++b) {
      if (kind[b] > 2 || tok[b] < 0 || tok[b] >= 4096) return 1;
      if (!prot[b] && kind[b] != 0) return 1;  /* only protected rows are gated */
      seq_out[b * (steps + 1) + t + 1] = tok[b];
    }
  }
  mg_stats_t st;
  CHECK(mg_stats(ctx, &st));
  printf("B=%d: steps %llu rows %llu protected %llu triggers %llu verified %llu repairs %llu\n", B,
         (unsigned long long)st.steps, (unsigned long long)st.rows, (unsigned long long)st.protected_rows,
         (unsigned long long)st.triggers, (unsigned long long)st.verified, (unsigned long long)st.repairs);
  if (st.steps != (uint64_t)steps || st.rows != (uint64_t)(steps * B) || st.protected_rows != (uint64_t)steps ||
      st.triggers != st.protected_rows || st.repairs > st.triggers)
    return 1;
  mg_destroy(ctx);
  cudaFree(tok_d);
  cudaFree(kind_d);
  cudaFree(buf.weights);
  cudaFree(buf.kv_fast);
  cudaFree(buf.kv_shadow);
  cudaFree(buf.workspace);
  return 0;
}

int main(int argc, char** argv) {
  const int steps = argc > 1 ? atoi(argv[1]) : 16;
  int32_t prompts[8][12];
  unsigned x = 12345u;
  for (int b = 0; b < 8; ++b)
    for (int i = 0; i < 12; ++i) {
      x = x * 1664525u + 1013904223u;
      prompts[b][i] = (int32_t)(x >> 20) % 4096;
    }
  int32_t* batched = calloc(8 * (steps + 1), 4);
  int32_t* alone = calloc(steps + 1, 4);
  if (run(8, steps, (const int32_t(*)[12])prompts, batched) || run(1, steps, (const int32_t(*)[12])prompts, alone)) {
    fprintf(stderr, "FAILED\n");
    return 1;
  }
  if (memcmp(batched, alone, (steps + 1) * 4) != 0) {
    fprintf(stderr, "FAILED: the protected request differs alone vs batched at tau = inf\n");
    return 1;
  }
  printf("ok: protected request identical alone vs in a batch of 8 over %d steps\n", steps);
  free(batched);
  free(alone);
  return 0;
}
