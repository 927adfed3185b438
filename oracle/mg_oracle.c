/*
 * oracle/mg_oracle.c -- plain, slow, obviously-correct CPU oracle of the
 * MarginGate per-step decode path (arxiv 2605.30218, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's CPU legs, never by the product path.  Shares no code with the
 * CUDA library.  Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp
 * (no FMA contraction, IEEE fp32).  OpenMP parallelises ONLY over
 * independent outputs (output features, vocabulary entries); every sum is
 * one thread's left-to-right loop, so results do not depend on the thread
 * count.
 *
 * Every arithmetic step follows DESIGN.md section 3 ("forward dataflow and
 * rounding points"), which restates SURVEY 8(c) steps 1-5.  Citations to
 * the paper are given per function.
 */
#include "mg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* bf16 <-> fp32: round to nearest, ties to even.      */
/* NaN -> quiet NaN, +-inf kept, overflow rounds to +-inf.             */
/* ------------------------------------------------------------------ */
uint16_t or_f32_to_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) {            /* inf or NaN */
    if (u & 0x007fffffu) return (uint16_t)((u >> 16) | 0x0040u);
    return (uint16_t)(u >> 16);
  }
  u += 0x7fffu + ((u >> 16) & 1u);                   /* RNE on the dropped 16 bits */
  return (uint16_t)(u >> 16);
}

float or_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline float bf(uint16_t h) { return or_bf16_to_f32(h); }

/* Contiguous equal chunks, remainder to the leading chunks
 * ("Chunk boundaries").  Returns start of chunk c. */
static inline int64_t chunk_start(int64_t n, int64_t S, int64_t c) {
  int64_t base = n / S, rem = n % S;
  return c * base + (c < rem ? c : rem);
}

/* chunked_dot: products in fp32 (exact for bf16 x bf16),
 * each chunk summed left to right, chunk partials summed left to right. */
float or_dot_bf16(const uint16_t* a, const uint16_t* b, int32_t n, int32_t splits) {
  int64_t S = splits < 1 ? 1 : splits;
  if (S > n) S = n > 0 ? n : 1;
  float total = 0.0f;
  for (int64_t c = 0; c < S; ++c) {
    int64_t lo = chunk_start(n, S, c), hi = chunk_start(n, S, c + 1);
    float part = 0.0f;
    for (int64_t i = lo; i < hi; ++i) part = part + bf(a[i]) * bf(b[i]);
    total = (c == 0) ? part : total + part;
  }
  return total;
}

/* ------------------------------------------------------------------ */
/* Counter-based weight generator. */
/* ------------------------------------------------------------------ */
uint64_t or_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* which (layer >= 0): 0 attn_norm 1 wq 2 wk 3 wv 4 wo 5 mlp_norm 6 wg 7 wu 8 wd 9 bq 10 bk 11 bv
 * which (layer == -1): 0 embed 1 final_norm 2 lm_head */
uint32_t or_tensor_id(const or_cfg* c, int32_t layer, int32_t which) {
  if (layer < 0) {
    if (which == 0) return 0u;
    return (uint32_t)(1 + 16 * c->n_layers + (which - 1));
  }
  return (uint32_t)(1 + 16 * layer + which);
}

/* kind 0: projection, sigma = 1/sqrt(fan_in); 1: embedding, sigma = 1;
 * 2: norm gain 1 + U(-1/8, 1/8); 3: bias, sigma = 0.02.
 * u = top 24 bits of splitmix64(seed ^ tid<<40 ^ idx), centred: u - 2^23.
 * w = bf16_rne(offset + (float)u * c), c rounded once from double. */
void or_gen_tensor(uint64_t seed, uint32_t tid, int64_t n, int32_t kind, int32_t fan_in, uint16_t* out) {
  float c, offset = 0.0f;
  switch (kind) {
    case 0: c = (float)(sqrt(3.0 / (double)fan_in) / 8388608.0); break;
    case 1: c = (float)(sqrt(3.0) / 8388608.0); break;
    case 2: c = (float)(0.125 / 8388608.0); offset = 1.0f; break;
    default: c = (float)(0.02 * sqrt(3.0) / 8388608.0); break;
  }
#pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t r = or_splitmix64(seed ^ ((uint64_t)tid << 40) ^ (uint64_t)i);
    int32_t u = (int32_t)(r >> 40) - 8388608;
    float prod = (float)u * c;
    out[i] = or_f32_to_bf16(offset + prod);
  }
}

/* ------------------------------------------------------------------ */
/* Op-level reference functions.                                       */
/* ------------------------------------------------------------------ */

/* RMSNorm: ss = sum x^2 (fp32, left to right); inv = 1/sqrtf(ss/d + eps);
 * xn_j = bf16((x_j * inv) * w_j).  BASELINE.json north_star: "fixed
 * RMSNorm tree, fp32 accumulation" (the GPU's tree differs; tolerance). */
void or_rmsnorm(const uint16_t* x, const uint16_t* w, int32_t T, int32_t d, float eps, uint16_t* out) {
  for (int32_t t = 0; t < T; ++t) {
    const uint16_t* xr = x + (int64_t)t * d;
    float ss = 0.0f;
    for (int32_t j = 0; j < d; ++j) { float v = bf(xr[j]); ss = ss + v * v; }
    float mean = ss / (float)d;
    float inv = 1.0f / sqrtf(mean + eps);
    for (int32_t j = 0; j < d; ++j) out[(int64_t)t * d + j] = or_f32_to_bf16((bf(xr[j]) * inv) * bf(w[j]));
  }
}

/* out[t][n] = sum_k x[t][k] * W[n][k]  (y = x W^T), chunked_dot with `splits`. */
void or_gemm(const uint16_t* x, const uint16_t* W, int32_t T, int32_t N, int32_t K, int32_t splits, float* out) {
  for (int32_t t = 0; t < T; ++t) {
#pragma omp parallel for schedule(static) if ((int64_t)N * K > 262144)
    for (int32_t n = 0; n < N; ++n)
      out[(int64_t)t * N + n] = or_dot_bf16(x + (int64_t)t * K, W + (int64_t)n * K, K, splits);
  }
}

/* RoPE, rotate-half pairs (i, i + hd/2):
 * inv_freq_i = theta^(-2i/hd) and angle = pos * inv_freq_i in double,
 * cos/sin rounded once to fp32. */
void or_rope_table(int32_t hd, float theta, int32_t pos, float* cos_out, float* sin_out) {
  for (int32_t i = 0; i < hd / 2; ++i) {
    double inv_freq = pow((double)theta, -(2.0 * (double)i) / (double)hd);
    double ang = (double)pos * inv_freq;
    cos_out[i] = (float)cos(ang);
    sin_out[i] = (float)sin(ang);
  }
}

/* a' = a*c - b*s, b' = b*c + a*s on the fp32 accumulator, then bf16. */
static void rope_head(const float* acc, const float* cs, const float* sn, int32_t hd, uint16_t* out) {
  int32_t h2 = hd / 2;
  for (int32_t i = 0; i < h2; ++i) {
    float a = acc[i], b = acc[i + h2];
    float ac = a * cs[i], bs = b * sn[i], bc = b * cs[i], as = a * sn[i];
    out[i] = or_f32_to_bf16(ac - bs);
    out[i + h2] = or_f32_to_bf16(bc + as);
  }
}

/* QKV epilogue: acc (+ bias as an fp32 add) -> RoPE(q), RoPE(k), v -> bf16.
 * Row layout of acc: [q heads | k heads | v heads], each head hd wide. */
void or_qkv_epilogue(const float* acc, const uint16_t* bias, const int32_t* pos, int32_t T, int32_t H,
                     int32_t KV, int32_t hd, float theta, uint16_t* q, uint16_t* k, uint16_t* v) {
  int32_t NQ = H * hd, NK = KV * hd, N = NQ + 2 * NK;
  float* tmp = (float*)malloc(sizeof(float) * (size_t)N);
  float* cs = (float*)malloc(sizeof(float) * (size_t)hd);
  float* sn = (float*)malloc(sizeof(float) * (size_t)hd);
  for (int32_t t = 0; t < T; ++t) {
    for (int32_t n = 0; n < N; ++n) {
      float a = acc[(int64_t)t * N + n];
      tmp[n] = bias ? a + bf(bias[n]) : a;
    }
    or_rope_table(hd, theta, pos[t], cs, sn);
    for (int32_t h = 0; h < H; ++h) rope_head(tmp + h * hd, cs, sn, hd, q + (int64_t)t * NQ + h * hd);
    for (int32_t h = 0; h < KV; ++h) rope_head(tmp + NQ + h * hd, cs, sn, hd, k + (int64_t)t * NK + h * hd);
    for (int32_t n = 0; n < NK; ++n) v[(int64_t)t * NK + n] = or_f32_to_bf16(tmp[NQ + NK + n]);
  }
  free(tmp); free(cs); free(sn);
}

/* Decode attention for one query token over keys 0..n_keys-1, GQA group
 * G = H/KV (query head h reads kv head h/G).  Scores in fp32:
 * s_j = (q . k_j) * fp32(1/sqrt(hd)); per chunk m = max, e = expf(s - m),
 * l = sum e, acc = sum e*v (left to right); chunks combined in index order
 * with weights expf(m_c - m*); o = bf16(acc / l).  SURVEY 8(c) step 4. */
static void or_attention_stream(const uint16_t* q, const uint16_t* K, const uint16_t* V, int32_t H, int32_t KV,
                                int32_t hd, int32_t n, int32_t key_stride, int32_t split_keys, uint16_t* o);

void or_attention(const uint16_t* q, const uint16_t* K, const uint16_t* V, int32_t H, int32_t KV, int32_t hd,
                  int32_t n, int32_t key_stride, int32_t chunk, int32_t splits, uint16_t* o) {
  if (chunk < 0) {
    or_attention_stream(q, K, V, H, KV, hd, n, key_stride, -chunk, o);
    return;
  }
  int32_t G = H / KV;
  float scale = (float)(1.0 / sqrt((double)hd));
  int64_t nch;
  if (chunk > 0) nch = (n + chunk - 1) / chunk;
  else { nch = splits < 1 ? 1 : splits; if (nch > n) nch = n; }
  float* s = (float*)malloc(sizeof(float) * (size_t)n);
  float* mc = (float*)malloc(sizeof(float) * (size_t)nch);
  float* lc = (float*)malloc(sizeof(float) * (size_t)nch);
  float* ac = (float*)malloc(sizeof(float) * (size_t)nch * hd);
  for (int32_t h = 0; h < H; ++h) {
    int32_t g = h / G;
    const uint16_t* qh = q + (int64_t)h * hd;
    const uint16_t* Kg = K + (int64_t)g * key_stride * hd;
    const uint16_t* Vg = V + (int64_t)g * key_stride * hd;
    for (int32_t j = 0; j < n; ++j) s[j] = or_dot_bf16(qh, Kg + (int64_t)j * hd, hd, 1) * scale;
    for (int64_t c = 0; c < nch; ++c) {
      int64_t lo, hi;
      if (chunk > 0) { lo = c * chunk; hi = lo + chunk; if (hi > n) hi = n; }
      else { lo = chunk_start(n, nch, c); hi = chunk_start(n, nch, c + 1); }
      float m = -INFINITY;
      for (int64_t j = lo; j < hi; ++j) m = s[j] > m ? s[j] : m;
      float l = 0.0f;
      float* a = ac + c * hd;
      for (int32_t d = 0; d < hd; ++d) a[d] = 0.0f;
      for (int64_t j = lo; j < hi; ++j) {
        float e = expf(s[j] - m);
        l = l + e;
        for (int32_t d = 0; d < hd; ++d) a[d] = a[d] + e * bf(Vg[j * hd + d]);
      }
      mc[c] = m; lc[c] = l;
    }
    float ms = -INFINITY;
    for (int64_t c = 0; c < nch; ++c) ms = mc[c] > ms ? mc[c] : ms;
    float L = 0.0f;
    float* out = (float*)malloc(sizeof(float) * (size_t)hd);
    for (int32_t d = 0; d < hd; ++d) out[d] = 0.0f;
    for (int64_t c = 0; c < nch; ++c) {
      float w = expf(mc[c] - ms);
      L = L + lc[c] * w;
      for (int32_t d = 0; d < hd; ++d) out[d] = out[d] + ac[c * hd + d] * w;
    }
    for (int32_t d = 0; d < hd; ++d) o[(int64_t)h * hd + d] = or_f32_to_bf16(out[d] / L);
    free(out);
  }
  free(s); free(mc); free(lc); free(ac);
}

/* Streamed form of the same attention (reading A14): keys cut
 * into splits of split_keys; inside a split, 16-key blocks dealt round-robin
 * to 4 streams (block b -> stream b mod 4).  Each stream keeps a running
 * (m, l, a) from (-inf, 0, 0); per block, in order:
 *   m' = max(m, max_j s_j), alpha = expf(m - m'), e_j = expf(s_j - m'),
 *   l = l*alpha + sum_j e_j,  a = a*alpha + sum_j e_j v_j,  m = m'.
 * The 4 streams, then the splits, are combined in index order with weights
 * expf(m_i - max_i m_i); one split: o = bf16(a / l) directly. */
static void or_attention_stream(const uint16_t* q, const uint16_t* K, const uint16_t* V, int32_t H, int32_t KV,
                                int32_t hd, int32_t n, int32_t key_stride, int32_t split_keys, uint16_t* o) {
  int32_t G = H / KV;
  float scale = (float)(1.0 / sqrt((double)hd));
  int32_t nsp = (n + split_keys - 1) / split_keys;
  float* s = (float*)malloc(sizeof(float) * (size_t)n);
  float* sm = (float*)malloc(sizeof(float) * 4);
  float* sl = (float*)malloc(sizeof(float) * 4);
  float* sa = (float*)malloc(sizeof(float) * 4 * hd);
  float* pm = (float*)malloc(sizeof(float) * (size_t)nsp);
  float* pl = (float*)malloc(sizeof(float) * (size_t)nsp);
  float* pa = (float*)malloc(sizeof(float) * (size_t)nsp * hd);
  for (int32_t h = 0; h < H; ++h) {
    const uint16_t* Kg = K + (int64_t)(h / G) * key_stride * hd;
    const uint16_t* Vg = V + (int64_t)(h / G) * key_stride * hd;
    for (int32_t j = 0; j < n; ++j) s[j] = or_dot_bf16(q + (int64_t)h * hd, Kg + (int64_t)j * hd, hd, 1) * scale;
    for (int32_t sp = 0; sp < nsp; ++sp) {
      int32_t lo = sp * split_keys, hi = lo + split_keys < n ? lo + split_keys : n;
      int32_t nblk = (hi - lo + 15) / 16;
      for (int32_t w = 0; w < 4; ++w) {
        float m = -INFINITY, l = 0.0f;
        float* a = sa + w * hd;
        for (int32_t d = 0; d < hd; ++d) a[d] = 0.0f;
        for (int32_t b = w; b < nblk; b += 4) {
          int32_t j0 = lo + 16 * b, j1 = j0 + 16 < hi ? j0 + 16 : hi;
          float mn = m;
          for (int32_t j = j0; j < j1; ++j) mn = s[j] > mn ? s[j] : mn;
          float alpha = expf(m - mn);
          float lb = 0.0f;
          for (int32_t j = j0; j < j1; ++j) lb = lb + expf(s[j] - mn);
          l = l * alpha + lb;
          for (int32_t d = 0; d < hd; ++d) {
            float ab = 0.0f;
            for (int32_t j = j0; j < j1; ++j) ab = ab + expf(s[j] - mn) * bf(Vg[(int64_t)j * hd + d]);
            a[d] = a[d] * alpha + ab;
          }
          m = mn;
        }
        sm[w] = m; sl[w] = l;
      }
      float M = -INFINITY;
      for (int32_t w = 0; w < 4; ++w) M = sm[w] > M ? sm[w] : M;
      pl[sp] = 0.0f;
      for (int32_t d = 0; d < hd; ++d) pa[(int64_t)sp * hd + d] = 0.0f;
      for (int32_t w = 0; w < 4; ++w) {
        float wt = expf(sm[w] - M);
        pl[sp] = pl[sp] + sl[w] * wt;
        for (int32_t d = 0; d < hd; ++d) pa[(int64_t)sp * hd + d] = pa[(int64_t)sp * hd + d] + sa[w * hd + d] * wt;
      }
      pm[sp] = M;
    }
    if (nsp == 1) {
      for (int32_t d = 0; d < hd; ++d) o[(int64_t)h * hd + d] = or_f32_to_bf16(pa[d] / pl[0]);
      continue;
    }
    float M = -INFINITY, L = 0.0f;
    for (int32_t sp = 0; sp < nsp; ++sp) M = pm[sp] > M ? pm[sp] : M;
    for (int32_t sp = 0; sp < nsp; ++sp) L = L + pl[sp] * expf(pm[sp] - M);
    for (int32_t d = 0; d < hd; ++d) {
      float acc = 0.0f;
      for (int32_t sp = 0; sp < nsp; ++sp) acc = acc + pa[(int64_t)sp * hd + d] * expf(pm[sp] - M);
      o[(int64_t)h * hd + d] = or_f32_to_bf16(acc / L);
    }
  }
  free(s); free(sm); free(sl); free(sa); free(pm); free(pl); free(pa);
}

/* residual: out = bf16(x + acc) (one fp32 add). */
void or_residual(const uint16_t* x, const float* acc, int64_t n, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = or_f32_to_bf16(bf(x[i]) + acc[i]);
}

/* SwiGLU: a = bf16((g / (1 + expf(-g))) * u). */
void or_swiglu(const float* g, const float* u, int64_t n, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    float t = expf(-g[i]);
    float den = 1.0f + t;
    float sg = g[i] / den;
    out[i] = or_f32_to_bf16(sg * u[i]);
  }
}

/* Top-2 margin: g = l(1) - l(2).  Total order: value
 * descending, then id ascending; the second entry is the best
 * entry other than i1, so a duplicated maximum gives g = 0.
 * NaN ranks as -inf. */
void or_top2(const float* logits, int32_t T, int32_t V, float* v1, int32_t* i1, float* v2, int32_t* i2,
             float* g, int32_t* nan_flag) {
  for (int32_t t = 0; t < T; ++t) {
    const float* l = logits + (int64_t)t * V;
    float b1 = -INFINITY, b2 = -INFINITY;
    int32_t j1 = -1, j2 = -1;
    for (int32_t j = 0; j < V; ++j) {
      float x = l[j];
      if (x != x) { if (nan_flag) *nan_flag = 1; x = -INFINITY; }
      if (j1 < 0 || x > b1) { b2 = b1; j2 = j1; b1 = x; j1 = j; }
      else if (j2 < 0 || x > b2) { b2 = x; j2 = j; }
    }
    v1[t] = b1; i1[t] = j1; v2[t] = b2; i2[t] = j2;
    g[t] = b1 - b2;
  }
}

/* Threshold trigger, PAPER.md:201 ("triggers the verifier when g < tau"),
 * protected requests only; rows in ascending order.
 * DESIGN.md A4/A7: tau = 0 never fires (pure BF16, r_verify = 0) and
 * tau = +inf always fires (always-on, r_verify = 1) -- also for
 * a margin of +inf (second logit -inf); a NaN margin (every logit NaN, ranked
 * -inf) fires for any tau > 0. */
static int gate_fires(float g, float tau) {
  return tau > 0.0f && (g < tau || isinf(tau) || g != g);
}

int32_t or_gate(const float* g, const uint8_t* prot, int32_t B, float tau, int32_t* rows_out) {
  int32_t n = 0;
  for (int32_t b = 0; b < B; ++b)
    if (prot[b] && gate_fires(g[b], tau)) rows_out[n++] = b;
  return n;
}

/* ------------------------------------------------------------------ */
/* Model and state.                                                    */
/* ------------------------------------------------------------------ */
struct or_model {
  or_cfg c;
  uint16_t* embed;     /* [V][d] */
  uint16_t* final_norm;
  uint16_t* lm;        /* [V][d] */
  uint16_t** layer_t;  /* [L*12] */
  int64_t* layer_n;    /* [L*12] */
};

static int64_t layer_tensor_numel(const or_cfg* c, int32_t which, int32_t* kind, int32_t* fan_in) {
  int64_t d = c->d_model, qd = (int64_t)c->n_heads * c->head_dim, kd = (int64_t)c->n_kv_heads * c->head_dim;
  int64_t f = c->d_ff;
  switch (which) {
    case 0: case 5: *kind = 2; *fan_in = 0; return d;
    case 1: *kind = 0; *fan_in = (int32_t)d; return qd * d;
    case 2: case 3: *kind = 0; *fan_in = (int32_t)d; return kd * d;
    case 4: *kind = 0; *fan_in = (int32_t)qd; return d * qd;
    case 6: case 7: *kind = 0; *fan_in = (int32_t)d; return f * d;
    case 8: *kind = 0; *fan_in = (int32_t)f; return d * f;
    case 9: *kind = 3; *fan_in = 0; return c->qkv_bias ? qd : 0;
    case 10: case 11: *kind = 3; *fan_in = 0; return c->qkv_bias ? kd : 0;
  }
  return 0;
}

or_model* or_model_create(const or_cfg* cfg) {
  or_model* m = (or_model*)calloc(1, sizeof(or_model));
  m->c = *cfg;
  int64_t V = cfg->vocab, d = cfg->d_model;
  int32_t L = cfg->n_layers;
  m->embed = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(V * d));
  or_gen_tensor(cfg->weight_seed, or_tensor_id(cfg, -1, 0), V * d, 1, 0, m->embed);
  m->final_norm = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)d);
  or_gen_tensor(cfg->weight_seed, or_tensor_id(cfg, -1, 1), d, 2, 0, m->final_norm);
  m->lm = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(V * d));
  or_gen_tensor(cfg->weight_seed, or_tensor_id(cfg, -1, 2), V * d, 0, (int32_t)d, m->lm);
  m->layer_t = (uint16_t**)calloc((size_t)L * 12, sizeof(uint16_t*));
  m->layer_n = (int64_t*)calloc((size_t)L * 12, sizeof(int64_t));
  for (int32_t l = 0; l < L; ++l)
    for (int32_t w = 0; w < 12; ++w) {
      int32_t kind, fan_in;
      int64_t n = layer_tensor_numel(cfg, w, &kind, &fan_in);
      m->layer_n[l * 12 + w] = n;
      if (n == 0) continue;
      m->layer_t[l * 12 + w] = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
      or_gen_tensor(cfg->weight_seed, or_tensor_id(cfg, l, w), n, kind, fan_in, m->layer_t[l * 12 + w]);
    }
  return m;
}

void or_model_free(or_model* m) {
  if (!m) return;
  free(m->embed); free(m->final_norm); free(m->lm);
  for (int32_t i = 0; i < m->c.n_layers * 12; ++i) free(m->layer_t[i]);
  free(m->layer_t); free(m->layer_n); free(m);
}

const uint16_t* or_model_tensor(const or_model* m, int32_t layer, int32_t which, int64_t* n_out) {
  if (layer < 0) {
    int64_t V = m->c.vocab, d = m->c.d_model;
    if (which == 0) { if (n_out) *n_out = V * d; return m->embed; }
    if (which == 1) { if (n_out) *n_out = d; return m->final_norm; }
    if (n_out) *n_out = V * d;
    return m->lm;
  }
  if (n_out) *n_out = m->layer_n[layer * 12 + which];
  return m->layer_t[layer * 12 + which];
}

struct or_state {
  const or_model* m;
  int32_t n_rows, max_seq;
  uint16_t* kv[2];      /* [which: 0 fast, 1 shadow] -> [row][L][2][KV][max_seq][hd] */
  int32_t* hist;        /* [row][max_seq + 1]: committed token consumed at position q */
  int32_t* pos;         /* next decode position p (= columns in the fast cache) */
  int32_t* shadow_len;  /* columns of the shadow cache that are final */
  int32_t repair_mode;  /* 0 column repair, 1 token-only ablation */
  uint64_t stats[9];
  uint64_t wstats[3];   /* window verifies (rows), rollbacks, rolled-back tokens */
};

static inline int64_t kv_index(const or_state* s, int32_t row, int32_t l, int32_t kvsel, int32_t h, int32_t q) {
  const or_cfg* c = &s->m->c;
  return ((((int64_t)row * c->n_layers + l) * 2 + kvsel) * c->n_kv_heads + h) * (int64_t)s->max_seq * c->head_dim +
         (int64_t)q * c->head_dim;
}

or_state* or_state_create(const or_model* m, int32_t n_rows, int32_t max_seq) {
  or_state* s = (or_state*)calloc(1, sizeof(or_state));
  const or_cfg* c = &m->c;
  s->m = m; s->n_rows = n_rows; s->max_seq = max_seq;
  size_t nkv = (size_t)n_rows * c->n_layers * 2 * c->n_kv_heads * (size_t)max_seq * c->head_dim;
  s->kv[0] = (uint16_t*)calloc(nkv, sizeof(uint16_t));
  s->kv[1] = (uint16_t*)calloc(nkv, sizeof(uint16_t));
  s->hist = (int32_t*)calloc((size_t)n_rows * (max_seq + 1), sizeof(int32_t));
  s->pos = (int32_t*)calloc((size_t)n_rows, sizeof(int32_t));
  s->shadow_len = (int32_t*)calloc((size_t)n_rows, sizeof(int32_t));
  return s;
}

void or_state_free(or_state* s) {
  if (!s) return;
  free(s->kv[0]); free(s->kv[1]); free(s->hist); free(s->pos); free(s->shadow_len); free(s);
}

/* One token of the decoder forward for `row` at
 * position q consuming token `tok`, reading and writing cache `which`
 * (0 fast, 1 shadow).  Appends this token's K/V column at q ("tentatively
 * appends the current token and K/V column"), attends keys
 * 0..q, and if logits != NULL writes the fp32 LM-head logits [V]. */
static void forward_token(or_state* s, int32_t which, int32_t row, int32_t q, int32_t tok, const or_sched* sc,
                          float* logits) {
  const or_model* m = s->m;
  const or_cfg* c = &m->c;
  int32_t d = c->d_model, H = c->n_heads, KV = c->n_kv_heads, hd = c->head_dim, F = c->d_ff;
  int32_t NQ = H * hd, NK = KV * hd, NQKV = NQ + 2 * NK;
  uint16_t* x = (uint16_t*)malloc(sizeof(uint16_t) * d);
  uint16_t* xn = (uint16_t*)malloc(sizeof(uint16_t) * d);
  float* acc = (float*)malloc(sizeof(float) * (size_t)(NQKV > 2 * F ? NQKV : 2 * F) + sizeof(float) * d);
  uint16_t* qv = (uint16_t*)malloc(sizeof(uint16_t) * NQ);
  uint16_t* kc = (uint16_t*)malloc(sizeof(uint16_t) * NK);
  uint16_t* vc = (uint16_t*)malloc(sizeof(uint16_t) * NK);
  uint16_t* att = (uint16_t*)malloc(sizeof(uint16_t) * NQ);
  uint16_t* a = (uint16_t*)malloc(sizeof(uint16_t) * F);

  memcpy(x, m->embed + (int64_t)tok * d, sizeof(uint16_t) * d);           /* a1: embed */
  for (int32_t l = 0; l < c->n_layers; ++l) {
    const uint16_t* const* T = (const uint16_t* const*)(m->layer_t + l * 12);
    or_rmsnorm(x, T[0], 1, d, c->rms_eps, xn);                            /* a2 */
    or_gemm(xn, T[1], 1, NQ, d, sc->split_qkv, acc);                      /* a3: q|k|v */
    or_gemm(xn, T[2], 1, NK, d, sc->split_qkv, acc + NQ);
    or_gemm(xn, T[3], 1, NK, d, sc->split_qkv, acc + NQ + NK);
    uint16_t* bias = NULL;
    if (c->qkv_bias) {
      bias = (uint16_t*)malloc(sizeof(uint16_t) * NQKV);
      memcpy(bias, T[9], sizeof(uint16_t) * NQ);
      memcpy(bias + NQ, T[10], sizeof(uint16_t) * NK);
      memcpy(bias + NQ + NK, T[11], sizeof(uint16_t) * NK);
    }
    or_qkv_epilogue(acc, bias, &q, 1, H, KV, hd, c->rope_theta, qv, kc, vc);
    free(bias);
    for (int32_t h = 0; h < KV; ++h) {                                     /* append column q */
      memcpy(s->kv[which] + kv_index(s, row, l, 0, h, q), kc + h * hd, sizeof(uint16_t) * hd);
      memcpy(s->kv[which] + kv_index(s, row, l, 1, h, q), vc + h * hd, sizeof(uint16_t) * hd);
    }
    or_attention(qv, s->kv[which] + kv_index(s, row, l, 0, 0, 0), s->kv[which] + kv_index(s, row, l, 1, 0, 0), H,
                 KV, hd, q + 1, s->max_seq, sc->attn_chunk, sc->attn_splits, att);        /* a4 */
    or_gemm(att, T[4], 1, d, NQ, sc->split_o, acc);                       /* a5: O + residual */
    or_residual(x, acc, d, x);
    or_rmsnorm(x, T[5], 1, d, c->rms_eps, xn);
    or_gemm(xn, T[6], 1, F, d, sc->split_gu, acc);                        /* a6: gate/up + SwiGLU */
    or_gemm(xn, T[7], 1, F, d, sc->split_gu, acc + F);
    or_swiglu(acc, acc + F, F, a);
    or_gemm(a, T[8], 1, d, F, sc->split_down, acc);                       /* a7: down + residual */
    or_residual(x, acc, d, x);
  }
  if (logits) {                                                            /* a8: final norm + LM head */
    or_rmsnorm(x, m->final_norm, 1, d, c->rms_eps, xn);
    or_gemm(xn, m->lm, 1, c->vocab, d, sc->split_lm, logits);
  }
  free(x); free(xn); free(acc); free(qv); free(kc); free(vc); free(att); free(a);
}

static void copy_column(or_state* s, int32_t from, int32_t to, int32_t row, int32_t q) {
  const or_cfg* c = &s->m->c;
  for (int32_t l = 0; l < c->n_layers; ++l)
    for (int32_t kvsel = 0; kvsel < 2; ++kvsel)
      for (int32_t h = 0; h < c->n_kv_heads; ++h) {
        int64_t i = kv_index(s, row, l, kvsel, h, q);
        memcpy(s->kv[to] + i, s->kv[from] + i, sizeof(uint16_t) * c->head_dim);
      }
}

int32_t or_prefill(or_state* s, int32_t row, const int32_t* prompt, int32_t len, const or_sched* det,
                   float* logits_out) {
  const or_cfg* c = &s->m->c;
  float* logits = (float*)malloc(sizeof(float) * (size_t)c->vocab);
  int32_t* h = s->hist + (int64_t)row * (s->max_seq + 1);
  for (int32_t q = 0; q < len; ++q) {
    h[q] = prompt[q];
    forward_token(s, 1, row, q, prompt[q], det, q == len - 1 ? logits : NULL);
  }
  for (int32_t q = 0; q < len; ++q) copy_column(s, 1, 0, row, q);
  float v1, v2, g; int32_t i1, i2, nan = 0;
  or_top2(logits, 1, c->vocab, &v1, &i1, &v2, &i2, &g, &nan);
  if (nan) s->stats[8] += 1;
  if (logits_out) memcpy(logits_out, logits, sizeof(float) * (size_t)c->vocab);
  h[len] = i1;
  s->pos[row] = len;
  s->shadow_len[row] = len;
  free(logits);
  return i1;
}

/* SPEC.md:76-84 injected perturbation: exactly zero at batch 1. */
static void inject_noise(float* logits, int32_t V, const or_sched* sc, int32_t B, int32_t row, int32_t pos) {
  if (!(sc->noise_amp > 0.0f) || B <= 1) return;
  for (int32_t v = 0; v < V; ++v) {
    uint64_t r = or_splitmix64(sc->noise_seed ^ ((uint64_t)B << 56) ^ ((uint64_t)row << 44) ^
                               ((uint64_t)pos << 20) ^ (uint64_t)v);
    int32_t u = (int32_t)(r >> 40) - 8388608;
    logits[v] = logits[v] + sc->noise_amp * ((float)u * (float)(1.0 / 8388608.0));
  }
}

int32_t or_step(or_state* s, const int32_t* rows, int32_t B, const uint8_t* prot, float tau,
                const or_sched* fast, const or_sched* det, const uint8_t* forced_trig, const int32_t* forced_out,
                const uint8_t* forced_kind, int32_t* f_tok, float* g, float* fv1, float* fv2, uint8_t* trig,
                int32_t* v_tok, float* v_g, uint8_t* kind, int32_t* out_tok, float* fast_logits) {
  const or_cfg* c = &s->m->c;
  int32_t V = c->vocab;
  float* logits = (float*)malloc(sizeof(float) * (size_t)V);
  int32_t* ft = (int32_t*)malloc(sizeof(int32_t) * B);
  float* gg = (float*)malloc(sizeof(float) * B);
  uint8_t* tr = (uint8_t*)calloc((size_t)B, 1);
  int32_t nan = 0;

  /* (1) BF16 batched fast step + fused top-2. */
  for (int32_t b = 0; b < B; ++b) {
    int32_t r = rows[b], p = s->pos[r];
    int32_t tok = s->hist[(int64_t)r * (s->max_seq + 1) + p];
    forward_token(s, 0, r, p, tok, fast, logits);
    inject_noise(logits, V, fast, B, r, p);
    if (fast_logits) memcpy(fast_logits + (int64_t)b * V, logits, sizeof(float) * V);
    float v1, v2; int32_t i1, i2;
    or_top2(logits, 1, V, &v1, &i1, &v2, &i2, &gg[b], &nan);
    ft[b] = i1;
    if (f_tok) f_tok[b] = i1;
    if (g) g[b] = gg[b];
    if (fv1) fv1[b] = v1;
    if (fv2) fv2[b] = v2;
  }
  /* (2) gate + compaction. */
  int32_t n_trig = 0;
  for (int32_t b = 0; b < B; ++b) {
    tr[b] = forced_trig ? forced_trig[b] : (uint8_t)(prot[b] && gate_fires(gg[b], tau));
    n_trig += tr[b];
    if (trig) trig[b] = tr[b];
  }
  /* (3) deterministic verifier on the gated rows, ascending:
   * catch the row's shadow cache up over shadow_len..p with the det schedule
   * and take the argmax at p. */
  int32_t* vt = (int32_t*)malloc(sizeof(int32_t) * B);
  for (int32_t b = 0; b < B; ++b) {
    vt[b] = -1;
    if (v_tok) v_tok[b] = -1;
    if (v_g) v_g[b] = 0.0f;
    if (!tr[b]) continue;
    int32_t r = rows[b], p = s->pos[r];
    int32_t* h = s->hist + (int64_t)r * (s->max_seq + 1);
    for (int32_t q = s->shadow_len[r]; q <= p; ++q) {
      forward_token(s, 1, r, q, h[q], det, q == p ? logits : NULL);
      s->stats[7] += 1;
    }
    s->shadow_len[r] = p + 1;
    float v1, v2, gv; int32_t i1, i2;
    or_top2(logits, 1, V, &v1, &i1, &v2, &i2, &gv, &nan);
    vt[b] = i1;
    if (v_tok) v_tok[b] = i1;
    if (v_g) v_g[b] = gv;
  }
  if (n_trig > 0) s->stats[6] += 1;
  /* (4) commit: fast | verified | repair of the single column p. */
  for (int32_t b = 0; b < B; ++b) {
    int32_t r = rows[b], p = s->pos[r];
    uint8_t k;
    int32_t out;
    if (forced_out) {
      out = forced_out[b];
      k = forced_kind ? forced_kind[b] : (uint8_t)(tr[b] ? (vt[b] == ft[b] ? 1 : 2) : 0);
    } else if (!tr[b]) { k = 0; out = ft[b]; }
    else if (vt[b] == ft[b]) { k = 1; out = ft[b]; }
    else { k = 2; out = vt[b]; }
    if (k == 2 && s->repair_mode == 0) copy_column(s, 1, 0, r, p);
    s->hist[(int64_t)r * (s->max_seq + 1) + p + 1] = out;
    s->pos[r] = p + 1;
    if (kind) kind[b] = k;
    if (out_tok) out_tok[b] = out;
    s->stats[1] += 1;
    s->stats[2] += prot[b] ? 1 : 0;
    s->stats[4] += k == 1;
    s->stats[5] += k == 2;
  }
  s->stats[0] += 1;
  s->stats[3] += (uint64_t)n_trig;
  if (nan) s->stats[8] += 1;
  free(logits); free(ft); free(gg); free(tr); free(vt);
  return n_trig;
}

int32_t or_state_pos(const or_state* s, int32_t row) { return s->pos[row]; }
int32_t or_state_shadow_len(const or_state* s, int32_t row) { return s->shadow_len[row]; }
int32_t or_state_token(const or_state* s, int32_t row, int32_t q) { return s->hist[(int64_t)row * (s->max_seq + 1) + q]; }

void or_state_column(const or_state* s, int32_t which, int32_t row, int32_t pos, uint16_t* out) {
  const or_cfg* c = &s->m->c;
  int64_t o = 0;
  for (int32_t l = 0; l < c->n_layers; ++l)
    for (int32_t kvsel = 0; kvsel < 2; ++kvsel)
      for (int32_t h = 0; h < c->n_kv_heads; ++h) {
        memcpy(out + o, s->kv[which] + kv_index(s, row, l, kvsel, h, pos), sizeof(uint16_t) * c->head_dim);
        o += c->head_dim;
      }
}

uint64_t or_state_digest(const or_state* s, int32_t which, int32_t skip_row, int32_t skip_pos) {
  const or_cfg* c = &s->m->c;
  uint64_t hsh = 1469598103934665603ull;
  for (int32_t r = 0; r < s->n_rows; ++r)
    for (int32_t l = 0; l < c->n_layers; ++l)
      for (int32_t kvsel = 0; kvsel < 2; ++kvsel)
        for (int32_t h = 0; h < c->n_kv_heads; ++h)
          for (int32_t q = 0; q < s->max_seq; ++q) {
            if (r == skip_row && q == skip_pos) continue;
            const uint16_t* p = s->kv[which] + kv_index(s, r, l, kvsel, h, q);
            for (int32_t d = 0; d < c->head_dim; ++d) {
              hsh ^= p[d];
              hsh *= 1099511628211ull;
            }
          }
  return hsh;
}

void or_state_stats(const or_state* s, uint64_t* out9) { memcpy(out9, s->stats, sizeof(s->stats)); }

/* Repair-action ablation (S4.4 "Repair-action ablation"): mode 1
 * emits the verifier token but leaves the tentative BF16 K/V column in place
 * ("token-only"); mode 0 (default) copies the verifier-produced column. */
void or_state_set_repair_mode(or_state* s, int32_t mode) { s->repair_mode = mode; }

/* LLM-42-style windowed verification with rollback ("keeps the
 * default path but verifies every token", "verifier setting
 * K=64", "restart-from-rollback"), in the
 * shadow-cache reading A1.  For each row r in rows[0..n):
 *   the tokens committed since the last verification, hist[shadow_len+1..pos],
 *   are checked in order: for q = shadow_len .. pos-1 the deterministic
 *   forward consumes hist[q] at position q (shadow cache) and its argmax v
 *   predicts position q+1.  At the first q with v != hist[q+1] the row rolls
 *   back: hist[q+1] = v, pos = shadow_len = q+1 (the tokens after q+1 are
 *   discarded; fast columns >= q+1 are rewritten by later steps).  Without a
 *   mismatch shadow_len = pos.
 * Outputs (nullable): new_pos[i] = pos after the call, last_tok[i] =
 * hist[new_pos], rolled_back[i] = tokens discarded.  Returns the total number
 * of discarded tokens. */
int32_t or_verify_window(or_state* s, const int32_t* rows, int32_t n, const or_sched* det, int32_t* new_pos,
                         int32_t* last_tok, int32_t* rolled_back) {
  const or_cfg* c = &s->m->c;
  float* logits = (float*)malloc(sizeof(float) * (size_t)c->vocab);
  int32_t total = 0;
  for (int32_t i = 0; i < n; ++i) {
    int32_t r = rows[i], p = s->pos[r], rb = 0;
    int32_t* h = s->hist + (int64_t)r * (s->max_seq + 1);
    for (int32_t q = s->shadow_len[r]; q < p; ++q) {
      forward_token(s, 1, r, q, h[q], det, logits);
      s->stats[7] += 1;
      float v1, v2, g; int32_t i1, i2, nan = 0;
      or_top2(logits, 1, c->vocab, &v1, &i1, &v2, &i2, &g, &nan);
      if (nan) s->stats[8] += 1;
      if (i1 != h[q + 1]) {      /* first disagreement: roll back to q+1 */
        rb = p - (q + 1);
        h[q + 1] = i1;
        p = q + 1;
        s->pos[r] = p;
        s->wstats[1] += 1;
        break;
      }
    }
    s->shadow_len[r] = p;
    s->wstats[0] += 1;
    s->wstats[2] += (uint64_t)rb;
    total += rb;
    if (new_pos) new_pos[i] = p;
    if (last_tok) last_tok[i] = h[p];
    if (rolled_back) rolled_back[i] = rb;
  }
  free(logits);
  return total;
}

void or_state_window_stats(const or_state* s, uint64_t* out3) { memcpy(out3, s->wstats, sizeof(s->wstats)); }
