/*
 * spmoe_oracle.c — CPU ORACLE for the SP-MoE verification-time expert path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, as
 * the checker (or as the timed CPU restatement of the reference path).  The
 * product path (paper_2510_10302_b200) never links or calls it.
 *
 * What it restates
 *   The reference package `moesim` contains no tensor arithmetic (SPEC.md:9,
 *   pkg/README.md:12-15), so the tensor half of the path is restated from the
 *   paper and pinned to the reference only where the reference has code:
 *     - top-k ordering (logit desc, index asc) = trace.top_k_indices
 *       (trace.py:28-37) / predictor.select_critical (predictor.py:100-106);
 *     - router projection of the draft hidden state = Algorithm 1 l.2-3
 *       Gates[l](s), TopK_Index;
 *     - expert SwiGLU E_i(x) and the gated sum of Eq. 1;
 *     - greedy acceptance: longest prefix + one correction/bonus token
 *       (PAPER.md:65,162), the deterministic counterpart of the Bernoulli
 *       acceptance in simcore.py:440-446.
 *   Parity for router logits, SwiGLU, combine and target logits is therefore
 *   anchored on the fixed-order arithmetic contract of include/spmoe.h rather
 *   than on reference golden vectors (SURVEY.md §8(c) "parity unpinned"
 *   list); top-k tie-break is pinned to the reference's own known answers
 *   (test_trace.py:41-43, test_predictor.py:57-70) in tests/.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, pthreads; parallel
 * loops on the persistent pool of oracle/pool.c).  No
 * FMA contraction, no fast-math: every float operation is an IEEE
 * round-to-nearest single-precision op in the order written.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "pool.h"

/* parallel loops: oracle/pool.c (persistent workers, contiguous spans) */
#define parallel_for oracle_parallel_for
typedef oracle_row_fn row_fn;

/* ------------------------------------------------------------------ */
/* scalar helpers                                                       */
/* ------------------------------------------------------------------ */
static inline float bf2f(uint16_t v) {
  union { uint32_t u; float f; } c;
  c.u = ((uint32_t)v) << 16;
  return c.f;
}

static inline uint16_t f2bf(float f) {
  union { uint32_t u; float f; } c;
  c.f = f;
  uint32_t u = c.u;
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static inline float u2f(uint32_t u) {
  union { uint32_t u; float f; } c;
  c.u = u;
  return c.f;
}

/* Deterministic exp: same constants and op order as spmoe_common.cuh. */
float oracle_det_exp(float x) {
  if (x < -86.0f) return 0.0f;
  if (x > 88.0f) return u2f(0x7f800000u);
  const float n = rintf(x * 1.44269504f);
  float r = x - n * 0.693145752f;
  r = r - n * 1.42860677e-06f;
  float p = 1.98412698e-04f;
  p = p * r + 1.38888889e-03f;
  p = p * r + 8.33333333e-03f;
  p = p * r + 4.16666667e-02f;
  p = p * r + 1.66666667e-01f;
  p = p * r + 0.5f;
  p = p * r + 1.0f;
  p = p * r + 1.0f;
  const int ni = (int)n;
  return p * u2f((uint32_t)(ni + 127) << 23);
}

float oracle_det_silu(float g) { return g / (1.0f + oracle_det_exp(-g)); }

/*
 * Fixed-order dot product of two bf16 vectors of length n (n % 8 == 0):
 * lane j (0..31) accumulates chunks c = j, j+32, ... ascending, elements
 * 0..7 of each chunk in order; then the xor-butterfly 16,8,4,2,1, whose
 * lane-0 value is the pairwise tree below.
 */
float oracle_dot_fixed(const uint16_t* a, const uint16_t* b, int n) {
  float lane[32] = {0};
  const int nch = n / 8;
  /* chunk groups outer, lanes inner: each lane still sees its chunks in
   * ascending order, but the 32 short chains overlap in the pipeline */
  for (int c0 = 0; c0 < nch; c0 += 32) {
    for (int j = 0; j < 32 && c0 + j < nch; ++j) {
      const uint16_t* pa = a + 8 * (c0 + j);
      const uint16_t* pb = b + 8 * (c0 + j);
      float acc = lane[j];
      for (int v = 0; v < 8; ++v) acc = acc + bf2f(pa[v]) * bf2f(pb[v]);
      lane[j] = acc;
    }
  }
  for (int w = 16; w >= 1; w >>= 1)
    for (int j = 0; j < w; ++j) lane[j] = lane[j] + lane[j + w];
  return lane[0];
}

/* ------------------------------------------------------------------ */
/* K1 router_topk                                                       */
/* ------------------------------------------------------------------ */
void oracle_router_topk(const uint16_t* x, const uint16_t* wg, int T, int H, int E, int k,
                        int renorm, float* weights, int32_t* idx, float* logits,
                        const uint16_t* sg_w, float* sg_out) {
  float* lg = (float*)malloc(sizeof(float) * (size_t)(E > 0 ? E : 1));
  int* taken = (int*)malloc(sizeof(int) * (size_t)(E > 0 ? E : 1));
  int* sel = (int*)malloc(sizeof(int) * (size_t)(k > 0 ? k : 1));
  for (int t = 0; t < T; ++t) {
    const uint16_t* xt = x + (size_t)t * H;
    for (int e = 0; e < E; ++e) lg[e] = oracle_dot_fixed(xt, wg + (size_t)e * H, H);
    if (logits)
      for (int e = 0; e < E; ++e) logits[(size_t)t * E + e] = lg[e];
    if (sg_w && sg_out) sg_out[t] = 1.0f / (1.0f + oracle_det_exp(-oracle_dot_fixed(xt, sg_w, H)));
    memset(taken, 0, sizeof(int) * (size_t)E);
    for (int i = 0; i < k; ++i) {
      int best = -1;
      float bv = 0.0f;
      for (int e = 0; e < E; ++e) {
        if (taken[e]) continue;
        if (best < 0 || lg[e] > bv) { best = e; bv = lg[e]; }
      }
      sel[i] = best;
      taken[best] = 1;
    }
    const float m = lg[sel[0]];
    float sum = 0.0f;
    if (renorm) {
      for (int i = 0; i < k; ++i) sum = sum + oracle_det_exp(lg[sel[i]] - m);
    } else {
      for (int e = 0; e < E; ++e) sum = sum + oracle_det_exp(lg[e] - m);
    }
    for (int i = 0; i < k; ++i) {
      weights[(size_t)t * k + i] = oracle_det_exp(lg[sel[i]] - m) / sum;
      idx[(size_t)t * k + i] = sel[i];
    }
  }
  free(lg);
  free(taken);
  free(sel);
}

/* ------------------------------------------------------------------ */
/* K2 permute                                                           */
/* ------------------------------------------------------------------ */
void oracle_moe_permute(const int32_t* idx, int T, int k, int E, int32_t* offsets,
                        int32_t* perm_token, int32_t* inv_pos) {
  const int n = T * k;
  int acc = 0;
  for (int e = 0; e < E; ++e) {
    offsets[e] = acc;
    for (int j = 0; j < n; ++j)
      if (idx[j] == e) {
        perm_token[acc] = j / k;
        inv_pos[j] = acc;
        ++acc;
      }
  }
  offsets[E] = acc;
}

/* ------------------------------------------------------------------ */
/* K3 expert SwiGLU over per-expert blobs W1[F,H] | W3[F,H] | W2[H,F]   */
/* ------------------------------------------------------------------ */
/*
 * blobs[e] -> expert e's blob (NULL = expert not computed); rows of y for
 * experts with a NULL blob are left untouched.  h_out [T*k, F] bf16 and
 * y [T*k, H] f32 use the permuted row order of oracle_moe_permute.
 */
typedef struct {
  const uint16_t *w1, *w3, *w2, *x;
  const int32_t* perm;
  uint16_t* h_out;
  float* y;
  int H, F, o0, o1;
} ffn_ctx;

static void ffn_up_row(void* c, int64_t f) {
  ffn_ctx* p = (ffn_ctx*)c;
  for (int q = p->o0; q < p->o1; ++q) {
    const uint16_t* xt = p->x + (size_t)p->perm[q] * p->H;
    const float g = oracle_dot_fixed(p->w1 + (size_t)f * p->H, xt, p->H);
    const float u = oracle_dot_fixed(p->w3 + (size_t)f * p->H, xt, p->H);
    p->h_out[(size_t)q * p->F + f] = f2bf(oracle_det_silu(g) * u);
  }
}

static void ffn_down_row(void* c, int64_t hr) {
  ffn_ctx* p = (ffn_ctx*)c;
  for (int q = p->o0; q < p->o1; ++q)
    p->y[(size_t)q * p->H + hr] =
        oracle_dot_fixed(p->w2 + (size_t)hr * p->F, p->h_out + (size_t)q * p->F, p->F);
}

void oracle_expert_ffn(const uint16_t* const* blobs, const uint16_t* x, int T, int H, int F,
                       int E, const int32_t* offsets, const int32_t* perm_token, uint16_t* h_out,
                       float* y) {
  (void)T;
  for (int e = 0; e < E; ++e) {
    const uint16_t* blob = blobs[e];
    const int o0 = offsets[e], o1 = offsets[e + 1];
    if (!blob || o1 <= o0) continue;
    ffn_ctx c = {blob, blob + (size_t)F * H, blob + 2 * (size_t)F * H, x, perm_token,
                 h_out, y, H, F, o0, o1};
    parallel_for(F, ffn_up_row, &c);
    parallel_for(H, ffn_down_row, &c);
  }
}

/* ------------------------------------------------------------------ */
/* K4 combine                                                           */
/* ------------------------------------------------------------------ */
void oracle_moe_combine(const float* y, const int32_t* inv_pos, const float* w, int T, int H,
                        int k, const float* ys, const float* sg, const uint16_t* residual,
                        uint16_t* out) {
  for (int t = 0; t < T; ++t)
    for (int h = 0; h < H; ++h) {
      float acc = 0.0f;
      for (int i = 0; i < k; ++i) {
        const int pos = inv_pos[t * k + i];
        if (pos < 0) continue;
        const float wi = w ? w[t * k + i] : 1.0f;
        const float prod = wi * y[(size_t)pos * H + h];
        acc = acc + prod;
      }
      if (ys) {
        const float g = sg ? sg[t] : 1.0f;
        const float prod = g * ys[(size_t)t * H + h];
        acc = acc + prod;
      }
      if (residual) {
        const float r = bf2f(residual[(size_t)t * H + h]);
        out[(size_t)t * H + h] = f2bf(r + acc);
      } else {
        out[(size_t)t * H + h] = f2bf(acc);
      }
    }
}

/* ------------------------------------------------------------------ */
/* K6 greedy acceptance                                                 */
/* ------------------------------------------------------------------ */
static inline int better(float v, int i, float bv, int bi) {
  if (v != v) return 0;
  if (bv != bv) return 1;
  return (v > bv) || (v == bv && i < bi);
}

void oracle_argmax_rows(const float* logits, int64_t ld, int rows, int V, int32_t* out) {
  for (int r = 0; r < rows; ++r) {
    const float* row = logits + (size_t)r * ld;
    float bv = u2f(0x7fc00000u);
    int bi = 0x7fffffff;
    for (int i = 0; i < V; ++i)
      if (better(row[i], i, bv, bi)) { bv = row[i]; bi = i; }
    out[r] = (bi == 0x7fffffff) ? 0 : bi;
  }
}

void oracle_greedy_accept(const float* logits, int64_t ld, const int32_t* draft, int B, int N,
                          int V, int32_t* amax, int32_t* result) {
  oracle_argmax_rows(logits, ld, B * (N + 1), V, amax);
  for (int b = 0; b < B; ++b) {
    int a = 0;
    while (a < N && draft[b * N + a] == amax[b * (N + 1) + a]) ++a;
    result[2 * b] = a;
    result[2 * b + 1] = amax[b * (N + 1) + a];
  }
}

/* ------------------------------------------------------------------ */
/* deterministic init (splitmix64 counter hash, Irwin-Hall(4))          */
/* ------------------------------------------------------------------ */
static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct {
  uint16_t* dst;
  uint64_t seed, offset;
  float scale;
  int64_t n, block;
} fill_ctx;

static void fill_block(void* c, int64_t b) {
  fill_ctx* p = (fill_ctx*)c;
  const int64_t lo = b * p->block;
  int64_t hi = lo + p->block;
  if (hi > p->n) hi = p->n;
  for (int64_t i = lo; i < hi; ++i) {
    const uint64_t h = splitmix64(p->seed ^ splitmix64(p->offset + (uint64_t)i));
    const int s = (int)(h & 0xffff) + (int)((h >> 16) & 0xffff) + (int)((h >> 32) & 0xffff) +
                  (int)(h >> 48);
    p->dst[i] = f2bf((float)(s - 131070) * p->scale);
  }
}

void oracle_fill_normal_bf16(uint16_t* dst, int64_t n, uint64_t seed, uint64_t offset,
                             float std) {
  fill_ctx c = {dst, seed, offset, std * 0x1.bb67aep-16f, n, 1 << 16};
  parallel_for((n + c.block - 1) / c.block, fill_block, &c);
}
