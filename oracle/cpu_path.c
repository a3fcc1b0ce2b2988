/*
 * cpu_path.c — the SP-MoE draft/verify forward on the host cores: the CPU
 * restatement that bench.py times as the reference arm / cpu_baseline, and
 * that the end-to-end parity tests run as the oracle of the whole SD loop.
 *
 * TEST INFRASTRUCTURE ONLY (see spmoe_oracle.c).  Same determinism contract
 * as the kernels and the scalar oracles (spmoe_oracle.c, forward_oracle.c),
 * only laid out for SIMD: weight rows are stored LANE-MAJOR ("LM"), so the
 * 32 fixed-order lane accumulators of one dot product become two 16-wide
 * vectors:
 *
 *   raw row   w[k], k = 256 g + 8 j + v     (lane j, chunk 32 g + j, elem v)
 *   LM row    wl[256 g + 32 v + j] = w[256 g + 8 j + v]   (zero-padded to
 *             Kp = 256 * ceil(K / 256))
 *
 * For each (g, v) in order, acc[j] = acc[j] + w * x for all 32 lanes at
 * once: lane j still adds chunk 32g+j's elements v = 0..7 in order, chunks
 * ascending -- exactly oracle_dot_fixed -- and zero padding adds +0 to an
 * accumulator that is never -0.  The butterfly at the end is scalar.
 * Activations are LM fp32 (converted once per call).  tests/test_cpu_path.py
 * pins every function here against the scalar oracles bit for bit.
 *
 * Vector code: GCC vector extensions, compiled per ISA with target_clones
 * (AVX-512 / AVX2 / generic; -ffp-contract=off keeps mul and add separate).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "pool.h"

float oracle_det_silu(float g);
float oracle_rms_scale(const uint16_t* x, int H, float eps);
void oracle_rms_norm(const uint16_t* x, const uint16_t* w, int rows, int H, float eps,
                     uint16_t* out);
void oracle_rope_kv(const uint16_t* qkv, const float* cos_t, const float* sin_t,
                    const int64_t* start, int B, int T, int nh, int nkv, int hd, int S,
                    int max_pos, uint16_t* q_out, uint16_t* kc, uint16_t* vc);
void oracle_attention(const uint16_t* q, const uint16_t* kc, const uint16_t* vc,
                      const int64_t* start, int B, int T, int nh, int nkv, int hd, int S,
                      float scale, uint16_t* out);

#define SIMD_CLONES __attribute__((target_clones("avx512f", "avx2", "default")))

typedef float v16f __attribute__((vector_size(64), aligned(4)));
typedef uint32_t v16u __attribute__((vector_size(64), aligned(4)));
typedef uint16_t v16h __attribute__((vector_size(32), aligned(2)));

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

int cpu_lm_len(int K) { return (K + 255) / 256 * 256; }

/* ------------------------------------------------------------------ */
/* layout conversion                                                    */
/* ------------------------------------------------------------------ */
typedef struct {
  const uint16_t* raw;
  int K, Kp;
  uint16_t* out;
} pack_ctx;

static void pack_row(void* c, int64_t r) {
  pack_ctx* p = (pack_ctx*)c;
  const uint16_t* src = p->raw + (size_t)r * p->K;
  uint16_t* dst = p->out + (size_t)r * p->Kp;
  for (int g = 0; g < p->Kp / 256; ++g)
    for (int v = 0; v < 8; ++v)
      for (int j = 0; j < 32; ++j) {
        const int k = 256 * g + 8 * j + v;
        dst[256 * g + 32 * v + j] = k < p->K ? src[k] : 0;
      }
}

/* raw [rows, K] bf16 -> LM [rows, Kp] bf16 */
void cpu_pack_lm(const uint16_t* raw, int64_t rows, int K, uint16_t* out) {
  pack_ctx c = {raw, K, cpu_lm_len(K), out};
  oracle_parallel_for(rows, pack_row, &c);
}

/* bf16 [T, K] (row stride ldx) -> LM fp32 [T, Kp] */
static void act_lm(const uint16_t* x, int64_t ldx, int T, int K, float* out) {
  const int Kp = cpu_lm_len(K);
  for (int t = 0; t < T; ++t) {
    const uint16_t* src = x + (size_t)t * ldx;
    float* dst = out + (size_t)t * Kp;
    for (int g = 0; g < Kp / 256; ++g)
      for (int v = 0; v < 8; ++v)
        for (int j = 0; j < 32; ++j) {
          const int k = 256 * g + 8 * j + v;
          dst[256 * g + 32 * v + j] = k < K ? bf2f(src[k]) : 0.0f;
        }
  }
}

/* ------------------------------------------------------------------ */
/* LM dot products of one weight row against TB token rows              */
/* ------------------------------------------------------------------ */
static inline float butterfly(const float* l32) {
  float lane[32];
  memcpy(lane, l32, sizeof(lane));
  for (int w = 16; w >= 1; w >>= 1)
    for (int j = 0; j < w; ++j) lane[j] = lane[j] + lane[j + w];
  return lane[0];
}

static inline __attribute__((always_inline)) v16f cvt16(const uint16_t* p) {
  v16h h;
  memcpy(&h, p, sizeof(h));
  v16u u = __builtin_convertvector(h, v16u) << 16;
  return (v16f)u;
}

static inline __attribute__((always_inline)) v16f ld16(const float* p) {
  v16f v;
  memcpy(&v, p, sizeof(v));
  return v;
}

#define DEF_DOT(TB)                                                                        \
  SIMD_CLONES static void dot_lm_##TB(const uint16_t* w, int Kp, const float* x, int ldx, \
                                      float* out) {                                      \
    v16f a0[TB], a1[TB];                                                                 \
    for (int t = 0; t < TB; ++t) {                                                       \
      a0[t] = (v16f){0};                                                                 \
      a1[t] = (v16f){0};                                                                 \
    }                                                                                    \
    for (int o = 0; o < Kp; o += 32) {                                                   \
      const v16f w0 = cvt16(w + o), w1 = cvt16(w + o + 16);                              \
      for (int t = 0; t < TB; ++t) {                                                     \
        const v16f p0 = w0 * ld16(x + (size_t)t * ldx + o);                              \
        const v16f p1 = w1 * ld16(x + (size_t)t * ldx + o + 16);                         \
        a0[t] = a0[t] + p0;                                                              \
        a1[t] = a1[t] + p1;                                                              \
      }                                                                                  \
    }                                                                                    \
    for (int t = 0; t < TB; ++t) {                                                       \
      float l32[32];                                                                     \
      memcpy(l32, &a0[t], 64);                                                           \
      memcpy(l32 + 16, &a1[t], 64);                                                      \
      out[t] = butterfly(l32);                                                           \
    }                                                                                    \
  }
DEF_DOT(1)
DEF_DOT(2)
DEF_DOT(4)
DEF_DOT(8)

/* out[t] = dot(w row, x token t) for t < T (x: LM fp32 rows, stride ldx) */
static void dot_lm(const uint16_t* w, int Kp, const float* x, int ldx, int T, float* out) {
  int t = 0;
  for (; T - t >= 8; t += 8) dot_lm_8(w, Kp, x + (size_t)t * ldx, ldx, out + t);
  if (T - t >= 4) { dot_lm_4(w, Kp, x + (size_t)t * ldx, ldx, out + t); t += 4; }
  if (T - t >= 2) { dot_lm_2(w, Kp, x + (size_t)t * ldx, ldx, out + t); t += 2; }
  if (T - t >= 1) { dot_lm_1(w, Kp, x + (size_t)t * ldx, ldx, out + t); t += 1; }
}

/* ------------------------------------------------------------------ */
/* K9 linear over an LM weight [N, Kp]                                  */
/* ------------------------------------------------------------------ */
typedef struct {
  const uint16_t* w;
  int Kp, N, T;
  const float* x;
  float* y_f32;
  int64_t ldy;
  uint16_t* y_bf16;
  const uint16_t* resid;
} lml_ctx;

#define ROW_BLOCK 16

static void lml_rows(void* c, int64_t blk) {
  lml_ctx* p = (lml_ctx*)c;
  float s[256];
  for (int64_t n = blk * ROW_BLOCK; n < (blk + 1) * ROW_BLOCK && n < p->N; ++n) {
    for (int t0 = 0; t0 < p->T; t0 += 256) {
      const int nt = p->T - t0 < 256 ? p->T - t0 : 256;
      dot_lm(p->w + (size_t)n * p->Kp, p->Kp, p->x + (size_t)t0 * p->Kp, p->Kp, nt, s);
      for (int t = 0; t < nt; ++t) {
        const size_t tt = (size_t)(t0 + t);
        if (p->y_f32) p->y_f32[tt * p->ldy + n] = s[t];
        if (p->y_bf16) {
          uint16_t o = f2bf(s[t]);
          if (p->resid) o = f2bf(bf2f(p->resid[tt * p->N + n]) + bf2f(o));
          p->y_bf16[tt * p->N + n] = o;
        }
      }
    }
  }
}

/* y = x W^T for raw bf16 x [T, K] (stride ldx; RMSNorm'd first when norm_w)
 * and an LM weight [N, Kp]; outputs as spmoe_linear. */
void cpu_linear(const uint16_t* w_lm, const uint16_t* x, int64_t ldx, int T, int K, int N,
                const uint16_t* norm_w, float eps, float* y_f32, int64_t ldy, uint16_t* y_bf16,
                const uint16_t* resid) {
  const int Kp = cpu_lm_len(K);
  float* xl = (float*)malloc(sizeof(float) * (size_t)(T > 0 ? T : 1) * Kp);
  uint16_t* xn = norm_w ? (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(T > 0 ? T : 1) * K) : NULL;
  if (norm_w) {
    for (int t = 0; t < T; ++t) oracle_rms_norm(x + (size_t)t * ldx, norm_w, 1, K, eps, xn + (size_t)t * K);
    act_lm(xn, K, T, K, xl);
  } else {
    act_lm(x, ldx, T, K, xl);
  }
  lml_ctx c = {w_lm, Kp, N, T, xl, y_f32, ldy, y_bf16, resid};
  oracle_parallel_for((N + ROW_BLOCK - 1) / ROW_BLOCK, lml_rows, &c);
  free(xl);
  free(xn);
}

/* ------------------------------------------------------------------ */
/* one expert's SwiGLU (K3) over an LM blob W1'[F,Hp] | W3'[F,Hp] |     */
/* W2'[H,Fp]:  h[q] = bf16(silu(W1 x) * (W3 x)),  y[q] = W2 h[q] (fp32) */
/* for the token rows x[perm[q]], q < n                                 */
/* ------------------------------------------------------------------ */
typedef struct {
  const uint16_t *w1, *w3, *w2;
  int H, F, Hp, Fp, n;
  const float* xl;  /* [n, Hp] */
  uint16_t* h;      /* [n, F] */
  const float* hl;  /* [n, Fp] */
  float* y;         /* rows y[q * ldy] */
  int64_t ldy;
} ffn_ctx;

static void ffn_up_rows(void* c, int64_t blk) {
  ffn_ctx* p = (ffn_ctx*)c;
  float g[256], u[256];
  for (int64_t f = blk * ROW_BLOCK; f < (blk + 1) * ROW_BLOCK && f < p->F; ++f)
    for (int q0 = 0; q0 < p->n; q0 += 256) {
      const int nq = p->n - q0 < 256 ? p->n - q0 : 256;
      dot_lm(p->w1 + (size_t)f * p->Hp, p->Hp, p->xl + (size_t)q0 * p->Hp, p->Hp, nq, g);
      dot_lm(p->w3 + (size_t)f * p->Hp, p->Hp, p->xl + (size_t)q0 * p->Hp, p->Hp, nq, u);
      for (int q = 0; q < nq; ++q) {
        const float hv = oracle_det_silu(g[q]) * u[q];
        p->h[(size_t)(q0 + q) * p->F + f] = f2bf(hv);
      }
    }
}

static void ffn_down_rows(void* c, int64_t blk) {
  ffn_ctx* p = (ffn_ctx*)c;
  float s[256];
  for (int64_t r = blk * ROW_BLOCK; r < (blk + 1) * ROW_BLOCK && r < p->H; ++r)
    for (int q0 = 0; q0 < p->n; q0 += 256) {
      const int nq = p->n - q0 < 256 ? p->n - q0 : 256;
      dot_lm(p->w2 + (size_t)r * p->Fp, p->Fp, p->hl + (size_t)q0 * p->Fp, p->Fp, nq, s);
      for (int q = 0; q < nq; ++q) p->y[(size_t)(q0 + q) * p->ldy + r] = s[q];
    }
}

/* blob_lm: one expert in LM layout; x [*, H] bf16 rows gathered by perm
 * (perm == NULL: rows 0..n-1); y [n, H] fp32 (row stride H); h [n, F] bf16
 * out (may be NULL: internal scratch). */
void cpu_expert_ffn(const uint16_t* blob_lm, int H, int F, const uint16_t* x, const int32_t* perm,
                    int n, uint16_t* h, float* y) {
  if (n <= 0) return;
  const int Hp = cpu_lm_len(H), Fp = cpu_lm_len(F);
  uint16_t* xg = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n * H);
  for (int q = 0; q < n; ++q) memcpy(xg + (size_t)q * H, x + (size_t)(perm ? perm[q] : q) * H, 2 * (size_t)H);
  float* xl = (float*)malloc(sizeof(float) * (size_t)n * Hp);
  act_lm(xg, H, n, H, xl);
  uint16_t* hh = h ? h : (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n * F);
  ffn_ctx c = {blob_lm, blob_lm + (size_t)F * Hp, blob_lm + 2 * (size_t)F * Hp, H, F, Hp, Fp, n, xl, hh,
               NULL, y, H};
  oracle_parallel_for((F + ROW_BLOCK - 1) / ROW_BLOCK, ffn_up_rows, &c);
  float* hl = (float*)malloc(sizeof(float) * (size_t)n * Fp);
  act_lm(hh, F, n, F, hl);
  c.hl = hl;
  oracle_parallel_for((H + ROW_BLOCK - 1) / ROW_BLOCK, ffn_down_rows, &c);
  free(hl);
  if (!h) free(hh);
  free(xl);
  free(xg);
}

/* LM blob elements of an expert / dense FFN of width F at hidden H */
int64_t cpu_blob_lm_elems(int H, int F) {
  return 2 * (int64_t)F * cpu_lm_len(H) + (int64_t)H * cpu_lm_len(F);
}

/* raw blob W1[F,H] | W3[F,H] | W2[H,F] -> LM blob */
void cpu_pack_blob(const uint16_t* raw, int H, int F, uint16_t* out) {
  const int Hp = cpu_lm_len(H);
  cpu_pack_lm(raw, F, H, out);
  cpu_pack_lm(raw + (size_t)F * H, F, H, out + (size_t)F * Hp);
  cpu_pack_lm(raw + 2 * (size_t)F * H, H, F, out + 2 * (size_t)F * Hp);
}

/* ------------------------------------------------------------------ */
/* attention half of a decoder layer (model.attention_block):           */
/* x <- bf16(x + bf16(attn(RMSNorm(x)) W_o^T)), KV appended             */
/* ------------------------------------------------------------------ */
void cpu_attn_block(uint16_t* x, int B, int T, int H, const uint16_t* wqkv_lm,
                    const uint16_t* wo_lm, const uint16_t* norm_w, float eps, int nh, int nkv,
                    int hd, const float* cos_t, const float* sin_t, int max_pos,
                    const int64_t* start, uint16_t* kc, uint16_t* vc, int S, float scale) {
  const int BT = B * T, Q = (nh + 2 * nkv) * hd, O = nh * hd;
  uint16_t* qkv = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)BT * Q);
  uint16_t* q = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)BT * O);
  uint16_t* o = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)BT * O);
  cpu_linear(wqkv_lm, x, H, BT, H, Q, norm_w, eps, NULL, 0, qkv, NULL);
  oracle_rope_kv(qkv, cos_t, sin_t, start, B, T, nh, nkv, hd, S, max_pos, q, kc, vc);
  oracle_attention(q, kc, vc, start, B, T, nh, nkv, hd, S, scale, o);
  cpu_linear(wo_lm, o, O, BT, O, H, NULL, 0.0f, NULL, 0, x, x);
  free(qkv);
  free(q);
  free(o);
}

/* ------------------------------------------------------------------ */
/* weight construction helpers (the CPU restatement of                  */
/* model.build_weights; elementwise, so results do not depend on the    */
/* thread split)                                                        */
/* ------------------------------------------------------------------ */
typedef struct {
  const uint16_t* a;
  uint16_t* b;
  float* acc;
  const float* cacc;
  int64_t n;
  float s;
} elt_ctx;

#define ELT_BLOCK (1 << 16)

static void upcycle_blk(void* c, int64_t blk) {
  elt_ctx* p = (elt_ctx*)c;
  const int64_t hi = (blk + 1) * ELT_BLOCK < p->n ? (blk + 1) * ELT_BLOCK : p->n;
  for (int64_t i = blk * ELT_BLOCK; i < hi; ++i) {
    const float d = bf2f(p->b[i]) * p->s;
    p->b[i] = f2bf(bf2f(p->a[i]) + d);
  }
}

/* dev <- bf16(base + dev * spread): the upcycled expert of model.gen_expert */
void cpu_upcycle(const uint16_t* base, uint16_t* dev, int64_t n, float spread) {
  elt_ctx c = {base, dev, NULL, NULL, n, spread};
  oracle_parallel_for((n + ELT_BLOCK - 1) / ELT_BLOCK, upcycle_blk, &c);
}

static void accum_blk(void* c, int64_t blk) {
  elt_ctx* p = (elt_ctx*)c;
  const int64_t hi = (blk + 1) * ELT_BLOCK < p->n ? (blk + 1) * ELT_BLOCK : p->n;
  for (int64_t i = blk * ELT_BLOCK; i < hi; ++i) p->acc[i] = p->acc[i] + bf2f(p->a[i]);
}

/* acc += float(x) (the draft proxy's running expert sum) */
void cpu_accum(float* acc, const uint16_t* x, int64_t n) {
  elt_ctx c = {x, NULL, acc, NULL, n, 0.0f};
  oracle_parallel_for((n + ELT_BLOCK - 1) / ELT_BLOCK, accum_blk, &c);
}

static void mean_blk(void* c, int64_t blk) {
  elt_ctx* p = (elt_ctx*)c;
  const int64_t hi = (blk + 1) * ELT_BLOCK < p->n ? (blk + 1) * ELT_BLOCK : p->n;
  for (int64_t i = blk * ELT_BLOCK; i < hi; ++i) p->b[i] = f2bf(p->cacc[i] / p->s);
}

/* out = bf16(acc / div) */
void cpu_div_bf16(const float* acc, int64_t n, float div, uint16_t* out) {
  elt_ctx c = {NULL, out, NULL, acc, n, div};
  oracle_parallel_for((n + ELT_BLOCK - 1) / ELT_BLOCK, mean_blk, &c);
}

static void scale_blk(void* c, int64_t blk) {
  elt_ctx* p = (elt_ctx*)c;
  const int64_t hi = (blk + 1) * ELT_BLOCK < p->n ? (blk + 1) * ELT_BLOCK : p->n;
  for (int64_t i = blk * ELT_BLOCK; i < hi; ++i) p->b[i] = f2bf(bf2f(p->b[i]) * p->s);
}

/* x = bf16(float(x) * s) */
void cpu_scale_bf16(uint16_t* x, int64_t n, float s) {
  elt_ctx c = {NULL, x, NULL, NULL, n, s};
  oracle_parallel_for((n + ELT_BLOCK - 1) / ELT_BLOCK, scale_blk, &c);
}
