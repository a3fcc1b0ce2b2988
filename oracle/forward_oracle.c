/*
 * forward_oracle.c — CPU ORACLE for the layer block around the MoE: the K9
 * projections (qkv, W_o, lm_head), RMSNorm, RoPE + KV append and the cached
 * causal GQA attention of the draft and target forwards.
 *
 * TEST INFRASTRUCTURE ONLY (see spmoe_oracle.c): restates, operation for
 * operation, the determinism contract of include/spmoe.h as implemented by
 * paper_2510_10302_b200/csrc/spmoe_attn.cu and spmoe_kernels.cu (K9), so the
 * whole draft/target forward -- and therefore the greedy accepted-token
 * sequence -- is reproducible on the CPU bit for bit.
 *
 * Reference anchors: the reference package has no tensor code;
 * these pieces are the "draft forward with the MLP-input hook" and "target
 * verify pass outside the MoE" of SURVEY.md §8(f) rows 1-2 (simcore.py:
 * 323-359 compute slots), in the standard
 * Mixtral/Qwen/DeepSeek decoder form (RMSNorm, rotate-half RoPE, GQA).
 *
 * Every float operation is an IEEE single-precision op in the order
 * written (-ffp-contract=off, no fast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "pool.h"

float oracle_dot_fixed(const uint16_t* a, const uint16_t* b, int n);
float oracle_det_exp(float x);

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

/* ------------------------------------------------------------------ */
/* RMSNorm: s = 1 / sqrt(dot_fixed(x, x) / H + eps); y = bf16((x*s)*w)   */
/* (spmoe_attn.cu rms_norm_kernel, spmoe_kernels.cu rms_scale_row)      */
/* ------------------------------------------------------------------ */
float oracle_rms_scale(const uint16_t* x, int H, float eps) {
  const float ss = oracle_dot_fixed(x, x, H);
  const float mean = ss / (float)H;
  const float v = mean + eps;
  return 1.0f / sqrtf(v);
}

void oracle_rms_norm(const uint16_t* x, const uint16_t* w, int rows, int H, float eps,
                     uint16_t* out) {
  for (int r = 0; r < rows; ++r) {
    const uint16_t* xr = x + (size_t)r * H;
    const float s = oracle_rms_scale(xr, H, eps);
    for (int i = 0; i < H; ++i) {
      const float a = bf2f(xr[i]) * s;
      out[(size_t)r * H + i] = f2bf(a * bf2f(w[i]));
    }
  }
}

/* ------------------------------------------------------------------ */
/* K9 linear                                                            */
/* ------------------------------------------------------------------ */
typedef struct {
  const uint16_t *w, *xin, *resid;
  int T, K, N;
  float* y_f32;
  int64_t ldy;
  uint16_t* y_bf16;
} lin_ctx;

static void lin_row(void* c, int64_t n) {
  lin_ctx* p = (lin_ctx*)c;
  const uint16_t* wr = p->w + (size_t)n * p->K;
  for (int t = 0; t < p->T; ++t) {
    const float s = oracle_dot_fixed(wr, p->xin + (size_t)t * p->K, p->K);
    if (p->y_f32) p->y_f32[(size_t)t * p->ldy + n] = s;
    if (p->y_bf16) {
      uint16_t o = f2bf(s);
      if (p->resid) o = f2bf(bf2f(p->resid[(size_t)t * p->N + n]) + bf2f(o));
      p->y_bf16[(size_t)t * p->N + n] = o;
    }
  }
}

void oracle_linear(const uint16_t* w, const uint16_t* x, int64_t ldx, int T, int K, int N,
                   const uint16_t* norm_w, float eps, float* y_f32, int64_t ldy, uint16_t* y_bf16,
                   const uint16_t* resid) {
  uint16_t* xin = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(T > 0 ? T : 1) * K);
  for (int t = 0; t < T; ++t) {
    if (norm_w)
      oracle_rms_norm(x + (size_t)t * ldx, norm_w, 1, K, eps, xin + (size_t)t * K);
    else
      memcpy(xin + (size_t)t * K, x + (size_t)t * ldx, sizeof(uint16_t) * K);
  }
  /* resid may alias y_bf16: each element is read then written by its own
   * (row, token) step, as on the GPU */
  lin_ctx c = {w, xin, resid, T, K, N, y_f32, ldy, y_bf16};
  oracle_parallel_for(N, lin_row, &c);
  free(xin);
}

/* ------------------------------------------------------------------ */
/* RoPE + KV append (rope_kv_kernel)                                    */
/* ------------------------------------------------------------------ */
void oracle_rope_kv(const uint16_t* qkv, const float* cos_t, const float* sin_t,
                    const int64_t* start, int B, int T, int nh, int nkv, int hd, int S,
                    int max_pos, uint16_t* q_out, uint16_t* kc, uint16_t* vc) {
  const int half = hd / 2, total = (nh + 2 * nkv) * hd;
  for (int b = 0; b < B; ++b)
    for (int t = 0; t < T; ++t) {
      const int64_t pos = start[b] + t;
      if (pos < 0 || pos >= S || pos >= max_pos) continue;
      const uint16_t* src = qkv + ((size_t)b * T + t) * total;
      const float* cs = cos_t + pos * hd;
      const float* sn = sin_t + pos * hd;
      for (int i = 0; i < total; ++i) {
        const int head = i / hd, d = i % hd;
        if (head < nh + nkv) {
          const float x = bf2f(src[i]);
          const int pd = d < half ? d + half : d - half;
          const float xp = bf2f(src[head * hd + pd]);
          const float rot = d < half ? -xp : xp;
          const float t1 = x * cs[d];
          const float t2 = rot * sn[d];
          const uint16_t y = f2bf(t1 + t2);
          if (head < nh)
            q_out[(((size_t)b * nh + head) * T + t) * hd + d] = y;
          else
            kc[(((size_t)b * nkv + (head - nh)) * S + pos) * hd + d] = y;
        } else {
          vc[(((size_t)b * nkv + (head - nh - nkv)) * S + pos) * hd + d] = src[i];
        }
      }
    }
}

/* ------------------------------------------------------------------ */
/* cached causal GQA attention (attn_kernel): the fixed order of        */
/* spmoe_attn.cu -- lane-blocked score dots + butterfly, det_exp(s-max), */
/* 8 key streams (key mod 8) merged in stream order, IEEE division      */
/* ------------------------------------------------------------------ */
#define ATTN_STREAMS 8

typedef struct {
  const uint16_t *q, *kc, *vc;
  const int64_t* start;
  int T, nh, nkv, hd, S;
  float scale;
  uint16_t* out;
} attn_ctx;

static float score_fixed(const float* qs, const uint16_t* k, int hd) {
  float lane[32];
  const int pl = hd / 32;
  for (int l = 0; l < 32; ++l) {
    float acc = 0.0f;
    for (int j = 0; j < pl; ++j) {
      const float prod = qs[l * pl + j] * bf2f(k[l * pl + j]);
      acc = acc + prod;
    }
    lane[l] = acc;
  }
  for (int w = 16; w >= 1; w >>= 1)
    for (int j = 0; j < w; ++j) lane[j] = lane[j] + lane[j + w];
  return lane[0];
}

static void attn_row(void* c, int64_t r) {
  attn_ctx* p = (attn_ctx*)c;
  const int hd = p->hd, S = p->S;
  const int t = (int)(r % p->T);
  const int h = (int)((r / p->T) % p->nh);
  const int b = (int)(r / ((int64_t)p->T * p->nh));
  const int kh = h / (p->nh / p->nkv);
  const int64_t pos = p->start[b] + t;
  int64_t kl = pos + 1;
  if (kl > S) kl = S;
  float qs[256];
  const uint16_t* qr = p->q + (((size_t)b * p->nh + h) * p->T + t) * hd;
  for (int d = 0; d < hd; ++d) qs[d] = bf2f(qr[d]) * p->scale;
  const uint16_t* kb = p->kc + ((size_t)b * p->nkv + kh) * (size_t)S * hd;
  const uint16_t* vb = p->vc + ((size_t)b * p->nkv + kh) * (size_t)S * hd;
  float* pr = (float*)malloc(sizeof(float) * (size_t)(kl > 0 ? kl : 1));
  float m = -INFINITY;
  for (int64_t j = 0; j < kl; ++j) {
    pr[j] = score_fixed(qs, kb + j * hd, hd);
    m = fmaxf(m, pr[j]);
  }
  for (int64_t j = 0; j < kl; ++j) pr[j] = oracle_det_exp(pr[j] - m);
  float num[256], den = 0.0f;
  for (int d = 0; d < hd; ++d) num[d] = 0.0f;
  for (int w = 0; w < ATTN_STREAMS; ++w) {
    float lw = 0.0f, accw[256];
    for (int d = 0; d < hd; ++d) accw[d] = 0.0f;
    for (int64_t j = w; j < kl; j += ATTN_STREAMS) {
      lw = lw + pr[j];
      for (int d = 0; d < hd; ++d) {
        const float prod = pr[j] * bf2f(vb[j * hd + d]);
        accw[d] = accw[d] + prod;
      }
    }
    den = den + lw;
    for (int d = 0; d < hd; ++d) num[d] = num[d] + accw[d];
  }
  uint16_t* o = p->out + (((size_t)b * p->T + t) * p->nh + h) * hd;
  for (int d = 0; d < hd; ++d) o[d] = f2bf(num[d] / den);
  free(pr);
}

void oracle_attention(const uint16_t* q, const uint16_t* kc, const uint16_t* vc,
                      const int64_t* start, int B, int T, int nh, int nkv, int hd, int S,
                      float scale, uint16_t* out) {
  attn_ctx c = {q, kc, vc, start, T, nh, nkv, hd, S, scale, out};
  oracle_parallel_for((int64_t)B * nh * T, attn_row, &c);
}
