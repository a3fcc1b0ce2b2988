// spmoe_attn.cu — the target/draft layer block around the MoE (SURVEY.md
// §8(f) rows 1-2: draft forward and the verify pass outside the MoE) as
// fused sm_100a kernels instead of ~30 small framework kernels per layer:
//
//   rms_norm_kernel   y = bf16((x * r) * w), r = 1/sqrt(mean(x^2) + eps), one
//                     warp per row (HF Mixtral/Qwen/DeepSeek RMSNorm)
//   rope_kv_kernel    split the fused qkv projection, rotate q and k
//                     (rotate-half RoPE), write q in [B, nh, T, hd] and append
//                     k, v to the layer's KV cache [B, nkv, S, hd] at each
//                     sequence's own positions
//   attn_kernel       causal GQA attention of T new queries over the cached
//                     keys 0..pos, two-pass softmax in fp32, output
//                     [B, T, nh*hd] bf16 ready for the W_o projection
//
// Every operation follows the determinism contract of include/spmoe.h, so
// the CPU oracle (oracle/forward_oracle.c) reproduces each output bit for
// bit: fixed-order reductions, IEEE mul/add/div/sqrt written out with
// __f*_rn (never contracted), det_exp instead of the SFU exp.  The
// projections around them are K9 linear launches (spmoe_kernels.cu).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spmoe.h"
#include "spmoe_common.cuh"

using namespace spmoe;

namespace {

// ------------------------------------------------------------------ RMSNorm
// One CTA per row; H % 8 == 0.  Warp 0 computes ss = dot_fixed(x, x)
// (lane-strided 8-value chunks, butterfly) and r = 1 / sqrt(ss / H + eps);
// every thread of the CTA then writes its chunks of y = bf16((x * r) * w)
// (elementwise: the split does not change a bit).
__global__ void __launch_bounds__(256) rms_norm_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w,
                                                       int rows, int H, float eps, uint16_t* __restrict__ out) {
  __shared__ float s_r;
  grid_dep_trigger();  // a following K9 (lm_head) may start streaming its weights
  const int row = blockIdx.x;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)row * H);
  const int n8 = H / 8;
  if (threadIdx.x < 32) {
    float ss = 0.0f;
    // loads of U rounds in flight together; the FMA order is unchanged
    constexpr int U = 8;
    for (int c0 = lane; c0 < n8; c0 += 32 * U) {
      uint4 xa[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c0 + 32 * u < n8) xa[u] = xr[c0 + 32 * u];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c0 + 32 * u < n8) {
          float a[8];
          unpack8(xa[u], a);
#pragma unroll
          for (int v = 0; v < 8; ++v) ss = fmaf(a[v], a[v], ss);  // bf16 squares are exact
        }
      }
    }
    ss = warp_sum_fixed(ss);
    if (lane == 0) s_r = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)H), eps)));
  }
  __syncthreads();
  const float r = s_r;
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* orow = reinterpret_cast<uint4*>(out + (int64_t)row * H);
  for (int i = threadIdx.x; i < n8; i += blockDim.x) {
    const uint4 v = xr[i], g = wr[i];
    const uint32_t u[4] = {v.x, v.y, v.z, v.w}, gw[4] = {g.x, g.y, g.z, g.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float lo = __fmul_rn(__fmul_rn(bf16_lo(u[j]), r), bf16_lo(gw[j]));
      const float hi = __fmul_rn(__fmul_rn(bf16_hi(u[j]), r), bf16_hi(gw[j]));
      o[j] = (uint32_t)f32_to_bf16(lo) | ((uint32_t)f32_to_bf16(hi) << 16);
    }
    orow[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ------------------------------------------------------------- RoPE + KV
// grid.x = token row, grid.y = 256-element slices of the row's nh + 2 nkv
// heads' dims: one element per thread, so a row's loads are all in flight
// at once (elementwise, the arithmetic does not depend on the split).
// y[d] = bf16(x[d] * cos[pos][d] + rot[d] * sin[pos][d]), rot = [-x2, x1],
// the two products and the sum each IEEE-rounded.  Positions at or beyond
// the cache (S) or the RoPE table (max_pos) write nothing (the host checks
// lengths before launching; this keeps a bad position from corrupting
// memory).
__global__ void __launch_bounds__(256) rope_kv_kernel(const uint16_t* __restrict__ qkv, const float* __restrict__ cos_t,
                                                      const float* __restrict__ sin_t, const int64_t* __restrict__ start,
                                                      int T, int nh, int nkv, int hd, int S, int max_pos,
                                                      uint16_t* __restrict__ q_out, uint16_t* __restrict__ kc,
                                                      uint16_t* __restrict__ vc) {
  const int row = blockIdx.x;  // b * T + t
  const int b = row / T, t = row % T;
  const int64_t pos = start[b] + t;
  if (pos < 0 || pos >= S || pos >= max_pos) return;
  const uint16_t* src = qkv + (int64_t)row * (nh + 2 * nkv) * hd;
  const float* cs = cos_t + pos * hd;
  const float* sn = sin_t + pos * hd;
  const int half = hd / 2;
  const int total = (nh + 2 * nkv) * hd;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < total; i += gridDim.y * blockDim.x) {
    const int head = i / hd, d = i % hd;
    const float x = bf16_to_f32(src[i]);
    if (head < nh + nkv) {
      const int pd = d < half ? d + half : d - half;
      const float xp = bf16_to_f32(src[head * hd + pd]);
      const float rot = d < half ? -xp : xp;
      const uint16_t y = f32_to_bf16(__fadd_rn(__fmul_rn(x, cs[d]), __fmul_rn(rot, sn[d])));
      if (head < nh) {
        q_out[(((int64_t)b * nh + head) * T + t) * hd + d] = y;
      } else {
        const int kh = head - nh;
        kc[(((int64_t)b * nkv + kh) * S + pos) * hd + d] = y;
      }
    } else {
      const int vh = head - nh - nkv;
      vc[(((int64_t)b * nkv + vh) * S + pos) * hd + d] = src[i];
    }
  }
}

// ------------------------------------------------------------ attention
// One CTA (NW = 8 warps) per (b, head, chunk of QC queries: 1 for a
// verify / draft step's few queries -- more CTAs in flight --, 8 for a
// prefill; QC only groups queries, it is not part of the order).  The fixed
// order, restated by oracle_attention:
//   qs[d]  = q[d] * scale
//   s_j    = sum_d qs[d] * k_j[d]: lane l sums its PL = hd/32 consecutive
//            dims in order, then the xor butterfly 16,8,4,2,1
//   m      = max_j s_j over the causal keys j <= pos
//   p_j    = det_exp(s_j - m)
//   stream w (= warp w) sums its keys j = w, w+8, w+16, ... ascending:
//            l_w = sum p_j,  acc_w[d] = sum p_j * v_j[d]
//   l = l_0 + l_1 + ... + l_7 (in w order), acc[d] likewise,
//   out[d] = bf16(acc[d] / l).
// Pass 1 keeps the scores of the chunk in shared memory ([QC][S] fp32).
constexpr int kAttnQCMax = 8;
constexpr int kAttnNW = 8;

// The PL bf16 of row `key` that lane owns (dims lane*PL ..), as fp32: one
// 8-byte (PL = 4) or 4-byte (PL = 2) load.
template <int PL>
__device__ __forceinline__ void load_row(const uint16_t* base, int key, int hd, int lane, float (&out)[PL]) {
  const uint16_t* p = base + (int64_t)key * hd + lane * PL;
  if constexpr (PL == 4) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
    out[0] = bf16_lo(w.x);
    out[1] = bf16_hi(w.x);
    out[2] = bf16_lo(w.y);
    out[3] = bf16_hi(w.y);
  } else {
#pragma unroll
    for (int j = 0; j < PL; ++j) out[j] = bf16_to_f32(p[j]);
  }
}

template <int HD, int QC>
__global__ void __launch_bounds__(32 * kAttnNW) attn_kernel(const uint16_t* __restrict__ q,
                                                         const uint16_t* __restrict__ kc,
                                                         const uint16_t* __restrict__ vc,
                                                         const int64_t* __restrict__ start, int T, int nh, int nkv,
                                                         int S, float scale, uint16_t* __restrict__ out) {
  constexpr int NW = kAttnNW;
  constexpr int PL = HD / 32;  // dims per lane
  grid_dep_trigger();  // the following K9 (W_o) may start streaming its weights
  extern __shared__ __align__(16) float sm[];
  float* s_p = sm;                        // [QC][S] scores, then probabilities
  float* s_acc = s_p + (int64_t)QC * S;   // [NW][QC][HD]
  float* s_l = s_acc + NW * QC * HD;      // [NW][QC]
  const int nqc = (T + QC - 1) / QC;
  const int qc = blockIdx.x % nqc;
  const int h = (blockIdx.x / nqc) % nh;
  const int b = blockIdx.x / (nqc * nh);
  const int kh = h / (nh / nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = qc * QC;
  const int nq = min(QC, T - t0);
  const int64_t p0 = start[b] + t0;  // position of the chunk's first query
  const int klen = (int)min((int64_t)S, p0 + nq);  // keys 0 .. last query's position
  float qv[QC][PL];
#pragma unroll
  for (int i = 0; i < QC; ++i)
#pragma unroll
    for (int j = 0; j < PL; ++j)
      qv[i][j] = i < nq ? __fmul_rn(bf16_to_f32(q[(((int64_t)b * nh + h) * T + t0 + i) * HD + lane * PL + j]), scale)
                        : 0.0f;
  const uint16_t* kb = kc + ((int64_t)b * nkv + kh) * S * HD;
  const uint16_t* vb = vc + ((int64_t)b * nkv + kh) * S * HD;
  // pass 1: scores.  The K rows of KU keys are loaded together (one vector
  // load per lane per key) before their dot products: same arithmetic per
  // key, KU memory latencies overlapped instead of one per key.
  constexpr int KU = 4;
  for (int key0 = warp; key0 < klen; key0 += NW * KU) {
    float kv[KU][PL];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int key = key0 + u * NW;
      load_row<PL>(kb, key < klen ? key : key0, HD, lane, kv[u]);
    }
    // every (key, query) lane partial first, then the xor butterflies of
    // all of them level by level (the same per-value order as
    // warp_sum_fixed, with KU*QC independent shuffle chains in flight)
    float sp[KU][QC];
#pragma unroll
    for (int u = 0; u < KU; ++u)
#pragma unroll
      for (int i = 0; i < QC; ++i) {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < PL; ++j) acc = __fadd_rn(acc, __fmul_rn(qv[i][j], kv[u][j]));
        sp[u][i] = acc;
      }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
      for (int u = 0; u < KU; ++u)
#pragma unroll
        for (int i = 0; i < QC; ++i) sp[u][i] = __fadd_rn(sp[u][i], __shfl_xor_sync(SPMOE_FULL_MASK, sp[u][i], off));
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int key = key0 + u * NW;
#pragma unroll
        for (int i = 0; i < QC; ++i)
          if (key < klen && i < nq && key <= p0 + i) s_p[i * S + key] = sp[u][i];  // causal keys only
      }
    }
  }
  __syncthreads();
  // max and probabilities: warp i owns query i
  if (warp < nq) {
    const int kl = (int)min((int64_t)S, p0 + warp + 1);
    float* row = s_p + warp * S;
    float m = -INFINITY;
    for (int j = lane; j < kl; j += 32) m = fmaxf(m, row[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(SPMOE_FULL_MASK, m, o));
    for (int j = lane; j < kl; j += 32) row[j] = det_exp(__fsub_rn(row[j], m));
  }
  __syncthreads();
  // pass 2: stream w = warp w, keys ascending
  float l[QC], acc[QC][PL];
#pragma unroll
  for (int i = 0; i < QC; ++i) {
    l[i] = 0.0f;
#pragma unroll
    for (int j = 0; j < PL; ++j) acc[i][j] = 0.0f;
  }
  for (int key0 = warp; key0 < klen; key0 += NW * KU) {
    float vv[KU][PL];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int key = key0 + u * NW;
      load_row<PL>(vb, key < klen ? key : key0, HD, lane, vv[u]);
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {  // keys ascending: the stream's fixed order
      const int key = key0 + u * NW;
      if (key >= klen) break;
#pragma unroll
      for (int i = 0; i < QC; ++i) {
        if (i >= nq || key > p0 + i) continue;
        const float pj = s_p[i * S + key];
        l[i] = __fadd_rn(l[i], pj);
#pragma unroll
        for (int j = 0; j < PL; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(pj, vv[u][j]));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < QC; ++i) {
#pragma unroll
    for (int j = 0; j < PL; ++j) s_acc[(warp * QC + i) * HD + lane * PL + j] = acc[i][j];
    if (lane == 0) s_l[warp * QC + i] = l[i];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nq * HD; idx += blockDim.x) {
    const int i = idx / HD, d = idx % HD;
    float den = 0.0f, num = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      den = __fadd_rn(den, s_l[w * QC + i]);
      num = __fadd_rn(num, s_acc[(w * QC + i) * HD + d]);
    }
    out[(((int64_t)b * T + t0 + i) * nh + h) * HD + d] = f32_to_bf16(__fdiv_rn(num, den));
  }
}

size_t attn_smem(int S, int hd, int qc) {
  return ((size_t)qc * S + (size_t)kAttnNW * qc * hd + kAttnNW * qc) * sizeof(float);
}

constexpr size_t kAttnSmemCap = 200 * 1024;

}  // namespace

extern "C" {

int spmoe_rms_norm(const uint16_t* x, const uint16_t* w, int rows, int H, float eps, uint16_t* out, void* stream) {
  if (rows < 0 || H <= 0 || H % 8 || !x || !w || !out) return (int)cudaErrorInvalidValue;
  if (rows == 0) return 0;
  rms_norm_kernel<<<rows, 256, 0, (cudaStream_t)stream>>>(x, w, rows, H, eps, out);
  return (int)cudaGetLastError();
}

int spmoe_rope_kv(const uint16_t* qkv, const float* cos_t, const float* sin_t, const int64_t* start, int B, int T,
                  int nh, int nkv, int hd, int S, int max_pos, uint16_t* q_out, uint16_t* k_cache,
                  uint16_t* v_cache, void* stream) {
  if (B < 0 || T < 0 || nh < 1 || nkv < 1 || nh % nkv || hd % 2 || S < 1 || max_pos < 1 || !qkv || !q_out ||
      !k_cache || !v_cache || !cos_t || !sin_t || !start)
    return (int)cudaErrorInvalidValue;
  if (B * T == 0) return 0;
  const int slices = ((nh + 2 * nkv) * hd + 255) / 256;
  rope_kv_kernel<<<dim3(B * T, slices), 256, 0, (cudaStream_t)stream>>>(qkv, cos_t, sin_t, start, T, nh, nkv, hd, S,
                                                                      max_pos, q_out, k_cache, v_cache);
  return (int)cudaGetLastError();
}

int spmoe_attention(const uint16_t* q, const uint16_t* k_cache, const uint16_t* v_cache, const int64_t* start,
                    int B, int T, int nh, int nkv, int hd, int S, float scale, uint16_t* out, void* stream) {
  if (B < 0 || T < 0 || nh < 1 || nkv < 1 || nh % nkv || (hd != 64 && hd != 128) || S < 1 || !q || !out ||
      !k_cache || !v_cache || !start)
    return (int)cudaErrorInvalidValue;
  if (B * T == 0) return 0;
  // a verify / draft step (T <= 8 queries): one query per CTA, B*nh*T CTAs
  const int qc = T <= kAttnQCMax ? 1 : kAttnQCMax;
  const size_t smem = attn_smem(S, hd, qc);
  if (smem > kAttnSmemCap) return (int)cudaErrorInvalidValue;
  const int nqc = (T + qc - 1) / qc;
  const dim3 grid(B * nh * nqc);
  cudaStream_t st = (cudaStream_t)stream;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attn_kernel<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAttnSmemCap);
    cudaFuncSetAttribute(attn_kernel<64, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAttnSmemCap);
    cudaFuncSetAttribute(attn_kernel<128, kAttnQCMax>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAttnSmemCap);
    cudaFuncSetAttribute(attn_kernel<64, kAttnQCMax>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAttnSmemCap);
    configured = true;
  }
  if (hd == 128 && qc == 1)
    attn_kernel<128, 1><<<grid, 32 * kAttnNW, smem, st>>>(q, k_cache, v_cache, start, T, nh, nkv, S, scale, out);
  else if (hd == 128)
    attn_kernel<128, kAttnQCMax><<<grid, 32 * kAttnNW, smem, st>>>(q, k_cache, v_cache, start, T, nh, nkv, S, scale,
                                                                   out);
  else if (qc == 1)
    attn_kernel<64, 1><<<grid, 32 * kAttnNW, smem, st>>>(q, k_cache, v_cache, start, T, nh, nkv, S, scale, out);
  else
    attn_kernel<64, kAttnQCMax><<<grid, 32 * kAttnNW, smem, st>>>(q, k_cache, v_cache, start, T, nh, nkv, S, scale,
                                                                  out);
  return (int)cudaGetLastError();
}

}  // extern "C"
