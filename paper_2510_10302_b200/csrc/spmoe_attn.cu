// spmoe_attn.cu — the target/draft layer block around the MoE (SURVEY.md
// §8(f) rows 1-2: draft forward and the verify pass outside the MoE) as
// three fused sm_100a kernels instead of ~30 small framework kernels per
// layer:
//
//   rms_norm_kernel   y = bf16(x * rsqrt(mean(x^2) + eps) * w), one warp per
//                     row, fp32 (HF Mixtral/Qwen/DeepSeek RMSNorm)
//   rope_kv_kernel    split the fused qkv projection, rotate q and k
//                     (rotate-half RoPE, fp32 math, bf16 out), write q in
//                     [B, nh, T, hd] and append k, v to the layer's KV cache
//                     [B, nkv, S, hd] at each sequence's own positions
//   attn_kernel       causal GQA attention of T new queries over the cached
//                     keys 0..pos, online softmax in fp32, output
//                     [B, T, nh*hd] bf16 ready for the W_o projection
//
// These are latency-bound (a few KB to a few MB per launch); the projections
// around them are cuBLAS GEMMs (weight-bandwidth bound).  Numerics follow
// the PyTorch reference within bf16 rounding of the attention output;
// routing parity is unaffected because the oracle checks each MoE layer on
// the GPU's own layer input.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spmoe.h"
#include "spmoe_common.cuh"

using namespace spmoe;

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ RMSNorm
// One warp per row; H % 8 == 0; 16-byte loads.
__global__ void __launch_bounds__(256) rms_norm_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w,
                                                       int rows, int H, float eps, uint16_t* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)warp * H);
  const int n8 = H / 8;
  float ss = 0.0f;
  for (int i = lane; i < n8; i += 32) {
    const uint4 v = xr[i];
    const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float a = bf16_lo(u[j]), b = bf16_hi(u[j]);
      ss += a * a + b * b;
    }
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / (float)H + eps);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* orow = reinterpret_cast<uint4*>(out + (int64_t)warp * H);
  for (int i = lane; i < n8; i += 32) {
    const uint4 v = xr[i], g = wr[i];
    const uint32_t u[4] = {v.x, v.y, v.z, v.w}, gw[4] = {g.x, g.y, g.z, g.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // fp32 (x * r) * w, one rounding to bf16 (as the PyTorch reference)
      const float lo = (bf16_lo(u[j]) * r) * bf16_lo(gw[j]);
      const float hi = (bf16_hi(u[j]) * r) * bf16_hi(gw[j]);
      o[j] = (uint32_t)f32_to_bf16(lo) | ((uint32_t)f32_to_bf16(hi) << 16);
    }
    orow[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ------------------------------------------------------------- RoPE + KV
// One CTA per (token row); threads walk the nh + 2 nkv heads' dims.
__global__ void __launch_bounds__(256) rope_kv_kernel(const uint16_t* __restrict__ qkv, const float* __restrict__ cos_t,
                                                      const float* __restrict__ sin_t, const int64_t* __restrict__ start,
                                                      int T, int nh, int nkv, int hd, int S,
                                                      uint16_t* __restrict__ q_out, uint16_t* __restrict__ kc,
                                                      uint16_t* __restrict__ vc) {
  const int row = blockIdx.x;  // b * T + t
  const int b = row / T, t = row % T;
  const int64_t pos = start[b] + t;
  const uint16_t* src = qkv + (int64_t)row * (nh + 2 * nkv) * hd;
  const float* cs = cos_t + pos * hd;
  const float* sn = sin_t + pos * hd;
  const int half = hd / 2;
  const int total = (nh + 2 * nkv) * hd;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int head = i / hd, d = i % hd;
    const float x = bf16_to_f32(src[i]);
    if (head < nh + nkv) {
      // rotate_half: [-x2, x1]
      const int pd = d < half ? d + half : d - half;
      const float xp = bf16_to_f32(src[head * hd + pd]);
      const float rot = d < half ? -xp : xp;
      const uint16_t y = f32_to_bf16(x * cs[d] + rot * sn[d]);
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
// One CTA (NW warps) per (b, head, chunk of QC queries).  Each warp owns a
// strided subset of the keys and keeps, per query, an online-softmax state
// (max, sum, acc[hd/32 per lane]); the warps merge through shared memory.
template <int HD, int QC, int NW>
__global__ void __launch_bounds__(32 * NW) attn_kernel(const uint16_t* __restrict__ q, const uint16_t* __restrict__ kc,
                                                   const uint16_t* __restrict__ vc, const int64_t* __restrict__ start,
                                                   int T, int nh, int nkv, int S, float scale,
                                                   uint16_t* __restrict__ out) {
  constexpr int PL = HD / 32;  // dims per lane
  const int nqc = (T + QC - 1) / QC;
  const int qc = blockIdx.x % nqc;
  const int h = (blockIdx.x / nqc) % nh;
  const int b = blockIdx.x / (nqc * nh);
  const int kh = h / (nh / nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = qc * QC;
  const int nq = min(QC, T - t0);
  const int64_t p0 = start[b];
  const int klen = (int)(p0 + t0 + nq);  // keys 0 .. last query's position
  float qv[QC][PL];
#pragma unroll
  for (int i = 0; i < QC; ++i)
#pragma unroll
    for (int j = 0; j < PL; ++j)
      qv[i][j] = i < nq ? bf16_to_f32(q[(((int64_t)b * nh + h) * T + t0 + i) * HD + lane * PL + j]) * scale : 0.0f;
  float m[QC], l[QC], acc[QC][PL];
#pragma unroll
  for (int i = 0; i < QC; ++i) {
    m[i] = -INFINITY;
    l[i] = 0.0f;
#pragma unroll
    for (int j = 0; j < PL; ++j) acc[i][j] = 0.0f;
  }
  const uint16_t* kb = kc + ((int64_t)b * nkv + kh) * S * HD;
  const uint16_t* vb = vc + ((int64_t)b * nkv + kh) * S * HD;
  for (int key = warp; key < klen; key += NW) {
    float kv[PL], vv[PL];
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      kv[j] = bf16_to_f32(kb[(int64_t)key * HD + lane * PL + j]);
      vv[j] = bf16_to_f32(vb[(int64_t)key * HD + lane * PL + j]);
    }
#pragma unroll
    for (int i = 0; i < QC; ++i) {
      if (i >= nq || key > p0 + t0 + i) continue;  // causal (warp-uniform)
      float s = 0.0f;
#pragma unroll
      for (int j = 0; j < PL; ++j) s += qv[i][j] * kv[j];
      s = warp_sum(s);
      const float mn = fmaxf(m[i], s);
      const float c = __expf(m[i] - mn), pexp = __expf(s - mn);
      l[i] = l[i] * c + pexp;
#pragma unroll
      for (int j = 0; j < PL; ++j) acc[i][j] = acc[i][j] * c + pexp * vv[j];
      m[i] = mn;
    }
  }
  // merge the 4 warps' states
  __shared__ float sm_m[NW][QC], sm_l[NW][QC];
  __shared__ float sm_acc[NW][QC][HD];
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < QC; ++i) {
      sm_m[warp][i] = m[i];
      sm_l[warp][i] = l[i];
    }
#pragma unroll
  for (int i = 0; i < QC; ++i)
#pragma unroll
    for (int j = 0; j < PL; ++j) sm_acc[warp][i][lane * PL + j] = acc[i][j];
  __syncthreads();
  for (int idx = threadIdx.x; idx < nq * HD; idx += blockDim.x) {
    const int i = idx / HD, d = idx % HD;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) mx = fmaxf(mx, sm_m[w][i]);
    float den = 0.0f, num = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      if (sm_m[w][i] == -INFINITY) continue;
      const float c = __expf(sm_m[w][i] - mx);
      den += sm_l[w][i] * c;
      num += sm_acc[w][i][d] * c;
    }
    out[(((int64_t)b * T + t0 + i) * nh + h) * HD + d] = f32_to_bf16(num / den);
  }
}

}  // namespace

extern "C" {

int spmoe_rms_norm(const uint16_t* x, const uint16_t* w, int rows, int H, float eps, uint16_t* out, void* stream) {
  if (rows < 0 || H <= 0 || H % 8 || !x || !w || !out) return (int)cudaErrorInvalidValue;
  if (rows == 0) return 0;
  const int threads = 256, per = threads / 32;
  rms_norm_kernel<<<(rows + per - 1) / per, threads, 0, (cudaStream_t)stream>>>(x, w, rows, H, eps, out);
  return (int)cudaGetLastError();
}

int spmoe_rope_kv(const uint16_t* qkv, const float* cos_t, const float* sin_t, const int64_t* start, int B, int T,
                  int nh, int nkv, int hd, int S, uint16_t* q_out, uint16_t* k_cache, uint16_t* v_cache,
                  void* stream) {
  if (B < 0 || T < 0 || nh < 1 || nkv < 1 || nh % nkv || hd % 2 || !qkv || !q_out || !k_cache || !v_cache)
    return (int)cudaErrorInvalidValue;
  if (B * T == 0) return 0;
  rope_kv_kernel<<<B * T, 256, 0, (cudaStream_t)stream>>>(qkv, cos_t, sin_t, start, T, nh, nkv, hd, S, q_out,
                                                          k_cache, v_cache);
  return (int)cudaGetLastError();
}

int spmoe_attention(const uint16_t* q, const uint16_t* k_cache, const uint16_t* v_cache, const int64_t* start,
                    int B, int T, int nh, int nkv, int hd, int S, float scale, uint16_t* out, void* stream) {
  if (B < 0 || T < 0 || nh < 1 || nkv < 1 || nh % nkv || (hd != 64 && hd != 128) || !q || !out)
    return (int)cudaErrorInvalidValue;
  if (B * T == 0) return 0;
  constexpr int QC = 8;  // T = N + 1 <= 9 verify tokens: one or two chunks
  const int nqc = (T + QC - 1) / QC;
  const dim3 grid(B * nh * nqc);
  cudaStream_t st = (cudaStream_t)stream;
  if (hd == 128)
    attn_kernel<128, QC, 8><<<grid, 256, 0, st>>>(q, k_cache, v_cache, start, T, nh, nkv, S, scale, out);
  else
    attn_kernel<64, QC, 8><<<grid, 256, 0, st>>>(q, k_cache, v_cache, start, T, nh, nkv, S, scale, out);
  return (int)cudaGetLastError();
}

}  // extern "C"
