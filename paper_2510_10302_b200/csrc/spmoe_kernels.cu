// spmoe_kernels.cu — sm_100a kernels of the SP-MoE verification-time expert
// path: K1 router_topk, K2 moe_permute, K3 expert_ffn (weight-streaming
// grouped SwiGLU over the HBM slot pool), K4 moe_combine, K6 greedy_accept,
// plus the deterministic counter-hash weight init.  C ABI in include/spmoe.h.
#include "spmoe_common.cuh"
#include "../../include/spmoe.h"

#include <stdio.h>
#include <stdlib.h>

using namespace spmoe;

namespace {

int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return (int)e;
}

// ---------------------------------------------------------------------------
// K1 router_topk: one CTA per token.  Warps compute the E logits with the
// fixed-order dot product; thread 0 selects the top-k by (logit desc, index
// asc) and forms the softmax weights with det_exp and sequential sums.
// ---------------------------------------------------------------------------
constexpr int kRouterThreads = 256;
constexpr int kMaxExperts = 256;

__global__ void __launch_bounds__(kRouterThreads)
router_topk_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ wg, int H,
                   int E, int k, int renorm, float* __restrict__ weights,
                   int32_t* __restrict__ idx, float* __restrict__ logits_out,
                   int32_t* __restrict__ host_idx, const uint16_t* __restrict__ sg_w,
                   float* __restrict__ shared_gate) {
  __shared__ float s_logit[kMaxExperts + 1];
  const int t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = kRouterThreads / 32;
  const int nchunks = H >> 3;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t)t * H);
  const int nrows = E + (sg_w != nullptr ? 1 : 0);
  for (int e = warp; e < nrows; e += nwarps) {
    const uint16_t* wrow = (e < E) ? wg + (size_t)e * H : sg_w;
    const uint4* wr = reinterpret_cast<const uint4*>(wrow);
    float acc = 0.0f;
    // the loads of U chunk rounds are issued before any of their FMAs (one
    // memory round trip per U rounds instead of per round); the FMAs still
    // run chunk j, j+32, j+64, ... in order -- the fixed-order contract
    constexpr int U = 8;
    for (int c0 = lane; c0 < nchunks; c0 += 32 * U) {
      uint4 xa[U], wb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        if (c < nchunks) {
          xa[u] = __ldg(xr + c);
          wb[u] = __ldg(wr + c);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c0 + 32 * u < nchunks) {
          float a[8], b[8];
          unpack8(xa[u], a);
          unpack8(wb[u], b);
#pragma unroll
          for (int v = 0; v < 8; ++v) acc = fmaf(a[v], b[v], acc);  // exact products
        }
      }
    }
    acc = warp_sum_fixed(acc);
    if (lane == 0) s_logit[e] = acc;
  }
  __syncthreads();
  __shared__ int s_sel[kMaxExperts];
  if (warp == 0) {
    // top-k by warp argmax rounds: value descending, lowest index on ties
    // (the strictly-greater scan of the oracle), E <= 256 = 8 per lane
    uint32_t taken = 0;  // bit j: expert lane + 32 j already selected
    for (int i = 0; i < k; ++i) {
      float bv = 0.0f;
      int best = -1;
      for (int j = 0; j < (E + 31) / 32; ++j) {
        const int e = lane + 32 * j;
        if (e < E && !(taken & (1u << j))) {
          const float v = s_logit[e];
          if (best < 0 || v > bv) { best = e; bv = v; }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(SPMOE_FULL_MASK, bv, o);
        const int oe = __shfl_xor_sync(SPMOE_FULL_MASK, best, o);
        if (oe >= 0 && (best < 0 || ov > bv || (ov == bv && oe < best))) { best = oe; bv = ov; }
      }
      if ((best & 31) == lane) taken |= 1u << (best >> 5);
      if (lane == 0) s_sel[i] = best;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (logits_out != nullptr)
      for (int e = 0; e < E; ++e) logits_out[(size_t)t * E + e] = s_logit[e];
    if (sg_w != nullptr && shared_gate != nullptr)
      shared_gate[t] = __fdiv_rn(1.0f, __fadd_rn(1.0f, det_exp(-s_logit[E])));
    const int* sel = s_sel;
    const float m = s_logit[sel[0]];
    float sum = 0.0f;
    if (renorm) {
      for (int i = 0; i < k; ++i) sum = __fadd_rn(sum, det_exp(__fsub_rn(s_logit[sel[i]], m)));
    } else {
      for (int e = 0; e < E; ++e) sum = __fadd_rn(sum, det_exp(__fsub_rn(s_logit[e], m)));
    }
    for (int i = 0; i < k; ++i) {
      const float ex = det_exp(__fsub_rn(s_logit[sel[i]], m));
      weights[(size_t)t * k + i] = __fdiv_rn(ex, sum);
      idx[(size_t)t * k + i] = sel[i];
      if (host_idx != nullptr) host_idx[(size_t)t * k + i] = sel[i];
    }
    // make the zero-copy indices visible to the host before any later
    // signal (spmoe_signal_bump) can be observed
    if (host_idx != nullptr) __threadfence_system();
  }
}

// Host-visible completion counter in mapped pinned memory: stream-ordered
// after the kernels whose results the host waits for; graph-capturable (the
// increment happens on the device at replay time).
__global__ void signal_bump_kernel(volatile int32_t* flag) {
  __threadfence_system();
  *flag = *flag + 1;
  __threadfence_system();
}

// ---------------------------------------------------------------------------
// K2 moe_permute: single CTA; thread e owns expert e and scans the routed
// (token, choice) pairs in order, so the permutation is stable by token.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
moe_permute_kernel(const int32_t* __restrict__ idx, int T, int k, int E,
                   int32_t* __restrict__ offsets, int32_t* __restrict__ perm_token,
                   int32_t* __restrict__ inv_pos) {
  __shared__ int s_cnt[kMaxExperts + 1];
  const int n = T * k;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int c = 0;
    for (int j = 0; j < n; ++j) c += (idx[j] == e);
    s_cnt[e] = c;
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int e = idx[j];
    if (e < 0 || e >= E) inv_pos[j] = -1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      const int c = s_cnt[e];
      s_cnt[e] = acc;
      offsets[e] = acc;
      acc += c;
    }
    offsets[E] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int p = s_cnt[e];
    for (int j = 0; j < n; ++j) {
      if (idx[j] == e) {
        perm_token[p] = j / k;
        inv_pos[j] = p;
        ++p;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3 expert_ffn.  Weight-streaming grouped SwiGLU: every warp owns whole
// weight rows (one row of W1 and the matching row of W3 in the up phase, one
// row of W2 in the down phase) and streams them once from HBM with 16-byte
// no-allocate loads, UNR loads in flight per lane; the routed tokens'
// activations are re-read through L1.  Rows of all active experts are laid
// end to end and dealt round-robin to the global warp index, so the load is
// balanced to one row across the 148 SMs.  Dot products follow the fixed
// order of the determinism contract (lane-strided chunks, butterfly).
// ---------------------------------------------------------------------------
constexpr int kFfnThreads = 512;
constexpr int kMaxFfnExperts = 64;

struct FfnParams {
  const uint16_t* pool;
  int64_t slot_elems;
  uint64_t mask;
  const uint16_t* x;       // up: [T, H] activations
  const uint16_t* h;       // down: [T*k, F] SwiGLU activations
  uint16_t* h_out;         // up output
  float* y;                // down output [T*k, H]
  const int32_t* offsets;  // [E+1]
  const int32_t* perm;     // [T*k]
  int T, H, F, E, k;
  int slot[kMaxFfnExperts];
};

// Collect the active experts (mask bit set and at least one routed row) into
// shared memory; returns their count.
__device__ __forceinline__ int gather_active(const FfnParams& p, int* s_active, int* s_off) {
  __shared__ int s_n;
  if (threadIdx.x < 32) {
    int base = 0;
    for (int e0 = 0; e0 < p.E; e0 += 32) {
      const int e = e0 + threadIdx.x;
      bool on = false;
      int o0 = 0, o1 = 0;
      if (e < p.E) {
        o0 = p.offsets[e];
        o1 = p.offsets[e + 1];
        on = ((p.mask >> e) & 1ull) && (o1 > o0);
      }
      const unsigned b = __ballot_sync(SPMOE_FULL_MASK, on);
      if (on) {
        const int pos = base + __popc(b & ((1u << threadIdx.x) - 1u));
        s_active[pos] = e;
      }
      if (e < p.E) { s_off[e] = o0; s_off[e + 1] = o1; }
      base += __popc(b);
    }
    if (threadIdx.x == 0) s_n = base;
  }
  __syncthreads();
  return s_n;
}

// One warp row: acc[r][t] += dot(weight row r, activation row t) over nchunks
// 16-byte chunks in the lane-strided fixed order; weights stream from HBM
// straight into registers (UNR chunks per row in flight per lane), the
// activation chunks come from the CTA's shared-memory stage.
template <int TT, int NR, int UNR>
__device__ __forceinline__ void stream_rows(const uint4* const (&wr)[NR], const uint4* act, int act_stride,
                                            int nt, int nchunks, int lane, float (&acc)[NR][TT]) {
  for (int base = 0; base < nchunks; base += 32 * UNR) {
    uint4 w[NR][UNR];
#pragma unroll
    for (int i = 0; i < UNR; ++i) {
      const int c = base + lane + 32 * i;
#pragma unroll
      for (int r = 0; r < NR; ++r)
        w[r][i] = (c < nchunks) ? ldg_stream(wr[r] + c) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < UNR; ++i) {
      const int c = base + lane + 32 * i;
      if (c < nchunks) {
        float wf[NR][8];
#pragma unroll
        for (int r = 0; r < NR; ++r) unpack8(w[r][i], wf[r]);
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          if (t < nt) {
            float af[8];
            unpack8(act[t * act_stride + c], af);
#pragma unroll
            for (int v = 0; v < 8; ++v)
#pragma unroll
              for (int r = 0; r < NR; ++r) acc[r][t] = fmaf(wf[r][v], af[v], acc[r][t]);
          }
        }
      }
    }
  }
}

// Same dot products with the activations pre-widened to fp32 in shared
// memory (two float4 planes per 16-byte chunk: elements 0-3 and 4-7, so the
// lanes' loads stay contiguous): no per-row bf16 unpack of the activations,
// identical FMA order.
template <int UNR>
__device__ __forceinline__ void load_round(const uint4* wr, int base, int nchunks, int lane, uint4 (&w)[UNR]) {
#pragma unroll
  for (int i = 0; i < UNR; ++i) {
    const int c = base + lane + 32 * i;
    w[i] = (c < nchunks) ? ldg_stream(wr + c) : make_uint4(0u, 0u, 0u, 0u);
  }
}

// Two weight rows per pass sharing every activation load (half the shared-
// memory traffic per row); each row's FMA chains keep their order.  Software
// pipelined: round r+1's loads are issued before round r's FMAs.
template <int TT, int UNR>
__device__ __forceinline__ void stream_rows2_f32(const uint4* wr0, const uint4* wr1, const float4* act, int nchunks,
                                                 int lane, float (&acc0)[TT], float (&acc1)[TT],
                                                 uint4 (&w0)[UNR], uint4 (&w1)[UNR]) {
  // w0 / w1 arrive holding round 0 (the caller may have issued it early)
  for (int base = 0; base < nchunks; base += 32 * UNR) {
    uint4 n0[UNR], n1[UNR];
    load_round<UNR>(wr0, base + 32 * UNR, nchunks, lane, n0);
    load_round<UNR>(wr1, base + 32 * UNR, nchunks, lane, n1);
#pragma unroll
    for (int i = 0; i < UNR; ++i) {
      const int c = base + lane + 32 * i;
      if (c < nchunks) {
        float wf0[8], wf1[8];
        unpack8(w0[i], wf0);
        unpack8(w1[i], wf1);
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const float4 a0 = act[(2 * t) * nchunks + c], a1 = act[(2 * t + 1) * nchunks + c];
          const float af[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            acc0[t] = fmaf(wf0[v], af[v], acc0[t]);
            acc1[t] = fmaf(wf1[v], af[v], acc1[t]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < UNR; ++i) {
      w0[i] = n0[i];
      w1[i] = n1[i];
    }
  }
}

template <int TT, int UNR, bool FULL>
__device__ __forceinline__ void stream_rows_f32(const uint4* wr, const float4* act, int nchunks, int nt, int lane,
                                                float (&acc)[TT]) {
  uint4 w[UNR];
  load_round<UNR>(wr, 0, nchunks, lane, w);
  for (int base = 0; base < nchunks; base += 32 * UNR) {
    uint4 nw[UNR];
    load_round<UNR>(wr, base + 32 * UNR, nchunks, lane, nw);
#pragma unroll
    for (int i = 0; i < UNR; ++i) {
      const int c = base + lane + 32 * i;
      if (c < nchunks) {
        float wf[8];
        unpack8(w[i], wf);
        if (FULL) {
          // every token row present: no branches, the TT independent FMA
          // chains interleave (each keeps its own element order)
          float af[TT][8];
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            const float4 a0 = act[(2 * t) * nchunks + c], a1 = act[(2 * t + 1) * nchunks + c];
            af[t][0] = a0.x; af[t][1] = a0.y; af[t][2] = a0.z; af[t][3] = a0.w;
            af[t][4] = a1.x; af[t][5] = a1.y; af[t][6] = a1.z; af[t][7] = a1.w;
          }
#pragma unroll
          for (int v = 0; v < 8; ++v)
#pragma unroll
            for (int t = 0; t < TT; ++t) acc[t] = fmaf(wf[v], af[t][v], acc[t]);
        } else {
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            if (t < nt) {
              const float4 a0 = act[(2 * t) * nchunks + c], a1 = act[(2 * t + 1) * nchunks + c];
              const float af[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
              for (int v = 0; v < 8; ++v) acc[t] = fmaf(wf[v], af[v], acc[t]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < UNR; ++i) w[i] = nw[i];
  }
}

// K3 phase kernel.  UP: rows f of W1 and W3 (NR=2, K=H) -> h = bf16(silu(g)*u);
// DOWN: rows h of W2 (NR=1, K=F) -> y fp32.  The (active expert, 16-row
// tile) space is split into one contiguous range per CTA (balanced to one
// tile, at most a couple of expert switches per CTA); a switch restages the
// expert's routed-token activations [TT][K] in shared memory.  Warp w owns
// row w of every tile.
template <bool UP, int TT>
__global__ void __launch_bounds__(kFfnThreads, 1) ffn_kernel(const FfnParams p) {
  extern __shared__ __align__(16) uint4 s_act[];
  __shared__ int s_active[kMaxFfnExperts];
  __shared__ int s_off[kMaxFfnExperts + 1];
  constexpr int NR = UP ? 2 : 1;
  constexpr int UNR = UP ? 8 : 16;
  constexpr int kRowsPerTile = kFfnThreads / 32;
  const int n_active = gather_active(p, s_active, s_off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = UP ? p.H : p.F;            // reduction length
  const int R = UP ? p.F : p.H;            // rows per expert
  const int nchunks = K >> 3;
  const int tpe = (R + kRowsPerTile - 1) / kRowsPerTile;
  const int64_t total = (int64_t)n_active * tpe;
  const int64_t t_begin = total * blockIdx.x / gridDim.x;
  const int64_t t_end = total * (blockIdx.x + 1) / gridDim.x;
  int cur_e = -1, cur_t0 = -1;
  for (int64_t tile = t_begin; tile < t_end; ++tile) {
    const int a = (int)(tile / tpe);
    const int row = (int)(tile - (int64_t)a * tpe) * kRowsPerTile + warp;
    const int e = s_active[a];
    const int off = s_off[e];
    const int cnt = s_off[e + 1] - off;
    const uint16_t* blob = p.pool + (int64_t)p.slot[e] * p.slot_elems;
    for (int t0 = 0; t0 < cnt; t0 += TT) {
      const int nt = min(TT, cnt - t0);
      if (e != cur_e || t0 != cur_t0) {
        __syncthreads();  // every warp is done with the previous stage
        for (int q = threadIdx.x; q < nt * nchunks; q += kFfnThreads) {
          const int t = q / nchunks, c = q - t * nchunks;
          const uint16_t* src = UP ? p.x + (int64_t)p.perm[off + t0 + t] * p.H
                                   : p.h + (int64_t)(off + t0 + t) * p.F;
          s_act[t * nchunks + c] = __ldg(reinterpret_cast<const uint4*>(src) + c);
        }
        __syncthreads();
        cur_e = e;
        cur_t0 = t0;
      }
      if (row >= R) continue;
      const uint4* wr[NR];
      if (UP) {
        wr[0] = reinterpret_cast<const uint4*>(blob + (int64_t)row * p.H);
        wr[NR - 1] = reinterpret_cast<const uint4*>(blob + ((int64_t)p.F + row) * p.H);
      } else {
        wr[0] = reinterpret_cast<const uint4*>(blob + 2 * (int64_t)p.F * p.H + (int64_t)row * p.F);
      }
      float acc[NR][TT];
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int t = 0; t < TT; ++t) acc[r][t] = 0.0f;
      stream_rows<TT, NR, UNR>(wr, s_act, nchunks, nt, nchunks, lane, acc);
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        if (t < nt) {
          const float s0 = warp_sum_fixed(acc[0][t]);
          if (UP) {
            const float s1 = warp_sum_fixed(acc[NR - 1][t]);
            if (lane == t) {
              const float hv = __fmul_rn(det_silu(s0), s1);
              p.h_out[(int64_t)(off + t0 + t) * p.F + row] = f32_to_bf16(hv);
            }
          } else if (lane == t) {
            p.y[(int64_t)(off + t0 + t) * p.H + row] = s0;
          }
        }
      }
    }
  }
}

constexpr int kActSmemCap = 200 * 1024;

// ---------------------------------------------------------------------------
// K9 linear: y[t][n] = dot_fixed(W[n,:], x[t,:]) for the projections around
// the MoE (fused qkv, W_o, lm_head) -- the same weight-streaming warp-per-row
// scheme and fixed reduction order as K3's down phase, so the whole forward
// (not just the MoE) is reproducible on the CPU oracle bit for bit.  Rows are
// dealt in 16-row tiles, one contiguous tile range per CTA; the T activation
// rows are staged in shared memory TT at a time (prefill re-streams the
// weights once per TT-token group).
//
// Optional fused pieces, each with the arithmetic of its standalone kernel:
//   norm_w != null : stage RMSNorm(x) (rms_norm_kernel's exact arithmetic)
//                    instead of x -- norm -> projection in one launch;
//   resid  != null : out = bf16(resid + bf16(y)) (the residual add of the
//                    torch graph `x = x + proj(o)`), else out = bf16(y);
//   y_f32  != null : raw fp32 dot products (lm_head logits).
// ---------------------------------------------------------------------------
struct LinParams {
  const uint16_t* w;     // [N, K]
  const uint16_t* x;     // [T, K] (row stride ldx elements)
  const uint16_t* norm_w;
  float eps;
  int64_t ldx;
  int T, K, N;
  float* y_f32;          // [T, ldy]
  int64_t ldy;
  uint16_t* y_bf16;      // [T, N]
  const uint16_t* resid; // [T, N] (may alias y_bf16)
};

// Fixed-order RMSNorm scale of one row (one warp): ss = dot_fixed(x, x),
// r = 1 / sqrt(ss / H + eps) with IEEE division and square root.
__device__ __forceinline__ float rms_scale_row(const uint4* xr, int nchunks, int H, float eps, int lane) {
  float acc = 0.0f;
  // loads of U rounds issued before their FMAs; FMA order unchanged
  constexpr int U = 8;
  for (int c0 = lane; c0 < nchunks; c0 += 32 * U) {
    uint4 xa[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + 32 * u < nchunks) xa[u] = __ldg(xr + c0 + 32 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c0 + 32 * u < nchunks) {
        float a[8];
        unpack8(xa[u], a);
#pragma unroll
        for (int v = 0; v < 8; ++v) acc = fmaf(a[v], a[v], acc);  // exact squares
      }
    }
  }
  acc = warp_sum_fixed(acc);
  const float mean = __fdiv_rn(acc, (float)H);
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(mean, eps)));
}

// y = bf16((x * r) * w), two IEEE products.
__device__ __forceinline__ uint32_t rms_apply2(uint32_t xw, uint32_t gw, float r) {
  const float lo = __fmul_rn(__fmul_rn(bf16_lo(xw), r), bf16_lo(gw));
  const float hi = __fmul_rn(__fmul_rn(bf16_hi(xw), r), bf16_hi(gw));
  return (uint32_t)f32_to_bf16(lo) | ((uint32_t)f32_to_bf16(hi) << 16);
}

template <int TT>
__global__ void __launch_bounds__(kFfnThreads, 1) linear_kernel(const LinParams p) {
  // activations widened to fp32: plane 2t (elements 0-3 of every chunk) and
  // plane 2t+1 (elements 4-7) of token t
  extern __shared__ __align__(16) float4 s_actf[];
  __shared__ float s_r[TT];
  constexpr int kRowsPerTile = kFfnThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nchunks = p.K >> 3;
  const int r_begin = (int)((int64_t)p.N * blockIdx.x / gridDim.x);
  const int r_end = (int)((int64_t)p.N * (blockIdx.x + 1) / gridDim.x);
  constexpr int U2 = TT <= 2 ? 4 : 2;  // pair rounds (more would spill at TT >= 3)
  // Launched with programmatic stream serialization: the weights are not
  // written by the preceding kernel, so the first two rounds of this warp's
  // first row pair are requested into L2 before the grid dependency (x,
  // resid) resolves -- while the previous kernel drains and during the
  // activation stage below.
  grid_dep_trigger();
  {
    const int row0 = r_begin + warp;
    if (row0 + kRowsPerTile < r_end) {
      const uint4* a = reinterpret_cast<const uint4*>(p.w + (int64_t)row0 * p.K);
      const uint4* b = reinterpret_cast<const uint4*>(p.w + (int64_t)(row0 + kRowsPerTile) * p.K);
#pragma unroll
      for (int i = 0; i < 2 * U2; ++i) {
        const int c = lane + 32 * i;
        if (c < nchunks) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a + c));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(b + c));
        }
      }
    }
  }
  grid_dep_wait();
  if (r_begin >= r_end) return;
  for (int t0 = 0; t0 < p.T; t0 += TT) {
    const int nt = min(TT, p.T - t0);
    __syncthreads();  // previous group's readers are done
    if (p.norm_w != nullptr) {
      for (int t = warp; t < nt; t += kFfnThreads / 32)
        s_r[t] = rms_scale_row(reinterpret_cast<const uint4*>(p.x + (int64_t)(t0 + t) * p.ldx), nchunks, p.K,
                               p.eps, lane);
      __syncthreads();
    }
    for (int q = threadIdx.x; q < nt * nchunks; q += kFfnThreads) {
      const int t = q / nchunks, c = q - t * nchunks;
      uint4 v = __ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)(t0 + t) * p.ldx) + c);
      if (p.norm_w != nullptr) {
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(p.norm_w) + c);
        const float r = s_r[t];
        v = make_uint4(rms_apply2(v.x, g.x, r), rms_apply2(v.y, g.y, r), rms_apply2(v.z, g.z, r),
                       rms_apply2(v.w, g.w, r));
      }
      float f[8];
      unpack8(v, f);
      s_actf[(2 * t) * nchunks + c] = make_float4(f[0], f[1], f[2], f[3]);
      s_actf[(2 * t + 1) * nchunks + c] = make_float4(f[4], f[5], f[6], f[7]);
    }
    __syncthreads();
    // this CTA's rows [r_begin, r_end); warp w takes rows r_begin + w + 16 k,
    // two at a time while it has two (full token groups), else one
    auto emit = [&](int row, const float (&acc)[TT]) {
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        if (t < nt) {
          const float sum = warp_sum_fixed(acc[t]);
          if (lane == t) {
            const int64_t tt = t0 + t;
            if (p.y_f32 != nullptr) p.y_f32[tt * p.ldy + row] = sum;
            if (p.y_bf16 != nullptr) {
              uint16_t o = f32_to_bf16(sum);
              if (p.resid != nullptr)
                o = f32_to_bf16(__fadd_rn(bf16_to_f32(p.resid[tt * p.N + row]), bf16_to_f32(o)));
              p.y_bf16[tt * p.N + row] = o;
            }
          }
        }
      }
    };
    int row = r_begin + warp;
    if (nt == TT) {
      for (; row + kRowsPerTile < r_end; row += 2 * kRowsPerTile) {
        float acc0[TT], acc1[TT];
#pragma unroll
        for (int t = 0; t < TT; ++t) acc0[t] = acc1[t] = 0.0f;
        const uint4* w0p = reinterpret_cast<const uint4*>(p.w + (int64_t)row * p.K);
        const uint4* w1p = reinterpret_cast<const uint4*>(p.w + (int64_t)(row + kRowsPerTile) * p.K);
        uint4 w0[U2], w1[U2];
        load_round<U2>(w0p, 0, nchunks, lane, w0);
        load_round<U2>(w1p, 0, nchunks, lane, w1);
        stream_rows2_f32<TT, U2>(w0p, w1p, s_actf, nchunks, lane, acc0, acc1, w0, w1);
        emit(row, acc0);
        emit(row + kRowsPerTile, acc1);
      }
    }
    for (; row < r_end; row += kRowsPerTile) {
      const uint4* wr = reinterpret_cast<const uint4*>(p.w + (int64_t)row * p.K);
      float acc[TT];
#pragma unroll
      for (int t = 0; t < TT; ++t) acc[t] = 0.0f;
      if (nt == TT)
        stream_rows_f32<TT, (TT <= 2 ? 8 : 4), true>(wr, s_actf, nchunks, nt, lane, acc);
      else
        stream_rows_f32<TT, (TT <= 2 ? 8 : 4), false>(wr, s_actf, nchunks, nt, lane, acc);
      emit(row, acc);
    }
  }
}

template <int TT>
int launch_linear(const LinParams& p, cudaStream_t s) {
  const size_t smem = (size_t)TT * p.K * 4;  // fp32 activation stage
  if (smem > (size_t)kActSmemCap) return (int)cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(linear_kernel<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kActSmemCap);
    configured = true;
  }
  const int tiles = (p.N + 15) / 16;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFfnThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const int no_pdl = getenv("SPMOE_NO_PDL") != nullptr;  // A/B switch
  cfg.numAttrs = no_pdl ? 0 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, linear_kernel<TT>, p);
  return e != cudaSuccess ? (int)e : launch_status();
}

// Register tile: the smallest of 1/2/4/8 covering the hint that also fits
// the activation stage (TT x K bf16) in shared memory.
int pick_tile(int hint, int K) {
  int tt = hint <= 0 ? 8 : hint <= 1 ? 1 : hint <= 2 ? 2 : hint <= 4 ? 4 : 8;
  while (tt > 1 && (size_t)tt * K * 2 > (size_t)kActSmemCap) tt >>= 1;
  return tt;
}

template <bool UP, int TT>
int launch_ffn(const FfnParams& p, cudaStream_t s) {
  const int K = UP ? p.H : p.F;
  const size_t smem = (size_t)TT * K * 2;
  if (smem > (size_t)kActSmemCap) return (int)cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ffn_kernel<UP, TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kActSmemCap);
    configured = true;
  }
  ffn_kernel<UP, TT><<<num_sms(), kFfnThreads, smem, s>>>(p);
  return launch_status();
}

template <bool UP>
int launch_ffn_tt(const FfnParams& p, int hint, cudaStream_t s) {
  switch (pick_tile(hint, UP ? p.H : p.F)) {
    case 1: return launch_ffn<UP, 1>(p, s);
    case 2: return launch_ffn<UP, 2>(p, s);
    case 4: return launch_ffn<UP, 4>(p, s);
    default: return launch_ffn<UP, 8>(p, s);
  }
}

bool fill_params(FfnParams& p, const uint16_t* pool, int64_t slot_elems,
                 const int32_t* slot_of_expert, uint64_t mask, int T, int H, int F, int E, int k,
                 const int32_t* offsets, const int32_t* perm) {
  if (pool == nullptr || slot_of_expert == nullptr || offsets == nullptr) return false;
  if (T < 0 || H <= 0 || F <= 0 || E <= 0 || E > kMaxFfnExperts || k <= 0) return false;
  if ((H & 7) || (F & 7)) return false;
  p.pool = pool;
  p.slot_elems = slot_elems;
  p.mask = mask;
  p.offsets = offsets;
  p.perm = perm;
  p.T = T; p.H = H; p.F = F; p.E = E; p.k = k;
  for (int e = 0; e < E; ++e) p.slot[e] = ((mask >> e) & 1ull) ? slot_of_expert[e] : 0;
  for (int e = E; e < kMaxFfnExperts; ++e) p.slot[e] = 0;
  return true;
}

// ---------------------------------------------------------------------------
// K4 moe_combine: one thread per 4 consecutive hidden elements.
// ---------------------------------------------------------------------------
__global__ void moe_combine_kernel(const float* __restrict__ y, const int32_t* __restrict__ inv_pos,
                                   const float* __restrict__ w, int H, int k,
                                   const float* __restrict__ ys, const float* __restrict__ sg,
                                   const uint16_t* residual, uint16_t* out) {
  grid_dep_trigger();  // a following K9 may start streaming its weights
  const int t = blockIdx.y;
  const int h0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (h0 >= H) return;
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int i = 0; i < k; ++i) {
    const int pos = inv_pos[t * k + i];
    if (pos < 0) continue;
    const float wi = (w != nullptr) ? w[t * k + i] : 1.0f;
    const float4 v = *reinterpret_cast<const float4*>(y + (int64_t)pos * H + h0);
    acc[0] = __fadd_rn(acc[0], __fmul_rn(wi, v.x));
    acc[1] = __fadd_rn(acc[1], __fmul_rn(wi, v.y));
    acc[2] = __fadd_rn(acc[2], __fmul_rn(wi, v.z));
    acc[3] = __fadd_rn(acc[3], __fmul_rn(wi, v.w));
  }
  if (ys != nullptr) {
    const float g = (sg != nullptr) ? sg[t] : 1.0f;
    const float4 v = *reinterpret_cast<const float4*>(ys + (int64_t)t * H + h0);
    acc[0] = __fadd_rn(acc[0], __fmul_rn(g, v.x));
    acc[1] = __fadd_rn(acc[1], __fmul_rn(g, v.y));
    acc[2] = __fadd_rn(acc[2], __fmul_rn(g, v.z));
    acc[3] = __fadd_rn(acc[3], __fmul_rn(g, v.w));
  }
  uint16_t o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float r = (residual != nullptr) ? bf16_to_f32(residual[(int64_t)t * H + h0 + j]) : 0.0f;
    o[j] = f32_to_bf16(residual != nullptr ? __fadd_rn(r, acc[j]) : acc[j]);
  }
  uint2 packed;
  packed.x = (uint32_t)o[0] | ((uint32_t)o[1] << 16);
  packed.y = (uint32_t)o[2] | ((uint32_t)o[3] << 16);
  *reinterpret_cast<uint2*>(out + (int64_t)t * H + h0) = packed;
}

// ---------------------------------------------------------------------------
// K6 greedy acceptance: row argmax (ties -> lowest index), then the longest
// matching prefix per sequence.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  // total order: larger value first, then lower index; NaN never wins
  if (v != v) return false;
  if (bv != bv) return true;
  return (v > bv) || (v == bv && i < bi);
}

__global__ void __launch_bounds__(1024)
argmax_rows_kernel(const float* __restrict__ logits, int64_t ld, int V, int32_t* __restrict__ out) {
  __shared__ float s_v[32];
  __shared__ int s_i[32];
  const float* row = logits + (int64_t)blockIdx.x * ld;
  float bv = __uint_as_float(0x7fc00000u);
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = row[i];
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const float ov = __shfl_xor_sync(SPMOE_FULL_MASK, bv, off);
    const int oi = __shfl_xor_sync(SPMOE_FULL_MASK, bi, off);
    if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_v[warp] = bv; s_i[warp] = bi; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    bv = (lane < nw) ? s_v[lane] : __uint_as_float(0x7fc00000u);
    bi = (lane < nw) ? s_i[lane] : 0x7fffffff;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const float ov = __shfl_xor_sync(SPMOE_FULL_MASK, bv, off);
      const int oi = __shfl_xor_sync(SPMOE_FULL_MASK, bi, off);
      if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) out[blockIdx.x] = (bi == 0x7fffffff) ? 0 : bi;
  }
}

__global__ void accept_prefix_kernel(const int32_t* __restrict__ amax, const int32_t* __restrict__ draft,
                                     int B, int N, int32_t* __restrict__ result) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int a = 0;
  while (a < N && draft[b * N + a] == amax[b * (N + 1) + a]) ++a;
  result[b * 2 + 0] = a;
  result[b * 2 + 1] = amax[b * (N + 1) + a];
}

// ---------------------------------------------------------------------------
// Deterministic init: splitmix64 counter hash -> Irwin-Hall(4) normal.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_normal_kernel(uint16_t* __restrict__ dst, int64_t n, uint64_t seed,
                                   uint64_t offset, float scale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t hsh = splitmix64(seed ^ splitmix64(offset + (uint64_t)i));
    const int s = (int)(hsh & 0xffff) + (int)((hsh >> 16) & 0xffff) +
                  (int)((hsh >> 32) & 0xffff) + (int)(hsh >> 48);
    dst[i] = f32_to_bf16(__fmul_rn((float)(s - 131070), scale));
  }
}

// ---------------------------------------------------------------------------
// Row gather for the expert-parallel exchange: dst[j] = src[idx[j] / div].
// W = 16-byte words when rows allow it, else 4-byte words; one CTA per row
// batch, consecutive threads on consecutive words (coalesced).
// ---------------------------------------------------------------------------
template <typename W>
__global__ void gather_rows_kernel(const W* __restrict__ src, const int32_t* __restrict__ idx, int n,
                                   int div, int64_t words, W* __restrict__ dst) {
  for (int j = blockIdx.x; j < n; j += gridDim.x) {
    const int64_t r = idx[j] / div;
    const W* s = src + r * words;
    W* d = dst + (int64_t)j * words;
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) d[w] = s[w];
  }
}

}  // namespace

K3Timing& spmoe::k3_timing() {
  static thread_local K3Timing t;
  return t;
}

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int spmoe_abi_version(void) { return 100; }

const char* spmoe_status_string(int status) {
  if (status == -1) return "spmoe: cache contract violation (CacheError)";
  return cudaGetErrorString((cudaError_t)status);
}

int spmoe_router_topk(const uint16_t* x, const uint16_t* w_gate, int T, int H, int E, int k,
                      int renorm, float* weights, int32_t* idx, float* logits, int32_t* host_idx,
                      const uint16_t* shared_gate_w, float* shared_gate, void* stream) {
  if (T < 0 || H <= 0 || (H & 7) || E <= 0 || E > kMaxExperts || k < 1 || k > E)
    return (int)cudaErrorInvalidValue;
  if (T == 0) return 0;
  if (!x || !w_gate || !weights || !idx) return (int)cudaErrorInvalidValue;
  router_topk_kernel<<<T, kRouterThreads, 0, (cudaStream_t)stream>>>(
      x, w_gate, H, E, k, renorm, weights, idx, logits, host_idx, shared_gate_w, shared_gate);
  return launch_status();
}

int spmoe_moe_permute(const int32_t* idx, int T, int k, int E, int32_t* expert_offsets,
                      int32_t* perm_token, int32_t* inv_pos, void* stream) {
  if (T < 0 || k < 1 || E < 1 || E > kMaxExperts) return (int)cudaErrorInvalidValue;
  if (!expert_offsets) return (int)cudaErrorInvalidValue;
  if (T > 0 && (!idx || !perm_token || !inv_pos)) return (int)cudaErrorInvalidValue;
  moe_permute_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(idx, T, k, E, expert_offsets,
                                                          perm_token, inv_pos);
  return launch_status();
}

int spmoe_expert_ffn_up(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                        uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E,
                        int k, const int32_t* expert_offsets, const int32_t* perm_token,
                        uint16_t* h_scratch, int max_tokens_per_expert, void* stream) {
  FfnParams p{};
  if (!fill_params(p, pool, slot_elems, slot_of_expert, expert_mask, T, H, F, E, k,
                   expert_offsets, perm_token))
    return (int)cudaErrorInvalidValue;
  if (T == 0 || expert_mask == 0) return 0;
  if (!x || !perm_token || !h_scratch) return (int)cudaErrorInvalidValue;
  p.x = x;
  p.h_out = h_scratch;
  const int grid = num_sms();
  cudaStream_t s = (cudaStream_t)stream;
  (void)grid;
  return launch_ffn_tt<true>(p, max_tokens_per_expert, s);
}

int spmoe_expert_ffn_down(const uint16_t* pool, int64_t slot_elems,
                          const int32_t* slot_of_expert, uint64_t expert_mask, int T, int H,
                          int F, int E, int k, const int32_t* expert_offsets,
                          const uint16_t* h_scratch, float* y, int max_tokens_per_expert,
                          void* stream) {
  FfnParams p{};
  if (!fill_params(p, pool, slot_elems, slot_of_expert, expert_mask, T, H, F, E, k,
                   expert_offsets, nullptr))
    return (int)cudaErrorInvalidValue;
  if (T == 0 || expert_mask == 0) return 0;
  if (!h_scratch || !y) return (int)cudaErrorInvalidValue;
  p.h = h_scratch;
  p.y = y;
  const int grid = num_sms();
  cudaStream_t s = (cudaStream_t)stream;
  (void)grid;
  return launch_ffn_tt<false>(p, max_tokens_per_expert, s);
}

int spmoe_expert_ffn(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                     uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E, int k,
                     const int32_t* expert_offsets, const int32_t* perm_token,
                     uint16_t* h_scratch, float* y, int max_tokens_per_expert, void* stream) {
  const K3Timing tm = k3_timing();
  k3_timing() = K3Timing{};
  if (tm.start) cudaEventRecord(tm.start, (cudaStream_t)stream);
  int st = spmoe_expert_ffn_up(pool, slot_elems, slot_of_expert, expert_mask, x, T, H, F, E, k,
                               expert_offsets, perm_token, h_scratch, max_tokens_per_expert,
                               stream);
  if (st) return st;
  st = spmoe_expert_ffn_down(pool, slot_elems, slot_of_expert, expert_mask, T, H, F, E, k,
                             expert_offsets, h_scratch, y, max_tokens_per_expert, stream);
  if (tm.end) cudaEventRecord(tm.end, (cudaStream_t)stream);
  return st;
}

int spmoe_linear(const uint16_t* w, const uint16_t* x, int64_t ldx, int T, int K, int N,
                 const uint16_t* norm_w, float eps, float* y_f32, int64_t ldy, uint16_t* y_bf16,
                 const uint16_t* resid, void* stream) {
  if (T < 0 || K <= 0 || (K & 7) || N <= 0 || ldx < K || (ldx & 7)) return (int)cudaErrorInvalidValue;
  if (T == 0) return 0;
  if (!w || !x || (!y_f32 && !y_bf16) || (y_f32 && ldy < N) || (resid && !y_bf16))
    return (int)cudaErrorInvalidValue;
  LinParams p{};
  p.w = w; p.x = x; p.norm_w = norm_w; p.eps = eps; p.ldx = ldx;
  p.T = T; p.K = K; p.N = N;
  p.y_f32 = y_f32; p.ldy = ldy; p.y_bf16 = y_bf16; p.resid = resid;
  // the register tile matches T exactly up to 8 rows (no predicated-off
  // token lanes in the inner loop), then 16-row groups
  int tt = T <= 8 ? T : 16;
  while (tt > 1 && (size_t)tt * K * 4 > (size_t)kActSmemCap) tt = tt > 8 ? 8 : tt / 2;
  cudaStream_t s = (cudaStream_t)stream;
  switch (tt) {
    case 1: return launch_linear<1>(p, s);
    case 2: return launch_linear<2>(p, s);
    case 3: return launch_linear<3>(p, s);
    case 4: return launch_linear<4>(p, s);
    case 5: return launch_linear<5>(p, s);
    case 6: return launch_linear<6>(p, s);
    case 7: return launch_linear<7>(p, s);
    case 8: return launch_linear<8>(p, s);
    default: return launch_linear<16>(p, s);
  }
}

int spmoe_gather_rows(const void* src, const int32_t* idx, int n, int div, int64_t row_bytes,
                      void* dst, void* stream) {
  if (n < 0 || div < 1 || row_bytes <= 0 || (row_bytes & 3)) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  if (!src || !idx || !dst) return (int)cudaErrorInvalidValue;
  const int grid = n < 4 * num_sms() ? n : 4 * num_sms();
  cudaStream_t s = (cudaStream_t)stream;
  const bool vec = !(row_bytes & 15) && !((uintptr_t)src & 15) && !((uintptr_t)dst & 15);
  if (vec)
    gather_rows_kernel<uint4><<<grid, 256, 0, s>>>((const uint4*)src, idx, n, div, row_bytes / 16,
                                                   (uint4*)dst);
  else
    gather_rows_kernel<uint32_t><<<grid, 256, 0, s>>>((const uint32_t*)src, idx, n, div,
                                                      row_bytes / 4, (uint32_t*)dst);
  return launch_status();
}

int spmoe_k3_devtiming(void* span) {
  k3_timing().dspan = span;
  return 0;
}

int spmoe_k3_timing(void* start, void* end) {
  k3_timing().start = (cudaEvent_t)start;
  k3_timing().end = (cudaEvent_t)end;
  return 0;
}

int spmoe_moe_combine(const float* y, const int32_t* inv_pos, const float* weights, int T, int H,
                      int k, const float* y_shared, const float* shared_gate,
                      const uint16_t* residual, uint16_t* out, void* stream) {
  if (T < 0 || H <= 0 || (H & 3) || k < 0) return (int)cudaErrorInvalidValue;
  if (T == 0) return 0;
  if (!out || (k > 0 && (!y || !inv_pos))) return (int)cudaErrorInvalidValue;
  const int threads = 128;
  dim3 grid((H / 4 + threads - 1) / threads, T);
  moe_combine_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(y, inv_pos, weights, H, k,
                                                                 y_shared, shared_gate, residual,
                                                                 out);
  return launch_status();
}

int spmoe_argmax_rows(const float* logits, int64_t ld, int rows, int V, int32_t* out,
                      void* stream) {
  if (rows < 0 || V <= 0 || ld < V) return (int)cudaErrorInvalidValue;
  if (rows == 0) return 0;
  if (!logits || !out) return (int)cudaErrorInvalidValue;
  argmax_rows_kernel<<<rows, 1024, 0, (cudaStream_t)stream>>>(logits, ld, V, out);
  return launch_status();
}

int spmoe_greedy_accept(const float* logits, int64_t ld, const int32_t* draft, int B, int N,
                        int V, int32_t* argmax_out, int32_t* result, void* stream) {
  if (B < 0 || N < 0 || V <= 0 || ld < V) return (int)cudaErrorInvalidValue;
  if (B == 0) return 0;
  if (!logits || !argmax_out || !result || (N > 0 && !draft)) return (int)cudaErrorInvalidValue;
  int st = spmoe_argmax_rows(logits, ld, B * (N + 1), V, argmax_out, stream);
  if (st) return st;
  accept_prefix_kernel<<<(B + 127) / 128, 128, 0, (cudaStream_t)stream>>>(argmax_out, draft, B,
                                                                          N, result);
  return launch_status();
}

int spmoe_signal_bump(int32_t* flag, void* stream) {
  if (!flag) return (int)cudaErrorInvalidValue;
  signal_bump_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flag);
  return launch_status();
}

int spmoe_h2d_batch(void* const* dst, const void* const* src, const size_t* bytes, int n,
                    void* stream) {
  if (n < 0 || (n > 0 && (!dst || !src || !bytes))) return (int)cudaErrorInvalidValue;
  for (int i = 0; i < n; ++i) {
    cudaError_t e = cudaMemcpyAsync(dst[i], src[i], bytes[i], cudaMemcpyHostToDevice,
                                    (cudaStream_t)stream);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

int spmoe_fill_normal_bf16(uint16_t* dst, int64_t n, uint64_t seed, uint64_t offset, float std,
                           void* stream) {
  if (n < 0 || (n > 0 && !dst)) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  const float scale = std * 0x1.bb67aep-16f;  // sqrt(3)/65536, Irwin-Hall(4) -> N(0,1)
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  fill_normal_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(dst, n, seed, offset,
                                                                              scale);
  return launch_status();
}

}  // extern "C"
