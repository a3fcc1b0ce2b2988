// spmoe_codec.cu — XC, the lossless exponent coding of expert blobs that
// cross the host link (format: include/spmoe.h, "XC").
//
// Why: with an offload budget the verify stage is bound by the pinned
// host -> HBM copies of routed experts (IoChannel.transfer,
// prefetch.py:45-74; PAPER.md:242 measures expert loading at 69.4 % of
// decode latency).  Copying fewer bytes per expert is the only lever left
// once the copy engine runs at the link's peak.  A bf16 weight's 8-bit
// exponent carries ~2.5 bits of entropy, so XC sends 1 byte of
// sign|mantissa + a 2-bit exponent code (+ a 4-bit secondary code for the
// ~27 % of values outside the top-3 exponents) and the copy stream's
// decode kernel rebuilds the exact bf16 bits in the HBM slot.
//
// Kernels (all one CTA of 256 threads per 4096-value coding block; thread t
// owns values 16t..16t+15 of its block):
//   xc_hist_kernel   exponent histogram per segment (per-warp smem bins)
//   xc_count_kernel  per block: escape words and exceptions
//   xc_scan_kernel   exclusive prefix of the per-block counts (1 CTA)
//   xc_write_kernel  sign|mantissa bytes, 2-bit codes, escape nibbles,
//                    exceptions
//   xc_decode_kernel the inverse; HBM-bound (reads ~1.39 B, writes 2 B per
//                    value)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/spmoe.h"

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 16;
static_assert(kThreads * kPerThread == SPMOE_XC_BLOCK, "block geometry");
constexpr int kMaxSecWords = SPMOE_XC_BLOCK / 8;  // all values escaped
constexpr uint8_t kExcLut = (15u << 2) | 3u;

struct Lut {
  uint8_t v[256];  // (secondary code << 2) | primary code
};

// Block-wide exclusive prefix of `v` over the 256 threads; *total = sum.
__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      const int s = warp_sums[w];
      warp_sums[w] = acc;
      acc += s;
    }
    warp_sums[kThreads / 32] = acc;
  }
  __syncthreads();
  const int ex = warp_sums[warp] + inc - v;
  *total = warp_sums[kThreads / 32];
  return ex;
}

__device__ __forceinline__ void load16(const uint16_t* __restrict__ src, uint32_t (&w)[8]) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(src));
  const uint4 b = __ldg(reinterpret_cast<const uint4*>(src) + 1);
  w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
  w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}

__device__ __forceinline__ uint32_t val_of(const uint32_t (&w)[8], int j) {
  return (w[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
}

// --------------------------------------------------------------- histogram
__global__ void __launch_bounds__(kThreads) xc_hist_kernel(const uint16_t* __restrict__ src, int64_t n,
                                                           uint32_t* __restrict__ hist) {
  __shared__ uint32_t bins[kThreads / 32][256];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (kThreads / 32) * 256; i += kThreads) (&bins[0][0])[i] = 0;
  __syncthreads();
  const int64_t n8 = n / 8;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n8; i += (int64_t)gridDim.x * kThreads) {
    const uint4 v = __ldg(s4 + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      atomicAdd(&bins[warp][(w[j] >> 7) & 0xffu], 1u);
      atomicAdd(&bins[warp][(w[j] >> 23) & 0xffu], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += kThreads) {
    uint32_t s = 0;
    for (int w = 0; w < kThreads / 32; ++w) s += bins[w][b];
    if (s) atomicAdd(&hist[b], s);
  }
}

// ------------------------------------------------------------------ count
__global__ void __launch_bounds__(kThreads) xc_count_kernel(const uint16_t* __restrict__ src, const Lut lut,
                                                            uint32_t* __restrict__ bsec,
                                                            uint32_t* __restrict__ bexc) {
  __shared__ uint8_t s_lut[256];
  __shared__ int warp_sums[kThreads / 32 + 1];
  s_lut[threadIdx.x] = lut.v[threadIdx.x];
  __syncthreads();
  const int64_t blk = blockIdx.x;
  uint32_t w[8];
  load16(src + blk * SPMOE_XC_BLOCK + threadIdx.x * kPerThread, w);
  int c = 0, ce = 0;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    const uint8_t l = s_lut[(val_of(w, j) >> 7) & 0xffu];
    c += (l & 3u) == 3u;
    ce += l == kExcLut;
  }
  int tot_c, tot_e;
  block_exclusive_scan(c, warp_sums, &tot_c);
  __syncthreads();
  block_exclusive_scan(ce, warp_sums, &tot_e);
  if (threadIdx.x == 0) {
    bsec[blk] = (uint32_t)((tot_c + 7) / 8);
    bexc[blk] = (uint32_t)tot_e;
  }
}

// In-place exclusive prefix over a[0..n) with a[n] = total (one CTA).
__global__ void __launch_bounds__(1024) xc_scan_kernel(uint32_t* __restrict__ a, int64_t n) {
  __shared__ uint64_t part[1024];
  const int64_t per = (n + 1023) / 1024;
  const int64_t lo = threadIdx.x * per, hi = min(n, lo + per);
  uint64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += a[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int i = 0; i < 1024; ++i) {
      const uint64_t v = part[i];
      part[i] = acc;
      acc += v;
    }
    a[n] = (uint32_t)acc;
  }
  __syncthreads();
  uint64_t acc = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) {
    const uint32_t v = a[i];
    a[i] = (uint32_t)acc;
    acc += v;
  }
}

// ------------------------------------------------------------------ write
struct WriteParams {
  const uint16_t* src;
  uint8_t* sm;
  uint32_t* pc;
  uint32_t* sec;
  uint32_t* exc;
  const uint32_t* bsec;
  const uint32_t* bexc;
  Lut lut;
};

__global__ void __launch_bounds__(kThreads) xc_write_kernel(const WriteParams p) {
  __shared__ uint8_t s_lut[256];
  __shared__ uint32_t s_sec[kMaxSecWords];
  __shared__ int warp_sums[kThreads / 32 + 1];
  s_lut[threadIdx.x] = p.lut.v[threadIdx.x];
  for (int i = threadIdx.x; i < kMaxSecWords; i += kThreads) s_sec[i] = 0;
  __syncthreads();
  const int64_t blk = blockIdx.x;
  const int64_t base = blk * SPMOE_XC_BLOCK + threadIdx.x * kPerThread;
  uint32_t w[8];
  load16(p.src + base, w);
  uint32_t code = 0, smw[4] = {0, 0, 0, 0};
  int c = 0, ce = 0;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    const uint32_t v = val_of(w, j);
    const uint8_t l = s_lut[(v >> 7) & 0xffu];
    code |= (uint32_t)(l & 3u) << (2 * j);
    smw[j >> 2] |= (((v >> 8) & 0x80u) | (v & 0x7fu)) << (8 * (j & 3));
    c += (l & 3u) == 3u;
    ce += l == kExcLut;
  }
  reinterpret_cast<uint4*>(p.sm)[base / 16] = make_uint4(smw[0], smw[1], smw[2], smw[3]);
  p.pc[base / 16] = code;
  int tot;
  int q = block_exclusive_scan(c, warp_sums, &tot);
  __syncthreads();
  int r = block_exclusive_scan(ce, warp_sums, &tot);
  const uint32_t e0 = p.bexc[blk];
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    const uint32_t v = val_of(w, j);
    const uint8_t l = s_lut[(v >> 7) & 0xffu];
    if ((l & 3u) == 3u) {
      atomicOr(&s_sec[q >> 3], (uint32_t)(l >> 2) << ((q & 7) * 4));
      ++q;
      if (l == kExcLut) p.exc[e0 + r++] = ((uint32_t)(threadIdx.x * kPerThread + j) << 8) | ((v >> 7) & 0xffu);
    }
  }
  __syncthreads();
  const uint32_t s0 = p.bsec[blk], nw = p.bsec[blk + 1] - s0;
  for (uint32_t i = threadIdx.x; i < nw; i += kThreads) p.sec[s0 + i] = s_sec[i];
}

// ----------------------------------------------------------------- decode
// Persistent CTAs, each owning a contiguous range of coding blocks.  Thread 0
// streams the next blocks' sm / pc / escape words into a shared-memory ring
// with bulk async copies (cp.async.bulk + mbarrier complete_tx) while the
// CTA decodes the current block, so HBM latency is hidden behind decode
// work.  Thread t decodes values 8t..8t+7 and 2048+8t..2048+8t+7 of the
// block: every 16-byte output store of a warp is contiguous.
constexpr int kDecStages = 3;
constexpr int kSecBytes = SPMOE_XC_BLOCK / 2 + 16;  // all escaped + alignment slack
constexpr int kStageBytes = SPMOE_XC_BLOCK + SPMOE_XC_BLOCK / 4 + kSecBytes;
constexpr int kMaxBlocksPerCta = 1023;

struct DecSeg {
  const uint8_t* sm;
  const uint32_t* pc;
  const uint32_t* sec;
  const uint32_t* bsec;
  const uint32_t* bexc;
  const uint32_t* exc;
  uint16_t* dst;
  uint32_t blk0, nblk;
  uint32_t prim;  // prim[0] | prim[1] << 8 | prim[2] << 16
  uint8_t sec_tab[16];
};

struct DecParams {
  DecSeg seg[SPMOE_XC_MAX_SEG];
  int nseg;
  uint32_t total;
};

__device__ __forceinline__ uint32_t smem_u32(const void* q) { return (uint32_t)__cvta_generic_to_shared(q); }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ int seg_of(const DecParams& p, uint32_t gb) {
  int si = 0;
#pragma unroll
  for (int i = 1; i < SPMOE_XC_MAX_SEG; ++i)
    if (i < p.nseg && gb >= p.seg[i].blk0) si = i;
  return si;
}

// Exponent of secondary code nib (0..14) from the segment's table held in
// four registers (byte i of t[i/4]); two byte-permutes and a select, no
// shared-memory lookup.
__device__ __forceinline__ uint32_t sec_exp(const uint32_t (&t)[4], uint32_t nib) {
  const uint32_t lo = __byte_perm(t[0], t[1], nib & 7u);
  const uint32_t hi = __byte_perm(t[2], t[3], nib & 7u);
  return (nib < 8u ? lo : hi) & 0xffu;
}

// Exception exponent of block position pos (code 15), from the block's
// ascending (position << 8 | exponent) list.
__device__ __noinline__ uint32_t exc_exp(const uint32_t* bexc, const uint32_t* exc, uint32_t lb, uint32_t pos) {
  const uint32_t x0 = __ldg(bexc + lb), x1 = __ldg(bexc + lb + 1);
  for (uint32_t x = x0; x < x1; ++x) {
    const uint32_t ent = __ldg(exc + x);
    if ((ent >> 8) == pos) return ent & 0xffu;
  }
  return 0u;
}

// Decode 8 values of one segment.  c16 = their 2-bit codes, sm_lo/sm_hi =
// their sign|mantissa bytes, q = nibble index of their first escape in the
// block's escape words s_sec.  Pairs are built with byte permutes and a
// 16-entry pair table (exponent fields of two codes, escapes 0); escaped
// values then OR in their exponent: the k-th escape of the group reads
// nibble k of the 8-nibble window starting at q, branch-free.
__device__ __forceinline__ uint4 decode8(uint32_t c16, uint32_t sm_lo, uint32_t sm_hi, const uint32_t* s_sec,
                                         int q, const uint32_t* lut2, const uint32_t (&tab)[4], const DecSeg& S,
                                         uint32_t lb, uint32_t pos0) {
  uint32_t o[4];
#pragma unroll
  for (int pr = 0; pr < 4; ++pr) {
    const uint32_t smw = pr < 2 ? sm_lo : sm_hi;
    const uint32_t k = 2 * (pr & 1);
    // bytes k, k+1 of smw -> the low bytes of the two 16-bit halves
    const uint32_t w = __byte_perm(smw, 0u, k | (4u << 4) | ((k + 1) << 8) | (4u << 12));
    o[pr] = ((w & 0x00800080u) << 8) | (w & 0x007f007fu) | lut2[(c16 >> (4 * pr)) & 15u];
  }
  const uint32_t esc = c16 & (c16 >> 1) & 0x5555u;
  if (esc) {
    const uint32_t w0 = s_sec[q >> 3], w1 = s_sec[(q >> 3) + 1];
    const uint32_t win = __funnelshift_r(w0, w1, (q & 7) * 4);  // nibbles q .. q+7
    bool exc = false;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t r = __popc(esc & ((1u << (2 * j)) - 1u));
      const uint32_t nib = (win >> (4 * r)) & 15u;
      const bool is = (esc >> (2 * j)) & 1u;
      exc |= is && nib == 15u;
      const uint32_t e = is ? sec_exp(tab, nib) : 0u;
      o[j >> 1] |= (e << 7) << (16 * (j & 1));
    }
    if (exc) {
#pragma unroll 1
      for (int j = 0; j < 8; ++j) {
        const uint32_t r = __popc(esc & ((1u << (2 * j)) - 1u));
        if (((esc >> (2 * j)) & 1u) && ((win >> (4 * r)) & 15u) == 15u) {
          const uint32_t e = exc_exp(S.bexc, S.exc, lb, pos0 + j);
          const uint32_t add = (e << 7) << (16 * (j & 1));
          const int wsel = j >> 1;
          o[0] |= wsel == 0 ? add : 0u;
          o[1] |= wsel == 1 ? add : 0u;
          o[2] |= wsel == 2 ? add : 0u;
          o[3] |= wsel == 3 ? add : 0u;
        }
      }
    }
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// Decode CTAs are 128 threads; thread t owns values 1024g + 8t .. +7 for the
// four groups g of its block (every 16-byte store of a warp is contiguous).
constexpr int kDecThreads = 128;

__global__ void __launch_bounds__(kDecThreads) xc_decode_kernel(const DecParams p) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full[kDecStages];
  __shared__ uint32_t s_bsec[kMaxBlocksPerCta + 1];
  __shared__ uint32_t s_lut2[SPMOE_XC_MAX_SEG][16];
  __shared__ uint2 warp_sums[2][kDecThreads / 32];
  const uint32_t b0 = (uint32_t)(((uint64_t)blockIdx.x * p.total) / gridDim.x);
  const uint32_t b1 = (uint32_t)(((uint64_t)(blockIdx.x + 1) * p.total) / gridDim.x);
  const int n = (int)(b1 - b0);
  // escape-word offsets of this CTA's blocks (and the one after the last)
  for (int i = threadIdx.x; i <= n; i += kDecThreads) {
    const uint32_t gb = b0 + i;
    const DecSeg& S = p.seg[seg_of(p, i < n ? gb : gb - 1)];
    s_bsec[i] = __ldg(S.bsec + (gb - S.blk0));
  }
  if (threadIdx.x < SPMOE_XC_MAX_SEG * 16) {
    const int g = threadIdx.x / 16, c = threadIdx.x % 16;
    const DecSeg& S = p.seg[g];
    const uint32_t c0 = c & 3u, c1 = c >> 2;
    const uint32_t e0 = c0 < 3 ? ((S.prim >> (8 * c0)) & 0xffu) << 7 : 0u;
    const uint32_t e1 = c1 < 3 ? ((S.prim >> (8 * c1)) & 0xffu) << 7 : 0u;
    s_lut2[g][c] = e0 | (e1 << 16);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDecStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // thread 0: start the copies of local block i into stage i % kDecStages
  auto issue = [&](int i) {
    const uint32_t gb = b0 + i;
    const DecSeg& S = p.seg[seg_of(p, gb)];
    const uint32_t lb = gb - S.blk0;
    uint8_t* st = ring + (i % kDecStages) * kStageBytes;
    // block i's escape words [s0, s1) end where block i+1's begin, except at
    // a segment boundary, where the segment's own table entry nblk is used
    const uint32_t s0 = s_bsec[i];
    const uint32_t s1 = (lb + 1 == S.nblk) ? __ldg(S.bsec + S.nblk) : s_bsec[i + 1];
    const uint32_t a = (s0 * 4) & ~15u;
    const uint32_t len = (((s1 * 4) + 15) & ~15u) - a;
    uint64_t* bar = &full[i % kDecStages];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"((uint32_t)(SPMOE_XC_BLOCK + SPMOE_XC_BLOCK / 4) + len)
                 : "memory");
    bulk_g2s(st, S.sm + (uint64_t)lb * SPMOE_XC_BLOCK, SPMOE_XC_BLOCK, bar);
    bulk_g2s(st + SPMOE_XC_BLOCK, S.pc + (uint64_t)lb * (SPMOE_XC_BLOCK / 16), SPMOE_XC_BLOCK / 4, bar);
    if (len) bulk_g2s(st + SPMOE_XC_BLOCK + SPMOE_XC_BLOCK / 4, (const uint8_t*)S.sec + a, len, bar);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < kDecStages - 1 && i < n; ++i) issue(i);

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int si = -1;
  uint32_t tab[4] = {0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    const uint32_t gb = b0 + i;
    const int sj = seg_of(p, gb);
    const DecSeg& S = p.seg[sj];
    if (sj != si) {
      si = sj;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tab[k] = (uint32_t)S.sec_tab[4 * k] | ((uint32_t)S.sec_tab[4 * k + 1] << 8) |
                 ((uint32_t)S.sec_tab[4 * k + 2] << 16) | ((uint32_t)S.sec_tab[4 * k + 3] << 24);
    }
    const uint32_t lb = gb - S.blk0;
    const uint8_t* st = ring + (i % kDecStages) * kStageBytes;
    mbar_wait_parity(&full[i % kDecStages], (uint32_t)(i / kDecStages) & 1u);
    const uint32_t* s_pc = (const uint32_t*)(st + SPMOE_XC_BLOCK);
    const uint32_t sh = 16 * (t & 1);
    uint32_t c[4];
    int v01 = 0, v23 = 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      c[g] = (s_pc[64 * g + (t >> 1)] >> sh) & 0xffffu;
      const int e = __popc(c[g] & (c[g] >> 1) & 0x5555u);
      if (g < 2) v01 |= e << (16 * g); else v23 |= e << (16 * (g - 2));
    }
    // escapes of the four groups, two packed per int: two warp scans
    int i01 = v01, i23 = v23;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u01 = __shfl_up_sync(0xffffffffu, i01, o);
      const int u23 = __shfl_up_sync(0xffffffffu, i23, o);
      if (lane >= o) {
        i01 += u01;
        i23 += u23;
      }
    }
    uint2* ws = warp_sums[i & 1];
    if (lane == 31) ws[warp] = make_uint2((uint32_t)i01, (uint32_t)i23);
    // one barrier per block: publishes the warp sums and proves every thread
    // is done with block i-1, so its stage can be refilled
    __syncthreads();
    if (threadIdx.x == 0 && i + kDecStages - 1 < n) issue(i + kDecStages - 1);
    uint32_t b01 = 0, b23 = 0, t01 = 0, t23 = 0;
#pragma unroll
    for (int w = 0; w < kDecThreads / 32; ++w) {
      const uint2 s_ = ws[w];
      b01 += w < warp ? s_.x : 0u;
      b23 += w < warp ? s_.y : 0u;
      t01 += s_.x;
      t23 += s_.y;
    }
    const uint32_t p01 = b01 + (uint32_t)(i01 - v01), p23 = b23 + (uint32_t)(i23 - v23);
    // escapes of group g precede those of group g+1 (value order)
    const uint32_t tg0 = t01 & 0xffffu, tg1 = t01 >> 16, tg2 = t23 & 0xffffu;
    int q[4];
    q[0] = (int)(p01 & 0xffffu);
    q[1] = (int)(tg0 + (p01 >> 16));
    q[2] = (int)(tg0 + tg1 + (p23 & 0xffffu));
    q[3] = (int)(tg0 + tg1 + tg2 + (p23 >> 16));
    const uint32_t* s_sec = (const uint32_t*)(st + SPMOE_XC_BLOCK + SPMOE_XC_BLOCK / 4) + (s_bsec[i] & 3u);
    uint16_t* d = S.dst + (uint64_t)lb * SPMOE_XC_BLOCK;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint2 m = *(const uint2*)(st + 1024 * g + 8 * t);
      const uint4 o = decode8(c[g], m.x, m.y, s_sec, q[g], s_lut2[sj], tab, S, lb, 1024 * g + 8 * t);
      reinterpret_cast<uint4*>(d + 1024 * g)[t] = o;
    }
  }
}

inline uint64_t align256(uint64_t x) { return (x + 255) & ~uint64_t(255); }
inline int64_t nblocks(int64_t n) { return n / SPMOE_XC_BLOCK; }

// work layout per segment: hist[256] | bsec[nb+1] | bexc[nb+1]  (u32)
inline size_t seg_work_words(int64_t n) { return 256 + 2 * (size_t)(nblocks(n) + 1); }

// Code tables from a histogram: exponents by (count desc, exponent asc).
void choose_tables(const uint32_t* hist, spmoe_xc_segment* seg, Lut* lut) {
  int order[256];
  for (int i = 0; i < 256; ++i) order[i] = i;
  std::stable_sort(order, order + 256, [&](int a, int b) { return hist[a] > hist[b]; });
  std::memset(seg->prim, 0, sizeof(seg->prim));
  std::memset(seg->sec, 0, sizeof(seg->sec));
  for (int i = 0; i < 256; ++i) lut->v[i] = kExcLut;
  for (int r = 0; r < 3; ++r) {
    seg->prim[r] = (uint8_t)order[r];
    lut->v[order[r]] = (uint8_t)r;
  }
  for (int r = 0; r < 15; ++r) {
    seg->sec[r] = (uint8_t)order[3 + r];
    lut->v[order[3 + r]] = (uint8_t)((r << 2) | 3);
  }
}

void lut_of(const spmoe_xc_segment& seg, Lut* lut) {
  for (int i = 0; i < 256; ++i) lut->v[i] = kExcLut;
  for (int r = 0; r < 3; ++r) lut->v[seg.prim[r]] = (uint8_t)r;
  for (int r = 0; r < 15; ++r) lut->v[seg.sec[r]] = (uint8_t)((r << 2) | 3);
}

bool valid_segments(int nseg, const int64_t* seg_n) {
  if (nseg < 1 || nseg > SPMOE_XC_MAX_SEG || !seg_n) return false;
  for (int i = 0; i < nseg; ++i)
    if (seg_n[i] <= 0 || seg_n[i] % SPMOE_XC_BLOCK) return false;
  return true;
}

}  // namespace

extern "C" {

size_t spmoe_xc_work_bytes(int nseg, const int64_t* seg_n) {
  if (!valid_segments(nseg, seg_n)) return 0;
  size_t w = 0;
  for (int i = 0; i < nseg; ++i) w += seg_work_words(seg_n[i]);
  return w * sizeof(uint32_t);
}

int spmoe_xc_plan(const uint16_t* src, int nseg, const int64_t* seg_n, void* work, spmoe_xc_header* hdr,
                  void* stream) {
  if (!valid_segments(nseg, seg_n) || !src || !work || !hdr) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* wk = (uint32_t*)work;
  cudaError_t e = cudaMemsetAsync(wk, 0, spmoe_xc_work_bytes(nseg, seg_n), st);
  if (e != cudaSuccess) return (int)e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // 1. histograms
  size_t off = 0;
  const uint16_t* s = src;
  for (int i = 0; i < nseg; ++i) {
    const int64_t n = seg_n[i];
    const int grid = (int)std::min<int64_t>((int64_t)sms * 8, (n / 8 + kThreads - 1) / kThreads);
    xc_hist_kernel<<<grid, kThreads, 0, st>>>(s, n, wk + off);
    off += seg_work_words(n);
    s += n;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  std::vector<uint32_t> host(spmoe_xc_work_bytes(nseg, seg_n) / 4);
  if ((e = cudaMemcpyAsync(host.data(), wk, host.size() * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return (int)e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
  std::memset(hdr, 0, sizeof(*hdr));
  hdr->magic = SPMOE_XC_MAGIC;
  hdr->nseg = (uint32_t)nseg;
  // 2. tables, per-block counts, prefixes
  off = 0;
  s = src;
  for (int i = 0; i < nseg; ++i) {
    const int64_t n = seg_n[i], nb = nblocks(n);
    Lut lut;
    choose_tables(host.data() + off, &hdr->seg[i], &lut);
    hdr->seg[i].n = (uint64_t)n;
    uint32_t* bsec = wk + off + 256;
    uint32_t* bexc = bsec + nb + 1;
    xc_count_kernel<<<(unsigned)nb, kThreads, 0, st>>>(s, lut, bsec, bexc);
    xc_scan_kernel<<<1, 1024, 0, st>>>(bsec, nb);
    xc_scan_kernel<<<1, 1024, 0, st>>>(bexc, nb);
    off += seg_work_words(n);
    s += n;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  std::vector<uint32_t> tot(2 * nseg);
  off = 0;
  for (int i = 0; i < nseg; ++i) {
    const int64_t nb = nblocks(seg_n[i]);
    cudaMemcpyAsync(&tot[2 * i], wk + off + 256 + nb, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&tot[2 * i + 1], wk + off + 256 + 2 * (nb + 1) - 1, 4, cudaMemcpyDeviceToHost, st);
    off += seg_work_words(seg_n[i]);
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
  // 3. layout
  uint64_t pos = 512, raw = 0;
  for (int i = 0; i < nseg; ++i) {
    spmoe_xc_segment& g = hdr->seg[i];
    const int64_t n = seg_n[i], nb = nblocks(n);
    g.sec_words = tot[2 * i];
    g.n_exc = tot[2 * i + 1];
    g.off_sm = pos; pos = align256(pos + (uint64_t)n);
    g.off_pc = pos; pos = align256(pos + (uint64_t)n / 4);
    g.off_sec = pos; pos = align256(pos + (uint64_t)g.sec_words * 4);
    g.off_bsec = pos; pos = align256(pos + (uint64_t)(nb + 1) * 4);
    g.off_bexc = pos; pos = align256(pos + (uint64_t)(nb + 1) * 4);
    g.off_exc = pos; pos = align256(pos + (uint64_t)g.n_exc * 4);
    raw += 2 * (uint64_t)n;
  }
  hdr->blob_bytes = pos;
  hdr->raw_bytes = raw;
  return 0;
}

int spmoe_xc_encode(const uint16_t* src, const spmoe_xc_header* hdr, const void* work, uint8_t* blob,
                    void* stream) {
  if (!src || !hdr || !work || !blob || hdr->magic != SPMOE_XC_MAGIC) return (int)cudaErrorInvalidValue;
  int64_t seg_n[SPMOE_XC_MAX_SEG];
  for (uint32_t i = 0; i < hdr->nseg && i < SPMOE_XC_MAX_SEG; ++i) seg_n[i] = (int64_t)hdr->seg[i].n;
  if (!valid_segments((int)hdr->nseg, seg_n)) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(blob, 0, hdr->blob_bytes, st);
  if (e != cudaSuccess) return (int)e;
  const uint32_t* wk = (const uint32_t*)work;
  size_t off = 0;
  const uint16_t* s = src;
  for (uint32_t i = 0; i < hdr->nseg; ++i) {
    const spmoe_xc_segment& g = hdr->seg[i];
    const int64_t n = (int64_t)g.n, nb = nblocks(n);
    WriteParams p;
    p.src = s;
    p.sm = blob + g.off_sm;
    p.pc = (uint32_t*)(blob + g.off_pc);
    p.sec = (uint32_t*)(blob + g.off_sec);
    p.exc = (uint32_t*)(blob + g.off_exc);
    p.bsec = wk + off + 256;
    p.bexc = wk + off + 256 + nb + 1;
    lut_of(g, &p.lut);
    xc_write_kernel<<<(unsigned)nb, kThreads, 0, st>>>(p);
    cudaMemcpyAsync(blob + g.off_bsec, p.bsec, (nb + 1) * 4, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(blob + g.off_bexc, p.bexc, (nb + 1) * 4, cudaMemcpyDeviceToDevice, st);
    off += seg_work_words(n);
    s += n;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  if ((e = cudaMemcpyAsync(blob, hdr, sizeof(*hdr), cudaMemcpyHostToDevice, st)) != cudaSuccess) return (int)e;
  return (int)cudaStreamSynchronize(st);
}

int spmoe_xc_decode_segments(const uint8_t* blob, const spmoe_xc_header* hdr, int first, int count,
                              uint16_t* dst, void* stream) {
  if (!blob || !hdr || !dst || hdr->magic != SPMOE_XC_MAGIC || hdr->nseg < 1 || hdr->nseg > SPMOE_XC_MAX_SEG ||
      first < 0 || count < 1 || first + count > (int)hdr->nseg)
    return (int)cudaErrorInvalidValue;
  DecParams p;
  std::memset(&p, 0, sizeof(p));
  p.nseg = count;
  uint32_t blk = 0;
  uint16_t* d = dst;
  for (int i = 0; i < first; ++i) d += hdr->seg[i].n;
  for (int j = 0; j < count; ++j) {
    const spmoe_xc_segment& g = hdr->seg[first + j];
    if (g.n == 0 || g.n % SPMOE_XC_BLOCK) return (int)cudaErrorInvalidValue;
    DecSeg& S = p.seg[j];
    S.sm = blob + g.off_sm;
    S.pc = (const uint32_t*)(blob + g.off_pc);
    S.sec = (const uint32_t*)(blob + g.off_sec);
    S.bsec = (const uint32_t*)(blob + g.off_bsec);
    S.bexc = (const uint32_t*)(blob + g.off_bexc);
    S.exc = (const uint32_t*)(blob + g.off_exc);
    S.dst = d;
    S.blk0 = blk;
    S.nblk = (uint32_t)(g.n / SPMOE_XC_BLOCK);
    S.prim = (uint32_t)g.prim[0] | ((uint32_t)g.prim[1] << 8) | ((uint32_t)g.prim[2] << 16);
    std::memcpy(S.sec_tab, g.sec, 16);
    blk += S.nblk;
    d += g.n;
  }
  p.total = blk;
  static int sms = 0;
  static bool attr = false;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int smem = kDecStages * kStageBytes;
  if (!attr) {
    cudaFuncSetAttribute(xc_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  // 8 CTAs of 128 threads per SM (ring + tables ~26 KB each), at most
  // kMaxBlocksPerCta blocks each
  uint32_t grid = (uint32_t)std::max(1, 8 * sms);
  grid = std::max(grid, (blk + kMaxBlocksPerCta - 1) / kMaxBlocksPerCta);
  grid = std::min(grid, blk);
  xc_decode_kernel<<<grid, kDecThreads, smem, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

int spmoe_xc_decode(const uint8_t* blob, const spmoe_xc_header* hdr, uint16_t* dst, void* stream) {
  if (!hdr) return (int)cudaErrorInvalidValue;
  return spmoe_xc_decode_segments(blob, hdr, 0, (int)hdr->nseg, dst, stream);
}

}  // extern "C"
