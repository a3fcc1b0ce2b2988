// spmoe_codec.cu — XC, the lossless exponent coding of expert blobs that
// cross the host link (format SXC5: include/spmoe.h, "XC").
//
// Why: with an offload budget the verify stage is bound by the pinned
// host -> HBM copies of routed experts (IoChannel.transfer,
// prefetch.py:45-74; PAPER.md:242 measures expert loading at 69.4 % of
// decode latency).  Copying fewer bytes per expert is the only lever left
// once the copy engine runs at the link's peak.  A bf16 weight's 8-bit
// exponent carries ~2.5 bits of entropy, so XC sends 1 byte of
// sign|mantissa plus the exponent as a 4-bit offset from the segment's base
// exponent (15 = escape, exponent in a per-block exception list) in a
// per-segment canonical Huffman code (<= 12 bits), and the copy path's
// decode kernel rebuilds the exact bf16 bits in the HBM slot.
//
// Geometry: 4096-value coding blocks, each split into 32 lane substreams of
// 128 values, so ONE WARP decodes a block: lane l walks its own substream
// with a 4096-entry shared-memory table (12-bit peek -> up to five 4-bit
// symbols), parks the symbols in shared memory, and the warp then assembles
// bf16 values with byte permutes and 16-byte coalesced stores and patches
// the block's escaped exponents.
//
// Kernels:
//   xc_hist_kernel    exponent histogram per segment (per-warp smem bins)
//   xc_count_kernel   per block and lane: code bits; per block: bit or word
//                     mode, words and escapes
//   xc_scan_kernel    exclusive prefix of the per-block counts (1 CTA)
//   xc_write_kernel   sign|mantissa bytes, lane substreams (bit-contiguous),
//                     exceptions
//   xc_decode_kernel  the inverse; HBM-bound target (reads ~1.35 B, writes
//                     2 B per value)
// Code construction (host) restates oracle/xc_oracle.c exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/spmoe.h"
#include "spmoe_common.cuh"

namespace {

constexpr int kThreads = 256;  // 8 warps: 8 blocks per CTA pass
constexpr int kWarps = kThreads / 32;
constexpr int kLanes = SPMOE_XC_LANES;
constexpr int kPerLane = SPMOE_XC_BLOCK / kLanes;  // 128
constexpr int kLmax = SPMOE_XC_LMAX;
constexpr int kLutSize = 1 << kLmax;
constexpr int kNsym = SPMOE_XC_NSYM;
constexpr int kEsc = kNsym - 1;
static_assert(kLanes == 32, "one warp per coding block");

// Per EXPONENT (the kernels index by exponent): the code of its symbol.
struct Codes {
  uint16_t rev[256];  // bit-reversed canonical code of the exponent's symbol
  uint8_t len[256];   // its length (0 = absent)
  uint32_t base;      // exponents [base, base + 14] are in the window
};

__host__ __device__ __forceinline__ bool escaped(uint32_t e, uint32_t base) { return e - base >= (uint32_t)kEsc; }

// --------------------------------------------------------------- histogram
__global__ void __launch_bounds__(kThreads) xc_hist_kernel(const uint16_t* __restrict__ src, int64_t n,
                                                           uint32_t* __restrict__ hist) {
  __shared__ uint32_t bins[kWarps][256];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * 256; i += kThreads) (&bins[0][0])[i] = 0;
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
    for (int w = 0; w < kWarps; ++w) s += bins[w][b];
    if (s) atomicAdd(&hist[b], s);
  }
}

// Lane l's 128 values of block blk, 8 at a time (uint4 loads).
__device__ __forceinline__ void lane_vals(const uint16_t* src, int64_t blk, int lane, int q, uint32_t (&w)[4]) {
  const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + blk * SPMOE_XC_BLOCK + lane * kPerLane) + q);
  w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
}

// ------------------------------------------------------------------ count
// One warp per block: lane word counts and the block's total.
// Per lane: its code bits (bit mode: minus the block's shortest lane) or
// words (word mode, when the lanes spread over more than 255 bits).
__device__ __forceinline__ uint32_t lane_bits_of(uint32_t v, uint32_t lbase) {
  return (lbase >> 15) ? 32u * v : (lbase & 0x7fffu) + v;
}

// One warp per block: lane lengths, the block's mode, words and escapes.
__global__ void __launch_bounds__(kThreads) xc_count_kernel(const uint16_t* __restrict__ src, int64_t nb,
                                                            const Codes c, uint32_t* __restrict__ bwords,
                                                            uint8_t* __restrict__ lanes, uint16_t* __restrict__ lbase,
                                                            uint32_t* __restrict__ bexc) {
  __shared__ uint8_t s_len[256];
  s_len[threadIdx.x] = c.len[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t blk = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (blk >= nb) return;
  uint32_t bits = 0, nx = 0;
  for (int q = 0; q < kPerLane / 8; ++q) {
    uint32_t w[4];
    lane_vals(src, blk, lane, q, w);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t e0 = (w[j] >> 7) & 0xffu, e1 = (w[j] >> 23) & 0xffu;
      bits += s_len[e0] + s_len[e1];
      nx += (uint32_t)escaped(e0, c.base) + (uint32_t)escaped(e1, c.base);
    }
  }
  const uint32_t words = (bits + 31) / 32;
  uint32_t lo = bits, hi = bits, tbits = bits, twords = words;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    tbits += __shfl_xor_sync(0xffffffffu, tbits, o);
    twords += __shfl_xor_sync(0xffffffffu, twords, o);
    nx += __shfl_xor_sync(0xffffffffu, nx, o);
  }
  const bool word_mode = hi - lo > 255;
  lanes[blk * kLanes + lane] = (uint8_t)(word_mode ? words : bits - lo);
  if (lane == 0) {
    lbase[blk] = (uint16_t)(word_mode ? 0x8000u : lo);
    bwords[blk] = word_mode ? twords : (tbits + 31) / 32;
    bexc[blk] = nx;
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
  int64_t nb;
  uint8_t* sm;
  uint32_t* ex;
  const uint32_t* bofs;
  const uint8_t* lanes;
  const uint16_t* lbase;
  const uint32_t* xofs;  // first exception of each block
  uint32_t* xrec;
  Codes c;
};

// One warp per block: lane l packs its 128 codes LSB first into its words.
__global__ void __launch_bounds__(kThreads) xc_write_kernel(const WriteParams p) {
  __shared__ uint8_t s_len[256];
  __shared__ uint16_t s_rev[256];
  s_len[threadIdx.x] = p.c.len[threadIdx.x];
  s_rev[threadIdx.x] = p.c.rev[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t blk = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (blk >= p.nb) return;
  // this lane's first bit: the block's first word + the bits of the lanes
  // before it (word mode: their whole words)
  const uint32_t lbits = lane_bits_of(p.lanes[blk * kLanes + lane], p.lbase[blk]);
  uint32_t pre = lbits;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += u;
  }
  const uint32_t start = pre - lbits;
  // neighbouring lanes share boundary words: OR into the zeroed stream
  uint32_t* out = p.ex + p.bofs[blk] + (start >> 5);
  // this lane's exceptions follow those of the lanes before it
  uint32_t nx = 0;
  for (int q = 0; q < kPerLane / 8; ++q) {
    uint32_t w[4];
    lane_vals(p.src, blk, lane, q, w);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      nx += (uint32_t)escaped((w[j] >> 7) & 0xffu, p.c.base) + (uint32_t)escaped((w[j] >> 23) & 0xffu, p.c.base);
  }
  uint32_t xpre = nx;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, xpre, o);
    if (lane >= o) xpre += u;
  }
  uint32_t* xout = p.xrec + p.xofs[blk] + (xpre - nx);
  uint64_t buf = 0;
  int nbits = (int)(start & 31);
  for (int q = 0; q < kPerLane / 8; ++q) {
    uint32_t w[4];
    lane_vals(p.src, blk, lane, q, w);
    uint32_t smw[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t v = (w[j >> 1] >> (16 * (j & 1))) & 0xffffu;
      const uint32_t e = (v >> 7) & 0xffu;
      if (escaped(e, p.c.base)) *xout++ = ((uint32_t)(lane * kPerLane + 8 * q + j) << 8) | e;
      smw[j >> 2] |= (((v >> 8) & 0x80u) | (v & 0x7fu)) << (8 * (j & 3));
      buf |= (uint64_t)s_rev[e] << nbits;
      nbits += s_len[e];
      if (nbits >= 32) {
        atomicOr(out++, (uint32_t)buf);
        buf >>= 32;
        nbits -= 32;
      }
    }
    *reinterpret_cast<uint2*>(p.sm + blk * SPMOE_XC_BLOCK + lane * kPerLane + 8 * q) = make_uint2(smw[0], smw[1]);
  }
  if (nbits > 0) atomicOr(out, (uint32_t)buf);
}

// ----------------------------------------------------------------- decode
struct DecSeg {
  const uint32_t* lut2;  // the blob's multi-symbol table
  const uint8_t* sm;
  const uint32_t* ex;
  const uint32_t* bofs;
  const uint8_t* lanes;
  const uint16_t* lbase;
  const uint32_t* xofs;
  const uint32_t* xrec;
  uint16_t* dst;
  uint32_t nblk;
  uint32_t base4;  // base exponent in every byte
};

struct DecParams {
  DecSeg seg[SPMOE_XC_MAX_SEG];
  spmoe::DevSpan* span;  // optional device-clock timing of this launch
  int stream_stores;     // evict-first (.cs) output stores (default; SPMOE_XC_STCS=0 disables, A/B switch)
};

// Symbols of one block, lane-major: lane l's 128 symbols are 16 words of 8
// nibbles (value order, LSB first) in row l, pitch 17 words (the lane-major
// writes are conflict-free; the value-order reads of the assembly conflict
// 2-way on one bank pair).
constexpr int kRowWords = kPerLane / 8;
constexpr int kRowPitch = kRowWords + 1;
// A block's code words are staged in shared memory before the lanes walk
// them (Gaussian weights: ~346 words; 400 ~ 3.1 bits per value); longer runs
// are read from global memory directly.
constexpr int kStageWords = 400;
constexpr int kDecWarps = 16;
constexpr int kDecThreads = 32 * kDecWarps;
// staged run: up to 3 words of 16-byte alignment slack + the run + 3 peek
// words, rounded up to 16 bytes (one bulk copy per block)
constexpr int kStageAlloc = 412;
static_assert(kStageAlloc * 4 >= ((12 + (kStageWords + 3) * 4 + 15) & ~15), "stage too small");
constexpr int kWarpSmemWords = kStageAlloc + kLanes * kRowPitch;
static_assert(kWarpSmemWords % 4 == 0, "warp buffers stay 16-byte aligned");
// dynamic shared memory (the 16 KB table is a static array)
constexpr int kDecSmemBytes = kDecWarps * kWarpSmemWords * 4 + kDecWarps * 8;

__device__ __forceinline__ uint32_t sh_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// One lane's substream -> its 128 symbols (row `erow`).  kStaged: the code
// words are in shared memory (the common case; refills are shared loads
// that rotate the window registers in place), else in global memory (an
// over-long block).  Up to five symbols per lookup; they queue in a
// register and leave as whole words.
template <bool kStaged>
__device__ __forceinline__ void decode_lane(const uint32_t* __restrict__ s_lut2, const uint32_t* wp, uint32_t pos,
                                            uint32_t* __restrict__ erow) {
  // bit window = (nxt:cur) >> pos, pos < 32: at least 33 valid bits; the
  // word after nxt is fetched one refill ahead, so a refill never waits on
  // a load (the only load on the serial chain is the table lookup)
  uint32_t cur = wp[0], nxt = wp[1], ahead = wp[2];
  wp += 3;
  uint64_t q = 0;
  uint32_t nq = 0;  // queued bits (4 per symbol)
  if (kStaged) {
    // 32-bit shared addresses throughout: table, refill pointer, symbol row
    const uint32_t lut = sh_u32(s_lut2);
    uint32_t sp = sh_u32(wp), ea = sh_u32(erow);
    const uint32_t eend = ea + 4 * kRowWords;
    while (ea < eend) {
      uint32_t e;
      asm volatile(
          "{\n"
          ".reg .b32 t;\n"
          "and.b32 t, %1, 4095;\n"
          "mad.lo.u32 t, t, 4, %2;\n"
          "ld.shared.u32 %0, [t];\n"
          "}\n"
          : "=r"(e)
          : "r"(__funnelshift_r(cur, nxt, pos)), "r"(lut));
      q |= (uint64_t)(e & 0xfffffu) << nq;  // nibbles past the count are zero
      nq += (e >> 20) & 31u;
      if (nq >= 32) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ea), "r"((uint32_t)q));
        ea += 4;
        q >>= 32;
        nq -= 32;
      }
      pos += e >> 25;
      // refill: rotate the window registers in place
      asm volatile(
          "{\n"
          ".reg .pred p;\n"
          "setp.ge.u32 p, %3, 32;\n"
          "@p mov.b32 %0, %1;\n"
          "@p mov.b32 %1, %2;\n"
          "@p ld.shared.u32 %2, [%4];\n"
          "@p add.u32 %4, %4, 4;\n"
          "@p sub.u32 %3, %3, 32;\n"
          "}\n"
          : "+r"(cur), "+r"(nxt), "+r"(ahead), "+r"(pos), "+r"(sp));
    }
  } else {
    for (int wi = 0; wi < kRowWords;) {
      const uint32_t e = s_lut2[__funnelshift_r(cur, nxt, pos) & (kLutSize - 1)];
      q |= (uint64_t)(e & 0xfffffu) << nq;
      nq += (e >> 20) & 31u;
      if (nq >= 32) {
        erow[wi++] = (uint32_t)q;
        q >>= 32;
        nq -= 32;
      }
      pos += e >> 25;
      if (pos >= 32) {
        pos -= 32;
        cur = nxt;
        nxt = ahead;
        ahead = *wp++;
      }
    }
  }
}

// grid.y = segment; each warp decodes whole blocks of its segment.  The
// registers are budgeted for 2 resident CTAs per SM (3 fit in shared memory,
// but at 40 registers the decode runs 30 % slower); the first kSmPre of the 16
// sign|mantissa rounds are fetched before the serial decode (all 16: +2 %).
constexpr int kDecCtas = 2;
constexpr int kSmPre = 8;
__global__ void __launch_bounds__(kDecThreads, kDecCtas) xc_decode_kernel(const DecParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  // multi-symbol table: entry p (12 peeked bits) = up to five whole codes:
  // syms (4 bits each) | 4 count << 20 | bits << 25
  __shared__ __align__(16) uint32_t s_lut2[kLutSize];
  uint8_t* wbase = dsm;
  spmoe::span_begin(p.span);
  const DecSeg& S = p.seg[blockIdx.y];
  // the segment's multi-symbol table, precomputed in the blob (lut2)
  for (int i = threadIdx.x; i < kLutSize / 4; i += kDecThreads)
    reinterpret_cast<uint4*>(s_lut2)[i] = __ldg(reinterpret_cast<const uint4*>(S.lut2) + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* stage = reinterpret_cast<uint32_t*>(wbase) + warp * kWarpSmemWords;
  uint32_t* ew = stage + kStageAlloc;
  // the block's code words arrive by one bulk copy (async proxy) per block,
  // completing on this warp's mbarrier
  uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase + kDecWarps * kWarpSmemWords * 4) + warp;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sh_u32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  uint32_t* erow = ew + lane * kRowPitch;  // this lane's symbol row
  const uint32_t base4 = S.base4;
  // warp-major block order: the last, partial wave's blocks go to one warp
  // of many CTAs (one per SM) instead of every warp of a few CTAs
  for (uint32_t blk = warp * gridDim.x + blockIdx.x; blk < S.nblk; blk += gridDim.x * kDecWarps) {
    // this lane's substream: block start + bits of the lanes before it
    const uint32_t lbits = lane_bits_of(__ldg(S.lanes + (uint64_t)blk * kLanes + lane), __ldg(S.lbase + blk));
    uint32_t pre = lbits;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += u;
    }
    const uint32_t start = pre - lbits;
    const uint32_t w0 = __ldg(S.bofs + blk), nw = __ldg(S.bofs + blk + 1) - w0;
    const uint32_t x0 = __ldg(S.xofs + blk), x1 = __ldg(S.xofs + blk + 1);
    const uint32_t* run = S.ex + w0;
    // the first sign|mantissa rounds are fetched before the serial decode
    const uint8_t* smb = S.sm + (uint64_t)blk * SPMOE_XC_BLOCK;
    uint2 sm[kSmPre];
#pragma unroll
    for (int it = 0; it < kSmPre; ++it) sm[it] = __ldg(reinterpret_cast<const uint2*>(smb) + it * 32 + lane);
    if (nw <= (uint32_t)kStageWords) {
      const uint32_t delta = (uint32_t)((uintptr_t)run & 15);  // 0, 4, 8 or 12
      if (lane == 0) {
        // the run + 3 peek words from its 16-byte-aligned start, rounded up
        // to 16 bytes: past the stream's 8 slack bytes come the segment's
        // block offsets, so the copy never leaves the segment
        const uint32_t bytes = (delta + (nw + 3) * 4 + 15) & ~15u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after last block's reads
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sh_u32(mbar)), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                sh_u32(stage)),
            "l"(reinterpret_cast<const uint8_t*>(run) - delta), "r"(bytes), "r"(sh_u32(mbar))
            : "memory");
      }
      asm volatile(
          "{\n"
          ".reg .pred p;\n"
          "XCW_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra XCW_%=;\n"
          "}\n" ::"r"(sh_u32(mbar)),
          "r"(phase)
          : "memory");
      phase ^= 1;
      decode_lane<true>(s_lut2, stage + (delta >> 2) + (start >> 5), start & 31, erow);
    } else {
      decode_lane<false>(s_lut2, run + (start >> 5), start & 31, erow);
    }
    __syncwarp();
    // assembly: 16 rounds of 8 consecutive values per lane (one symbol
    // word), 16-byte stores
    uint16_t* dst = S.dst + (uint64_t)blk * SPMOE_XC_BLOCK;
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const uint32_t r = (uint32_t)(it * 32 + lane) >> 4, off = (uint32_t)lane & 15;
      const uint32_t nib = ew[r * kRowPitch + off];
      const uint32_t lo = nib & 0x0f0f0f0fu, hi = (nib >> 4) & 0x0f0f0f0fu;
      // exponents of values 0..3 and 4..7 (no byte carries: base <= 240)
      const uint32_t ea = __byte_perm(lo, hi, 0x5140) + base4, eb = __byte_perm(lo, hi, 0x7362) + base4;
      const uint2 m = it < kSmPre ? sm[it] : __ldg(reinterpret_cast<const uint2*>(smb) + it * 32 + lane);
      uint32_t o[4];
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        const uint32_t smw = pr < 2 ? m.x : m.y;
        const uint32_t exw = pr < 2 ? ea : eb;
        const uint32_t k = 2 * (pr & 1);
        const uint32_t sel = k | (4u << 4) | ((k + 1) << 8) | (4u << 12);
        const uint32_t ws = __byte_perm(smw, 0u, sel), we = __byte_perm(exw, 0u, sel);
        o[pr] = ((ws & 0x00800080u) << 8) | (ws & 0x007f007fu) | (we << 7);
      }
      if (p.stream_stores)
        __stcs(reinterpret_cast<uint4*>(dst) + it * 32 + lane, make_uint4(o[0], o[1], o[2], o[3]));
      else
        reinterpret_cast<uint4*>(dst)[it * 32 + lane] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    // escaped exponents (rare for weights): rewrite those values; __syncwarp
    // orders them after the assembly's stores of the same addresses
    if (x1 > x0) {
      __syncwarp();
      for (uint32_t i = x0 + lane; i < x1; i += 32) {
        const uint32_t rec = __ldg(S.xrec + i), idx = rec >> 8;
        const uint32_t b = __ldg(smb + idx);
        dst[idx] = (uint16_t)(((b & 0x80u) << 8) | ((rec & 0xffu) << 7) | (b & 0x7fu));
      }
    }
    __syncwarp();
  }
  spmoe::span_end(p.span);
}

inline uint64_t align256(uint64_t x) { return (x + 255) & ~uint64_t(255); }
inline int64_t nblocks(int64_t n) { return n / SPMOE_XC_BLOCK; }

// work layout per segment (u32 words):
//   hist[256] | bofs[nb+1] | lanes[nb*32 bytes] | xofs[nb+1] | lbase[nb u16]
inline size_t seg_lanes_words(int64_t n) { return (size_t)nblocks(n) * kLanes / 4; }
inline size_t seg_xofs_word(int64_t n) { return 256 + (size_t)(nblocks(n) + 1) + seg_lanes_words(n); }
inline size_t seg_lbase_word(int64_t n) { return seg_xofs_word(n) + (size_t)(nblocks(n) + 1); }
inline size_t seg_work_words(int64_t n) { return seg_lbase_word(n) + (size_t)(nblocks(n) + 1) / 2; }

// The segment's base exponent (restates oracle_xc_base, oracle/xc_oracle.c):
// the lowest b <= 240 whose window [b, b + 14] holds the most values.
uint32_t base_of(const uint32_t* hist) {
  uint32_t best = 0;
  uint64_t best_mass = 0;
  for (uint32_t b = 0; b <= 240; ++b) {
    uint64_t m = 0;
    for (uint32_t e = b; e < b + kEsc; ++e) m += hist[e];
    if (m > best_mass) {
      best_mass = m;
      best = b;
    }
  }
  return best;
}

// Code lengths of the 16 symbols (restates oracle_xc_code_lengths).
void code_lengths(const uint64_t* cnt, uint8_t len[kNsym]) {
  std::memset(len, 0, kNsym);
  int sym[kNsym], n = 0;
  for (int s = 0; s < kNsym; ++s)
    if (cnt[s]) sym[n++] = s;
  if (n == 0) return;
  if (n == 1) {
    len[sym[0]] = 1;
    return;
  }
  std::stable_sort(sym, sym + n, [&](int a, int b) { return cnt[a] < cnt[b]; });
  uint64_t w[2 * kNsym];
  int parent[2 * kNsym], depth[2 * kNsym];
  for (int i = 0; i < n; ++i) w[i] = cnt[sym[i]];
  int li = 0, ii = n, next = n;
  for (int k = 0; k < n - 1; ++k) {
    int pick[2];
    for (int t = 0; t < 2; ++t) {
      if (li < n && (ii == next || w[li] <= w[ii])) pick[t] = li++;
      else pick[t] = ii++;
    }
    w[next] = w[pick[0]] + w[pick[1]];
    parent[pick[0]] = parent[pick[1]] = next;
    ++next;
  }
  const int root = 2 * n - 2;
  depth[root] = 0;
  for (int v = root - 1; v >= 0; --v) depth[v] = depth[parent[v]] + 1;
  int maxlen = 0;
  for (int i = 0; i < n; ++i) {
    len[sym[i]] = (uint8_t)depth[i];
    maxlen = std::max(maxlen, depth[i]);
  }
  if (maxlen <= kLmax) return;
  int64_t kraft = 0;
  for (int s = 0; s < kNsym; ++s) {
    if (!len[s]) continue;
    if (len[s] > kLmax) len[s] = kLmax;
    kraft += (int64_t)1 << (kLmax - len[s]);
  }
  while (kraft > ((int64_t)1 << kLmax)) {
    int best = -1;
    for (int s = 0; s < kNsym; ++s) {
      if (!len[s] || len[s] >= kLmax) continue;
      if (best < 0 || len[s] > len[best] ||
          (len[s] == len[best] && (cnt[s] < cnt[best] || (cnt[s] == cnt[best] && s > best))))
        best = s;
    }
    kraft -= (int64_t)1 << (kLmax - len[best] - 1);
    len[best]++;
  }
}

// Canonical codes of the 16 symbols, bit-reversed (LSB-first packing).
void sym_codes(const uint8_t len[kNsym], uint16_t rev[kNsym]) {
  std::memset(rev, 0, sizeof(uint16_t) * kNsym);
  uint32_t code = 0;
  int prev = 0;
  for (int L = 1; L <= kLmax; ++L)
    for (int s = 0; s < kNsym; ++s) {
      if (len[s] != L) continue;
      if (prev) code <<= (L - prev);
      prev = L;
      uint32_t r = 0;
      for (int b = 0; b < L; ++b) r |= ((code >> b) & 1u) << (L - 1 - b);
      rev[s] = (uint16_t)r;
      ++code;
    }
}

// Per-exponent code table for the encoder kernels.
void codes_of(const spmoe_xc_segment& g, Codes* c) {
  uint16_t rev[kNsym];
  sym_codes(g.len, rev);
  for (uint32_t e = 0; e < 256; ++e) {
    const uint32_t y = escaped(e, g.base) ? (uint32_t)kEsc : e - g.base;
    c->rev[e] = rev[y];
    c->len[e] = g.len[y];
  }
  c->base = g.base;
}

// Single-symbol table: entry q = symbol | length << 8 (restates oracle_xc_lut).
void lut_of(const uint8_t len[kNsym], uint16_t* lut) {
  uint16_t rev[kNsym];
  sym_codes(len, rev);
  std::memset(lut, 0, sizeof(uint16_t) * kLutSize);
  for (int s = 0; s < kNsym; ++s) {
    const int L = len[s];
    if (!L) continue;
    for (uint32_t q = 0; q < (1u << (kLmax - L)); ++q) lut[rev[s] | (q << L)] = (uint16_t)(s | (L << 8));
  }
}

// Multi-symbol table (restated in oracle_xc_lut2, oracle/xc_oracle.c): up to
// five whole codes in the 12 peeked bits.
void lut2_of(const uint16_t* lut, uint32_t* lut2) {
  for (uint32_t q = 0; q < (uint32_t)kLutSize; ++q) {
    const uint32_t e0 = lut[q];
    uint32_t tot = e0 >> 8, cnt = 1, syms = e0 & 0xfu;
    if (tot == 0) tot = 1;  // unused pattern of an incomplete code: always progress
    while (cnt < 5) {
      const uint32_t e = lut[q >> tot], l = e >> 8;
      if (!l || tot + l > (uint32_t)kLmax) break;
      syms |= (e & 0xfu) << (4 * cnt);
      ++cnt;
      tot += l;
    }
    lut2[q] = syms | ((4 * cnt) << 20) | (tot << 25);
  }
}

bool valid_segments(int nseg, const int64_t* seg_n) {
  if (nseg < 1 || nseg > SPMOE_XC_MAX_SEG || !seg_n) return false;
  for (int i = 0; i < nseg; ++i)
    if (seg_n[i] <= 0 || seg_n[i] % SPMOE_XC_BLOCK) return false;
  return true;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
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
  const int sms = num_sms();
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
  std::vector<uint32_t> hist(256 * nseg);
  off = 0;
  for (int i = 0; i < nseg; ++i) {
    cudaMemcpyAsync(&hist[256 * i], wk + off, 256 * 4, cudaMemcpyDeviceToHost, st);
    off += seg_work_words(seg_n[i]);
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
  std::memset(hdr, 0, sizeof(*hdr));
  hdr->magic = SPMOE_XC_MAGIC;
  hdr->nseg = (uint32_t)nseg;
  // 2. base, codes, per-block word and exception counts, prefixes
  off = 0;
  s = src;
  for (int i = 0; i < nseg; ++i) {
    const int64_t n = seg_n[i], nb = nblocks(n);
    spmoe_xc_segment& g = hdr->seg[i];
    const uint32_t* h = &hist[256 * i];
    g.base = base_of(h);
    uint64_t cnt[kNsym] = {};
    for (uint32_t x = 0; x < 256; ++x) cnt[escaped(x, g.base) ? kEsc : x - g.base] += h[x];
    code_lengths(cnt, g.len);
    g.n = (uint64_t)n;
    Codes c;
    codes_of(g, &c);
    uint32_t* bofs = wk + off + 256;
    uint8_t* lanes = (uint8_t*)(bofs + nb + 1);
    uint32_t* xofs = wk + off + seg_xofs_word(n);
    uint16_t* lbase = (uint16_t*)(wk + off + seg_lbase_word(n));
    xc_count_kernel<<<(unsigned)((nb + kWarps - 1) / kWarps), kThreads, 0, st>>>(s, nb, c, bofs, lanes, lbase, xofs);
    xc_scan_kernel<<<1, 1024, 0, st>>>(bofs, nb);
    xc_scan_kernel<<<1, 1024, 0, st>>>(xofs, nb);
    off += seg_work_words(n);
    s += n;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  std::vector<uint32_t> tot(2 * nseg);
  off = 0;
  for (int i = 0; i < nseg; ++i) {
    cudaMemcpyAsync(&tot[2 * i], wk + off + 256 + nblocks(seg_n[i]), 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&tot[2 * i + 1], wk + off + seg_xofs_word(seg_n[i]) + nblocks(seg_n[i]), 4,
                    cudaMemcpyDeviceToHost, st);
    off += seg_work_words(seg_n[i]);
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
  // 3. layout
  uint64_t pos = align256(sizeof(spmoe_xc_header)), raw = 0;
  for (int i = 0; i < nseg; ++i) {
    spmoe_xc_segment& g = hdr->seg[i];
    const int64_t n = seg_n[i], nb = nblocks(n);
    g.ex_words = tot[2 * i];
    g.n_exc = tot[2 * i + 1];
    g.off_lut = pos; pos = align256(pos + 4 * (uint64_t)kLutSize);
    g.off_sm = pos; pos = align256(pos + (uint64_t)n);
    g.off_ex = pos; pos = align256(pos + (uint64_t)g.ex_words * 4 + 8);
    g.off_bofs = pos; pos = align256(pos + (uint64_t)(nb + 1) * 4);
    g.off_lanes = pos; pos = align256(pos + (uint64_t)nb * kLanes);
    g.off_lbase = pos; pos = align256(pos + (uint64_t)nb * 2);
    g.off_xofs = pos; pos = align256(pos + (uint64_t)(nb + 1) * 4);
    g.off_xrec = pos; pos = align256(pos + (uint64_t)g.n_exc * 4);
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
  for (uint32_t i = 0; i < hdr->nseg; ++i)
    if (hdr->seg[i].base > 240) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(blob, 0, hdr->blob_bytes, st);
  if (e != cudaSuccess) return (int)e;
  const uint32_t* wk = (const uint32_t*)work;
  std::vector<uint16_t> luts((size_t)hdr->nseg * kLutSize);
  std::vector<uint32_t> luts2((size_t)hdr->nseg * kLutSize);
  size_t off = 0;
  const uint16_t* s = src;
  for (uint32_t i = 0; i < hdr->nseg; ++i) {
    const spmoe_xc_segment& g = hdr->seg[i];
    const int64_t n = (int64_t)g.n, nb = nblocks(n);
    WriteParams p;
    p.src = s;
    p.nb = nb;
    p.sm = blob + g.off_sm;
    p.ex = (uint32_t*)(blob + g.off_ex);
    p.bofs = wk + off + 256;
    p.lanes = (const uint8_t*)(p.bofs + nb + 1);
    p.xofs = wk + off + seg_xofs_word(n);
    p.lbase = (const uint16_t*)(wk + off + seg_lbase_word(n));
    p.xrec = (uint32_t*)(blob + g.off_xrec);
    codes_of(g, &p.c);
    xc_write_kernel<<<(unsigned)((nb + kWarps - 1) / kWarps), kThreads, 0, st>>>(p);
    cudaMemcpyAsync(blob + g.off_bofs, p.bofs, (nb + 1) * 4, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(blob + g.off_lanes, p.lanes, nb * kLanes, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(blob + g.off_xofs, p.xofs, (nb + 1) * 4, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(blob + g.off_lbase, p.lbase, nb * 2, cudaMemcpyDeviceToDevice, st);
    lut_of(g.len, &luts[(size_t)i * kLutSize]);
    lut2_of(&luts[(size_t)i * kLutSize], &luts2[(size_t)i * kLutSize]);
    cudaMemcpyAsync(blob + g.off_lut, &luts2[(size_t)i * kLutSize], 4 * kLutSize, cudaMemcpyHostToDevice, st);
    off += seg_work_words(n);
    s += n;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  if ((e = cudaMemcpyAsync(blob, hdr, sizeof(*hdr), cudaMemcpyHostToDevice, st)) != cudaSuccess) return (int)e;
  return (int)cudaStreamSynchronize(st);  // luts / luts2 / hdr are host memory
}

int spmoe_xc_decode_segments_timed(const uint8_t* blob, const spmoe_xc_header* hdr, int first, int count,
                                   uint16_t* dst, void* stream, void* span) {
  if (!blob || !hdr || !dst || hdr->magic != SPMOE_XC_MAGIC || hdr->nseg < 1 || hdr->nseg > SPMOE_XC_MAX_SEG ||
      first < 0 || count < 1 || first + count > (int)hdr->nseg)
    return (int)cudaErrorInvalidValue;
  DecParams p;
  std::memset(&p, 0, sizeof(p));
  p.span = (spmoe::DevSpan*)span;
  static const int stcs = [] {
    // evict-first output stores: in the SD loop 0.605 -> 0.624 of the copy
    // peak and the concurrent multi-expert K3 launches 346 -> 320 us
    // (tools/ab_stcs.sh, one box)
    const char* v = getenv("SPMOE_XC_STCS");
    return v && v[0] == '0' ? 0 : 1;
  }();
  p.stream_stores = stcs;
  uint16_t* d = dst;
  for (int i = 0; i < first; ++i) d += hdr->seg[i].n;
  uint32_t maxblk = 0;
  for (int j = 0; j < count; ++j) {
    const spmoe_xc_segment& g = hdr->seg[first + j];
    if (g.n == 0 || g.n % SPMOE_XC_BLOCK) return (int)cudaErrorInvalidValue;
    DecSeg& S = p.seg[j];
    S.lut2 = (const uint32_t*)(blob + g.off_lut);
    S.sm = blob + g.off_sm;
    S.ex = (const uint32_t*)(blob + g.off_ex);
    S.bofs = (const uint32_t*)(blob + g.off_bofs);
    S.lanes = blob + g.off_lanes;
    S.lbase = (const uint16_t*)(blob + g.off_lbase);
    S.xofs = (const uint32_t*)(blob + g.off_xofs);
    S.xrec = (const uint32_t*)(blob + g.off_xrec);
    S.dst = d;
    S.nblk = (uint32_t)(g.n / SPMOE_XC_BLOCK);
    if (g.base > 240) return (int)cudaErrorInvalidValue;
    S.base4 = g.base * 0x01010101u;
    maxblk = std::max(maxblk, S.nblk);
    d += g.n;
  }
  static const bool attr = [] {
    cudaFuncSetAttribute(xc_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmemBytes);
    return true;
  }();
  (void)attr;
  const uint32_t want = (uint32_t)std::max(1, kDecCtas * num_sms() / count);
  const uint32_t gx = std::max(1u, std::min(want, (maxblk + kDecWarps - 1) / kDecWarps));
  xc_decode_kernel<<<dim3(gx, count), kDecThreads, kDecSmemBytes, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

int spmoe_xc_decode_segments(const uint8_t* blob, const spmoe_xc_header* hdr, int first, int count,
                             uint16_t* dst, void* stream) {
  return spmoe_xc_decode_segments_timed(blob, hdr, first, count, dst, stream, nullptr);
}

int spmoe_xc_decode(const uint8_t* blob, const spmoe_xc_header* hdr, uint16_t* dst, void* stream) {
  if (!hdr) return (int)cudaErrorInvalidValue;
  return spmoe_xc_decode_segments(blob, hdr, 0, (int)hdr->nseg, dst, stream);
}

}  // extern "C"
