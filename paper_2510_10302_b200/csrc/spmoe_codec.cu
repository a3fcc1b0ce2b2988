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
};

__global__ void __launch_bounds__(kThreads) xc_decode_kernel(const DecParams p) {
  __shared__ uint32_t s_sec[kMaxSecWords];
  __shared__ uint8_t s_tab[16];
  __shared__ int warp_sums[kThreads / 32 + 1];
  int si = 0;
#pragma unroll
  for (int i = 1; i < SPMOE_XC_MAX_SEG; ++i)
    if (i < p.nseg && blockIdx.x >= p.seg[i].blk0) si = i;
  const DecSeg& S = p.seg[si];
  const uint32_t lb = blockIdx.x - S.blk0;
  const int64_t vbase = (int64_t)lb * SPMOE_XC_BLOCK + threadIdx.x * kPerThread;
  const uint32_t w = __ldg(S.pc + vbase / 16);
  const uint4 smv = __ldg(reinterpret_cast<const uint4*>(S.sm) + vbase / 16);
  const uint32_t s0 = __ldg(S.bsec + lb), nw = __ldg(S.bsec + lb + 1) - s0;
  for (uint32_t i = threadIdx.x; i < nw; i += kThreads) s_sec[i] = __ldg(S.sec + s0 + i);
  if (threadIdx.x < 16) s_tab[threadIdx.x] = S.sec_tab[threadIdx.x];
  const uint32_t esc = w & (w >> 1) & 0x55555555u;
  int tot;
  int q = block_exclusive_scan(__popc(esc), warp_sums, &tot);  // syncs: s_sec/s_tab visible
  const uint32_t smw[4] = {smv.x, smv.y, smv.z, smv.w};
  uint32_t out[8];
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    const uint32_t c = (w >> (2 * j)) & 3u;
    const uint32_t b = (smw[j >> 2] >> (8 * (j & 3))) & 0xffu;
    uint32_t e;
    if (c < 3u) {
      e = (S.prim >> (8 * c)) & 0xffu;
    } else {
      const uint32_t nib = (s_sec[q >> 3] >> ((q & 7) * 4)) & 15u;
      ++q;
      if (nib < 15u) {
        e = s_tab[nib];
      } else {
        // exception: (position << 8) | exponent, ascending in the block
        const uint32_t pos = threadIdx.x * kPerThread + j;
        const uint32_t x0 = __ldg(S.bexc + lb), x1 = __ldg(S.bexc + lb + 1);
        e = 0;
        for (uint32_t x = x0; x < x1; ++x) {
          const uint32_t ent = __ldg(S.exc + x);
          if ((ent >> 8) == pos) {
            e = ent & 0xffu;
            break;
          }
        }
      }
    }
    const uint32_t v = ((b & 0x80u) << 8) | (e << 7) | (b & 0x7fu);
    if (j & 1) out[j >> 1] |= v << 16; else out[j >> 1] = v;
  }
  uint4* d = reinterpret_cast<uint4*>(S.dst + vbase);
  d[0] = make_uint4(out[0], out[1], out[2], out[3]);
  d[1] = make_uint4(out[4], out[5], out[6], out[7]);
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

int spmoe_xc_decode(const uint8_t* blob, const spmoe_xc_header* hdr, uint16_t* dst, void* stream) {
  if (!blob || !hdr || !dst || hdr->magic != SPMOE_XC_MAGIC || hdr->nseg < 1 || hdr->nseg > SPMOE_XC_MAX_SEG)
    return (int)cudaErrorInvalidValue;
  DecParams p;
  std::memset(&p, 0, sizeof(p));
  p.nseg = (int)hdr->nseg;
  uint32_t blk = 0;
  uint16_t* d = dst;
  for (uint32_t i = 0; i < hdr->nseg; ++i) {
    const spmoe_xc_segment& g = hdr->seg[i];
    if (g.n == 0 || g.n % SPMOE_XC_BLOCK) return (int)cudaErrorInvalidValue;
    DecSeg& S = p.seg[i];
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
  xc_decode_kernel<<<blk, kThreads, 0, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

}  // extern "C"
