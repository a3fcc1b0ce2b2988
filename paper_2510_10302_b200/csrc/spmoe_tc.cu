// spmoe_tc.cu — tcgen05/TMEM/TMA path of K3 (grouped SwiGLU over the HBM
// slot pool) for sm_100a.
//
// Swap-AB: the expert weight rows are the MMA's M dimension (tiles of 128
// rows), the routed tokens of one expert are N (padded to a multiple of 16,
// at most 64 per tile), K is the reduction (H for the up phase, F for the
// down phase).  Weight tiles [128 x 64] and activation tiles [64 x 64] are
// fetched by TMA (128B swizzle) from 3-D tensor maps over the slot pool
// (slot = outer coordinate, so no per-expert descriptor rebuilds) into a
// multi-stage shared-memory ring; one elected thread issues tcgen05.mma
// (kind::f16, bf16 x bf16 -> fp32) into a double-buffered TMEM accumulator;
// four epilogue warps drain TMEM with tcgen05.ld and apply SiLU*up (up
// phase) or write fp32 partial sums (down phase, split-K, reduced in a fixed
// order afterwards).
//
// Numerics: fp32 accumulation in the tensor core's order, so results match
// the CPU oracle within fp32 rounding (tolerance documented in
// tests/test_tc_gpu.py) rather than bit for bit; the CUDA-core path of
// spmoe_kernels.cu is the bit-exact one.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>

#include "../../include/spmoe.h"
#include "spmoe_common.cuh"

using namespace spmoe;

namespace tc {

constexpr int BM = 128;  // weight rows per tile (UMMA M)
constexpr int BK = 64;   // K elements per stage (128 bytes: one swizzle atom row)
constexpr int BN = 64;   // max tokens per tile (activation box rows)
constexpr int kThreads = 192;  // warp 0 TMA, warp 1 MMA + TMEM alloc, warps 2-5 epilogue
constexpr int kMaxExperts = 64;
constexpr int kTmemCols = 256;

struct Params {
  uint64_t mask;
  const int32_t* offsets;
  uint16_t* h_out;  // up, split 1: [rows, F] bf16
  float* g_part;    // up, split > 1: [split][rows, F] fp32 (gate), then up
  float* y_part;    // down: [split][rows, H] fp32 (split 1: y itself)
  DevSpan* span_end;  // optional device-clock span closed by this launch
  int E, H, F, rows, split;
  int slot[kMaxExperts];
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Programmatic dependent launch: a kernel lets the next one in its stream
// start launching (its CTAs then run their prologue on free SMs), and that
// one waits for this grid's completion and memory before touching its
// inputs.  Both are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
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

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Same with an L2 cache policy (createpolicy): weights are read once per
// launch, so they stream through L2 as evict-first and leave the lines a
// preceding decode just wrote (the slot's last segment) for the reads that
// follow.
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Four arbitrary rows of a 2-D map with box {64, 1}: 4 x 128 B land as
// consecutive 128-byte rows at dst (the 128B swizzle follows the shared
// memory address, so a group at a 512-byte offset is rows 4..7 of its atom).
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int r0, int r1,
                                            int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

// K-major operand, 128-byte swizzle, 8-row atoms of 1024 bytes (SBO), LBO
// unused (1), descriptor version 1 (sm100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128.
__device__ __forceinline__ uint32_t instr_desc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 lanes x 16 columns of 32-bit from TMEM (one row per thread).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32"
      " {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------ tile list
// Tiles enumerate (active expert, token chunk of <= BN, 128-row block,
// K split); every role walks the same static sequence.
struct TileList {
  int n_active;
  int active[kMaxExperts];
  int start[kMaxExperts + 1];  // prefix of tiles per active expert
};

__device__ __forceinline__ void build_tiles(const Params& p, int mtiles, int split, TileList* tl) {
  if (threadIdx.x == 0) {
    int n = 0, acc = 0;
    for (int e = 0; e < p.E; ++e) {
      const int cnt = p.offsets[e + 1] - p.offsets[e];
      if (((p.mask >> e) & 1ull) && cnt > 0) {
        tl->active[n] = e;
        tl->start[n] = acc;
        acc += ((cnt + BN - 1) / BN) * mtiles * split;
        ++n;
      }
    }
    tl->start[n] = acc;
    tl->n_active = n;
  }
}

struct Tile {
  int e, n0, ntok, m0, kb0, kb1, ks;
};

__device__ __forceinline__ Tile decode(const Params& p, const TileList& tl, int tile, int mtiles, int split,
                                       int kblocks) {
  int a = 0;
  while (tile >= tl.start[a + 1]) ++a;
  int r = tile - tl.start[a];
  Tile t;
  t.e = tl.active[a];
  t.ks = r % split;
  r /= split;
  t.m0 = (r % mtiles) * BM;
  r /= mtiles;
  t.n0 = r * BN;
  const int cnt = p.offsets[t.e + 1] - p.offsets[t.e];
  t.ntok = min(BN, cnt - t.n0);
  t.kb0 = kblocks * t.ks / split;
  t.kb1 = kblocks * (t.ks + 1) / split;
  return t;
}

template <bool UP, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
ffn_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_act,
              const Params p) {
  constexpr int A_BYTES = BM * BK * 2;          // 16 KB weight tile
  constexpr int B_BYTES = BN * BK * 2;          // 8 KB activation tile
  constexpr int NA = UP ? 2 : 1;                // W1 + W3 tiles in the up phase
  constexpr int STAGE_BYTES = NA * A_BYTES + B_BYTES;
  constexpr int ACC_COLS = UP ? 2 * BN : BN;    // g | u, or y
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ TileList tl;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = UP ? p.H : p.F;
  const int R = UP ? p.F : p.H;
  const int kblocks = K / BK;
  const int mtiles = R / BM;
  const int split = p.split;
  pdl_launch_dependents();

  build_tiles(p, mtiles, split, &tl);  // offsets come from K2, two launches back
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  const int ntiles = tl.start[tl.n_active];
  pdl_wait();  // the previous kernel's activations / partials are complete

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const Tile t = decode(p, tl, tile, mtiles, split, kblocks);
        const int slot = p.slot[t.e];
        const int arow = p.offsets[t.e] + t.n0;
        for (int kb = t.kb0; kb < t.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
          tma_load_3d(st, &map_w, &full_bar[stage], kb * BK, t.m0, slot);
          if (UP) tma_load_3d(st + A_BYTES, &map_w, &full_bar[stage], kb * BK, p.F + t.m0, slot);
          tma_load_2d(st + NA * A_BYTES, &map_act, &full_bar[stage], kb * BK, arow);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread)
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const Tile t = decode(p, tl, tile, mtiles, split, kblocks);
        const int n = ((t.ntok + 15) / 16) * 16;
        const uint32_t idesc = instr_desc(n);
        mbar_wait(&tempty_bar[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * ACC_COLS;
        for (int kb = t.kb0; kb < t.kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * STAGE_BYTES;
          const uint64_t a0 = smem_desc_sw128(st);
          const uint64_t a1 = smem_desc_sw128(st + A_BYTES);
          const uint64_t b0 = smem_desc_sw128(st + NA * A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t accum = (kb > t.kb0 || k > 0) ? 1u : 0u;
            // +32 bytes per K=16 step inside the swizzle atom (desc units of 16 B)
            umma(d, a0 + 2 * k, b0 + 2 * k, idesc, accum);
            if (UP) umma(d + BN, a1 + 2 * k, b0 + 2 * k, idesc, accum);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5, TMEM lane quarter = warp % 4
    const int q = warp & 3;
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const Tile t = decode(p, tl, tile, mtiles, split, kblocks);
      mbar_wait(&tfull_bar[acc], aphase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + acc * ACC_COLS;
      const int row = t.m0 + 32 * q + lane;
      const int64_t prow = p.offsets[t.e] + t.n0;
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        if (c0 < t.ntok) {  // warp-uniform
          float g[16], u[16];
          tmem_ld16(taddr + c0, g);
          if (UP) tmem_ld16(taddr + BN + c0, u);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            if (c0 + c < t.ntok) {
              if (UP) {
                if (split == 1) {
                  p.h_out[(prow + c0 + c) * p.F + row] = f32_to_bf16(__fmul_rn(det_silu(g[c]), u[c]));
                } else {
                  const int64_t i = ((int64_t)t.ks * p.rows + prow + c0 + c) * p.F + row;
                  p.g_part[i] = g[c];
                  p.g_part[(int64_t)split * p.rows * p.F + i] = u[c];
                }
              } else {
                p.y_part[((int64_t)t.ks * p.rows + prow + c0 + c) * p.H + row] = g[c];
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
  span_end(p.span_end);
}

// ------------------------------------------------------------------ fused
// One persistent cooperative launch for both phases of one K3 call: every
// CTA walks its up tiles, its epilogue signals a grid-wide counter once its
// last h store is visible, and the down phase starts; the TMA producer
// issues the W2 (A operand) loads of its first STAGES down stages before
// waiting for the counter (weights do not depend on h), so the barrier and
// the W2 ramp overlap the up phase's tail.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
ffn_tc_fused_kernel(const __grid_constant__ CUtensorMap map_wu, const __grid_constant__ CUtensorMap map_x,
                    const __grid_constant__ CUtensorMap map_wd, const __grid_constant__ CUtensorMap map_h,
                    const Params p, uint32_t* grid_sync) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = 2 * A_BYTES + B_BYTES;  // sized for the up phase
  constexpr int UP_TX = 2 * A_BYTES + B_BYTES;
  constexpr int DN_TX = A_BYTES + B_BYTES;
  constexpr int ACC_COLS = 2 * BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ TileList tl_up, tl_dn;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb_up = p.H / BK, kb_dn = p.F / BK;
  const int mt_up = p.F / BM, mt_dn = p.H / BM;
  const int split = p.split;

  build_tiles(p, mt_up, 1, &tl_up);
  build_tiles(p, mt_dn, split, &tl_dn);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  const int n_up = tl_up.start[tl_up.n_active];
  const int n_dn = tl_dn.start[tl_dn.n_active];

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < n_up; tile += gridDim.x) {
        const Tile t = decode(p, tl_up, tile, mt_up, 1, kb_up);
        const int slot = p.slot[t.e];
        const int arow = p.offsets[t.e] + t.n0;
        for (int kb = t.kb0; kb < t.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full_bar[stage], UP_TX);
          tma_load_3d(st, &map_wu, &full_bar[stage], kb * BK, t.m0, slot);
          tma_load_3d(st + A_BYTES, &map_wu, &full_bar[stage], kb * BK, p.F + t.m0, slot);
          tma_load_2d(st + 2 * A_BYTES, &map_x, &full_bar[stage], kb * BK, arow);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      // down phase: W2 loads run ahead of the grid barrier for up to STAGES
      // stages; their h loads are issued once every up tile is stored
      int pend_stage[STAGES], pend_kb[STAGES], pend_row[STAGES];
      int npend = 0;
      bool synced = false;
      for (int tile = blockIdx.x; tile < n_dn; tile += gridDim.x) {
        const Tile t = decode(p, tl_dn, tile, mt_dn, split, kb_dn);
        const int slot = p.slot[t.e];
        const int arow = p.offsets[t.e] + t.n0;
        for (int kb = t.kb0; kb < t.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full_bar[stage], DN_TX);
          tma_load_3d(st, &map_wd, &full_bar[stage], kb * BK, t.m0, slot);
          if (synced) {
            tma_load_2d(st + A_BYTES, &map_h, &full_bar[stage], kb * BK, arow);
          } else {
            pend_stage[npend] = stage;
            pend_kb[npend] = kb;
            pend_row[npend] = arow;
            if (++npend == STAGES) {
              while (ld_acquire_u32(grid_sync) < gridDim.x) __nanosleep(64);
              asm volatile("fence.proxy.async.global;" ::: "memory");
              for (int i = 0; i < npend; ++i)
                tma_load_2d(smem + pend_stage[i] * STAGE_BYTES + A_BYTES, &map_h, &full_bar[pend_stage[i]],
                            pend_kb[i] * BK, pend_row[i]);
              npend = 0;
              synced = true;
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (!synced && npend > 0) {
        while (ld_acquire_u32(grid_sync) < gridDim.x) __nanosleep(64);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        for (int i = 0; i < npend; ++i)
          tma_load_2d(smem + pend_stage[i] * STAGE_BYTES + A_BYTES, &map_h, &full_bar[pend_stage[i]],
                      pend_kb[i] * BK, pend_row[i]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int ph = 0; ph < 2; ++ph) {
        const bool up = ph == 0;
        const int ntile = up ? n_up : n_dn;
        for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
          const Tile t = up ? decode(p, tl_up, tile, mt_up, 1, kb_up) : decode(p, tl_dn, tile, mt_dn, split, kb_dn);
          const uint32_t idesc = instr_desc(((t.ntok + 15) / 16) * 16);
          mbar_wait(&tempty_bar[acc], aphase ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + acc * ACC_COLS;
          for (int kb = t.kb0; kb < t.kb1; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            uint8_t* st = smem + stage * STAGE_BYTES;
            const uint64_t a0 = smem_desc_sw128(st);
            const uint64_t a1 = smem_desc_sw128(st + A_BYTES);
            const uint64_t b0 = smem_desc_sw128(st + (up ? 2 * A_BYTES : A_BYTES));
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint32_t accum = (kb > t.kb0 || k > 0) ? 1u : 0u;
              umma(d, a0 + 2 * k, b0 + 2 * k, idesc, accum);
              if (up) umma(d + BN, a1 + 2 * k, b0 + 2 * k, idesc, accum);
            }
            umma_commit(&empty_bar[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          umma_commit(&tfull_bar[acc]);
          if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
      }
    }
  } else {
    const int q = warp & 3;
    int acc = 0;
    uint32_t aphase = 0;
    for (int ph = 0; ph < 2; ++ph) {
      const bool up = ph == 0;
      const int ntile = up ? n_up : n_dn;
      for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const Tile t = up ? decode(p, tl_up, tile, mt_up, 1, kb_up) : decode(p, tl_dn, tile, mt_dn, split, kb_dn);
        mbar_wait(&tfull_bar[acc], aphase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + acc * ACC_COLS;
        const int row = t.m0 + 32 * q + lane;
        const int64_t prow = p.offsets[t.e] + t.n0;
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 16) {
          if (c0 < t.ntok) {
            float g[16], u[16];
            tmem_ld16(taddr + c0, g);
            if (up) tmem_ld16(taddr + BN + c0, u);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              if (c0 + c < t.ntok) {
                if (up) {
                  p.h_out[(prow + c0 + c) * p.F + row] = f32_to_bf16(__fmul_rn(det_silu(g[c]), u[c]));
                } else {
                  p.y_part[((int64_t)t.ks * p.rows + prow + c0 + c) * p.H + row] = g[c];
                }
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty_bar[acc]);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
      if (up) {
        // every h store of this CTA is done: publish to the grid (release +
        // generic->async proxy fence for the TMA readers in other CTAs)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          atomicAdd(grid_sync, 1u);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// ------------------------------------------------------------ unit-fused
// ONE launch per K3 call, no grid-wide dependency: a work UNIT is (expert e,
// 128-feature block m).  Its up part streams W1/W3 rows [128m, 128m+128)
// over all of H and yields h[:, 128m:128m+128]; that h block is exactly
// the K-slice of the down phase that W2[:, 128m:128m+128] multiplies, so
// the same CTA runs the down part straight from shared memory (h never
// round-trips through HBM or waits for other CTAs) and writes a partial y_m
// per 128-row output tile; a PDL-chained second launch sums the F/128
// partials of every element in a fixed order (its CTAs are resident and
// waiting before this kernel ends).  (Letting the last unit of each tile
// reduce it inside this kernel was measured 5-50x slower: the slowest CTA
// ends up last on every tile and serialises all the reductions.)  An
// expert's bits depend only on its own units, never on which experts share
// the launch.
// Tokens per expert <= 16 (one N=16 MMA): the SD verify regime.
constexpr int UN = 16;  // tokens per unit (MMA N)
#ifndef SPMOE_UNIT_NY
#define SPMOE_UNIT_NY 2
#endif
constexpr int kUnitNY = SPMOE_UNIT_NY;  // down-phase y accumulators in TMEM (ring)
constexpr int kUnitTmemCols = 32 + 16 * kUnitNY <= 64 ? 64 : 32 + 16 * kUnitNY <= 128 ? 128 : 256;

struct UnitParams {
  const int32_t* offsets;
  const int32_t* perm_token;  // token (row of x) of every routed row, K2 order
  DevSpan* span;
  uint16_t* h_out;      // [rows, F] bf16 (optional copy of h for callers/tests)
  float* y_part;        // [F/128][rows, H] fp32 partials
  int H, F, rows, n_active;
  int active[kMaxExperts];
  int slot[kMaxExperts];
};

#ifdef SPMOE_UNIT_STAMPS
// diagnostic build only (tools/k3_unit_stamps.py): per-CTA globaltimer
// stamps of the unit kernel's phases
__device__ unsigned long long* g_unit_stamps = nullptr;
#define UNIT_STAMP(i)                                                        \
  do {                                                                       \
    if (g_unit_stamps && u == (int)blockIdx.x) {                             \
      unsigned long long t_;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      g_unit_stamps[blockIdx.x * 8 + (i)] = t_;                              \
    }                                                                        \
  } while (0)
#else
#define UNIT_STAMP(i) \
  do {                \
  } while (0)
#endif

template <int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
ffn_tc_unit_kernel(const __grid_constant__ CUtensorMap map_wu, const __grid_constant__ CUtensorMap map_x,
                   const __grid_constant__ CUtensorMap map_wd, const UnitParams p) {
  constexpr int A_BYTES = BM * BK * 2;                // 16 KB weight box
  constexpr int X_BYTES = UN * BK * 2;                // 2 KB: 16 rows of x_perm x 64 features
  constexpr int STAGE_BYTES = 2 * A_BYTES + X_BYTES;  // up: W1 + W3 + x; down: two W2 k-blocks
  constexpr int HB_BYTES = UN * BK * 2;               // one 64-feature k-block of h (K-major, SW128)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* hb = smem + STAGES * STAGE_BYTES;  // h block as the down MMA's B operand: 2 x [16 x 64]
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], gu_full, h_ready, y_full[kUnitNY], y_empty[kUnitNY];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb_up = p.H / BK;
  const int mt_up = p.F / BM;  // units per expert
  const int mt_dn = p.H / BM;  // down M-tiles per unit
  const int n_units = p.n_active * mt_up;
  pdl_launch_dependents();
  span_begin(p.span);
  if (threadIdx.x == 0) {
    { const int u = blockIdx.x; UNIT_STAMP(0); }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&gu_full, 1);
    mbar_init(&h_ready, 128);
    for (int s = 0; s < kUnitNY; ++s) {
      mbar_init(&y_full[s], 1);
      mbar_init(&y_empty[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_wu) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_wd) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
  }
  if (warp == 1) {
    // columns: g [0,16) | u [16,32) | y ring: kUnitNY x 16 from 32
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kUnitTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {
      { const int u = blockIdx.x; UNIT_STAMP(1); }
      // ---------------- TMA producer: per unit, the up stream then the
      // W2 column block (weights never depend on h, so the down loads run
      // ahead while the epilogue turns the up accumulators into h).  x_perm
      // comes from the gather kernel this launch is PDL-chained to: the
      // weight boxes of the first STAGES stages go out before waiting for it.
      // x rows come straight from x by TMA gather4 (rows perm_token[arow ..
      // arow + 16), clamped to the unit's last token: the extra MMA columns
      // are never read back), so no gather kernel precedes this one.
      int stage = 0;
      uint32_t phase = 0;
      bool waited = false;
      int pend_stage[STAGES], pend_kb[STAGES], npend = 0;
      int xr[UN];
      const uint64_t ef = l2_evict_first_policy();
      // offsets / perm_token are read only after griddepcontrol.wait, so
      // whichever kernel precedes this one in the stream may produce them
      auto x_rows = [&](int e) {
        const int arow = p.offsets[e];
        const int ntok = max(1, min(UN, p.offsets[e + 1] - arow));
#pragma unroll
        for (int i = 0; i < UN; ++i) xr[i] = p.perm_token[arow + min(i, ntok - 1)];
      };
      auto load_x = [&](uint8_t* dst, uint64_t* bar, int kb) {
#pragma unroll
        for (int g = 0; g < UN / 4; ++g)
          tma_gather4(dst + g * 512, &map_x, bar, kb * BK, xr[4 * g], xr[4 * g + 1], xr[4 * g + 2], xr[4 * g + 3]);
      };
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int a = u / mt_up, m = u - a * mt_up;
        const int e = p.active[a], slot = p.slot[a];
        if (waited) x_rows(e);
        for (int kb = 0; kb < kb_up; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
          tma_load_3d_hint(st, &map_wu, &full_bar[stage], kb * BK, m * BM, slot, ef);
          tma_load_3d_hint(st + A_BYTES, &map_wu, &full_bar[stage], kb * BK, p.F + m * BM, slot, ef);
          if (waited) {
            load_x(st + 2 * A_BYTES, &full_bar[stage], kb);
          } else {
            // the first stages' weights go out before the dependency on the
            // producer of x / perm_token resolves
            pend_stage[npend] = stage;
            pend_kb[npend] = kb;
            if (++npend == STAGES || kb + 1 == kb_up) {
              pdl_wait();
              x_rows(e);
              for (int i = 0; i < npend; ++i)
                load_x(smem + pend_stage[i] * STAGE_BYTES + 2 * A_BYTES, &full_bar[pend_stage[i]], pend_kb[i]);
              npend = 0;
              waited = true;
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        for (int j = 0; j < mt_dn; ++j) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full_bar[stage], 2 * A_BYTES);
          tma_load_3d_hint(st, &map_wd, &full_bar[stage], m * BM, j * BM, slot, ef);
          tma_load_3d_hint(st + A_BYTES, &map_wd, &full_bar[stage], m * BM + BK, j * BM, slot, ef);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        UNIT_STAMP(6);
      }
      if (!waited) pdl_wait();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      const uint32_t idesc = instr_desc(UN);
      const uint32_t d_g = tmem_base, d_u = tmem_base + 16;
      int stage = 0, acc = 0;
      uint32_t phase = 0, hphase = 0, aphase = 0;
      const uint64_t hb0 = smem_desc_sw128(hb), hb1 = smem_desc_sw128(hb + HB_BYTES);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        // up: g, u accumulators (free: the previous unit's down MMAs, issued
        // after its h_ready, imply its epilogue has drained them)
        for (int kb = 0; kb < kb_up; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          if (kb == 0) UNIT_STAMP(2);
          tc_fence_after();
          uint8_t* st = smem + stage * STAGE_BYTES;
          const uint64_t a0 = smem_desc_sw128(st), a1 = smem_desc_sw128(st + A_BYTES);
          const uint64_t b0 = smem_desc_sw128(st + 2 * A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t accum = (kb > 0 || k > 0) ? 1u : 0u;
            umma(d_g, a0 + 2 * k, b0 + 2 * k, idesc, accum);
            umma(d_u, a1 + 2 * k, b0 + 2 * k, idesc, accum);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&gu_full);
        UNIT_STAMP(3);
        // down: B = this unit's h block from shared memory
        mbar_wait(&h_ready, hphase);
        hphase ^= 1;
        UNIT_STAMP(5);
        tc_fence_after();
        for (int j = 0; j < mt_dn; ++j) {
          mbar_wait(&y_empty[acc], aphase ^ 1);
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * STAGE_BYTES;
          const uint64_t a0 = smem_desc_sw128(st), a1 = smem_desc_sw128(st + A_BYTES);
          const uint32_t d = tmem_base + 32 + 16 * acc;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) umma(d, a0 + 2 * k, hb0 + 2 * k, idesc, k > 0 ? 1u : 0u);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) umma(d, a1 + 2 * k, hb1 + 2 * k, idesc, 1u);
          umma_commit(&empty_bar[stage]);
          umma_commit(&y_full[acc]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (++acc == kUnitNY) { acc = 0; aphase ^= 1; }
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5, TMEM lane quarter q = warp % 4
    const int q = warp & 3;
    const int fl = 32 * q + lane;  // feature row within the unit (up), h row within the tile (down)
    int acc = 0;
    uint32_t gphase = 0, aphase = 0;
    const int64_t plane = (int64_t)p.rows * p.H;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int a = u / mt_up, m = u - a * mt_up;
      const int e = p.active[a];
      mbar_wait(&gu_full, gphase);  // after the producer's griddepcontrol.wait (x box -> MMA -> commit)
      gphase ^= 1;
      tc_fence_after();
      const int r0 = p.offsets[e];
      const int ntok = min(UN, p.offsets[e + 1] - r0);
      float g[16], v[16];
      const uint32_t lq = (uint32_t)(32 * q) << 16;
      tmem_ld16(tmem_base + lq, g);
      tmem_ld16(tmem_base + lq + 16, v);
      tmem_wait_ld();
      // h -> shared memory in the K-major 128B-swizzled layout the down
      // MMA reads: k-block fl / 64, row = token, 16-byte chunk XOR row % 8
      uint8_t* hk = hb + (fl >> 6) * HB_BYTES;
      const int k = fl & 63;
#pragma unroll
      for (int n = 0; n < UN; ++n) {
        const uint16_t hv = n < ntok ? f32_to_bf16(__fmul_rn(det_silu(g[n]), v[n])) : (uint16_t)0;
        const uint32_t off = (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + ((((k >> 3) ^ (n & 7)) << 4)) + (k & 7) * 2);
        *reinterpret_cast<uint16_t*>(hk + off) = hv;
        if (p.h_out && n < ntok) p.h_out[(int64_t)(r0 + n) * p.F + m * BM + fl] = hv;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
      tc_fence_before();
      mbar_arrive(&h_ready);
      if (threadIdx.x == 64) UNIT_STAMP(4);
      float* yp = p.y_part + (int64_t)m * plane;
      for (int j = 0; j < mt_dn; ++j) {
        mbar_wait(&y_full[acc], aphase);
        tc_fence_after();
        float y[16];
        tmem_ld16(tmem_base + lq + 32 + 16 * acc, y);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&y_empty[acc]);
        if (++acc == kUnitNY) { acc = 0; aphase ^= 1; }
        const int col = j * BM + fl;
#pragma unroll
        for (int n = 0; n < UN; ++n)
          if (n < ntok) __stcg(yp + (int64_t)(r0 + n) * p.H + col, y[n]);
      }
      if (threadIdx.x == 64) UNIT_STAMP(7);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kUnitTmemCols));
  }
}

// y[r, :] = sum over the F/128 unit partials of r's expert, for the rows of
// experts in `mask`.  Eight threads per output element each add a
// contiguous eighth of the partials in order, then the eight sums combine
// in a fixed tree (shuffles): deterministic, and the partials' loads are
// in flight together.
__global__ void reduce_units_kernel(const float* __restrict__ part, int nparts, int rows, int H,
                                    const int32_t* __restrict__ offsets, int E, uint64_t mask,
                                    float* __restrict__ y, DevSpan* span) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t n = (int64_t)rows * H;
  const int sub = threadIdx.x & 7;
  const int per = (nparts + 7) / 8;
  const int s0 = sub * per, s1 = min(nparts, s0 + per);
  for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3; i0 < n;
       i0 += ((int64_t)gridDim.x * blockDim.x) >> 3) {
    const int r = (int)(i0 / H);
    int e = 0;
    while (e < E - 1 && r >= offsets[e + 1]) ++e;
    const bool live = (mask >> e) & 1ull;  // uniform over the 8 lanes of an element
    float s = 0.0f;
    if (live && s0 < s1) {
      float v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = (s0 + t < s1) ? __ldcg(part + (int64_t)(s0 + t) * n + i0) : 0.0f;
      s = v[0];
#pragma unroll
      for (int t = 1; t < 16; ++t)
        if (s0 + t < s1) s = __fadd_rn(s, v[t]);
      for (int t = s0 + 16; t < s1; ++t) s = __fadd_rn(s, __ldcg(part + (int64_t)t * n + i0));
    }
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
    if (live && sub == 0) y[i0] = s;
  }
  span_end(span);
}

// y[r, :] = sum_s y_part[s][r, :] in split order (deterministic), only for
// rows of experts in this launch's mask (other rows keep their values).
__global__ void reduce_split_kernel(const float* __restrict__ part, int split, int rows, int H,
                                    const int32_t* __restrict__ offsets, int E, uint64_t mask,
                                    float* __restrict__ y, DevSpan* span) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t n = (int64_t)rows * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / H);
    int e = 0;
    while (e < E - 1 && r >= offsets[e + 1]) ++e;
    if (!((mask >> e) & 1ull)) continue;
    float s = part[i];
    for (int k = 1; k < split; ++k) s = __fadd_rn(s, part[(int64_t)k * n + i]);
    y[i] = s;
  }
  span_end(span);
}

// h[r, f] = bf16(silu(sum_s g) * sum_s u), split order, masked rows only.
__global__ void reduce_swiglu_kernel(const float* __restrict__ part, int split, int rows, int F,
                                     const int32_t* __restrict__ offsets, int E, uint64_t mask,
                                     uint16_t* __restrict__ h) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t n = (int64_t)rows * F;
  const float* up = part + (int64_t)split * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / F);
    int e = 0;
    while (e < E - 1 && r >= offsets[e + 1]) ++e;
    if (!((mask >> e) & 1ull)) continue;
    float g = part[i], u = up[i];
    for (int k = 1; k < split; ++k) {
      g = __fadd_rn(g, part[(int64_t)k * n + i]);
      u = __fadd_rn(u, up[(int64_t)k * n + i]);
    }
    h[i] = f32_to_bf16(__fmul_rn(det_silu(g), u));
  }
}

// x_perm[r] = x[perm[r]] (activation rows grouped by expert for TMA).
__global__ void gather_rows_kernel(const uint16_t* __restrict__ x, const int32_t* __restrict__ perm,
                                   const int32_t* __restrict__ offsets, int E, int H, uint16_t* __restrict__ out,
                                   DevSpan* span) {
  span_begin(span);
  pdl_launch_dependents();  // launched normally: its inputs are complete
  const int rows = offsets[E];
  const int nch = H >> 3;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)rows * nch;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / nch), c = (int)(i - (int64_t)r * nch);
    reinterpret_cast<uint4*>(out + (int64_t)r * H)[c] =
        reinterpret_cast<const uint4*>(x + (int64_t)perm[r] * H)[c];
  }
}

// -------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)ptr;
  }
  return fn;
}

// bf16 tensor map, 128B swizzle, box = {64, box_rows, 1}; dims/strides in
// elements / bytes, innermost first.
bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
              uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[3], s[2];
  cuuint32_t box[3] = {(cuuint32_t)BK, box_rows, 1}, es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) d[i] = dims[i];
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)rank, const_cast<void*>(base), d, s, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Launch with programmatic stream serialization (see pdl_wait).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const int no_pdl = getenv("SPMOE_NO_PDL") != nullptr;  // A/B switch
  cfg.numAttrs = no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <bool UP, int STAGES>
int launch(const CUtensorMap& mw, const CUtensorMap& ma, const Params& p, int nsms, cudaStream_t s) {
  constexpr int NA = UP ? 2 : 1;
  constexpr int STAGE_BYTES = NA * BM * BK * 2 + BN * BK * 2;
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ffn_tc_kernel<UP, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  return (int)launch_pdl(ffn_tc_kernel<UP, STAGES>, dim3(nsms), dim3(kThreads), smem, s, mw, ma, p);
}

}  // namespace tc

extern "C" int spmoe_expert_ffn_tc(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                                   uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E, int k,
                                   const int32_t* expert_offsets, const int32_t* perm_token, uint16_t* x_perm,
                                   uint16_t* h_scratch, float* y, float* workspace, int split_up, int split_dn,
                                   void* stream) {
  using namespace tc;
  if (!pool || !slot_of_expert || !expert_offsets || T < 0 || E < 1 || E > kMaxExperts || k < 1)
    return (int)cudaErrorInvalidValue;
  if (H % BM || F % BM || H % BK || F % BK || split_up < 1 || split_dn < 1) return (int)cudaErrorInvalidValue;
  if (split_up > H / BK || split_dn > F / BK) return (int)cudaErrorInvalidValue;
  if (T == 0 || expert_mask == 0) return 0;
  if (!x || !perm_token || !x_perm || !h_scratch || !y || ((split_up > 1 || split_dn > 1) && !workspace))
    return (int)cudaErrorInvalidValue;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, nsms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsms, cudaDevAttrMultiProcessorCount, dev);
  const int rows = T * k;
  Params p{};
  p.mask = expert_mask;
  p.offsets = expert_offsets;
  p.h_out = h_scratch;
  p.g_part = workspace;
  p.E = E;
  p.H = H;
  p.F = F;
  p.rows = rows;
  int max_slot = 0;
  for (int e = 0; e < E; ++e) {
    p.slot[e] = ((expert_mask >> e) & 1ull) ? slot_of_expert[e] : 0;
    if (p.slot[e] > max_slot) max_slot = p.slot[e];
  }
  int st = 0;
  CUtensorMap mw_up, ma_up, mw_dn, ma_dn;
  const uint64_t sb = (uint64_t)slot_elems * 2;
  {
    const uint64_t d[3] = {(uint64_t)H, (uint64_t)2 * F, (uint64_t)max_slot + 1};
    const uint64_t str[2] = {(uint64_t)H * 2, sb};
    if (!make_map(&mw_up, pool, 3, d, str, BM)) return (int)cudaErrorInvalidValue;
    const uint64_t da[2] = {(uint64_t)H, (uint64_t)rows};
    const uint64_t sa[1] = {(uint64_t)H * 2};
    if (!make_map(&ma_up, x_perm, 2, da, sa, BN)) return (int)cudaErrorInvalidValue;
  }
  {
    const uint64_t d[3] = {(uint64_t)F, (uint64_t)H, (uint64_t)max_slot + 1};
    const uint64_t str[2] = {(uint64_t)F * 2, sb};
    if (!make_map(&mw_dn, pool + (int64_t)2 * F * H, 3, d, str, BM)) return (int)cudaErrorInvalidValue;
    const uint64_t da[2] = {(uint64_t)F, (uint64_t)rows};
    const uint64_t sa[1] = {(uint64_t)F * 2};
    if (!make_map(&ma_dn, h_scratch, 2, da, sa, BN)) return (int)cudaErrorInvalidValue;
  }
  DevSpan* span = (DevSpan*)k3_timing().dspan;
  k3_timing_begin(s);
  gather_rows_kernel<<<nsms, 256, 0, s>>>(x, perm_token, expert_offsets, E, H, x_perm, span);
  p.split = split_up;
  st = launch<true, 5>(mw_up, ma_up, p, nsms, s);
  if (st) return st;
  if (split_up > 1) {
    st = (int)launch_pdl(reduce_swiglu_kernel, dim3(nsms * 4), dim3(256), 0, s, (const float*)workspace, split_up,
                         rows, F, expert_offsets, E, expert_mask, h_scratch);
    if (st) return st;
  }
  p.split = split_dn;
  p.y_part = split_dn > 1 ? workspace : y;
  p.span_end = split_dn > 1 ? nullptr : span;
  st = launch<false, 8>(mw_dn, ma_dn, p, nsms, s);
  if (st) return st;
  if (split_dn > 1) {
    st = (int)launch_pdl(reduce_split_kernel, dim3(nsms * 4), dim3(256), 0, s, (const float*)workspace, split_dn,
                         rows, H, expert_offsets, E, expert_mask, y, span);
  }
  k3_timing_end(s);
  return st;
}

extern "C" int spmoe_expert_ffn_tc_fused(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                                         uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E,
                                         int k, const int32_t* expert_offsets, const int32_t* perm_token,
                                         uint16_t* x_perm, uint16_t* h_scratch, float* y, float* workspace,
                                         int split_dn, uint32_t* grid_sync, void* stream) {
  using namespace tc;
  if (!pool || !slot_of_expert || !expert_offsets || !grid_sync || T < 0 || E < 1 || E > kMaxExperts || k < 1)
    return (int)cudaErrorInvalidValue;
  if (H % BM || F % BM || split_dn < 1 || split_dn > F / BK) return (int)cudaErrorInvalidValue;
  if (T == 0 || expert_mask == 0) return 0;
  if (!x || !perm_token || !x_perm || !h_scratch || !y || (split_dn > 1 && !workspace))
    return (int)cudaErrorInvalidValue;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, nsms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsms, cudaDevAttrMultiProcessorCount, dev);
  const int rows = T * k;
  Params p{};
  p.mask = expert_mask;
  p.offsets = expert_offsets;
  p.h_out = h_scratch;
  p.y_part = split_dn > 1 ? workspace : y;
  p.E = E;
  p.H = H;
  p.F = F;
  p.rows = rows;
  p.split = split_dn;
  int max_slot = 0;
  for (int e = 0; e < E; ++e) {
    p.slot[e] = ((expert_mask >> e) & 1ull) ? slot_of_expert[e] : 0;
    if (p.slot[e] > max_slot) max_slot = p.slot[e];
  }
  int st = 0;
  CUtensorMap mwu, mx, mwd, mh;
  const uint64_t sb = (uint64_t)slot_elems * 2;
  {
    const uint64_t d[3] = {(uint64_t)H, (uint64_t)2 * F, (uint64_t)max_slot + 1};
    const uint64_t str[2] = {(uint64_t)H * 2, sb};
    if (!make_map(&mwu, pool, 3, d, str, BM)) return (int)cudaErrorInvalidValue;
    const uint64_t da[2] = {(uint64_t)H, (uint64_t)rows};
    const uint64_t sa[1] = {(uint64_t)H * 2};
    if (!make_map(&mx, x_perm, 2, da, sa, BN)) return (int)cudaErrorInvalidValue;
    const uint64_t d2[3] = {(uint64_t)F, (uint64_t)H, (uint64_t)max_slot + 1};
    const uint64_t str2[2] = {(uint64_t)F * 2, sb};
    if (!make_map(&mwd, pool + (int64_t)2 * F * H, 3, d2, str2, BM)) return (int)cudaErrorInvalidValue;
    const uint64_t dh[2] = {(uint64_t)F, (uint64_t)rows};
    const uint64_t sh[1] = {(uint64_t)F * 2};
    if (!make_map(&mh, h_scratch, 2, dh, sh, BN)) return (int)cudaErrorInvalidValue;
  }
  constexpr int STAGES = 5;
  const size_t smem = (size_t)STAGES * (2 * BM * BK * 2 + BN * BK * 2) + 1024;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ffn_tc_fused_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  void* args[] = {(void*)&mwu, (void*)&mx, (void*)&mwd, (void*)&mh, (void*)&p, (void*)&grid_sync};
  k3_timing_begin(s);
  gather_rows_kernel<<<nsms, 256, 0, s>>>(x, perm_token, expert_offsets, E, H, x_perm, nullptr);
  st = (int)cudaMemsetAsync(grid_sync, 0, sizeof(uint32_t), s);
  if (st) return st;
  st = (int)cudaLaunchCooperativeKernel((const void*)ffn_tc_fused_kernel<STAGES>, dim3(nsms), dim3(kThreads), args,
                                        smem, s);
  if (st) return st;
  if (split_dn > 1) {
    st = (int)launch_pdl(reduce_split_kernel, dim3(nsms * 4), dim3(256), 0, s, (const float*)workspace, split_dn,
                         rows, H, expert_offsets, E, expert_mask, y, (DevSpan*)nullptr);
  }
  k3_timing_end(s);
  return st;
}

extern "C" int spmoe_expert_ffn_tc_units(const uint16_t* pool, int64_t slot_elems, const int32_t* slot_of_expert,
                                         uint64_t expert_mask, const uint16_t* x, int T, int H, int F, int E,
                                         int k, const int32_t* expert_offsets, const int32_t* perm_token,
                                         int max_tokens_per_expert, uint16_t* x_perm, uint16_t* h_scratch,
                                         float* y, float* workspace, void* stream) {
  using namespace tc;
  if (!pool || !slot_of_expert || !expert_offsets || T < 0 || E < 1 || E > kMaxExperts || k < 1)
    return (int)cudaErrorInvalidValue;
  if (H % BM || F % BM || max_tokens_per_expert < 0 || max_tokens_per_expert > UN)
    return (int)cudaErrorInvalidValue;
  if (T == 0 || expert_mask == 0) return 0;
  (void)x_perm;  // the unit kernel gathers x rows itself (TMA gather4); kept for the ABI
  if (!x || !perm_token || !y || !workspace) return (int)cudaErrorInvalidValue;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, nsms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsms, cudaDevAttrMultiProcessorCount, dev);
  const int rows = T * k;
  UnitParams p{};
  p.offsets = expert_offsets;
  p.h_out = h_scratch;
  p.y_part = workspace;
  p.H = H;
  p.F = F;
  p.rows = rows;
  int max_slot = 0;
  for (int e = 0; e < E; ++e) {
    if (!((expert_mask >> e) & 1ull)) continue;
    p.active[p.n_active] = e;
    p.slot[p.n_active] = slot_of_expert[e];
    max_slot = max(max_slot, slot_of_expert[e]);
    ++p.n_active;
  }
  CUtensorMap mwu, mx, mwd;
  const uint64_t sb = (uint64_t)slot_elems * 2;
  {
    const uint64_t d[3] = {(uint64_t)H, (uint64_t)2 * F, (uint64_t)max_slot + 1};
    const uint64_t str[2] = {(uint64_t)H * 2, sb};
    if (!make_map(&mwu, pool, 3, d, str, BM)) return (int)cudaErrorInvalidValue;
    const uint64_t da[2] = {(uint64_t)H, (uint64_t)T};
    const uint64_t sa[1] = {(uint64_t)H * 2};
    if (!make_map(&mx, x, 2, da, sa, 1)) return (int)cudaErrorInvalidValue;  // gather4 rows of x
    const uint64_t d2[3] = {(uint64_t)F, (uint64_t)H, (uint64_t)max_slot + 1};
    const uint64_t str2[2] = {(uint64_t)F * 2, sb};
    if (!make_map(&mwd, pool + (int64_t)2 * F * H, 3, d2, str2, BM)) return (int)cudaErrorInvalidValue;
  }
  constexpr int STAGES = 6;
  const size_t smem = (size_t)STAGES * (2 * BM * BK * 2 + UN * BK * 2) + 2 * UN * BK * 2 + 1024;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ffn_tc_unit_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  const int units = p.n_active * (F / BM);
  DevSpan* span = (DevSpan*)k3_timing().dspan;
  p.perm_token = perm_token;
  p.span = span;
  k3_timing_begin(s);
  int st = (int)launch_pdl(ffn_tc_unit_kernel<STAGES>, dim3(min(units, nsms)), dim3(kThreads), smem, s, mwu, mx, mwd,
                           p);
  if (st) return st;
  st = (int)launch_pdl(reduce_units_kernel, dim3(nsms * 2), dim3(256), 0, s, (const float*)workspace, F / BM, rows, H,
                       expert_offsets, E, expert_mask, y, span);
  k3_timing_end(s);
  return st;
}

#ifdef SPMOE_UNIT_STAMPS
extern "C" int spmoe_debug_unit_stamps(void* buf) {
  unsigned long long* p = (unsigned long long*)buf;
  return (int)cudaMemcpyToSymbol(tc::g_unit_stamps, &p, sizeof(p));
}
#endif

/* floats of workspace: the F/128 partial planes of [rows, H] */
extern "C" int64_t spmoe_expert_ffn_tc_units_workspace_floats(int rows, int H, int F) {
  return (int64_t)(F / 128) * rows * H;
}
