// How fast can ONE SM stream weights from HBM into shared memory, and does
// the access pattern matter?  (Design input for K3's single-expert calls,
// which run their up phase on 112 of 148 SMs.)
//
// Each CTA has one producer thread keeping S stages in flight and one
// consumer thread releasing them (no math).  Patterns:
//   tile128 : 3-D TMA boxes [64 cols x 128 rows] (128B swizzle) over a
//             [rows, 4096] bf16 matrix, tile-major like K3's up phase
//             (one CTA walks its 128-row tiles, 64 k-blocks each)
//   tile256 : same with [64 x 256] boxes (32 KB per instruction)
//   bulk    : 1-D cp.async.bulk of contiguous 16 KB chunks (a pre-tiled layout)
// Prints per CTA count G: aggregate GB/s and GB/s per active SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

constexpr int kCols = 4096;  // K (hidden)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}

// mode 0: tensor boxes of BOXR rows; mode 1: bulk contiguous chunks
template <int MODE, int BOXR, int S>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const char* base,
                                                       int tiles_per_cta, unsigned* sink) {
  constexpr int STAGE = BOXR * 64 * 2;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int kblocks = kCols / 64;
  const int n_iter = tiles_per_cta * kblocks * (128 / BOXR > 0 ? 1 : 1);
  // tile rows per CTA: BOXR rows per tile
  if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t ph = 0;
    for (int it = 0; it < n_iter; ++it) {
      const int t = blockIdx.x * tiles_per_cta + it / kblocks, kb = it % kblocks;
      wait_bar(&empty[stage], ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[stage])), "r"(STAGE)
                   : "memory");
      if (MODE == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
            "[%2];" ::"r"(su32(sm + stage * STAGE)),
            "l"(&map), "r"(su32(&full[stage])), "r"(kb * 64), "r"(t * BOXR)
            : "memory");
      } else {
        const char* src = base + ((size_t)t * kblocks + kb) * STAGE;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(sm + stage * STAGE)),
            "l"(src), "r"(STAGE), "r"(su32(&full[stage]))
            : "memory");
      }
      if (++stage == S) { stage = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int stage = 0;
    uint32_t ph = 0;
    unsigned acc = 0;
    for (int it = 0; it < n_iter; ++it) {
      wait_bar(&full[stage], ph);
      acc += sm[stage * STAGE + (it & 1023)];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[stage])) : "memory");
      if (++stage == S) { stage = 0; ph ^= 1; }
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE, int BOXR, int S>
void run(const char* name, void* buf, size_t rows, unsigned* sink, EncodeFn enc) {
  CUtensorMap map;
  cuuint64_t d[2] = {(cuuint64_t)kCols, (cuuint64_t)rows}, st[1] = {(cuuint64_t)kCols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)BOXR}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  constexpr int STAGE = BOXR * 64 * 2;
  const size_t smem = (size_t)S * STAGE + 1024;
  cudaFuncSetAttribute(stream_kernel<MODE, BOXR, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const size_t tile_bytes = (size_t)BOXR * kCols * 2;
  const int total_tiles = (int)(rows / BOXR);
  for (int G : {16, 32, 64, 112, 128, 148, 296}) {
    // each CTA streams 8 MB (or as many whole tiles as fit)
    int tpc = (int)((8u << 20) / tile_bytes);
    if (tpc < 1) tpc = 1;
    if ((size_t)G * tpc > (size_t)total_tiles) tpc = total_tiles / G;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      stream_kernel<MODE, BOXR, S><<<G, 64, smem>>>(map, (const char*)buf, tpc, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double bytes = (double)G * tpc * tile_bytes;
    const int active = G > 148 ? 148 : G;
    printf("%-8s S=%2d stage=%5d B  G=%3d  %8.1f GB/s  %6.1f GB/s/SM  (%.1f us)\n", name, S, STAGE, G,
           bytes / best / 1e6, bytes / best / 1e6 / active, best * 1e3);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
}

int main() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)ptr;
  const size_t rows = 28672 * 12;  // 12 experts' W1|W3 (2.8 GB): no L2 reuse
  void* buf;
  cudaMalloc(&buf, rows * kCols * 2);
  cudaMemset(buf, 1, rows * kCols * 2);
  unsigned* sink;
  cudaMalloc(&sink, 64);
  run<0, 128, 4>("tile128", buf, rows, sink, enc);
  run<0, 128, 8>("tile128", buf, rows, sink, enc);
  run<0, 128, 12>("tile128", buf, rows, sink, enc);
  run<0, 256, 4>("tile256", buf, rows, sink, enc);
  run<0, 256, 6>("tile256", buf, rows, sink, enc);
  run<1, 128, 4>("bulk16k", buf, rows, sink, enc);
  run<1, 128, 8>("bulk16k", buf, rows, sink, enc);
  run<1, 128, 12>("bulk16k", buf, rows, sink, enc);
  run<1, 256, 6>("bulk32k", buf, rows, sink, enc);
  return 0;
}
