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
#include <initializer_list>
#include <ctime>
#include <cstring>
#include <cstdlib>
#include <sys/mman.h>

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
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap map2, const char* base,
                                                       int tiles_per_cta, unsigned* sink,
                                                       unsigned long long* stamps) {
  constexpr int STAGE = BOXR * 64 * 2;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  if (threadIdx.x == 0 && stamps) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(&stamps[0], t);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int kblocks = kCols / 64;
  const int n_iter = MODE == 2 ? 64 : MODE == 3 ? 192 : tiles_per_cta * kblocks;
  // tile rows per CTA: BOXR rows per tile
  if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t ph = 0;
    for (int it = 0; it < n_iter; ++it) {
      const int t = blockIdx.x * tiles_per_cta + it / kblocks, kb = it % kblocks;
      wait_bar(&empty[stage], ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[stage])), "r"(STAGE)
                   : "memory");
      if (MODE >= 2) {
        // K3 unit stream: (MODE 3) W1 then W3 tile m over all 64 k-blocks,
        // then (MODE 2, 3) W2's 128-column block m as 32 row tiles x 2 boxes
        const int m = blockIdx.x % 112, ex = blockIdx.x / 112;
        const int n_up = MODE == 3 ? 2 * kblocks : 0;
        int c0, r0;
        const CUtensorMap* mp;
        if (it < n_up) {
          mp = &map;
          c0 = (it >> 1) * 64;
          r0 = ex * 28672 + (it & 1) * 14336 + m * 128;
        } else {
          const int d = it - n_up;
          mp = &map2;
          c0 = m * 128 + (d & 1) * 64;
          r0 = ex * 4096 + (d >> 1) * 128;
        }
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
            "[%2];" ::"r"(su32(sm + stage * STAGE)),
            "l"(mp), "r"(su32(&full[stage])), "r"(c0), "r"(r0)
            : "memory");
      } else if (MODE == 0) {
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
    if (stamps) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(&stamps[1], t);
    }
  }
}

__global__ void stamp_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// optional concurrent pinned H2D copy during every timed launch
static void* g_h2d_src = nullptr;
static void* g_h2d_dst = nullptr;
static size_t g_h2d_bytes = 0;
static cudaStream_t g_side = nullptr;
static unsigned long long* g_stamps = nullptr;
static bool g_graph = false;
static float g_gap0 = 0, g_gap1 = 0;  // us: stamp kernel -> first CTA start, last CTA end -> stamp kernel  // launch the kernel as a pre-uploaded CUDA graph

static CUtensorMap g_map2;  // W2-shaped [rows, 14336] map for MODE 2/3
template <int MODE, int BOXR, int S>
void run(const char* name, void* buf, size_t rows, unsigned* sink, EncodeFn enc, int per_cta_mb = 8,
         std::initializer_list<int> grids = {16, 32, 64, 112, 128, 148, 296}) {
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
  for (int G : grids) {
    // each CTA streams per_cta_mb MB (or as many whole tiles as fit)
    int tpc = (int)(((size_t)per_cta_mb << 20) / tile_bytes);
    if (tpc < 1) tpc = 1;
    if ((size_t)G * tpc > (size_t)total_tiles) tpc = total_tiles / G;
    if (MODE >= 2) tpc = 0;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f, best_in = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      unsigned long long init[2] = {~0ull, 0ull};
      cudaMemcpy(g_stamps, init, sizeof(init), cudaMemcpyHostToDevice);
      cudaDeviceSynchronize();
      cudaGraphExec_t ge = nullptr;
      cudaStream_t cs = nullptr;
      if (g_graph) {
        cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        cudaGraph_t gr;
        cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        stream_kernel<MODE, BOXR, S><<<G, 64, smem, cs>>>(map, g_map2, (const char*)buf, tpc, sink, g_stamps);
        cudaStreamEndCapture(cs, &gr);
        cudaGraphInstantiate(&ge, gr, 0);
        cudaGraphUpload(ge, cs);
        cudaStreamSynchronize(cs);
        cudaGraphDestroy(gr);
      }
      if (g_h2d_bytes) {
        cudaMemcpyAsync(g_h2d_dst, g_h2d_src, g_h2d_bytes, cudaMemcpyHostToDevice, g_side);
        struct timespec ts2 = {0, 200000};
        nanosleep(&ts2, nullptr);
      }
      cudaEventRecord(a, cs);
      stamp_kernel<<<1, 1, 0, cs>>>(g_stamps + 2);
      if (g_graph) cudaGraphLaunch(ge, cs);
      else stream_kernel<MODE, BOXR, S><<<G, 64, smem, cs>>>(map, g_map2, (const char*)buf, tpc, sink, g_stamps);
      stamp_kernel<<<1, 1, 0, cs>>>(g_stamps + 3);
      cudaEventRecord(b, cs);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
      if (ge) cudaGraphExecDestroy(ge);
      if (cs) cudaStreamDestroy(cs);
      unsigned long long st[4];
      cudaMemcpy(st, g_stamps, sizeof(st), cudaMemcpyDeviceToHost);
      const float in_ms = (float)(st[1] - st[0]) / 1e6f;
      if (in_ms < best_in) {
        best_in = in_ms;
        g_gap0 = (float)(st[0] - st[2]) / 1e3f;
        g_gap1 = (float)(st[3] - st[1]) / 1e3f;
      }
    }
    const double bytes = MODE == 2 ? (double)G * 64 * STAGE : MODE == 3 ? (double)G * 192 * STAGE
                                                                      : (double)G * tpc * tile_bytes;
    const int active = G > 148 ? 148 : G;
    printf("%-8s S=%2d stage=%5d B  G=%3d  %2d MB/CTA  %8.1f GB/s  %6.1f GB/s/SM  (%.1f us events, %.1f us first CTA start -> last CTA end; gaps %.1f / %.1f us)\n",
           name, S, STAGE, G, tpc * (int)(tile_bytes >> 20), bytes / best / 1e6, bytes / best / 1e6 / active, best * 1e3,
           best_in * 1e3, g_gap0, g_gap1);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
}

int main(int argc, char** argv) {
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
  cudaMalloc(&g_stamps, 32);
  if (argc > 1 && !strcmp(argv[1], "unit")) {
    // K3's single-expert unit stream without math: up (W1|W3 tile m) 2 MB,
    // down (W2 column block m, 256 B per row at a 28 KB stride) 1 MB
    void* w2;
    const size_t rows2 = 4096 * 12;
    cudaMalloc(&w2, rows2 * 14336 * 2);
    cudaMemset(w2, 1, rows2 * 14336 * 2);
    cuuint64_t d[2] = {14336, (cuuint64_t)rows2}, st[1] = {14336 * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&g_map2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w2, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int rep = 0; rep < 2; ++rep) {
      run<0, 128, 12>("tile128", buf, rows, sink, enc, 2, {112});
      run<0, 128, 12>("tile128", buf, rows, sink, enc, 3, {112});
      run<2, 128, 12>("down", buf, rows, sink, enc, 1, {112, 224, 448});
      run<3, 128, 12>("unit", buf, rows, sink, enc, 3, {112, 224});
      run<3, 128, 8>("unit", buf, rows, sink, enc, 3, {112});
    }
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "h2dsrc")) {
    // does the pinned source's page size change the penalty?  cudaMallocHost
    // vs 2 MB-aligned THP-advised memory registered with cudaHostRegister vs
    // hugetlbfs pages
    system("cat /sys/kernel/mm/transparent_hugepage/enabled; grep -i huge /proc/meminfo");
    g_h2d_bytes = 1ull << 30;
    cudaMalloc(&g_h2d_dst, g_h2d_bytes);
    cudaStreamCreateWithFlags(&g_side, cudaStreamNonBlocking);
    for (int kind = 0; kind < 3; ++kind) {
      void* src = nullptr;
      const char* nm = "";
      if (kind == 0) {
        cudaMallocHost(&src, g_h2d_bytes);
        nm = "cudaMallocHost";
      } else if (kind == 1) {
        if (posix_memalign(&src, 2u << 20, g_h2d_bytes)) src = nullptr;
        if (src) {
          madvise(src, g_h2d_bytes, MADV_HUGEPAGE);
          memset(src, 1, g_h2d_bytes);
          if (cudaHostRegister(src, g_h2d_bytes, cudaHostRegisterPortable) != cudaSuccess) src = nullptr;
        }
        nm = "THP+cudaHostRegister";
      } else {
        src = mmap(nullptr, g_h2d_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB, -1, 0);
        if (src == MAP_FAILED) src = nullptr;
        if (src) {
          memset(src, 1, g_h2d_bytes);
          if (cudaHostRegister(src, g_h2d_bytes, cudaHostRegisterPortable) != cudaSuccess) src = nullptr;
        }
        nm = "hugetlb+cudaHostRegister";
      }
      if (!src) {
        printf("# %s: unavailable\n", nm);
        cudaGetLastError();
        continue;
      }
      system("grep -i AnonHugePages /proc/meminfo");
      g_h2d_src = src;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, g_side);
      cudaMemcpyAsync(g_h2d_dst, src, g_h2d_bytes, cudaMemcpyHostToDevice, g_side);
      cudaEventRecord(b, g_side);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("# source %s: H2D %.1f GB/s\n", nm, g_h2d_bytes / ms / 1e6);
      run<0, 128, 8>("tile128", buf, rows, sink, enc, 3, {112});
      run<0, 128, 8>("tile128", buf, rows, sink, enc, 8, {148});
    }
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "h2d")) {
    // the same streaming with a 1 GiB pinned H2D copy in flight
    g_h2d_bytes = 1ull << 30;
    cudaMallocHost(&g_h2d_src, g_h2d_bytes);
    cudaMalloc(&g_h2d_dst, g_h2d_bytes);
    cudaStreamCreateWithFlags(&g_side, cudaStreamNonBlocking);
    for (int pass = 0; pass < 4; ++pass) {
      g_graph = pass >= 2;
      printf("# concurrent H2D: %s, %s\n", pass & 1 ? "on" : "off", g_graph ? "CUDA graph launch" : "stream launch");
      if (!(pass & 1)) g_h2d_bytes = 0; else g_h2d_bytes = 1ull << 30;
      run<0, 128, 8>("tile128", buf, rows, sink, enc, 3, {112, 148});
      run<0, 128, 8>("tile128", buf, rows, sink, enc, 8, {112, 148});
      run<1, 128, 8>("bulk16k", buf, rows, sink, enc, 8, {148});
    }
    return 0;
  }
  if (argc > 1) {
    // short streams: K3's single-expert up phase is 2 MB per CTA on 112 CTAs
    for (int mb : {1, 2, 3, 4, 8}) {
      run<0, 128, 8>("tile128", buf, rows, sink, enc, mb, {112, 148});
      run<0, 128, 12>("tile128", buf, rows, sink, enc, mb, {112, 148});
    }
    return 0;
  }
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
