// Can SMs pull pinned host memory over PCIe at the copy engine's rate?
// Reads a 1 GiB pinned buffer through its UVA pointer with G CTAs x 256
// threads, 8 independent 16-byte loads in flight per thread; prints GB/s
// per CTA count, next to cudaMemcpyAsync H2D of the same buffer, and the
// same through TMA bulk copies (one thread per CTA, 8 x 16 KB in flight).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zero_copy_read zero_copy_read.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_host(const uint4* __restrict__ src, size_t n16, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcv(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc.x ^= v[k].x; acc.y ^= v[k].y; acc.z ^= v[k].z; acc.w ^= v[k].w; }
  }
  for (; i < n16; i += stride) { uint4 v = __ldcv(src + i); acc.x ^= v.x; }
  if (acc.x == 0x12345678u) sink[0] = acc;
}


// TMA bulk copies (cp.async.bulk global -> shared) of host memory: one
// thread per CTA keeps kStages chunks of kChunk bytes in flight.
constexpr int kChunk = 16384, kStages = 8;
__global__ void bulk_read_host(const char* __restrict__ src, size_t bytes, uint4* sink) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bar[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nchunks = bytes / kChunk;
  unsigned phase[kStages] = {0};
  size_t issued = 0, done = 0;
  size_t c = blockIdx.x;
  auto issue = [&](int s, size_t chunk) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * kChunk);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                 "l"(src + chunk * kChunk), "r"(kChunk), "r"(b) : "memory");
  };
  for (int s = 0; s < kStages && c < nchunks; ++s, c += gridDim.x, ++issued) issue(s, c);
  unsigned acc = 0;
  int s = 0;
  while (done < issued) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(b),
                 "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    acc ^= *(volatile unsigned*)(smem + s * kChunk);
    ++done;
    if (c < nchunks) { issue(s, c); c += gridDim.x; ++issued; }
    s = (s + 1) % kStages;
  }
  if (acc == 0x12345678u) sink[0] = make_uint4(acc, 0, 0, 0);
}

int main() {
  const size_t bytes = 1ull << 30;
  void* h = nullptr;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  for (size_t i = 0; i < bytes; i += 4096) ((char*)h)[i] = (char)i;
  void* d = nullptr;
  cudaMalloc(&d, bytes);
  uint4* sink = nullptr;
  cudaMalloc(&sink, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0;
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(a);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("{\"memcpy_h2d_gbs\": %.1f}\n", bytes / (ms / 1e3) / 1e9);
  const int grids[] = {4, 8, 16, 32, 64, 148, 296};
  for (int g : grids) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      read_host<<<g, 256>>>((const uint4*)h, bytes / 16, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("{\"ctas\": %d, \"zero_copy_gbs\": %.1f, \"err\": \"%s\"}\n", g, bytes / (ms / 1e3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(bulk_read_host, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk);
  for (int g : grids) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      bulk_read_host<<<g, 32, kStages * kChunk>>>((const char*)h, bytes, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("{\"ctas\": %d, \"bulk_copy_gbs\": %.1f, \"err\": \"%s\"}\n", g, bytes / (ms / 1e3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  // both at once: the copy engine on one stream, SM reads of a second
  // pinned buffer on another; total bytes / wall time of the pair
  void* h2 = nullptr;
  cudaHostAlloc(&h2, bytes, cudaHostAllocMapped);
  for (size_t i = 0; i < bytes; i += 4096) ((char*)h2)[i] = (char)i;
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  const int mix[] = {8, 32, 148};
  for (int g : mix) {
    for (int frac = 1; frac <= 4; frac *= 2) {  // SM share: bytes / (frac+1)... CE gets the rest
      const size_t sm_bytes = (bytes / (frac + 1)) & ~(size_t)(kChunk - 1);
      const size_t ce_bytes = bytes - sm_bytes;
      float t = 0;
      for (int r = 0; r < 2; ++r) {
        cudaDeviceSynchronize();
        cudaEventRecord(a, 0);
        cudaStreamWaitEvent(s1, a, 0);
        cudaStreamWaitEvent(s2, a, 0);
        cudaMemcpyAsync(d, h, ce_bytes, cudaMemcpyHostToDevice, s1);
        read_host<<<g, 256, 0, s2>>>((const uint4*)h2, sm_bytes / 16, sink);
        cudaEvent_t e1, e2;
        cudaEventCreate(&e1);
        cudaEventCreate(&e2);
        cudaEventRecord(e1, s1);
        cudaEventRecord(e2, s2);
        cudaStreamWaitEvent(0, e1, 0);
        cudaStreamWaitEvent(0, e2, 0);
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&t, a, b);
      }
      printf("{\"ctas\": %d, \"sm_share\": %.2f, \"ce_plus_sm_gbs\": %.1f}\n", g, (double)sm_bytes / bytes,
             bytes / (t / 1e3) / 1e9);
    }
  }
  return 0;
}
