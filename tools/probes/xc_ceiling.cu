// Memory ceiling of the XC decode's access pattern on one Mixtral W1 segment
// (14336 blocks of 4096 values): what would the decode take if the Huffman
// walk were free?  Kernels, each timed back to back with CUDA events:
//   read_only   stream the 59 MB of sign|mantissa bytes once
//   write_only  write the 117 MB output (16-byte evict-first stores)
//   copyish     the decode's exact traffic: one warp per block reads its
//               4 KB of sign|mantissa bytes and ~1.4 KB of code words and
//               writes its 8 KB of bf16 with a constant exponent, same grid
//               (2 CTAs x 16 warps per SM) and block order as the decoder
//   memcpy      cudaMemcpyAsync device-to-device of the 117 MB output size
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xc_ceiling xc_ceiling.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kBlock = 4096;
constexpr int kBlocks = 14336;
constexpr int kExWords = 346;  // ~2.7 bits per value of code words per block

template <int WARPS>
__global__ void __launch_bounds__(32 * WARPS) copyish(const uint8_t* __restrict__ sm, const uint32_t* __restrict__ ex,
                                                  uint16_t* __restrict__ dst, unsigned* sink) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t acc = 0;
  for (uint32_t blk = warp * gridDim.x + blockIdx.x; blk < kBlocks; blk += gridDim.x * WARPS) {
    const uint32_t* run = ex + (size_t)blk * kExWords;
    for (int i = lane; i < kExWords; i += 32) acc += __ldg(run + i);
    const uint8_t* smb = sm + (size_t)blk * kBlock;
    uint16_t* d = dst + (size_t)blk * kBlock;
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const uint2 m = __ldg(reinterpret_cast<const uint2*>(smb) + it * 32 + lane);
      uint32_t o[4];
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        const uint32_t smw = pr < 2 ? m.x : m.y;
        const uint32_t k = 2 * (pr & 1);
        const uint32_t sel = k | (4u << 4) | ((k + 1) << 8) | (4u << 12);
        const uint32_t ws = __byte_perm(smw, 0u, sel);
        o[pr] = ((ws & 0x00800080u) << 8) | (ws & 0x007f007fu) | 0x3c003c00u;
      }
      __stcs(reinterpret_cast<uint4*>(d) + it * 32 + lane, make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void read_only(const uint4* __restrict__ src, size_t n16, unsigned* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void write_only(uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    __stcs(dst + i, make_uint4(i, i, i, i));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t sm_bytes = (size_t)kBlocks * kBlock, ex_bytes = (size_t)kBlocks * kExWords * 4;
  const size_t out_bytes = 2 * sm_bytes;
  uint8_t *sm, *out, *out2;
  uint32_t* ex;
  unsigned* sink;
  cudaMalloc(&sm, sm_bytes);
  cudaMalloc(&ex, ex_bytes);
  cudaMalloc(&out, out_bytes);
  cudaMalloc(&out2, out_bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(sm, 1, sm_bytes);
  cudaMemset(ex, 2, ex_bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double in_b = (double)(sm_bytes + ex_bytes), alg = in_b + out_bytes;
  auto run = [&](const char* name, double bytes, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    cudaEventRecord(a);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double us = 1e3 * ms / reps;
    printf("{\"kernel\": \"%s\", \"us\": %.2f, \"gbs\": %.1f, \"alg_gbs_of_decode\": %.1f}\n", name, us,
           bytes / us / 1e3, alg / us / 1e3);
  };
  run("copyish 16w x 2/SM (the decoder's grid)", alg, [&] { copyish<16><<<2 * sms, 512>>>(sm, ex, (uint16_t*)out, sink); });
  run("copyish 16w x 4/SM", alg, [&] { copyish<16><<<4 * sms, 512>>>(sm, ex, (uint16_t*)out, sink); });
  run("copyish 8w x 2/SM", alg, [&] { copyish<8><<<2 * sms, 256>>>(sm, ex, (uint16_t*)out, sink); });
  run("copyish 8w x 3/SM", alg, [&] { copyish<8><<<3 * sms, 256>>>(sm, ex, (uint16_t*)out, sink); });
  run("copyish 32w x 2/SM", alg, [&] { copyish<32><<<2 * sms, 1024>>>(sm, ex, (uint16_t*)out, sink); });
  run("copyish 16w x 1/SM", alg, [&] { copyish<16><<<sms, 512>>>(sm, ex, (uint16_t*)out, sink); });
  run("read_only", (double)sm_bytes, [&] { read_only<<<4 * sms, 512>>>((const uint4*)sm, sm_bytes / 16, sink); });
  run("write_only", (double)out_bytes, [&] { write_only<<<4 * sms, 512>>>((uint4*)out, out_bytes / 16); });
  run("memcpy_d2d", 2.0 * out_bytes, [&] { cudaMemcpyAsync(out2, out, out_bytes, cudaMemcpyDeviceToDevice); });
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
