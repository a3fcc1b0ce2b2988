// Shared device helpers for the spmoe sm_100a kernels.
//
// Everything numeric here is part of the determinism contract in
// include/spmoe.h: the CPU oracle (oracle/spmoe_oracle.c) restates each
// helper operation for operation.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define SPMOE_FULL_MASK 0xffffffffu

namespace spmoe {

// Optional CUDA events for the next K3 call on this host thread: recorded
// right before its first kernel and after its last (spmoe_k3_timing), so a
// measured duration excludes host-side launch preparation.
struct K3Timing {
  cudaEvent_t start = nullptr, end = nullptr;
  void* dspan = nullptr;  // DevSpan* (spmoe_k3_devtiming)
};

// Device-clock span of one launch (or one chain of launches): t0 = the
// globaltimer (ns) when the first CTA of the first kernel starts, t1 = when
// the last CTA of the last kernel ends.  Zero-initialised by the host; CUDA
// events around launches are skewed by tens of microseconds while the host
// link is saturated (tools/probes/tma_stream.cu h2d), the device clock is
// not.
struct DevSpan {
  unsigned long long t0, t1;
};
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// thread 0 of every CTA; the earliest CTA wins
__device__ __forceinline__ void span_begin(DevSpan* s) {
  if (s && threadIdx.x == 0) atomicCAS(&s->t0, 0ull, globaltimer_ns());
}
// every thread of the CTA (contains a __syncthreads)
__device__ __forceinline__ void span_end(DevSpan* s) {
  if (!s) return;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&s->t1, globaltimer_ns());
}
K3Timing& k3_timing();
inline void k3_timing_begin(cudaStream_t s) {
  if (k3_timing().start) cudaEventRecord(k3_timing().start, s);
}
inline void k3_timing_end(cudaStream_t s) {
  if (k3_timing().end) cudaEventRecord(k3_timing().end, s);
  k3_timing() = K3Timing{};
}

// bf16 -> f32 for the low / high half of a packed 32-bit word (exact).
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }
__device__ __forceinline__ float bf16_to_f32(uint16_t v) { return __uint_as_float(((uint32_t)v) << 16); }

// f32 -> bf16 round-to-nearest-even (NaN -> canonical quiet NaN).
__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// Deterministic exp: Cody-Waite reduction + degree-7 Taylor polynomial with
// explicit IEEE round-to-nearest mul/add (never contracted to FMA), scaled by
// an exactly constructed power of two.  Identical bits to det_exp() in the
// C oracle.  Inputs below -86 flush to 0, above 88 saturate to +inf.
__device__ __forceinline__ float det_exp(float x) {
  if (x < -86.0f) return 0.0f;
  if (x > 88.0f) return __uint_as_float(0x7f800000u);
  const float n = rintf(__fmul_rn(x, 1.44269504f));
  float r = __fsub_rn(x, __fmul_rn(n, 0.693145752f));
  r = __fsub_rn(r, __fmul_rn(n, 1.42860677e-06f));
  float p = 1.98412698e-04f;
  p = __fadd_rn(__fmul_rn(p, r), 1.38888889e-03f);
  p = __fadd_rn(__fmul_rn(p, r), 8.33333333e-03f);
  p = __fadd_rn(__fmul_rn(p, r), 4.16666667e-02f);
  p = __fadd_rn(__fmul_rn(p, r), 1.66666667e-01f);
  p = __fadd_rn(__fmul_rn(p, r), 0.5f);
  p = __fadd_rn(__fmul_rn(p, r), 1.0f);
  p = __fadd_rn(__fmul_rn(p, r), 1.0f);
  const int ni = (int)n;
  return __fmul_rn(p, __uint_as_float((uint32_t)(ni + 127) << 23));
}

// silu(g) = g / (1 + exp(-g)), IEEE division.
__device__ __forceinline__ float det_silu(float g) {
  return __fdiv_rn(g, __fadd_rn(1.0f, det_exp(-g)));
}

// Butterfly sum over the 32 lanes, offsets 16,8,4,2,1 (all lanes end equal).
__device__ __forceinline__ float warp_sum_fixed(float v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
    v = __fadd_rn(v, __shfl_xor_sync(SPMOE_FULL_MASK, v, off));
  return v;
}

// Streaming 16-byte load of read-once weights: read-only path, no L1
// allocation, 256-byte L2 prefetch granularity.
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Programmatic dependent launch for the non-tcgen05 kernels (spmoe_tc.cu
// has its own copies): grid_dep_trigger lets the next kernel in the stream,
// if launched with the attribute, get scheduled now; grid_dep_wait blocks
// until the previous grid has completed and its writes are visible.  Both
// are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void grid_dep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 16-byte load of re-used activations (L1-cached read-only path).
__device__ __forceinline__ uint4 ldg_act(const uint4* p) { return __ldg(p); }

__device__ __forceinline__ void unpack8(const uint4& v, float f[8]) {
  f[0] = bf16_lo(v.x); f[1] = bf16_hi(v.x);
  f[2] = bf16_lo(v.y); f[3] = bf16_hi(v.y);
  f[4] = bf16_lo(v.z); f[5] = bf16_hi(v.z);
  f[6] = bf16_lo(v.w); f[7] = bf16_hi(v.w);
}

}  // namespace spmoe
