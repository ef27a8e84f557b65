// common.cuh -- shared device primitives for the B200 kNN-graph path.
//
// * exact-order distances: the reference accumulates sqrt(sum (a-b)^2) in fp32
//   one dimension at a time with separately rounded sub/mul/add and a final
//   sqrtss (core.hpp:23-30).  Every kernel here computes
//   a distance with that exact operation order (explicit __fsub_rn / __fmul_rn
//   / __fadd_rn so ptxas can never contract to FFMA), which makes stored
//   distances bit-identical to the reference's recomputation and lets every
//   (dist,id) comparison decide exactly as the CPU does.
// * packed keys: (float_bits(dist) << 32) | id.  dist >= 0, so u64 order is the
//   reference tie rule closer() (core.hpp:136-139).
// * counter-based SplitMix64: draw m of a stream seeded s is
//   mix(s + (m+1)*gamma) (rng.hpp:16-21), so streams are random-access.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace knng_b200 {

using u32 = uint32_t;
using u64 = uint64_t;

constexpr u64 kEmptyKey = ~0ull;
constexpr u64 kGamma = 0x9e3779b97f4a7c15ull;
constexpr unsigned kFull = 0xffffffffu;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define KNNG_CUDA(expr)                                                                   \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::knng_b200::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                   " at " + __FILE__ + ":" + std::to_string(__LINE__));   \
  } while (0)

// Every kernel launch is followed by KNNG_LAUNCH_CHECK(), which also counts it
// (process-wide; read through knng_kernel_launches()).
inline std::atomic<unsigned long long>& launch_counter() {
  static std::atomic<unsigned long long> c{0};
  return c;
}
#define KNNG_LAUNCH_CHECK()                                               \
  do {                                                                    \
    ::knng_b200::launch_counter().fetch_add(1, std::memory_order_relaxed); \
    KNNG_CUDA(cudaGetLastError());                                        \
  } while (0)

// ---------------------------------------------------------------------------
// SplitMix64 (rng.hpp:12-63)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ u64 sm64_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct Rng {
  u64 state;
  __host__ __device__ __forceinline__ explicit Rng(u64 s) : state(s) {}
  __host__ __device__ __forceinline__ u64 next_u64() { return sm64_mix(state += kGamma); }
  __host__ __device__ __forceinline__ u64 next_below(u64 bound) {
#ifdef __CUDA_ARCH__
    return __umul64hi(next_u64(), bound);
#else
    return (u64)(((unsigned __int128)next_u64() * bound) >> 64);
#endif
  }
};

__host__ __device__ __forceinline__ u64 mix_seed(u64 a, u64 b) {
  Rng r(a ^ (b * kGamma + 0xd1b54a32d192ed03ull));
  return r.next_u64();
}

// Draw m (0-based) of the stream that Rng(s) would produce.
__host__ __device__ __forceinline__ u64 sm64_draw(u64 s, u64 m) {
  return sm64_mix(s + (m + 1) * kGamma);
}

__device__ __forceinline__ u64 mulhi64(u64 x, u64 b) { return __umul64hi(x, b); }

// ---------------------------------------------------------------------------
// packed (dist, id) keys
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ u64 pack_key(float d, u32 id) {
#ifdef __CUDA_ARCH__
  return ((u64)__float_as_uint(d) << 32) | id;
#else
  u32 b;
  memcpy(&b, &d, 4);
  return ((u64)b << 32) | id;
#endif
}
__host__ __device__ __forceinline__ u32 key_id(u64 k) { return (u32)k; }
__device__ __forceinline__ float key_dist(u64 k) { return __uint_as_float((u32)(k >> 32)); }

// ---------------------------------------------------------------------------
// exact-order distance (core.hpp:23-30)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float sq_step(float acc, float a, float b) {
  const float t = __fsub_rn(a, b);
  return __fadd_rn(acc, __fmul_rn(t, t));
}

// Two dims at once: the differences and squares use Blackwell's packed
// FADD2/FMUL2 (IEEE round-to-nearest per component, identical to the scalar
// ops); the accumulation stays scalar and sequential.  A packed accumulate
// would be contracted by ptxas into FFMA2 (single rounding) -- measured to
// change 31% of distances -- so the adds must not be f32x2.
__device__ __forceinline__ float sq_step2(float acc, float a0, float a1, float b0, float b1) {
  unsigned long long A, B, T;
  asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(T) : "l"(A), "l"(B));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(T) : "l"(T));
  float s0, s1;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(s0), "=f"(s1) : "l"(T));
  return __fadd_rn(__fadd_rn(acc, s0), s1);
}

__device__ __forceinline__ float sq_step4(float acc, float4 a, float4 b) {
  acc = sq_step2(acc, a.x, a.y, b.x, b.y);
  return sq_step2(acc, a.z, a.w, b.z, b.w);
}

// ---------------------------------------------------------------------------
// cosine (core.hpp:41-55): dot, na and nb are three independent sequential
// chains.  A row's norm chain does not depend on its partner, so it is
// computed once per row (row_norms_device) and only the dot runs per pair;
// the finish repeats the reference's operations in order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float dot_step(float acc, float a, float b) {
  return __fadd_rn(acc, __fmul_rn(a, b));
}
__device__ __forceinline__ float dot_step2(float acc, float a0, float a1, float b0, float b1) {
  unsigned long long A, B, T;
  asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(T) : "l"(A), "l"(B));
  float s0, s1;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(s0), "=f"(s1) : "l"(T));
  return __fadd_rn(__fadd_rn(acc, s0), s1);
}
__device__ __forceinline__ float dot_step4(float acc, float4 a, float4 b) {
  acc = dot_step2(acc, a.x, a.y, b.x, b.y);
  return dot_step2(acc, a.z, a.w, b.z, b.w);
}
__device__ __forceinline__ float cos_finish(float dot, float na, float nb) {
  if (na == 0.0f || nb == 0.0f) return 1.0f;
  const float v = __fsub_rn(1.0f, __fdiv_rn(dot, __fmul_rn(__fsqrt_rn(na), __fsqrt_rn(nb))));
  return v < 0.0f ? 0.0f : v;
}

// Metric-generic steps: kCos selects the dot chain, else the L2 chain.
template <bool kCos>
__device__ __forceinline__ float m_step4(float acc, float4 a, float4 b) {
  return kCos ? dot_step4(acc, a, b) : sq_step4(acc, a, b);
}
template <bool kCos>
__device__ __forceinline__ float m_step(float acc, float a, float b) {
  return kCos ? dot_step(acc, a, b) : sq_step(acc, a, b);
}
// Distance from a finished accumulator; na/nb (row norm chains) read only for cosine.
template <bool kCos>
__device__ __forceinline__ float m_finish(float acc, float na, float nb) {
  return kCos ? cos_finish(acc, na, nb) : __fsqrt_rn(acc);
}

// Full exact distance between two global/shared rows.
__device__ __forceinline__ float l2_exact(const float* __restrict__ a,
                                          const float* __restrict__ b, int d) {
  float acc = 0.0f;
  int i = 0;
  if ((((uintptr_t)a | (uintptr_t)b) & 15) == 0) {
    for (; i + 4 <= d; i += 4)
      acc = sq_step4(acc, *reinterpret_cast<const float4*>(a + i),
                     *reinterpret_cast<const float4*>(b + i));
  }
  for (; i < d; ++i) acc = sq_step(acc, a[i], b[i]);
  return __fsqrt_rn(acc);
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Bitonic sort of one u64 key per lane, ascending across lanes 0..31.
__device__ __forceinline__ u64 warp_sort32(u64 v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const u64 other = __shfl_xor_sync(kFull, v, stride);
      const bool up = ((lane & size) == 0);
      const bool lower = ((lane & stride) == 0);
      // keep min if (lower && up) || (!lower && !up)
      const bool take_min = (lower == up);
      v = take_min ? (other < v ? other : v) : (other > v ? other : v);
    }
  }
  return v;
}

template <class T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}

}  // namespace knng_b200
