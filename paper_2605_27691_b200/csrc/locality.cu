// locality.cu -- a spatial processing order for a point set.
//
// The reference's ids carry no spatial locality (the generator assigns
// cluster = i mod c, a partition is a random permutation), so work that walks
// the data in id order -- the remote-refine searches, NN-Descent's offers --
// touches cache lines all over HBM.  locality_order() returns a permutation in
// which spatially near points are near each other: a 3-D Morton (Z-order) code
// of three seeded random projections, 10 bits per axis, sorted stably (ties
// keep id order).  Consumers only change the ORDER in which independent work
// runs (the search: tests bit-identical) or renumber a build internally.
#include <algorithm>

#include "locality.hpp"
#include "radix.hpp"

namespace knng_b200 {
namespace {

constexpr int kAxes = 3;
constexpr int kBits = 10;

// projections p[i][a] = <x_i, R_a>, and per-axis min / max (as ordered ints):
// warp per row, lanes over the dims (coalesced row reads), shuffle-reduced
// (a fixed order: the projection only has to be deterministic)
__global__ void k_project(const float* __restrict__ X, u64 n, int d, const float* __restrict__ R,
                          float* __restrict__ P, int* __restrict__ mn, int* __restrict__ mx) {
  __shared__ float sR[kAxes * 1024];
  for (int t = threadIdx.x; t < kAxes * d && t < kAxes * 1024; t += blockDim.x) sR[t] = R[t];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  int lmin[kAxes], lmax[kAxes];
#pragma unroll
  for (int a = 0; a < kAxes; ++a) {
    lmin[a] = 0x7fffffff;
    lmax[a] = (int)0x80000000;
  }
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 i = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    float acc[kAxes] = {0.f, 0.f, 0.f};
    const float* xr = X + i * (u64)d;
    for (int j = lane; j < d; j += 32) {
      const float v = xr[j];
#pragma unroll
      for (int a = 0; a < kAxes; ++a) acc[a] = fmaf(v, sR[a * d + j], acc[a]);
    }
#pragma unroll
    for (int a = 0; a < kAxes; ++a) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], o);
      if (lane == a) P[i * kAxes + a] = acc[a];
      // float -> order-preserving int
      int b = __float_as_int(acc[a]);
      b = b >= 0 ? b : b ^ 0x7fffffff;
      lmin[a] = min(lmin[a], b);
      lmax[a] = max(lmax[a], b);
    }
  }
#pragma unroll
  for (int a = 0; a < kAxes; ++a) {
    if (lane == 0) {
      atomicMin(mn + a, lmin[a]);
      atomicMax(mx + a, lmax[a]);
    }
  }
}

// seeded projection directions (Box-Muller from the counter-based stream) and
// the min / max identities: generated on the device, so the call makes no
// host copy or synchronisation (a build starts its GPU work at once)
__global__ void k_dirs(u64 seed, int count, float* __restrict__ R, int* __restrict__ mm) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
    const u64 a = sm64_mix(seed + (2ull * t + 1) * kGamma);
    const u64 b = sm64_mix(seed + (2ull * t + 2) * kGamma);
    const float u1 = ((float)(a >> 40) + 1.0f) * (1.0f / 16777217.0f);
    const float u2 = (float)(b >> 40) * (1.0f / 16777216.0f);
    R[t] = sqrtf(-2.0f * logf(u1)) * cosf(6.2831853f * u2);
  }
  if (blockIdx.x == 0 && threadIdx.x < 2 * kAxes)
    mm[threadIdx.x] = threadIdx.x < kAxes ? 0x7fffffff : (int)0x80000000;
}

__device__ __forceinline__ float unord(int b) { return __int_as_float(b >= 0 ? b : b ^ 0x7fffffff); }

__global__ void k_morton(const float* __restrict__ P, u64 n, const int* __restrict__ mn,
                         const int* __restrict__ mx, u32* __restrict__ code,
                         u32* __restrict__ idx) {
  float lo[kAxes], scale[kAxes];
#pragma unroll
  for (int a = 0; a < kAxes; ++a) {
    lo[a] = unord(mn[a]);
    const float span = unord(mx[a]) - lo[a];
    scale[a] = span > 0.f ? (float)((1 << kBits) - 1) / span : 0.f;
  }
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    u32 c = 0;
#pragma unroll
    for (int a = 0; a < kAxes; ++a) {
      u32 q = (u32)fminf(fmaxf((P[i * kAxes + a] - lo[a]) * scale[a], 0.f),
                         (float)((1 << kBits) - 1));
#pragma unroll
      for (int b = 0; b < kBits; ++b) c |= ((q >> b) & 1u) << (kAxes * b + a);
    }
    code[i] = c;
    idx[i] = (u32)i;
  }
}

}  // namespace

void locality_order(const Runner& r, const float* X, uint64_t n, int d, uint64_t seed,
                    uint32_t* order) {
  require(d > 0 && d <= 1024, "locality_order: 1 <= d <= 1024");
  if (n == 0) return;
  DeviceGuard g(r.device);
  DBuf<float> dR(r, (size_t)kAxes * d), P(r, n * kAxes);
  DBuf<int> mm(r, 2 * kAxes);
  k_dirs<<<ceil_div(kAxes * d, 256), 256, 0, r.stream>>>(seed, kAxes * d, dR.p, mm.p);
  KNNG_LAUNCH_CHECK();
  const unsigned grid = (unsigned)std::min<u64>(ceil_div<u64>(n, 256), (u64)r.num_sms * 8);
  const unsigned pgrid = (unsigned)std::min<u64>(ceil_div<u64>(n, 8), (u64)r.num_sms * 16);
  k_project<<<pgrid, 256, 0, r.stream>>>(X, n, d, dR.p, P.p, mm.p, mm.p + kAxes);
  KNNG_LAUNCH_CHECK();
  DBuf<u32> code(r, n), tk(r, n), tv(r, n);
  k_morton<<<grid, 256, 0, r.stream>>>(P.p, n, mm.p, mm.p + kAxes, code.p, order);
  KNNG_LAUNCH_CHECK();
  bool in_tmp = false;
  radix_sort_pairs(r, code.p, order, tk.p, tv.p, n, (1u << (kAxes * kBits)) - 1, &in_tmp);
  if (in_tmp)
    KNNG_CUDA(cudaMemcpyAsync(order, tv.p, n * 4, cudaMemcpyDeviceToDevice, r.stream));
}

}  // namespace knng_b200
