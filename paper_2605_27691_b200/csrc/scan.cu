// scan.cu -- exclusive prefix sum u32 -> u64 (CSR offsets for the reverse
// neighbor lists of sample_neighbors / optimize_graph).  Three passes:
// per-block scan of 4096 items, scan of the block totals, add-back.
#include "runtime.hpp"

namespace knng_b200 {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ u64 warp_incl_scan(u64 v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 t = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total.
__device__ __forceinline__ u64 block_excl_scan(u64 v, u64* s_warp, u64& total) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const u64 incl = warp_incl_scan(v);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const u64 w = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
    const u64 wi = warp_incl_scan(w);
    s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  total = s_warp[32];
  const u64 r = incl - v + s_warp[warp];
  __syncthreads();
  return r;
}

__global__ __launch_bounds__(kScanThreads) void k_scan_tiles(const u32* __restrict__ in,
                                                             u64* __restrict__ out,
                                                             u64* __restrict__ bsum, u64 n) {
  __shared__ u64 s_warp[33];
  const u64 base = (u64)blockIdx.x * kScanTile + (u64)threadIdx.x * kScanItems;
  u64 v[kScanItems];
  u64 local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0;
    local += v[i];
  }
  u64 total;
  u64 run = block_excl_scan(local, s_warp, total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ __launch_bounds__(kScanThreads) void k_scan_bsums(u64* __restrict__ bsum, u64 nb,
                                                             u64* __restrict__ out_total) {
  __shared__ u64 s_warp[33];
  u64 carry = 0;
  for (u64 base = 0; base < nb; base += kScanThreads) {
    const u64 i = base + threadIdx.x;
    const u64 v = i < nb ? bsum[i] : 0;
    u64 total;
    const u64 ex = block_excl_scan(v, s_warp, total);
    if (i < nb) bsum[i] = ex + carry;
    carry += total;
  }
  if (threadIdx.x == 0) *out_total = carry;
}

__global__ void k_scan_add(u64* __restrict__ out, const u64* __restrict__ bsum, u64 n) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += bsum[i / kScanTile];
}

}  // namespace

void exclusive_scan_u32(const Runner& r, const uint32_t* in, uint64_t* out, uint64_t n) {
  if (n == 0) {
    KNNG_CUDA(cudaMemsetAsync(out, 0, sizeof(u64), r.stream));
    return;
  }
  const u64 nb = ceil_div<u64>(n, kScanTile);
  u64* bsum = static_cast<u64*>(r.scratch(Runner::kScrScan, nb * sizeof(u64)));
  k_scan_tiles<<<(unsigned)nb, kScanThreads, 0, r.stream>>>(in, out, bsum, n);
  KNNG_LAUNCH_CHECK();
  k_scan_bsums<<<1, kScanThreads, 0, r.stream>>>(bsum, nb, out + n);
  KNNG_LAUNCH_CHECK();
  k_scan_add<<<(unsigned)ceil_div<u64>(n, 256), 256, 0, r.stream>>>(out, bsum, n);
  KNNG_LAUNCH_CHECK();
}

}  // namespace knng_b200
