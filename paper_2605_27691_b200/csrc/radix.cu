// radix.cu -- stable LSD radix sort of (u32 key, u32 value) pairs by key.
//
// Used to transpose the forward neighbor samples into reverse lists: pairs
// (target, source) are emitted in ascending source order, so a stable sort by
// target yields every reverse list already in ascending source order -- the
// order of the reference's serial transpose (nndescent.cpp:108-113).
//
// One pass per 8-bit digit (passes = bytes of the largest key):
//   k_radix_count   tile of 2048 items per CTA; each warp walks its 256 items
//                   in order (8 rounds of 32) with __match_any_sync, giving
//                   per-warp digit counts -> per-(digit, tile) totals.
//   scan            digit-major exclusive scan -> global base of (digit, tile).
//   k_radix_scatter same walk; the stable rank of an item is the tile base of
//                   its digit + the counts of earlier warps + its rank within
//                   the warp (earlier rounds, then earlier lanes).
#include "radix.hpp"

namespace knng_b200 {
namespace {

constexpr int kRT = 256;             // threads per CTA
constexpr int kRW = kRT / 32;        // warps
constexpr int kRItems = 8;           // rounds per warp
constexpr int kTile = kRT * kRItems; // 2048 items per tile
constexpr int kDigits = 256;

// n_dev (optional): the live element count, read on the device (<= n)
__device__ __forceinline__ u64 live_count(u64 n, const u64* n_dev) {
  if (n_dev == nullptr) return n;
  const u64 m = *n_dev;
  return m < n ? m : n;
}

__global__ __launch_bounds__(kRT) void k_radix_count(const u32* __restrict__ keys, u64 n_cap,
                                                     const u64* __restrict__ n_dev, int shift,
                                                     u32* __restrict__ hist, u64 ntiles) {
  __shared__ u32 s_cnt[kRW][kDigits];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const u64 n = live_count(n_cap, n_dev);
  if ((u64)blockIdx.x * kTile >= n) {  // empty tile: zero column
    for (int d = threadIdx.x; d < kDigits; d += kRT) hist[(u64)d * ntiles + blockIdx.x] = 0;
    return;
  }
  for (int d = threadIdx.x; d < kRW * kDigits; d += kRT) (&s_cnt[0][0])[d] = 0;
  __syncthreads();
  const u64 t0 = (u64)blockIdx.x * kTile + (u64)warp * 32 * kRItems;
  for (int r = 0; r < kRItems; ++r) {
    const u64 i = t0 + (u64)r * 32 + lane;
    const bool valid = i < n;
    const u32 dg = valid ? (keys[i] >> shift) & 0xffu : 0xffffffffu;
    const unsigned peers = __match_any_sync(kFull, dg);
    if (valid && (__ffs(peers) - 1) == (int)lane) s_cnt[warp][dg] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kDigits; d += kRT) {
    u32 t = 0;
    for (int w = 0; w < kRW; ++w) t += s_cnt[w][d];
    hist[(u64)d * ntiles + blockIdx.x] = t;
  }
}

__global__ __launch_bounds__(kRT) void k_radix_scatter(const u32* __restrict__ keys,
                                                       const u32* __restrict__ vals, u64 n_cap,
                                                       const u64* __restrict__ n_dev, int shift,
                                                       const u64* __restrict__ base,
                                                       u64 ntiles, u32* __restrict__ okeys,
                                                       u32* __restrict__ ovals) {
  __shared__ u32 s_cnt[kRW][kDigits];
  __shared__ u32 s_pre[kRW][kDigits];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const u64 n = live_count(n_cap, n_dev);
  if ((u64)blockIdx.x * kTile >= n) return;
  for (int d = threadIdx.x; d < kRW * kDigits; d += kRT) (&s_cnt[0][0])[d] = 0;
  __syncthreads();
  const u64 t0 = (u64)blockIdx.x * kTile + (u64)warp * 32 * kRItems;
  u32 dgs[kRItems], rank[kRItems];
  for (int r = 0; r < kRItems; ++r) {
    const u64 i = t0 + (u64)r * 32 + lane;
    const bool valid = i < n;
    const u32 dg = valid ? (keys[i] >> shift) & 0xffu : 0xffffffffu;
    const unsigned peers = __match_any_sync(kFull, dg);
    dgs[r] = dg;
    rank[r] = 0;
    if (valid) rank[r] = s_cnt[warp][dg] + __popc(peers & lanemask_lt());
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == (int)lane) s_cnt[warp][dg] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps per digit, plus the global (digit, tile) base
  for (int d = threadIdx.x; d < kDigits; d += kRT) {
    u32 run = 0;
    for (int w = 0; w < kRW; ++w) {
      s_pre[w][d] = run;
      run += s_cnt[w][d];
    }
  }
  __syncthreads();
  for (int r = 0; r < kRItems; ++r) {
    const u64 i = t0 + (u64)r * 32 + lane;
    if (i < n) {
      const u32 dg = dgs[r];
      const u64 pos = base[(u64)dg * ntiles + blockIdx.x] + s_pre[warp][dg] + rank[r];
      okeys[pos] = keys[i];
      ovals[pos] = vals[i];
    }
  }
}

}  // namespace

namespace {

void sort_impl(const Runner& r, u32* keys, u32* vals, u32* tmp_keys, u32* tmp_vals, u64 n,
               const u64* n_dev, u32 max_key, bool* result_in_tmp) {
  const u64 ntiles = ceil_div<u64>(n ? n : 1, (u64)kTile);
  int passes = 0;
  for (u64 m = max_key; m; m >>= 8) ++passes;
  if (passes == 0) passes = 1;
  u32* hist = static_cast<u32*>(r.scratch(Runner::kScrRadixHist, (u64)kDigits * ntiles * 4));
  u64* base = static_cast<u64*>(r.scratch(Runner::kScrRadixBase, ((u64)kDigits * ntiles + 1) * 8));
  u32 *ik = keys, *iv = vals, *ok = tmp_keys, *ov = tmp_vals;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    k_radix_count<<<(unsigned)ntiles, kRT, 0, r.stream>>>(ik, n, n_dev, shift, hist, ntiles);
    KNNG_LAUNCH_CHECK();
    exclusive_scan_u32(r, hist, base, (u64)kDigits * ntiles);
    k_radix_scatter<<<(unsigned)ntiles, kRT, 0, r.stream>>>(ik, iv, n, n_dev, shift, base,
                                                            ntiles, ok, ov);
    KNNG_LAUNCH_CHECK();
    std::swap(ik, ok);
    std::swap(iv, ov);
  }
  *result_in_tmp = (ik == tmp_keys);
}

}  // namespace

void radix_sort_pairs(const Runner& r, u32* keys, u32* vals, u32* tmp_keys, u32* tmp_vals,
                      uint64_t n, uint32_t max_key, bool* result_in_tmp) {
  sort_impl(r, keys, vals, tmp_keys, tmp_vals, n, nullptr, max_key, result_in_tmp);
}

void radix_sort_pairs_dev(const Runner& r, u32* keys, u32* vals, u32* tmp_keys, u32* tmp_vals,
                          uint64_t capacity, const uint64_t* n_dev, uint32_t max_key,
                          bool* result_in_tmp) {
  sort_impl(r, keys, vals, tmp_keys, tmp_vals, capacity, n_dev, max_key, result_in_tmp);
}

}  // namespace knng_b200
