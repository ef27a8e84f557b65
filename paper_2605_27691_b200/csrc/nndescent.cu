// nndescent.cu -- B200 lock-free NN-Descent (north_star item 2).
//
// nn_descent_device builds on a Morton renumbering of the points (locality.cu)
// from 2^17 points on and maps the graph back.  Per iteration
// (nndescent.cpp:247-257):
//   k_sample_fwd   warp per point: forward new/old samples, exactly the
//                  reference's sampling stream (nndescent.cpp:80-104)
//   reverse lists  the serial transpose (:108-113): sources scattered into
//                  their targets' segments (k_rev_scatter; old entries only
//                  for targets that join, through a joins bitmap), a segment
//                  longer than the bound ranked in ascending source order
//                  (k_rev_select_rank / _long) and sampled with the
//                  reference's rng stream (:114-127) -- the picks equal the
//                  sorted path's (the stable radix sort + k_rev_select path
//                  serves sample_neighbors and KNNG_REV_SORT=1)
//   k_join         persistent CTAs over batches of points (join.cu): dedup'd
//                  new/old lists (:135-153), feature rows staged in smem with
//                  cp.async, 4x4 register micro-tiles of exact-order
//                  distances, offers (:157-197) resolved by 64-bit packed
//                  (dist,id) atomicMin cascades into hashed 4-way candidate
//                  buckets that keep the 4 smallest distinct keys -- lock-free
//                  and order-independent, so the build is deterministic;
//                  iteration 0 runs in slices with an exact bucket bound on
//                  the offer filter between them (k_bucket_bound)
//   k_apply        warp per point: the row becomes the k smallest of
//                  (row U candidates) with knn_insert semantics (:199-223),
//                  the candidates taken in ascending key order (accepted =
//                  kept), worst refreshed; only touched points once sparse.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "join.hpp"
#include "nndescent.hpp"

#include <chrono>
#include "locality.hpp"
#include "radix.hpp"
#include "refine_kernels.hpp"

namespace knng_b200 {
namespace {

constexpr u32 kNone = 0xffffffffu;

__device__ __forceinline__ u32 kmask_of(u32 k) { return k >= 32 ? kFull : ((1u << k) - 1u); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// sample_distinct(bound, B, rng) rng.hpp:66-87 with the whole warp: the rng
// stream is counter-addressed (draw m = sm64_draw(s, m)), so lane l evaluates
// draw m0 + l; first occurrences that are not yet picked are taken in draw
// order until B are picked -- the same picks, in the same order, as the serial
// loop.  s_pick[i] (warp scratch) receives pick i; returns the draws consumed
// (the serial loop's rng position afterwards).  Needs B <= 32 and B < bound.
__device__ u32 warp_sample_distinct(u64 s, u64 m0, u64 bound, u32 B, u32* s_pick) {
  const unsigned lane = lane_id();
  u32 got = 0;
  u64 m = m0;
  while (true) {
    const u32 x = (u32)__umul64hi(sm64_draw(s, m + lane), bound);
    const unsigned grp = __match_any_sync(kFull, x);
    bool fresh = (__ffs(grp) - 1) == (int)lane;  // first occurrence in this batch
    for (u32 j = 0; j < got; ++j) fresh = fresh && s_pick[j] != x;
    const unsigned fb = __ballot_sync(kFull, fresh);
    const u32 before = __popc(fb & lanemask_lt());
    const bool take = fresh && got + before < B;
    if (take) s_pick[got + before] = x;
    const unsigned last = __ballot_sync(kFull, take && got + before == B - 1);
    __syncwarp();
    if (last) return (u32)(m - m0) + (u32)__ffs(last);
    got += __popc(fb);
    m += 32;
  }
}

// ---------------------------------------------------------------------------
// init_random_graph nndescent.cpp:29-62 -- warp per row
// ---------------------------------------------------------------------------
constexpr u32 kInitDims = 64;  // dims per staging round (d % 4 == 0 path)

constexpr int kInitThreads = 128;  // 4 warps: 4 x 8.7 KB staging fits static smem

template <bool kCos>
__global__ __launch_bounds__(kInitThreads) void k_init(const float* __restrict__ X, u64 n, int d, u32 k,
                                              u64 seed, u64* __restrict__ keys,
                                              u32* __restrict__ flags,
                                              float* __restrict__ worst,
                                              const float* __restrict__ nrm) {
  // per warp: 32 staged rows x (kInitDims + 4) floats | 32 picks
  __shared__ __align__(16) float s_rows[kInitThreads / 32][32 * (kInitDims + 4)];
  __shared__ u32 s_pick[kInitThreads / 32][32];
  const unsigned lane = lane_id(), w = threadIdx.x >> 5;
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  const bool vec = (d % 4) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  constexpr u32 kStride = kInitDims + 4;  // stride/4 odd: conflict-free LDS.128 by row
  for (u64 r = (((u64)blockIdx.x * blockDim.x) >> 5) + w; r < n; r += warps) {
    // k distinct non-self ids: sample_distinct(n - 1, k) in draw order, then
    // the reference's skip-self shift (x >= r -> x + 1)
    warp_sample_distinct(mix_seed(seed, r), 0, n - 1, k, s_pick[w]);
    u32 my_id = kNone;
    if (lane < k) {
      my_id = s_pick[w][lane];
      if (my_id >= r) ++my_id;
    }
    const float* xr = X + r * (u64)d;
    float acc = 0.0f;
    if (vec) {
      // stage the k neighbor rows chunk by chunk (coalesced cp.async, one
      // 16-byte piece per lane, 2 rows per warp instruction at 64 dims) and
      // sum each lane's own row in the reference's order
      float* st = s_rows[w];
      for (int c0 = 0; c0 < d; c0 += kInitDims) {
        const int cl = min((int)kInitDims, d - c0);
        const u32 pieces = (u32)cl / 4;          // 16-byte pieces per row
        for (u32 e0 = 0; e0 < k * pieces; e0 += 32) {  // warp-uniform trips
          const u32 e = e0 + lane;
          const u32 j = e / pieces, q = e - j * pieces;
          const u32 idj = __shfl_sync(kFull, my_id, j < 32 ? j : 0);
          if (e < k * pieces) cp_async16(st + j * kStride + q * 4, X + (u64)idj * d + c0 + q * 4);
        }
        cp_async_wait_all();
        __syncwarp();
        if (lane < k) {
          const float* my = st + lane * kStride;
          for (int i = 0; i < cl; i += 4)
            acc = m_step4<kCos>(acc, *reinterpret_cast<const float4*>(xr + c0 + i),
                           *reinterpret_cast<const float4*>(my + i));
        }
        __syncwarp();
      }
    } else if (lane < k) {
      const float* xo = X + (u64)my_id * d;
      for (int i = 0; i < d; ++i) acc = m_step<kCos>(acc, xr[i], xo[i]);
    }
    u64 key = kEmptyKey;
    if (lane < k)
      key = pack_key(m_finish<kCos>(acc, kCos ? nrm[r] : 0.0f, kCos ? nrm[my_id] : 0.0f), my_id);
    key = warp_sort32(key);
    if (lane < k) keys[r * k + lane] = key;
    const u64 last = __shfl_sync(kFull, key, k - 1);
    if (lane == 0) {
      flags[r] = kmask_of(k);
      worst[r] = key_dist(last);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// sample_neighbors, forward half (nndescent.cpp:80-104) -- warp per point
// ---------------------------------------------------------------------------
__global__ __launch_bounds__(256) void k_sample_fwd(const u64* __restrict__ keys,
                                                    u32* __restrict__ flags, u64 n, u32 k,
                                                    u32 B, u64 iter_seed, u32* __restrict__ nf,
                                                    u32* __restrict__ nfn, u32* __restrict__ of,
                                                    u32* __restrict__ ofn,
                                                    u32* __restrict__ cnt_new,
                                                    u32* __restrict__ cnt_old, bool count_old) {
  __shared__ u32 s_scr[8][64];  // per warp: picks | rank -> lane
  const unsigned lane = lane_id();
  const u32 km = kmask_of(k);
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 p = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); p < n; p += warps) {
    const u32 id = lane < k ? key_id(keys[p * k + lane]) : kNone;
    const u32 fm = flags[p] & km;
    const bool isnew = (fm >> lane) & 1u;
    const u32 np = __popc(fm);
    const unsigned lt = lanemask_lt();
    if (lane < k && !isnew) {
      of[p * k + __popc(~fm & km & lt)] = id;
      if (count_old) atomicAdd(&cnt_old[id], 1u);
    }
    if (np <= B) {
      if (isnew) {
        nf[p * B + __popc(fm & lt)] = id;
        atomicAdd(&cnt_new[id], 1u);
      }
      if (lane == 0) {
        nfn[p] = np;
        ofn[p] = k - np;
        flags[p] = 0;
      }
    } else {
      // sample_distinct(np, B, Rng(mix_seed(iter_seed, p))) rng.hpp:66-87:
      // pick i = the rank (among the new entries) of the i-th sampled one
      u32* sp = s_scr[threadIdx.x >> 5];
      u32* sr = sp + 32;
      if (isnew) sr[__popc(fm & lt)] = lane;  // rank -> lane
      warp_sample_distinct(mix_seed(iter_seed, p), 0, np, B, sp);
      u32 src = 0;
      if (lane < B) src = sr[sp[lane]];
      const u32 idv = __shfl_sync(kFull, id, src);
      if (lane < B) {
        nf[p * B + lane] = idv;
        atomicAdd(&cnt_new[idv], 1u);
      }
      const u32 cleared = __reduce_or_sync(kFull, lane < B ? (1u << src) : 0u);
      if (lane == 0) {
        nfn[p] = B;
        ofn[p] = k - np;
        flags[p] = fm & ~cleared;
      }
      __syncwarp();
    }
  }
}

// Reverse lists: (target, source) pairs emitted compacted in ascending
// source order (prefix offsets per source), so a stable radix sort by target
// lays out every reverse list in ascending source order -- the order of the
// reference's serial transpose (nndescent.cpp:108-113).
//
// Inside nn_descent the old pairs are pruned to targets that have a new
// entry (a new forward sample or a new reverse one): only those points join
// (new x new, new x old -- nndescent.cpp:157-171), and each target's reverse
// sample uses its own rng, so the lists of the joining points are unchanged
// while late iterations sort a small fraction of the n*k old entries.
__device__ __forceinline__ bool joins(u32 t, const u32* __restrict__ nfn,
                                      const u32* __restrict__ cnt_new) {
  return nfn[t] > 0 || cnt_new[t] > 0;
}
// the same predicate as a bitmap (n bits: 1.25 MB at 10M points, L2-resident)
// -- the prune's random lookups hit it instead of two n-entry arrays
__device__ __forceinline__ bool joins_bit(u32 t, const u32* __restrict__ bits) {
  return (__ldg(bits + (t >> 5)) >> (t & 31)) & 1u;
}
// warp per 32 points
__global__ __launch_bounds__(256) void k_join_bits(u64 n, const u32* __restrict__ nfn,
                                                   const u32* __restrict__ cnt_new,
                                                   u32* __restrict__ bits) {
  const unsigned lane = lane_id();
  const u64 words = (n + 31) >> 5;
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 w = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); w < words; w += warps) {
    const u64 t = w * 32 + lane;
    const unsigned b = __ballot_sync(kFull, t < n && joins((u32)t, nfn, cnt_new));
    if (lane == 0) bits[w] = b;
  }
}

// warp per source: how many of its old entries survive the prune; counts
// the surviving reverse entries per target
__global__ __launch_bounds__(256) void k_old_count(u64 n, u32 k, const u32* __restrict__ of,
                                                   const u32* __restrict__ ofn,
                                                   const u32* __restrict__ jbits,
                                                   u32* __restrict__ src_cnt,
                                                   u32* __restrict__ cnt_old) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 p = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); p < n; p += warps) {
    bool keep = false;
    if (lane < ofn[p]) {
      const u32 t = of[p * k + lane];
      keep = joins_bit(t, jbits);
      if (keep) atomicAdd(&cnt_old[t], 1u);
    }
    const unsigned kb = __ballot_sync(kFull, keep);
    if (lane == 0) src_cnt[p] = __popc(kb);
  }
}

// warp per source: write its (kept) entries at src_off[p] + rank
__global__ __launch_bounds__(256) void k_emit_pairs(u64 n, u32 width, const u32* __restrict__ fwd,
                                                    const u32* __restrict__ cnt,
                                                    const u64* __restrict__ src_off,
                                                    const u32* __restrict__ jbits,
                                                    u32* __restrict__ keys,
                                                    u32* __restrict__ vals) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 p = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); p < n; p += warps) {
    bool keep = false;
    u32 t = 0;
    if (lane < cnt[p]) {
      t = fwd[p * width + lane];
      keep = jbits == nullptr || joins_bit(t, jbits);
    }
    const unsigned kb = __ballot_sync(kFull, keep);
    if (keep) {
      const u64 pos = src_off[p] + __popc(kb & lanemask_lt());
      keys[pos] = t;
      vals[pos] = (u32)p;
    }
  }
}

// Reverse sampling nndescent.cpp:114-127: the segment of v, ranked in
// ascending source order (= the serial transpose order), sampled with
// Rng(mix_seed(iter_seed, 2^63|v)) shared by new_rev then old_rev.
__global__ __launch_bounds__(256) void k_rev_select(u64 n, u32 B, u64 iter_seed,
                                                    const u64* __restrict__ off_new,
                                                    const u32* __restrict__ buf_new,
                                                    const u64* __restrict__ off_old,
                                                    const u32* __restrict__ buf_old,
                                                    u32* __restrict__ nr, u32* __restrict__ nrn,
                                                    u32* __restrict__ orv,
                                                    u32* __restrict__ orn) {
  __shared__ u32 s_scr[8][32];  // per warp: picks
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 v = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); v < n; v += warps) {
    const u64 rs = mix_seed(iter_seed, 0x8000000000000000ull | v);
    u64 drawn = 0;  // rng position, shared by new_rev then old_rev
    u32* sp = s_scr[threadIdx.x >> 5];
    for (int which = 0; which < 2; ++which) {
      const u64* off = which ? off_old : off_new;
      const u32* buf = which ? buf_old : buf_new;
      u32* out = (which ? orv : nr) + v * B;
      u32* outn = which ? orn : nrn;
      const u64 lo = off[v];
      const u32 len = (u32)(off[v + 1] - lo);
      const u32* seg = buf + lo;
      if (len <= B) {  // already in ascending source order
        if (lane < len) out[lane] = seg[lane];
        if (lane == 0) outn[v] = len;
        continue;
      }
      // sample_distinct(len, B, rng) rng.hpp:66-87 over the sorted segment
      drawn += warp_sample_distinct(rs, drawn, len, B, sp);
      if (lane < B) out[lane] = seg[sp[lane]];
      if (lane == 0) outn[v] = B;
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// Reverse lists inside nn_descent without the sort.  Only the SET of a
// reverse list matters to the join when it is not sampled (the join lists are
// deduplicated unions, and every pair they produce is offered to
// order-independent buckets), so sources are scattered straight into their
// targets' segments with per-target atomic cursors.  A segment longer than
// the bound is sampled by RANK in ascending source order (the reference's
// serial transpose order, nndescent.cpp:108-127): k_rev_select_rank ranks it
// (warp bitonic sort <= 32, rank counting in smem <= kRankSmem, rank counting
// in global memory beyond), so the picks equal the sorted path's.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rev_put(u32 t, bool on, u32 p, const u64* __restrict__ off,
                                        u32* __restrict__ cur, u32* __restrict__ buf) {
  // lanes of one warp often share a hub target: one atomic per distinct target
  const unsigned act = __ballot_sync(kFull, on);
  if (!on) return;
  const unsigned grp = __match_any_sync(act, t);
  const int leader = __ffs(grp) - 1;
  u32 base = 0;
  if ((int)lane_id() == leader) base = atomicAdd(&cur[t], (u32)__popc(grp));
  base = __shfl_sync(grp, base, leader);
  buf[off[t] + base + __popc(grp & lanemask_lt())] = p;
}

// lane = source (32 consecutive sources per warp), one list slot per round
__global__ __launch_bounds__(256) void k_rev_scatter(u64 n, u32 k, u32 B, const u32* __restrict__ nf,
                                                     const u32* __restrict__ nfn,
                                                     const u32* __restrict__ of,
                                                     const u32* __restrict__ ofn,
                                                     const u32* __restrict__ jbits,
                                                     const u64* __restrict__ off_new,
                                                     const u64* __restrict__ off_old,
                                                     u32* __restrict__ cur_new,
                                                     u32* __restrict__ cur_old,
                                                     u32* __restrict__ buf_new,
                                                     u32* __restrict__ buf_old) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 p0 = ((((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5)) * 32; p0 < n;
       p0 += warps * 32) {
    const u64 p = p0 + lane;
    const bool live = p < n;
    const u32 cn = live ? nfn[p] : 0, co = live ? ofn[p] : 0;
    const u32 mx = __reduce_max_sync(kFull, cn > co ? cn : co);
    for (u32 j = 0; j < mx; ++j) {
      const bool on_n = j < cn;
      const u32 tn = on_n ? nf[p * B + j] : 0;
      rev_put(tn, on_n, (u32)p, off_new, cur_new, buf_new);
      bool on_o = j < co;
      const u32 to = on_o ? of[p * k + j] : 0;
      on_o = on_o && joins_bit(to, jbits);
      rev_put(to, on_o, (u32)p, off_old, cur_old, buf_old);
    }
  }
}

constexpr u32 kRankSmem = 512;  // per-warp smem rank sort capacity

// Ascending bitonic sort of 32 R keys held R per lane (element j*32 + lane in
// v[j]); strides >= 32 compare registers of one lane, shorter ones shuffle.
template <int R>
__device__ __forceinline__ void warp_sort_regs(u32 (&v)[R], unsigned lane) {
#pragma unroll
  for (unsigned size = 2; size <= 32u * R; size <<= 1)
#pragma unroll
    for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const unsigned js = stride >> 5;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (j & js) continue;
          const unsigned e = (unsigned)j * 32 + lane;
          const bool up = (e & size) == 0;
          const u32 a = v[j], b = v[j ^ js];
          if ((a > b) == up) {
            v[j] = b;
            v[j ^ js] = a;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const unsigned e = (unsigned)j * 32 + lane;
          const u32 o = __shfl_xor_sync(kFull, v[j], stride);
          const bool keep_min = ((lane & stride) == 0) == ((e & size) == 0);
          v[j] = keep_min ? min(v[j], o) : max(v[j], o);
        }
      }
    }
}
// pick the element of rank r (all lanes take part; r < 32 R)
template <int R>
__device__ __forceinline__ u32 warp_pick_regs(const u32 (&v)[R], u32 r) {
  u32 out = 0;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const u32 x = __shfl_sync(kFull, v[j], r & 31);
    if ((r >> 5) == (u32)j) out = x;
  }
  return out;
}

__global__ __launch_bounds__(256) void k_rev_select_rank(u64 n, u32 B, u64 iter_seed,
                                                         const u64* __restrict__ off_new,
                                                         const u32* __restrict__ buf_new,
                                                         const u64* __restrict__ off_old,
                                                         const u32* __restrict__ buf_old,
                                                         u32* __restrict__ nr,
                                                         u32* __restrict__ nrn,
                                                         u32* __restrict__ orv,
                                                         u32* __restrict__ orn,
                                                         u32* __restrict__ long_cnt,
                                                         u32* __restrict__ long_rec) {
  __shared__ u32 s_pick[8][32];
  __shared__ u32 s_seg[8][kRankSmem];
  const unsigned lane = lane_id();
  const int w = threadIdx.x >> 5;
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 v = (((u64)blockIdx.x * blockDim.x) >> 5) + w; v < n; v += warps) {
    const u64 rs = mix_seed(iter_seed, 0x8000000000000000ull | v);
    u64 drawn = 0;  // rng position, shared by new_rev then old_rev
    u32* sp = s_pick[w];
    for (int which = 0; which < 2; ++which) {
      const u64* off = which ? off_old : off_new;
      const u32* buf = which ? buf_old : buf_new;
      u32* out = (which ? orv : nr) + v * B;
      u32* outn = which ? orn : nrn;
      const u64 lo = off[v];
      const u32 len = (u32)(off[v + 1] - lo);
      const u32* seg = buf + lo;
      if (len <= B) {  // taken whole: its order is irrelevant to the join
        if (lane < len) out[lane] = seg[lane];
        if (lane == 0) outn[v] = len;
        continue;
      }
      drawn += warp_sample_distinct(rs, drawn, len, B, sp);
      if (len <= 32) {
        // ascending sort across the warp, then pick ranks
        u32 v[1] = {lane < len ? seg[lane] : 0xffffffffu};
        warp_sort_regs<1>(v, lane);
        const u32 pick = warp_pick_regs<1>(v, lane < B ? sp[lane] : 0);
        if (lane < B) out[lane] = pick;
      } else if (len <= 64) {
        u32 v[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) v[j] = j * 32 + lane < len ? seg[j * 32 + lane] : 0xffffffffu;
        warp_sort_regs<2>(v, lane);
        const u32 pick = warp_pick_regs<2>(v, lane < B ? sp[lane] : 0);
        if (lane < B) out[lane] = pick;
      } else if (len <= 128) {
        u32 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = j * 32 + lane < len ? seg[j * 32 + lane] : 0xffffffffu;
        warp_sort_regs<4>(v, lane);
        const u32 pick = warp_pick_regs<4>(v, lane < B ? sp[lane] : 0);
        if (lane < B) out[lane] = pick;
      } else if (len <= kRankSmem) {
        // bitonic sort of the segment (padded to a power of two) in smem
        u32* ss = s_seg[w];
        u32 m = 64;
        while (m < len) m <<= 1;
        for (u32 i = lane; i < m; i += 32) ss[i] = i < len ? seg[i] : 0xffffffffu;
        __syncwarp();
        for (u32 size = 2; size <= m; size <<= 1)
          for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
            for (u32 i = lane; i < m; i += 32) {
              const u32 partner = i ^ stride;
              if (partner > i) {
                const u32 a0 = ss[i], a1 = ss[partner];
                const bool up = (i & size) == 0;
                if ((a0 > a1) == up) {
                  ss[i] = a1;
                  ss[partner] = a0;
                }
              }
            }
            __syncwarp();
          }
        if (lane < B) out[lane] = ss[sp[lane]];
        __syncwarp();
      } else {
        // long (hub) segment: deferred to k_rev_select_long (radix select)
        u32 slot = 0;
        if (lane == 0) slot = atomicAdd(long_cnt, 1u);
        slot = __shfl_sync(kFull, slot, 0);
        u32* rec = long_rec + (u64)slot * (2 + 32);
        if (lane == 0) {
          rec[0] = (u32)v;
          rec[1] = (u32)which;
        }
        if (lane < B) rec[2 + lane] = sp[lane];
      }
      if (lane == 0) outn[v] = B;
      __syncwarp();
    }
  }
}

// Hub segments (longer than kRankSmem): one CTA each selects the elements of
// the B sampled ranks by radix select -- 8-bit digits from the top bits that
// vary; after the last pass each rank's prefix IS its element (sources in a
// segment are distinct).  O(len) per pass:
//   * ranks whose prefixes agree so far form a group with one histogram; the
//     element -> group map of the next pass is a (group, digit) table, and a
//     segment of <= kLongCache entries is kept in shared memory with its
//     group byte, so an element costs a few shared-memory operations per
//     pass (longer ones re-read HBM and match the <= B group prefixes);
//   * each rank finds its bin by a warp scan of its group's 256 bins.
constexpr u32 kLongCache = 8192;
constexpr size_t kLongSmem = 32 * 256 * 4 + kLongCache * 4 + kLongCache + 32 * 256;

__global__ __launch_bounds__(256) void k_rev_select_long(u64 n_src, u32 B,
                                                         const u64* __restrict__ off_new,
                                                         const u32* __restrict__ buf_new,
                                                         const u64* __restrict__ off_old,
                                                         const u32* __restrict__ buf_old,
                                                         u32* __restrict__ nr,
                                                         u32* __restrict__ orv,
                                                         const u32* __restrict__ long_cnt,
                                                         const u32* __restrict__ long_rec) {
  extern __shared__ __align__(16) unsigned char smem_long[];
  u32* hist = reinterpret_cast<u32*>(smem_long);              // [32][256]
  u32* xs = hist + 32 * 256;                                   // [kLongCache]
  unsigned char* grp = reinterpret_cast<unsigned char*>(xs + kLongCache);  // [kLongCache]
  unsigned char* child = grp + kLongCache;                     // [32][256]
  __shared__ u32 prefix[32], remain[32], gid[32], gpre[32], bin_of[32];
  __shared__ int G;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const u32 nrec = *long_cnt;
  int top = 0;
  while (top < 32 && (n_src >> top) > 0) ++top;
  const int first_shift = top > 8 ? ((top - 8 + 7) / 8) * 8 : 0;
  for (u32 e = blockIdx.x; e < nrec; e += gridDim.x) {
    const u32* rec = long_rec + (u64)e * (2 + 32);
    const u64 v = rec[0];
    const int which = (int)rec[1];
    const u64* off = which ? off_old : off_new;
    const u32* seg = (which ? buf_old : buf_new) + off[v];
    const u32 len = (u32)(off[v + 1] - off[v]);
    const bool cached = len <= kLongCache;
    if (cached)
      for (u32 i = threadIdx.x; i < len; i += blockDim.x) {
        xs[i] = seg[i];
        grp[i] = 0;
      }
    if (threadIdx.x < B) {
      prefix[threadIdx.x] = 0;
      remain[threadIdx.x] = rec[2 + threadIdx.x];
      gid[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) {
      G = 1;
      gpre[0] = 0;
    }
    __syncthreads();
    int prev_shift = -1;  // the digit that indexes `child` (previous pass)
    for (int shift = first_shift; shift >= 0; shift -= 8) {
      const int g_n = G;
      for (u32 i = threadIdx.x; i < (u32)g_n * 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const u32 hi_mask = shift >= 24 ? 0u : (0xffffffffu << (shift + 8));
      for (u32 i = threadIdx.x; i < len; i += blockDim.x) {
        u32 x, g;
        if (cached) {
          // the element's group moves by the previous pass's (group, digit)
          x = xs[i];
          g = grp[i];
          if (prev_shift >= 0 && g != 0xff) {
            g = child[g * 256 + ((x >> prev_shift) & 255)];
            grp[i] = (unsigned char)g;
          }
        } else {
          x = seg[i];
          g = 0xff;
          for (int b = 0; b < g_n; ++b)
            if ((x & hi_mask) == (gpre[b] & hi_mask)) {
              g = b;
              break;
            }
        }
        if (g != 0xff) atomicAdd(&hist[g * 256 + ((x >> shift) & 255)], 1u);
      }
      __syncthreads();
      // rank r (warp r % 8): lane l scans bins 8l..8l+7 of the rank's group
      for (u32 r = warp; r < B; r += blockDim.x >> 5) {
        const u32* h = hist + gid[r] * 256 + lane * 8;
        u32 c[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          c[j] = h[j];
          tot += c[j];
        }
        u32 incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 t = __shfl_up_sync(kFull, incl, o);
          if ((int)lane >= o) incl += t;
        }
        const u32 excl = incl - tot, want = remain[r];
        // the lane whose range holds rank `want`
        const unsigned hit = __ballot_sync(kFull, excl <= want && want < incl);
        if ((int)lane == __ffs(hit) - 1) {
          u32 acc = excl, bin = lane * 8;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (acc + c[j] > want) break;
            acc += c[j];
            ++bin;
          }
          bin_of[r] = bin;
          prefix[r] |= bin << shift;
          remain[r] = want - acc;
        }
      }
      __syncthreads();
      if (shift == 0) break;
      // next groups (warp 0, lane = rank): ranks with the same (group, bin)
      // share one; `child` maps an element's (group, digit) to it
      if (warp == 0) {
        const bool live = lane < B;
        const u32 key = live ? gid[lane] * 256 + bin_of[lane] : 0xffffffffu;
        const unsigned same = __match_any_sync(kFull, key);
        const int leader = __ffs(same) - 1;
        const unsigned leaders = __ballot_sync(kFull, live && leader == (int)lane);
        const u32 ng = __popc(leaders & ((1u << leader) - 1u));
        // clear this pass's table rows, then the leaders write theirs
        for (u32 i = lane; i < (u32)g_n * 64; i += 32)
          reinterpret_cast<u32*>(child)[i] = 0xffffffffu;
        __syncwarp();
        if (live && leader == (int)lane) {
          child[key] = (unsigned char)ng;
          gpre[ng] = prefix[lane];
        }
        if (live) gid[lane] = ng;
        if (lane == 0) G = __popc(leaders);
      }
      prev_shift = shift;
      __syncthreads();
    }
    if (threadIdx.x < B) (which ? orv : nr)[v * B + threadIdx.x] = prefix[threadIdx.x];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// apply_candidates nndescent.cpp:199-223 -- warp per point
// ---------------------------------------------------------------------------
// The reference inserts a point's buffered candidates with knn_insert in
// buffer order (core.cpp:99-112: duplicates of row ids and non-improvements
// rejected, the rest shifted in).  The row it ends with is the k smallest of
// (row U candidates) whatever the order; the count of accepted inserts
// depends on the order (a candidate accepted and later pushed out counts).
// The buffer order is the join threads' arrival order there; here the
// candidates are applied in ascending key order -- one valid buffer order --
// for which "accepted" = "kept": the count is the number of new entries the
// row ends with.
//
// Many candidates (early iterations: ~50 per point): two 32-key bitonic
// sorts, a bitonic merge keeping the 32 smallest candidates and one more
// merge against the row (with the new-entry flags), ~400 instructions per
// point.  Few candidates: knn_insert one at a time (~40 each).
//
// With X set the buckets hold LOWER BOUNDS of the exact distances (the
// tensor-core join, join_tc.cu): every candidate whose bound beats the row's
// current worst gets its exact-order distance recomputed here (core.hpp:23-30),
// so the inserted keys -- and the decisions of knn_insert -- are exact.
__device__ __forceinline__ u64 shfl64(u64 v, int src) { return __shfl_sync(kFull, v, src); }
__device__ __forceinline__ u64 shfl_xor64(u64 v, int m) { return __shfl_xor_sync(kFull, v, m); }

// ascending bitonic sort of one key per lane
__device__ __forceinline__ u64 warp_sort_asc(u64 v, unsigned lane) {
#pragma unroll
  for (unsigned size = 2; size <= 32; size <<= 1)
#pragma unroll
    for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
      const u64 o = shfl_xor64(v, stride);
      const bool keep_min = ((lane & stride) == 0) == ((lane & size) == 0);
      v = keep_min ? (o < v ? o : v) : (o > v ? o : v);
    }
  return v;
}
// a bitonic sequence of one key per lane -> ascending
__device__ __forceinline__ u64 warp_merge_asc(u64 v, unsigned lane) {
#pragma unroll
  for (unsigned stride = 16; stride > 0; stride >>= 1) {
    const u64 o = shfl_xor64(v, stride);
    v = (lane & stride) == 0 ? (o < v ? o : v) : (o > v ? o : v);
  }
  return v;
}

constexpr u32 kApplySerialMax = 8;  // candidates up to which knn_insert runs one by one

// Only points an offer reached (touched, set by k_offer) can hold candidates:
// a warp takes 32 points, reads their touched bytes at once and visits the
// set ones.  Used once offers get sparse (the iteration before queued fewer
// than 4 per point); with touched null every point is visited (k_offer then
// writes no flags -- early iterations reach almost every point anyway).
__global__ __launch_bounds__(256) void k_apply(u64 n, u32 k, u32 S, u64* __restrict__ keys,
                                               u32* __restrict__ flags,
                                               float* __restrict__ worst,
                                               u64* __restrict__ slots,
                                               u64* __restrict__ counters,
                                               const float* __restrict__ X, int d,
                                               uint8_t* __restrict__ touched) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  u64 acc_total = 0;
  for (u64 p0 = ((((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5)) * 32; p0 < n;
       p0 += warps * 32) {
   const bool mine = p0 + lane < n && (!touched || touched[p0 + lane]);
   if (mine && touched) touched[p0 + lane] = 0;
   unsigned todo = __ballot_sync(kFull, mine);
   while (todo) {
    const u64 p = p0 + (__ffs(todo) - 1);
    todo &= todo - 1;
    u64* sl = slots + p * S;
    // the buffer (S <= 64: two keys per lane), reset as it is read
    u64 c[2];
    bool any = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const u32 si = h * 32 + lane;
      c[h] = si < S ? sl[si] : kEmptyKey;
      const bool filled = c[h] != kEmptyKey;
      if (filled) sl[si] = kEmptyKey;  // CandidateBuffer::reset
      any |= __any_sync(kFull, filled);
    }
    if (!any) continue;
    u64 rk = lane < k ? keys[p * k + lane] : kEmptyKey;
    u32 fl = lane < k ? (flags[p] >> lane) & 1u : 0u;
    const u64 last = shfl64(rk, k - 1);
    u32 nv = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (X && c[h] < last) {
        const u32 v = key_id(c[h]);
        c[h] = pack_key(l2_exact(X + p * (u64)d, X + (u64)v * d, d), v);
      }
      if (c[h] >= last) c[h] = kEmptyKey;  // non-improvement (filled or not)
      // duplicate of a row id: its key equals that row entry's (same exact
      // distance), found by a binary search of the sorted row
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const u64 x = shfl64(rk, lo + step - 1);
        if (x < c[h]) lo += step;
      }
      const u64 at = shfl64(rk, lo & 31);
      if (c[h] != kEmptyKey && lo < (int)k && at == c[h]) c[h] = kEmptyKey;
      nv += __popc(__ballot_sync(kFull, c[h] != kEmptyKey));
    }
    if (nv == 0) continue;
    u32 kept = 0;
    if (nv <= kApplySerialMax) {
      // knn_insert one by one (the kept row is order-independent)
      u32 from_c = 0;
      u64 lst = last;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        unsigned mask = __ballot_sync(kFull, c[h] != kEmptyKey);
        while (mask) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1;
          const u64 cc = shfl64(c[h], src);
          if (cc >= lst) continue;
          const u32 pos = __popc(__ballot_sync(kFull, lane < k && rk < cc));
          const u64 up = __shfl_up_sync(kFull, rk, 1);
          const u32 upf = __shfl_up_sync(kFull, fl | (from_c << 1), 1);
          if (lane > pos && lane < k) {
            rk = up;
            fl = upf & 1u;
            from_c = upf >> 1;
          }
          if (lane == pos) {
            rk = cc;
            fl = 1;
            from_c = 1;
          }
          lst = shfl64(rk, k - 1);
        }
      }
      kept = __popc(__ballot_sync(kFull, lane < k && from_c));
    } else {
      // the 32 smallest candidates, ascending: sort both halves, then the
      // elementwise min of one and the other reversed is bitonic
      const u64 a = warp_sort_asc(c[0], lane);
      const u64 b = warp_sort_asc(c[1], lane);
      const u64 br = shfl64(b, 31 - lane);
      const u64 cs = warp_merge_asc(a < br ? a : br, lane);
      // the k smallest of row U candidates (rows pad lanes >= k with empty
      // keys), new-entry flags following their keys
      const u64 cr = shfl64(cs, 31 - lane);
      const bool take_c = cr < rk;
      u64 v = take_c ? cr : rk;
      u32 f = take_c ? 3u : fl;  // bit 1: from the candidates
#pragma unroll
      for (unsigned stride = 16; stride > 0; stride >>= 1) {
        const u64 o = shfl_xor64(v, stride);
        const u32 of = __shfl_xor_sync(kFull, f, stride);
        const bool lower = (lane & stride) == 0;
        if (lower ? (o < v) : (o > v)) {
          v = o;
          f = of;
        }
      }
      rk = v;
      fl = f & 1u;
      kept = __popc(__ballot_sync(kFull, lane < k && (f & 2u)));
    }
    if (kept) {
      if (lane < k) keys[p * k + lane] = rk;
      const unsigned fmask = __ballot_sync(kFull, fl && lane < k);
      const u64 nl = shfl64(rk, k - 1);
      if (lane == 0) {
        flags[p] = fmask;
        worst[p] = key_dist(nl);
      }
      acc_total += kept;
    }
   }
  }
  if (lane == 0 && acc_total)
    atomicAdd(reinterpret_cast<unsigned long long*>(counters + kCntAccepted), acc_total);
}

// Filter refresh between join slices of a dense iteration: worst[p] =
// min(worst[p], just above the k-th smallest key in p's buckets).  Bucket
// keys only decrease (a bucket keeps its W smallest distinct keys), and every
// bucket key ends up in row U buckets -- a key equal to a row entry IS that
// entry -- so at the end row U buckets still holds >= k keys at or below the
// bound: a later offer above it can neither enter the final top-k nor, being
// larger than every key it could displace that matters, change which keys
// below it the buckets keep.  k_apply's result is unchanged; the offers
// shrink.  (Exact keys only: not with the tensor-core join's lower bounds.)
__global__ __launch_bounds__(256) void k_bucket_bound(u64 n, u32 k, u32 S,
                                                      float* __restrict__ worst,
                                                      const u64* __restrict__ slots) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 p = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); p < n; p += warps) {
    const u64* sl = slots + p * S;
    const u64 c0 = lane < S ? sl[lane] : kEmptyKey;
    const u64 c1 = 32 + lane < S ? sl[32 + lane] : kEmptyKey;
    const unsigned full = __ballot_sync(kFull, c0 != kEmptyKey);
    const unsigned full1 = __ballot_sync(kFull, c1 != kEmptyKey);
    if ((u32)(__popc(full) + __popc(full1)) < k) continue;  // fewer than k keys: no bound
    const u64 a = warp_sort_asc(c0, lane);
    const u64 b = warp_sort_asc(c1, lane);
    const u64 br = shfl64(b, 31 - lane);
    const u64 cs = warp_merge_asc(a < br ? a : br, lane);
    const u64 kth = shfl64(cs, k - 1);
    if (lane == 0) {
      const float w = nextafterf(key_dist(kth), INFINITY);
      if (w < worst[p]) worst[p] = w;
    }
  }
}

// More than 64 buffered slots per point (candidate_capacity > 64): the same
// semantics, knn_insert one candidate at a time over 32-slot chunks.
__global__ __launch_bounds__(256) void k_apply_wide(u64 n, u32 k, u32 S, u64* __restrict__ keys,
                                                    u32* __restrict__ flags,
                                                    float* __restrict__ worst,
                                                    u64* __restrict__ slots,
                                                    u64* __restrict__ counters,
                                                    const float* __restrict__ X, int d) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  u64 acc_total = 0;
  for (u64 p = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); p < n; p += warps) {
    u64* sl = slots + p * S;
    u64 rk = kEmptyKey, last = 0;
    u32 fl = 0, from_c = 0;
    bool loaded = false;
    for (u32 c0 = 0; c0 < S; c0 += 32) {
      const u32 si = c0 + lane;
      u64 cc = si < S ? sl[si] : kEmptyKey;
      const bool filled = cc != kEmptyKey;
      if (filled) sl[si] = kEmptyKey;  // CandidateBuffer::reset
      if (!__any_sync(kFull, filled)) continue;
      if (!loaded) {
        loaded = true;
        rk = lane < k ? keys[p * k + lane] : kEmptyKey;
        fl = lane < k ? (flags[p] >> lane) & 1u : 0u;
        last = shfl64(rk, k - 1);
      }
      if (X && filled && cc < last) {
        const u32 v = key_id(cc);
        cc = pack_key(l2_exact(X + p * (u64)d, X + (u64)v * d, d), v);
      }
      unsigned mask = __ballot_sync(kFull, filled && cc < last);
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const u64 c = shfl64(cc, src);
        if (c >= last) continue;
        if (__ballot_sync(kFull, lane < k && key_id(rk) == key_id(c))) continue;
        const u32 pos = __popc(__ballot_sync(kFull, lane < k && rk < c));
        const u64 up = __shfl_up_sync(kFull, rk, 1);
        const u32 upf = __shfl_up_sync(kFull, fl | (from_c << 1), 1);
        if (lane > pos && lane < k) {
          rk = up;
          fl = upf & 1u;
          from_c = upf >> 1;
        }
        if (lane == pos) {
          rk = c;
          fl = 1;
          from_c = 1;
        }
        last = shfl64(rk, k - 1);
      }
    }
    const u32 kept = __popc(__ballot_sync(kFull, lane < k && from_c));
    if (kept) {
      if (lane < k) keys[p * k + lane] = rk;
      const unsigned fmask = __ballot_sync(kFull, fl && lane < k);
      if (lane == 0) {
        flags[p] = fmask;
        worst[p] = key_dist(last);
      }
      acc_total += kept;
    }
  }
  if (lane == 0 && acc_total)
    atomicAdd(reinterpret_cast<unsigned long long*>(counters + kCntAccepted), acc_total);
}

// ---------------------------------------------------------------------------
// layout conversion
// ---------------------------------------------------------------------------
__global__ void k_export(const u64* __restrict__ keys, const u32* __restrict__ flags, u64 n,
                         u32 k, u32 shift, u32* __restrict__ ids, float* __restrict__ dists,
                         uint8_t* __restrict__ f8) {
  const u64 total = n * k;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (u64)gridDim.x * blockDim.x) {
    const u64 key = keys[i];
    if (ids) ids[i] = key_id(key) + shift;
    if (dists) dists[i] = key_dist(key);
    if (f8) f8[i] = flags ? (uint8_t)((flags[i / k] >> (i % k)) & 1u) : 0;
  }
}

__global__ __launch_bounds__(256) void k_import(const u32* __restrict__ ids,
                                                const float* __restrict__ dists,
                                                const uint8_t* __restrict__ f8, u64 n, u32 k,
                                                u64* __restrict__ keys,
                                                u32* __restrict__ flags) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 r = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    bool f = false;
    if (lane < k) {
      keys[r * k + lane] = pack_key(dists[r * k + lane], ids[r * k + lane]);
      f = f8 ? f8[r * k + lane] != 0 : false;
    }
    const unsigned m = __ballot_sync(kFull, f);
    if (flags && lane == 0) flags[r] = m;
  }
}

unsigned warp_grid(const Runner& r, u64 items) {
  const u64 want = ceil_div<u64>(items, 8);
  const u64 cap = (u64)r.num_sms * 16;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

uint32_t bound_of(double rho, uint32_t k) {
  return (uint32_t)std::ceil(rho * (double)k);
}

}  // namespace

void validate_nnd(const NndParams& p, uint64_t n) {
  require(!(p.rho <= 0.0 || p.rho > 1.0), "nn_descent: rho must be in (0, 1]");
  require(p.delta >= 0.0, "nn_descent: delta must be >= 0");
  const uint64_t cap = p.candidate_capacity ? p.candidate_capacity : 2ull * p.k;
  require(cap >= p.k, "nn_descent: candidate_capacity must be >= k");
  require(p.k >= 1 && p.k < n, "init_random_graph: need 1 <= k < N");
  require(p.k <= 32, "nn_descent: the B200 path supports k <= 32");
  require(n < 0xffffffffull, "nn_descent: N must fit a 32-bit point id");
}

namespace {
void launch_init(const Runner& r, const DevRows& ds, u32 k, u64 seed, u64* keys, u32* flags,
                 float* worst) {
  const unsigned g =
      (unsigned)std::min<u64>(ceil_div<u64>(ds.n, kInitThreads / 32), (u64)r.num_sms * 32);
  if (ds.nrm)
    k_init<true><<<g, kInitThreads, 0, r.stream>>>(ds.x, ds.n, ds.d, k, seed, keys, flags, worst,
                                                   ds.nrm);
  else
    k_init<false><<<g, kInitThreads, 0, r.stream>>>(ds.x, ds.n, ds.d, k, seed, keys, flags, worst,
                                                    nullptr);
  KNNG_LAUNCH_CHECK();
}
}  // namespace

void init_random_graph_device(Runner& r, const DevRows& ds, uint32_t k, uint64_t seed,
                              uint64_t* keys, uint32_t* flags) {
  require(k >= 1 && k < ds.n, "init_random_graph: need 1 <= k < N");
  require(k <= 32, "init_random_graph: the B200 path supports k <= 32");
  DBuf<float> worst(r, ds.n);
  launch_init(r, ds, k, seed, keys, flags, worst.p);
}

namespace {


// Which reverse-list path nn_descent takes (both give bit-identical graphs,
// tests/test_parity_gpu.py): the scatter path unless KNNG_REV_SORT=1.  With
// segments of <= 32 ranked by a warp sort and 33-512 in shared memory it won
// at 1M points (sampling 24.9 -> 21.6 ms per build) and lost at 10M
// (2.24 -> 2.65 s; profiles/r02_sampling_paths.md); ranking 33-128 in
// registers (warp_sort_regs) and the joins bitmap turned that around.
bool rev_sort_forced(uint64_t n) {
  const char* v = std::getenv("KNNG_REV_SORT");
  if (v && v[0] == '1') return true;
  (void)n;
  // the scatter path at every size since its segments of 33-128 entries are
  // ranked in registers: 10M x 96 clustered(16) builds 3.86 s vs 4.13 s
  // sorted, 5M 1.51 vs 1.57 s (round 2; before, the sort won beyond 2M)
  return false;
}

void sample_into(Runner& r, uint64_t n, uint32_t k, uint32_t B, uint64_t iter_seed,
                 const uint64_t* keys, uint32_t* flags, SampleLists& s, RevCsr& c, bool prune_old,
                 uint64_t* launches) {
  const unsigned g = warp_grid(r, n);
  double t_lap = slow_trace_on() ? trace_clock_ms() : 0;
  auto lap = [&](const char* what) {
    if (!slow_trace_on()) return;
    const double t = trace_clock_ms();
    if (t - t_lap > 5.0)
      std::fprintf(stderr, "[knng slow] t %.1f dev %d sample_into %s host %.1f ms\n", t, r.device,
                   what, t - t_lap);
    t_lap = t;
  };
  c.cnt_new.zero();
  c.cnt_old.zero();
  k_sample_fwd<<<g, 256, 0, r.stream>>>(keys, flags, n, k, B, iter_seed, s.nf.p, s.nfn.p,
                                        s.of.p, s.ofn.p, c.cnt_new.p, c.cnt_old.p, !prune_old);
  KNNG_LAUNCH_CHECK();
  lap("zero+sample_fwd");
  if (prune_old) {
    k_join_bits<<<warp_grid(r, (n + 31) / 32), 256, 0, r.stream>>>(n, s.nfn.p, c.cnt_new.p,
                                                                    c.join_bits.p);
    KNNG_LAUNCH_CHECK();
    k_old_count<<<g, 256, 0, r.stream>>>(n, k, s.of.p, s.ofn.p, c.join_bits.p, c.src_cnt.p,
                                         c.cnt_old.p);
    KNNG_LAUNCH_CHECK();
    exclusive_scan_u32(r, c.src_cnt.p, c.src_off_old.p, n);
  } else {
    exclusive_scan_u32(r, s.ofn.p, c.src_off_old.p, n);
  }
  lap("old_count+scan");
  if (prune_old && !rev_sort_forced(n)) {
    // inside nn_descent: scatter + rank-sampled reverse lists (no sort)
    exclusive_scan_u32(r, c.cnt_new.p, c.off_new.p, n);
    exclusive_scan_u32(r, c.cnt_old.p, c.off_old.p, n);
    c.cur_new.zero();
    c.cur_old.zero();
    k_rev_scatter<<<g, 256, 0, r.stream>>>(n, k, B, s.nf.p, s.nfn.p, s.of.p, s.ofn.p,
                                           c.join_bits.p, c.off_new.p, c.off_old.p, c.cur_new.p,
                                           c.cur_old.p, c.key_new.p, c.key_old.p);
    KNNG_LAUNCH_CHECK();
    c.long_cnt.zero();
    k_rev_select_rank<<<g, 256, 0, r.stream>>>(n, B, iter_seed, c.off_new.p, c.key_new.p,
                                               c.off_old.p, c.key_old.p, s.nr.p, s.nrn.p,
                                               s.orv.p, s.orn.p, c.long_cnt.p, c.long_rec.p);
    KNNG_LAUNCH_CHECK();
    // (idempotent; cheap next to the sampling launches)
    KNNG_CUDA(cudaFuncSetAttribute(k_rev_select_long,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLongSmem));
    k_rev_select_long<<<r.num_sms * 2, 256, kLongSmem, r.stream>>>(n, B, c.off_new.p, c.key_new.p,
                                                           c.off_old.p, c.key_old.p, s.nr.p,
                                                           s.orv.p, c.long_cnt.p, c.long_rec.p);
    KNNG_LAUNCH_CHECK();
    if (launches) *launches += 4 + 3 + 2 * 3 + 3;
    return;
  }
  exclusive_scan_u32(r, s.nfn.p, c.src_off_new.p, n);
  exclusive_scan_u32(r, c.cnt_new.p, c.off_new.p, n);
  exclusive_scan_u32(r, c.cnt_old.p, c.off_old.p, n);
  lap("scans");
  k_emit_pairs<<<g, 256, 0, r.stream>>>(n, B, s.nf.p, s.nfn.p, c.src_off_new.p, nullptr,
                                        c.key_new.p, c.val_new.p);
  KNNG_LAUNCH_CHECK();
  k_emit_pairs<<<g, 256, 0, r.stream>>>(n, k, s.of.p, s.ofn.p, c.src_off_old.p,
                                        prune_old ? c.join_bits.p : nullptr, c.key_old.p,
                                        c.val_old.p);
  KNNG_LAUNCH_CHECK();
  lap("emit");
  // sorts read their element counts (src_off[n]) on the device: no host sync
  bool tn = false, to = false;
  const u32 maxk = (u32)(n ? n - 1 : 0);
  radix_sort_pairs_dev(r, c.key_new.p, c.val_new.p, c.tk_new.p, c.tv_new.p, n * B,
                       c.src_off_new.p + n, maxk, &tn);
  radix_sort_pairs_dev(r, c.key_old.p, c.val_old.p, c.tk_old.p, c.tv_old.p, n * k,
                       c.src_off_old.p + n, maxk, &to);
  lap("sorts");
  k_rev_select<<<g, 256, 0, r.stream>>>(n, B, iter_seed, c.off_new.p, tn ? c.tv_new.p : c.val_new.p,
                                        c.off_old.p, to ? c.tv_old.p : c.val_old.p, s.nr.p,
                                        s.nrn.p, s.orv.p, s.orn.p);
  KNNG_LAUNCH_CHECK();
  if (launches) *launches += 4 + (prune_old ? 3 : 1) + 4 * 3 + 2 * 9;
}

void alloc_lists(Runner& r, uint64_t n, uint32_t k, uint32_t B, SampleLists& s, RevCsr& c) {
  s.bound = B;
  const u64 b = B ? B : 1;
  s.nf.alloc(r, n * b);
  s.nfn.alloc(r, n);
  s.of.alloc(r, n * k);
  s.ofn.alloc(r, n);
  s.nr.alloc(r, n * b);
  s.nrn.alloc(r, n);
  s.orv.alloc(r, n * b);
  s.orn.alloc(r, n);
  c.cnt_new.alloc(r, n);
  c.cnt_old.alloc(r, n);
  c.join_bits.alloc(r, (n + 31) / 32 + 1);
  c.cur_new.alloc(r, n);
  c.cur_old.alloc(r, n);
  // hub segments (> kRankSmem entries): at most (new + old entries) / kRankSmem
  c.long_cnt.alloc(r, 1);
  c.long_rec.alloc(r, (n * (b + k) / kRankSmem + 2) * (2 + 32));
  c.off_new.alloc(r, n + 1);
  c.off_old.alloc(r, n + 1);
  c.src_cnt.alloc(r, n);
  c.src_off_new.alloc(r, n + 1);
  c.src_off_old.alloc(r, n + 1);
  c.key_new.alloc(r, n * b);
  c.val_new.alloc(r, n * b);
  c.tk_new.alloc(r, n * b);
  c.tv_new.alloc(r, n * b);
  c.key_old.alloc(r, n * k);
  c.val_old.alloc(r, n * k);
  c.tk_old.alloc(r, n * k);
  c.tv_old.alloc(r, n * k);
}

}  // namespace

void sample_neighbors_device(Runner& r, uint64_t n, uint32_t k, double rho, uint64_t seed,
                             uint64_t iter, const uint64_t* keys, uint32_t* flags,
                             SampleLists& out) {
  require(!(rho <= 0.0 || rho > 1.0), "sample_neighbors: rho must be in (0, 1]");
  require(k >= 1 && k <= 32, "sample_neighbors: the B200 path supports 1 <= k <= 32");
  const uint32_t B = bound_of(rho, k);
  RevCsr c;
  alloc_lists(r, n, k, B, out, c);
  sample_into(r, n, k, B, mix_seed(seed, 0x5a3f1e00ull + iter), keys, flags, out, c, false,
              nullptr);
}

namespace {
// buffer of at least `count` entries: the workspace's (grown if short) or `own`
template <class T>
T* ws_buf(Runner& r, DBuf<T>* ws, DBuf<T>& own, uint64_t count) {
  DBuf<T>& b = ws ? *ws : own;
  if (b.n < count) b.alloc(r, count);
  return b.p;
}
}  // namespace

namespace {
void nn_descent_core(Runner& r, const DevRows& ds, const NndParams& p, uint64_t* keys,
                     uint32_t* flags, NndStats* st, bool time_kernels, NndWorkspace* ws) {
  const u64 n = ds.n;
  const u32 k = p.k;
  const u32 B = bound_of(p.rho, k);
  const u32 cap = (u32)(p.candidate_capacity ? p.candidate_capacity : 2ull * k);
  const u32 ways = cap < kWays ? cap : kWays;
  const u32 nb = cap / ways;
  const u32 S = nb * ways;
  DeviceGuard guard(r.device);

  StageTimer tm(time_kernels, r.stream);
  const auto t_call = std::chrono::steady_clock::now();

  // per-build buffers: the context's workspace (grow-only, reused across
  // builds on this device), else owned by this call
  NndWorkspace own_ws;
  NndWorkspace& W = ws ? *ws : own_ws;
  float* worst_p = ws_buf(r, &W.worst, W.worst, n);
  u64* slots_p = ws_buf(r, &W.slots, W.slots, n * S);
  KNNG_CUDA(cudaMemsetAsync(slots_p, 0xff, n * S * sizeof(u64), r.stream));
  uint8_t* touched_p = ws_buf(r, &W.touched, W.touched, n);
  KNNG_CUDA(cudaMemsetAsync(touched_p, 0, n, r.stream));
  u64* counters_p = ws_buf(r, &W.counters, W.counters, kNumCounters);
  auto zero_counters = [&] {
    KNNG_CUDA(cudaMemsetAsync(counters_p, 0, kNumCounters * sizeof(u64), r.stream));
  };
  HBuf<u64> hcount(kNumCounters);
  if (W.lists_n < n || W.lists_k != k || W.lists_b != B) {
    alloc_lists(r, n, k, B, W.lists, W.rev);
    W.lists_n = n;
    W.lists_k = k;
    W.lists_b = B;
  }
  SampleLists& s = W.lists;
  RevCsr& c = W.rev;
  uint64_t launches = 0;

  launch_init(r, ds, k, p.seed, keys, flags, worst_p);
  ++launches;
  tm.tick(kStInit);

  // join lists (compact per point) + join launch shape
  const JoinPlan plan = plan_join(r, ds.d, k, B);
  u32* L_cnt_p = ws_buf(r, &W.L_cnt, W.L_cnt, n);
  u32* L_ids_p = ws_buf(r, &W.L_ids, W.L_ids, n * plan.RMAX);
  // Offer queue: each point chunk owns a region sized for its worst case (2
  // offers per pair, max pairs C(2B,2) + 2B(k+B)), so nothing can overflow;
  // points are processed in slices to bound the queue (budget below).
  // memory available to stream-ordered allocations: free device memory plus
  // what the pool holds unused from earlier calls (cudaMemGetInfo counts that
  // as used, so the budget -- and the queue size -- drifted between builds
  // and a later build had to map tens of GB afresh)
  // the slicing is decided once per (n, queue-region) shape and kept in the
  // workspace: a warm build makes no memory query
  u64 chunks_per_slice = W.q_chunks_per_slice;
  if (!(W.q_n == n && W.q_per_chunk == plan.q_per_chunk && chunks_per_slice)) {
    size_t free_b = 0, total_b = 0;
    KNNG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    {
      cudaMemPool_t pool;
      uint64_t reserved = 0, used = 0;
      if (cudaDeviceGetDefaultMemPool(&pool, r.device) == cudaSuccess &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) ==
              cudaSuccess &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
          reserved > used)
        free_b += reserved - used;
      cudaGetLastError();
    }
    free_b += W.q_key.n * 8 + W.q_tgt.n * 4;  // reused below
    // up to 64 GB of worst-case queue (B200: 180 GB HBM): C2 runs as a single
    // slice (one join + one offer launch per iteration)
    const u64 budget = std::min<u64>(64ull << 30, free_b / 3);
    chunks_per_slice = std::max<u64>(1, budget / (plan.q_per_chunk * 12));
    chunks_per_slice = std::min<u64>(chunks_per_slice, ceil_div<u64>(n, (u64)kJoinChunk));
    W.q_chunks_per_slice = chunks_per_slice;
    W.q_per_chunk = plan.q_per_chunk;
    W.q_n = n;
  }
  u64 slice = chunks_per_slice * kJoinChunk;
  if (slice > n) slice = n;
  u32* q_fill_p = ws_buf(r, &W.q_fill, W.q_fill, chunks_per_slice);
  u64* q_key_p = ws_buf(r, &W.q_key, W.q_key, chunks_per_slice * plan.q_per_chunk);
  u32* q_tgt_p = ws_buf(r, &W.q_tgt, W.q_tgt, chunks_per_slice * plan.q_per_chunk);
  u32* chunk_ctr_p = ws_buf(r, &W.chunk_ctr, W.chunk_ctr, 1);
  // points with a new entry, compacted: late iterations join a small fraction
  u32* act_p = ws_buf(r, &W.act, W.act, n);
  u32* act_flag_p = ws_buf(r, &W.act_flag, W.act_flag, n);
  u64* act_off_p = ws_buf(r, &W.act_off, W.act_off, n + 1);
  JoinLaunch jl;
  jl.act = act_p;
  jl.X = ds.x;
  jl.nrm = ds.nrm;
  jl.d = ds.d;
  jl.n_rows = n;
  const bool use_tc = join_tc_supported(ds.x, ds.d, k, B, ds.nrm != nullptr);
  jl.L_ids = L_ids_p;
  jl.L_cnt = L_cnt_p;
  jl.worst = worst_p;
  jl.chunk_counter = chunk_ctr_p;
  jl.q_key = q_key_p;
  jl.q_tgt = q_tgt_p;
  jl.q_fill = q_fill_p;
  jl.counters = counters_p;

  if (st) *st = NndStats{};
  const double threshold = p.delta * (double)k * (double)n;
  cudaEvent_t iter_done;
  KNNG_CUDA(cudaEventCreateWithFlags(&iter_done, cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t e;
    ~EvGuard() { cudaEventDestroy(e); }
  } iter_done_guard{iter_done};
  u64 prev_offers = ~0ull;  // offers queued by the previous iteration
  // KNNG_BOUND_SLICES (1 = off): join slices of a dense iteration
  u64 bound_slices = 4;
  if (const char* v = std::getenv("KNNG_BOUND_SLICES")) bound_slices = std::max(1, std::atoi(v));
  for (u64 iter = 0; iter < p.max_iters; ++iter) {
    const bool use_touched = S <= 64 && prev_offers < 4 * n;
    zero_counters();
    const u64 iter_seed = mix_seed(p.seed, 0x5a3f1e00ull + iter);
    sample_into(r, n, k, B, iter_seed, keys, flags, s, c, true, &launches);
    tm.tick(kStSample);
    launch_join_lists(r, n, k, B, plan.RMAX, s.nf.p, s.nfn.p, s.of.p, s.ofn.p, s.nr.p, s.nrn.p,
                      s.orv.p, s.orn.p, L_ids_p, L_cnt_p);
    ++launches;
    tm.tick(kStLists);
    build_active_list(r, n, L_cnt_p, act_flag_p, act_off_p, act_p);
    launches += 5;
    // the active count stays on the device: every slice is launched and its
    // kernels bound themselves by it (no host round trip mid-iteration; the
    // slices past the count exit at once)
    jl.n_live = act_off_p + n;
    // iteration 0 (random rows: nearly every pair passes the row filter)
    // runs the join in bound_slices slices with k_bucket_bound tightening
    // the filter between them (later dense iterations gain too little to pay
    // for the extra passes: C2 offers 216M -> 154M in iteration 2)
    const bool bound = !use_tc && S <= 64 && bound_slices > 1 && iter == 0;
    u64 it_slice = slice;
    if (bound) {
      const u64 want = ceil_div<u64>(ceil_div<u64>(n, bound_slices), (u64)kJoinChunk) * kJoinChunk;
      if (want < it_slice) it_slice = want;
    }
    const u64 nslices = ceil_div<u64>(n, it_slice);
    for (u64 si = 0; si < nslices; ++si) {
      jl.p_lo = si * it_slice;
      jl.p_hi = std::min<u64>(n, jl.p_lo + it_slice);
      KNNG_CUDA(cudaMemsetAsync(chunk_ctr_p, 0, sizeof(u32), r.stream));
      tm.tick(kStLists);
      if (use_tc) {
        KNNG_CUDA(cudaMemsetAsync(q_fill_p, 0, chunks_per_slice * sizeof(u32), r.stream));
        launch_join_tc(r, plan, jl);
      } else {
        launch_join(r, plan, jl);
      }
      tm.tick(kStJoin);
      launch_offer(r, plan, q_key_p, q_tgt_p, q_fill_p,
                   (u32)ceil_div<u64>(jl.p_hi - jl.p_lo, (u64)kJoinChunk), slots_p, S, nb, ways,
                   counters_p, jl.p_lo, jl.n_live, n, use_touched ? touched_p : nullptr);
      tm.tick(kStOffer);
      launches += 2;
      if (bound && si + 1 < nslices) {
        k_bucket_bound<<<warp_grid(r, n), 256, 0, r.stream>>>(n, k, S, worst_p, slots_p);
        KNNG_LAUNCH_CHECK();
        ++launches;
        tm.tick(kStOffer);
      }
    }
    if (S <= 64)
      k_apply<<<warp_grid(r, (n + 31) / 32), 256, 0, r.stream>>>(
          n, k, S, keys, flags, worst_p, slots_p, counters_p, use_tc ? ds.x : nullptr, ds.d,
          use_touched ? touched_p : nullptr);
    else
      k_apply_wide<<<warp_grid(r, n), 256, 0, r.stream>>>(n, k, S, keys, flags, worst_p, slots_p,
                                                          counters_p, use_tc ? ds.x : nullptr,
                                                          ds.d);
    KNNG_LAUNCH_CHECK();
    launches += 1;
    tm.tick(kStApply);
    KNNG_CUDA(cudaMemcpyAsync(hcount.p, counters_p, kNumCounters * sizeof(u64),
                              cudaMemcpyDeviceToHost, r.stream));
    // busy-poll the iteration's end: a sleeping cudaStreamSynchronize woke
    // up late now and then, idling the GPU before the next iteration (up to
    // ~7 ms per iteration, seen as a variable 'sample' stage)
    KNNG_CUDA(cudaEventRecord(iter_done, r.stream));
    while (cudaEventQuery(iter_done) == cudaErrorNotReady) {
    }
    KNNG_CUDA(cudaGetLastError());
    tm.tick(kStSync);
    const u64 accepted = hcount.p[kCntAccepted];
    prev_offers = hcount.p[kCntOffers];
    if (std::getenv("KNNG_TRACE"))
      std::fprintf(stderr, "[knng nnd] dev %d t %.1f ms iter %llu pairs %llu offers %llu seen %llu accepted %llu\n",
                   r.device,
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call).count(),
                   (unsigned long long)iter, (unsigned long long)hcount.p[kCntPairs],
                   (unsigned long long)hcount.p[kCntOffers],
                   (unsigned long long)hcount.p[kCntOfferSeen], (unsigned long long)accepted);
    if (st) {
      st->accepted_per_iter.push_back(accepted);
      st->iterations = iter + 1;
      st->pairs += hcount.p[kCntPairs];
      st->staged_rows += hcount.p[kCntStagedRows];
      st->offers += hcount.p[kCntOffers];
      st->offers_per_iter.push_back(hcount.p[kCntOffers]);
      st->pairs_per_iter.push_back(hcount.p[kCntPairs]);
      st->join_launches += nslices;
    }
    if ((double)accepted < threshold) break;
  }
  tm.tick(kStSync);
  if (time_kernels && st) {
    r.sync();
    tm.accumulate(st->stage_ms, 8);
    st->join_ms = st->stage_ms[kStJoin];
    st->offer_ms = st->stage_ms[kStOffer];
    st->total_ms = tm.total_ms();
  }
  if (st) st->launches = launches;
  if (slow_trace_on())
    std::fprintf(stderr, "[knng slow] t %.1f dev %d nnd epilogue done\n", trace_clock_ms(), r.device);
}

__global__ void k_gather_f32(const float* __restrict__ src, const u32* __restrict__ order, u64 n,
                             float* __restrict__ dst) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x)
    dst[i] = src[order[i]];
}

// Row i of the renumbered build is point order[i]: relabel its ids, restore
// the (dist, id) order among equal distances (ties are the only entries the
// relabelling can reorder) and store it as row order[i], flags following
// their entries.  One warp per row (k <= 32).
__global__ __launch_bounds__(256) void k_unrenumber(const u64* __restrict__ kin,
                                                    const u32* __restrict__ fin,
                                                    const u32* __restrict__ order, u64 n, u32 k,
                                                    u64* __restrict__ kout,
                                                    u32* __restrict__ fout) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 i = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    u64 key = ~0ull;
    u32 f = 0;
    if (lane < k) {
      key = kin[i * k + lane];
      if (key != ~0ull) key = (key & 0xffffffff00000000ull) | order[key_id(key)];
      f = (fin[i] >> lane) & 1u;
    }
    // an inversion can only sit between equal distances; sort when one exists
    const u64 prev = __shfl_up_sync(0xffffffffu, key, 1);
    if (__any_sync(0xffffffffu, lane > 0 && lane < k && prev > key)) {
      // bitonic sort of 32 (key, flag) pairs
      for (unsigned size = 2; size <= 32; size <<= 1)
        for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
          const u64 ok = __shfl_xor_sync(0xffffffffu, key, stride);
          const u32 of = __shfl_xor_sync(0xffffffffu, f, stride);
          const bool up = ((lane & size) == 0);
          const bool lower = ((lane & stride) == 0);
          const bool take = lower == up ? ok < key : ok > key;
          if (take) {
            key = ok;
            f = of;
          }
        }
    }
    const u64 dst = order[i];
    if (lane < k) kout[dst * k + lane] = key;
    const u32 bits = __ballot_sync(0xffffffffu, lane < k && f);
    if (lane == 0) fout[dst] = bits;
  }
}
}  // namespace

// NN-Descent on a locality renumbering of the points: the build runs on the
// rows permuted into a Morton order of random projections (locality.cu), so
// a point's neighbours -- and the rows a join tile gathers, the slots an offer
// hits -- sit close together in HBM.  The renumbered build is a deterministic
// function of (points, seed) like the plain one (its random streams attach to
// the new ids); the graph comes back in the caller's numbering and order.
// C2: 174.1 -> 161.2 ms per build (profiles/r02_renumber.md).
// KNNG_NND_RENUMBER=0 builds in the given numbering.
void nn_descent_device(Runner& r, const DevRows& ds, const NndParams& p, uint64_t* keys,
                       uint32_t* flags, NndStats* st, bool time_kernels, NndWorkspace* ws) {
  validate_nnd(p, ds.n);
  const u64 n = ds.n;
  const char* env = std::getenv("KNNG_NND_RENUMBER");
  const bool renumber = n >= (1ull << 17) && ds.d <= 1024 && !(env && *env && atoi(env) == 0);
  if (!renumber) {
    nn_descent_core(r, ds, p, keys, flags, st, time_kernels, ws);
    return;
  }
  DeviceGuard guard(r.device);
  const auto t0 = std::chrono::steady_clock::now();
  const u32 k = p.k;
  DBuf<u32> order(r, n);
  locality_order(r, ds.x, n, ds.d, mix_seed(p.seed, 0x10ca11e5ull), order.p);
  DBuf<float> xr(r, n * (u64)ds.d), nr;
  gather_rows_device(r, ds.x, ds.d, order.p, n, xr.p);
  const unsigned g = (unsigned)std::min<u64>(ceil_div<u64>(n, 256), (u64)r.num_sms * 32);
  if (ds.nrm) {
    nr.alloc(r, n);
    k_gather_f32<<<g, 256, 0, r.stream>>>(ds.nrm, order.p, n, nr.p);
    KNNG_LAUNCH_CHECK();
  }
  DBuf<u64> kr(r, n * k);
  DBuf<u32> fr(r, n);
  const double pre_ms = time_kernels
                            ? (r.sync(), 1e3 * std::chrono::duration<double>(
                                               std::chrono::steady_clock::now() - t0).count())
                            : 0.0;
  nn_descent_core(r, DevRows{xr.p, n, ds.d, ds.nrm ? nr.p : nullptr}, p, kr.p, fr.p, st,
                  time_kernels, ws);
  const auto t1 = std::chrono::steady_clock::now();
  k_unrenumber<<<warp_grid(r, n), 256, 0, r.stream>>>(kr.p, fr.p, order.p, n, k, keys, flags);
  KNNG_LAUNCH_CHECK();
  if (st) st->launches += 6;
  if (time_kernels && st) {
    r.sync();
    const double post_ms =
        1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    st->stage_ms[kStInit] += pre_ms + post_ms;
    st->total_ms += pre_ms + post_ms;
  }
}

void export_graph_device(const Runner& r, const uint64_t* keys, const uint32_t* flags,
                         uint64_t n, uint32_t k, uint32_t id_shift, uint32_t* ids, float* dists,
                         uint8_t* flags_u8) {
  const u64 total = n * k;
  if (!total) return;
  const unsigned g = (unsigned)std::min<u64>(ceil_div<u64>(total, 256), (u64)r.num_sms * 32);
  k_export<<<g, 256, 0, r.stream>>>(keys, flags, n, k, id_shift, ids, dists, flags_u8);
  KNNG_LAUNCH_CHECK();
}

void import_graph_device(const Runner& r, const uint32_t* ids, const float* dists,
                         const uint8_t* flags_u8, uint64_t n, uint32_t k, uint64_t* keys,
                         uint32_t* flags) {
  if (!n) return;
  k_import<<<warp_grid(r, n), 256, 0, r.stream>>>(ids, dists, flags_u8, n, k, keys, flags);
  KNNG_LAUNCH_CHECK();
}

}  // namespace knng_b200
