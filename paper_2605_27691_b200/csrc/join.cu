// join.cu -- NN-Descent local join (nndescent.cpp:135-197) on the B200.
//
//   k_join_lists  warp per point: build_join_lists (:135-153) -- new = nf U nr,
//                 old = (of U orv) \ new, first occurrence wins -- written
//                 compactly (L_ids[p * RMAX ..], L_cnt[p] = nn | na << 16).
//   k_join        persistent CTAs (two per SM), a software pipeline over
//                 batches of points: while batch b is computed from one smem
//                 buffer, the feature rows of batch b+1 stream into the other
//                 with cp.async (16 B, coalesced per row).  A batch packs as
//                 many points as fit; its 4x4 micro-tiles -- per point a
//                 trapezoid of 4-entry blocks (new blocks x all blocks, j > i;
//                 see tiles_of), rows interleaved so consecutive threads read
//                 consecutive smem rows (conflict-free LDS.128) -- are spread
//                 over all 256 threads.  Distances are exact-order (common.cuh),
//                 filtered by the worst snapshot (nndescent.hpp:39-40) and the
//                 survivors appended to the chunk's offer queue in HBM.
//   k_offer       resolves queued offers into the 4-way candidate buckets with
//                 atomicMin cascades (lock-free, order-independent).
#include <algorithm>
#include <cstdlib>

#include "join.hpp"
#include "nndescent.hpp"

namespace knng_b200 {
namespace {

constexpr u32 kNone = 0xffffffffu;
#ifndef KNNG_JOIN_THREADS
#define KNNG_JOIN_THREADS 256
#endif
#ifndef KNNG_JOIN_CTAS
#define KNNG_JOIN_CTAS 2
#endif
#ifndef KNNG_JOIN_UNROLL
#define KNNG_JOIN_UNROLL 4  // unroll of the 4-dim micro-tile step (1/2/4: 102.2/99.3/97.4 ms per C2 build)
#endif
constexpr int kJUnroll = KNNG_JOIN_UNROLL;
constexpr int kJT = KNNG_JOIN_THREADS;  // threads per join CTA
constexpr int kJCtas = KNNG_JOIN_CTAS;  // resident join CTAs per SM (latency overlap)
constexpr int kTPT = 1;                 // micro-tiles per thread
constexpr int kMaxTiles = kJT * kTPT;   // tiles per batch
constexpr int G = kJoinChunk;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Bucket of candidate v in point u's candidate buffer (kWays slots each).
__device__ __forceinline__ u32 bucket_hash(u32 u, u32 v, u32 nb) {
  u32 x = v * 0x9E3779B1u + u * 0x85EBCA77u;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  x *= 0x297A2D39u;
  x ^= x >> 15;
  return x % nb;
}

// Lock-free offers (k_offer) given a snapshot of the bucket.  The bucket keeps its W
// smallest distinct (dist,id) keys in ascending order: each step atomicMin's
// the carried key into one slot and carries the larger of (old, key) onward.
// Slots only decrease, so whatever the interleaving the final bucket is the W
// smallest distinct keys offered (order-independent -> deterministic build).
// Any snapshot is safe: a key >= the snapshot tail can never be among the W
// smallest, a key equal to a snapshot entry is already buffered (or displaced
// by smaller ones), and every slot before the snapshot insertion position
// already holds a smaller key, so the cascade starts there.
// ---------------------------------------------------------------------------
// k_join_lists
// ---------------------------------------------------------------------------
__global__ __launch_bounds__(256) void k_join_lists(u64 n, u32 k, u32 B, int RMAX,
                                                    const u32* __restrict__ nf,
                                                    const u32* __restrict__ nfn,
                                                    const u32* __restrict__ of,
                                                    const u32* __restrict__ ofn,
                                                    const u32* __restrict__ nr,
                                                    const u32* __restrict__ nrn,
                                                    const u32* __restrict__ orv,
                                                    const u32* __restrict__ orn,
                                                    u32* __restrict__ L_ids,
                                                    u32* __restrict__ L_cnt) {
  __shared__ u32 s_list[8][128];
  // per-warp membership hash of the list so far (<= 128 of 256 slots used):
  // a candidate is checked in O(1) probes instead of against every entry
  constexpr u32 kHash = 256;
  __shared__ u32 s_hash[8][kHash];
  const unsigned lane = lane_id(), w = threadIdx.x >> 5;
  u32* lst = s_list[w];
  u32* hs = s_hash[w];
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  auto slot_of = [](u32 c) { return (c * 0x9E3779B1u) >> 24; };  // top 8 bits
  for (u64 p = (((u64)blockIdx.x * blockDim.x) >> 5) + w; p < n; p += warps) {
    // no new entry: the point has no new x new / new x old pair (:157-171);
    // an empty descriptor keeps the join from gathering its old list at all
    if (nfn[p] + nrn[p] == 0) {
      if (lane == 0) L_cnt[p] = 0;
      continue;
    }
    for (u32 t = lane; t < kHash; t += 32) hs[t] = kNone;
    __syncwarp();
    int cnt = 0, nn = 0;
    for (int src = 0; src < 4; ++src) {
      const u32* base = src == 0 ? nf + p * B : src == 1 ? nr + p * B : src == 2 ? of + p * k
                                                                                 : orv + p * B;
      const u32 len = src == 0 ? nfn[p] : src == 1 ? nrn[p] : src == 2 ? ofn[p] : orn[p];
      for (u32 b0 = 0; b0 < len; b0 += 32) {
        const bool valid = b0 + lane < len;
        const u32 c = valid ? base[b0 + lane] : kNone;
        const unsigned m = __match_any_sync(kFull, c);
        bool keep = valid && (__ffs(m) - 1 == (int)lane);
        if (keep) {
          for (u32 h = slot_of(c);; h = (h + 1) & (kHash - 1)) {
            const u32 v = hs[h];
            if (v == c) {
              keep = false;
              break;
            }
            if (v == kNone) break;
          }
        }
        const unsigned kb = __ballot_sync(kFull, keep);
        if (keep) {
          lst[cnt + __popc(kb & lanemask_lt())] = c;
          // kept candidates are distinct: claim the first free slot
          for (u32 h = slot_of(c);; h = (h + 1) & (kHash - 1))
            if (atomicCAS(&hs[h], kNone, c) == kNone) break;
        }
        cnt += __popc(kb);
        __syncwarp();
      }
      if (src == 1) nn = cnt;
    }
    for (int t = lane; t < cnt; t += 32) L_ids[p * RMAX + t] = lst[t];
    if (lane == 0) L_cnt[p] = (u32)nn | ((u32)cnt << 16);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// k_offer
// ---------------------------------------------------------------------------
#ifndef KNNG_OFFER_BATCH
#define KNNG_OFFER_BATCH 2
#endif
constexpr int kOfferBatch = KNNG_OFFER_BATCH;  // offers per thread (independent atomics per round)

// Targets outside [t_lo, t_hi) are skipped (target-range passes, opt-in via
// KNNG_OFFER_PASSES; see launch_offer).
__global__ __launch_bounds__(256) void k_offer(const u64* __restrict__ q_key,
                                               const u32* __restrict__ q_tgt,
                                               const u32* __restrict__ q_fill, u64 q_per_chunk,
                                               u32 chunks, u64* __restrict__ slots, u32 S,
                                               u32 nb, u32 ways, u64* __restrict__ counters,
                                               u64 p_lo, const u64* __restrict__ n_live,
                                               u32 t_lo, u32 t_hi,
                                               uint8_t* __restrict__ touched) {
  if (n_live) {  // the slice's live chunk count, read on the device
    const u64 live = *n_live;
    const u64 hi = live < p_lo ? 0 : live - p_lo;
    const u64 c = (hi + G - 1) / G;
    if (c < chunks) chunks = (u32)c;
  }
  for (u32 region = blockIdx.x; region < chunks; region += gridDim.x) {
    const u32 fill = q_fill[region];
    if (threadIdx.x == 0 && counters && t_lo == 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(counters + kCntOfferSeen), (u64)fill);
    const u64 base = (u64)region * q_per_chunk;
    // warp-uniform trip count + __syncwarp: lanes that leave the cascade early
    // must not race ahead, or the warp splits into 1-2-lane groups
    for (u32 e_base = 0; e_base < fill; e_base += kOfferBatch * blockDim.x) {
      const u32 e0 = e_base + threadIdx.x;
      u64 key[kOfferBatch];
      u64* bk[kOfferBatch];
      u32 pos[kOfferBatch];
      u32 key_tgt[kOfferBatch];
#pragma unroll
      for (int i = 0; i < kOfferBatch; ++i) {
        const u32 e = e0 + i * blockDim.x;
        bk[i] = nullptr;
        if (e < fill) {
          const u32 tgt = q_tgt[base + e];
          key_tgt[i] = tgt;
          if (tgt >= t_lo && tgt < t_hi) {
            key[i] = q_key[base + e];
            bk[i] = slots + (u64)tgt * S + (u64)bucket_hash(tgt, key_id(key[i]), nb) * ways;
          }
        }
      }
      // L2-coherent snapshots (L1 lines would go stale under the atomics);
      // the cascade of each offer starts at its snapshot insertion position
#pragma unroll
      for (int i = 0; i < kOfferBatch; ++i) {
        pos[i] = 4;
        if (!bk[i]) continue;
        u64 sn[4];
        if (ways == 4) {
          const ulonglong2 lo = __ldcg(reinterpret_cast<const ulonglong2*>(bk[i]));
          const ulonglong2 hi = __ldcg(reinterpret_cast<const ulonglong2*>(bk[i] + 2));
          sn[0] = lo.x;
          sn[1] = lo.y;
          sn[2] = hi.x;
          sn[3] = hi.y;
        } else {
#pragma unroll
          for (u32 w = 0; w < 4; ++w) sn[w] = w < ways ? __ldcg(bk[i] + w) : kEmptyKey;
        }
        u32 p = 0;
        bool dup = false;
#pragma unroll
        for (u32 w = 0; w < 4; ++w) {
          dup |= (w < ways && sn[w] == key[i]);
          p += (w < ways && sn[w] < key[i]) ? 1u : 0u;
        }
        pos[i] = (dup || p >= ways) ? 4u : p;
        // the target's buffer may change: k_apply visits touched points only
        if (touched && pos[i] < ways) touched[key_tgt[i]] = 1;
      }
      // rounds: one independent atomicMin per live offer (pipelined), then
      // carry the larger of (old, key) to the next slot (the cascade above)
#pragma unroll
      for (int round = 0; round < 4; ++round) {
        u64 old[kOfferBatch];
#pragma unroll
        for (int i = 0; i < kOfferBatch; ++i)
          if (pos[i] < ways)
            old[i] = atomicMin(reinterpret_cast<unsigned long long*>(bk[i] + pos[i]),
                               (unsigned long long)key[i]);
#pragma unroll
        for (int i = 0; i < kOfferBatch; ++i) {
          if (pos[i] >= ways) continue;
          if (old[i] == key[i]) {
            pos[i] = 4;
            continue;
          }
          key[i] = old[i] > key[i] ? old[i] : key[i];
          pos[i] = key[i] == kEmptyKey ? 4u : pos[i] + 1;
        }
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// k_join
// ---------------------------------------------------------------------------
struct JoinArgs {
  const float* X;
  const float* nrm;  // cosine norm chains (null: l2)
  int d;
  const u32* L_ids;
  const u32* L_cnt;
  int RMAX;
  const float* worst;
  const u32* act;  // active point list (null: points p_lo..p_hi themselves)
  u64 p_lo, p_hi;
  const u64* n_live;  // device count bounding p_hi (null: none)
  u32* chunk_counter;
  u64* q_key;
  u32* q_tgt;
  u32* q_fill;
  u64 q_per_chunk;
  int DC, DCP, RB;
  u64* counters;
  // (-0.0f, -0.0f): the addend of the paired squares' FFMA2 (see sq_pairs);
  // a kernel argument, so ptxas cannot see it is a no-op addend
  unsigned long long negz2;
};

// Tiling of one point's pairs (nndescent.cpp:157-171: new x new with i < j,
// new x old).  The point's list (new entries, then old) is cut into blocks of
// 4 logical entries; block b of the list pairs with blocks b' >= b: a
// "trapezoid" of 4x4 micro-tiles over rows = the new blocks (RT of them) and
// columns = all blocks (CT), rt*ct - rt(rt-1)/2 tiles.  A pair (i, j) of
// logical entries is evaluated iff i < nn, j < na and j > i -- every new x new
// pair once (as i < j), every new x old pair once.  Merging the new and old
// column ranges leaves one padded column block per point (the separate
// triangle + rectangle of round 1 padded both, ~15% more tile slots).
// smem layout of a point: logical entry e = 4 blk + w sits at slot w*CT + blk,
// so micro-tile rows {4 ti + r} are slots ti + CT r and consecutive tiles of a
// thread row read consecutive smem rows (conflict-free LDS.128).
__device__ __forceinline__ int tiles_of(u32 cnt) {
  const int nn = cnt & 0xffff, na = cnt >> 16;
  const int rt = (nn + 3) >> 2, ct = (na + 3) >> 2;
  return (nn == 0 || na < 2) ? 0 : rt * ct - rt * (rt - 1) / 2;
}
// smem rows one point takes (4 CT, padding slots included)
__device__ __forceinline__ int slots_of(u32 cnt) { return (((int)(cnt >> 16) + 3) >> 2) * 4; }

// A 4x4 micro-tile of one point: rows = logical entries 4 ti + r (slots
// ti + CT r), columns = logical entries 4 tj + c (slots tj + CT c), tj >= ti.
struct Tile {
  int pt;          // point slot in the chunk (-1: none)
  int row0, rstr;  // batch smem row of row 0, stride
  int col0, cstr;  // batch smem row of column 0, stride
  int nn, na;
  int ti, tj;
};

// per meta slot (2): s_ids[G*RMAX] u32 | s_cnt[G] | s_pid[G] | hdr[4]
// (the worst snapshot is read from HBM/L2 per tile row and column: 4 MB at
// 1M points stays L2-resident, and the smem it would take buys ~70 more
// staged rows per batch, i.e. more tiles per CTA barrier)
// per desc slot (2): s_rb[G+1] | s_tb[G+1] | hdr[4]
// misc[16] | x[2][(RB+4)*DCP]
// Slots are addressed arithmetically (base + slot * stride) so nothing lands
// in local memory.
struct Smem {
  unsigned char* meta;  // slot m at meta + m * meta_bytes
  unsigned char* desc;  // slot q at desc + q * desc_bytes
  int* misc;            // [0..15] warp sums, [16] chunk grab
  float* x0;            // buffer b at x0 + b * xstride
  int RMAX;
  u32 meta_bytes, desc_bytes, xstride;
  __device__ u32* ids(int m) const { return reinterpret_cast<u32*>(meta + m * meta_bytes); }
  __device__ u32* cnt(int m) const {
    return reinterpret_cast<u32*>(meta + m * meta_bytes + G * RMAX * 4);
  }
  __device__ u32* pid(int m) const {
    return reinterpret_cast<u32*>(meta + m * meta_bytes + G * RMAX * 4 + G * 4);
  }
  __device__ int* mhdr(int m) const {  // [0] chunk, [1] np, [2] offers queued
    return reinterpret_cast<int*>(meta + m * meta_bytes + G * RMAX * 4 + G * 8);
  }
  __device__ int* rb(int q) const { return reinterpret_cast<int*>(desc + q * desc_bytes); }
  __device__ int* tb(int q) const { return rb(q) + (G + 1); }
  // [0] meta, [1] jb, [2] je, [3] first tile of point jb, [4] next point, [5] its first tile
  __device__ int* dhdr(int q) const { return rb(q) + 2 * (G + 1); }
  __device__ u32* rowid(int q) const { return reinterpret_cast<u32*>(rb(q) + 2 * (G + 1) + 8); }
  __device__ float* x(int b) const { return x0 + b * xstride; }
};

__host__ __device__ inline size_t desc_slot_bytes(int RB) {
  return ((size_t)(2 * (G + 1) + 8) * 4 + (size_t)RB * 4 + 15) & ~size_t(15);
}

__device__ __forceinline__ Smem carve(unsigned char* base, int RMAX, int RB, int DCP) {
  Smem s;
  s.RMAX = RMAX;
  s.meta_bytes = (u32)((size_t)G * RMAX * 4 + G * 8 + 16);
  s.desc_bytes = (u32)desc_slot_bytes(RB);
  s.meta = base;
  s.desc = base + 2 * s.meta_bytes;
  s.misc = reinterpret_cast<int*>(s.desc + 2 * s.desc_bytes);
  size_t off = 2 * (size_t)s.meta_bytes + 2 * (size_t)s.desc_bytes + 128;
  off = (off + 15) & ~size_t(15);
  s.x0 = reinterpret_cast<float*>(base + off);
  s.xstride = (u32)((RB + 4) * DCP);
  return s;
}

__host__ __device__ inline size_t join_smem_bytes(int RMAX, int RB, int DCP) {
  size_t off = 2 * ((size_t)G * RMAX * 4 + G * 8 + 16) + 2 * desc_slot_bytes(RB) + 128;
  off = (off + 15) & ~size_t(15);
  return off + 2 * (size_t)(RB + 4) * DCP * 4;
}

// Grab the next chunk into meta slot m; returns false when the slice is done.
__device__ bool load_chunk(const JoinArgs& a, const Smem& s, int m) {
  const int tid = threadIdx.x;
  __syncthreads();  // slot m is no longer read by anyone
  if (tid == 0) s.misc[16] = (int)atomicAdd(a.chunk_counter, 1u);
  __syncthreads();
  const u32 chunk = (u32)s.misc[16];
  u64 p_hi = a.p_hi;
  if (a.n_live) {
    const u64 live = *a.n_live;
    if (live < p_hi) p_hi = live;
  }
  const u64 p0 = a.p_lo + (u64)chunk * G;
  if (p0 >= p_hi) return false;
  const int np = (p_hi - p0) < (u64)G ? (int)(p_hi - p0) : G;
  if (tid < np) {
    const u32 pt = a.act ? a.act[p0 + tid] : (u32)(p0 + tid);
    s.pid(m)[tid] = pt;
    s.cnt(m)[tid] = a.L_cnt[pt];
  }
  __syncthreads();
  // warp per point, lane per list entry (no index division; empty slots skipped)
  for (int j = tid >> 5; j < np; j += kJT / 32) {
    const int na = (int)(s.cnt(m)[j] >> 16);
    const u32* src = a.L_ids + (u64)s.pid(m)[j] * a.RMAX;
    for (int i = tid & 31; i < na; i += 32) s.ids(m)[j * a.RMAX + i] = src[i];
  }
  if (tid == 0) {
    s.mhdr(m)[0] = (int)chunk;
    s.mhdr(m)[1] = np;
    s.mhdr(m)[2] = 0;  // offers queued for this chunk (shared atomic)
  }
  __syncthreads();
  return true;
}

// Warp 0 packs the tiles of meta slot m, starting at tile t0 of point jb,
// into desc slot q: whole points while rows fit, and the tile budget is filled
// exactly -- a point whose tiles do not all fit is split, the rest of it opens
// the next batch (its rows are staged in both; every tile is computed once).
// Lane l looks at point jb + l (a chunk has <= 32 points): inclusive warp
// scans of rows and tiles give the first point that overflows either budget
// -- the same cut as a serial walk, in log2(32) steps instead of a
// single-thread loop the other 255 threads wait for at the next barrier.
__device__ void form_batch(const JoinArgs& a, const Smem& s, int q, int m, int jb, int t0) {
  static_assert(G <= 32, "form_batch: one lane per chunk point");
  if (threadIdx.x >= 32) return;
  const unsigned lane = lane_id();
  const int np = s.mhdr(m)[1];
  const int j = jb + (int)lane;
  const bool live = j < np;
  const u32 c = live ? s.cnt(m)[j] : 0u;
  const int tt = live ? tiles_of(c) : 0;
  const int avail = tt - (lane == 0 ? t0 : 0);
  const int rows_j = tt ? slots_of(c) : 0;
  int R = rows_j, T = avail;  // inclusive prefix sums
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int r = __shfl_up_sync(kFull, R, o), t = __shfl_up_sync(kFull, T, o);
    if ((int)lane >= o) {
      R += r;
      T += t;
    }
  }
  // first overflowing point: rows (never the batch's first point) or tiles
  const unsigned rcut = __ballot_sync(kFull, live && lane > 0 && R > a.RB);
  const unsigned tcut = __ballot_sync(kFull, live && T > kMaxTiles);
  const int lr = rcut ? __ffs(rcut) - 1 : 32, lt = tcut ? __ffs(tcut) - 1 : 32;
  const int live_n = np - jb;
  int ncnt, jn, tn = 0, take = -1;
  if (lr <= lt) {  // rows full (or the chunk ends) before the tile budget
    ncnt = min(lr, live_n);
    jn = jb + ncnt;
  } else {          // tile budget: point lt is split (or excluded when nothing fits)
    const int before = __shfl_sync(kFull, T - avail, lt);  // tiles before point lt
    take = kMaxTiles - before;
    if (take <= 0) {
      ncnt = lt;
      jn = jb + lt;
    } else {
      ncnt = lt + 1;
      jn = jb + lt;
      tn = (lt == 0 ? t0 : 0) + take;
    }
  }
  // exclusive prefixes = the points' first row / tile in the batch
  const int Rx = R - rows_j, Tx = T - avail;
  if ((int)lane < ncnt) {
    s.rb(q)[j] = Rx;
    s.tb(q)[j] = Tx;
  }
  const int last = ncnt - 1;
  int rows_end = 0, tiles_end = 0;
  if (ncnt > 0) {
    rows_end = __shfl_sync(kFull, R, last);
    tiles_end = __shfl_sync(kFull, Tx, last) +
                (take > 0 && last == lt ? take : __shfl_sync(kFull, avail, last));
  }
  // list rows staged (padding slots excluded): the algorithmic rows
  int real = (int)lane < ncnt && tt ? (int)(c >> 16) : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) real += __shfl_xor_sync(kFull, real, o);
  if (lane == 0) {
    const int je = jb + ncnt;
    s.rb(q)[je] = rows_end;
    s.tb(q)[je] = tiles_end;
    s.dhdr(q)[0] = m;
    s.dhdr(q)[1] = jb;
    s.dhdr(q)[2] = je;
    s.dhdr(q)[3] = t0;
    s.dhdr(q)[4] = jn;
    s.dhdr(q)[5] = tn;
    s.dhdr(q)[6] = real;
  }
}

// Stage dims [c0, c0+dc) of every row of desc q into buffer buf (async).
// Row -> point id table of desc q (all threads; once per batch).  Row r
// belongs to the last point j with rb[j] <= r (zero-row points share rb).
template <bool kPair>
__device__ void fill_rowids(const JoinArgs& a, const Smem& s, int q) {
  const int m = s.dhdr(q)[0], jb = s.dhdr(q)[1], je = s.dhdr(q)[2];
  const int* rb = s.rb(q);
  const int rows = rb[je];
  u32* rowid = s.rowid(q);
  for (int r = threadIdx.x; r < rows; r += kJT) {
    int lo = jb, hi = je - 1;  // last j in [jb, je) with rb[j] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rb[mid] <= r) lo = mid; else hi = mid - 1;
    }
    // slot -> logical entry (slot = w * CT + blk holds entry 4 blk + w); the
    // padding slots of the last block stage the point's first row (unused)
    const u32 c = s.cnt(m)[lo];
    const int na = (int)(c >> 16), ct = (na + 3) >> 2;
    const int slot = r - rb[lo];
    int e;
    if (kPair) {  // slot = 2 pair-row + parity, pair-row = (w >> 1) CT + blk
      const int pr = slot >> 1, h = pr >= ct;
      e = (pr - h * ct) * 4 + 2 * h + (slot & 1);
    } else {
      e = (slot % ct) * 4 + slot / ct;
    }
    rowid[r] = s.ids(m)[lo * a.RMAX + (e < na ? e : 0)];
  }
}

// Stage dims [c0, c0+dc) of every row of desc q into buffer buf (async,
// one 16-byte cp.async per thread per step, all lanes busy).
template <bool kPair>
__device__ void issue_rows(const JoinArgs& a, const Smem& s, int q, int c0, int buf) {
  const int je = s.dhdr(q)[2];
  const int rows = s.rb(q)[je];
  const int dc = min(a.DC, a.d - c0);
  const u32* rowid = s.rowid(q);
  float* xb = s.x(buf);
  if (kPair) {
    // pair layout: slots 2i, 2i+1 share pair-row i (stride 2 DCP), their
    // values interleaved per dim.  Thread -> (pair-row, 4-dim quad): 8
    // four-byte cp.async fill 32 contiguous smem bytes from 16 B of each
    // row (one address computation per 8 elements; the quads of a warp
    // cover whole 128-B row segments, L1-cached across the 8 copies)
    const int qd = dc >> 2, ppi = kJT / qd;
    const int p0 = (int)threadIdx.x / qd, q4 = (int)threadIdx.x - p0 * qd;
    if (p0 < ppi) {
      const float* src = a.X + c0 + q4 * 4;
      float* dst = xb + q4 * 8;
      const uint2* rid2 = reinterpret_cast<const uint2*>(rowid);
      for (int pr = p0; pr < (rows >> 1); pr += ppi) {
        const uint2 id = rid2[pr];
        const float* s0 = src + (u64)id.x * (u64)a.d;
        const float* s1 = src + (u64)id.y * (u64)a.d;
        float* d0 = dst + pr * 2 * a.DCP;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          cp_async4(d0 + 2 * k, s0 + k);
          cp_async4(d0 + 2 * k + 1, s1 + k);
        }
      }
    }
  } else if ((a.d & 3) == 0) {
    // thread -> (row r0 + k * rpi, 16-byte piece c4): one division per call
    const int qd = dc >> 2, rpi = kJT / qd;
    const int r0 = (int)threadIdx.x / qd, c4 = (int)threadIdx.x - r0 * qd;
    if (r0 < rpi) {
      const float* src = a.X + c0 + c4 * 4;
      float* dst = xb + c4 * 4;
      for (int r = r0; r < rows; r += rpi)
        cp_async16(dst + r * a.DCP, src + (u64)rowid[r] * (u64)a.d);
    }
  } else {
    for (int e = threadIdx.x; e < rows * dc; e += kJT) {
      const int r = e / dc, cc = e - r * dc;
      xb[r * a.DCP + cc] = a.X[(u64)rowid[r] * a.d + c0 + cc];
    }
  }
  cp_async_commit();
}

template <bool kPair>
__device__ __forceinline__ Tile decode_tile(const Smem& s, int q, int t) {
  Tile T;
  const int m = s.dhdr(q)[0], jb = s.dhdr(q)[1], je = s.dhdr(q)[2];
  if (t >= s.tb(q)[je]) {
    T.pt = -1;
    return T;
  }
  int j = jb;
  while (j + 1 < je && s.tb(q)[j + 1] <= t) ++j;
  const u32 c = s.cnt(m)[j];
  const int nn = c & 0xffff, na = c >> 16;
  const int ct = (na + 3) >> 2;
  int lt = t - s.tb(q)[j] + (j == jb ? s.dhdr(q)[3] : 0);
  int ti = 0;  // row block ti owns the tiles tj = ti .. ct-1
  while (lt >= ct - ti) {
    lt -= ct - ti;
    ++ti;
  }
  T.pt = j;
  T.nn = nn;
  T.na = na;
  T.ti = ti;
  T.tj = ti + lt;
  // pair layout: row0 / col0 index pair-rows (entries 4 ti + {0,1} and
  // 4 ti + {2,3} sit in pair-rows ti and ct + ti of the point)
  const int base = kPair ? s.rb(q)[j] >> 1 : s.rb(q)[j];
  T.row0 = base + ti;
  T.col0 = base + T.tj;
  T.rstr = T.cstr = ct;
  return T;
}

// Two pairs at once, exact order: T = (b0 - a, b1 - a) with FADD2 (a
// broadcast; b - a is the exact negation of a - b, so squares are equal),
// P = T*T + (-0) with FFMA2 (x*y + -0 rounds once, = the rounded product),
// acc += P with FADD2 -- every pair still sums round(acc + round(t*t)) dim by
// dim.  A plain FMUL2 + FADD2 would be contracted into FFMA2 by ptxas (one
// rounding); the runtime -0 addend blocks that.  1.5 instructions per
// pair-dim instead of 2 (FADD2 sub + FMUL2 + two scalar FADDs per two dims).
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
template <bool kCos>
__device__ __forceinline__ void step_pairs(unsigned long long& acc, float a, float b0, float b1,
                                           unsigned long long negz2) {
  const unsigned long long A = pack2(a, a), B = pack2(b0, b1);
  unsigned long long P;
  if (kCos) {
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(P) : "l"(B), "l"(A), "l"(negz2));
  } else {
    unsigned long long T;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(T) : "l"(B), "l"(A));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(P) : "l"(T), "l"(negz2));
  }
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc) : "l"(acc), "l"(P));
}

template <bool kCos, bool kPair>
__global__ __launch_bounds__(kJT, kJCtas) void k_join(JoinArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Smem s = carve(smem, a.RMAX, a.RB, a.DCP);
  const int tid = threadIdx.x;
  const unsigned lane = lane_id();
  u64 my_pairs = 0, my_rows = 0, my_offers = 0;
  int pend_chunk = -1, pend_m = 0;  // chunk completed by the last batch (uniform)

  // prologue: first chunk, first batch, first dim chunk
  if (!load_chunk(a, s, 0)) return;
  int cq = 0, cc0 = 0, cbuf = 0;  // current unit: desc slot, dim offset, buffer
  form_batch(a, s, 0, 0, 0, 0);
  __syncthreads();
  fill_rowids<kPair>(a, s, 0);
  __syncthreads();
  issue_rows<kPair>(a, s, 0, 0, 0);

  Tile T[kTPT];
  float acc[kTPT][4][4];
  while (true) {
    // One barrier per unit: after it the current unit's rows have landed
    // (every thread waited for its own copies) and everyone is done with the
    // previous unit -- its buffer, and at a batch change its desc slot.  The
    // next unit's rows are then issued into that buffer while this one is
    // computed.
    cp_async_wait<0>();
    __syncthreads();
    if (pend_chunk >= 0) {
      // the chunk's offers are all queued (slot pend_m is reloaded only two
      // chunks later: its counter is final)
      if (tid == 0) {
        const u32 f = (u32)s.mhdr(pend_m)[2];
        a.q_fill[pend_chunk] = f;
        my_offers += f;
      }
      pend_chunk = -1;
    }
    // ---- next unit: next dim chunk of this batch, next batch, or next chunk
    int nq = cq, nc0 = cc0 + a.DC, nbuf = cbuf ^ 1;
    bool have_next = true;
    if (nc0 >= a.d) {
      nc0 = 0;
      nq = cq ^ 1;
      const int m = s.dhdr(cq)[0];
      const int jn = s.dhdr(cq)[4], tn = s.dhdr(cq)[5];
      if (jn < s.mhdr(m)[1]) {
        form_batch(a, s, nq, m, jn, tn);
      } else if (load_chunk(a, s, m ^ 1)) {
        form_batch(a, s, nq, m ^ 1, 0, 0);
      } else {
        have_next = false;
      }
      __syncthreads();
      if (have_next) {
        fill_rowids<kPair>(a, s, nq);
        __syncthreads();
      }
    }
    if (have_next) issue_rows<kPair>(a, s, nq, nc0, nbuf);

    // ---- compute the current unit
    const int m = s.dhdr(cq)[0];
    if (cc0 == 0) {
#pragma unroll
      for (int t = 0; t < kTPT; ++t) T[t] = decode_tile<kPair>(s, cq, tid + t * kJT);
#pragma unroll
      for (int t = 0; t < kTPT; ++t)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[t][r][c] = 0.0f;
      if (tid == 0) my_rows += (u64)s.dhdr(cq)[6];
    }
    if (kPair) {
      const float* xb = s.x(cbuf);
      const int dc = min(a.DC, a.d - cc0);  // a multiple of 4 (d % 4 == 0)
#pragma unroll
      for (int t = 0; t < kTPT; ++t) {
        if (T[t].pt < 0) continue;
        unsigned long long acc2[4][2];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 2; ++c) acc2[r][c] = pack2(acc[t][r][2 * c], acc[t][r][2 * c + 1]);
        // pair-rows: h = 0 holds entries {0,1} of the block, h = 1 entries {2,3}
        const float* pa[2];
        const float* pb[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          pa[h] = xb + (T[t].row0 + T[t].rstr * h) * 2 * a.DCP;
          pb[h] = xb + (T[t].col0 + T[t].cstr * h) * 2 * a.DCP;
        }
        // two dims per 16-B smem word: (e0[j], e1[j], e0[j+1], e1[j+1]) of
        // each pair-row; groups of 8 dims with immediate offsets off
        // pointers advanced once per group (dc is a multiple of 4)
        auto two_dims = [&](const float4 (&va)[2], const float4 (&vb)[2]) {
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const float4& A = va[r >> 1];
              const float av = j == 0 ? ((r & 1) ? A.y : A.x) : ((r & 1) ? A.w : A.z);
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                if (j == 0)
                  step_pairs<kCos>(acc2[r][c], av, vb[c].x, vb[c].y, a.negz2);
                else
                  step_pairs<kCos>(acc2[r][c], av, vb[c].z, vb[c].w, a.negz2);
              }
            }
        };
        const float *a0 = pa[0], *a1 = pa[1], *b0 = pb[0], *b1 = pb[1];
        const int dc8 = dc & ~7;
        for (int dd = 0; dd < dc8; dd += 8) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 va[2] = {*reinterpret_cast<const float4*>(a0 + 4 * u),
                                  *reinterpret_cast<const float4*>(a1 + 4 * u)};
            const float4 vb[2] = {*reinterpret_cast<const float4*>(b0 + 4 * u),
                                  *reinterpret_cast<const float4*>(b1 + 4 * u)};
            two_dims(va, vb);
          }
          a0 += 16;
          a1 += 16;
          b0 += 16;
          b1 += 16;
        }
        if (dc8 < dc) {  // 4 more dims
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const float4 va[2] = {*reinterpret_cast<const float4*>(a0 + 4 * u),
                                  *reinterpret_cast<const float4*>(a1 + 4 * u)};
            const float4 vb[2] = {*reinterpret_cast<const float4*>(b0 + 4 * u),
                                  *reinterpret_cast<const float4*>(b1 + 4 * u)};
            two_dims(va, vb);
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            asm("mov.b64 {%0,%1}, %2;" : "=f"(acc[t][r][2 * c]), "=f"(acc[t][r][2 * c + 1])
                : "l"(acc2[r][c]));
      }
    } else {
      const float* xb = s.x(cbuf);
      const int dc = min(a.DC, a.d - cc0);
      const int dc4 = dc & ~3;
#pragma unroll
      for (int t = 0; t < kTPT; ++t) {
        if (T[t].pt < 0) continue;
        const float* ra[4];
        const float* rb[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) ra[r] = xb + (T[t].row0 + T[t].rstr * r) * a.DCP;
#pragma unroll
        for (int c = 0; c < 4; ++c) rb[c] = xb + (T[t].col0 + T[t].cstr * c) * a.DCP;
#pragma unroll kJUnroll
        for (int dd = 0; dd < dc4; dd += 4) {
          float4 va[4], vb[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) va[r] = *reinterpret_cast<const float4*>(ra[r] + dd);
#pragma unroll
          for (int c = 0; c < 4; ++c) vb[c] = *reinterpret_cast<const float4*>(rb[c] + dd);
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[t][r][c] = m_step4<kCos>(acc[t][r][c], va[r], vb[c]);
        }
        for (int dd = dc4; dd < dc; ++dd) {
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              acc[t][r][c] = m_step<kCos>(acc[t][r][c], ra[r][dd], rb[c][dd]);
        }
      }
    }

    // ---- offers after the last dim chunk (nndescent.cpp:160-171)
    if (cc0 + a.DC >= a.d) {
      u32 pass_mask[kTPT];
      int my_q = 0;
#pragma unroll
      for (int t = 0; t < kTPT; ++t) {
        pass_mask[t] = 0;
        if (T[t].pt < 0) continue;
        const int lb = T[t].pt * a.RMAX;
        // ids, worst snapshots (and cosine norm chains) of the tile's 4 rows and 4 columns
        u32 rid[4], cid[4];
        float rw[4], cw[4], rn[4], cn[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int i = 4 * T[t].ti + q4, jj = 4 * T[t].tj + q4;
          rid[q4] = i < T[t].nn ? s.ids(m)[lb + i] : 0u;
          cid[q4] = jj < T[t].na ? s.ids(m)[lb + jj] : 0u;
          rw[q4] = i < T[t].nn ? __ldg(a.worst + rid[q4]) : 0.0f;
          cw[q4] = jj < T[t].na ? __ldg(a.worst + cid[q4]) : 0.0f;
          rn[q4] = kCos ? __ldg(a.nrm + rid[q4]) : 0.0f;
          cn[q4] = kCos ? __ldg(a.nrm + cid[q4]) : 0.0f;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int i = 4 * T[t].ti + r;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int jj = 4 * T[t].tj + c;
            const bool valid = i < T[t].nn && jj < T[t].na && jj > i;
            if (!valid) continue;
            const float dist = m_finish<kCos>(acc[t][r][c], rn[r], cn[c]);
            acc[t][r][c] = dist;
            ++my_pairs;
            const int bit = (r * 4 + c) * 2;
            if (dist < rw[r]) pass_mask[t] |= 1u << bit;
            if (dist < cw[c]) pass_mask[t] |= 2u << bit;
          }
        }
        my_q += __popc(pass_mask[t]);
      }
      // queue order is irrelevant (bucket inserts are order-independent):
      // each warp reserves one run of slots with a shared atomic, then every
      // (pair, direction) bit position is written by one ballot -- the
      // passing lanes store to consecutive slots (coalesced, branch-free)
      const u32 chunk = (u32)s.mhdr(m)[0];
      u64* qk = a.q_key + (u64)chunk * a.q_per_chunk;
      u32* qt = a.q_tgt + (u64)chunk * a.q_per_chunk;
      const int wq = __reduce_add_sync(kFull, (unsigned)my_q);
      u32 wbase = 0;
      if (lane == 0 && wq) wbase = (u32)atomicAdd(&s.mhdr(m)[2], wq);
      u32 slot = __shfl_sync(kFull, wbase, 0);
#pragma unroll
      for (int t = 0; t < kTPT; ++t) {
        const u32 pm = pass_mask[t];
        if (!__any_sync(kFull, pm != 0)) continue;
        const int lb = T[t].pt * a.RMAX;
#pragma unroll
        for (int rc = 0; rc < 16; ++rc) {
          const u32 two = (pm >> (rc * 2)) & 3u;
          if (!__any_sync(kFull, two != 0)) continue;
          const int r = rc >> 2, c = rc & 3;
          u32 u = 0, v = 0;
          float dist = 0.0f;
          if (two) {
            u = s.ids(m)[lb + 4 * T[t].ti + r];
            v = s.ids(m)[lb + 4 * T[t].tj + c];
            dist = acc[t][r][c];
          }
#pragma unroll
          for (int dir = 0; dir < 2; ++dir) {
            const bool on = (two >> dir) & 1u;
            const unsigned mb = __ballot_sync(kFull, on);
            if (on) {
              const u32 at = slot + __popc(mb & lanemask_lt());
              qk[at] = pack_key(dist, dir ? u : v);
              qt[at] = dir ? v : u;
            }
            slot += __popc(mb);
          }
        }
      }
      if (s.dhdr(cq)[4] >= s.mhdr(m)[1]) {  // chunk complete: fill after the barrier
        pend_chunk = (int)chunk;
        pend_m = m;
      }
    }
    if (!have_next) break;
    cq = nq;
    cc0 = nc0;
    cbuf = nbuf;
  }
  __syncthreads();
  if (pend_chunk >= 0 && tid == 0) {
    const u32 f = (u32)s.mhdr(pend_m)[2];
    a.q_fill[pend_chunk] = f;
    my_offers += f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_pairs += __shfl_xor_sync(kFull, my_pairs, o);
  if (lane == 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + kCntPairs), my_pairs);
  if (tid == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + kCntOffers), my_offers);
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + kCntStagedRows), my_rows);
  }
}

__global__ void k_active_flags(u64 n, const u32* __restrict__ L_cnt, u32* __restrict__ flag) {
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (u64)gridDim.x * blockDim.x)
    flag[p] = L_cnt[p] != 0;
}
__global__ void k_active_compact(u64 n, const u32* __restrict__ L_cnt, const u64* __restrict__ off,
                                 u32* __restrict__ act) {
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (u64)gridDim.x * blockDim.x)
    if (L_cnt[p]) act[off[p]] = (u32)p;
}

unsigned warp_grid(const Runner& r, u64 items) {
  const u64 want = ceil_div<u64>(items, 8);
  const u64 cap = (u64)r.num_sms * 16;
  return (unsigned)std::max<u64>(1, std::min(want, cap));
}

}  // namespace

JoinPlan plan_join(const Runner& r, int d, uint32_t k, uint32_t B) {
  JoinPlan p;
  const int max_rows = (int)(2 * B + k + B);
  p.RMAX = (max_rows + 3) & ~3;
  // Stage DC dims at a time (default 32); the exact-order accumulators carry
  // across the dim slices (registers), so the summation order is unchanged.
  // A narrower slice fits more rows (points) per batch: KNNG_JOIN_DC tunes it.
  int dc = 32;
  if (const char* v = std::getenv("KNNG_JOIN_DC")) dc = std::max(8, (std::atoi(v) + 7) & ~7);
  p.DC = d <= dc ? ((d + 7) & ~7) : dc;
  // pair layout (opt-in KNNG_JOIN_PAIR=1, d % 4 == 0): pair-row stride
  // 2 (DC + 2) floats = DC/2 + 1 16-B units, odd; else row stride DC + 4 =
  // DC/4 + 1 units, odd -- consecutive (pair-)rows are conflict-free for
  // LDS.128.  Measured on C2: join 102.8 ms vs 88.0 (the interleaving
  // 4-byte cp.async staging costs more than the 25% fewer math
  // instructions save; profiles/r02_join_pair.md)
  const char* pv = std::getenv("KNNG_JOIN_PAIR");
  p.pair = (d % 4 == 0) && pv && *pv && std::atoi(pv) != 0;
  p.DCP = p.pair ? p.DC + 2 : p.DC + 4;
  int smem_max = 0;
  KNNG_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, r.device));
  // largest RB whose footprint fits (2 feature buffers + 2 row-id tables)
  int rb = 1024;
  int smem_sm = 0;
  KNNG_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, r.device));
  // kJCtas CTAs must fit one SM (1 KB reserved per CTA)
  smem_max = std::min(smem_max, smem_sm / kJCtas - 1024);
  while (rb > 0 && join_smem_bytes(p.RMAX, rb, p.DCP) + 1024 > (size_t)smem_max) rb -= 8;
  // a point takes up to RMAX smem rows (its list, padded to whole 4-blocks)
  require(rb >= p.RMAX, "nn_descent: feature rows too wide for the join's smem batches");
  p.RB = rb;
  p.smem = join_smem_bytes(p.RMAX, p.RB, p.DCP);
  KNNG_CUDA(cudaFuncSetAttribute(k_join<false, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  KNNG_CUDA(cudaFuncSetAttribute(k_join<true, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  KNNG_CUDA(cudaFuncSetAttribute(k_join<false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  KNNG_CUDA(cudaFuncSetAttribute(k_join<true, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  int per_sm = 0;
  if (p.pair)
    KNNG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_join<false, true>, kJT,
                                                            p.smem));
  else
    KNNG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_join<false, false>, kJT,
                                                            p.smem));
  p.grid = (unsigned)r.num_sms * (unsigned)std::max(per_sm, 1);
  const uint64_t nn_max = 2ull * B, no_max = (uint64_t)k + B;
  const uint64_t max_offers_pp = 2 * (nn_max * (nn_max - 1) / 2 + nn_max * no_max);
  p.q_per_chunk = (uint64_t)G * max_offers_pp;
  return p;
}

void launch_join_lists(const Runner& r, uint64_t n, uint32_t k, uint32_t B, int RMAX,
                       const uint32_t* nf, const uint32_t* nfn, const uint32_t* of,
                       const uint32_t* ofn, const uint32_t* nr, const uint32_t* nrn,
                       const uint32_t* orv, const uint32_t* orn, uint32_t* L_ids,
                       uint32_t* L_cnt) {
  k_join_lists<<<warp_grid(r, n), 256, 0, r.stream>>>(n, k, B, RMAX, nf, nfn, of, ofn, nr, nrn,
                                                      orv, orn, L_ids, L_cnt);
  KNNG_LAUNCH_CHECK();
}

void build_active_list(const Runner& r, uint64_t n, const uint32_t* L_cnt, uint32_t* flag,
                       uint64_t* off, uint32_t* act) {
  const unsigned g = (unsigned)std::min<u64>(ceil_div<u64>(n ? n : 1, 256), (u64)r.num_sms * 16);
  k_active_flags<<<g, 256, 0, r.stream>>>(n, L_cnt, flag);
  KNNG_LAUNCH_CHECK();
  exclusive_scan_u32(r, flag, off, n);
  k_active_compact<<<g, 256, 0, r.stream>>>(n, L_cnt, off, act);
  KNNG_LAUNCH_CHECK();
}

void launch_join(const Runner& r, const JoinPlan& plan, const JoinLaunch& l) {
  JoinArgs a{};
  a.X = l.X;
  a.nrm = l.nrm;
  a.d = l.d;
  a.L_ids = l.L_ids;
  a.L_cnt = l.L_cnt;
  a.RMAX = plan.RMAX;
  a.worst = l.worst;
  a.act = l.act;
  a.p_lo = l.p_lo;
  a.p_hi = l.p_hi;
  a.n_live = l.n_live;
  a.chunk_counter = l.chunk_counter;
  a.q_key = l.q_key;
  a.q_tgt = l.q_tgt;
  a.q_fill = l.q_fill;
  a.q_per_chunk = plan.q_per_chunk;
  a.DC = plan.DC;
  a.DCP = plan.DCP;
  a.RB = plan.RB;
  a.counters = l.counters;
  a.negz2 = 0x8000000080000000ull;
  if (plan.pair) {
    if (a.nrm)
      k_join<true, true><<<plan.grid, kJT, plan.smem, r.stream>>>(a);
    else
      k_join<false, true><<<plan.grid, kJT, plan.smem, r.stream>>>(a);
  } else if (a.nrm) {
    k_join<true, false><<<plan.grid, kJT, plan.smem, r.stream>>>(a);
  } else {
    k_join<false, false><<<plan.grid, kJT, plan.smem, r.stream>>>(a);
  }
  KNNG_LAUNCH_CHECK();
}

void launch_offer(const Runner& r, const JoinPlan& plan, const uint64_t* q_key,
                  const uint32_t* q_tgt, const uint32_t* q_fill, uint32_t chunks,
                  uint64_t* slots, uint32_t S, uint32_t nb, uint32_t ways, uint64_t* counters,
                  uint64_t p_lo, const uint64_t* n_live, uint64_t n_points,
                  uint8_t* touched) {
  if (!chunks) return;
  const unsigned grid = (unsigned)std::min<uint64_t>(chunks, (uint64_t)r.num_sms * 8);
  // one pass by default: target-range passes with L2-resident bucket rows
  // (KNNG_OFFER_PASSES) measured slower on C2 -- 4 passes 71.8 ms, 8 passes
  // 115 ms per build vs 43.3 ms for one (profiles/r02_offer_passes.md)
  uint64_t passes = 1;
  if (const char* v = std::getenv("KNNG_OFFER_PASSES")) passes = std::max(1, std::atoi(v));
  if (passes > 64 || !n_points) passes = 1;
  const uint64_t per = (n_points + passes - 1) / passes;
  for (uint64_t b = 0; b < passes; ++b) {
    const u32 lo = (u32)std::min<uint64_t>(b * per, n_points);
    const u32 hi = (u32)std::min<uint64_t>((b + 1) * per, n_points);
    k_offer<<<grid, 256, 0, r.stream>>>(q_key, q_tgt, q_fill, plan.q_per_chunk, chunks, slots,
                                        S, nb, ways, counters, p_lo, n_live, lo,
                                        passes == 1 ? 0xffffffffu : hi, touched);
    KNNG_LAUNCH_CHECK();
  }
}

}  // namespace knng_b200
