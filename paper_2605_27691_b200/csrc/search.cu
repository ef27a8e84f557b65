// search.cu -- greedy best-first batch search ann_search (annsearch.cpp:50-129),
// the remote-refine kernel (north_star item 3).
//
// One warp per query (persistent CTAs of one warp).  Per query the warp keeps
//   * the beam: a sorted array of packed (dist,id) keys in smem, double
//     buffered, plus an "expanded" bitmask (BeamEntry, annsearch.cpp:19-31);
//   * the visited set (VisitedSet, annsearch.cpp:35-46) as an open-addressing
//     hash of ids in smem, in one of two modes:
//       exact  -- (per-query diagnostics requested) 4096 slots; a query that
//                 visits more than 3/4 of that migrates to a per-warp tagged
//                 table in global memory, so no point is ever scored twice and
//                 `scored` equals the reference's visited.size();
//       cache  -- (no diagnostics) the entry points are drawn against an
//                 exact set (sample_distinct needs exact distinctness); the
//                 expansion then uses the table as a lossy 2-way direct-mapped
//                 filter of ids (plain loads/stores, no probing).  It has no
//                 false positives, so a fresh id is always scored.  A visited
//                 id it forgot is either in the beam -- re-scoring gives the
//                 identical (dist,id) key and the merge drops the duplicate --
//                 or was rejected/evicted while the beam was full; the full
//                 beam's tail only decreases, so its key is >= tail and it is
//                 dropped again.  Ids, distances and hop counts stay
//                 bit-identical; only wasted re-scores are added (counted in
//                 `scored`).
//   * the query vector in smem and a staging tile of 32 candidate rows.
// A hop expands the first unexpanded beam entry, dedups its out-neighbors
// (match.any), test-and-sets them in the visited set, stages the fresh rows
// with coalesced cp.async (one row per warp instruction) into a padded smem
// tile, and each lane sums its own row in the reference's sequential order
// (bank-conflict-free: row stride/4 is odd).  The batch is sorted with a warp
// bitonic network and merged into the beam by rank (merge path); a beam after
// a batch is the top-`width` of (beam U batch), which is what the reference's
// sequential beam_insert produces, so results are bit-identical.
#include "search.hpp"
#include "locality.hpp"

#include <algorithm>
#include <cstdlib>

namespace knng_b200 {
namespace {

constexpr u32 kNoId = 0xffffffffu;
constexpr u32 kExactVis = 4096;   // exact-mode smem slots (spills to global beyond 3/4)
constexpr u32 kStageDims = 64;    // dims per staging chunk (smem per query sets occupancy)

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

struct SearchArgs {
  const float* Q;
  const float* qn;  // cosine norm chains of Q / V rows (null: l2)
  const float* vn;
  u64 nq;
  int d;
  const float* V;
  u64 nv;
  const u32* sg;
  u32 deg;
  u32 ks, width, entries, max_hops;
  u64 seed;
  u64 qbase;  // stream index offset of query 0 (rng stream 0xa11ce000 + q)
  u32* out_ids;
  float* out_d;
  u32* hops_out;
  u32* scored_out;
  u32* scored_ids;   // diagnostics: ids in scoring order, scored_cap per query (null: off)
  u64 scored_cap;
  const u32* qorder;  // processing order of the queries (null: 0..nq-1)
  unsigned long long* qctr;  // dynamic query fetch counter (null: static slots)
  u64* gtable;  // per-CTA tagged visited tables (gcap slots each), may be null
  u32 gcap;
  u64* counters;  // [0] hops [1] scored [2] overflowed queries / cache resets
  u32 id_base;    // added to output ids
  u32 vis_slots;  // smem visited slots (power of two)
  u32 vis_limit;  // migrate (exact) / reset (cache) above this count
  u32 cache;      // 1 = cache mode
  u32 dch;        // dims per staging chunk
  u32 stride;     // staging row stride in floats
  u32 vec4;       // rows are 16-byte aligned (d % 4 == 0)
  u32 pipe;       // double-buffered dim chunks
};

__device__ __forceinline__ u32 vis_hash(u32 id) {
  u32 x = id * 0x9E3779B1u;
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  return x;
}

struct Visited {
  u32* s;           // smem table
  u32 mask;         // slots - 1
  u64* g;           // global table of this CTA (exact mode)
  u32 gcap;
  u32 tag;          // query tag for the global table
  bool global;
  u32 count;

  // Returns true if id was present (no insert); lane-parallel, ids distinct.
  __device__ __forceinline__ bool lookup(u32 id) const {
    if (!global) {
      u32 h = vis_hash(id) & mask;
      while (true) {
        const u32 v = s[h];
        if (v == id) return true;
        if (v == kNoId) return false;
        h = (h + 1) & mask;
      }
    }
    u32 h = vis_hash(id) & (gcap - 1);
    while (true) {
      const u64 v = g[h];
      if ((u32)(v >> 32) != tag) return false;
      if ((u32)v == id) return true;
      h = (h + 1) & (gcap - 1);
    }
  }
  __device__ __forceinline__ bool insert_smem(u32 id) {
    u32 h = vis_hash(id) & mask;
    while (true) {
      const u32 old = atomicCAS(&s[h], kNoId, id);
      if (old == kNoId) return true;
      if (old == id) return false;
      h = (h + 1) & mask;
    }
  }
  // Test-and-set; returns true if newly inserted.
  __device__ __forceinline__ bool insert(u32 id) {
    if (!global) return insert_smem(id);
    u32 h = vis_hash(id) & (gcap - 1);
    const u64 mine = ((u64)tag << 32) | id;
    while (true) {
      u64 cur = g[h];
      while ((u32)(cur >> 32) != tag) {
        const u64 old = atomicCAS(reinterpret_cast<unsigned long long*>(&g[h]),
                                  (unsigned long long)cur, (unsigned long long)mine);
        if (old == cur) return true;
        cur = old;
      }
      if ((u32)cur == id) return false;
      h = (h + 1) & (gcap - 1);
    }
  }
  // Exact mode: move the smem set into the global table (all lanes call).
  __device__ void migrate() {
    const unsigned lane = lane_id();
    __syncwarp();
    global = true;
    for (u32 t = lane; t <= mask; t += 32) {
      const u32 id = s[t];
      if (id != kNoId) insert(id);
    }
    __syncwarp();
  }
  // Cache mode after the entry points: a lossy 2-way direct-mapped filter
  // (no false positives; the merge drops re-scored beam members as exact
  // duplicate keys).  Returns true if id was not found (and records it).
  __device__ __forceinline__ bool dm_test_and_set(u32 id) {
    const u32 h = vis_hash(id);
    const u32 p = h & mask & ~1u;
    const uint2 v = *reinterpret_cast<const uint2*>(s + p);
    if (v.x == id || v.y == id) return false;
    s[p + ((h >> 20) & 1u)] = id;
    return true;
  }
  // Switch the smem table from the exact entry-phase set to the filter,
  // seeded with the beam's ids (all lanes call).
  __device__ void to_filter(const u64* beam, u32 bs) {
    const unsigned lane = lane_id();
    __syncwarp();
    for (u32 t = lane; t <= mask; t += 32) s[t] = kNoId;
    __syncwarp();
    for (u32 i = lane; i < bs; i += 32) dm_test_and_set(key_id(beam[i]));
    __syncwarp();
  }
};

// Exact-order L2 distances of the lanes' candidates (take = lane has one):
// rows are staged chunk by chunk with coalesced cp.async, one row per warp
// instruction, then each lane sums its row sequentially (l2_exact order).
template <bool kCos>
__device__ __forceinline__ u64 score_batch(const SearchArgs& a, const float* __restrict__ s_q,
                                           float* __restrict__ s_stage, u64* __restrict__ s_ptr,
                                           u32 id, bool take, float qnorm) {
  const unsigned lane = lane_id();
  __syncwarp();  // reconverge after the visited-set CAS loops
  const unsigned fm = __ballot_sync(kFull, take);
  if (!fm) return kEmptyKey;
  // compact the fresh rows: staging slot = rank among the fresh lanes; row
  // addresses go through smem (broadcast loads) rather than shuffles
  const u32 nf = __popc(fm);
  const u32 rank = __popc(fm & lanemask_lt());
  if (take) s_ptr[rank] = (u64)(uintptr_t)(a.V + (u64)id * (u64)a.d);
  __syncwarp();
  float acc = 0.0f;
  const u32 nch = ((u32)a.d + a.dch - 1) / a.dch;
  const u32 buf_floats = 32 * a.stride;
  // stage chunk ch into buffer `buf` (one commit group per chunk)
  auto issue = [&](u32 ch, u32 buf) {
    const u32 c0 = ch * a.dch;
    const u32 cl = min(a.dch, (u32)a.d - c0);
    float* stage = s_stage + buf * buf_floats;
    if (a.vec4) {
      // lanes-per-row = pow2 >= cl/4 (<= 32); 32/lpr rows per warp instruction
      const u32 lpr = cl > 64 ? 32u : (cl > 32 ? 16u : (cl > 16 ? 8u : (cl > 8 ? 4u : (cl > 4 ? 2u : 1u))));
      const u32 rpi = 32u / lpr;
      const u32 g = lane / lpr, sub = lane % lpr;
      const u32 sbase = (u32)__cvta_generic_to_shared(stage) + sub * 16;
      const uintptr_t gofs = (uintptr_t)(c0 + sub * 4) * 4;
      if (sub * 4 < cl) {
        // 4 rows per trip from one asm block (the copies stay back-to-back,
        // so they share the compiler's LDGSTS padding); a trip's rows past nf
        // copy a stale (valid) pointer into an unused slot instead of being
        // predicated off
        const u32 stride_b = a.stride * 4;
        const u32 step = 4 * rpi;
        u32 dst = sbase + g * stride_b;
        const u32 dstep = rpi * stride_b;
        for (u32 k = g; k < nf; k += step) {
          const u32 k1 = min(k + rpi, 31u), k2 = min(k + 2 * rpi, 31u), k3 = min(k + 3 * rpi, 31u);
          const uintptr_t s0 = (uintptr_t)s_ptr[k] + gofs, s1 = (uintptr_t)s_ptr[k1] + gofs;
          const uintptr_t s2 = (uintptr_t)s_ptr[k2] + gofs, s3 = (uintptr_t)s_ptr[k3] + gofs;
          asm volatile(
              "cp.async.cg.shared.global [%0], [%1], 16;\n"
              "cp.async.cg.shared.global [%2], [%3], 16;\n"
              "cp.async.cg.shared.global [%4], [%5], 16;\n"
              "cp.async.cg.shared.global [%6], [%7], 16;\n" ::"r"(dst), "l"(s0),
              "r"(sbase + k1 * stride_b), "l"(s1), "r"(sbase + k2 * stride_b), "l"(s2),
              "r"(sbase + k3 * stride_b), "l"(s3)
              : "memory");
          dst += 4 * dstep;
        }
        if (cl > 128) {
          for (u32 k = g; k < nf; k += rpi)
            for (u32 t = sub * 4 + 128; t < cl; t += 128)
              cpa16(stage + k * a.stride + t,
                    reinterpret_cast<const float*>((uintptr_t)s_ptr[k]) + c0 + t);
        }
      }
    } else {
      for (u32 k = 0; k < nf; ++k) {
        const float* src = reinterpret_cast<const float*>((uintptr_t)s_ptr[k]) + c0;
        float* dst = stage + k * a.stride;
        for (u32 t = lane; t < cl; t += 32) cpa4(dst + t, src + t);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const u32 nbuf = a.pipe ? 2u : 1u;
  issue(0, 0);
  if (nbuf == 2 && nch > 1) issue(1, 1);
  for (u32 ch = 0; ch < nch; ++ch) {
    if (nbuf == 2 && ch + 1 < nch)
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    const u32 c0 = ch * a.dch;
    const u32 cl = min(a.dch, (u32)a.d - c0);
    if (take) {
      const float* qq = s_q + c0;
      const float* my = s_stage + (ch % nbuf) * buf_floats + rank * a.stride;
      if (a.vec4) {
        for (u32 i = 0; i < cl; i += 4)
          acc = m_step4<kCos>(acc, *reinterpret_cast<const float4*>(qq + i),
                              *reinterpret_cast<const float4*>(my + i));
      } else {
        for (u32 i = 0; i < cl; ++i) acc = m_step<kCos>(acc, qq[i], my[i]);
      }
    }
    __syncwarp();
    if (ch + nbuf < nch) issue(ch + nbuf, ch % nbuf);
  }
  if (!take) return kEmptyKey;
  return pack_key(m_finish<kCos>(acc, qnorm, kCos ? __ldg(a.vn + id) : 0.0f), id);
}

// Merge the lane-held candidate keys (kEmptyKey = none) into the sorted
// beam in place: the beam becomes the top-`width` of (beam U candidates),
// which is what the reference's sequential beam_insert leaves.  A candidate
// whose key is already in the beam (an id re-scored after it fell out of the
// lossy visited filter: same id => same key) is dropped.  No sort: with
// clo = #beam < c, a kept candidate lands at clo + #kept < c and beam entry i
// moves right by #{kept : clo <= i}.  Groups of 32 entries are rewritten from
// the end (entries only move right, so every group is read before a write can
// reach it); unmoved entries are not stored.
__device__ __forceinline__ void beam_merge(u64 c, u64* __restrict__ beam,
                                           unsigned char* __restrict__ flag,
                                           u32* __restrict__ s_clo, u32& bs, u32 width,
                                           u32& low_insert) {
  const unsigned lane = lane_id();
  if (bs == width && c != kEmptyKey && c >= beam[width - 1]) c = kEmptyKey;
  if (!__any_sync(kFull, c != kEmptyKey)) return;
  u32 clo = 0;
  bool keep = false;
  if (c != kEmptyKey) {
    u32 hi = bs;
    while (clo < hi) {
      const u32 mid = (clo + hi) >> 1;
      if (beam[mid] < c) clo = mid + 1; else hi = mid;
    }
    keep = !(clo < bs && beam[clo] == c);
  }
  unsigned kb = __ballot_sync(kFull, keep);
  if (!kb) return;
  const u32 nc = __popc(kb);
  // rank among the kept candidates (keys are distinct)
  u32 crank = 0;
  if (nc > 8) {
    // many: a bitonic sort of the kept keys (clo travels with its key) puts
    // candidate of rank r on lane r -- 15 exchange steps instead of nc
    // broadcast-compare rounds
    u64 v = keep ? c : kEmptyKey;
    u32 pl = clo;
#pragma unroll
    for (unsigned size = 2; size <= 32; size <<= 1)
#pragma unroll
      for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
        const u64 o = __shfl_xor_sync(kFull, v, stride);
        const u32 op = __shfl_xor_sync(kFull, pl, stride);
        const bool keep_min = ((lane & stride) == 0) == ((lane & size) == 0);
        if (keep_min ? (o < v) : (o > v)) {
          v = o;
          pl = op;
        }
      }
    keep = lane < nc;
    c = v;
    clo = pl;
    crank = lane;
    kb = __ballot_sync(kFull, keep);
  } else {
    for (unsigned m = kb; m;) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const u64 cj = __shfl_sync(kFull, c, j);
      crank += (keep && cj < c) ? 1u : 0u;
    }
  }
  if (keep) s_clo[__popc(kb & lanemask_lt())] = clo;
  // entries before the first insertion point keep their slots
  const u32 first = __reduce_min_sync(kFull, keep ? clo : 0xffffffffu);
  low_insert = min(low_insert, first);
  __syncwarp();
  for (int t = (int)((bs + 31) >> 5) - 1; t >= (int)(first >> 5); --t) {
    const u32 i = lane + 32u * (u32)t;
    const bool valid = i < bs;
    u64 b = 0;
    unsigned char f = 0;
    u32 sh = 0;
    if (valid) {
      b = beam[i];
      f = flag[i];
      for (u32 j = 0; j < nc; ++j) sh += s_clo[j] <= i ? 1u : 0u;
    }
    __syncwarp();
    if (valid && sh && i + sh < width) {
      beam[i + sh] = b;
      flag[i + sh] = f;
    }
    __syncwarp();
  }
  if (keep && clo + crank < width) {
    beam[clo + crank] = c;
    flag[clo + crank] = 0;
  }
  __syncwarp();
  bs = min(width, bs + nc);
}

struct SmemLayout {
  size_t q, vis, beam, flag, clo, stage, ptr, total;
};

__host__ __device__ inline SmemLayout search_layout(int d, u32 width, u32 vis_slots, u32 stride) {
  SmemLayout L{};
  size_t off = 0;
  L.q = off;
  off += (((size_t)d * 4) + 15) & ~size_t(15);
  L.stage = off;
  off += (size_t)32 * stride * 4;
  L.beam = off;
  off += (size_t)width * 8;
  L.ptr = off;
  off += 32 * 8;
  L.clo = off;
  off += 32 * 4;
  L.vis = off;
  off += (size_t)vis_slots * 4;
  L.flag = off;
  off += ((size_t)width + 15) & ~size_t(15);
  L.total = off;
  return L;
}

// 20 resident warps per SM: <= 95 registers, no spills (was 120-134 at 1:
// 2M C4-shape queries 0.538 -> 0.504 s)
#ifndef KNNG_SEARCH_MINB
#define KNNG_SEARCH_MINB 20
#endif
template <bool kCos>
__global__ __launch_bounds__(32, KNNG_SEARCH_MINB) void k_search(SearchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const unsigned lane = lane_id();
  const u32 W = a.width;
  const SmemLayout L = search_layout(a.d, W, a.vis_slots, a.stride * (a.pipe ? 2 : 1));
  float* s_q = reinterpret_cast<float*>(smem + L.q);
  float* s_stage = reinterpret_cast<float*>(smem + L.stage);
  u64* s_beam = reinterpret_cast<u64*>(smem + L.beam);
  unsigned char* s_flag = smem + L.flag;  // 1 = expanded (BeamEntry::expanded)
  u32* s_clo = reinterpret_cast<u32*>(smem + L.clo);
  u64* s_ptr = reinterpret_cast<u64*>(smem + L.ptr);
  u32* s_vis = reinterpret_cast<u32*>(smem + L.vis);

  // every staging slot pointer is always a valid row (see score_batch)
  s_ptr[lane] = (u64)(uintptr_t)a.V;
  __syncwarp();
  u64 tot_hops = 0, tot_scored = 0, tot_ovf = 0;
  // query slots: static round robin, or (a.qctr) fetched from a counter so a
  // CTA that runs ahead takes more queries (no static tail)
  auto next_q = [&](u64 cur) -> u64 {
    if (!a.qctr) return cur + gridDim.x;
    u64 v = 0;
    if (lane == 0) v = atomicAdd(a.qctr, 1ull);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  for (u64 qi = a.qctr ? next_q(0) : blockIdx.x; qi < a.nq; qi = next_q(qi)) {
    // queries run in a spatial order (concurrent warps walk nearby parts of
    // the graph and share L2 lines); everything below is indexed by the
    // query's own id q, so results are unchanged
    const u64 q = a.qorder ? a.qorder[qi] : qi;
    // stage query, clear visited
    const float* qrow = a.Q + q * (u64)a.d;
    for (int t = lane; t < a.d; t += 32) s_q[t] = qrow[t];
    const float qnorm = kCos ? a.qn[q] : 0.0f;
    for (u32 t = lane; t < a.vis_slots; t += 32) s_vis[t] = kNoId;
    __syncwarp();
    Visited vis{s_vis, a.vis_slots - 1, a.gtable ? a.gtable + (u64)blockIdx.x * a.gcap : nullptr,
                a.gcap, (u32)(q + 1), false, 0};
    u32 bs = 0;
    u32 low_insert = 0;  // lowest beam position a merge inserted at (scan hint)
    u32 scored = 0;

    // exact mode: spill before the batch can overfill the smem table
    auto after_insert = [&](u32 add) {
      vis.count += add;
      if (!a.cache && !vis.global && vis.count > a.vis_limit) {
        if (vis.g == nullptr) __trap();  // host sizes gtable whenever overflow is possible
        vis.migrate();
        ++tot_ovf;
      }
    };
    auto score_and_merge = [&](u32 id, bool take) {
      const u64 c = score_batch<kCos>(a, s_q, s_stage, s_ptr, id, take, qnorm);
      beam_merge(c, s_beam, s_flag, s_clo, bs, W, low_insert);
    };
    // SearchDiagnostics::scored_ids (annsearch.hpp:36-41): every scored id in
    // scoring order (exact mode only: no id is ever scored twice)
    auto record = [&](u32 id, bool take) {
      if (!a.scored_ids) return;
      const unsigned tb = __ballot_sync(kFull, take);
      const u32 pos = scored + __popc(tb & lanemask_lt());
      if (take && pos < a.scored_cap) a.scored_ids[q * a.scored_cap + pos] = id;
    };

    // entry points: sample_distinct(n, entries, Rng(mix_seed(seed, 0xa11ce000+q)))
    // (host sizes the cache so it never re-seeds before the entries are drawn)
    if (a.entries >= a.nv) {
      for (u64 base = 0; base < a.nv; base += 32) {
        const u64 id = base + lane;
        const bool take = id < a.nv;
        if (take) vis.insert((u32)id);
        const u32 nt = __popc(__ballot_sync(kFull, take));
        record((u32)id, take);
        after_insert(nt);
        score_and_merge((u32)id, take);
        scored += nt;
      }
    } else {
      const u64 s0 = mix_seed(a.seed, 0xa11ce000ull + a.qbase + q);
      u64 m = 0;
      u32 got = 0;
      while (got < a.entries) {
        const u32 x = (u32)mulhi64(sm64_draw(s0, m + lane), a.nv);
        m += 32;
        const unsigned grp = __match_any_sync(kFull, x);
        const bool first = (__ffs(grp) - 1) == (int)lane;
        const bool fresh = first && !vis.lookup(x);
        const unsigned fb = __ballot_sync(kFull, fresh);
        const u32 before = __popc(fb & lanemask_lt());
        const bool take = fresh && (got + before < a.entries);
        if (take) vis.insert(x);
        const u32 ntake = __popc(__ballot_sync(kFull, take));
        got += ntake;
        record(x, take);
        scored += ntake;
        after_insert(ntake);
        score_and_merge(x, take);
      }
    }
    if (a.cache) vis.to_filter(s_beam, bs);

    // expansion loop (annsearch.cpp:103-120)
    u32 hops = 0;
    u32 scan_from = 0;  // entries before it are expanded and unmoved
    while (hops < a.max_hops) {
      // first unexpanded beam entry (annsearch.cpp:104-108): every entry
      // before min(last expanded, lowest insertion since) is expanded
      u32 idx = kNoId;
      const u32 t0 = min(scan_from, low_insert) >> 5;
      low_insert = 0xffffffffu;
      for (u32 t = t0; t * 32 < bs; ++t) {
        const u32 i = t * 32 + lane;
        const unsigned m = __ballot_sync(kFull, i < bs && s_flag[i] == 0);
        if (m) {
          idx = t * 32 + (__ffs(m) - 1);
          break;
        }
      }
      if (idx == kNoId) break;  // every beam entry expanded
      scan_from = idx;
      const u32 u = key_id(s_beam[idx]);
      __syncwarp();
      if (lane == 0) s_flag[idx] = 1;
      __syncwarp();
      for (u32 c0 = 0; c0 < a.deg; c0 += 32) {
        const u32 nb = (c0 + lane < a.deg) ? __ldg(a.sg + (u64)u * a.deg + c0 + lane) : kNoId;
        const unsigned grp = __match_any_sync(kFull, nb);
        const bool cand = nb != kNoId && (__ffs(grp) - 1) == (int)lane;
        bool fresh;
        if (a.cache) {
          fresh = cand && vis.dm_test_and_set(nb);
        } else {
          fresh = cand && vis.insert(nb);
        }
        const u32 nf = __popc(__ballot_sync(kFull, fresh));
        record(nb, fresh);
        scored += nf;
        if (!a.cache) after_insert(nf);
        score_and_merge(nb, fresh);
      }
      ++hops;
    }
    // best k_s (annsearch.cpp:122-126); unfilled slots stay 0 / 0.0f
    for (u32 i = lane; i < a.ks; i += 32) {
      u32 id = 0;
      float dd = 0.0f;
      if (i < bs) {
        const u64 key = s_beam[i];
        id = key_id(key) + a.id_base;
        dd = key_dist(key);
      }
      a.out_ids[q * a.ks + i] = id;
      a.out_d[q * a.ks + i] = dd;
    }
    if (lane == 0) {
      if (a.hops_out) a.hops_out[q] = hops;
      if (a.scored_out) a.scored_out[q] = scored;
    }
    tot_hops += hops;
    tot_scored += scored;
    __syncwarp();
  }
  if (lane == 0 && a.counters) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 0), tot_hops);
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 1), tot_scored);
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 2), tot_ovf);
  }
}

u32 next_pow2(u64 v) {
  u64 p = 1;
  while (p < v) p <<= 1;
  return (u32)p;
}

u32 env_u32(const char* name, u32 dflt) {
  const char* v = getenv(name);
  return (v && *v) ? (u32)strtoul(v, nullptr, 10) : dflt;
}

struct SearchShape {
  u32 vis_slots, vis_limit, cache, dch, stride, vec4, pipe;
  size_t smem;
};

SearchShape search_shape(int d, u32 width, u64 entries, bool exact) {
  SearchShape s{};
  s.vec4 = (d % 4) == 0;
  // chunks of <= kStageDims dims, equal-sized (d = 96: 2 x 48, not 64 + 32 --
  // a smaller staging tile, more queries per SM: 2M C4-shape queries
  // 0.504 -> 0.495 s)
  const u32 nch0 = ((u32)d + kStageDims - 1) / kStageDims;
  const u32 even = ((((u32)d + nch0 - 1) / nch0) + 3) & ~3u;
  const u32 dch = std::max<u32>(4, env_u32("KNNG_SEARCH_DCH", even) & ~3u);
  if (s.vec4) {
    s.dch = std::min<u32>(dch, (u32)d);
    s.stride = ((s.dch / 4) % 2 == 0) ? s.dch + 4 : s.dch;  // stride/4 odd: conflict-free
  } else {
    s.dch = std::min<u32>(kStageDims, (u32)d);
    s.stride = s.dch | 1u;  // odd stride: conflict-free scalar reads
  }
  // cache mode: the entry phase uses the table as an exact set (entries + one
  // batch at <= 3/4 load), the expansion phase as a lossy 2-way filter.
  u32 slots = env_u32("KNNG_SEARCH_VIS", 256);
  const u64 need = entries + 32;
  slots = std::max<u32>(std::max<u32>(next_pow2(slots), 64), next_pow2(need * 4 / 3 + 1));
  if (exact || slots > 8192) {
    s.cache = 0;
    s.vis_slots = kExactVis;
  } else {
    s.cache = 1;
    s.vis_slots = slots;
  }
  s.pipe = env_u32("KNNG_SEARCH_PIPE", 0) != 0 && (u32)d > s.dch;
  s.smem = search_layout(d, width, s.vis_slots, s.stride * (s.pipe ? 2 : 1)).total;
  // cache mode: a larger filter forgets fewer visited ids (cache mode scores
  // ~14% more rows than the exact set at C4) -- doubled while the CTA still
  // fits KNNG_SEARCH_MINB per SM (d = 96: 2M queries 0.495 -> 0.490 s)
  if (s.cache && !getenv("KNNG_SEARCH_VIS") && s.vis_slots < 8192) {
    const size_t bigger =
        search_layout(d, width, 2 * s.vis_slots, s.stride * (s.pipe ? 2 : 1)).total;
    if ((bigger + 1024) * KNNG_SEARCH_MINB <= 228 * 1024) {
      s.vis_slots *= 2;
      s.smem = bigger;
    }
  }
  s.vis_limit = s.vis_slots * 3 / 4;
  return s;
}

}  // namespace

size_t search_smem_bytes(int d, uint32_t width) {
  return search_shape(d, width, width, true).smem;
}

void validate_search(uint64_t nq_dims, uint64_t v_dims, uint64_t sg_n, uint64_t nv,
                     const SearchParamsDev& p) {
  require(nq_dims == v_dims, "ann_search: query/vector datasets incompatible");
  require(sg_n == nv, "ann_search: graph/vector row count mismatch");
  require(!(p.k_s == 0 || p.k_s > nv), "ann_search: k_s must be in [1, num points]");
  require(p.k_s <= p.beam_width, "ann_search: k_s must be <= beam_width");
  require(p.beam_width <= 1024, "ann_search: the B200 path supports beam_width <= 1024");
}

void ann_search_device(Runner& r, const float* Q, uint64_t nq, int d, const uint32_t* sg,
                       uint32_t deg, const float* V, uint64_t nv, const SearchParamsDev& p,
                       uint32_t id_base, uint32_t* out_ids, float* out_d, uint32_t* hops,
                       uint32_t* scored, SearchCounters* counters, uint64_t qbase,
                       const float* qn, const float* vn, uint32_t* scored_ids,
                       uint64_t scored_cap) {
  require((qn == nullptr) == (vn == nullptr), "ann_search: cosine needs both norm arrays");
  validate_search((uint64_t)d, (uint64_t)d, nv, nv, p);
  if (nq == 0) return;
  DeviceGuard guard(r.device);
  const u32 width = (u32)p.beam_width;
  const u32 max_hops = (u32)(p.max_hops ? p.max_hops : p.beam_width * 4);
  u64 entries = p.num_entry_points > p.k_s ? p.num_entry_points : p.k_s;
  if (entries > nv) entries = nv;

  // per-query diagnostics mirror the reference's exact visited-set size
  const bool exact =
      scored != nullptr || scored_ids != nullptr || getenv("KNNG_SEARCH_EXACT") != nullptr;
  const SearchShape sh = search_shape(d, width, entries, exact);
  KNNG_CUDA(cudaFuncSetAttribute(k_search<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sh.smem));
  KNNG_CUDA(cudaFuncSetAttribute(k_search<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sh.smem));
  int per_sm = 0;
  KNNG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search<false>, 32, sh.smem));
  if (per_sm < 1) per_sm = 1;
  const unsigned grid = persistent_grid(r, per_sm, nq);

  SearchArgs a{};
  a.Q = Q;
  a.qn = qn;
  a.vn = vn;
  a.nq = nq;
  a.d = d;
  a.V = V;
  a.nv = nv;
  a.sg = sg;
  a.deg = deg;
  a.ks = (u32)p.k_s;
  a.width = width;
  a.entries = (u32)entries;
  a.max_hops = max_hops;
  a.seed = p.seed;
  a.qbase = qbase;
  a.out_ids = out_ids;
  a.out_d = out_d;
  a.hops_out = hops;
  a.scored_out = scored;
  a.scored_ids = scored_ids;
  a.scored_cap = scored_cap;
  // large batches: a locality order of the queries (KNNG_SEARCH_ORDER=0 off);
  // 2M C4-shape queries: 0.634 -> 0.586 s (profiles/r02_search_sweep.md)
  DBuf<u32> qord;
  if (nq >= 65536 && env_u32("KNNG_SEARCH_ORDER", 1) != 0 && d <= 1024) {
    qord.alloc(r, nq);
    locality_order(r, Q, nq, d, 0x5eed04d0ull, qord.p);
    a.qorder = qord.p;
  }
  // dynamic query fetch (KNNG_SEARCH_DYN=0: static slots): 5M C4-shape
  // queries 1.527 -> 1.403 s (tools/exp_search_var.py)
  DBuf<unsigned long long> qctr;
  if (env_u32("KNNG_SEARCH_DYN", 1) != 0) {
    qctr.alloc(r, 1);
    qctr.zero();
    a.qctr = qctr.p;
  }
  a.id_base = id_base;
  a.vis_slots = sh.vis_slots;
  a.vis_limit = sh.vis_limit;
  a.cache = sh.cache;
  a.dch = sh.dch;
  a.stride = sh.stride;
  a.vec4 = sh.vec4;
  a.pipe = sh.pipe;

  // exact mode: worst-case visited count of one query = entries + hops * deg
  const u64 bound = entries + (u64)max_hops * deg + 32;
  DBuf<u64> gtab;
  if (!sh.cache && bound > (u64)sh.vis_limit) {
    a.gcap = next_pow2(2 * bound);
    gtab.alloc(r, (u64)grid * a.gcap);
    gtab.zero();
    a.gtable = gtab.p;
  }
  DBuf<u64> cnt(r, 4);
  cnt.zero();
  a.counters = cnt.p;
  if (qn)
    k_search<true><<<grid, 32, sh.smem, r.stream>>>(a);
  else
    k_search<false><<<grid, 32, sh.smem, r.stream>>>(a);
  KNNG_LAUNCH_CHECK();
  if (counters) {
    u64 h[4];
    KNNG_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, r.stream));
    r.sync();
    counters->hops += h[0];
    counters->scored += h[1];
    counters->overflowed += h[2];
    counters->launches += 1;
  }
}

}  // namespace knng_b200
