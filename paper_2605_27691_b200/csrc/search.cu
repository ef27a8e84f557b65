// search.cu -- greedy best-first batch search ann_search (annsearch.cpp:50-129),
// the remote-refine kernel (north_star item 3).
//
// One warp per query (persistent CTAs of one warp).  Per query the warp keeps
//   * the beam: a sorted array of packed (dist,id) keys in smem, double
//     buffered, plus an "expanded" bitmask (BeamEntry, annsearch.cpp:19-31);
//   * the visited set: an exact open-addressing hash of ids in smem (4096
//     slots); if a query ever visits more than 3/4 of that, the set migrates
//     to a per-warp tagged table in global memory, so membership stays exact
//     (VisitedSet, annsearch.cpp:35-46) -- no point is ever scored twice;
//   * the query vector in smem.
// A hop expands the first unexpanded beam entry, dedups its out-neighbors
// (match.any), test-and-sets them in the visited set, scores the new ones with
// exact-order distances (one lane per candidate), sorts the batch with a warp
// bitonic network and merges it into the beam by rank (merge path).  A beam
// after a batch is the top-`width` of (beam U batch), which is what the
// reference's sequential beam_insert produces, so results are bit-identical.
#include "search.hpp"

namespace knng_b200 {
namespace {

constexpr u32 kNoId = 0xffffffffu;
constexpr int kVisH = 4096;            // smem visited slots
constexpr int kVisLimit = kVisH * 3 / 4;

struct SearchArgs {
  const float* Q;
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
  u64* gtable;  // per-CTA tagged visited tables (gcap slots each), may be null
  u32 gcap;
  u64* counters;  // [0] hops [1] scored [2] overflowed queries
  u32 id_base;    // added to output ids
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
  u64* g;           // global table of this CTA
  u32 gcap;
  u32 tag;          // query tag for the global table
  bool global;
  u32 count;

  // Returns true if id was present (no insert); lane-parallel, ids distinct.
  __device__ __forceinline__ bool lookup(u32 id) const {
    if (!global) {
      u32 h = vis_hash(id) & (kVisH - 1);
      while (true) {
        const u32 v = s[h];
        if (v == id) return true;
        if (v == kNoId) return false;
        h = (h + 1) & (kVisH - 1);
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
  // Test-and-set; returns true if newly inserted.
  __device__ __forceinline__ bool insert(u32 id) {
    if (!global) {
      u32 h = vis_hash(id) & (kVisH - 1);
      while (true) {
        const u32 old = atomicCAS(&s[h], kNoId, id);
        if (old == kNoId) return true;
        if (old == id) return false;
        h = (h + 1) & (kVisH - 1);
      }
    }
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
  // Move the smem set into the global table (all lanes call).
  __device__ void migrate() {
    const unsigned lane = lane_id();
    __syncwarp();
    global = true;
    for (int t = lane; t < kVisH; t += 32) {
      const u32 id = s[t];
      if (id != kNoId) insert(id);
    }
    __syncwarp();
  }
};

// Merge the lane-held candidate keys (kEmptyKey = none) into the beam.
__device__ __forceinline__ void beam_merge(u64 c, u64* __restrict__ s_beam, u32* __restrict__ s_exp,
                                           u64* __restrict__ s_cand, int& cur, u32& bs, u32 width) {
  const unsigned lane = lane_id();
  if (bs == width && c != kEmptyKey && c >= s_beam[cur * width + width - 1]) c = kEmptyKey;
  if (!__any_sync(kFull, c != kEmptyKey)) return;
  c = warp_sort32(c);
  const u32 nc = __popc(__ballot_sync(kFull, c != kEmptyKey));
  s_cand[lane] = c;
  const int nxt = cur ^ 1;
  const u32 words = (width + 31) >> 5;
  u64* dst = s_beam + nxt * width;
  u32* dexp = s_exp + nxt * 32;
  const u64* src = s_beam + cur * width;
  const u32* sexp = s_exp + cur * 32;
  if (lane < words) dexp[lane] = 0;
  __syncwarp();
  // beam entries: new position = i + #cands < b
  for (u32 i = lane; i < bs; i += 32) {
    const u64 b = src[i];
    u32 lo = 0, hi = nc;
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if (s_cand[mid] < b) lo = mid + 1; else hi = mid;
    }
    const u32 pos = i + lo;
    if (pos < width) {
      dst[pos] = b;
      if ((sexp[i >> 5] >> (i & 31)) & 1u) atomicOr(&dexp[pos >> 5], 1u << (pos & 31));
    }
  }
  // candidates: new position = j + #beam < c
  if (lane < nc) {
    u32 lo = 0, hi = bs;
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if (src[mid] < c) lo = mid + 1; else hi = mid;
    }
    const u32 pos = lane + lo;
    if (pos < width) dst[pos] = c;
  }
  __syncwarp();
  cur = nxt;
  bs = min(width, bs + nc);
}

__global__ __launch_bounds__(32) void k_search(SearchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const unsigned lane = lane_id();
  const u32 W = a.width;
  // layout
  float* s_q = reinterpret_cast<float*>(smem);
  size_t off = (((size_t)a.d * 4) + 15) & ~size_t(15);
  u32* s_vis = reinterpret_cast<u32*>(smem + off);
  off += (size_t)kVisH * 4;
  u64* s_beam = reinterpret_cast<u64*>(smem + off);
  off += (size_t)2 * W * 8;
  u64* s_cand = reinterpret_cast<u64*>(smem + off);
  off += 32 * 8;
  u32* s_exp = reinterpret_cast<u32*>(smem + off);  // 2 x 32 words

  u64 tot_hops = 0, tot_scored = 0, tot_ovf = 0;
  for (u64 q = blockIdx.x; q < a.nq; q += gridDim.x) {
    // stage query, clear visited
    const float* qrow = a.Q + q * (u64)a.d;
    for (int t = lane; t < a.d; t += 32) s_q[t] = qrow[t];
    for (int t = lane; t < kVisH; t += 32) s_vis[t] = kNoId;
    __syncwarp();
    Visited vis{s_vis, a.gtable ? a.gtable + (u64)blockIdx.x * a.gcap : nullptr, a.gcap,
                (u32)(q + 1), false, 0};
    int cur = 0;
    u32 bs = 0;
    u32 scored = 0;

    auto score_and_merge = [&](u32 id, bool take) {
      u64 c = kEmptyKey;
      if (take) c = pack_key(l2_exact(s_q, a.V + (u64)id * a.d, a.d), id);
      beam_merge(c, s_beam, s_exp, s_cand, cur, bs, W);
    };
    auto maybe_migrate = [&](u32 add) {
      vis.count += add;
      if (!vis.global && vis.count > (u32)kVisLimit) {
        if (vis.g == nullptr) __trap();  // host sizes gtable whenever overflow is possible
        vis.migrate();
        ++tot_ovf;
      }
    };

    // entry points: sample_distinct(n, entries, Rng(mix_seed(seed, 0xa11ce000+q)))
    if (a.entries >= a.nv) {
      for (u64 base = 0; base < a.nv; base += 32) {
        const u64 id = base + lane;
        const bool take = id < a.nv;
        if (take) vis.insert((u32)id);
        maybe_migrate(__popc(__ballot_sync(kFull, take)));
        score_and_merge((u32)id, take);
        scored += __popc(__ballot_sync(kFull, take));
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
        scored += ntake;
        maybe_migrate(ntake);
        score_and_merge(x, take);
      }
    }

    // expansion loop (annsearch.cpp:103-120)
    u32 hops = 0;
    while (hops < a.max_hops) {
      const u32 words = (bs + 31) >> 5;
      u32 w = 0;
      if (lane < words) {
        const u32 valid = (lane == words - 1 && (bs & 31)) ? ((1u << (bs & 31)) - 1u) : kFull;
        w = ~s_exp[cur * 32 + lane] & valid;
      }
      const unsigned nz = __ballot_sync(kFull, w != 0);
      if (!nz) break;  // every beam entry expanded
      const int wl = __ffs(nz) - 1;
      const u32 wv = __shfl_sync(kFull, w, wl);
      const u32 idx = (u32)wl * 32 + (__ffs(wv) - 1);
      const u32 u = key_id(s_beam[cur * W + idx]);
      __syncwarp();
      if (lane == 0) s_exp[cur * 32 + (idx >> 5)] |= 1u << (idx & 31);
      __syncwarp();
      for (u32 c0 = 0; c0 < a.deg; c0 += 32) {
        const u32 nb = (c0 + lane < a.deg) ? a.sg[(u64)u * a.deg + c0 + lane] : kNoId;
        const unsigned grp = __match_any_sync(kFull, nb);
        const bool cand = nb != kNoId && (__ffs(grp) - 1) == (int)lane;
        const bool fresh = cand && vis.insert(nb);
        const u32 nf = __popc(__ballot_sync(kFull, fresh));
        scored += nf;
        maybe_migrate(nf);
        score_and_merge(nb, fresh);
      }
      ++hops;
    }
    // best k_s (annsearch.cpp:122-126); unfilled slots stay 0 / 0.0f
    for (u32 i = lane; i < a.ks; i += 32) {
      u32 id = 0;
      float dd = 0.0f;
      if (i < bs) {
        const u64 key = s_beam[cur * W + i];
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

}  // namespace

size_t search_smem_bytes(int d, uint32_t width) {
  size_t off = (((size_t)d * 4) + 15) & ~size_t(15);
  off += (size_t)kVisH * 4 + (size_t)2 * width * 8 + 32 * 8 + 2 * 32 * 4;
  return off;
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
                       uint32_t* scored, SearchCounters* counters, uint64_t qbase) {
  validate_search((uint64_t)d, (uint64_t)d, nv, nv, p);
  if (nq == 0) return;
  DeviceGuard guard(r.device);
  const u32 width = (u32)p.beam_width;
  const u32 max_hops = (u32)(p.max_hops ? p.max_hops : p.beam_width * 4);
  u64 entries = p.num_entry_points > p.k_s ? p.num_entry_points : p.k_s;
  if (entries > nv) entries = nv;

  const size_t smem = search_smem_bytes(d, width);
  KNNG_CUDA(cudaFuncSetAttribute(k_search, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  int per_sm = 0;
  KNNG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search, 32, smem));
  if (per_sm < 1) per_sm = 1;
  const unsigned grid = persistent_grid(r, per_sm, nq);

  SearchArgs a{};
  a.Q = Q;
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
  a.id_base = id_base;

  // worst-case visited count of one query: entries + hops * deg
  const u64 bound = entries + (u64)max_hops * deg + 32;
  DBuf<u64> gtab;
  if (bound > (u64)kVisLimit) {
    a.gcap = next_pow2(2 * bound);
    gtab.alloc(r, (u64)grid * a.gcap);
    gtab.zero();
    a.gtable = gtab.p;
  }
  DBuf<u64> cnt(r, 4);
  cnt.zero();
  a.counters = cnt.p;
  k_search<<<grid, 32, smem, r.stream>>>(a);
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
