// refine_kernels.cu -- partition (K1), merge_results_into (K8),
// translate_to_external (K9) and row gathers on the B200.
//
// * partition_dataset refine.cpp:86-126: the reference's serial Fisher-Yates
//   (rng.hpp:90-96) executed in parallel by deterministic reservations: swap t
//   exchanges positions (n-1-t, j_t) with j_t = next_below(draw t, n-t) read
//   from the counter-addressed SplitMix64 stream; in each round every pending
//   swap atomicMin-reserves both positions with its index and commits only if
//   it owns both, so conflicting swaps execute in sequential order.  The
//   permutation is bit-identical to the serial shuffle.
// * merge_rows core.cpp:114-134 as a warp-per-row segmented merge by rank
//   (b first on equal keys), first-occurrence id dedup, truncation to k.
// * translate_to_external refine.cpp:395-416: ids mapped, row re-sorted by
//   (dist, external id), scattered to its external row.
#include <algorithm>
#include <vector>

#include "refine_kernels.hpp"

namespace knng_b200 {
namespace {

__global__ void k_iota(u32* __restrict__ perm, u64 n) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x)
    perm[i] = (u32)i;
}

__global__ void k_shuffle_init(u32* __restrict__ perm, u32* __restrict__ res,
                               u32* __restrict__ jdraw, u32* __restrict__ pend, u64 n, u64 s0) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    perm[i] = (u32)i;
    res[i] = 0xffffffffu;
    if (i + 1 < n) {
      // swap t = i: position a = n-1-t with j = next_below(n - t)
      jdraw[i] = (u32)mulhi64(sm64_draw(s0, i), n - i);
      pend[i] = (u32)i;
    }
  }
}

__global__ void k_shuffle_reserve(const u32* __restrict__ pend, u64 cnt,
                                  const u32* __restrict__ jdraw, u32* __restrict__ res, u64 n) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (u64)gridDim.x * blockDim.x) {
    const u32 t = pend[i];
    atomicMin(&res[n - 1 - t], t);
    atomicMin(&res[jdraw[t]], t);
  }
}

__global__ void k_shuffle_commit(const u32* __restrict__ pend, u64 cnt,
                                 const u32* __restrict__ jdraw, const u32* __restrict__ res,
                                 u32* __restrict__ perm, u32* __restrict__ next,
                                 unsigned long long* __restrict__ next_cnt, u64 n) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (u64)gridDim.x * blockDim.x) {
    const u32 t = pend[i];
    const u64 a = n - 1 - t, b = jdraw[t];
    if (res[a] == t && res[b] == t) {
      const u32 x = perm[a];
      perm[a] = perm[b];
      perm[b] = x;
    } else {
      next[atomicAdd(next_cnt, 1ull)] = t;
    }
  }
}

__global__ void k_shuffle_reset(const u32* __restrict__ pend, u64 cnt,
                                const u32* __restrict__ jdraw, u32* __restrict__ res, u64 n) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (u64)gridDim.x * blockDim.x) {
    const u32 t = pend[i];
    res[n - 1 - t] = 0xffffffffu;
    res[jdraw[t]] = 0xffffffffu;
  }
}

__global__ __launch_bounds__(256) void k_gather_rows(const float* __restrict__ X, int d,
                                                     const u32* __restrict__ idx, u64 rows,
                                                     float* __restrict__ out) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  const bool vec = (d & 3) == 0;
  for (u64 r = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const float* src = X + (u64)idx[r] * d;
    float* dst = out + r * d;
    if (vec) {
      for (int c = lane * 4; c < d; c += 128)
        *reinterpret_cast<float4*>(dst + c) = *reinterpret_cast<const float4*>(src + c);
    } else {
      for (int c = lane; c < d; c += 32) dst[c] = src[c];
    }
  }
}

// merge_rows core.cpp:114-134 for every row: a = na sorted keys (+ optional
// flag mask), b = nb result entries (ids + id_base, dists); out = first k
// distinct-by-id entries of the merged order (b first on equal keys).  The
// output may alias a (each warp reads its row before writing).
__global__ __launch_bounds__(256) void k_merge_rows(const u64* akeys, const u32* aflags, u32 na,
                                                    const u32* __restrict__ bid,
                                                    const float* __restrict__ bd, u32 nb,
                                                    u32 id_base, u64 rows, u32 k, u64* okeys,
                                                    u32* oflags, u32* __restrict__ ocount) {
  __shared__ u64 s_key[8][64];
  __shared__ u32 s_flag[8][64];
  const unsigned lane = lane_id(), w = threadIdx.x >> 5;
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 r = (((u64)blockIdx.x * blockDim.x) >> 5) + w; r < rows; r += warps) {
    const u64 ak = lane < na ? akeys[r * na + lane] : kEmptyKey;
    const u32 af = aflags ? ((aflags[r] >> lane) & 1u) : 0u;
    const u64 bk = lane < nb ? pack_key(bd[r * nb + lane], bid[r * nb + lane] + id_base) : kEmptyKey;
    u32 ca = 0, cb = 0;
    for (u32 t = 0; t < 32; ++t) {
      const u64 bt = __shfl_sync(kFull, bk, t);
      const u64 at = __shfl_sync(kFull, ak, t);
      ca += (t < nb && bt <= ak) ? 1u : 0u;  // b goes first on equal keys
      cb += (t < na && at < bk) ? 1u : 0u;
    }
    if (lane < na) {
      s_key[w][lane + ca] = ak;
      s_flag[w][lane + ca] = af;
    }
    if (lane < nb) {
      s_key[w][lane + cb] = bk;
      s_flag[w][lane + cb] = 0;
    }
    __syncwarp();
    const u32 tot = na + nb;
    u32 outc = 0;
    u64 mykey = kEmptyKey;
    u32 myflag = 0;
    for (u32 h = 0; h < tot; h += 32) {
      const u32 pos = h + lane;
      bool keep = false;
      u64 e = kEmptyKey;
      u32 ef = 0;
      if (pos < tot) {
        e = s_key[w][pos];
        ef = s_flag[w][pos];
        keep = true;
        for (u32 q = 0; q < pos; ++q)
          if (key_id(s_key[w][q]) == key_id(e)) keep = false;
      }
      const unsigned b = __ballot_sync(kFull, keep);
      const u32 idx = outc + __popc(b & lanemask_lt());
      for (u32 src = 0; src < 32; ++src) {
        if (!((b >> src) & 1u)) continue;
        const u64 ev = __shfl_sync(kFull, e, src);
        const u32 fv = __shfl_sync(kFull, ef, src);
        const u32 iv = __shfl_sync(kFull, idx, src);
        if (iv == lane) {
          mykey = ev;
          myflag = fv;
        }
      }
      outc += __popc(b);
    }
    __syncwarp();
    if (lane < k) okeys[r * k + lane] = mykey;
    const unsigned fm = __ballot_sync(kFull, lane < k && myflag);
    if (lane == 0) {
      if (oflags) oflags[r] = fm;
      if (ocount) ocount[r] = outc < k ? outc : k;
    }
  }
}

// translate_to_external: rows [0, n) of the internal-order graph (row g is
// internal id g) -> external row to_external[g], ids mapped, re-sorted.
// row g of keys is internal row row_base + g; scattered to its external row
// (full graph) or kept at g with its external row id in out_rows (compact)
__global__ __launch_bounds__(256) void k_translate(const u64* __restrict__ keys, u64 n, u32 k,
                                                   const u32* __restrict__ to_ext,
                                                   u32* __restrict__ out_ids,
                                                   float* __restrict__ out_d, u64 row_base,
                                                   u32* __restrict__ out_rows) {
  const unsigned lane = lane_id();
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 g = (((u64)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); g < n; g += warps) {
    u64 key = kEmptyKey;
    if (lane < k) {
      const u64 kk = keys[g * k + lane];
      key = ((kk >> 32) << 32) | to_ext[key_id(kk)];
    }
    key = warp_sort32(key);
    const u64 ext_row = to_ext[row_base + g];
    const u64 dst = out_rows ? g : ext_row;
    if (out_rows && lane == 0) out_rows[g] = (u32)ext_row;
    if (lane < k) {
      out_ids[dst * k + lane] = key_id(key);
      out_d[dst * k + lane] = key_dist(key);
    }
  }
}

__global__ void k_shift_ids(u64* __restrict__ keys, u64 count, int64_t delta) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (u64)gridDim.x * blockDim.x) {
    const u64 key = keys[i];
    keys[i] = (key & 0xffffffff00000000ull) | (u32)((int64_t)key_id(key) + delta);
  }
}

unsigned elem_grid(const Runner& r, u64 items) {
  const u64 want = ceil_div<u64>(items, 256);
  const u64 cap = (u64)r.num_sms * 32;
  return (unsigned)std::max<u64>(1, std::min(want, cap));
}
unsigned warp_grid(const Runner& r, u64 items) {
  const u64 want = ceil_div<u64>(items, 8);
  const u64 cap = (u64)r.num_sms * 16;
  return (unsigned)std::max<u64>(1, std::min(want, cap));
}

}  // namespace

void partition_device(Runner& r, uint64_t n, uint32_t ranks, uint64_t seed, uint32_t* to_external,
                      std::vector<uint64_t>& offsets, uint64_t* rounds_out) {
  require(!(ranks == 0 || ranks > n), "partition_dataset: need 1 <= P <= N");
  require(n < 0xffffffffull, "partition_dataset: N must fit a 32-bit point id");
  DeviceGuard guard(r.device);
  offsets.assign(ranks + 1, 0);
  const u64 base = n / ranks, extra = n % ranks;
  for (u32 q = 0; q < ranks; ++q) offsets[q + 1] = offsets[q] + base + (q < extra ? 1 : 0);
  uint64_t rounds = 0;
  if (ranks == 1 || n < 2) {
    // identity (refine.cpp:93-98)
    k_iota<<<elem_grid(r, n), 256, 0, r.stream>>>(to_external, n);
    KNNG_LAUNCH_CHECK();
    if (rounds_out) *rounds_out = 0;
    return;
  }
  const u64 s0 = mix_seed(seed, 0x9a71710ull);
  DBuf<u32> res(r, n), jd(r, n), pa(r, n), pb(r, n);
  DBuf<unsigned long long> cnt(r, 1);
  k_shuffle_init<<<elem_grid(r, n), 256, 0, r.stream>>>(to_external, res.p, jd.p, pa.p, n, s0);
  KNNG_LAUNCH_CHECK();
  u64 pending = n - 1;
  u32* cur = pa.p;
  u32* nxt = pb.p;
  // each round's pending count comes back through pinned memory, polled on
  // an event (a pageable copy + sleeping stream sync per round stalled the
  // host by up to ~0.7 s now and then with four ranks per box)
  HBuf<unsigned long long> hc(1);
  cudaEvent_t done;
  KNNG_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t e;
    ~EvGuard() { cudaEventDestroy(e); }
  } done_guard{done};
  while (pending) {
    ++rounds;
    cnt.zero();
    const unsigned g = elem_grid(r, pending);
    k_shuffle_reserve<<<g, 256, 0, r.stream>>>(cur, pending, jd.p, res.p, n);
    KNNG_LAUNCH_CHECK();
    k_shuffle_commit<<<g, 256, 0, r.stream>>>(cur, pending, jd.p, res.p, to_external, nxt, cnt.p,
                                              n);
    KNNG_LAUNCH_CHECK();
    k_shuffle_reset<<<g, 256, 0, r.stream>>>(cur, pending, jd.p, res.p, n);
    KNNG_LAUNCH_CHECK();
    KNNG_CUDA(cudaMemcpyAsync(hc.p, cnt.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              r.stream));
    KNNG_CUDA(cudaEventRecord(done, r.stream));
    while (cudaEventQuery(done) == cudaErrorNotReady) {
    }
    KNNG_CUDA(cudaGetLastError());
    pending = hc.p[0];
    std::swap(cur, nxt);
  }
  if (rounds_out) *rounds_out = rounds;
}

void gather_rows_device(const Runner& r, const float* X, int d, const uint32_t* idx, uint64_t rows,
                        float* out) {
  if (!rows) return;
  k_gather_rows<<<warp_grid(r, rows), 256, 0, r.stream>>>(X, d, idx, rows, out);
  KNNG_LAUNCH_CHECK();
}

void merge_rows_device(const Runner& r, const uint64_t* akeys, const uint32_t* aflags,
                       uint32_t na, const uint32_t* bid, const float* bd, uint32_t nb,
                       uint32_t id_base, uint64_t rows, uint32_t k, uint64_t* okeys,
                       uint32_t* oflags, uint32_t* ocount) {
  require(na <= 32 && nb <= 32 && k >= 1 && k <= 32,
          "merge_rows: the B200 path supports rows of <= 32 entries");
  if (!rows) return;
  k_merge_rows<<<warp_grid(r, rows), 256, 0, r.stream>>>(akeys, aflags, na, bid, bd, nb, id_base,
                                                         rows, k, okeys, oflags, ocount);
  KNNG_LAUNCH_CHECK();
}

void merge_results_device(const Runner& r, uint64_t* keys, uint32_t* flags, uint64_t n, uint32_t k,
                          const uint32_t* rid, const float* rd, uint32_t ks, uint32_t id_base) {
  merge_rows_device(r, keys, flags, k, rid, rd, ks, id_base, n, k, keys, flags, nullptr);
}

void shift_ids_device(const Runner& r, uint64_t* keys, uint64_t count, int64_t delta) {
  if (!count || !delta) return;
  k_shift_ids<<<elem_grid(r, count), 256, 0, r.stream>>>(keys, count, delta);
  KNNG_LAUNCH_CHECK();
}

void translate_device(const Runner& r, const uint64_t* keys, uint64_t n, uint32_t k,
                      const uint32_t* to_ext, uint32_t* out_ids, float* out_d) {
  if (!n) return;
  k_translate<<<warp_grid(r, n), 256, 0, r.stream>>>(keys, n, k, to_ext, out_ids, out_d, 0,
                                                     nullptr);
  KNNG_LAUNCH_CHECK();
}

void translate_rows_device(const Runner& r, const uint64_t* keys, uint64_t rows, uint32_t k,
                           const uint32_t* to_ext, uint64_t row_base, uint32_t* out_ids,
                           float* out_d, uint32_t* out_rows) {
  if (!rows) return;
  k_translate<<<warp_grid(r, rows), 256, 0, r.stream>>>(keys, rows, k, to_ext, out_ids, out_d,
                                                        row_base, out_rows);
  KNNG_LAUNCH_CHECK();
}

}  // namespace knng_b200
