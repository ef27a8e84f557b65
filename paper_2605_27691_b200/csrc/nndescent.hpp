// nndescent.hpp -- B200 lock-free NN-Descent local build (north_star item 2).
//
// Reference: nndescent.cpp:225-259 (nn_descent), :29-62 (init_random_graph),
// :64-129 (sample_neighbors), :135-197 (build_join_lists + local_join),
// :199-223 (apply_candidates), nndescent.hpp:12-20 (NnDescentParams).
//
// Device graph layout: keys[n*k] u64 packed (dist,id) sorted ascending per row,
// flags[n] u32 bitmask of "new" entries (k <= 32), worst[n] f32 = dist of
// row[k-1] (CandidateBuffer::worst, nndescent.hpp:58-60).
#pragma once

#include <cstdint>
#include <vector>

#include "runtime.hpp"

namespace knng_b200 {

struct NndParams {
  uint32_t k = 32;
  double delta = 0.0001;
  double rho = 0.5;
  uint64_t max_iters = 100;
  uint64_t candidate_capacity = 0;  // 0 -> 2k
  uint64_t seed = 0;
};

// Device counters written by the kernels (read back once per iteration).
enum NndStage : int { kStInit = 0, kStSample, kStLists, kStJoin, kStOffer, kStApply, kStSync };

enum NndCounter : int {
  kCntAccepted = 0,    // accepted inserts, ascending-key order = entries kept (nndescent.cpp:213)
  kCntPairs = 1,       // sigma evaluations (JoinCounts::pairs)
  kCntStagedRows = 2,  // feature rows staged into smem by the join (algorithmic bytes)
  kCntOffers = 3,      // offers passing the worst filter (atomicMin issued)
  kCntJoinPoints = 4,  // points with >= 1 pair
  kCntOfferSeen = 5,   // queue entries walked by k_offer
  kCntActive = 6,      // host scratch: points with a new entry this iteration
  kNumCounters = 8
};

struct NndStats {
  std::vector<uint64_t> accepted_per_iter;
  std::vector<uint64_t> offers_per_iter;
  std::vector<uint64_t> pairs_per_iter;
  uint64_t iterations = 0;
  uint64_t pairs = 0;
  uint64_t staged_rows = 0;
  uint64_t offers = 0;
  // Device time of the join kernel summed over iterations (CUDA events on the
  // launching stream) and of the whole build.
  double join_ms = 0.0;
  double offer_ms = 0.0;  // k_offer (atomicMin cascades), summed
  double total_ms = 0.0;
  // device time per stage: init, sample (fwd + transpose + reverse select),
  // join lists, join, offer, apply, readback/host gap
  double stage_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t join_launches = 0;
  uint64_t launches = 0;  // all kernels launched by the build
};

// Dataset on the runner's device, row-major n x d f32, L2.
struct DevRows {
  const float* x = nullptr;
  uint64_t n = 0;
  int d = 0;
  const float* nrm = nullptr;  // cosine norm chains (row_norms_device); null -> l2
};

void validate_nnd(const NndParams& p, uint64_t n);

// Grow-only buffers of a build (offer queue, candidate buckets, join lists),
// kept by a context across builds on one device: a fresh ~50 GB set per build
// occasionally made the pool map memory anew while the GPU waited.
struct SampleLists {
  uint32_t bound = 0;
  DBuf<uint32_t> nf, nfn, of, ofn, nr, nrn, orv, orn;
};
// reverse-list scratch of one sampling pass (counts, offsets, pair buffers)
struct RevCsr {
  DBuf<uint32_t> cnt_new, cnt_old, src_cnt, cur_new, cur_old, long_cnt, long_rec;
  DBuf<uint32_t> join_bits;  // joins(t) per point (n bits), for the old-list prune
  DBuf<uint64_t> off_new, off_old, src_off_new, src_off_old;
  DBuf<uint32_t> key_new, val_new, key_old, val_old, tk_new, tv_new, tk_old, tv_old;
};

struct NndWorkspace {
  DBuf<uint64_t> q_key, slots;
  DBuf<uint32_t> q_tgt, L_ids;
  // every other per-build buffer, so a build in a warm context issues no
  // allocation and no memory query (sized for the largest n / k / B seen)
  SampleLists lists;
  RevCsr rev;
  uint64_t lists_n = 0;
  uint32_t lists_k = 0, lists_b = 0;
  DBuf<float> worst;
  DBuf<uint8_t> touched;  // points an offer reached this iteration (k_offer -> k_apply)
  DBuf<uint64_t> counters, act_off;
  DBuf<uint32_t> L_cnt, act, act_flag, q_fill, chunk_ctr;
  uint64_t q_chunks_per_slice = 0;  // offer-queue slicing decided once per shape
  uint64_t q_per_chunk = 0, q_n = 0;
};

// Full build.  keys/flags must hold n*k / n entries on the runner's device.
void nn_descent_device(Runner& r, const DevRows& ds, const NndParams& p, uint64_t* keys,
                       uint32_t* flags, NndStats* stats, bool time_kernels,
                       NndWorkspace* ws = nullptr);

// Individual stages (exposed for parity tests through the C-ABI).
void init_random_graph_device(Runner& r, const DevRows& ds, uint32_t k, uint64_t seed,
                              uint64_t* keys, uint32_t* flags);

void sample_neighbors_device(Runner& r, uint64_t n, uint32_t k, double rho, uint64_t seed,
                             uint64_t iter, const uint64_t* keys, uint32_t* flags,
                             SampleLists& out);

// keys -> ids / dists / u8 flags (KnnGraph layout, core.hpp:156-179).
void export_graph_device(const Runner& r, const uint64_t* keys, const uint32_t* flags,
                         uint64_t n, uint32_t k, uint32_t id_shift, uint32_t* ids,
                         float* dists, uint8_t* flags_u8);
// ids / dists (+ optional u8 flags) -> keys (+ flag masks).
void import_graph_device(const Runner& r, const uint32_t* ids, const float* dists,
                         const uint8_t* flags_u8, uint64_t n, uint32_t k, uint64_t* keys,
                         uint32_t* flags);

}  // namespace knng_b200
