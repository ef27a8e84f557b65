// join.hpp -- the NN-Descent local join (nndescent.cpp:135-197) on the B200:
// compact join lists, the pipelined exact-distance join kernel and the
// lock-free offer resolution into the 4-way candidate buckets.
#pragma once

#include <cstdint>

#include "runtime.hpp"

namespace knng_b200 {

constexpr uint32_t kWays = 4;  // candidate slots per hash bucket

struct JoinPlan {
  int RMAX = 0;       // list capacity per point (>= 2B + k + B, multiple of 4)
  int DC = 0, DCP = 0;  // dims per staged chunk, smem row stride (floats)
  int pair = 0;         // pair layout (d % 4 == 0): two rows interleaved per dim
  int RB = 0;         // rows per staged batch
  size_t smem = 0;    // dynamic smem of k_join
  unsigned grid = 0;  // persistent CTAs (one per SM)
  uint64_t q_per_chunk = 0;  // offer-queue entries per point chunk
};

constexpr int kJoinChunk = 32;  // points per dynamically scheduled chunk

JoinPlan plan_join(const Runner& r, int d, uint32_t k, uint32_t B);

// Build the compact join lists of every point from the sampled lists.
void launch_join_lists(const Runner& r, uint64_t n, uint32_t k, uint32_t B, int RMAX,
                       const uint32_t* nf, const uint32_t* nfn, const uint32_t* of,
                       const uint32_t* ofn, const uint32_t* nr, const uint32_t* nrn,
                       const uint32_t* orv, const uint32_t* orn, uint32_t* L_ids,
                       uint32_t* L_cnt);

struct JoinLaunch {
  const float* X = nullptr;
  const float* nrm = nullptr;  // cosine norm chains (null: l2)
  int d = 0;
  uint64_t n_rows = 0;  // rows of X (the tensor-core join's TMA map)
  const uint32_t* L_ids = nullptr;
  const uint32_t* L_cnt = nullptr;
  const float* worst = nullptr;
  const uint32_t* act = nullptr;  // active point list; [p_lo, p_hi) index it (null: points)
  uint64_t p_lo = 0, p_hi = 0;
  const uint64_t* n_live = nullptr;  // device count bounding p_hi (null: none)
  uint32_t* chunk_counter = nullptr;  // zeroed before each launch
  uint64_t* q_key = nullptr;
  uint32_t* q_tgt = nullptr;
  uint32_t* q_fill = nullptr;
  uint64_t* counters = nullptr;  // kCntPairs / kCntOffers / kCntStagedRows
};

void launch_join(const Runner& r, const JoinPlan& plan, const JoinLaunch& a);

// Tensor-core join (join_tc.cu): tf32 Gram of the centred list rows decides,
// offers carry a lower bound of the exact distance (k_apply recomputes the
// exact distance of every candidate it may insert).  l2, d % 4 == 0, lists of
// <= 128 rows; opt-in with KNNG_JOIN=tc (the exact-order kernel above is the
// default: it measured faster).
bool join_tc_supported(const float* X, int d, uint32_t k, uint32_t B, bool cosine);
void launch_join_tc(const Runner& r, const JoinPlan& plan, const JoinLaunch& a);

// act[0 .. off[n]) = the points whose join descriptor is non-empty (a new
// entry exists), ascending; flag/off are scratch (n and n + 1 entries).
void build_active_list(const Runner& r, uint64_t n, const uint32_t* L_cnt, uint32_t* flag,
                       uint64_t* off, uint32_t* act);

// Resolve the queued offers of `chunks` chunk regions into the buckets.
void launch_offer(const Runner& r, const JoinPlan& plan, const uint64_t* q_key,
                  const uint32_t* q_tgt, const uint32_t* q_fill, uint32_t chunks,
                  uint64_t* slots, uint32_t S, uint32_t nb, uint32_t ways,
                  uint64_t* counters = nullptr, uint64_t p_lo = 0,
                  const uint64_t* n_live = nullptr, uint64_t n_points = 0,
                  uint8_t* touched = nullptr);

}  // namespace knng_b200
