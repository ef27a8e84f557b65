// search.hpp -- ann_search on the B200 (annsearch.cpp:50-129).
#pragma once

#include <cstdint>

#include "runtime.hpp"

namespace knng_b200 {

struct SearchParamsDev {
  uint64_t k_s = 10;
  uint64_t beam_width = 64;
  uint64_t num_entry_points = 16;
  uint64_t max_hops = 0;  // 0 -> 4 * beam_width
  uint64_t seed = 0;
};

struct SearchCounters {
  uint64_t hops = 0;
  uint64_t scored = 0;
  uint64_t overflowed = 0;  // queries whose visited set spilled to global memory
  uint64_t launches = 0;
};

void validate_search(uint64_t q_dims, uint64_t v_dims, uint64_t sg_n, uint64_t nv,
                     const SearchParamsDev& p);
size_t search_smem_bytes(int d, uint32_t width);

// Q: nq x d queries, V: nv x d vectors, sg: nv x deg ids into V; all on the
// runner's device.  Output ids get id_base added (refine merges global ids).
// Query q uses rng stream mix_seed(seed, 0xa11ce000 + qbase + q).
void ann_search_device(Runner& r, const float* Q, uint64_t nq, int d, const uint32_t* sg,
                       uint32_t deg, const float* V, uint64_t nv, const SearchParamsDev& p,
                       uint32_t id_base, uint32_t* out_ids, float* out_d, uint32_t* hops,
                       uint32_t* scored, SearchCounters* counters, uint64_t qbase = 0,
                       const float* qn = nullptr, const float* vn = nullptr,  // cosine norms
                       uint32_t* scored_ids = nullptr, uint64_t scored_cap = 0);

}  // namespace knng_b200
