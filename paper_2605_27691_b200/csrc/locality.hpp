// locality.hpp -- a spatial processing order of a point set (locality.cu).
#pragma once

#include <cstdint>

#include "runtime.hpp"

namespace knng_b200 {

// order[0..n): a permutation of 0..n-1 in which spatially near rows of X
// (n x d f32, on r's device) are near each other (Morton order of three
// seeded random projections; ties keep id order).  Deterministic.
void locality_order(const Runner& r, const float* X, uint64_t n, int d, uint64_t seed,
                    uint32_t* order);

}  // namespace knng_b200
