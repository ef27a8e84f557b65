// radix.hpp -- stable LSD radix sort of (u32 key, u32 value) pairs.
#pragma once

#include <cstdint>

#include "runtime.hpp"

namespace knng_b200 {

// Sorts n pairs by key (stable).  Ping-pongs between (keys, vals) and (tmp_keys,
// tmp_vals); *result_in_tmp says which pair holds the sorted output.  Keys
// above max_key are not allowed (they decide the number of 8-bit passes).
void radix_sort_pairs(const Runner& r, uint32_t* keys, uint32_t* vals, uint32_t* tmp_keys,
                      uint32_t* tmp_vals, uint64_t n, uint32_t max_key, bool* result_in_tmp);
// Same, sorting the first *n_dev (read on the device, <= capacity) pairs:
// tiles past the live count exit at once, so no host round trip is needed.
void radix_sort_pairs_dev(const Runner& r, uint32_t* keys, uint32_t* vals, uint32_t* tmp_keys,
                          uint32_t* tmp_vals, uint64_t capacity, const uint64_t* n_dev,
                          uint32_t max_key, bool* result_in_tmp);

}  // namespace knng_b200
