// refine_kernels.hpp -- partition / merge / translate kernels (refine.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "runtime.hpp"

namespace knng_b200 {

// partition_dataset refine.cpp:86-126: to_external (device, n entries) is the
// bit-exact serial Fisher-Yates permutation; offsets (host) the ceil split.
void partition_device(Runner& r, uint64_t n, uint32_t ranks, uint64_t seed,
                      uint32_t* to_external, std::vector<uint64_t>& offsets,
                      uint64_t* rounds = nullptr);
// out[i] = X[idx[i]] (rows of d floats)
void gather_rows_device(const Runner& r, const float* X, int d, const uint32_t* idx,
                        uint64_t rows, float* out);
// merge_rows core.cpp:114-134, batched (see k_merge_rows); okeys may alias akeys.
void merge_rows_device(const Runner& r, const uint64_t* akeys, const uint32_t* aflags,
                       uint32_t na, const uint32_t* bid, const float* bd, uint32_t nb,
                       uint32_t id_base, uint64_t rows, uint32_t k, uint64_t* okeys,
                       uint32_t* oflags, uint32_t* ocount);
// merge_results_into refine.cpp:49-60 -> merge_rows core.cpp:114-134, in place.
void merge_results_device(const Runner& r, uint64_t* keys, uint32_t* flags, uint64_t n,
                          uint32_t k, const uint32_t* rid, const float* rd, uint32_t ks,
                          uint32_t id_base);
// shift_ids refine.cpp:42-45 on packed keys (row order is preserved).
void shift_ids_device(const Runner& r, uint64_t* keys, uint64_t count, int64_t delta);
// translate_to_external refine.cpp:395-416 for an internal-order N x k graph.
void translate_device(const Runner& r, const uint64_t* keys, uint64_t n, uint32_t k,
                      const uint32_t* to_ext, uint32_t* out_ids, float* out_d);
// The same for internal rows [row_base, row_base + rows) of one rank, written
// compactly: row g -> out row g, external row id -> out_rows[g].
void translate_rows_device(const Runner& r, const uint64_t* keys, uint64_t rows, uint32_t k,
                           const uint32_t* to_ext, uint64_t row_base, uint32_t* out_ids,
                           float* out_d, uint32_t* out_rows);

// Exact k-NN (brute_force_knng evalio.cpp:125-147) of rows[0..q) against all n
// rows of X (self excluded), k <= 32; keys out q x k.  nrm = the rows' norm
// chains (row_norms_device) selects the cosine metric; null -> l2.
void brute_force_rows_device(Runner& r, const float* X, uint64_t n, int d, const uint64_t* rows,
                             uint64_t q, uint32_t k, uint32_t* out_ids, float* out_d,
                             const float* nrm = nullptr);

// Cosine norm chains (core.hpp:44-49) of rows [0, n) of X into out[n].
void row_norms_device(const Runner& r, const float* X, uint64_t n, int d, float* out);

}  // namespace knng_b200
