// graphopt.hpp -- optimize_graph on the B200 (graphopt.cpp:24-105).
#pragma once

#include <cstdint>

#include "runtime.hpp"

namespace knng_b200 {

// keys: n x k packed (dist, id + id_base) rows on the runner's device; X: the
// n x d rows the ids index (after subtracting id_base).  Writes n x out_degree
// ids (local) to sg.
void optimize_graph_device(Runner& r, const uint64_t* keys, uint64_t n, uint32_t k,
                           uint32_t id_base, const float* X, int d, uint32_t out_degree,
                           uint32_t* sg, uint64_t* launches = nullptr,
                           const float* nrm = nullptr);  // nrm: cosine norm chains

}  // namespace knng_b200
