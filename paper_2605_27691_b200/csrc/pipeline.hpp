// pipeline.hpp -- build_distributed (refine.cpp:504-586) on B200s:
// partition -> per-rank local NN-Descent -> binary-tree refine -> grouped
// merge -> flat refine -> translate to external ids.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "nndescent.hpp"
#include "search.hpp"
#include "world.hpp"

namespace knng_b200 {

struct RefineCfg {
  uint64_t ranks = 1;
  uint64_t groups = 2;
  uint64_t k = 32;
  uint64_t k_s = 0;         // 0 -> k
  uint64_t out_degree = 0;  // 0 -> k
  NndParams nn;
  SearchParamsDev search;
  bool skip_tree_phase = false;
  bool double_buffer = false;
  bool capture_snapshots = false;
  uint64_t max_concat_bytes = 0;
  uint64_t seed = 0;
  bool cosine = false;    // MetricKind::cosine (core.hpp:41-55): kernels run the dot chain
  bool u8_elems = false;  // input rows were u8 (expanded to f32 on the device): wire sizes
                          // and footprint estimates use 1 byte per element
};

struct DistResult {
  double local_s = 0, tree_s = 0, merge_s = 0, flat_s = 0, etc_s = 0, partition_s = 0;
  uint64_t levels = 0, merge_epoch = 0, flat_epoch = 0;
  std::vector<GetRecord> comm_log;
  // local build statistics summed over ranks
  uint64_t nnd_iterations_max = 0, nnd_pairs = 0, nnd_staged_rows = 0;
  double join_ms_max = 0;
  SearchCounters search;
  // snapshots (capture_snapshots): label + N x k graph in external order
  std::vector<std::string> snap_labels;
  std::vector<std::vector<uint32_t>> snap_ids;
  std::vector<std::vector<float>> snap_dists;
};

// effective_groups refine.cpp:160-183: M, or P when the tree phase is skipped
// (skip_tree_phase, or the max_concat_bytes estimate exceeded).
uint64_t effective_group_count(const std::vector<uint64_t>& offsets, const RefineCfg& cfg, int d);

// Tree schedule helpers (refine.cpp:128-149).
uint64_t tree_levels(uint64_t ranks, uint64_t groups);
struct TreeLevel {
  uint64_t group_lo = 0, group_hi = 0;
  std::vector<uint64_t> partners;
};
TreeLevel tree_schedule(uint64_t ranks, uint64_t groups, uint64_t rank, uint64_t level);

// Devices the ranks run on: rank r -> devices[r % devices.size()].
// X: n x d f32 rows (host or device memory of devices[0]).  Output N x k ids /
// dists in external order, host or device (out_on_device: devices[0]).
void build_distributed(const std::vector<int>& devices, const float* X, bool x_on_device,
                       uint64_t n, int d, const RefineCfg& cfg, uint32_t* out_ids,
                       float* out_dists, bool out_on_device, DistResult* res);

// One rank of build_distributed in this process (one process per GPU):
// every rank passes the same full dataset; the partition is recomputed
// identically, the rank builds and refines its block on `device`, and the
// cross-rank pulls go through a ProcWorld over the caller's host transport.
// Outputs: the rank's rows in external ids (rows x k) and each row's external
// id; returns the row count (<= ceil(n / ranks)).  Collective: every rank of
// the transport must call it with the same arguments.
uint64_t build_distributed_rank(int device, size_t rank, size_t ranks, const HostTransport& t,
                                const float* X, bool x_on_device, uint64_t n, int d,
                                const RefineCfg& cfg, uint32_t* out_ids, float* out_dists,
                                uint32_t* out_rows, bool out_on_device, DistResult* res,
                                Runner* base = nullptr, NndWorkspace* ws = nullptr);

// Refinement only, from given local graphs (internal global ids, rank blocks
// at offsets) -- the world-level drivers binary_tree_refine -> grouped_merge
// -> flat_refine (mode 0) or all_to_all_refine (mode 1), refine.hpp:117-136.
// X_perm: rows in internal order (host).  ids/dists updated in place (host).
void refine_from_local(const std::vector<int>& devices, const float* X_perm, uint64_t n, int d,
                       const RefineCfg& cfg, const std::vector<uint64_t>& offsets, uint32_t* ids,
                       float* dists, int mode, DistResult* res);

// One world-level phase driver (1 all_to_all_refine, 2 binary_tree_refine,
// 3 grouped_merge, 4 flat_refine, refine.cpp:430-502) on a world starting at epoch `epoch0`.
// sg_in / sg_out: per-rank blocks (group_n(rank) x out_degree), rank order.
void refine_phase(const std::vector<int>& devices, const float* X_perm, uint64_t n, int d,
                  const RefineCfg& cfg, const std::vector<uint64_t>& offsets, int phase,
                  uint64_t epoch0, uint32_t* ids, float* dists, const uint32_t* sg_in,
                  uint32_t* sg_out, DistResult* res, uint64_t* epoch_out);

}  // namespace knng_b200
