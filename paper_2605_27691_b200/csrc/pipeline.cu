// pipeline.cu -- build_distributed (refine.cpp:504-586) on B200s.
//
// One host thread per rank (run_ranks, distsim.hpp:113-198), rank r on GPU
// devices[r % G] with its own stream.  Every rank-side phase body mirrors the
// reference line by line; the arithmetic runs in the kernels of
// nndescent.cu / graphopt.cu / search.cu / refine_kernels.cu and every
// cross-rank transfer is a one-sided NVLink peer pull through ThreadWorld.
#include "pipeline.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <memory>
#include <thread>

#include "graphopt.hpp"
#include "refine_kernels.hpp"

namespace knng_b200 {

namespace {

bool is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; }
uint64_t log2_exact(uint64_t v) {
  uint64_t l = 0;
  while ((uint64_t{1} << l) < v) ++l;
  return l;
}
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// KNNG_TRACE=1: per-rank phase timestamps (seconds since the call began)
double g_trace_t0 = 0;
void trace(size_t rank, const char* what) {
  static const bool on = std::getenv("KNNG_TRACE") != nullptr;
  if (on) std::fprintf(stderr, "[knng dist] rank %zu %-14s %8.1f ms\n", rank, what,
                       1e3 * (now_s() - g_trace_t0));
}

// KNNG_TRACE=2: also stamps inside phases, after draining the rank's stream
// (diagnosis only: it removes the overlap of the stamped steps)
struct RankState;
void trace_synced(RankState& R, const char* what);

const char* kDataset = "dataset";
const char* kGraph = "graph";
const char* kSGraph = "sgraph";

// a rank's runner: owned (fresh stream) or borrowed (the caller's persistent
// one, whose scratch buffers then survive across builds)
using RunnerPtr = std::unique_ptr<Runner, void (*)(Runner*)>;
RunnerPtr owned_runner(int dev) { return RunnerPtr(new Runner(dev), [](Runner* p) { delete p; }); }
RunnerPtr borrowed_runner(Runner* r) { return RunnerPtr(r, [](Runner*) {}); }

struct Shared {
  const RefineCfg* cfg = nullptr;
  std::vector<uint64_t> offsets;
  int d = 0;
  uint64_t k = 0, ks = 0, od = 0, groups = 1, levels = 0;
  SearchParamsDev sp;
  World* world = nullptr;
};

struct RankState {
  size_t rank = 0;
  RunnerPtr runner{nullptr, [](Runner*) {}};
  DBuf<float> local_x;
  uint64_t n_local = 0;
  DBuf<u64> keys;  // graph rows in internal global ids
  std::vector<DBuf<u64>> snaps;
  double local_t = 0, tree_t = 0, merge_t = 0, flat_t = 0;
  NndStats nst;
  SearchCounters sc;
  NndWorkspace* ws = nullptr;  // reusable local-build buffers (per-rank driver)
};

uint64_t size_of(const Shared& S, uint64_t r) { return S.offsets[r + 1] - S.offsets[r]; }

// validate_config refine.cpp:359-378
void validate_config(const std::vector<uint64_t>& offsets, const RefineCfg& cfg) {
  const uint64_t p = offsets.size() - 1;
  require(is_pow2(p), "refine: P must be a power of two");
  if (p > 1)
    require(is_pow2(cfg.groups) && cfg.groups >= 2 && cfg.groups <= p,
            "refine: M must be a power of two with 2 <= M <= P");
  uint64_t min_block = offsets[1] - offsets[0];
  for (uint64_t r = 1; r < p; ++r) min_block = std::min(min_block, offsets[r + 1] - offsets[r]);
  require(cfg.k < min_block, "refine: k must be < points per rank");
  const uint64_t ks = cfg.k_s ? cfg.k_s : cfg.k;
  require(ks <= min_block, "refine: k_s must be <= points per rank");
  const uint64_t od = cfg.out_degree ? cfg.out_degree : cfg.k;
  require(od <= cfg.k, "refine: out_degree must be <= k");
}

// effective_groups refine.cpp:160-183
uint64_t effective_groups(const std::vector<uint64_t>& offsets, const RefineCfg& cfg, int d) {
  const uint64_t p = offsets.size() - 1;
  if (p == 1) return 1;
  bool skip = cfg.skip_tree_phase;
  if (!skip && cfg.max_concat_bytes != 0) {
    const uint64_t gs = p / cfg.groups;
    uint64_t span = 0;
    for (uint64_t g = 0; g < cfg.groups; ++g)
      span = std::max(span, offsets[(g + 1) * gs] - offsets[g * gs]);
    const uint64_t od = cfg.out_degree ? cfg.out_degree : cfg.k;
    const uint64_t esz = cfg.u8_elems ? 1 : 4;  // refine.cpp:175-176
    const uint64_t est = span * ((uint64_t)d * esz + cfg.k * 8 + od * 4);
    if (est > cfg.max_concat_bytes) skip = true;
  }
  return skip ? p : cfg.groups;
}

// Cosine norm chains of n rows (row_norms_device); empty (p == null -> l2)
// unless the build runs the cosine metric.
DBuf<float> norms_of(const Shared& S, Runner& r, const float* x, uint64_t n) {
  DBuf<float> out;
  if (!S.cfg->cosine) return out;
  out.alloc(r, n ? n : 1);
  row_norms_device(r, x, n, S.d, out.p);
  return out;
}

void trace_synced(RankState& R, const char* what) {
  static const bool on = [] {
    const char* v = std::getenv("KNNG_TRACE");
    return v && std::atoi(v) >= 2;
  }();
  if (!on) return;
  R.runner->sync();
  trace(R.rank, what);
}

void pull_rows(Shared& S, RankState& R, uint64_t j, const char* name, void* dst) {
  S.world->get(R.rank, j, name, dst, *R.runner);
}
// the same pull, issued on another stream of the rank's device
void pull_rows_on(Shared& S, RankState& R, uint64_t j, const char* name, void* dst, Runner& on) {
  S.world->get(R.rank, j, name, dst, on);
}

// search the local points against (sg, vectors) and fold results into the
// rank's graph (refine.cpp:212-214, 332-333)
void search_and_merge(Shared& S, RankState& R, const u32* sg, const float* vec, uint64_t nvec,
                      uint64_t id_base) {
  Runner& r = *R.runner;
  DBuf<u32> rid(r, R.n_local * S.ks);
  DBuf<float> rd(r, R.n_local * S.ks);
  const DBuf<float> qn = norms_of(S, r, R.local_x.p, R.n_local), vn = norms_of(S, r, vec, nvec);
  ann_search_device(r, R.local_x.p, R.n_local, S.d, sg, (u32)S.od, vec, nvec, S.sp,
                    (u32)id_base, rid.p, rd.p, nullptr, nullptr, &R.sc, 0, qn.p, vn.p);
  trace_synced(R, "  search");
  merge_results_device(r, R.keys.p, nullptr, R.n_local, (u32)S.k, rid.p, rd.p, (u32)S.ks, 0);
}

void snapshot(RankState& R, uint64_t k) {
  Runner& r = *R.runner;
  R.snaps.emplace_back(r, R.n_local * k);
  KNNG_CUDA(cudaMemcpyAsync(R.snaps.back().p, R.keys.p, R.n_local * k * 8,
                            cudaMemcpyDeviceToDevice, r.stream));
}

// tree_level_rank refine.cpp:189-230
void tree_level(Shared& S, RankState& R, uint64_t level, DBuf<float>& span_x, uint64_t& span_lo,
                uint64_t& span_n) {
  Runner& r = *R.runner;
  const TreeLevel sched = tree_schedule(S.offsets.size() - 1, S.groups, R.rank, level);
  const uint64_t base = S.offsets[sched.partners.front()];
  const uint64_t cnt = S.offsets[sched.partners.back() + 1] - base;
  DBuf<float> px(r, cnt * S.d);
  DBuf<u64> pk(r, cnt * S.k);
  for (uint64_t j : sched.partners) {
    const uint64_t at = S.offsets[j] - base;
    pull_rows(S, R, j, kDataset, px.p + at * S.d);
    pull_rows(S, R, j, kGraph, pk.p + at * S.k);
  }
  trace_synced(R, "tree pulled");
  DBuf<u32> sg(r, cnt * S.od);
  {
    const DBuf<float> pn = norms_of(S, r, px.p, cnt);
    optimize_graph_device(r, pk.p, cnt, (u32)S.k, (u32)base, px.p, S.d, (u32)S.od, sg.p, nullptr,
                          pn.p);
  }
  trace_synced(R, "tree optimized");
  search_and_merge(S, R, sg.p, px.p, cnt, base);
  trace_synced(R, "tree merged");
  // accumulate the span dataset in rank order (refine.cpp:216-226)
  DBuf<float> ns(r, (span_n + cnt) * S.d);
  const size_t row = (size_t)S.d * 4;
  if (base < span_lo) {
    KNNG_CUDA(cudaMemcpyAsync(ns.p, px.p, cnt * row, cudaMemcpyDeviceToDevice, r.stream));
    KNNG_CUDA(cudaMemcpyAsync(ns.p + cnt * S.d, span_x.p, span_n * row, cudaMemcpyDeviceToDevice,
                              r.stream));
    span_lo = base;
  } else {
    KNNG_CUDA(cudaMemcpyAsync(ns.p, span_x.p, span_n * row, cudaMemcpyDeviceToDevice, r.stream));
    KNNG_CUDA(cudaMemcpyAsync(ns.p + span_n * S.d, px.p, cnt * row, cudaMemcpyDeviceToDevice,
                              r.stream));
  }
  span_n += cnt;
  span_x = std::move(ns);
  S.world->publish(R.rank, kGraph, R.keys.p, R.n_local * S.k * 8,
                   wire_region_size(RegionKind::knng, R.n_local, S.k), r);
  trace_synced(R, "tree published");
  S.world->barrier(R.rank, r);
}

// grouped_merge_rank refine.cpp:256-293; returns the group search graph.
// span_x == nullptr: the standalone driver (refine.cpp:272-283) -- the
// members' datasets are pulled too (graph then dataset per member).
DBuf<u32> grouped_merge(Shared& S, RankState& R, const float* span_x, uint64_t span_n) {
  Runner& r = *R.runner;
  const uint64_t p = S.offsets.size() - 1;
  const uint64_t gsz = p / S.groups;
  const uint64_t glo = (R.rank / gsz) * gsz, ghi = glo + gsz;
  const uint64_t base = S.offsets[glo];
  const uint64_t cnt = S.offsets[ghi] - base;
  DBuf<float> group_x;
  if (!span_x) group_x.alloc(r, cnt * S.d);
  require(!span_x || cnt == span_n, "grouped_merge: span/group size mismatch");
  DBuf<u64> concat(r, cnt * S.k);
  for (uint64_t j = glo; j < ghi; ++j) {
    u64* dst = concat.p + (S.offsets[j] - base) * S.k;
    float* xdst = span_x ? nullptr : group_x.p + (S.offsets[j] - base) * S.d;
    if (j == R.rank) {
      KNNG_CUDA(cudaMemcpyAsync(dst, R.keys.p, R.n_local * S.k * 8, cudaMemcpyDeviceToDevice,
                                r.stream));
      if (xdst)
        KNNG_CUDA(cudaMemcpyAsync(xdst, R.local_x.p, R.n_local * S.d * 4,
                                  cudaMemcpyDeviceToDevice, r.stream));
    } else {
      pull_rows(S, R, j, kGraph, dst);
      if (xdst) pull_rows(S, R, j, kDataset, xdst);
    }
  }
  if (!span_x) span_x = group_x.p;
  DBuf<u32> gs(r, cnt * S.od);
  {
    const DBuf<float> sn = norms_of(S, r, span_x, cnt);
    optimize_graph_device(r, concat.p, cnt, (u32)S.k, (u32)base, span_x, S.d, (u32)S.od, gs.p,
                          nullptr, sn.p);
  }
  S.world->publish(R.rank, kSGraph, gs.p, cnt * S.od * 4,
                   wire_region_size(RegionKind::sgraph, cnt, S.od), r);
  S.world->barrier(R.rank, r);
  return gs;
}

// flat_refine_rank refine.cpp:300-351
void flat_refine_double_buffered(Shared& S, RankState& R);

void flat_refine(Shared& S, RankState& R) {
  Runner& r = *R.runner;
  if (S.groups <= 1) return;
  if (S.cfg->double_buffer && S.groups > 2) return flat_refine_double_buffered(S, R);
  const uint64_t p = S.offsets.size() - 1;
  const uint64_t gsz = p / S.groups;
  const uint64_t my_group = R.rank / gsz, pos = R.rank % gsz;
  for (uint64_t step = 1; step < S.groups; ++step) {
    const uint64_t grp = (my_group + step) % S.groups;
    const uint64_t base = S.offsets[grp * gsz];
    const uint64_t cnt = S.offsets[(grp + 1) * gsz] - base;
    DBuf<u32> sg(r, cnt * S.od);
    // same-position rank in the target group, staggered across pullers
    pull_rows(S, R, grp * gsz + pos, kSGraph, sg.p);
    DBuf<float> vx(r, cnt * S.d);
    for (uint64_t j = grp * gsz; j < (grp + 1) * gsz; ++j)
      pull_rows(S, R, j, kDataset, vx.p + (S.offsets[j] - base) * S.d);
    trace_synced(R, "flat pulled");
    search_and_merge(S, R, sg.p, vx.p, cnt, base);
    trace_synced(R, "flat searched");
  }
  r.sync();
}

// double_buffer (refine.cpp:343-350): the next group's pulls (its search graph
// from the same-position rank + the member datasets, one-sided copies over
// NVLink) run on a second stream while the current group is searched; two
// buffer sets alternate, each reused only after the search that read it is
// done.  Same gets, same results -- only the overlap differs.
void flat_refine_double_buffered(Shared& S, RankState& R) {
  Runner& r = *R.runner;
  const uint64_t p = S.offsets.size() - 1;
  const uint64_t gsz = p / S.groups;
  const uint64_t my_group = R.rank / gsz, pos = R.rank % gsz;
  uint64_t max_cnt = 0;
  for (uint64_t g = 0; g < S.groups; ++g)
    max_cnt = std::max<uint64_t>(max_cnt, S.offsets[(g + 1) * gsz] - S.offsets[g * gsz]);
  DBuf<u32> sg[2] = {DBuf<u32>(r, max_cnt * S.od), DBuf<u32>(r, max_cnt * S.od)};
  DBuf<float> vx[2] = {DBuf<float>(r, max_cnt * S.d), DBuf<float>(r, max_cnt * S.d)};
  cudaStream_t side_s = nullptr;
  KNNG_CUDA(cudaStreamCreateWithFlags(&side_s, cudaStreamNonBlocking));
  cudaEvent_t landed[2], freed[2];
  for (int b = 0; b < 2; ++b) {
    KNNG_CUDA(cudaEventCreateWithFlags(&landed[b], cudaEventDisableTiming));
    KNNG_CUDA(cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming));
    KNNG_CUDA(cudaEventRecord(freed[b], r.stream));  // buffers allocated on r.stream
  }
  struct Cleanup {
    cudaStream_t s;
    cudaEvent_t* e;
    ~Cleanup() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  };
  cudaEvent_t evs[4] = {landed[0], landed[1], freed[0], freed[1]};
  Cleanup cleanup{side_s, evs};
  Runner side(r.device, side_s);
  auto fetch = [&](uint64_t step, int b) {
    const uint64_t grp = (my_group + step) % S.groups;
    const uint64_t base = S.offsets[grp * gsz];
    KNNG_CUDA(cudaStreamWaitEvent(side_s, freed[b], 0));
    pull_rows_on(S, R, grp * gsz + pos, kSGraph, sg[b].p, side);
    for (uint64_t j = grp * gsz; j < (grp + 1) * gsz; ++j)
      pull_rows_on(S, R, j, kDataset, vx[b].p + (S.offsets[j] - base) * S.d, side);
    KNNG_CUDA(cudaEventRecord(landed[b], side_s));
  };
  fetch(1, 0);
  for (uint64_t step = 1; step < S.groups; ++step) {
    const int b = (int)((step - 1) & 1);
    if (step + 1 < S.groups) fetch(step + 1, b ^ 1);
    const uint64_t grp = (my_group + step) % S.groups;
    const uint64_t base = S.offsets[grp * gsz];
    const uint64_t cnt = S.offsets[(grp + 1) * gsz] - base;
    KNNG_CUDA(cudaStreamWaitEvent(r.stream, landed[b], 0));
    search_and_merge(S, R, sg[b].p, vx[b].p, cnt, base);
    KNNG_CUDA(cudaEventRecord(freed[b], r.stream));
  }
  r.sync();
}

// all_to_all_refine refine.cpp:473-502
void a2a_refine(Shared& S, RankState& R) {
  Runner& r = *R.runner;
  const uint64_t p = S.offsets.size() - 1;
  DBuf<u32> own(r, R.n_local * S.od);
  {
    const DBuf<float> ln = norms_of(S, r, R.local_x.p, R.n_local);
    optimize_graph_device(r, R.keys.p, R.n_local, (u32)S.k, (u32)S.offsets[R.rank], R.local_x.p,
                          S.d, (u32)S.od, own.p, nullptr, ln.p);
  }
  S.world->publish(R.rank, kDataset, R.local_x.p, R.n_local * S.d * 4,
                   wire_region_size(RegionKind::dataset, R.n_local, S.d, S.cfg->u8_elems), r);
  S.world->publish(R.rank, kSGraph, own.p, R.n_local * S.od * 4,
                   wire_region_size(RegionKind::sgraph, R.n_local, S.od), r);
  S.world->barrier(R.rank, r);
  for (uint64_t step = 1; step < p; ++step) {
    const uint64_t j = (R.rank + step) % p;
    const uint64_t cnt = size_of(S, j);
    DBuf<u32> sg(r, cnt * S.od);
    DBuf<float> vx(r, cnt * S.d);
    pull_rows(S, R, j, kSGraph, sg.p);
    pull_rows(S, R, j, kDataset, vx.p);
    search_and_merge(S, R, sg.p, vx.p, cnt, S.offsets[j]);
  }
  r.sync();
}

// The refine body of build_distributed refine.cpp:532-549 (after the local
// build), shared with the standalone drivers.
void refine_rank(Shared& S, RankState& R, bool capture) {
  Runner& r = *R.runner;
  S.world->publish(R.rank, kDataset, R.local_x.p, R.n_local * S.d * 4,
                   wire_region_size(RegionKind::dataset, R.n_local, S.d, S.cfg->u8_elems), r);
  S.world->publish(R.rank, kGraph, R.keys.p, R.n_local * S.k * 8,
                   wire_region_size(RegionKind::knng, R.n_local, S.k), r);
  S.world->barrier(R.rank, r);
  trace(R.rank, "published");

  double t = now_s();
  DBuf<float> span_x(r, R.n_local * S.d);
  KNNG_CUDA(cudaMemcpyAsync(span_x.p, R.local_x.p, R.n_local * S.d * 4, cudaMemcpyDeviceToDevice,
                            r.stream));
  uint64_t span_lo = S.offsets[R.rank], span_n = R.n_local;
  for (uint64_t level = 0; level < S.levels; ++level) {
    tree_level(S, R, level, span_x, span_lo, span_n);
    if (capture) snapshot(R, S.k);
  }
  r.sync();
  R.tree_t = now_s() - t;
  trace(R.rank, "tree");

  t = now_s();
  DBuf<u32> gs = grouped_merge(S, R, span_x.p, span_n);
  r.sync();
  R.merge_t = now_s() - t;
  trace(R.rank, "merge");

  t = now_s();
  flat_refine(S, R);
  R.flat_t = now_s() - t;
  trace(R.rank, "flat");
  if (capture) snapshot(R, S.k);
  r.sync();
}

// local_build_rank refine.cpp:380-390: nn_descent on the rank's rows, seed
// mix(nn.seed, rank) for P > 1, ids shifted to internal global ids
void local_build_rank(Shared& S, const RefineCfg& cfg, RankState& R) {
  Runner& r = *R.runner;
  DeviceGuard g(r.device);
  const double t = now_s();
  const uint64_t p = S.offsets.size() - 1;
  NndParams np = cfg.nn;
  np.k = (uint32_t)cfg.k;
  np.seed = p == 1 ? cfg.nn.seed : mix_seed(cfg.nn.seed, R.rank);  // refine.cpp:385
  DBuf<u32> flags(r, R.n_local);
  const DBuf<float> ln = norms_of(S, r, R.local_x.p, R.n_local);
  nn_descent_device(r, DevRows{R.local_x.p, R.n_local, S.d, ln.p}, np, R.keys.p, flags.p, &R.nst,
                    true, R.ws);
  shift_ids_device(r, R.keys.p, R.n_local * S.k, (int64_t)S.offsets[R.rank]);
  r.sync();
  R.local_t = now_s() - t;
  trace(R.rank, "local");
  if (cfg.capture_snapshots) snapshot(R, S.k);
}

// run body(rank) on one thread per rank; first genuine failure rethrown
// (RankRunner distsim.hpp:113-153)
template <class Body>
void run_ranks(World& world, size_t p, Body&& body) {
  std::vector<std::exception_ptr> errors(p);
  std::vector<std::thread> threads;
  threads.reserve(p);
  for (size_t i = 0; i < p; ++i) {
    threads.emplace_back([&, i] {
      try {
        body(i);
      } catch (...) {
        errors[i] = std::current_exception();
        world.abort("rank " + std::to_string(i) + " failed");
      }
    });
  }
  for (auto& t : threads) t.join();
  std::exception_ptr first;
  for (auto& e : errors) {
    if (!e) continue;
    if (!first) first = e;
    try {
      std::rethrow_exception(e);
    } catch (const WorldAborted&) {
    } catch (...) {
      first = e;
      break;
    }
  }
  if (first) std::rethrow_exception(first);
}

Shared make_shared_state(const RefineCfg& cfg, const std::vector<uint64_t>& offsets, int d) {
  Shared S;
  S.cfg = &cfg;
  S.offsets = offsets;
  S.d = d;
  S.k = cfg.k;
  S.ks = cfg.k_s ? cfg.k_s : cfg.k;
  S.od = cfg.out_degree ? cfg.out_degree : cfg.k;
  S.groups = effective_groups(offsets, cfg, d);
  S.levels = tree_levels(offsets.size() - 1, S.groups);
  // effective_search_params refine.cpp:153-158
  S.sp = cfg.search;
  S.sp.k_s = S.ks;
  return S;
}

// Assemble per-rank key buffers (internal order) on device 0 and translate.
void translate_all(Runner& r0, std::vector<RankState>& ranks, const std::vector<uint64_t>& offsets,
                   uint64_t k, const u32* to_ext, uint32_t* out_ids, float* out_d,
                   bool out_on_device, int which_snap) {
  const uint64_t n = offsets.back();
  DBuf<u64> all(r0, n * k);
  for (auto& R : ranks) {
    const u64* src = which_snap < 0 ? R.keys.p : R.snaps[which_snap].p;
    R.runner->sync();
    if (R.runner->device == r0.device)
      KNNG_CUDA(cudaMemcpyAsync(all.p + offsets[R.rank] * k, src, R.n_local * k * 8,
                                cudaMemcpyDeviceToDevice, r0.stream));
    else
      KNNG_CUDA(cudaMemcpyPeerAsync(all.p + offsets[R.rank] * k, r0.device, src,
                                    R.runner->device, R.n_local * k * 8, r0.stream));
  }
  if (out_on_device) {
    translate_device(r0, all.p, n, (u32)k, to_ext, out_ids, out_d);
  } else {
    DBuf<u32> ti(r0, n * k);
    DBuf<float> td(r0, n * k);
    translate_device(r0, all.p, n, (u32)k, to_ext, ti.p, td.p);
    d2h_host(r0, out_ids, ti.p, n * k * 4);
    d2h_host(r0, out_d, td.p, n * k * 4);
  }
  r0.sync();
}

void fill_result(Shared& S, std::vector<RankState>& ranks, World* world, DistResult* res) {
  if (!res) return;
  for (auto& R : ranks) {
    res->local_s = std::max(res->local_s, R.local_t);
    res->tree_s = std::max(res->tree_s, R.tree_t);
    res->merge_s = std::max(res->merge_s, R.merge_t);
    res->flat_s = std::max(res->flat_s, R.flat_t);
    res->nnd_iterations_max = std::max<uint64_t>(res->nnd_iterations_max, R.nst.iterations);
    res->nnd_pairs += R.nst.pairs;
    res->nnd_staged_rows += R.nst.staged_rows;
    res->join_ms_max = std::max(res->join_ms_max, R.nst.join_ms);
    res->search.hops += R.sc.hops;
    res->search.scored += R.sc.scored;
    res->search.overflowed += R.sc.overflowed;
    res->search.launches += R.sc.launches;
  }
  const uint64_t p = S.offsets.size() - 1;
  res->levels = S.levels;
  res->merge_epoch = p == 1 ? 0 : S.levels + 1;
  res->flat_epoch = p == 1 ? 0 : S.levels + 2;
  if (world) res->comm_log = world->comm_log();
}

}  // namespace

uint64_t effective_group_count(const std::vector<uint64_t>& offsets, const RefineCfg& cfg,
                               int d) {
  return effective_groups(offsets, cfg, d);
}

uint64_t tree_levels(uint64_t ranks, uint64_t groups) {
  require(is_pow2(ranks) && is_pow2(groups) && groups <= ranks, "tree_levels: invalid P or M");
  return log2_exact(ranks / groups);
}

TreeLevel tree_schedule(uint64_t ranks, uint64_t groups, uint64_t rank, uint64_t level) {
  const uint64_t levels = tree_levels(ranks, groups);
  require(rank < ranks, "tree_schedule: rank out of range");
  require(level < levels, "tree_schedule: level out of range");
  const uint64_t size = uint64_t{1} << level;
  const uint64_t block = rank / size;
  TreeLevel t;
  t.group_lo = block * size;
  t.group_hi = t.group_lo + size;
  const uint64_t plo = (block ^ 1u) * size;
  t.partners.resize(size);
  for (uint64_t i = 0; i < size; ++i) t.partners[i] = plo + i;
  return t;
}

void build_distributed(const std::vector<int>& devices, const float* X, bool x_on_device,
                       uint64_t n, int d, const RefineCfg& cfg, uint32_t* out_ids,
                       float* out_dists, bool out_on_device, DistResult* res) {
  require(!devices.empty(), "build_distributed: no CUDA device");
  const uint64_t p = cfg.ranks;
  require(!(p == 0 || p > n), "partition_dataset: need 1 <= P <= N");
  Runner r0(devices[0]);
  DeviceGuard g0(r0.device);
  double t0 = now_s();
  g_trace_t0 = t0;
  // dataset resident on device 0
  DBuf<float> xdev;
  const float* Xd = X;
  if (!x_on_device) {
    xdev.alloc(r0, n * d);
    KNNG_CUDA(cudaMemcpyAsync(xdev.p, X, n * (uint64_t)d * 4, cudaMemcpyHostToDevice, r0.stream));
    Xd = xdev.p;
  }
  // partition refine.cpp:86-126 (bit-exact permutation on the GPU)
  DBuf<u32> to_ext(r0, n);
  std::vector<uint64_t> offsets;
  partition_device(r0, n, (uint32_t)p, cfg.seed, to_ext.p, offsets);
  validate_config(offsets, cfg);
  Shared S = make_shared_state(cfg, offsets, d);
  std::vector<RankState> ranks(p);
  for (uint64_t i = 0; i < p; ++i) {
    RankState& R = ranks[i];
    R.rank = i;
    R.runner = owned_runner(devices[i % devices.size()]);
    R.n_local = size_of(S, i);
    R.local_x.alloc(*R.runner, R.n_local * d);
    R.keys.alloc(*R.runner, R.n_local * S.k);
  }
  {
    // gather each rank's rows: to_external block -> rows (on device 0), then
    // NVLink peer copy to the rank's GPU
    for (auto& R : ranks) {
      DBuf<float> tmp(r0, R.n_local * d);
      gather_rows_device(r0, Xd, d, to_ext.p + offsets[R.rank], R.n_local, tmp.p);
      r0.sync();
      R.runner->sync();
      if (R.runner->device == r0.device)
        KNNG_CUDA(cudaMemcpyAsync(R.local_x.p, tmp.p, R.n_local * d * 4,
                                  cudaMemcpyDeviceToDevice, r0.stream));
      else
        KNNG_CUDA(cudaMemcpyPeerAsync(R.local_x.p, R.runner->device, tmp.p, r0.device,
                                      R.n_local * d * 4, r0.stream));
      r0.sync();
    }
    if (!x_on_device) xdev.release();
  }
  if (res) res->partition_s = now_s() - t0;
  trace(0, "partitioned");

  auto local_build = [&](RankState& R) { local_build_rank(S, cfg, R); };

  std::unique_ptr<ThreadWorld> world;
  if (p == 1) {
    local_build(ranks[0]);
  } else {
    world = std::make_unique<ThreadWorld>(p);
    S.world = world.get();
    run_ranks(*world, p, [&](size_t i) {
      RankState& R = ranks[i];
      DeviceGuard g(R.runner->device);
      local_build(R);
      refine_rank(S, R, cfg.capture_snapshots);
    });
  }
  const double te = now_s();
  trace(0, "ranks joined");
  translate_all(r0, ranks, offsets, S.k, to_ext.p, out_ids, out_dists, out_on_device, -1);
  trace(0, "translated");
  if (res) {
    fill_result(S, ranks, world.get(), res);
    res->etc_s = now_s() - te;
    if (cfg.capture_snapshots) {
      const size_t ns = ranks[0].snaps.size();
      for (size_t s = 0; s < ns; ++s) {
        std::string label = s == 0 ? "local"
                            : (s <= S.levels ? "tree_level_" + std::to_string(s - 1) : "flat");
        res->snap_labels.push_back(label);
        res->snap_ids.emplace_back(n * S.k);
        res->snap_dists.emplace_back(n * S.k);
        translate_all(r0, ranks, offsets, S.k, to_ext.p, res->snap_ids.back().data(),
                      res->snap_dists.back().data(), false, (int)s);
      }
    }
  }
}

void refine_from_local(const std::vector<int>& devices, const float* X_perm, uint64_t n, int d,
                       const RefineCfg& cfg, const std::vector<uint64_t>& offsets, uint32_t* ids,
                       float* dists, int mode, DistResult* res) {
  require(!devices.empty(), "refine: no CUDA device");
  require(offsets.size() == cfg.ranks + 1 && offsets.back() == n, "refine: bad offsets");
  validate_config(offsets, cfg);
  Shared S = make_shared_state(cfg, offsets, d);
  const uint64_t p = cfg.ranks;
  std::vector<RankState> ranks(p);
  for (uint64_t i = 0; i < p; ++i) {
    RankState& R = ranks[i];
    R.rank = i;
    R.runner = owned_runner(devices[i % devices.size()]);
    Runner& r = *R.runner;
    DeviceGuard g(r.device);
    R.n_local = size_of(S, i);
    R.local_x.alloc(r, R.n_local * d);
    R.keys.alloc(r, R.n_local * S.k);
    KNNG_CUDA(cudaMemcpyAsync(R.local_x.p, X_perm + offsets[i] * d, R.n_local * d * 4,
                              cudaMemcpyHostToDevice, r.stream));
    DBuf<u32> ti(r, R.n_local * S.k);
    DBuf<float> td(r, R.n_local * S.k);
    KNNG_CUDA(cudaMemcpyAsync(ti.p, ids + offsets[i] * S.k, R.n_local * S.k * 4,
                              cudaMemcpyHostToDevice, r.stream));
    KNNG_CUDA(cudaMemcpyAsync(td.p, dists + offsets[i] * S.k, R.n_local * S.k * 4,
                              cudaMemcpyHostToDevice, r.stream));
    import_graph_device(r, ti.p, td.p, nullptr, R.n_local, (u32)S.k, R.keys.p, nullptr);
    r.sync();
  }
  ThreadWorld world(p);
  S.world = &world;
  if (p > 1) {
    run_ranks(world, p, [&](size_t i) {
      RankState& R = ranks[i];
      DeviceGuard g(R.runner->device);
      if (mode == 1)
        a2a_refine(S, R);
      else
        refine_rank(S, R, false);
    });
  }
  for (auto& R : ranks) {
    Runner& r = *R.runner;
    DeviceGuard g(r.device);
    DBuf<u32> ti(r, R.n_local * S.k);
    DBuf<float> td(r, R.n_local * S.k);
    export_graph_device(r, R.keys.p, nullptr, R.n_local, (u32)S.k, 0, ti.p, td.p, nullptr);
    KNNG_CUDA(cudaMemcpyAsync(ids + offsets[R.rank] * S.k, ti.p, R.n_local * S.k * 4,
                              cudaMemcpyDeviceToHost, r.stream));
    KNNG_CUDA(cudaMemcpyAsync(dists + offsets[R.rank] * S.k, td.p, R.n_local * S.k * 4,
                              cudaMemcpyDeviceToHost, r.stream));
    r.sync();
  }
  fill_result(S, ranks, &world, res);
}

// The world-level phase drivers one at a time (refine.cpp:430-502): each
// publishes what its phase needs, barriers, and runs its phase on every rank.
//   phase 1 all_to_all_refine:  ids/dists in/out
// The world starts at epoch `epoch0` (the caller's RankWorld may have run
// earlier drivers); `epoch_out` receives its epoch at the end.
//   phase 2 binary_tree_refine: ids/dists in/out
//   phase 3 grouped_merge:      sg_out[rank block] = the rank's group search graph
//   phase 4 flat_refine:        sg_in[rank block] = group_graphs[rank]; ids/dists in/out
// sg blocks: rank r's block holds group_n(r) x out_degree ids, blocks in rank order.
void refine_phase(const std::vector<int>& devices, const float* X_perm, uint64_t n, int d,
                  const RefineCfg& cfg, const std::vector<uint64_t>& offsets, int phase,
                  uint64_t epoch0, uint32_t* ids, float* dists, const uint32_t* sg_in,
                  uint32_t* sg_out, DistResult* res, uint64_t* epoch_out) {
  require(!devices.empty(), "refine: no CUDA device");
  require(offsets.size() == cfg.ranks + 1 && offsets.back() == n, "refine: bad offsets");
  require(phase >= 1 && phase <= 4, "refine: unknown phase");
  validate_config(offsets, cfg);
  Shared S = make_shared_state(cfg, offsets, d);
  const uint64_t p = cfg.ranks;
  const uint64_t gsz = p / S.groups;
  auto group_n = [&](uint64_t r) {
    const uint64_t glo = (r / gsz) * gsz;
    return S.offsets[glo + gsz] - S.offsets[glo];
  };
  std::vector<uint64_t> sg_off(p + 1, 0);
  for (uint64_t r = 0; r < p; ++r) sg_off[r + 1] = sg_off[r] + group_n(r) * S.od;
  require(phase <= 2 || (phase == 3 ? sg_out != nullptr : sg_in != nullptr),
          "refine: search-graph buffer expected");
  std::vector<RankState> ranks(p);
  for (uint64_t i = 0; i < p; ++i) {
    RankState& R = ranks[i];
    R.rank = i;
    R.runner = owned_runner(devices[i % devices.size()]);
    Runner& r = *R.runner;
    DeviceGuard g(r.device);
    R.n_local = size_of(S, i);
    R.local_x.alloc(r, R.n_local * d);
    R.keys.alloc(r, R.n_local * S.k);
    KNNG_CUDA(cudaMemcpyAsync(R.local_x.p, X_perm + offsets[i] * d, R.n_local * d * 4,
                              cudaMemcpyHostToDevice, r.stream));
    DBuf<u32> ti(r, R.n_local * S.k);
    DBuf<float> td(r, R.n_local * S.k);
    KNNG_CUDA(cudaMemcpyAsync(ti.p, ids + offsets[i] * S.k, R.n_local * S.k * 4,
                              cudaMemcpyHostToDevice, r.stream));
    KNNG_CUDA(cudaMemcpyAsync(td.p, dists + offsets[i] * S.k, R.n_local * S.k * 4,
                              cudaMemcpyHostToDevice, r.stream));
    import_graph_device(r, ti.p, td.p, nullptr, R.n_local, (u32)S.k, R.keys.p, nullptr);
    r.sync();
  }
  ThreadWorld world(p, std::chrono::seconds(600), epoch0);
  S.world = &world;
  run_ranks(world, p, [&](size_t i) {
    RankState& R = ranks[i];
    Runner& r = *R.runner;
    DeviceGuard g(r.device);
    if (phase == 1) {  // all_to_all_refine publishes and barriers itself
      const double t = now_s();
      a2a_refine(S, R);
      R.flat_t = now_s() - t;
      return;
    }
    S.world->publish(R.rank, kDataset, R.local_x.p, R.n_local * S.d * 4,
                     wire_region_size(RegionKind::dataset, R.n_local, S.d, S.cfg->u8_elems), r);
    if (phase == 4) {
      const uint64_t cnt = group_n(i);
      DBuf<u32> gs(r, cnt * S.od);
      KNNG_CUDA(cudaMemcpyAsync(gs.p, sg_in + sg_off[i], cnt * S.od * 4, cudaMemcpyHostToDevice,
                                r.stream));
      S.world->publish(R.rank, kSGraph, gs.p, cnt * S.od * 4,
                       wire_region_size(RegionKind::sgraph, cnt, S.od), r);
    } else {
      S.world->publish(R.rank, kGraph, R.keys.p, R.n_local * S.k * 8,
                       wire_region_size(RegionKind::knng, R.n_local, S.k), r);
    }
    S.world->barrier(R.rank, r);
    const double t = now_s();
    if (phase == 2) {
      DBuf<float> span_x(r, R.n_local * S.d);
      KNNG_CUDA(cudaMemcpyAsync(span_x.p, R.local_x.p, R.n_local * S.d * 4,
                                cudaMemcpyDeviceToDevice, r.stream));
      uint64_t span_lo = S.offsets[R.rank], span_n = R.n_local;
      for (uint64_t level = 0; level < S.levels; ++level)
        tree_level(S, R, level, span_x, span_lo, span_n);
      r.sync();
      R.tree_t = now_s() - t;
    } else if (phase == 3) {
      DBuf<u32> gs = grouped_merge(S, R, nullptr, 0);
      KNNG_CUDA(cudaMemcpyAsync(sg_out + sg_off[i], gs.p, group_n(i) * S.od * 4,
                                cudaMemcpyDeviceToHost, r.stream));
      r.sync();
      R.merge_t = now_s() - t;
    } else {
      flat_refine(S, R);
      R.flat_t = now_s() - t;
    }
  });
  if (phase != 3) {
    for (auto& R : ranks) {
      Runner& r = *R.runner;
      DeviceGuard g(r.device);
      DBuf<u32> ti(r, R.n_local * S.k);
      DBuf<float> td(r, R.n_local * S.k);
      export_graph_device(r, R.keys.p, nullptr, R.n_local, (u32)S.k, 0, ti.p, td.p, nullptr);
      KNNG_CUDA(cudaMemcpyAsync(ids + offsets[R.rank] * S.k, ti.p, R.n_local * S.k * 4,
                                cudaMemcpyDeviceToHost, r.stream));
      KNNG_CUDA(cudaMemcpyAsync(dists + offsets[R.rank] * S.k, td.p, R.n_local * S.k * 4,
                                cudaMemcpyDeviceToHost, r.stream));
      r.sync();
    }
  }
  fill_result(S, ranks, &world, res);
  if (epoch_out) *epoch_out = world.epoch();
}

uint64_t build_distributed_rank(int device, size_t rank, size_t ranks, const HostTransport& t,
                                const float* X, bool x_on_device, uint64_t n, int d,
                                const RefineCfg& cfg_in, uint32_t* out_ids, float* out_dists,
                                uint32_t* out_rows, bool out_on_device, DistResult* res,
                                Runner* base, NndWorkspace* ws) {
  RefineCfg cfg = cfg_in;
  cfg.ranks = ranks;
  require(rank < ranks, "build_distributed: rank out of range");
  require(!(ranks == 0 || ranks > n), "partition_dataset: need 1 <= P <= N");
  require(!cfg.capture_snapshots, "build_distributed: snapshots need the single-process driver");
  // the rank state (and its runner/stream) is declared first so it outlives
  // every buffer below that frees on its stream
  std::vector<RankState> one(1);
  RankState& R = one[0];
  R.rank = rank;
  // on the caller's persistent runner when given (its workspace and scratch
  // buffers are stream-ordered on it and reused across builds), else a fresh one
  R.runner = base ? borrowed_runner(base) : owned_runner(device);
  R.ws = ws;
  Runner& r = *R.runner;
  DeviceGuard g(r.device);
  const double t0 = now_s();
  g_trace_t0 = t0;
  DBuf<float> xdev;
  const float* Xd = X;
  if (!x_on_device) {
    // A rank needs only its own block (remote rows arrive over NVLink from
    // their owners), but its rows are a random 1/P of the dataset: gathering
    // them zero-copy over PCIe (KNNG_ZEROCOPY=1, pinned memory only) made
    // many small random reads -- C4 N = 2 e2e 3.80 s per step vs 2.81 s with
    // one bulk copy of the whole dataset and a gather on the device (the
    // default).
    void* mapped = nullptr;
    const char* zc = std::getenv("KNNG_ZEROCOPY");
    const bool zero_copy = zc && *zc && std::atoi(zc) != 0;
    if (zero_copy &&
        cudaHostGetDevicePointer(&mapped, const_cast<float*>(X), 0) == cudaSuccess && mapped) {
      Xd = static_cast<const float*>(mapped);
    } else {
      cudaGetLastError();
      xdev.alloc(r, n * d);
      KNNG_CUDA(cudaMemcpyAsync(xdev.p, X, n * (uint64_t)d * 4, cudaMemcpyHostToDevice,
                                r.stream));
      Xd = xdev.p;
    }
  }
  // every rank computes the same permutation (refine.cpp:86-126, bit-exact)
  DBuf<u32> to_ext(r, n);
  std::vector<uint64_t> offsets;
  partition_device(r, n, (uint32_t)ranks, cfg.seed, to_ext.p, offsets);
  validate_config(offsets, cfg);
  Shared S = make_shared_state(cfg, offsets, d);
  R.n_local = size_of(S, rank);
  R.local_x.alloc(r, R.n_local * d);
  R.keys.alloc(r, R.n_local * S.k);
  gather_rows_device(r, Xd, d, to_ext.p + offsets[rank], R.n_local, R.local_x.p);
  if (!x_on_device) xdev.release();
  r.sync();
  if (res) res->partition_s = now_s() - t0;
  std::unique_ptr<ProcWorld> world;
  if (ranks > 1) {
    world = std::make_unique<ProcWorld>(ranks, rank, t);
    S.world = world.get();
  }
  try {
    local_build_rank(S, cfg, R);
    // failure injection for the abort-propagation test (tests/test_multiprocess_gpu.py)
    if (const char* f = std::getenv("KNNG_INJECT_FAIL_RANK"))
      if (std::atoi(f) == (int)rank)
        throw std::runtime_error("injected failure at rank " + std::to_string(rank));
    if (ranks > 1) refine_rank(S, R, false);
  } catch (const std::exception& e) {
    // a failing rank aborts the world so that its peers' barriers return
    // WorldAborted instead of waiting for it (RankRunner distsim.hpp:127-129)
    if (world) world->abort("rank " + std::to_string(rank) + " failed: " + e.what());
    throw;
  }
  const double te = now_s();
  if (out_on_device) {
    translate_rows_device(r, R.keys.p, R.n_local, (u32)S.k, to_ext.p, offsets[rank], out_ids,
                          out_dists, out_rows);
  } else {
    DBuf<u32> ti(r, R.n_local * S.k), tr(r, R.n_local);
    DBuf<float> td(r, R.n_local * S.k);
    translate_rows_device(r, R.keys.p, R.n_local, (u32)S.k, to_ext.p, offsets[rank], ti.p, td.p,
                          tr.p);
    d2h_host(r, out_ids, ti.p, R.n_local * S.k * 4);
    d2h_host(r, out_dists, td.p, R.n_local * S.k * 4);
    d2h_host(r, out_rows, tr.p, R.n_local * 4);
  }
  r.sync();
  if (res) {
    fill_result(S, one, nullptr, res);
    res->etc_s = now_s() - te;
    if (world) res->comm_log = world->gather_comm_log();
  }
  return R.n_local;
}

}  // namespace knng_b200
