// knng_b200.hpp -- header-only C++ drop-in for the reference's public API
// (/root/reference/proj/include/knng/*.hpp) on top of the C-ABI in knng_c.h.
//
// A reference user swaps `#include "knng/..."` for this header and links
// libknng_b200.so: same namespace, type names, field names, function
// signatures and exception classes for the kNN-graph construction path
// (partition -> local build -> remote refine -> merge -> graph output).
// Internal building blocks of the CPU implementation that the GPU design does
// not have (CandidateBuffer, NeighborSamples' vectors, local_join,
// parallel_for) are not part of this surface; see INTEGRATION.md.  The
// host-side parts of the reference API (Rng, wire regions, RankWorld and its
// world-level phase drivers, the cost model) are in knng_b200_host.hpp,
// included at the end; include/knng/*.hpp forward the reference's header
// names here, so the reference's own sources compile unchanged against it.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <filesystem>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "knng_c.h"

namespace knng {

using PointId = std::uint32_t;
enum class ElemKind : std::uint8_t { f32 = 0, u8 = 1 };
enum class MetricKind : std::uint8_t { l2 = 0, cosine = 1 };
enum class IdSpace : std::uint8_t { local = 0, global = 1 };

// exception classes (distsim.hpp:19-26, evalio.hpp:14-16)
struct WorldError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct WorldAborted : WorldError {
  using WorldError::WorldError;
};
struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(knng_status s) {
  if (s == KNNG_OK) return;
  const std::string m = knng_last_error();
  switch (s) {
    case KNNG_EINVAL: throw std::invalid_argument(m);
    case KNNG_EWORLD: throw WorldError(m);
    case KNNG_EABORTED: throw WorldAborted(m);
    case KNNG_EFORMAT: throw FormatError(m);
    case KNNG_ELOGIC: throw std::logic_error(m);
    case KNNG_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(m);
  }
}
// One context per process (knng_c.h threading rule), created on first use.
inline knng_ctx* ctx() {
  static std::unique_ptr<knng_ctx, void (*)(knng_ctx*)> c = [] {
    knng_ctx* h = nullptr;
    check(knng_ctx_create(0, &h));
    return std::unique_ptr<knng_ctx, void (*)(knng_ctx*)>(h, knng_ctx_destroy);
  }();
  return c.get();
}
}  // namespace detail

inline const char* to_string(MetricKind m) { return m == MetricKind::l2 ? "l2" : "cosine"; }
inline MetricKind metric_from_string(const std::string& s) {
  if (s == "l2") return MetricKind::l2;
  if (s == "cosine") return MetricKind::cosine;
  throw std::invalid_argument("unknown metric: " + s);
}

// sigma core.hpp:23-55 on the host (the exact operation order of the
// reference: per dimension a separately rounded subtract, multiply and add,
// then sqrt -- compile callers with -ffp-contract=off).  The library computes
// every distance of a build on the GPU in this same order; these host forms
// serve measurement code and Dataset::row_distance.
namespace detail {
template <class T>
inline float l2_exact(const T* a, const T* b, std::size_t d) {
  float acc = 0.0f;
  for (std::size_t i = 0; i < d; ++i) {
    const float t = static_cast<float>(a[i]) - static_cast<float>(b[i]);
    const float sq = t * t;
    acc = acc + sq;
  }
  return std::sqrt(acc);
}
inline float l2_f32(const float* a, const float* b, std::size_t d) { return l2_exact(a, b, d); }
inline float l2_u8(const std::uint8_t* a, const std::uint8_t* b, std::size_t d) {
  return l2_exact(a, b, d);
}
template <class T>
inline float cosine_t(const T* a, const T* b, std::size_t d) {
  float dot = 0.0f, na = 0.0f, nb = 0.0f;
  for (std::size_t i = 0; i < d; ++i) {
    const float x = static_cast<float>(a[i]), y = static_cast<float>(b[i]);
    const float xy = x * y, xx = x * x, yy = y * y;
    dot = dot + xy;
    na = na + xx;
    nb = nb + yy;
  }
  if (na == 0.0f || nb == 0.0f) return 1.0f;
  const float v = 1.0f - dot / (std::sqrt(na) * std::sqrt(nb));
  return v < 0.0f ? 0.0f : v;
}
}  // namespace detail

inline float distance(MetricKind m, std::span<const float> a, std::span<const float> b) {
  if (a.size() != b.size()) throw std::invalid_argument("distance: dimension mismatch");
  return m == MetricKind::l2 ? detail::l2_f32(a.data(), b.data(), a.size())
                             : detail::cosine_t(a.data(), b.data(), a.size());
}
inline float distance(MetricKind m, std::span<const std::uint8_t> a,
                      std::span<const std::uint8_t> b) {
  if (a.size() != b.size()) throw std::invalid_argument("distance: dimension mismatch");
  return m == MetricKind::l2 ? detail::l2_u8(a.data(), b.data(), a.size())
                             : detail::cosine_t(a.data(), b.data(), a.size());
}

// Dataset core.hpp:67-105 (f32 or u8 rows; l2 or cosine)
struct Dataset {
  std::size_t num_points = 0;
  std::size_t dims = 0;
  ElemKind elem_kind = ElemKind::f32;
  MetricKind metric = MetricKind::l2;
  std::vector<float> f32;
  std::vector<std::uint8_t> u8;

  static Dataset empty(std::size_t dims, ElemKind kind, MetricKind metric) {
    Dataset d;
    d.dims = dims;
    d.elem_kind = kind;
    d.metric = metric;
    return d;
  }
  std::span<const float> frow(std::size_t i) const { return {f32.data() + i * dims, dims}; }
  std::span<const std::uint8_t> brow(std::size_t i) const {
    return {u8.data() + i * dims, dims};
  }
  float row_distance(std::size_t i, std::size_t j) const {
    if (elem_kind == ElemKind::f32)
      return metric == MetricKind::l2
                 ? detail::l2_f32(f32.data() + i * dims, f32.data() + j * dims, dims)
                 : detail::cosine_t(f32.data() + i * dims, f32.data() + j * dims, dims);
    return metric == MetricKind::l2
               ? detail::l2_u8(u8.data() + i * dims, u8.data() + j * dims, dims)
               : detail::cosine_t(u8.data() + i * dims, u8.data() + j * dims, dims);
  }
  Dataset slice(std::size_t begin, std::size_t count) const {
    if (begin + count > num_points) throw std::invalid_argument("Dataset::slice out of range");
    Dataset out = empty(dims, elem_kind, metric);
    out.num_points = count;
    if (elem_kind == ElemKind::f32)
      out.f32.assign(f32.begin() + begin * dims, f32.begin() + (begin + count) * dims);
    else
      out.u8.assign(u8.begin() + begin * dims, u8.begin() + (begin + count) * dims);
    return out;
  }
  void append(const Dataset& o) {
    if (o.dims != dims || o.elem_kind != elem_kind || o.metric != metric)
      throw std::invalid_argument("Dataset::append: incompatible dataset");
    if (elem_kind == ElemKind::f32)
      f32.insert(f32.end(), o.f32.begin(), o.f32.end());
    else
      u8.insert(u8.end(), o.u8.begin(), o.u8.end());
    num_points += o.num_points;
  }
  // FNV-1a over (num_points, dims), (elem kind, metric) and the payload bytes
  std::uint64_t content_hash() const {
    std::uint64_t h = 0xcbf29ce484222325ULL;
    auto mix = [&h](const void* p, std::size_t n) {
      const unsigned char* c = static_cast<const unsigned char*>(p);
      for (std::size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 0x100000001b3ULL;
    };
    const std::uint64_t shape[2] = {num_points, dims};
    const std::uint8_t tag[2] = {static_cast<std::uint8_t>(elem_kind),
                                 static_cast<std::uint8_t>(metric)};
    mix(shape, sizeof shape);
    mix(tag, sizeof tag);
    if (elem_kind == ElemKind::f32)
      mix(f32.data(), f32.size() * sizeof(float));
    else
      mix(u8.data(), u8.size());
    return h;
  }
  std::size_t payload_bytes() const {
    return elem_kind == ElemKind::f32 ? f32.size() * sizeof(float) : u8.size();
  }
  void validate() const {
    if ((elem_kind == ElemKind::f32 ? f32.size() : u8.size()) != num_points * dims)
      throw std::logic_error("Dataset: data length != num_points * dims");
  }
  knng_dataset view() const {
    const void* data = elem_kind == ElemKind::u8 ? static_cast<const void*>(u8.data())
                                                 : static_cast<const void*>(f32.data());
    return knng_dataset{data, num_points, dims, static_cast<std::uint8_t>(elem_kind),
                        static_cast<std::uint8_t>(metric), KNNG_MEM_HOST, 0};
  }
};

inline float cross_distance(const Dataset& a, std::size_t i, const Dataset& b, std::size_t j) {
  if (a.elem_kind == ElemKind::f32)
    return a.metric == MetricKind::l2
               ? detail::l2_f32(a.f32.data() + i * a.dims, b.f32.data() + j * b.dims, a.dims)
               : detail::cosine_t(a.f32.data() + i * a.dims, b.f32.data() + j * b.dims, a.dims);
  return a.metric == MetricKind::l2
             ? detail::l2_u8(a.u8.data() + i * a.dims, b.u8.data() + j * b.dims, a.dims)
             : detail::cosine_t(a.u8.data() + i * a.dims, b.u8.data() + j * b.dims, a.dims);
}

struct NeighborEntry {
  PointId id = 0;
  float dist = 0.0f;
  bool flag = false;
  bool operator==(const NeighborEntry& o) const { return id == o.id && dist == o.dist; }
};

// core.hpp:136-139
inline bool closer(const NeighborEntry& a, const NeighborEntry& b) {
  if (a.dist != b.dist) return a.dist < b.dist;
  return a.id < b.id;
}

// KnnGraph core.hpp:156-179
struct KnnGraph {
  std::size_t num_sources = 0;
  std::size_t k = 0;
  IdSpace id_space = IdSpace::local;
  std::vector<PointId> ids;
  std::vector<float> dists;
  std::vector<std::uint8_t> flags;

  static KnnGraph allocate(std::size_t n, std::size_t k, IdSpace space) {
    KnnGraph g;
    g.num_sources = n;
    g.k = k;
    g.id_space = space;
    g.ids.assign(n * k, 0);
    g.dists.assign(n * k, 0.0f);
    g.flags.assign(n * k, 0);
    return g;
  }
  std::span<const PointId> ids_row(std::size_t r) const { return {ids.data() + r * k, k}; }
  std::span<const float> dists_row(std::size_t r) const { return {dists.data() + r * k, k}; }
  std::span<PointId> ids_row(std::size_t r) { return {ids.data() + r * k, k}; }
  std::span<float> dists_row(std::size_t r) { return {dists.data() + r * k, k}; }
  std::vector<NeighborEntry> row_entries(std::size_t r) const {
    std::vector<NeighborEntry> e(k);
    for (std::size_t j = 0; j < k; ++j)
      e[j] = {ids[r * k + j], dists[r * k + j], !flags.empty() && flags[r * k + j] != 0};
    return e;
  }
  void set_row(std::size_t r, std::span<const NeighborEntry> e) {
    if (e.size() != k) throw std::invalid_argument("KnnGraph::set_row: wrong row length");
    for (std::size_t j = 0; j < k; ++j) {
      ids[r * k + j] = e[j].id;
      dists[r * k + j] = e[j].dist;
      if (!flags.empty()) flags[r * k + j] = e[j].flag ? 1 : 0;
    }
  }
  knng_graph view() {
    return knng_graph{ids.data(), dists.data(), flags.empty() ? nullptr : flags.data(),
                      num_sources, k, KNNG_MEM_HOST, {0, 0, 0, 0, 0, 0, 0}};
  }
};

// check_graph_invariants core.cpp:166-186: shape, non-negative distances, no
// self loop in local id space, rows sorted by (dist, id), no duplicate id.
inline void check_graph_invariants(const KnnGraph& g) {
  if (g.ids.size() != g.num_sources * g.k || g.dists.size() != g.ids.size())
    throw std::logic_error("KnnGraph: matrix shape mismatch");
  for (std::size_t r = 0; r < g.num_sources; ++r) {
    const PointId* id = g.ids.data() + r * g.k;
    const float* ds = g.dists.data() + r * g.k;
    for (std::size_t j = 0; j < g.k; ++j) {
      if (ds[j] < 0.0f) throw std::logic_error("KnnGraph: negative distance");
      if (g.id_space == IdSpace::local && id[j] == r)
        throw std::logic_error("KnnGraph: self-loop");
      if (j && !(ds[j - 1] < ds[j] || (ds[j - 1] == ds[j] && id[j - 1] < id[j])))
        throw std::logic_error("KnnGraph: row not sorted");
      for (std::size_t m = j + 1; m < g.k; ++m)
        if (id[m] == id[j]) throw std::logic_error("KnnGraph: duplicate id");
    }
  }
}

// merge_rows core.cpp:114-134 (on the GPU)
inline std::vector<NeighborEntry> merge_rows(std::span<const NeighborEntry> a,
                                             std::span<const NeighborEntry> b, std::size_t k) {
  std::vector<PointId> ai(a.size()), bi(b.size()), oi(k);
  std::vector<float> ad(a.size()), bd(b.size()), od(k);
  for (std::size_t i = 0; i < a.size(); ++i) ai[i] = a[i].id, ad[i] = a[i].dist;
  for (std::size_t i = 0; i < b.size(); ++i) bi[i] = b[i].id, bd[i] = b[i].dist;
  std::uint32_t cnt = 0;
  detail::check(knng_merge_rows(detail::ctx(), 0, 1, ai.data(), ad.data(), a.size(), bi.data(),
                                bd.data(), b.size(), k, oi.data(), od.data(), &cnt));
  std::vector<NeighborEntry> out(cnt);
  for (std::uint32_t i = 0; i < cnt; ++i) out[i] = {oi[i], od[i], false};
  return out;
}

// NnDescentParams / NnDescentStats nndescent.hpp:12-20, 113-116
struct NnDescentParams {
  std::size_t k = 32;
  double delta = 0.0001;
  double rho = 0.5;
  std::size_t max_iters = 100;
  std::size_t candidate_capacity = 0;
  std::uint64_t seed = 0;
  std::size_t workers = 0;
};
struct NnDescentStats {
  std::vector<std::size_t> accepted_per_iter;
  std::size_t iterations = 0;
};

inline KnnGraph init_random_graph(const Dataset& d, std::size_t k, std::uint64_t seed,
                                  std::size_t /*workers*/ = 0) {
  KnnGraph g = KnnGraph::allocate(d.num_points, k, IdSpace::local);
  const knng_dataset ds = d.view();
  knng_graph gv = g.view();
  detail::check(knng_init_random_graph(detail::ctx(), 0, &ds, k, seed, &gv));
  return g;
}

// nn_descent nndescent.cpp:225-259
inline KnnGraph nn_descent(const Dataset& d, const NnDescentParams& p,
                           NnDescentStats* stats = nullptr) {
  KnnGraph g = KnnGraph::allocate(d.num_points, p.k, IdSpace::local);
  const knng_dataset ds = d.view();
  const knng_nnd_params cp{p.k, p.delta, p.rho, p.max_iters, p.candidate_capacity, p.seed,
                           p.workers};
  std::vector<std::uint64_t> acc(p.max_iters ? p.max_iters : 1);
  knng_nnd_stats st{};
  st.accepted_per_iter = acc.data();
  st.accepted_cap = acc.size();
  knng_graph gv = g.view();
  detail::check(knng_nn_descent(detail::ctx(), 0, &ds, &cp, &gv, stats ? &st : nullptr));
  if (stats) {
    stats->iterations = st.iterations;
    stats->accepted_per_iter.assign(acc.begin(), acc.begin() + st.iterations);
  }
  return g;
}

// SearchGraph graphopt.hpp:13-25
struct SearchGraph {
  std::size_t num_sources = 0;
  std::size_t out_degree = 0;
  IdSpace id_space = IdSpace::local;
  std::vector<PointId> ids;
  std::span<const PointId> row(std::size_t r) const {
    return {ids.data() + r * out_degree, out_degree};
  }
  std::span<PointId> row(std::size_t r) { return {ids.data() + r * out_degree, out_degree}; }
};

// optimize_graph graphopt.cpp:24-105 (bit-identical to the reference)
inline SearchGraph optimize_graph(const KnnGraph& g, const Dataset& d, std::size_t out_degree,
                                  std::size_t /*workers*/ = 0) {
  SearchGraph sg;
  sg.num_sources = g.num_sources;
  sg.out_degree = out_degree ? out_degree : g.k;
  sg.id_space = g.id_space;
  if (sg.out_degree > g.k) throw std::invalid_argument("optimize_graph: out_degree must be <= k");
  sg.ids.assign(sg.num_sources * sg.out_degree, 0);
  KnnGraph copy = g;
  knng_graph gv = copy.view();
  gv.flags = nullptr;
  const knng_dataset ds = d.view();
  detail::check(knng_optimize_graph(detail::ctx(), 0, &gv, &ds, out_degree, sg.ids.data()));
  return sg;
}

// SearchParams / SearchResult / SearchDiagnostics annsearch.hpp:12-41
struct SearchParams {
  std::size_t k_s = 10;
  std::size_t beam_width = 64;
  std::size_t num_entry_points = 16;
  std::size_t max_hops = 0;
  std::uint64_t seed = 0;
  std::size_t workers = 0;
};
struct SearchResult {
  std::size_t num_queries = 0;
  std::size_t k_s = 0;
  std::vector<PointId> ids;
  std::vector<float> dists;
  std::span<const PointId> ids_row(std::size_t q) const { return {ids.data() + q * k_s, k_s}; }
  std::span<const float> dists_row(std::size_t q) const {
    return {dists.data() + q * k_s, k_s};
  }
};
struct SearchDiagnostics {
  bool collect_scored_ids = false;  // scored ids in scoring order (second, exact pass)
  std::vector<std::vector<PointId>> scored_ids;
  std::vector<std::size_t> hops;
  std::vector<std::size_t> scored;
};

// ann_search annsearch.cpp:50-129 (bit-identical to the reference)
inline SearchResult ann_search(const Dataset& q, const SearchGraph& sg, const Dataset& v,
                               const SearchParams& p, SearchDiagnostics* diag = nullptr) {
  SearchResult r;
  r.num_queries = q.num_points;
  r.k_s = p.k_s;
  r.ids.assign(q.num_points * p.k_s, 0);
  r.dists.assign(q.num_points * p.k_s, 0.0f);
  std::vector<std::uint32_t> hops(diag ? q.num_points : 0), scored(diag ? q.num_points : 0);
  const knng_dataset qd = q.view(), vd = v.view();
  const knng_search_params sp{p.k_s, p.beam_width, p.num_entry_points, p.max_hops, p.seed,
                              p.workers};
  static const std::uint32_t kNoRow = 0;
  detail::check(knng_ann_search(detail::ctx(), 0, &qd, sg.ids.empty() ? &kNoRow : sg.ids.data(),
                                sg.num_sources, sg.out_degree, &vd, &sp, KNNG_MEM_HOST,
                                r.ids.data(), r.dists.data(), diag ? hops.data() : nullptr,
                                diag ? scored.data() : nullptr));
  if (diag) {
    diag->hops.assign(hops.begin(), hops.end());
    diag->scored.assign(scored.begin(), scored.end());
    diag->scored_ids.clear();
    if (diag->collect_scored_ids) {
      // the search is deterministic: rerun with the exact per-query capacity
      std::uint64_t cap = 1;
      for (auto c : scored) cap = std::max<std::uint64_t>(cap, c);
      std::vector<std::uint32_t> ids(q.num_points * cap), h2(q.num_points), s2(q.num_points);
      SearchResult r2 = r;
      detail::check(knng_ann_search_scored_ids(
          detail::ctx(), 0, &qd, sg.ids.empty() ? &kNoRow : sg.ids.data(), sg.num_sources,
          sg.out_degree, &vd, &sp, KNNG_MEM_HOST, r2.ids.data(), r2.dists.data(), h2.data(),
          s2.data(), ids.data(), cap));
      for (std::size_t i = 0; i < q.num_points; ++i)
        diag->scored_ids.emplace_back(ids.begin() + i * cap, ids.begin() + i * cap + s2[i]);
    }
  }
  return r;
}

// Partition refine.hpp:57-70
struct Partition {
  std::vector<PointId> to_external;
  std::vector<std::size_t> offsets;
  std::vector<Dataset> locals;
  std::size_t num_ranks() const { return locals.size(); }
  std::size_t total_points() const { return to_external.size(); }
  std::size_t size_of(std::size_t r) const { return offsets[r + 1] - offsets[r]; }
};

inline Partition partition_dataset(const Dataset& d, std::size_t ranks, std::uint64_t seed) {
  Partition p;
  p.to_external.assign(d.num_points, 0);
  std::vector<std::uint64_t> off(ranks + 1, 0);
  std::vector<float> perm(d.num_points * d.dims);
  const knng_dataset ds = d.view();
  detail::check(knng_partition(detail::ctx(), 0, &ds, ranks, seed, KNNG_MEM_HOST,
                               p.to_external.data(), off.data(), perm.data()));
  p.offsets.assign(off.begin(), off.end());
  for (std::size_t r = 0; r < ranks; ++r) {
    Dataset l = Dataset::empty(d.dims, d.elem_kind, d.metric);
    l.num_points = p.size_of(r);
    l.f32.assign(perm.begin() + p.offsets[r] * d.dims, perm.begin() + p.offsets[r + 1] * d.dims);
    p.locals.push_back(std::move(l));
  }
  return p;
}

inline std::size_t tree_levels(std::size_t ranks, std::size_t groups) {
  std::uint64_t out = 0;
  detail::check(knng_tree_levels(ranks, groups, &out));
  return out;
}

struct TreeLevel {
  std::size_t group_lo = 0;
  std::size_t group_hi = 0;
  std::vector<std::size_t> partners;
};

inline TreeLevel tree_schedule(std::size_t ranks, std::size_t groups, std::size_t rank,
                               std::size_t level) {
  std::uint64_t lo = 0, hi = 0;
  std::vector<std::uint64_t> partners(ranks ? ranks : 1);
  detail::check(knng_tree_schedule(ranks, groups, rank, level, &lo, &hi, partners.data()));
  TreeLevel t;
  t.group_lo = lo;
  t.group_hi = hi;
  t.partners.assign(partners.begin(), partners.begin() + (std::size_t{1} << level));
  return t;
}

// RefineConfig / DistBuildResult refine.hpp:37-52, 91-107
struct RefineConfig {
  std::size_t ranks = 1;
  std::size_t groups = 2;
  std::size_t k = 32;
  std::size_t k_s = 0;
  std::size_t out_degree = 0;
  NnDescentParams nn;
  SearchParams search;
  bool skip_tree_phase = false;
  bool double_buffer = false;
  std::size_t max_concat_bytes = 0;
  std::uint64_t seed = 0;
  bool capture_snapshots = false;
};

struct GetRecord {
  std::size_t src = 0;
  std::size_t target = 0;
  std::string region;
  std::size_t bytes = 0;
  std::uint64_t epoch = 0;
};

struct PhaseSnapshot {
  std::string label;
  KnnGraph graph;
};

struct DistBuildResult {
  KnnGraph graph;
  struct Phases {
    double local_s = 0.0, tree_s = 0.0, merge_s = 0.0, flat_s = 0.0, etc_s = 0.0;
  } phases;
  std::size_t levels = 0;
  std::uint64_t merge_epoch = 0;
  std::uint64_t flat_epoch = 0;
  std::vector<GetRecord> comm_log;
  std::vector<PhaseSnapshot> snapshots;
};

namespace detail {
inline knng_refine_config to_c(const RefineConfig& cfg) {
  knng_refine_config c{};
  c.ranks = cfg.ranks;
  c.groups = cfg.groups;
  c.k = cfg.k;
  c.k_s = cfg.k_s;
  c.out_degree = cfg.out_degree;
  c.nn = knng_nnd_params{cfg.k, cfg.nn.delta, cfg.nn.rho, cfg.nn.max_iters,
                         cfg.nn.candidate_capacity, cfg.nn.seed, cfg.nn.workers};
  c.search = knng_search_params{cfg.search.k_s, cfg.search.beam_width, cfg.search.num_entry_points,
                                cfg.search.max_hops, cfg.search.seed, cfg.search.workers};
  c.skip_tree_phase = cfg.skip_tree_phase;
  c.double_buffer = cfg.double_buffer;
  c.capture_snapshots = cfg.capture_snapshots;
  c.max_concat_bytes = cfg.max_concat_bytes;
  c.seed = cfg.seed;
  return c;
}
inline std::vector<GetRecord> last_comm_log(std::uint64_t gets) {
  std::vector<knng_get_record> recs(gets ? gets : 1);
  std::uint64_t cnt = 0;
  check(knng_last_comm_log(ctx(), recs.data(), recs.size(), &cnt));
  std::vector<GetRecord> out;
  for (std::uint64_t i = 0; i < cnt && i < recs.size(); ++i)
    out.push_back({recs[i].src, recs[i].target, recs[i].region, recs[i].bytes, recs[i].epoch});
  return out;
}
}  // namespace detail

// build_distributed refine.cpp:504-586 (ranks on the context's GPUs)
inline DistBuildResult build_distributed(const Dataset& d, const RefineConfig& cfg) {
  DistBuildResult res;
  res.graph = KnnGraph::allocate(d.num_points, cfg.k, IdSpace::global);
  res.graph.flags.clear();
  knng_refine_config c = detail::to_c(cfg);
  const knng_dataset ds = d.view();
  knng_graph gv = res.graph.view();
  knng_dist_result r{};
  const std::size_t cells = d.num_points * cfg.k;
  const std::size_t cap = cfg.capture_snapshots ? 10 : 0;
  std::vector<std::uint32_t> si(cap * cells);
  std::vector<float> sd(cap * cells);
  detail::check(knng_build_distributed(detail::ctx(), &ds, &c, &gv, &r, cap ? si.data() : nullptr,
                                       cap ? sd.data() : nullptr, cap));
  res.phases = {r.local_s, r.tree_s, r.merge_s, r.flat_s, r.etc_s};
  res.levels = r.levels;
  res.merge_epoch = r.merge_epoch;
  res.flat_epoch = r.flat_epoch;
  std::vector<knng_get_record> recs(r.comm_gets ? r.comm_gets : 1);
  std::uint64_t cnt = 0;
  detail::check(knng_last_comm_log(detail::ctx(), recs.data(), recs.size(), &cnt));
  for (std::uint64_t i = 0; i < cnt; ++i)
    res.comm_log.push_back({recs[i].src, recs[i].target, recs[i].region, recs[i].bytes,
                            recs[i].epoch});
  for (std::uint64_t s = 0; s < r.num_snapshots && s < cap; ++s) {
    PhaseSnapshot ps;
    ps.label = s == 0 ? "local"
               : (s <= r.levels ? "tree_level_" + std::to_string(s - 1) : std::string("flat"));
    ps.graph = KnnGraph::allocate(d.num_points, cfg.k, IdSpace::global);
    ps.graph.ids.assign(si.begin() + s * cells, si.begin() + (s + 1) * cells);
    ps.graph.dists.assign(sd.begin() + s * cells, sd.begin() + (s + 1) * cells);
    res.snapshots.push_back(std::move(ps));
  }
  return res;
}

// search_throughput_probe annsearch.cpp:131-155 (annsearch.hpp:52-69)
struct ThroughputCase {
  std::size_t source_count = 0;
  const SearchGraph* sgraph = nullptr;
  const Dataset* vectors = nullptr;
};
struct ThroughputRow {
  std::size_t source_count = 0;
  std::size_t num_queries = 0;
  double seconds = 0.0;
  double qps = 0.0;
};
inline std::vector<ThroughputRow> search_throughput_probe(const std::vector<ThroughputCase>& cases,
                                                          const Dataset& queries,
                                                          const SearchParams& params) {
  std::vector<knng_dataset> vds(cases.size());
  std::vector<knng_throughput_case> cc(cases.size());
  for (std::size_t i = 0; i < cases.size(); ++i) {
    vds[i] = cases[i].vectors->view();
    cc[i] = knng_throughput_case{cases[i].source_count, cases[i].sgraph->ids.data(),
                                 cases[i].sgraph->num_sources, cases[i].sgraph->out_degree, &vds[i],
                                 KNNG_MEM_HOST};
  }
  const knng_dataset q = queries.view();
  const knng_search_params p{params.k_s, params.beam_width, params.num_entry_points,
                             params.max_hops, params.seed, params.workers};
  std::vector<knng_throughput_row> rows(cases.size());
  detail::check(knng_search_throughput_probe(detail::ctx(), 0, cc.data(), cc.size(), &q, &p,
                                             rows.data()));
  std::vector<ThroughputRow> out;
  for (const auto& r : rows) out.push_back({r.source_count, r.num_queries, r.seconds, r.qps});
  return out;
}

// One rank of build_distributed in this process (one process per GPU; B200
// extension, no reference counterpart).  `allgather(in, bytes, out)` must
// gather `bytes` from every rank into `out` in rank order (MPI_Allgather,
// torch.distributed, ...).  Returns this rank's rows (external ids) and, in
// `rows`, the external id of each row.
struct RankBuildResult {
  KnnGraph graph;  // rows x k
  std::vector<std::uint32_t> rows;
  DistBuildResult::Phases phases;
  std::vector<GetRecord> comm_log;  // every rank's gets
};

namespace detail {
template <class F>
int allgather_thunk(void* user, const void* in, std::uint64_t bytes, void* out) {
  try {
    (*static_cast<F*>(user))(in, static_cast<std::size_t>(bytes), out);
    return 0;
  } catch (...) {
    return 1;
  }
}
}  // namespace detail

template <class AllGather>
inline RankBuildResult build_distributed_rank(const Dataset& d, const RefineConfig& cfg,
                                              std::size_t rank, std::size_t world, int device,
                                              AllGather allgather) {
  knng_refine_config c{};
  c.ranks = world;
  c.groups = cfg.groups;
  c.k = cfg.k;
  c.k_s = cfg.k_s;
  c.out_degree = cfg.out_degree;
  c.nn = knng_nnd_params{cfg.k, cfg.nn.delta, cfg.nn.rho, cfg.nn.max_iters,
                         cfg.nn.candidate_capacity, cfg.nn.seed, cfg.nn.workers};
  c.search = knng_search_params{cfg.search.k_s, cfg.search.beam_width, cfg.search.num_entry_points,
                                cfg.search.max_hops, cfg.search.seed, cfg.search.workers};
  c.skip_tree_phase = cfg.skip_tree_phase;
  c.double_buffer = cfg.double_buffer;
  c.max_concat_bytes = cfg.max_concat_bytes;
  c.seed = cfg.seed;
  const std::size_t cap = (d.num_points + world - 1) / world;
  std::vector<std::uint32_t> ids(cap * cfg.k), rows(cap);
  std::vector<float> dists(cap * cfg.k);
  const knng_dataset ds = d.view();
  knng_dist_result r{};
  std::uint64_t n_rows = 0;
  detail::check(knng_build_distributed_rank(detail::ctx(), device, rank, world,
                                            &detail::allgather_thunk<AllGather>, &allgather, &ds,
                                            &c, ids.data(), dists.data(), rows.data(),
                                            KNNG_MEM_HOST, &n_rows, &r));
  RankBuildResult res;
  res.graph = KnnGraph::allocate(n_rows, cfg.k, IdSpace::global);
  res.graph.flags.clear();
  res.graph.ids.assign(ids.begin(), ids.begin() + n_rows * cfg.k);
  res.graph.dists.assign(dists.begin(), dists.begin() + n_rows * cfg.k);
  res.rows.assign(rows.begin(), rows.begin() + n_rows);
  res.phases = {r.local_s, r.tree_s, r.merge_s, r.flat_s, r.etc_s};
  std::vector<knng_get_record> recs(r.comm_gets ? r.comm_gets : 1);
  std::uint64_t cnt = 0;
  detail::check(knng_last_comm_log(detail::ctx(), recs.data(), recs.size(), &cnt));
  for (std::uint64_t i = 0; i < cnt; ++i)
    res.comm_log.push_back({recs[i].src, recs[i].target, recs[i].region, recs[i].bytes,
                            recs[i].epoch});
  return res;
}

// read_vecs / write_vecs / read_ivecs / write_ivecs evalio.hpp:17-31
inline Dataset read_vecs(const std::filesystem::path& path, ElemKind kind,
                         MetricKind metric = MetricKind::l2) {
  const int code = kind == ElemKind::f32 ? KNNG_ELEM_F32 : KNNG_ELEM_U8;
  std::uint64_t rows = 0, dims = 0;
  detail::check(knng_vecs_shape(path.string().c_str(), code, &rows, &dims));
  Dataset d = Dataset::empty(dims, kind, metric);
  d.num_points = rows;
  void* out;
  if (kind == ElemKind::f32) {
    d.f32.resize(rows * dims);
    out = d.f32.data();
  } else {
    d.u8.resize(rows * dims);
    out = d.u8.data();
  }
  detail::check(knng_read_vecs(nullptr, 0, path.string().c_str(), code, out, rows, dims,
                               KNNG_MEM_HOST));
  return d;
}
inline void write_vecs(const Dataset& d, const std::filesystem::path& path) {
  const bool f = d.elem_kind == ElemKind::f32;
  detail::check(knng_write_vecs(path.string().c_str(), f ? KNNG_ELEM_F32 : KNNG_ELEM_U8,
                                f ? static_cast<const void*>(d.f32.data())
                                  : static_cast<const void*>(d.u8.data()),
                                d.num_points, d.dims));
}
struct IdMatrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<std::int32_t> v;
};
inline IdMatrix read_ivecs(const std::filesystem::path& path) {
  std::uint64_t rows = 0, cols = 0;
  detail::check(knng_vecs_shape(path.string().c_str(), KNNG_ELEM_I32, &rows, &cols));
  IdMatrix m;
  m.rows = rows;
  m.cols = cols;
  m.v.resize(rows * cols);
  detail::check(knng_read_vecs(nullptr, 0, path.string().c_str(), KNNG_ELEM_I32, m.v.data(), rows,
                               cols, KNNG_MEM_HOST));
  return m;
}
inline void write_ivecs(const IdMatrix& m, const std::filesystem::path& path) {
  detail::check(knng_write_vecs(path.string().c_str(), KNNG_ELEM_I32, m.v.data(), m.rows, m.cols));
}

// evalio.hpp (measurement support)
enum class Distribution { uniform, gaussian, clustered };

inline Dataset gen_random_dataset(std::size_t n, std::size_t dims, Distribution dist,
                                  std::uint64_t seed, std::size_t clusters = 0,
                                  MetricKind metric = MetricKind::l2) {
  Dataset d = Dataset::empty(dims, ElemKind::f32, metric);
  d.num_points = n;
  d.f32.resize(n * dims);
  detail::check(knng_gen_random_dataset(n, dims, static_cast<int>(dist), seed, clusters,
                                        d.f32.data()));
  return d;
}

struct GroundTruth {
  KnnGraph graph;
  std::uint64_t dataset_hash = 0;
  std::size_t k = 0;
  MetricKind metric = MetricKind::l2;
};

inline GroundTruth brute_force_knng(const Dataset& d, std::size_t k, std::size_t /*workers*/ = 0) {
  GroundTruth gt;
  gt.k = k;
  gt.metric = d.metric;
  gt.dataset_hash = d.content_hash();
  gt.graph = KnnGraph::allocate(d.num_points, k, IdSpace::local);
  std::vector<std::uint64_t> rows(d.num_points);
  for (std::size_t i = 0; i < rows.size(); ++i) rows[i] = i;
  const knng_dataset ds = d.view();
  detail::check(knng_brute_force(detail::ctx(), 0, &ds, rows.data(), rows.size(), k, KNNG_MEM_HOST,
                                 gt.graph.ids.data(), gt.graph.dists.data()));
  return gt;
}

inline double recall_at_k(const KnnGraph& test, const KnnGraph& truth, std::size_t k_eval) {
  if (k_eval == 0 || k_eval > test.k || k_eval > truth.k)
    throw std::invalid_argument("recall_at_k: k_eval out of range");
  if (test.num_sources != truth.num_sources)
    throw std::invalid_argument("recall_at_k: graphs not comparable");
  std::size_t hits = 0;
  for (std::size_t r = 0; r < test.num_sources; ++r)
    for (std::size_t i = 0; i < k_eval; ++i)
      for (std::size_t j = 0; j < k_eval; ++j)
        if (test.ids[r * test.k + i] == truth.ids[r * truth.k + j]) {
          ++hits;
          break;
        }
  return static_cast<double>(hits) / static_cast<double>(test.num_sources * k_eval);
}
inline double recall_at_k(const KnnGraph& test, const GroundTruth& gt, std::size_t k_eval) {
  return recall_at_k(test, gt.graph, k_eval);
}

// distance_threshold_recall evalio.cpp:199-215 (host, measurement only): per
// row, the share of the first k_eval test distances <= the reference row's
// k_eval-th distance, averaged in row order.
inline double distance_threshold_recall(const KnnGraph& test, const KnnGraph& reference,
                                        std::size_t k_eval) {
  if (k_eval == 0 || k_eval > test.k || k_eval > reference.k)
    throw std::invalid_argument("distance_threshold_recall: k_eval out of range");
  if (test.num_sources != reference.num_sources)
    throw std::invalid_argument("distance_threshold_recall: graphs not comparable");
  double total = 0.0;
  for (std::size_t r = 0; r < test.num_sources; ++r) {
    const float thr = reference.dists[r * reference.k + k_eval - 1];
    std::size_t c = 0;
    while (c < test.k && test.dists[r * test.k + c] <= thr) ++c;
    total += static_cast<double>(std::min(c, k_eval)) / static_cast<double>(k_eval);
  }
  return total / static_cast<double>(test.num_sources);
}

inline void save_graph(const KnnGraph& g, const std::filesystem::path& path) {
  KnnGraph copy = g;
  knng_graph gv = copy.view();
  detail::check(knng_save_graph(&gv, path.string().c_str()));
}

inline KnnGraph load_graph(const std::filesystem::path& path, IdSpace space = IdSpace::global) {
  std::uint64_t n = 0, k = 0;
  detail::check(knng_load_graph_header(path.string().c_str(), &n, &k));
  KnnGraph g = KnnGraph::allocate(n, k, space);
  knng_graph gv = g.view();
  detail::check(knng_load_graph(path.string().c_str(), &gv));
  return g;
}

}  // namespace knng

#include "knng_b200_host.hpp"
