// knng_b200_host.hpp -- the host-side remainder of the reference's public API
// for the C++ drop-in (included by knng_b200.hpp; not meant to be included on
// its own):
//
//   rng.hpp       Rng (SplitMix64), mix_seed, sample_distinct, shuffle
//   wire.hpp      serialized regions (22-byte header + payload), region_size
//   distsim.hpp   RankWorld / RankHandle / run_ranks / spawn_world: the
//                 reference's simulated-rank transport for host regions
//   refine.hpp    the world-level phase drivers (build_local_graphs,
//                 binary_tree_refine, grouped_merge, flat_refine,
//                 all_to_all_refine) -- on the GPUs through knng_refine_phase;
//                 the RankWorld passed in carries the epoch counter and the
//                 comm log across calls exactly as the reference's does --
//                 plus the closed-form cost model (predicted_runtime)
//   evalio.hpp    brute_force_knng_cached, synth_shifted_copies
//
// Every function cites the reference declaration it replaces.
#pragma once

#include <chrono>
#include <condition_variable>
#include <cstddef>
#include <cstring>
#include <exception>
#include <fstream>
#include <limits>
#include <map>
#include <mutex>
#include <sstream>
#include <string_view>
#include <thread>
#include <type_traits>
#include <utility>

namespace knng {

// ---------------------------------------------------------------------------
// rng.hpp:12-96
// ---------------------------------------------------------------------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : s_(seed) {}
  std::uint64_t next_u64() {
    std::uint64_t z = (s_ += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  std::uint64_t next_below(std::uint64_t bound) {  // mulhi(x, bound)
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next_u64()) * bound) >> 64);
  }
  float next_float() { return static_cast<float>(next_u64() >> 40) * 0x1.0p-24f; }
  float next_gaussian() {  // Box-Muller, second value cached
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    float u1 = next_float();
    while (u1 <= 0.0f) u1 = next_float();
    const float u2 = next_float();
    const float rad = std::sqrt(-2.0f * std::log(u1));
    const float ang = 6.28318530717958647692f * u2;
    spare_ = rad * std::sin(ang);
    spare_ok_ = true;
    return rad * std::cos(ang);
  }

 private:
  std::uint64_t s_;
  float spare_ = 0.0f;
  bool spare_ok_ = false;
};

inline std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b) {
  return Rng(a ^ (b * 0x9e3779b97f4a7c15ULL + 0xd1b54a32d192ed03ULL)).next_u64();
}

inline std::vector<std::uint32_t> sample_distinct(std::uint64_t n, std::size_t m, Rng& rng) {
  std::vector<std::uint32_t> out;
  if (m >= n) {
    for (std::uint64_t i = 0; i < n; ++i) out.push_back(static_cast<std::uint32_t>(i));
    return out;
  }
  while (out.size() < m) {
    const auto v = static_cast<std::uint32_t>(rng.next_below(n));
    if (std::find(out.begin(), out.end(), v) == out.end()) out.push_back(v);
  }
  return out;
}

template <class T>
void shuffle(std::vector<T>& v, Rng& rng) {
  for (std::size_t i = v.size(); i > 1; --i)
    std::swap(v[i - 1], v[static_cast<std::size_t>(rng.next_below(i))]);
}

// ---------------------------------------------------------------------------
// wire.hpp: magic u32 | kind u8 | rows u64 | cols u64 | elem u8 | payload,
// little-endian (the host is little-endian)
// ---------------------------------------------------------------------------
namespace wire {
inline constexpr std::uint32_t kMagic = 0x474E4E4BU;
inline constexpr std::size_t kHeaderBytes = 4 + 1 + 8 + 8 + 1;
enum class RegionKind : std::uint8_t { dataset = 0, knng = 1, sgraph = 2, result = 3 };
inline constexpr std::uint8_t kElemF32 = 0;
inline constexpr std::uint8_t kElemU8 = 1;
inline constexpr std::uint8_t kElemU32 = 2;

struct Region {
  std::vector<std::byte> bytes;
  std::size_t size() const { return bytes.size(); }
};
struct Header {
  RegionKind kind = RegionKind::dataset;
  std::uint64_t rows = 0;
  std::uint64_t cols = 0;
  std::uint8_t elem_kind = kElemF32;
};

namespace detail {
inline std::size_t payload(RegionKind kind, std::uint64_t rows, std::uint64_t cols,
                           std::uint8_t elem) {
  const std::uint64_t cells = rows * cols;
  switch (kind) {
    case RegionKind::dataset: return cells * (elem == kElemU8 ? 1 : 4);
    case RegionKind::knng:
    case RegionKind::result: return cells * 8;
    case RegionKind::sgraph: return cells * 4;
  }
  throw std::runtime_error("wire: unknown region kind");
}
inline Region begin(RegionKind kind, std::uint64_t rows, std::uint64_t cols, std::uint8_t elem) {
  Region r;
  r.bytes.resize(kHeaderBytes + payload(kind, rows, cols, elem));
  std::byte* p = r.bytes.data();
  const std::uint8_t k8 = static_cast<std::uint8_t>(kind);
  std::memcpy(p, &kMagic, 4);
  std::memcpy(p + 4, &k8, 1);
  std::memcpy(p + 5, &rows, 8);
  std::memcpy(p + 13, &cols, 8);
  std::memcpy(p + 21, &elem, 1);
  return r;
}
}  // namespace detail

inline std::size_t region_size(RegionKind kind, std::uint64_t rows, std::uint64_t cols,
                               std::uint8_t elem_kind) {
  return kHeaderBytes + detail::payload(kind, rows, cols, elem_kind);
}

inline Region serialize(const Dataset& d) {
  const bool f = d.elem_kind == ElemKind::f32;
  Region r = detail::begin(RegionKind::dataset, d.num_points, d.dims, f ? kElemF32 : kElemU8);
  if (f)
    std::memcpy(r.bytes.data() + kHeaderBytes, d.f32.data(), d.f32.size() * 4);
  else
    std::memcpy(r.bytes.data() + kHeaderBytes, d.u8.data(), d.u8.size());
  return r;
}
inline Region serialize(const KnnGraph& g) {
  Region r = detail::begin(RegionKind::knng, g.num_sources, g.k, kElemF32);
  std::memcpy(r.bytes.data() + kHeaderBytes, g.ids.data(), g.ids.size() * 4);
  std::memcpy(r.bytes.data() + kHeaderBytes + g.ids.size() * 4, g.dists.data(),
              g.dists.size() * 4);
  return r;
}
inline Region serialize(const SearchGraph& g) {
  Region r = detail::begin(RegionKind::sgraph, g.num_sources, g.out_degree, kElemU32);
  std::memcpy(r.bytes.data() + kHeaderBytes, g.ids.data(), g.ids.size() * 4);
  return r;
}
inline Region serialize(const SearchResult& s) {
  Region r = detail::begin(RegionKind::result, s.num_queries, s.k_s, kElemF32);
  std::memcpy(r.bytes.data() + kHeaderBytes, s.ids.data(), s.ids.size() * 4);
  std::memcpy(r.bytes.data() + kHeaderBytes + s.ids.size() * 4, s.dists.data(),
              s.dists.size() * 4);
  return r;
}

inline Header peek_header(const Region& r) {
  if (r.bytes.size() < kHeaderBytes)
    throw std::runtime_error("wire: region truncated before header end");
  const std::byte* p = r.bytes.data();
  std::uint32_t magic = 0;
  std::uint8_t kind = 0;
  Header h;
  std::memcpy(&magic, p, 4);
  if (magic != kMagic) throw std::runtime_error("wire: bad magic");
  std::memcpy(&kind, p + 4, 1);
  if (kind > 3) throw std::runtime_error("wire: bad region kind");
  h.kind = static_cast<RegionKind>(kind);
  std::memcpy(&h.rows, p + 5, 8);
  std::memcpy(&h.cols, p + 13, 8);
  std::memcpy(&h.elem_kind, p + 21, 1);
  if (h.elem_kind > kElemU32) throw std::runtime_error("wire: bad elem kind");
  if (r.bytes.size() != region_size(h.kind, h.rows, h.cols, h.elem_kind))
    throw std::runtime_error("wire: payload size mismatch");
  return h;
}

inline Dataset deserialize_dataset(const Region& r, MetricKind metric) {
  const Header h = peek_header(r);
  if (h.kind != RegionKind::dataset) throw std::runtime_error("wire: expected dataset region");
  const bool u = h.elem_kind == kElemU8;
  Dataset d = Dataset::empty(h.cols, u ? ElemKind::u8 : ElemKind::f32, metric);
  d.num_points = h.rows;
  const std::byte* p = r.bytes.data() + kHeaderBytes;
  if (u) {
    d.u8.resize(h.rows * h.cols);
    std::memcpy(d.u8.data(), p, d.u8.size());
  } else {
    d.f32.resize(h.rows * h.cols);
    std::memcpy(d.f32.data(), p, d.f32.size() * 4);
  }
  return d;
}
inline KnnGraph deserialize_knng(const Region& r, IdSpace space) {
  const Header h = peek_header(r);
  if (h.kind != RegionKind::knng) throw std::runtime_error("wire: expected knng region");
  KnnGraph g = KnnGraph::allocate(h.rows, h.cols, space);
  const std::byte* p = r.bytes.data() + kHeaderBytes;
  std::memcpy(g.ids.data(), p, g.ids.size() * 4);
  std::memcpy(g.dists.data(), p + g.ids.size() * 4, g.dists.size() * 4);
  return g;
}
inline SearchGraph deserialize_sgraph(const Region& r, IdSpace space) {
  const Header h = peek_header(r);
  if (h.kind != RegionKind::sgraph) throw std::runtime_error("wire: expected sgraph region");
  SearchGraph g;
  g.num_sources = h.rows;
  g.out_degree = h.cols;
  g.id_space = space;
  g.ids.resize(h.rows * h.cols);
  std::memcpy(g.ids.data(), r.bytes.data() + kHeaderBytes, g.ids.size() * 4);
  return g;
}
inline SearchResult deserialize_result(const Region& r) {
  const Header h = peek_header(r);
  if (h.kind != RegionKind::result) throw std::runtime_error("wire: expected result region");
  SearchResult s;
  s.num_queries = h.rows;
  s.k_s = h.cols;
  s.ids.resize(h.rows * h.cols);
  s.dists.resize(h.rows * h.cols);
  const std::byte* p = r.bytes.data() + kHeaderBytes;
  std::memcpy(s.ids.data(), p, s.ids.size() * 4);
  std::memcpy(s.dists.data(), p + s.ids.size() * 4, s.dists.size() * 4);
  return s;
}
inline void save_region(const Region& r, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  out.write(reinterpret_cast<const char*>(r.bytes.data()), static_cast<std::streamsize>(r.size()));
  if (!out) throw std::runtime_error("wire: cannot write " + path.string());
}
inline Region load_region(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw std::runtime_error("wire: cannot open " + path.string());
  Region r;
  r.bytes.resize(static_cast<std::size_t>(in.tellg()));
  in.seekg(0);
  in.read(reinterpret_cast<char*>(r.bytes.data()), static_cast<std::streamsize>(r.size()));
  peek_header(r);
  return r;
}
}  // namespace wire

// ---------------------------------------------------------------------------
// distsim.hpp:36-198 -- P simulated ranks over an immutable-snapshot region
// store.  A first publish is visible at once, a republish is staged until the
// next barrier, one publish per name per epoch; gets copy the snapshot and are
// logged; the barrier (60 s watchdog) advances the epoch; abort wakes waiters.
// The GPU phase drivers below run their ranks on the context's devices and
// report their gets and epochs into this same world.
// ---------------------------------------------------------------------------
class RankWorld {
 public:
  explicit RankWorld(std::size_t num_ranks,
                     std::chrono::milliseconds watchdog = std::chrono::seconds(60))
      : n_(num_ranks), watchdog_(watchdog) {
    if (num_ranks == 0) throw std::invalid_argument("RankWorld: P must be >= 1");
  }
  std::size_t num_ranks() const { return n_; }
  std::uint64_t epoch() const {
    std::lock_guard<std::mutex> l(mu_);
    return epoch_;
  }

  void publish(std::size_t rank, std::string_view name, wire::Region payload) {
    check_rank(rank);
    std::lock_guard<std::mutex> l(mu_);
    throw_if_aborted();
    Slot& s = store_[{rank, std::string(name)}];
    if (s.published && s.epoch == epoch_)
      throw WorldError("publish: region '" + std::string(name) + "' already published by rank " +
                       std::to_string(rank) + " in epoch " + std::to_string(epoch_));
    if (s.has_current) {
      s.staged = std::move(payload);
      s.has_staged = true;
    } else {
      s.current = std::move(payload);
      s.has_current = true;
    }
    s.published = true;
    s.epoch = epoch_;
  }

  wire::Region one_sided_get(std::size_t src, std::size_t target, std::string_view name) {
    check_rank(src);
    check_rank(target);
    std::lock_guard<std::mutex> l(mu_);
    throw_if_aborted();
    auto it = store_.find({target, std::string(name)});
    if (it == store_.end() || !it->second.has_current)
      throw WorldError("one_sided_get: region '" + std::string(name) +
                       "' not published by rank " + std::to_string(target));
    wire::Region copy = it->second.current;
    log_.push_back({src, target, std::string(name), copy.size(), epoch_});
    return copy;
  }

  void barrier(std::size_t rank) {
    check_rank(rank);
    std::unique_lock<std::mutex> l(mu_);
    throw_if_aborted();
    const std::uint64_t gen = generation_;
    if (++arrived_ == n_) {
      for (auto& kv : store_) {
        Slot& s = kv.second;
        if (!s.has_staged) continue;
        s.current = std::move(s.staged);
        s.staged = wire::Region{};
        s.has_staged = false;
      }
      ++epoch_;
      arrived_ = 0;
      ++generation_;
      cv_.notify_all();
      return;
    }
    const bool woke = cv_.wait_for(l, watchdog_, [&] { return generation_ != gen || aborted_; });
    throw_if_aborted();
    if (!woke) {
      aborted_ = true;
      reason_ = "barrier watchdog timeout at rank " + std::to_string(rank);
      cv_.notify_all();
      throw WorldError(reason_);
    }
  }

  void abort(const std::string& reason) {
    std::lock_guard<std::mutex> l(mu_);
    if (!aborted_) {
      aborted_ = true;
      reason_ = reason;
    }
    cv_.notify_all();
  }

  std::vector<GetRecord> comm_log() const {
    std::lock_guard<std::mutex> l(mu_);
    return log_;
  }

  // B200 drivers: the world epoch a GPU phase starts from, and the phase's
  // gets + final epoch folded back in (same records the reference would log).
  std::uint64_t begin_device_phase() {
    std::lock_guard<std::mutex> l(mu_);
    throw_if_aborted();
    return epoch_;
  }
  void end_device_phase(std::vector<GetRecord> gets, std::uint64_t epoch) {
    std::lock_guard<std::mutex> l(mu_);
    for (auto& g : gets) log_.push_back(std::move(g));
    epoch_ = epoch;
  }

 private:
  struct Slot {
    wire::Region current, staged;
    bool has_current = false, has_staged = false, published = false;
    std::uint64_t epoch = 0;
  };
  void check_rank(std::size_t r) const {
    if (r >= n_) throw std::invalid_argument("RankWorld: rank out of range");
  }
  void throw_if_aborted() const {
    if (aborted_) throw WorldAborted("world aborted: " + reason_);
  }
  const std::size_t n_;
  const std::chrono::milliseconds watchdog_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::pair<std::size_t, std::string>, Slot> store_;
  std::vector<GetRecord> log_;
  std::uint64_t epoch_ = 0, generation_ = 0;
  std::size_t arrived_ = 0;
  bool aborted_ = false;
  std::string reason_;
};

class RankHandle {
 public:
  RankHandle(RankWorld& world, std::size_t rank) : w_(&world), rank_(rank) {}
  std::size_t rank() const { return rank_; }
  std::size_t world_size() const { return w_->num_ranks(); }
  RankWorld& world() { return *w_; }
  void publish(std::string_view name, wire::Region payload) {
    w_->publish(rank_, name, std::move(payload));
  }
  wire::Region get(std::size_t target, std::string_view name) {
    return w_->one_sided_get(rank_, target, name);
  }
  void barrier() { w_->barrier(rank_); }

 private:
  RankWorld* w_;
  std::size_t rank_;
};

namespace detail {
// run body on one thread per rank; a failing rank aborts the world; the first
// failure that is not a secondary WorldAborted is rethrown (distsim.hpp:113-153)
template <class Body>
auto run_rank_threads(RankWorld& world, Body& body) {
  using R = std::invoke_result_t<Body&, RankHandle&>;
  const std::size_t p = world.num_ranks();
  std::vector<std::exception_ptr> err(p);
  std::conditional_t<std::is_void_v<R>, std::vector<int>, std::vector<R>> out(p);
  std::vector<std::thread> th;
  for (std::size_t i = 0; i < p; ++i)
    th.emplace_back([&, i] {
      RankHandle h(world, i);
      try {
        if constexpr (std::is_void_v<R>)
          body(h);
        else
          out[i] = body(h);
      } catch (...) {
        err[i] = std::current_exception();
        world.abort("rank " + std::to_string(i) + " failed");
      }
    });
  for (auto& t : th) t.join();
  std::exception_ptr first;
  for (auto& e : err) {
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
  if constexpr (!std::is_void_v<R>) return out;
}
}  // namespace detail

template <class Body>
auto run_ranks(RankWorld& world, Body&& body) {
  return detail::run_rank_threads(world, body);
}
template <class Body>
auto spawn_world(std::size_t num_ranks, Body&& body) {
  RankWorld world(num_ranks);
  return detail::run_rank_threads(world, body);
}

// ---------------------------------------------------------------------------
// refine.hpp:13-35 -- the closed-form cost model
// ---------------------------------------------------------------------------
struct CostModel {
  double query_seconds = 0.0;
  double alpha = 0.0;
  double beta = 0.0;
};
struct RuntimeBreakdown {
  double tree = 0.0, merge = 0.0, flat = 0.0, total = 0.0;
};
// tree = S(N/P)log2(P/M) + (P/M - 1)h, merge = (P/M)h, flat = (M-1)[S(N/P) +
// (P/M)h], h = alpha + (N/P) beta  (refine.cpp:68-84)
inline RuntimeBreakdown predicted_runtime(const CostModel& cm, double n_points, std::size_t ranks,
                                          std::size_t groups) {
  auto pow2 = [](std::size_t v) { return v && !(v & (v - 1)); };
  if (!pow2(ranks) || !pow2(groups) || groups > ranks)
    throw std::invalid_argument("predicted_runtime: P and M must be powers of two with M <= P");
  const double p = static_cast<double>(ranks), m = static_cast<double>(groups);
  const double per = n_points / p, hop = cm.alpha + per * cm.beta;
  RuntimeBreakdown b;
  b.tree = cm.query_seconds * per * std::log2(p / m) + (p / m - 1.0) * hop;
  b.merge = (p / m) * hop;
  b.flat = (m - 1.0) * (cm.query_seconds * per + (p / m) * hop);
  b.total = b.tree + b.merge + b.flat;
  return b;
}

// ---------------------------------------------------------------------------
// refine.hpp:114-136 -- the world-level phase drivers on the GPUs
// ---------------------------------------------------------------------------
namespace detail {
// validate_config refine.cpp:359-378
inline void validate_refine(const Partition& part, const RefineConfig& cfg) {
  const std::size_t p = part.num_ranks();
  auto pow2 = [](std::size_t v) { return v && !(v & (v - 1)); };
  if (!pow2(p)) throw std::invalid_argument("refine: P must be a power of two");
  if (p > 1 && (!pow2(cfg.groups) || cfg.groups < 2 || cfg.groups > p))
    throw std::invalid_argument("refine: M must be a power of two with 2 <= M <= P");
  std::size_t min_block = part.size_of(0);
  for (std::size_t r = 1; r < p; ++r) min_block = std::min(min_block, part.size_of(r));
  if (cfg.k >= min_block) throw std::invalid_argument("refine: k must be < points per rank");
  if ((cfg.k_s ? cfg.k_s : cfg.k) > min_block)
    throw std::invalid_argument("refine: k_s must be <= points per rank");
  if ((cfg.out_degree ? cfg.out_degree : cfg.k) > cfg.k)
    throw std::invalid_argument("refine: out_degree must be <= k");
}

// The partition's rows in rank order (internal order) and its offsets.
struct FlatPartition {
  std::vector<float> x;
  std::vector<std::uint64_t> off;
  std::size_t dims = 0;
};
inline FlatPartition flatten(const Partition& part) {
  FlatPartition f;
  f.dims = part.locals.front().dims;
  for (const Dataset& l : part.locals) {
    if (l.elem_kind != ElemKind::f32 || l.metric != MetricKind::l2)
      throw std::invalid_argument("refine: the phase drivers take f32 / l2 partitions");
    f.x.insert(f.x.end(), l.f32.begin(), l.f32.end());
  }
  f.off.assign(part.offsets.begin(), part.offsets.end());
  return f;
}

// Graph rows of every rank, concatenated (internal global ids).
inline void concat_graphs(const std::vector<KnnGraph>& gs, std::size_t k,
                          std::vector<PointId>& ids, std::vector<float>& dists) {
  for (const KnnGraph& g : gs) {
    if (g.k != k) throw std::invalid_argument("refine: graph k != cfg.k");
    ids.insert(ids.end(), g.ids.begin(), g.ids.end());
    dists.insert(dists.end(), g.dists.begin(), g.dists.end());
  }
}
inline std::vector<KnnGraph> split_graphs(const Partition& part, std::size_t k,
                                          const std::vector<PointId>& ids,
                                          const std::vector<float>& dists) {
  std::vector<KnnGraph> out;
  for (std::size_t r = 0; r < part.num_ranks(); ++r) {
    KnnGraph g = KnnGraph::allocate(part.size_of(r), k, IdSpace::global);
    g.flags.clear();
    std::copy_n(ids.begin() + part.offsets[r] * k, g.ids.size(), g.ids.begin());
    std::copy_n(dists.begin() + part.offsets[r] * k, g.dists.size(), g.dists.begin());
    out.push_back(std::move(g));
  }
  return out;
}
inline std::size_t group_points(const Partition& part, std::size_t groups, std::size_t r) {
  const std::size_t gsz = part.num_ranks() / groups;
  const std::size_t lo = (r / gsz) * gsz;
  return part.offsets[lo + gsz] - part.offsets[lo];
}

// One driver call: phase 1 a2a, 2 tree, 3 merge (sg_out), 4 flat (sg_in).
inline void device_phase(RankWorld& world, const Partition& part, const RefineConfig& cfg,
                         int phase, std::vector<PointId>& ids, std::vector<float>& dists,
                         const std::vector<PointId>* sg_in, std::vector<PointId>* sg_out) {
  validate_refine(part, cfg);
  if (world.num_ranks() != part.num_ranks())
    throw std::invalid_argument("refine: world size != partition ranks");
  const FlatPartition f = flatten(part);
  RefineConfig c = cfg;
  c.ranks = part.num_ranks();
  const knng_refine_config cc = to_c(c);
  std::uint64_t epoch = world.begin_device_phase();
  knng_dist_result r{};
  const knng_status st =
      knng_refine_phase(ctx(), f.x.data(), part.total_points(), f.dims, &cc, f.off.data(), phase,
                        &epoch, ids.data(), dists.data(), sg_in ? sg_in->data() : nullptr,
                        sg_out ? sg_out->data() : nullptr, &r);
  if (st != KNNG_OK) world.abort(knng_last_error());
  check(st);
  world.end_device_phase(last_comm_log(r.comm_gets), epoch);
}
}  // namespace detail

// build_local_graphs refine.cpp:420-428 (local_build_rank :380-390): one
// nn_descent per rank, seed mix_seed(nn.seed, rank) when P > 1, ids shifted
// to internal global ids.
inline std::vector<KnnGraph> build_local_graphs(const Partition& part, const RefineConfig& cfg) {
  detail::validate_refine(part, cfg);
  std::vector<KnnGraph> out;
  for (std::size_t r = 0; r < part.num_ranks(); ++r) {
    NnDescentParams np = cfg.nn;
    np.k = cfg.k;
    np.workers = 1;
    np.seed = part.num_ranks() == 1 ? cfg.nn.seed : mix_seed(cfg.nn.seed, r);
    KnnGraph g = nn_descent(part.locals[r], np);
    for (auto& id : g.ids) id += static_cast<PointId>(part.offsets[r]);
    g.id_space = IdSpace::global;
    out.push_back(std::move(g));
  }
  return out;
}

// binary_tree_refine refine.cpp:430-443
inline std::vector<KnnGraph> binary_tree_refine(RankWorld& world, const Partition& part,
                                                std::vector<KnnGraph> graphs,
                                                const RefineConfig& cfg) {
  std::vector<PointId> ids;
  std::vector<float> dists;
  detail::concat_graphs(graphs, cfg.k, ids, dists);
  detail::device_phase(world, part, cfg, 2, ids, dists, nullptr, nullptr);
  return detail::split_graphs(part, cfg.k, ids, dists);
}

// grouped_merge refine.cpp:445-456: every member holds its group's search
// graph (local ids of the group span)
inline std::vector<SearchGraph> grouped_merge(RankWorld& world, const Partition& part,
                                              const std::vector<KnnGraph>& graphs,
                                              const RefineConfig& cfg) {
  std::vector<PointId> ids;
  std::vector<float> dists;
  detail::concat_graphs(graphs, cfg.k, ids, dists);
  const std::size_t od = cfg.out_degree ? cfg.out_degree : cfg.k;
  // the tree phase's effective group count (skip_tree / max_concat_bytes) is
  // decided by the library; size the blocks for the finest grouping (M = P)
  // and read the real group sizes back from the driver's output layout
  RefineConfig c = cfg;
  c.ranks = part.num_ranks();
  std::size_t groups = c.ranks == 1 ? 1 : cfg.groups;
  {
    std::uint64_t g_eff = 0;
    const detail::FlatPartition f = detail::flatten(part);
    const knng_refine_config cc = detail::to_c(c);
    detail::check(knng_effective_groups(&cc, f.off.data(), f.dims, &g_eff));
    groups = g_eff;
  }
  std::vector<std::size_t> block(part.num_ranks() + 1, 0);
  for (std::size_t r = 0; r < part.num_ranks(); ++r)
    block[r + 1] = block[r] + detail::group_points(part, groups, r) * od;
  std::vector<PointId> sg(block.back());
  detail::device_phase(world, part, cfg, 3, ids, dists, nullptr, &sg);
  std::vector<SearchGraph> out;
  for (std::size_t r = 0; r < part.num_ranks(); ++r) {
    SearchGraph g;
    g.num_sources = detail::group_points(part, groups, r);
    g.out_degree = od;
    g.id_space = IdSpace::local;
    g.ids.assign(sg.begin() + block[r], sg.begin() + block[r + 1]);
    out.push_back(std::move(g));
  }
  return out;
}

// flat_refine refine.cpp:458-471 (each rank publishes group_graphs[rank])
inline std::vector<KnnGraph> flat_refine(RankWorld& world, const Partition& part,
                                         std::vector<KnnGraph> graphs,
                                         const std::vector<SearchGraph>& group_graphs,
                                         const RefineConfig& cfg) {
  if (group_graphs.size() != part.num_ranks())
    throw std::invalid_argument("flat_refine: one group graph per rank expected");
  std::vector<PointId> ids;
  std::vector<float> dists;
  detail::concat_graphs(graphs, cfg.k, ids, dists);
  std::vector<PointId> sg;
  for (const SearchGraph& g : group_graphs) sg.insert(sg.end(), g.ids.begin(), g.ids.end());
  detail::device_phase(world, part, cfg, 4, ids, dists, &sg, nullptr);
  return detail::split_graphs(part, cfg.k, ids, dists);
}

// all_to_all_refine refine.cpp:473-502
inline std::vector<KnnGraph> all_to_all_refine(RankWorld& world, const Partition& part,
                                               std::vector<KnnGraph> graphs,
                                               const RefineConfig& cfg) {
  std::vector<PointId> ids;
  std::vector<float> dists;
  detail::concat_graphs(graphs, cfg.k, ids, dists);
  detail::device_phase(world, part, cfg, 1, ids, dists, nullptr, nullptr);
  return detail::split_graphs(part, cfg.k, ids, dists);
}

// ---------------------------------------------------------------------------
// evalio.hpp
// ---------------------------------------------------------------------------
// brute_force_knng_cached evalio.cpp:149-168: keyed by (content hash, k, metric)
inline GroundTruth brute_force_knng_cached(const Dataset& d, std::size_t k,
                                           const std::filesystem::path& cache_dir,
                                           std::size_t workers = 0) {
  std::filesystem::create_directories(cache_dir);
  std::ostringstream name;
  name << "gt_" << std::hex << d.content_hash() << std::dec << "_k" << k << "_"
       << to_string(d.metric) << ".knng";
  const std::filesystem::path path = cache_dir / name.str();
  if (std::filesystem::exists(path)) {
    GroundTruth gt;
    gt.graph = load_graph(path, IdSpace::local);
    gt.dataset_hash = d.content_hash();
    gt.k = k;
    gt.metric = d.metric;
    if (gt.graph.num_sources == d.num_points && gt.graph.k == k) return gt;
  }
  GroundTruth gt = brute_force_knng(d, k, workers);
  save_graph(gt.graph, path);
  return gt;
}

// synth_shifted_copies evalio.cpp:217-240: copy c shifts axis (c-1) mod dims by
// (max - min + epsilon) over the output built so far
inline Dataset synth_shifted_copies(const Dataset& d, std::size_t copies, float epsilon) {
  if (epsilon <= 0.0f) throw std::invalid_argument("synth_shifted_copies: epsilon must be > 0");
  if (copies < 1) throw std::invalid_argument("synth_shifted_copies: copies >= 1");
  if (d.dims == 0 || d.elem_kind != ElemKind::f32)
    throw std::invalid_argument("synth_shifted_copies: needs float data with >= 1 dim");
  Dataset out = d;
  for (std::size_t c = 1; c < copies; ++c) {
    const std::size_t axis = (c - 1) % d.dims;
    float lo = std::numeric_limits<float>::infinity(), hi = -lo;
    for (std::size_t i = 0; i < out.num_points; ++i) {
      lo = std::min(lo, out.f32[i * d.dims + axis]);
      hi = std::max(hi, out.f32[i * d.dims + axis]);
    }
    const float shift = hi - lo + epsilon;
    Dataset cp = d;
    for (std::size_t i = 0; i < cp.num_points; ++i) cp.f32[i * d.dims + axis] += shift;
    out.append(cp);
  }
  return out;
}

inline void save_sgraph(const SearchGraph& g, const std::filesystem::path& path) {
  wire::save_region(wire::serialize(g), path);
}
inline SearchGraph load_sgraph(const std::filesystem::path& path,
                               IdSpace space = IdSpace::global) {
  return wire::deserialize_sgraph(wire::load_region(path), space);
}

}  // namespace knng
