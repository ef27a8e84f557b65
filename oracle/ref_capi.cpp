// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shims over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libknng_ref.so).  Used to (1) mint the golden fixtures under
// tests/golden/ that pin the C restatement (knng_oracle.c) and the CUDA path,
// and (2) time the reference CPU path as bench.py's cpu_baseline /
// `--impl reference` arm.  Nothing in the product links this.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "knng/annsearch.hpp"
#include "knng/core.hpp"
#include "knng/distsim.hpp"
#include "knng/evalio.hpp"
#include "knng/graphopt.hpp"
#include "knng/nndescent.hpp"
#include "knng/refine.hpp"
#include "knng/rng.hpp"

using namespace knng;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 world error, 3 other exception
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const WorldError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// Metric of every dataset the shims build (kr_set_metric; default l2).
MetricKind g_metric = MetricKind::l2;

Dataset make_ds(const float* data, std::size_t n, std::size_t dims) {
  Dataset d = Dataset::empty(dims, ElemKind::f32, g_metric);
  d.num_points = n;
  d.f32.assign(data, data + n * dims);
  return d;
}

void put_graph(const KnnGraph& g, std::uint32_t* ids, float* dists, std::uint8_t* flags) {
  std::copy(g.ids.begin(), g.ids.end(), ids);
  std::copy(g.dists.begin(), g.dists.end(), dists);
  if (flags) {
    if (g.flags.empty())
      std::fill(flags, flags + g.ids.size(), 0);
    else
      std::copy(g.flags.begin(), g.flags.end(), flags);
  }
}

KnnGraph get_graph(const std::uint32_t* ids, const float* dists, std::size_t n,
                   std::size_t k, IdSpace space) {
  KnnGraph g = KnnGraph::allocate(n, k, space);
  std::copy(ids, ids + n * k, g.ids.begin());
  std::copy(dists, dists + n * k, g.dists.begin());
  return g;
}

struct CRefineCfg {
  std::uint64_t ranks, groups, k, k_s, out_degree;
  double delta, rho;
  std::uint64_t max_iters, cap, nn_seed;
  std::uint64_t beam_width, num_entry_points, max_hops, search_seed;
  std::uint64_t skip_tree, double_buffer, max_concat_bytes, seed;
};

RefineConfig to_cfg(const CRefineCfg* c) {
  RefineConfig cfg;
  cfg.ranks = c->ranks;
  cfg.groups = c->groups;
  cfg.k = c->k;
  cfg.k_s = c->k_s;
  cfg.out_degree = c->out_degree;
  cfg.nn.k = c->k;
  cfg.nn.delta = c->delta;
  cfg.nn.rho = c->rho;
  cfg.nn.max_iters = c->max_iters;
  cfg.nn.candidate_capacity = c->cap;
  cfg.nn.seed = c->nn_seed;
  cfg.search.beam_width = c->beam_width;
  cfg.search.num_entry_points = c->num_entry_points;
  cfg.search.max_hops = c->max_hops;
  cfg.search.seed = c->search_seed;
  cfg.skip_tree_phase = c->skip_tree != 0;
  cfg.double_buffer = c->double_buffer != 0;
  cfg.max_concat_bytes = c->max_concat_bytes;
  cfg.seed = c->seed;
  return cfg;
}

}  // namespace

extern "C" {

const char* kr_last_error() { return g_err.c_str(); }

unsigned kr_hardware_concurrency() { return std::thread::hardware_concurrency(); }

int kr_gen_random_dataset(std::uint64_t n, std::uint64_t dims, int dist,
                          std::uint64_t seed, std::uint64_t clusters, float* out) {
  return guard([&] {
    const Distribution dd = dist == 0   ? Distribution::uniform
                            : dist == 1 ? Distribution::gaussian
                                        : Distribution::clustered;
    const Dataset d = gen_random_dataset(n, dims, dd, seed, clusters);
    std::copy(d.f32.begin(), d.f32.end(), out);
  });
}

void kr_set_metric(int metric) { g_metric = metric ? MetricKind::cosine : MetricKind::l2; }

float kr_cosine(const float* a, const float* b, std::uint64_t d) {
  return distance(MetricKind::cosine, std::span<const float>(a, d), std::span<const float>(b, d));
}

float kr_l2(const float* a, const float* b, std::uint64_t d) {
  return distance(MetricKind::l2, std::span<const float>(a, d), std::span<const float>(b, d));
}

int kr_init_random_graph(const float* data, std::uint64_t n, std::uint64_t dims,
                         std::uint64_t k, std::uint64_t seed, std::uint32_t* ids,
                         float* dists, std::uint8_t* flags) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    put_graph(init_random_graph(d, k, seed, 1), ids, dists, flags);
  });
}

int kr_sample_neighbors(std::uint32_t* ids, float* dists, std::uint8_t* flags,
                        std::uint64_t n, std::uint64_t k, double rho, std::uint64_t seed,
                        std::uint64_t iter, std::uint32_t* new_fwd, std::uint32_t* new_fwd_n,
                        std::uint32_t* old_fwd, std::uint32_t* old_fwd_n,
                        std::uint32_t* new_rev, std::uint32_t* new_rev_n,
                        std::uint32_t* old_rev, std::uint32_t* old_rev_n) {
  return guard([&] {
    KnnGraph g = get_graph(ids, dists, n, k, IdSpace::local);
    std::copy(flags, flags + n * k, g.flags.begin());
    const NeighborSamples s = sample_neighbors(g, rho, seed, iter, 1);
    const std::size_t b = s.bound;
    for (std::size_t p = 0; p < n; ++p) {
      new_fwd_n[p] = static_cast<std::uint32_t>(s.new_fwd[p].size());
      std::copy(s.new_fwd[p].begin(), s.new_fwd[p].end(), new_fwd + p * b);
      old_fwd_n[p] = static_cast<std::uint32_t>(s.old_fwd[p].size());
      std::copy(s.old_fwd[p].begin(), s.old_fwd[p].end(), old_fwd + p * k);
      new_rev_n[p] = static_cast<std::uint32_t>(s.new_rev[p].size());
      std::copy(s.new_rev[p].begin(), s.new_rev[p].end(), new_rev + p * b);
      old_rev_n[p] = static_cast<std::uint32_t>(s.old_rev[p].size());
      std::copy(s.old_rev[p].begin(), s.old_rev[p].end(), old_rev + p * b);
    }
    std::copy(g.flags.begin(), g.flags.end(), flags);
  });
}

int kr_nn_descent(const float* data, std::uint64_t n, std::uint64_t dims, std::uint64_t k,
                  double delta, double rho, std::uint64_t max_iters, std::uint64_t cap,
                  std::uint64_t seed, std::uint64_t workers, std::uint32_t* ids,
                  float* dists, std::uint8_t* flags, std::uint64_t* accepted,
                  std::uint64_t* iterations, double* seconds) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    NnDescentParams p;
    p.k = k;
    p.delta = delta;
    p.rho = rho;
    p.max_iters = max_iters;
    p.candidate_capacity = cap;
    p.seed = seed;
    p.workers = workers;
    NnDescentStats st;
    const auto t0 = std::chrono::steady_clock::now();
    const KnnGraph g = nn_descent(d, p, &st);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    put_graph(g, ids, dists, flags);
    if (accepted)
      std::copy(st.accepted_per_iter.begin(), st.accepted_per_iter.end(), accepted);
    if (iterations) *iterations = st.iterations;
  });
}

int kr_optimize_graph(const std::uint32_t* ids, const float* dists, std::uint64_t n,
                      std::uint64_t k, const float* data, std::uint64_t dims,
                      std::uint64_t out_degree, std::uint32_t* sg_ids, std::uint64_t workers) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    const KnnGraph g = get_graph(ids, dists, n, k, IdSpace::local);
    const SearchGraph sg = optimize_graph(g, d, out_degree, workers);
    std::copy(sg.ids.begin(), sg.ids.end(), sg_ids);
  });
}

int kr_ann_search(const float* q, std::uint64_t nq, const std::uint32_t* sg_ids,
                  std::uint64_t sg_n, std::uint64_t deg, const float* v, std::uint64_t dims,
                  std::uint64_t k_s, std::uint64_t beam, std::uint64_t entries,
                  std::uint64_t max_hops, std::uint64_t seed, std::uint64_t workers,
                  std::uint32_t* out_ids, float* out_d, std::uint32_t* hops,
                  std::uint32_t* scored) {
  return guard([&] {
    const Dataset qd = make_ds(q, nq, dims);
    const Dataset vd = make_ds(v, sg_n, dims);
    SearchGraph sg;
    sg.num_sources = sg_n;
    sg.out_degree = deg;
    sg.ids.assign(sg_ids, sg_ids + sg_n * deg);
    SearchParams sp;
    sp.k_s = k_s;
    sp.beam_width = beam;
    sp.num_entry_points = entries;
    sp.max_hops = max_hops;
    sp.seed = seed;
    sp.workers = workers;
    SearchDiagnostics diag;
    diag.collect_scored_ids = scored != nullptr;
    const SearchResult r = ann_search(qd, sg, vd, sp, &diag);
    std::copy(r.ids.begin(), r.ids.end(), out_ids);
    std::copy(r.dists.begin(), r.dists.end(), out_d);
    for (std::size_t i = 0; i < nq; ++i) {
      if (hops) hops[i] = static_cast<std::uint32_t>(diag.hops[i]);
      if (scored) scored[i] = static_cast<std::uint32_t>(diag.scored_ids[i].size());
    }
  });
}

int kr_partition(const float* data, std::uint64_t n, std::uint64_t dims,
                 std::uint64_t ranks, std::uint64_t seed, std::uint32_t* to_external,
                 std::uint64_t* offsets, float* locals_concat) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    const Partition p = partition_dataset(d, ranks, seed);
    std::copy(p.to_external.begin(), p.to_external.end(), to_external);
    for (std::size_t r = 0; r <= ranks; ++r) offsets[r] = p.offsets[r];
    if (locals_concat) {
      std::size_t at = 0;
      for (const auto& l : p.locals) {
        std::copy(l.f32.begin(), l.f32.end(), locals_concat + at);
        at += l.f32.size();
      }
    }
  });
}

std::uint64_t kr_merge_rows(const std::uint32_t* a_ids, const float* a_d, std::uint64_t na,
                            const std::uint32_t* b_ids, const float* b_d, std::uint64_t nb,
                            std::uint64_t k, std::uint32_t* o_ids, float* o_d) {
  std::vector<NeighborEntry> a(na), b(nb);
  for (std::size_t i = 0; i < na; ++i) a[i] = {a_ids[i], a_d[i], false};
  for (std::size_t i = 0; i < nb; ++i) b[i] = {b_ids[i], b_d[i], false};
  const auto m = merge_rows(a, b, k);
  for (std::size_t i = 0; i < m.size(); ++i) {
    o_ids[i] = m[i].id;
    o_d[i] = m[i].dist;
  }
  return m.size();
}

int kr_brute_force(const float* data, std::uint64_t n, std::uint64_t dims, std::uint64_t k,
                   std::uint64_t workers, std::uint32_t* ids, float* dists) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    const GroundTruth gt = brute_force_knng(d, k, workers);
    put_graph(gt.graph, ids, dists, nullptr);
  });
}

int kr_build_distributed(const float* data, std::uint64_t n, std::uint64_t dims,
                         const CRefineCfg* c, std::uint32_t* ids, float* dists,
                         double* phases, std::uint64_t* comm_gets,
                         std::uint64_t* comm_bytes) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    const DistBuildResult r = build_distributed(d, to_cfg(c));
    put_graph(r.graph, ids, dists, nullptr);
    if (phases) {
      phases[0] = r.phases.local_s;
      phases[1] = r.phases.tree_s;
      phases[2] = r.phases.merge_s;
      phases[3] = r.phases.flat_s;
      phases[4] = r.phases.etc_s;
    }
    std::uint64_t gets = 0, bytes = 0;
    for (const auto& rec : r.comm_log) {
      ++gets;
      bytes += rec.bytes;
    }
    if (comm_gets) *comm_gets = gets;
    if (comm_bytes) *comm_bytes = bytes;
  });
}

// Local graphs (internal global ids, rank blocks concatenated) as built by
// build_local_graphs refine.cpp:420-428.
int kr_build_local_graphs(const float* data, std::uint64_t n, std::uint64_t dims,
                          const CRefineCfg* c, std::uint32_t* ids, float* dists) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    const RefineConfig cfg = to_cfg(c);
    const Partition part = partition_dataset(d, cfg.ranks, cfg.seed);
    const auto gs = build_local_graphs(part, cfg);
    std::size_t at = 0;
    for (const auto& g : gs) {
      std::copy(g.ids.begin(), g.ids.end(), ids + at);
      std::copy(g.dists.begin(), g.dists.end(), dists + at);
      at += g.ids.size();
    }
  });
}

// Refine the given local graphs with the standalone world drivers
// (binary_tree_refine -> grouped_merge -> flat_refine, refine.hpp:119-130) or
// all_to_all_refine (mode 1).  Graph rows updated in place (internal ids).
int kr_refine_from_local(const float* data, std::uint64_t n, std::uint64_t dims,
                         const CRefineCfg* c, std::uint32_t* ids, float* dists, int mode,
                         std::uint32_t* sg_out) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    const RefineConfig cfg = to_cfg(c);
    const Partition part = partition_dataset(d, cfg.ranks, cfg.seed);
    std::vector<KnnGraph> gs;
    for (std::size_t r = 0; r < cfg.ranks; ++r) {
      const std::size_t lo = part.offsets[r], cnt = part.size_of(r);
      gs.push_back(get_graph(ids + lo * cfg.k, dists + lo * cfg.k, cnt, cfg.k, IdSpace::global));
    }
    std::vector<KnnGraph> out;
    if (mode == 1) {
      RankWorld w(cfg.ranks);
      out = all_to_all_refine(w, part, gs, cfg);
    } else {
      RankWorld w1(cfg.ranks);
      auto g1 = binary_tree_refine(w1, part, gs, cfg);
      RankWorld w2(cfg.ranks);
      auto sgs = grouped_merge(w2, part, g1, cfg);
      if (sg_out) {
        // Group search graphs, one per group, in group order (every member
        // holds a byte-identical copy, test_refine.cpp:244-259).
        const std::size_t gsz = cfg.ranks / refine_detail::effective_groups(part, cfg);
        std::size_t at = 0;
        for (std::size_t r = 0; r < cfg.ranks; r += gsz) {
          std::copy(sgs[r].ids.begin(), sgs[r].ids.end(), sg_out + at);
          at += sgs[r].ids.size();
        }
      }
      RankWorld w3(cfg.ranks);
      out = flat_refine(w3, part, g1, sgs, cfg);
    }
    for (std::size_t r = 0; r < cfg.ranks; ++r) {
      const std::size_t lo = part.offsets[r];
      std::copy(out[r].ids.begin(), out[r].ids.end(), ids + lo * cfg.k);
      std::copy(out[r].dists.begin(), out[r].dists.end(), dists + lo * cfg.k);
    }
  });
}


// build_distributed (refine.cpp:504-586) at sizes where the reference's own
// driver cannot finish on this host: the P local builds run as P concurrent
// threads exactly as local_build_rank (refine.cpp:380-390: workers=1, seed
// mix_seed(nn.seed, rank) when P>1, ids shifted by offsets[rank]) -- the
// reference's build_local_graphs runs them one after another -- and the
// refine phases run through the public world drivers (refine.hpp:119-130)
// with a barrier watchdog of `watchdog_s` seconds instead of 60 s (ranks'
// multi-minute single-threaded phases finish more than a minute apart).
// Output: the N x k graph in external ids, rows sorted by (dist, ext id) as
// translate_to_external (refine.cpp:395-416).  phases = local, tree, merge, flat s.
int kr_build_distributed_staged(const float* data, std::uint64_t n, std::uint64_t dims,
                                const CRefineCfg* c, std::uint32_t* ids, float* dists,
                                double* phases, double watchdog_s) {
  return guard([&] {
    const Dataset d = make_ds(data, n, dims);
    const RefineConfig cfg = to_cfg(c);
    const Partition part = partition_dataset(d, cfg.ranks, cfg.seed);
    const std::size_t P = cfg.ranks;
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double>(b - a).count();
    };
    auto t0 = clk::now();
    std::vector<KnnGraph> gs(P);
    std::vector<std::exception_ptr> errs(P);
    {
      std::vector<std::thread> th;
      for (std::size_t r = 0; r < P; ++r)
        th.emplace_back([&, r] {
          try {
            NnDescentParams np = cfg.nn;
            np.k = cfg.k;
            np.workers = 1;
            np.seed = P == 1 ? cfg.nn.seed : mix_seed(cfg.nn.seed, r);
            KnnGraph g = nn_descent(part.locals[r], np);
            for (auto& id : g.ids) id += static_cast<std::uint32_t>(part.offsets[r]);
            g.id_space = IdSpace::global;
            gs[r] = std::move(g);
          } catch (...) {
            errs[r] = std::current_exception();
          }
        });
      for (auto& t : th) t.join();
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    }
    auto t1 = clk::now();
    const auto wd = std::chrono::milliseconds(static_cast<long long>(watchdog_s * 1000));
    RankWorld w1(P, wd);
    auto g1 = binary_tree_refine(w1, part, gs, cfg);
    auto t2 = clk::now();
    RankWorld w2(P, wd);
    auto sgs = grouped_merge(w2, part, g1, cfg);
    auto t3 = clk::now();
    RankWorld w3(P, wd);
    auto out = flat_refine(w3, part, g1, sgs, cfg);
    auto t4 = clk::now();
    const std::size_t k = cfg.k;
    for (std::size_t r = 0; r < P; ++r) {
      const KnnGraph& g = out[r];
      for (std::size_t row = 0; row < g.num_sources; ++row) {
        auto e = g.row_entries(row);
        for (auto& x : e) x.id = part.to_external[x.id];
        std::sort(e.begin(), e.end(),
                  [](const NeighborEntry& a, const NeighborEntry& b) { return closer(a, b); });
        const std::size_t ext = part.to_external[part.offsets[r] + row];
        for (std::size_t j = 0; j < k; ++j) {
          ids[ext * k + j] = e[j].id;
          dists[ext * k + j] = e[j].dist;
        }
      }
    }
    if (phases) {
      phases[0] = secs(t0, t1);
      phases[1] = secs(t1, t2);
      phases[2] = secs(t2, t3);
      phases[3] = secs(t3, t4);
    }
  });
}

}  // extern "C"
