// capi.cu -- the extern "C" drop-in boundary (include/knng_c.h).  Exceptions
// never cross it: each entry point maps the reference's exception classes to
// a status code and keeps e.what() for knng_last_error().
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/knng_c.h"
#include "graphopt.hpp"
#include "nndescent.hpp"
#include "pipeline.hpp"
#include "refine_kernels.hpp"
#include "search.hpp"

namespace knng_b200 {
void gen_random_dataset(uint64_t n, uint64_t dims, int dist, uint64_t seed, uint64_t clusters,
                        float* out);
void save_graph(const uint32_t* ids, const float* dists, uint64_t n, uint64_t k,
                const std::string& path);
void load_graph_header(const std::string& path, uint64_t* n, uint64_t* k);
void load_graph(const std::string& path, uint32_t* ids, float* dists, uint64_t n, uint64_t k);
void vecs_shape(const std::string& path, uint64_t esz, uint64_t* rows, uint64_t* dims);
void read_vecs(const std::string& path, uint64_t esz, void* out, uint64_t rows, uint64_t dims,
               const Runner* dev_runner);
void write_vecs(const std::string& path, const void* data, uint64_t rows, uint64_t dims,
                uint64_t esz);
}  // namespace knng_b200

using namespace knng_b200;

struct knng_ctx {
  std::vector<int> devices;
  std::vector<std::unique_ptr<Runner>> runners;  // one default runner per device
  // per-device NN-descent workspaces (declared after the runners: destroyed
  // first, while their streams exist)
  std::vector<std::unique_ptr<NndWorkspace>> nnd_ws;
  std::vector<GetRecord> last_log;
  Runner& runner(int dev) {
    for (size_t i = 0; i < devices.size(); ++i)
      if (devices[i] == dev) return *runners[i];
    throw std::invalid_argument("knng: device " + std::to_string(dev) + " not in this context");
  }
  NndWorkspace* workspace(int dev) {
    for (size_t i = 0; i < devices.size(); ++i)
      if (devices[i] == dev) {
        if (nnd_ws.size() < devices.size()) nnd_ws.resize(devices.size());
        if (!nnd_ws[i]) nnd_ws[i] = std::make_unique<NndWorkspace>();
        return nnd_ws[i].get();
      }
    throw std::invalid_argument("knng: device " + std::to_string(dev) + " not in this context");
  }
};

namespace {

thread_local std::string g_err;

// KNNG_TRACE=1: host timestamps of the phases of a C-ABI call on stderr.
struct HostTrace {
  const char* name;
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  explicit HostTrace(const char* n) : name(n), on(std::getenv("KNNG_TRACE") != nullptr) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[knng %s] %s %.3f ms (total %.3f)\n", name, what,
                 std::chrono::duration<double, std::milli>(t - last).count(),
                 std::chrono::duration<double, std::milli>(t - t0).count());
    last = t;
  }
  ~HostTrace() { mark("exit"); }
};

template <class F>
knng_status guard(F&& f) {
  try {
    f();
    return KNNG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return KNNG_EINVAL;
  } catch (const WorldAborted& e) {
    g_err = e.what();
    return KNNG_EABORTED;
  } catch (const WorldError& e) {
    g_err = e.what();
    return KNNG_EWORLD;
  } catch (const FormatError& e) {
    g_err = e.what();
    return KNNG_EFORMAT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return KNNG_ELOGIC;
  } catch (const CudaError& e) {
    g_err = e.what();
    return KNNG_ECUDA;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return KNNG_ENOMEM;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    const std::string w = e.what();
    return w.rfind("wire:", 0) == 0 ? KNNG_EFORMAT : KNNG_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KNNG_ERUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return KNNG_ERUNTIME;
  }
}

void check_ds(const knng_dataset* ds) {
  require(ds != nullptr && (ds->data != nullptr || ds->n == 0), "knng: null dataset");
  require(ds->elem_kind == KNNG_ELEM_F32 || ds->elem_kind == KNNG_ELEM_U8,
          "knng: unknown element kind");
  require(ds->metric == KNNG_METRIC_L2 || ds->metric == KNNG_METRIC_COS, "knng: unknown metric");
  require(ds->dims >= 1 && ds->dims <= (1u << 20), "knng: dims out of range");
}

// l2_u8 (core.hpp:32-39) promotes every byte to float before the sequential
// sum, and (float)a - (float)b and its square are exact: expanding u8 rows to
// f32 once gives bit-identical distances through the f32 kernels.
__global__ void k_u8_to_f32(const uint8_t* __restrict__ in, u64 count, float* __restrict__ out) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (u64)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}

// A dataset resident on the runner's device as f32 rows (copied in if host
// memory, expanded if u8).
struct DevData {
  DBuf<float> own;
  const float* p = nullptr;
  DBuf<float> nrm_own;  // cosine: per-row norm chains (core.hpp:44-49); else empty
  const float* nrm = nullptr;
};

void stage_rows(Runner& r, const knng_dataset* ds, DevData& out, int slot);
// Stage the rows, then (cosine) their norm chains: every kernel then runs only
// the per-pair dot chain and finishes with cos_finish (common.cuh).
void stage(Runner& r, const knng_dataset* ds, DevData& out, int slot = 0) {
  stage_rows(r, ds, out, slot);
  if (ds->metric == KNNG_METRIC_COS) {
    DeviceGuard g(r.device);
    out.nrm_own.alloc(r, ds->n ? ds->n : 1);
    row_norms_device(r, out.p, ds->n, (int)ds->dims, out.nrm_own.p);
    out.nrm = out.nrm_own.p;
  }
}
// slot: which runner scratch receives a host f32 dataset (a call staging two
// datasets uses 0 and 1); reused across calls, so repeated calls do not
// re-allocate hundreds of MB each time.
void stage_rows(Runner& r, const knng_dataset* ds, DevData& out, int slot) {
  check_ds(ds);
  DeviceGuard g(r.device);  // the caller's current device may be another GPU
  if (ds->elem_kind == KNNG_ELEM_U8) {
    const u64 cells = ds->n * ds->dims;
    out.own.alloc(r, cells);
    out.p = out.own.p;
    if (!cells) return;
    DBuf<uint8_t> tmp;
    const uint8_t* src = static_cast<const uint8_t*>(ds->data);
    if (ds->mem != KNNG_MEM_DEVICE) {
      tmp.alloc(r, cells);
      KNNG_CUDA(cudaMemcpyAsync(tmp.p, ds->data, cells, cudaMemcpyHostToDevice, r.stream));
      src = tmp.p;
    }
    const unsigned g = (unsigned)std::min<u64>(ceil_div<u64>(cells, 256), (u64)r.num_sms * 32);
    k_u8_to_f32<<<g, 256, 0, r.stream>>>(src, cells, out.own.p);
    KNNG_LAUNCH_CHECK();
    return;
  }
  if (ds->mem == KNNG_MEM_DEVICE) {
    out.p = static_cast<const float*>(ds->data);
    return;
  }
  float* dst = static_cast<float*>(
      r.scratch(slot ? Runner::kScrStage1 : Runner::kScrStage0, ds->n * ds->dims * 4 + 16));
  if (ds->n)
    KNNG_CUDA(cudaMemcpyAsync(dst, ds->data, ds->n * ds->dims * 4, cudaMemcpyHostToDevice,
                              r.stream));
  out.p = dst;
}

template <class T>
void copy_out(Runner& r, T* dst, const T* src, size_t count, bool dst_on_device) {
  if (!count) return;
  if (!dst_on_device) {
    d2h_host(r, dst, src, count * sizeof(T));
    return;
  }
  KNNG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToDevice, r.stream));
}
template <class T>
void copy_in(Runner& r, T* dst, const T* src, size_t count, bool src_on_device) {
  if (!count) return;
  KNNG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T),
                            src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            r.stream));
}

NndParams to_nnd(const knng_nnd_params* p) {
  NndParams o;
  o.k = (uint32_t)p->k;
  o.delta = p->delta;
  o.rho = p->rho;
  o.max_iters = p->max_iters;
  o.candidate_capacity = p->candidate_capacity;
  o.seed = p->seed;
  require(p->k <= 0xffffffffull, "nn_descent: k out of range");
  return o;
}

SearchParamsDev to_sp(const knng_search_params* p) {
  SearchParamsDev o;
  o.k_s = p->k_s;
  o.beam_width = p->beam_width;
  o.num_entry_points = p->num_entry_points;
  o.max_hops = p->max_hops;
  o.seed = p->seed;
  return o;
}

RefineCfg to_cfg(const knng_refine_config* c) {
  RefineCfg o;
  o.ranks = c->ranks;
  o.groups = c->groups;
  o.k = c->k;
  o.k_s = c->k_s;
  o.out_degree = c->out_degree;
  o.nn = to_nnd(&c->nn);
  o.nn.k = (uint32_t)c->k;
  o.search = to_sp(&c->search);
  o.skip_tree_phase = c->skip_tree_phase != 0;
  o.double_buffer = c->double_buffer != 0;
  o.capture_snapshots = c->capture_snapshots != 0;
  o.max_concat_bytes = c->max_concat_bytes;
  o.seed = c->seed;
  require(o.k >= 1 && o.k <= 32, "refine: the B200 path supports 1 <= k <= 32");
  return o;
}

void fill_dist_result(const DistResult& d, knng_dist_result* r) {
  if (!r) return;
  std::memset(r, 0, sizeof(*r));
  r->local_s = d.local_s;
  r->tree_s = d.tree_s;
  r->merge_s = d.merge_s;
  r->flat_s = d.flat_s;
  r->etc_s = d.etc_s;
  r->partition_s = d.partition_s;
  r->levels = d.levels;
  r->merge_epoch = d.merge_epoch;
  r->flat_epoch = d.flat_epoch;
  r->comm_gets = d.comm_log.size();
  for (const auto& g : d.comm_log) r->comm_bytes += g.bytes;
  r->search_hops = d.search.hops;
  r->search_scored = d.search.scored;
  r->nnd_pairs = d.nnd_pairs;
  r->nnd_iterations = d.nnd_iterations_max;
  r->num_snapshots = d.snap_labels.size();
}

// row_distance (core.hpp:82-93): l2_exact, or (nrm != null) the cosine dot
// chain in index order finished with the rows' norm chains.
__global__ void k_row_dist(const float* __restrict__ X, int d, const u32* __restrict__ i,
                           const u32* __restrict__ j, u64 count, float* __restrict__ out,
                           const float* __restrict__ nrm) {
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (u64)gridDim.x * blockDim.x) {
    const float* a = X + (u64)i[t] * d;
    const float* b = X + (u64)j[t] * d;
    if (!nrm) {
      out[t] = l2_exact(a, b, d);
      continue;
    }
    float dot = 0.0f;
    for (int e = 0; e < d; ++e) dot = dot_step(dot, a[e], b[e]);
    out[t] = cos_finish(dot, nrm[i[t]], nrm[j[t]]);
  }
}

__global__ void k_pack(const u32* __restrict__ ids, const float* __restrict__ dists, u64 count,
                       u64* __restrict__ keys) {
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (u64)gridDim.x * blockDim.x)
    keys[t] = pack_key(dists[t], ids[t]);
}

unsigned grid_for(const Runner& r, u64 count) {
  return (unsigned)std::max<u64>(1, std::min<u64>(ceil_div<u64>(count, 256), (u64)r.num_sms * 32));
}

}  // namespace

extern "C" {

int knng_abi_version(void) { return KNNG_ABI_VERSION; }

uint64_t knng_kernel_launches(void) { return launch_counter().load(std::memory_order_relaxed); }

const char* knng_last_error(void) { return g_err.c_str(); }

knng_status knng_ctx_create_on(const int* devices, int num_devices, knng_ctx** out) {
  return guard([&] {
    require(out != nullptr && devices != nullptr && num_devices > 0,
            "knng_ctx_create_on: null argument");
    int count = 0;
    KNNG_CUDA(cudaGetDeviceCount(&count));
    require(count > 0, "knng_ctx_create: no CUDA device");
    auto ctx = std::make_unique<knng_ctx>();
    for (int i = 0; i < num_devices; ++i) {
      require(devices[i] >= 0 && devices[i] < count, "knng_ctx_create_on: device out of range");
      ctx->devices.push_back(devices[i]);
      ctx->runners.push_back(std::make_unique<Runner>(devices[i]));
    }
    // NVLink peer access between every pair of the context's devices
    for (int ia = 0; ia < num_devices; ++ia) {
      const int a = devices[ia];
      DeviceGuard g(a);
      for (int ib = 0; ib < num_devices; ++ib) {
        const int b = devices[ib];
        if (a == b) continue;
        int ok = 0;
        KNNG_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
        if (!ok) continue;
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) KNNG_CUDA(e);
        cudaGetLastError();
        // Pool memory stays device-private: cross-GPU transfers are explicit
        // cudaMemcpyPeerAsync pulls (ThreadWorld), which need no pool mapping,
        // and mapping every pool allocation into all peers made pool growth
        // fail spuriously on 2-GPU boxes.
      }
    }
    *out = ctx.release();
  });
}

knng_status knng_ctx_create(int num_devices, knng_ctx** out) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) {
    cudaGetLastError();
    return guard([&] { throw CudaError("knng_ctx_create: no CUDA device"); });
  }
  if (num_devices <= 0 || num_devices > count) num_devices = count;
  std::vector<int> devs(num_devices);
  for (int d = 0; d < num_devices; ++d) devs[d] = d;
  return knng_ctx_create_on(devs.data(), num_devices, out);
}

void knng_ctx_destroy(knng_ctx* ctx) { delete ctx; }

knng_status knng_ctx_device_count(knng_ctx* ctx, int* out) {
  return guard([&] {
    require(ctx && out, "knng: null argument");
    *out = (int)ctx->devices.size();
  });
}

knng_status knng_ctx_stream(knng_ctx* ctx, int device, void** stream) {
  return guard([&] {
    require(ctx && stream, "knng: null argument");
    *stream = (void*)ctx->runner(device).stream;
  });
}

knng_status knng_row_distances(knng_ctx* ctx, int device, const knng_dataset* ds, const uint32_t* i,
                               const uint32_t* j, uint64_t count, float* out) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    DevData x;
    stage(r, ds, x);
    if (!count) return;
    DBuf<u32> di(r, count), dj(r, count);
    DBuf<float> dout(r, count);
    copy_in(r, di.p, i, count, false);
    copy_in(r, dj.p, j, count, false);
    k_row_dist<<<grid_for(r, count), 256, 0, r.stream>>>(x.p, (int)ds->dims, di.p, dj.p, count,
                                                         dout.p, x.nrm);
    KNNG_LAUNCH_CHECK();
    copy_out(r, out, dout.p, count, false);
    r.sync();
  });
}

knng_status knng_merge_rows(knng_ctx* ctx, int device, uint64_t rows, const uint32_t* a_ids,
                            const float* a_d, uint64_t na, const uint32_t* b_ids,
                            const float* b_d, uint64_t nb, uint64_t k, uint32_t* out_ids,
                            float* out_d, uint32_t* out_count) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(k >= 1 && k <= 32 && na <= 32 && nb <= 32,
            "merge_rows: the B200 path supports rows of <= 32 entries");
    if (!rows) return;
    DBuf<u32> ai(r, rows * na + 1), bi(r, rows * nb + 1), oi(r, rows * k), oc(r, rows);
    DBuf<float> ad(r, rows * na + 1), bdd(r, rows * nb + 1), od(r, rows * k);
    DBuf<u64> ak(r, rows * na + 1), ok(r, rows * k);
    copy_in(r, ai.p, a_ids, rows * na, false);
    copy_in(r, ad.p, a_d, rows * na, false);
    copy_in(r, bi.p, b_ids, rows * nb, false);
    copy_in(r, bdd.p, b_d, rows * nb, false);
    if (rows * na)
      k_pack<<<grid_for(r, rows * na), 256, 0, r.stream>>>(ai.p, ad.p, rows * na, ak.p);
      KNNG_LAUNCH_CHECK();
    merge_rows_device(r, ak.p, nullptr, (u32)na, bi.p, bdd.p, (u32)nb, 0, rows, (u32)k, ok.p,
                      nullptr, oc.p);
    export_graph_device(r, ok.p, nullptr, rows, (u32)k, 0, oi.p, od.p, nullptr);
    copy_out(r, out_ids, oi.p, rows * k, false);
    copy_out(r, out_d, od.p, rows * k, false);
    if (out_count) copy_out(r, out_count, oc.p, rows, false);
    r.sync();
  });
}

knng_status knng_init_random_graph(knng_ctx* ctx, int device, const knng_dataset* ds, uint64_t k,
                                   uint64_t seed, knng_graph* out) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    DevData x;
    stage(r, ds, x);
    require(out && out->n == ds->n && out->k == k, "init_random_graph: output shape mismatch");
    require(k >= 1 && k < ds->n, "init_random_graph: need 1 <= k < N");
    DBuf<u64> keys(r, ds->n * k);
    DBuf<u32> flags(r, ds->n);
    init_random_graph_device(r, DevRows{x.p, ds->n, (int)ds->dims, x.nrm}, (u32)k, seed, keys.p,
                             flags.p);
    const bool dev = out->mem == KNNG_MEM_DEVICE;
    DBuf<u32> ti;
    DBuf<float> td;
    DBuf<uint8_t> tf;
    uint32_t* oi = out->ids;
    float* od = out->dists;
    uint8_t* of = out->flags;
    if (!dev) {
      ti.alloc(r, ds->n * k);
      td.alloc(r, ds->n * k);
      tf.alloc(r, ds->n * k);
      oi = ti.p;
      od = td.p;
      of = out->flags ? tf.p : nullptr;
    }
    export_graph_device(r, keys.p, flags.p, ds->n, (u32)k, 0, oi, od, of);
    if (!dev) {
      copy_out(r, out->ids, ti.p, ds->n * k, false);
      copy_out(r, out->dists, td.p, ds->n * k, false);
      if (out->flags) copy_out(r, out->flags, tf.p, ds->n * k, false);
    }
    r.sync();
  });
}

knng_status knng_sample_neighbors(knng_ctx* ctx, int device, knng_graph* gph, double rho,
                                  uint64_t seed, uint64_t iter, uint32_t* new_fwd,
                                  uint32_t* new_fwd_n, uint32_t* old_fwd, uint32_t* old_fwd_n,
                                  uint32_t* new_rev, uint32_t* new_rev_n, uint32_t* old_rev,
                                  uint32_t* old_rev_n, uint64_t* bound) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(gph && gph->mem == KNNG_MEM_HOST && gph->flags, "sample_neighbors: host graph with flags");
    const u64 n = gph->n, k = gph->k;
    require(k >= 1 && k <= 32, "sample_neighbors: the B200 path supports 1 <= k <= 32");
    DBuf<u32> ti(r, n * k);
    DBuf<float> td(r, n * k);
    DBuf<uint8_t> tf(r, n * k);
    DBuf<u64> keys(r, n * k);
    DBuf<u32> flags(r, n);
    copy_in(r, ti.p, gph->ids, n * k, false);
    copy_in(r, td.p, gph->dists, n * k, false);
    copy_in(r, tf.p, gph->flags, n * k, false);
    import_graph_device(r, ti.p, td.p, tf.p, n, (u32)k, keys.p, flags.p);
    SampleLists s;
    sample_neighbors_device(r, n, (u32)k, rho, seed, iter, keys.p, flags.p, s);
    const u64 B = s.bound;
    export_graph_device(r, keys.p, flags.p, n, (u32)k, 0, nullptr, nullptr, tf.p);
    copy_out(r, gph->flags, tf.p, n * k, false);
    copy_out(r, new_fwd, s.nf.p, n * B, false);
    copy_out(r, new_fwd_n, s.nfn.p, n, false);
    copy_out(r, old_fwd, s.of.p, n * k, false);
    copy_out(r, old_fwd_n, s.ofn.p, n, false);
    copy_out(r, new_rev, s.nr.p, n * B, false);
    copy_out(r, new_rev_n, s.nrn.p, n, false);
    copy_out(r, old_rev, s.orv.p, n * B, false);
    copy_out(r, old_rev_n, s.orn.p, n, false);
    r.sync();
    if (bound) *bound = B;
  });
}

knng_status knng_nn_descent(knng_ctx* ctx, int device, const knng_dataset* ds,
                            const knng_nnd_params* params, knng_graph* out,
                            knng_nnd_stats* stats) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(params != nullptr && out != nullptr, "nn_descent: null argument");
    NndParams p = to_nnd(params);
    check_ds(ds);
    validate_nnd(p, ds->n);
    require(out->n == ds->n && out->k == p.k, "nn_descent: output shape mismatch");
    HostTrace tr("nn_descent");
    DevData x;
    stage(r, ds, x);
    const u64 n = ds->n, k = p.k;
    DBuf<u64> keys(r, n * k);
    DBuf<u32> flags(r, n);
    NndStats st;
    tr.mark("alloc");
    nn_descent_device(r, DevRows{x.p, n, (int)ds->dims, x.nrm}, p, keys.p, flags.p, &st,
                      stats != nullptr,
                      ctx->workspace(device));
    tr.mark("build");
    const bool dev = out->mem == KNNG_MEM_DEVICE;
    if (dev) {
      export_graph_device(r, keys.p, flags.p, n, (u32)k, 0, out->ids, out->dists, out->flags);
    } else {
      DBuf<u32> ti(r, n * k);
      DBuf<float> td(r, n * k);
      DBuf<uint8_t> tf(r, out->flags ? n * k : 0);
      export_graph_device(r, keys.p, flags.p, n, (u32)k, 0, ti.p, td.p,
                          out->flags ? tf.p : nullptr);
      copy_out(r, out->ids, ti.p, n * k, false);
      copy_out(r, out->dists, td.p, n * k, false);
      if (out->flags) copy_out(r, out->flags, tf.p, n * k, false);
      r.sync();
    }
    r.sync();
    if (stats) {
      stats->iterations = st.iterations;
      if (stats->accepted_per_iter)
        for (u64 i = 0; i < std::min<u64>(stats->accepted_cap, st.accepted_per_iter.size()); ++i)
          stats->accepted_per_iter[i] = st.accepted_per_iter[i];
      stats->pairs = st.pairs;
      stats->staged_rows = st.staged_rows;
      stats->offers = st.offers;
      stats->join_ms = st.join_ms;
      stats->total_ms = st.total_ms;
      stats->join_launches = st.join_launches;
      stats->offer_ms = st.offer_ms;
      for (int i = 0; i < 8; ++i) stats->stage_ms[i] = st.stage_ms[i];
      for (u64 i = 0; i < std::min<u64>(stats->accepted_cap, st.offers_per_iter.size()); ++i) {
        if (stats->offers_per_iter) stats->offers_per_iter[i] = st.offers_per_iter[i];
        if (stats->pairs_per_iter) stats->pairs_per_iter[i] = st.pairs_per_iter[i];
      }
      stats->launches = st.launches + 1;
    }
  });
}

knng_status knng_optimize_graph(knng_ctx* ctx, int device, const knng_graph* gph,
                                const knng_dataset* ds, uint64_t out_degree, uint32_t* sg_ids) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(gph && ds && sg_ids, "optimize_graph: null argument");
    if (out_degree == 0) out_degree = gph->k;
    require(out_degree <= gph->k, "optimize_graph: out_degree must be <= k");
    require(gph->n == ds->n, "optimize_graph: graph/dataset size mismatch");
    DevData x;
    stage(r, ds, x);
    const u64 n = gph->n, k = gph->k;
    const bool dev = gph->mem == KNNG_MEM_DEVICE;
    DBuf<u32> ti;
    DBuf<float> td;
    const u32* ids = gph->ids;
    const float* dd = gph->dists;
    if (!dev) {
      ti.alloc(r, n * k);
      td.alloc(r, n * k);
      copy_in(r, ti.p, gph->ids, n * k, false);
      copy_in(r, td.p, gph->dists, n * k, false);
      ids = ti.p;
      dd = td.p;
    }
    DBuf<u64> keys(r, n * k);
    import_graph_device(r, ids, dd, nullptr, n, (u32)k, keys.p, nullptr);
    if (dev) {
      optimize_graph_device(r, keys.p, n, (u32)k, 0, x.p, (int)ds->dims, (u32)out_degree, sg_ids,
                            nullptr, x.nrm);
    } else {
      DBuf<u32> sg(r, n * out_degree);
      optimize_graph_device(r, keys.p, n, (u32)k, 0, x.p, (int)ds->dims, (u32)out_degree, sg.p,
                            nullptr, x.nrm);
      copy_out(r, sg_ids, sg.p, n * out_degree, false);
      r.sync();
    }
    r.sync();
  });
}

static knng_status ann_search_impl(knng_ctx* ctx, int device, const knng_dataset* queries,
                            const uint32_t* sg_ids, uint64_t sg_n, uint64_t degree,
                            const knng_dataset* vectors, const knng_search_params* params,
                            uint8_t out_mem, uint32_t* out_ids, float* out_dists, uint32_t* hops,
                            uint32_t* scored, uint32_t* scored_ids, uint64_t scored_cap) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(queries && vectors && params, "ann_search: null argument");
    require(queries->dims == vectors->dims && queries->elem_kind == vectors->elem_kind &&
                queries->metric == vectors->metric,
            "ann_search: query/vector datasets incompatible");
    SearchParamsDev sp = to_sp(params);
    validate_search(queries->dims, vectors->dims, sg_n, vectors->n, sp);
    DevData q, v;
    stage(r, queries, q, 0);
    stage(r, vectors, v, 1);
    const u64 nq = queries->n;
    // the search graph: device if out_mem is device, else host
    DBuf<u32> sgd;
    const u32* sg = sg_ids;
    if (out_mem != KNNG_MEM_DEVICE) {
      sgd.alloc(r, sg_n * degree + 1);
      copy_in(r, sgd.p, sg_ids, sg_n * degree, false);
      sg = sgd.p;
    }
    if (nq == 0) return;
    const u64 ks = sp.k_s;
    if (out_mem == KNNG_MEM_DEVICE) {
      ann_search_device(r, q.p, nq, (int)queries->dims, sg, (u32)degree, v.p, vectors->n, sp, 0,
                        out_ids, out_dists, hops, scored, nullptr, 0, q.nrm, v.nrm, scored_ids,
                        scored_cap);
    } else {
      DBuf<u32> oi(r, nq * ks), hh(r, hops ? nq : 0), ss(r, scored ? nq : 0);
      DBuf<u32> si(r, scored_ids ? nq * scored_cap : 0);
      DBuf<float> od(r, nq * ks);
      ann_search_device(r, q.p, nq, (int)queries->dims, sg, (u32)degree, v.p, vectors->n, sp, 0,
                        oi.p, od.p, hops ? hh.p : nullptr, scored ? ss.p : nullptr, nullptr, 0,
                        q.nrm, v.nrm, scored_ids ? si.p : nullptr, scored_cap);
      if (scored_ids) copy_out(r, scored_ids, si.p, nq * scored_cap, false);
      copy_out(r, out_ids, oi.p, nq * ks, false);
      copy_out(r, out_dists, od.p, nq * ks, false);
      if (hops) copy_out(r, hops, hh.p, nq, false);
      if (scored) copy_out(r, scored, ss.p, nq, false);
      r.sync();
    }
    r.sync();
  });
}

knng_status knng_ann_search(knng_ctx* ctx, int device, const knng_dataset* queries,
                            const uint32_t* sg_ids, uint64_t sg_n, uint64_t degree,
                            const knng_dataset* vectors, const knng_search_params* params,
                            uint8_t out_mem, uint32_t* out_ids, float* out_dists, uint32_t* hops,
                            uint32_t* scored) {
  return ann_search_impl(ctx, device, queries, sg_ids, sg_n, degree, vectors, params, out_mem,
                         out_ids, out_dists, hops, scored, nullptr, 0);
}

knng_status knng_ann_search_scored_ids(knng_ctx* ctx, int device, const knng_dataset* queries,
                                       const uint32_t* sg_ids, uint64_t sg_n, uint64_t degree,
                                       const knng_dataset* vectors,
                                       const knng_search_params* params, uint8_t out_mem,
                                       uint32_t* out_ids, float* out_dists, uint32_t* hops,
                                       uint32_t* scored, uint32_t* scored_ids,
                                       uint64_t scored_cap) {
  if (!scored_ids || !scored) return ann_search_impl(ctx, device, queries, sg_ids, sg_n, degree,
                                                     vectors, params, out_mem, out_ids, out_dists,
                                                     hops, scored, nullptr, 0);
  return ann_search_impl(ctx, device, queries, sg_ids, sg_n, degree, vectors, params, out_mem,
                         out_ids, out_dists, hops, scored, scored_ids, scored_cap);
}

knng_status knng_search_throughput_probe(knng_ctx* ctx, int device,
                                         const knng_throughput_case* cases, uint64_t num_cases,
                                         const knng_dataset* queries,
                                         const knng_search_params* params,
                                         knng_throughput_row* rows) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(queries && params && (cases || num_cases == 0) && (rows || num_cases == 0),
            "search_throughput_probe: null argument");
    if (queries->n == 0)
      throw std::invalid_argument("search_throughput_probe: empty query set");  // :134-135
    for (uint64_t i = 1; i < num_cases; ++i)
      if (cases[i].source_count < cases[i - 1].source_count)
        throw std::invalid_argument("search_throughput_probe: sizes must ascend");  // :136-139
    const SearchParamsDev sp = to_sp(params);
    DevData q;
    stage(r, queries, q);
    const u64 nq = queries->n, ks = sp.k_s;
    DBuf<u32> oi(r, nq * ks);
    DBuf<float> od(r, nq * ks);
    cudaEvent_t e0, e1;
    KNNG_CUDA(cudaEventCreate(&e0));
    KNNG_CUDA(cudaEventCreate(&e1));
    struct Ev {
      cudaEvent_t a, b;
      ~Ev() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
    } ev{e0, e1};
    for (uint64_t i = 0; i < num_cases; ++i) {
      const knng_throughput_case& c = cases[i];
      require(c.vectors != nullptr && c.sg_ids != nullptr, "search_throughput_probe: null case");
      require(queries->dims == c.vectors->dims && queries->elem_kind == c.vectors->elem_kind &&
                  queries->metric == c.vectors->metric,
              "ann_search: query/vector datasets incompatible");
      validate_search(queries->dims, c.vectors->dims, c.sg_n, c.vectors->n, sp);
      DevData v;
      stage(r, c.vectors, v, 1);
      DBuf<u32> sgd;
      const u32* sg = c.sg_ids;
      if (c.sg_mem != KNNG_MEM_DEVICE) {
        sgd.alloc(r, c.sg_n * c.degree + 1);
        copy_in(r, sgd.p, c.sg_ids, c.sg_n * c.degree, false);
        sg = sgd.p;
      }
      r.sync();
      KNNG_CUDA(cudaEventRecord(e0, r.stream));
      ann_search_device(r, q.p, nq, (int)queries->dims, sg, (u32)c.degree, v.p, c.vectors->n, sp,
                        0, oi.p, od.p, nullptr, nullptr, nullptr, 0, q.nrm, v.nrm);
      KNNG_CUDA(cudaEventRecord(e1, r.stream));
      KNNG_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      KNNG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      knng_throughput_row& row = rows[i];
      row.source_count = c.source_count;
      row.num_queries = nq;
      row.seconds = ms / 1000.0;
      row.qps = row.seconds > 0.0 ? (double)nq / row.seconds : 0.0;
    }
  });
}

knng_status knng_partition(knng_ctx* ctx, int device, const knng_dataset* ds, uint64_t ranks,
                           uint64_t seed, uint8_t mem, uint32_t* to_external, uint64_t* offsets,
                           float* locals_out) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(ds && to_external && offsets, "partition_dataset: null argument");
    const u64 n = ds->n;
    require(!(ranks == 0 || ranks > n), "partition_dataset: need 1 <= P <= N");
    const bool dev = mem == KNNG_MEM_DEVICE;
    DBuf<u32> te;
    u32* tp = to_external;
    if (!dev) {
      te.alloc(r, n);
      tp = te.p;
    }
    std::vector<uint64_t> off;
    partition_device(r, n, (uint32_t)ranks, seed, tp, off);
    std::copy(off.begin(), off.end(), offsets);
    if (locals_out) {
      DevData x;
      stage(r, ds, x);
      if (dev) {
        gather_rows_device(r, x.p, (int)ds->dims, tp, n, locals_out);
      } else {
        DBuf<float> lo(r, n * ds->dims);
        gather_rows_device(r, x.p, (int)ds->dims, tp, n, lo.p);
        copy_out(r, locals_out, lo.p, n * ds->dims, false);
        r.sync();
      }
    }
    if (!dev) copy_out(r, to_external, te.p, n, false);
    r.sync();
  });
}

knng_status knng_tree_levels(uint64_t ranks, uint64_t groups, uint64_t* out) {
  return guard([&] { *out = tree_levels(ranks, groups); });
}

knng_status knng_tree_schedule(uint64_t ranks, uint64_t groups, uint64_t rank, uint64_t level,
                               uint64_t* group_lo, uint64_t* group_hi, uint64_t* partners) {
  return guard([&] {
    const TreeLevel t = tree_schedule(ranks, groups, rank, level);
    *group_lo = t.group_lo;
    *group_hi = t.group_hi;
    std::copy(t.partners.begin(), t.partners.end(), partners);
  });
}

knng_status knng_merge_results(knng_ctx* ctx, int device, knng_graph* gph, const uint32_t* res_ids,
                               const float* res_dists, uint64_t k_s, uint64_t id_base) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(gph && gph->mem == KNNG_MEM_HOST, "merge_results: host graph expected");
    const u64 n = gph->n, k = gph->k;
    require(k >= 1 && k <= 32 && k_s <= 32, "merge_rows: the B200 path supports k, k_s <= 32");
    DBuf<u32> ti(r, n * k), ri(r, n * k_s + 1);
    DBuf<float> td(r, n * k), rd(r, n * k_s + 1);
    DBuf<u64> keys(r, n * k);
    copy_in(r, ti.p, gph->ids, n * k, false);
    copy_in(r, td.p, gph->dists, n * k, false);
    copy_in(r, ri.p, res_ids, n * k_s, false);
    copy_in(r, rd.p, res_dists, n * k_s, false);
    import_graph_device(r, ti.p, td.p, nullptr, n, (u32)k, keys.p, nullptr);
    merge_results_device(r, keys.p, nullptr, n, (u32)k, ri.p, rd.p, (u32)k_s, (u32)id_base);
    export_graph_device(r, keys.p, nullptr, n, (u32)k, 0, ti.p, td.p, nullptr);
    copy_out(r, gph->ids, ti.p, n * k, false);
    copy_out(r, gph->dists, td.p, n * k, false);
    r.sync();
  });
}

knng_status knng_translate_to_external(knng_ctx* ctx, int device, const uint32_t* to_external,
                                       uint64_t n, uint64_t k, const uint32_t* ids,
                                       const float* dists, uint32_t* out_ids, float* out_dists) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(k >= 1 && k <= 32, "translate_to_external: the B200 path supports k <= 32");
    DBuf<u32> te(r, n), ti(r, n * k), oi(r, n * k);
    DBuf<float> td(r, n * k), od(r, n * k);
    DBuf<u64> keys(r, n * k);
    copy_in(r, te.p, to_external, n, false);
    copy_in(r, ti.p, ids, n * k, false);
    copy_in(r, td.p, dists, n * k, false);
    import_graph_device(r, ti.p, td.p, nullptr, n, (u32)k, keys.p, nullptr);
    translate_device(r, keys.p, n, (u32)k, te.p, oi.p, od.p);
    copy_out(r, out_ids, oi.p, n * k, false);
    copy_out(r, out_dists, od.p, n * k, false);
    r.sync();
  });
}

knng_status knng_build_distributed(knng_ctx* ctx, const knng_dataset* ds,
                                   const knng_refine_config* cfg, knng_graph* out,
                                   knng_dist_result* result, uint32_t* snap_ids, float* snap_dists,
                                   uint64_t snap_cap) {
  return guard([&] {
    require(ctx && ds && cfg && out, "build_distributed: null argument");
    check_ds(ds);
    RefineCfg c = to_cfg(cfg);
    c.cosine = ds->metric == KNNG_METRIC_COS;
    require(out->n == ds->n && out->k == c.k, "build_distributed: output shape mismatch");
    DistResult res;
    const float* xp = static_cast<const float*>(ds->data);
    bool x_dev = ds->mem == KNNG_MEM_DEVICE;
    DevData staged;
    if (ds->elem_kind == KNNG_ELEM_U8) {  // rows expanded to f32 on device 0
      stage(ctx->runner(ctx->devices[0]), ds, staged);
      ctx->runner(ctx->devices[0]).sync();
      xp = staged.p;
      x_dev = true;
      c.u8_elems = true;
    }
    build_distributed(ctx->devices, xp, x_dev, ds->n, (int)ds->dims, c, out->ids, out->dists,
                      out->mem == KNNG_MEM_DEVICE, &res);
    ctx->last_log = res.comm_log;
    fill_dist_result(res, result);
    if (snap_ids && snap_dists) {
      const u64 cells = ds->n * c.k;
      for (u64 s = 0; s < std::min<u64>(snap_cap, res.snap_labels.size()); ++s) {
        std::copy(res.snap_ids[s].begin(), res.snap_ids[s].end(), snap_ids + s * cells);
        std::copy(res.snap_dists[s].begin(), res.snap_dists[s].end(), snap_dists + s * cells);
      }
    }
  });
}

knng_status knng_build_distributed_rank(knng_ctx* ctx, int device, uint64_t rank,
                                        uint64_t world_size, knng_allgather_fn allgather,
                                        void* user, const knng_dataset* ds,
                                        const knng_refine_config* cfg, uint32_t* out_ids,
                                        float* out_dists, uint32_t* out_rows, int out_mem,
                                        uint64_t* rows_out, knng_dist_result* result) {
  return guard([&] {
    require(ctx && ds && cfg && out_ids && out_dists && out_rows && allgather,
            "build_distributed: null argument");
    ctx->runner(device);  // the device belongs to this context
    check_ds(ds);
    RefineCfg c = to_cfg(cfg);
    c.ranks = world_size;
    c.cosine = ds->metric == KNNG_METRIC_COS;
    HostTransport t;
    t.user = user;
    t.allgather = allgather;
    DistResult res;
    const float* xp = static_cast<const float*>(ds->data);
    bool x_dev = ds->mem == KNNG_MEM_DEVICE;
    DevData staged;
    if (ds->elem_kind == KNNG_ELEM_U8) {  // rows expanded to f32 on this rank's device
      stage(ctx->runner(device), ds, staged);
      ctx->runner(device).sync();
      xp = staged.p;
      x_dev = true;
      c.u8_elems = true;
    }
    const uint64_t rows = build_distributed_rank(
        device, (size_t)rank, (size_t)world_size, t, xp, x_dev, ds->n, (int)ds->dims, c, out_ids,
        out_dists, out_rows, out_mem == KNNG_MEM_DEVICE, &res, &ctx->runner(device),
        ctx->workspace(device));
    if (rows_out) *rows_out = rows;
    ctx->last_log = res.comm_log;
    fill_dist_result(res, result);
  });
}

knng_status knng_refine(knng_ctx* ctx, const float* x_perm, uint64_t n, uint64_t dims,
                        const knng_refine_config* cfg, const uint64_t* offsets, uint32_t* ids,
                        float* dists, int mode, knng_dist_result* result) {
  return guard([&] {
    require(ctx && x_perm && cfg && offsets && ids && dists, "refine: null argument");
    const RefineCfg c = to_cfg(cfg);
    std::vector<uint64_t> off(offsets, offsets + c.ranks + 1);
    DistResult res;
    refine_from_local(ctx->devices, x_perm, n, (int)dims, c, off, ids, dists, mode, &res);
    ctx->last_log = res.comm_log;
    fill_dist_result(res, result);
  });
}

knng_status knng_refine_phase(knng_ctx* ctx, const float* x_perm, uint64_t n, uint64_t dims,
                              const knng_refine_config* cfg, const uint64_t* offsets, int phase,
                              uint64_t* epoch, uint32_t* ids, float* dists,
                              const uint32_t* sg_in, uint32_t* sg_out,
                              knng_dist_result* result) {
  return guard([&] {
    require(ctx && x_perm && cfg && offsets && ids && dists && epoch, "refine: null argument");
    const RefineCfg c = to_cfg(cfg);
    std::vector<uint64_t> off(offsets, offsets + c.ranks + 1);
    DistResult res;
    refine_phase(ctx->devices, x_perm, n, (int)dims, c, off, phase, *epoch, ids, dists, sg_in,
                 sg_out, &res, epoch);
    ctx->last_log = res.comm_log;
    fill_dist_result(res, result);
  });
}

knng_status knng_effective_groups(const knng_refine_config* cfg, const uint64_t* offsets,
                                  uint64_t dims, uint64_t* groups) {
  return guard([&] {
    require(cfg && offsets && groups, "effective_groups: null argument");
    const RefineCfg c = to_cfg(cfg);
    std::vector<uint64_t> off(offsets, offsets + c.ranks + 1);
    *groups = effective_group_count(off, c, (int)dims);
  });
}

knng_status knng_last_comm_log(knng_ctx* ctx, knng_get_record* records, uint64_t cap,
                               uint64_t* count) {
  return guard([&] {
    require(ctx && count, "knng: null argument");
    *count = ctx->last_log.size();
    for (u64 i = 0; i < std::min<u64>(cap, ctx->last_log.size()); ++i) {
      const GetRecord& g = ctx->last_log[i];
      records[i].src = g.src;
      records[i].target = g.target;
      std::memset(records[i].region, 0, sizeof(records[i].region));
      std::strncpy(records[i].region, g.region.c_str(), sizeof(records[i].region) - 1);
      records[i].bytes = g.bytes;
      records[i].epoch = g.epoch;
    }
  });
}

knng_status knng_brute_force(knng_ctx* ctx, int device, const knng_dataset* ds,
                             const uint64_t* rows, uint64_t q, uint64_t k, uint8_t out_mem,
                             uint32_t* out_ids, float* out_dists) {
  return guard([&] {
    Runner& r = ctx->runner(device);
    DeviceGuard g(r.device);
    require(k < ds->n, "brute_force_knng: k must be < N");
    DevData x;
    stage(r, ds, x);
    DBuf<u64> rw(r, q + 1);
    copy_in(r, rw.p, rows, q, false);
    if (out_mem == KNNG_MEM_DEVICE) {
      brute_force_rows_device(r, x.p, ds->n, (int)ds->dims, rw.p, q, (u32)k, out_ids, out_dists,
                              x.nrm);
    } else {
      DBuf<u32> oi(r, q * k);
      DBuf<float> od(r, q * k);
      brute_force_rows_device(r, x.p, ds->n, (int)ds->dims, rw.p, q, (u32)k, oi.p, od.p, x.nrm);
      copy_out(r, out_ids, oi.p, q * k, false);
      copy_out(r, out_dists, od.p, q * k, false);
      r.sync();
    }
    r.sync();
  });
}

knng_status knng_gen_random_dataset(uint64_t n, uint64_t dims, int dist, uint64_t seed,
                                    uint64_t clusters, float* out) {
  return guard([&] { gen_random_dataset(n, dims, dist, seed, clusters, out); });
}

knng_status knng_save_graph(const knng_graph* g, const char* path) {
  return guard([&] {
    require(g && g->mem == KNNG_MEM_HOST && path, "save_graph: host graph and path expected");
    save_graph(g->ids, g->dists, g->n, g->k, path);
  });
}

knng_status knng_load_graph_header(const char* path, uint64_t* n, uint64_t* k) {
  return guard([&] { load_graph_header(path, n, k); });
}

knng_status knng_load_graph(const char* path, knng_graph* out) {
  return guard([&] {
    require(out && out->mem == KNNG_MEM_HOST, "load_graph: host graph expected");
    load_graph(path, out->ids, out->dists, out->n, out->k);
  });
}

static uint64_t vecs_esz(int elem) {
  require(elem == KNNG_ELEM_F32 || elem == KNNG_ELEM_U8 || elem == KNNG_ELEM_I32,
          "vecs: element kind must be f32 (.fvecs), u8 (.bvecs) or i32 (.ivecs)");
  return elem == KNNG_ELEM_U8 ? 1 : 4;
}

knng_status knng_vecs_shape(const char* path, int elem, uint64_t* rows, uint64_t* dims) {
  return guard([&] {
    require(path && rows && dims, "vecs: null argument");
    vecs_shape(path, vecs_esz(elem), rows, dims);
  });
}

knng_status knng_read_vecs(knng_ctx* ctx, int device, const char* path, int elem, void* out,
                           uint64_t rows, uint64_t dims, uint8_t mem) {
  return guard([&] {
    require(path && (out || rows == 0), "vecs: null argument");
    const Runner* r = nullptr;
    if (mem == KNNG_MEM_DEVICE) {
      require(ctx != nullptr, "read_vecs: a context is needed for device output");
      r = &ctx->runner(device);
    }
    read_vecs(path, vecs_esz(elem), out, rows, dims, r);
  });
}

knng_status knng_write_vecs(const char* path, int elem, const void* data, uint64_t rows,
                            uint64_t dims) {
  return guard([&] {
    require(path && (data || rows == 0), "vecs: null argument");
    write_vecs(path, data, rows, dims, vecs_esz(elem));
  });
}

}  // extern "C"
