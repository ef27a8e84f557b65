/*
 * knng_c.h -- C-ABI of the B200-native kNN-graph construction path
 * (libknng_b200.so).  Drop-in boundary for the reference's public C++ API
 * (/root/reference/proj/include/knng/ headers): every entry point below cites the
 * reference function it replaces.  Plain pointers and sizes only; no
 * exceptions cross the boundary (status codes map 1:1 onto the reference's
 * exception classes, knng_last_error() carries e.what()).
 *
 * Memory: every dataset / graph argument says where its buffers live
 * (KNNG_MEM_HOST or KNNG_MEM_DEVICE).  Host inputs are copied to the GPU and
 * host outputs copied back inside the call; device buffers must live on the
 * device the call runs on.  All calls are synchronous w.r.t. the host.
 *
 * Threading: one knng_ctx per process; a ctx is not thread-safe per call.
 * build_distributed runs one internal host thread per rank.
 */
#ifndef KNNG_C_H
#define KNNG_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNNG_ABI_VERSION 1

typedef enum {
  KNNG_OK = 0,
  KNNG_EINVAL = 1,   /* std::invalid_argument */
  KNNG_EWORLD = 2,   /* WorldError (distsim.hpp:19-21) */
  KNNG_EABORTED = 3, /* WorldAborted (distsim.hpp:24-26) */
  KNNG_EFORMAT = 4,  /* FormatError / wire corruption (evalio.hpp:14, wire.cpp:100) */
  KNNG_ELOGIC = 5,   /* std::logic_error (core.cpp:166-186) */
  KNNG_ECUDA = 6,    /* CUDA runtime failure */
  KNNG_ENOMEM = 7,
  KNNG_ERUNTIME = 8  /* any other std::runtime_error */
} knng_status;

enum { KNNG_MEM_HOST = 0, KNNG_MEM_DEVICE = 1 };
enum { KNNG_ELEM_F32 = 0, KNNG_ELEM_U8 = 1 };     /* ElemKind core.hpp:14 */
enum { KNNG_ELEM_I32 = 2 };                       /* .ivecs payload (IdMatrix, evalio.hpp:26-31) */
enum { KNNG_METRIC_L2 = 0, KNNG_METRIC_COS = 1 }; /* MetricKind core.hpp:15 */

typedef struct knng_ctx knng_ctx;

/* Dataset core.hpp:67-105: n x dims row-major. */
typedef struct {
  const void* data;
  uint64_t n;
  uint64_t dims;
  uint8_t elem_kind;
  uint8_t metric;
  uint8_t mem;
  uint8_t reserved;
} knng_dataset;

/* KnnGraph core.hpp:156-179: n x k ids + dists (+ optional u8 flags). */
typedef struct {
  uint32_t* ids;
  float* dists;
  uint8_t* flags; /* nullable */
  uint64_t n;
  uint64_t k;
  uint8_t mem;
  uint8_t reserved[7];
} knng_graph;

/* NnDescentParams nndescent.hpp:12-20 */
typedef struct {
  uint64_t k;
  double delta;
  double rho;
  uint64_t max_iters;
  uint64_t candidate_capacity; /* 0 -> 2k */
  uint64_t seed;
  uint64_t workers; /* accepted for API parity; the GPU ignores it */
} knng_nnd_params;

/* NnDescentStats nndescent.hpp:113-116 + device counters */
typedef struct {
  uint64_t iterations;
  uint64_t* accepted_per_iter; /* caller array of accepted_cap entries, nullable */
  uint64_t accepted_cap;
  uint64_t pairs;       /* sigma evaluations */
  uint64_t staged_rows; /* feature rows staged by the join (algorithmic bytes) */
  uint64_t offers;
  double join_ms;   /* device time of the join kernel, summed (CUDA events) */
  double total_ms;  /* device time of the whole build */
  uint64_t join_launches;
  uint64_t launches;
  double offer_ms; /* device time of the offer (atomicMin cascade) kernel, summed */
  /* device time per stage (ms): init, sample, join lists, join, offer, apply,
   * readback + host gaps, unused */
  double stage_ms[8];
  uint64_t* offers_per_iter; /* caller arrays of accepted_cap entries, nullable */
  uint64_t* pairs_per_iter;
} knng_nnd_stats;

/* SearchParams annsearch.hpp:12-19 */
typedef struct {
  uint64_t k_s;
  uint64_t beam_width;
  uint64_t num_entry_points;
  uint64_t max_hops; /* 0 -> 4 * beam_width */
  uint64_t seed;
  uint64_t workers; /* ignored */
} knng_search_params;

/* RefineConfig refine.hpp:37-52 */
typedef struct {
  uint64_t ranks;
  uint64_t groups;
  uint64_t k;
  uint64_t k_s;
  uint64_t out_degree;
  knng_nnd_params nn;
  knng_search_params search;
  uint8_t skip_tree_phase;
  uint8_t double_buffer;
  uint8_t capture_snapshots;
  uint8_t reserved[5];
  uint64_t max_concat_bytes;
  uint64_t seed;
} knng_refine_config;

/* DistBuildResult refine.hpp:91-107 */
typedef struct {
  double local_s, tree_s, merge_s, flat_s, etc_s, partition_s;
  uint64_t levels;
  uint64_t merge_epoch;
  uint64_t flat_epoch;
  uint64_t comm_gets;
  uint64_t comm_bytes; /* sum of wire region sizes, as the reference logs */
  uint64_t search_hops;
  uint64_t search_scored;
  uint64_t nnd_pairs;
  uint64_t nnd_iterations;
  uint64_t num_snapshots;
} knng_dist_result;

/* GetRecord distsim.hpp:28-34 */
typedef struct {
  uint64_t src;
  uint64_t target;
  char region[16];
  uint64_t bytes;
  uint64_t epoch;
} knng_get_record;

/* ---- library / context ----------------------------------------------- */
int knng_abi_version(void);
const char* knng_last_error(void);
/* Number of CUDA kernels this library has launched in this process (all
 * devices, all calls) -- launch accounting for benchmarks; no reference
 * counterpart. */
uint64_t knng_kernel_launches(void);
/* num_devices <= 0: every visible device.  Enables NVLink peer access. */
knng_status knng_ctx_create(int num_devices, knng_ctx** out);
/* A context on the listed devices only (e.g. one process per GPU: its own
 * device; peers are reached through IPC mappings, not contexts). */
knng_status knng_ctx_create_on(const int* devices, int num_devices, knng_ctx** out);
void knng_ctx_destroy(knng_ctx* ctx);
knng_status knng_ctx_device_count(knng_ctx* ctx, int* out);
/* The stream calls on `device` run on (for CUDA-event timing by callers). */
knng_status knng_ctx_stream(knng_ctx* ctx, int device, void** stream);

/* ---- core (core.hpp) ---------------------------------------------------- */
/* Batched exact distance sigma(x_i, x_j) (Dataset::row_distance core.hpp:84-95)
 * for `count` index pairs; i/j/out host arrays. */
knng_status knng_row_distances(knng_ctx* ctx, int device, const knng_dataset* ds,
                               const uint32_t* i, const uint32_t* j, uint64_t count,
                               float* out);
/* merge_rows core.cpp:114-134, batched: rows x (na | nb) sorted rows in, rows x k
 * out (+ per-row counts); host arrays. */
knng_status knng_merge_rows(knng_ctx* ctx, int device, uint64_t rows, const uint32_t* a_ids,
                            const float* a_d, uint64_t na, const uint32_t* b_ids,
                            const float* b_d, uint64_t nb, uint64_t k, uint32_t* out_ids,
                            float* out_d, uint32_t* out_count);

/* ---- nndescent (nndescent.hpp) ----------------------------------------- */
/* init_random_graph nndescent.cpp:29-62 */
knng_status knng_init_random_graph(knng_ctx* ctx, int device, const knng_dataset* ds,
                                   uint64_t k, uint64_t seed, knng_graph* out);
/* sample_neighbors nndescent.cpp:64-129 on a host graph (flags consumed in
 * place).  Lists are host arrays: new_fwd n x bound, old_fwd n x k, new_rev /
 * old_rev n x bound, with per-point counts.  Returns bound in *bound. */
knng_status knng_sample_neighbors(knng_ctx* ctx, int device, knng_graph* g, double rho,
                                  uint64_t seed, uint64_t iter, uint32_t* new_fwd,
                                  uint32_t* new_fwd_n, uint32_t* old_fwd, uint32_t* old_fwd_n,
                                  uint32_t* new_rev, uint32_t* new_rev_n, uint32_t* old_rev,
                                  uint32_t* old_rev_n, uint64_t* bound);
/* nn_descent nndescent.cpp:225-259 */
knng_status knng_nn_descent(knng_ctx* ctx, int device, const knng_dataset* ds,
                            const knng_nnd_params* params, knng_graph* out,
                            knng_nnd_stats* stats);

/* ---- graphopt / annsearch ---------------------------------------------- */
/* optimize_graph graphopt.cpp:24-105; sg_ids n x out_degree (mem = g->mem). */
knng_status knng_optimize_graph(knng_ctx* ctx, int device, const knng_graph* g,
                                const knng_dataset* ds, uint64_t out_degree, uint32_t* sg_ids);
/* ann_search annsearch.cpp:50-129; outputs nq x k_s in mem `out_mem`; hops /
 * scored (SearchDiagnostics annsearch.hpp:37-41) nullable, same mem. */
knng_status knng_ann_search(knng_ctx* ctx, int device, const knng_dataset* queries,
                            const uint32_t* sg_ids, uint64_t sg_n, uint64_t degree,
                            const knng_dataset* vectors, const knng_search_params* params,
                            uint8_t out_mem, uint32_t* out_ids, float* out_dists,
                            uint32_t* hops, uint32_t* scored);
/* ann_search with SearchDiagnostics::collect_scored_ids (annsearch.hpp:36-41):
 * additionally writes each query's scored ids in scoring order into
 * scored_ids[q * scored_cap ...] (the first min(scored[q], scored_cap) of
 * them); hops and scored are required.  Call with the scored counts of a first
 * knng_ann_search to size scored_cap exactly (the search is deterministic). */
knng_status knng_ann_search_scored_ids(knng_ctx* ctx, int device, const knng_dataset* queries,
                                       const uint32_t* sg_ids, uint64_t sg_n, uint64_t degree,
                                       const knng_dataset* vectors,
                                       const knng_search_params* params, uint8_t out_mem,
                                       uint32_t* out_ids, float* out_dists, uint32_t* hops,
                                       uint32_t* scored, uint32_t* scored_ids,
                                       uint64_t scored_cap);

/* search_throughput_probe annsearch.cpp:131-155 (ThroughputCase / Row,
 * annsearch.hpp:52-69): the batch search of `queries` against each case's
 * graph, cases in ascending source_count; seconds = device time of the
 * search (CUDA events on the context stream; inputs staged before timing).
 * sg_ids host or device per sg_mem. */
typedef struct {
  uint64_t source_count;
  const uint32_t* sg_ids;
  uint64_t sg_n, degree;
  const knng_dataset* vectors;
  uint8_t sg_mem;
} knng_throughput_case;
typedef struct {
  uint64_t source_count, num_queries;
  double seconds, qps;
} knng_throughput_row;
knng_status knng_search_throughput_probe(knng_ctx* ctx, int device,
                                         const knng_throughput_case* cases, uint64_t num_cases,
                                         const knng_dataset* queries,
                                         const knng_search_params* params,
                                         knng_throughput_row* rows);

/* ---- refine (refine.hpp) ----------------------------------------------- */
/* partition_dataset refine.cpp:86-126: to_external (n, mem `mem`) and offsets
 * (ranks+1, host).  locals_out (nullable, same mem): all rows in internal
 * order, i.e. Partition::locals concatenated. */
knng_status knng_partition(knng_ctx* ctx, int device, const knng_dataset* ds, uint64_t ranks,
                           uint64_t seed, uint8_t mem, uint32_t* to_external, uint64_t* offsets,
                           float* locals_out);
/* tree_levels / tree_schedule refine.cpp:128-149 */
knng_status knng_tree_levels(uint64_t ranks, uint64_t groups, uint64_t* out);
knng_status knng_tree_schedule(uint64_t ranks, uint64_t groups, uint64_t rank, uint64_t level,
                               uint64_t* group_lo, uint64_t* group_hi, uint64_t* partners);
/* merge_results_into refine.cpp:49-60: g (in place) with result rows + id_base */
knng_status knng_merge_results(knng_ctx* ctx, int device, knng_graph* g,
                               const uint32_t* res_ids, const float* res_dists, uint64_t k_s,
                               uint64_t id_base);
/* translate_to_external refine.cpp:395-416 (host arrays) */
knng_status knng_translate_to_external(knng_ctx* ctx, int device, const uint32_t* to_external,
                                       uint64_t n, uint64_t k, const uint32_t* ids,
                                       const float* dists, uint32_t* out_ids, float* out_dists);
/* build_distributed refine.cpp:504-586.  out: N x k external graph.  result,
 * snapshots (num x N x k host arrays, nullable) optional. */
knng_status knng_build_distributed(knng_ctx* ctx, const knng_dataset* ds,
                                   const knng_refine_config* cfg, knng_graph* out,
                                   knng_dist_result* result, uint32_t* snap_ids,
                                   float* snap_dists, uint64_t snap_cap);
/* Host transport for one-process-per-GPU builds: an all-gather -- out =
 * world_size consecutive blocks of `bytes`, in rank order.  Return 0 on
 * success (nonzero aborts the build with KNNG_EWORLD). */
typedef int (*knng_allgather_fn)(void* user, const void* in, uint64_t bytes, void* out);
/* One rank of build_distributed (refine.cpp:504-586) in this process, for
 * launches with one process per GPU (torchrun).  Collective: every rank calls
 * it with the same full dataset and config; the partition is recomputed
 * identically per rank, the rank's block is built and refined on `device`,
 * and published regions are shared as CUDA IPC handles exchanged with
 * `allgather` (pulls stay one-sided NVLink copies, RankWorld::one_sided_get).
 * Outputs (ceil(N / world_size) rows capacity, host or device per out_mem):
 * the rank's rows of the final graph in external ids (rows x k) and each
 * row's external id; *rows_out = the rank's row count.  result->comm_log
 * covers every rank's gets. */
knng_status knng_build_distributed_rank(knng_ctx* ctx, int device, uint64_t rank,
                                        uint64_t world_size, knng_allgather_fn allgather,
                                        void* user, const knng_dataset* ds,
                                        const knng_refine_config* cfg, uint32_t* out_ids,
                                        float* out_dists, uint32_t* out_rows, int out_mem,
                                        uint64_t* rows_out, knng_dist_result* result);
/* World-level drivers from given local graphs (internal global ids):
 * mode 0 = binary_tree_refine -> grouped_merge -> flat_refine,
 * mode 1 = all_to_all_refine (refine.hpp:117-136).  x_perm: rows in internal
 * order (host, f32, l2 metric: the raw-row signature carries no metric --
 * cosine datasets go through knng_build_distributed[_rank]); ids/dists
 * updated in place (host). */
knng_status knng_refine(knng_ctx* ctx, const float* x_perm, uint64_t n, uint64_t dims,
                        const knng_refine_config* cfg, const uint64_t* offsets, uint32_t* ids,
                        float* dists, int mode, knng_dist_result* result);
/* The world-level phase drivers one at a time (refine.hpp:119-136,
 * refine.cpp:430-502): phase 1 all_to_all_refine, 2 binary_tree_refine, 3
 * grouped_merge, 4 flat_refine.  Each publishes what its phase needs (dataset + graph, or
 * dataset + the rank's group search graph for flat_refine), barriers and runs
 * its phase on every rank, like the reference's drivers on a caller-owned
 * RankWorld: the world starts at epoch *epoch and *epoch receives its epoch at
 * the end (the C++ drop-in's RankWorld carries it between calls).  ids/dists:
 * n x k internal global ids, rank blocks at offsets, updated in place (phases
 * 1, 2 and 4).  sg_in (phase 4) / sg_out (phase 3): per-rank blocks in rank order,
 * block r = the search graph of rank r's group (group points x out_degree).
 * The gets are in knng_last_comm_log. */
knng_status knng_refine_phase(knng_ctx* ctx, const float* x_perm, uint64_t n, uint64_t dims,
                              const knng_refine_config* cfg, const uint64_t* offsets, int phase,
                              uint64_t* epoch, uint32_t* ids, float* dists,
                              const uint32_t* sg_in, uint32_t* sg_out,
                              knng_dist_result* result);
/* effective_groups refine.cpp:160-183: the group count the refine phases use
 * (cfg->groups, or P when skip_tree_phase is set or the max_concat_bytes
 * footprint estimate is exceeded); offsets = P + 1 rank block bounds. */
knng_status knng_effective_groups(const knng_refine_config* cfg, const uint64_t* offsets,
                                  uint64_t dims, uint64_t* groups);
/* Comm log of the last build_distributed / refine (RankWorld::comm_log). */
knng_status knng_last_comm_log(knng_ctx* ctx, knng_get_record* records, uint64_t cap,
                               uint64_t* count);

/* ---- evalio (measurement support, evalio.hpp) -------------------------- */
/* brute_force_knng evalio.cpp:125-147 for rows[0..q) (host) of ds; out q x k */
knng_status knng_brute_force(knng_ctx* ctx, int device, const knng_dataset* ds,
                             const uint64_t* rows, uint64_t q, uint64_t k, uint8_t out_mem,
                             uint32_t* out_ids, float* out_dists);
/* gen_random_dataset evalio.cpp:242-272 (host; dist 0 uniform, 1 gaussian,
 * 2 clustered) -- the reference's generator, bit-exact. */
knng_status knng_gen_random_dataset(uint64_t n, uint64_t dims, int dist, uint64_t seed,
                                    uint64_t clusters, float* out);
/* save_graph / load_graph evalio.cpp:274-280 + wire.cpp (22-byte header,
 * u32 ids, f32 dists, little-endian); host graphs. */
knng_status knng_save_graph(const knng_graph* g, const char* path);
knng_status knng_load_graph_header(const char* path, uint64_t* n, uint64_t* k);
knng_status knng_load_graph(const char* path, knng_graph* out);
/* read_vecs / write_vecs / read_ivecs / write_ivecs evalio.cpp:31-123: per row
 * a little-endian i32 dimension, then the row (.fvecs f32, .bvecs u8, .ivecs
 * i32 per `elem`).  vecs_shape validates every row (FormatError on a
 * truncated field/payload, a non-positive or inconsistent dimension) and
 * returns rows x dims; read_vecs fills rows x dims elements into host memory,
 * or into device memory through pinned staging buffers (mem = device). */
knng_status knng_vecs_shape(const char* path, int elem, uint64_t* rows, uint64_t* dims);
knng_status knng_read_vecs(knng_ctx* ctx, int device, const char* path, int elem, void* out,
                           uint64_t rows, uint64_t dims, uint8_t mem);
knng_status knng_write_vecs(const char* path, int elem, const void* data, uint64_t rows,
                            uint64_t dims);

#ifdef __cplusplus
}
#endif
#endif /* KNNG_C_H */
