/*
 * knng_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU algorithm (SOLANET desk-scale
 * implementation, /root/reference/proj) for the kNN-graph construction hot
 * path.  It is the checker for the B200 kernels in paper_2605_27691_b200/: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * The product library never links it and has no CPU fallback.
 *
 * Parity of this restatement is PINNED against the reference itself: the
 * recipe oracle/Makefile compiles the reference src/ .cpp files unchanged into
 * oracle/_ref/libknng_ref.so, tests/golden/make_golden.py runs it to mint the
 * fixtures in tests/golden/, and tests/test_oracle.py checks every function
 * below against those fixtures bit-for-bit.
 *
 * Every function cites the reference file:line it restates.  Semantics follow
 * the reference with workers = 1 (the deterministic schedule).
 */
#ifndef KNNG_ORACLE_H
#define KNNG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:12-96 ---------------------------------------------------- */
typedef struct {
  uint64_t state;
  float spare;
  int have_spare;
} ko_rng;

void ko_rng_init(ko_rng* r, uint64_t seed);
uint64_t ko_next_u64(ko_rng* r);
uint64_t ko_next_below(ko_rng* r, uint64_t bound);
float ko_next_float(ko_rng* r);
float ko_next_gaussian(ko_rng* r);
uint64_t ko_mix_seed(uint64_t a, uint64_t b);
/* sample_distinct rng.hpp:66-87; returns count written (min(m, n)). */
size_t ko_sample_distinct(uint64_t n, size_t m, ko_rng* r, uint32_t* out);
/* shuffle rng.hpp:90-96 over u32 */
void ko_shuffle_u32(uint32_t* v, size_t n, ko_rng* r);

/* ---- core.hpp:23-55 ---------------------------------------------------- */
float ko_l2_f32(const float* a, const float* b, size_t d);
float ko_l2_u8(const uint8_t* a, const uint8_t* b, size_t d);
float ko_cosine_f32(const float* a, const float* b, size_t d);
float ko_cosine_u8(const uint8_t* a, const uint8_t* b, size_t d);

/* Dataset descriptor: elem 0 = f32, 1 = u8; metric 0 = l2, 1 = cosine. */
typedef struct {
  const void* data;
  size_t n;
  size_t dims;
  int elem;
  int metric;
} ko_dataset;

float ko_row_distance(const ko_dataset* ds, size_t i, size_t j);
float ko_cross_distance(const ko_dataset* a, size_t i, const ko_dataset* b, size_t j);

/* ---- core.cpp:99-134 ---------------------------------------------------- */
typedef struct {
  uint32_t id;
  float dist;
  uint8_t flag;
} ko_entry;

int ko_closer(const ko_entry* a, const ko_entry* b);
int ko_knn_insert(ko_entry* row, size_t* fill, size_t k, const ko_entry* cand);
/* merge_rows core.cpp:114-134: returns count written to out (<= k). */
size_t ko_merge_rows(const ko_entry* a, size_t na, const ko_entry* b, size_t nb,
                     size_t k, ko_entry* out);
/* flat-array variant used by the Python tests: ids/dists row pairs. */
size_t ko_merge_rows_flat(const uint32_t* a_ids, const float* a_d, size_t na,
                          const uint32_t* b_ids, const float* b_d, size_t nb,
                          size_t k, uint32_t* o_ids, float* o_d);
/* check_graph_invariants core.cpp:166-186: 0 = ok, else a violation code. */
int ko_check_graph_invariants(const uint32_t* ids, const float* dists, size_t n,
                              size_t k, int local_space);

/* ---- evalio.cpp:242-272 ------------------------------------------------- */
/* dist: 0 uniform, 1 gaussian, 2 clustered. Returns 0 or -1 on invalid args. */
int ko_gen_random_dataset(size_t n, size_t dims, int dist, uint64_t seed,
                          size_t clusters, float* out);

/* ---- nndescent.cpp ------------------------------------------------------ */
int ko_init_random_graph(const ko_dataset* ds, size_t k, uint64_t seed,
                         uint32_t* ids, float* dists, uint8_t* flags);

/* sample_neighbors nndescent.cpp:64-129.  Outputs (caller-allocated):
 *   new_fwd [n*bound], old_fwd [n*k], new_rev [n*bound], old_rev [n*bound]
 * with per-point counts.  Flags are consumed in place.  Returns bound. */
size_t ko_sample_neighbors(uint32_t* ids, uint8_t* flags, size_t n, size_t k,
                           double rho, uint64_t seed, size_t iter,
                           uint32_t* new_fwd, uint32_t* new_fwd_n,
                           uint32_t* old_fwd, uint32_t* old_fwd_n,
                           uint32_t* new_rev, uint32_t* new_rev_n,
                           uint32_t* old_rev, uint32_t* old_rev_n);

typedef struct {
  size_t k;
  double delta;
  double rho;
  size_t max_iters;
  size_t candidate_capacity;
  uint64_t seed;
} ko_nnd_params;

/* nn_descent nndescent.cpp:225-259 at workers=1.  accepted_per_iter may be
 * NULL; otherwise it must hold max_iters entries.  Returns iterations or -1
 * on invalid arguments. */
long ko_nn_descent(const ko_dataset* ds, const ko_nnd_params* p, uint32_t* ids,
                   float* dists, uint8_t* flags, uint64_t* accepted_per_iter);

/* ---- graphopt.cpp:24-105 ----------------------------------------------- */
int ko_optimize_graph(const uint32_t* ids, const float* dists, size_t n, size_t k,
                      const ko_dataset* ds, size_t out_degree, uint32_t* sg_ids);

/* ---- annsearch.cpp:50-129 ---------------------------------------------- */
typedef struct {
  size_t k_s;
  size_t beam_width;
  size_t num_entry_points;
  size_t max_hops;
  uint64_t seed;
} ko_search_params;

/* hops / scored may be NULL (per-query diagnostics, annsearch.hpp:37-41). */
int ko_ann_search(const ko_dataset* q, const uint32_t* sg_ids, size_t sg_n,
                  size_t deg, const ko_dataset* v, const ko_search_params* p,
                  uint32_t* out_ids, float* out_dists, uint32_t* hops,
                  uint32_t* scored);

/* ---- refine.cpp ---------------------------------------------------------- */
int ko_partition(size_t n, size_t ranks, uint64_t seed, uint32_t* to_external,
                 uint64_t* offsets);
long ko_tree_levels(size_t ranks, size_t groups);
/* partners written to out (2^level entries); returns group_lo or -1. */
long ko_tree_schedule(size_t ranks, size_t groups, size_t rank, size_t level,
                      size_t* group_hi, size_t* partners);

typedef struct {
  size_t ranks;
  size_t groups;
  size_t k;
  size_t k_s;
  size_t out_degree;
  ko_nnd_params nn;
  ko_search_params search;
  int skip_tree_phase;
  size_t max_concat_bytes;
  uint64_t seed;
} ko_refine_config;

/* build_distributed refine.cpp:504-586 with the P ranks executed in lockstep
 * (every rank's work between two barriers reads only the snapshot published
 * before the first of them, exactly the RankWorld epoch rule
 * distsim.hpp:36-44).  Output: N x k graph in external ids / order. */
int ko_build_distributed(const ko_dataset* ds, const ko_refine_config* cfg,
                         uint32_t* ids, float* dists);

/* Refine only, from given per-rank local graphs (internal global ids,
 * rows of rank r at offsets[r]).  mode: 0 = tree+merge+flat (the
 * build_distributed body after local build), 1 = all_to_all_refine
 * refine.cpp:473-502.  Graph rows are updated in place (internal ids). */
int ko_refine_from_local(const ko_dataset* ds, const ko_refine_config* cfg,
                         const uint32_t* to_external, const uint64_t* offsets,
                         uint32_t* ids, float* dists, int mode);

/* translate_to_external refine.cpp:395-416 */
void ko_translate_to_external(const uint32_t* to_external, size_t n, size_t k,
                              const uint32_t* in_ids, const float* in_d,
                              uint32_t* out_ids, float* out_d);

/* ---- evalio.cpp:125-192 ------------------------------------------------ */
/* Exact k-NN of rows[0..q) of ds against all of ds (self excluded). */
int ko_brute_force_rows(const ko_dataset* ds, const uint64_t* rows, size_t q,
                        size_t k, uint32_t* ids, float* dists);
double ko_recall_rows(const uint32_t* test_ids, size_t test_k,
                      const uint32_t* truth_ids, size_t truth_k, size_t q,
                      size_t k_eval);

#ifdef __cplusplus
}
#endif
#endif
