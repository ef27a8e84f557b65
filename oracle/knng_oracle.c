/*
 * knng_oracle.c -- TEST INFRASTRUCTURE ONLY (see knng_oracle.h).
 *
 * CPU restatement of /root/reference/proj (C++20) in plain C, workers = 1.
 * Compile with -ffp-contract=off and without -ffast-math so every float op
 * rounds exactly as the reference's SSE code (subss/mulss/addss/sqrtss, no
 * FMA).
 */
#include "knng_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================== */
/* rng.hpp:12-96                                                             */
/* ======================================================================== */

void ko_rng_init(ko_rng* r, uint64_t seed) {
  r->state = seed;
  r->spare = 0.0f;
  r->have_spare = 0;
}

/* Rng::next_u64 rng.hpp:16-21 */
uint64_t ko_next_u64(ko_rng* r) {
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* Rng::next_below rng.hpp:24-27 (128-bit multiply-high) */
uint64_t ko_next_below(ko_rng* r, uint64_t bound) {
  return (uint64_t)(((unsigned __int128)ko_next_u64(r) * bound) >> 64);
}

/* Rng::next_float rng.hpp:30-32 */
float ko_next_float(ko_rng* r) {
  return (float)(ko_next_u64(r) >> 40) * 0x1.0p-24f;
}

/* Rng::next_gaussian rng.hpp:35-50 (Box-Muller, spare cached) */
float ko_next_gaussian(ko_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  float u1;
  do {
    u1 = ko_next_float(r);
  } while (u1 <= 0.0f);
  const float u2 = ko_next_float(r);
  const float rad = sqrtf(-2.0f * logf(u1));
  const float a = 6.28318530717958647692f * u2;
  r->spare = rad * sinf(a);
  r->have_spare = 1;
  return rad * cosf(a);
}

/* mix_seed rng.hpp:60-63 */
uint64_t ko_mix_seed(uint64_t a, uint64_t b) {
  ko_rng r;
  ko_rng_init(&r, a ^ (b * 0x9e3779b97f4a7c15ULL + 0xd1b54a32d192ed03ULL));
  return ko_next_u64(&r);
}

/* sample_distinct rng.hpp:66-87 */
size_t ko_sample_distinct(uint64_t n, size_t m, ko_rng* r, uint32_t* out) {
  if (m >= n) {
    for (size_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
    return (size_t)n;
  }
  size_t cnt = 0;
  while (cnt < m) {
    const uint32_t v = (uint32_t)ko_next_below(r, n);
    int dup = 0;
    for (size_t i = 0; i < cnt; ++i) {
      if (out[i] == v) {
        dup = 1;
        break;
      }
    }
    if (!dup) out[cnt++] = v;
  }
  return cnt;
}

/* shuffle rng.hpp:90-96 */
void ko_shuffle_u32(uint32_t* v, size_t n, ko_rng* r) {
  for (size_t i = n; i > 1; --i) {
    const size_t j = (size_t)ko_next_below(r, i);
    const uint32_t t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

/* ======================================================================== */
/* core.hpp:23-55, 84-123                                                    */
/* ======================================================================== */

float ko_l2_f32(const float* a, const float* b, size_t d) {
  float acc = 0.0f;
  for (size_t i = 0; i < d; ++i) {
    const float t = a[i] - b[i];
    acc += t * t;
  }
  return sqrtf(acc);
}

float ko_l2_u8(const uint8_t* a, const uint8_t* b, size_t d) {
  float acc = 0.0f;
  for (size_t i = 0; i < d; ++i) {
    const float t = (float)a[i] - (float)b[i];
    acc += t * t;
  }
  return sqrtf(acc);
}

#define KO_COSINE_BODY(T)                                   \
  float dot = 0.0f, na = 0.0f, nb = 0.0f;                   \
  for (size_t i = 0; i < d; ++i) {                          \
    const float x = (float)a[i];                            \
    const float y = (float)b[i];                            \
    dot += x * y;                                           \
    na += x * x;                                            \
    nb += y * y;                                            \
  }                                                         \
  if (na == 0.0f || nb == 0.0f) return 1.0f;                \
  const float v = 1.0f - dot / (sqrtf(na) * sqrtf(nb));     \
  return v < 0.0f ? 0.0f : v;

float ko_cosine_f32(const float* a, const float* b, size_t d) { KO_COSINE_BODY(float) }
float ko_cosine_u8(const uint8_t* a, const uint8_t* b, size_t d) { KO_COSINE_BODY(uint8_t) }

float ko_cross_distance(const ko_dataset* a, size_t i, const ko_dataset* b, size_t j) {
  const size_t d = a->dims;
  if (a->elem == 0) {
    const float* x = (const float*)a->data + i * d;
    const float* y = (const float*)b->data + j * d;
    return a->metric == 0 ? ko_l2_f32(x, y, d) : ko_cosine_f32(x, y, d);
  }
  const uint8_t* x = (const uint8_t*)a->data + i * d;
  const uint8_t* y = (const uint8_t*)b->data + j * d;
  return a->metric == 0 ? ko_l2_u8(x, y, d) : ko_cosine_u8(x, y, d);
}

float ko_row_distance(const ko_dataset* ds, size_t i, size_t j) {
  return ko_cross_distance(ds, i, ds, j);
}

/* ======================================================================== */
/* core.hpp:136-139, core.cpp:99-134, 166-186                                */
/* ======================================================================== */

int ko_closer(const ko_entry* a, const ko_entry* b) {
  if (a->dist != b->dist) return a->dist < b->dist;
  return a->id < b->id;
}

int ko_knn_insert(ko_entry* row, size_t* fill, size_t k, const ko_entry* cand) {
  for (size_t i = 0; i < *fill; ++i)
    if (row[i].id == cand->id) return 0;
  if (*fill >= k && !ko_closer(cand, &row[k - 1])) return 0;
  size_t pos = *fill < k ? *fill : k - 1;
  while (pos > 0 && ko_closer(cand, &row[pos - 1])) --pos;
  const size_t last = *fill < k ? *fill : k - 1;
  for (size_t i = last; i > pos; --i) row[i] = row[i - 1];
  row[pos] = *cand;
  if (*fill < k) ++*fill;
  return 1;
}

size_t ko_merge_rows(const ko_entry* a, size_t na, const ko_entry* b, size_t nb,
                     size_t k, ko_entry* out) {
  size_t i = 0, j = 0, cnt = 0;
  while (cnt < k && (i < na || j < nb)) {
    const ko_entry* e;
    if (j >= nb || (i < na && ko_closer(&a[i], &b[j])))
      e = &a[i++];
    else
      e = &b[j++];
    int dup = 0;
    for (size_t o = 0; o < cnt; ++o) {
      if (out[o].id == e->id) {
        dup = 1;
        break;
      }
    }
    if (!dup) out[cnt++] = *e;
  }
  return cnt;
}

size_t ko_merge_rows_flat(const uint32_t* a_ids, const float* a_d, size_t na,
                          const uint32_t* b_ids, const float* b_d, size_t nb,
                          size_t k, uint32_t* o_ids, float* o_d) {
  ko_entry* a = (ko_entry*)malloc(sizeof(ko_entry) * (na + 1));
  ko_entry* b = (ko_entry*)malloc(sizeof(ko_entry) * (nb + 1));
  ko_entry* o = (ko_entry*)malloc(sizeof(ko_entry) * (k + 1));
  for (size_t i = 0; i < na; ++i) a[i] = (ko_entry){a_ids[i], a_d[i], 0};
  for (size_t i = 0; i < nb; ++i) b[i] = (ko_entry){b_ids[i], b_d[i], 0};
  const size_t c = ko_merge_rows(a, na, b, nb, k, o);
  for (size_t i = 0; i < c; ++i) {
    o_ids[i] = o[i].id;
    o_d[i] = o[i].dist;
  }
  free(a);
  free(b);
  free(o);
  return c;
}

int ko_check_graph_invariants(const uint32_t* ids, const float* ds, size_t n,
                              size_t k, int local_space) {
  for (size_t r = 0; r < n; ++r) {
    const uint32_t* ir = ids + r * k;
    const float* dr = ds + r * k;
    for (size_t j = 0; j < k; ++j) {
      if (dr[j] < 0.0f) return 1;
      if (local_space && ir[j] == r) return 2;
      if (j > 0) {
        const int ordered = dr[j - 1] < dr[j] || (dr[j - 1] == dr[j] && ir[j - 1] < ir[j]);
        if (!ordered) return 3;
      }
      for (size_t m = j + 1; m < k; ++m)
        if (ir[j] == ir[m]) return 4;
    }
  }
  return 0;
}

static int entry_cmp(const void* x, const void* y) {
  const ko_entry* a = (const ko_entry*)x;
  const ko_entry* b = (const ko_entry*)y;
  if (ko_closer(a, b)) return -1;
  if (ko_closer(b, a)) return 1;
  return 0;
}

/* ======================================================================== */
/* evalio.cpp:242-272                                                        */
/* ======================================================================== */

int ko_gen_random_dataset(size_t n, size_t dims, int dist, uint64_t seed,
                          size_t clusters, float* out) {
  if (n == 0 || dims == 0) return -1;
  ko_rng rng;
  ko_rng_init(&rng, ko_mix_seed(seed, 0xda7a5e7ULL));
  const size_t total = n * dims;
  if (dist == 0) {
    for (size_t i = 0; i < total; ++i) out[i] = ko_next_float(&rng);
  } else if (dist == 1) {
    for (size_t i = 0; i < total; ++i) out[i] = ko_next_gaussian(&rng);
  } else {
    if (clusters == 0) return -1;
    float* centers = (float*)malloc(sizeof(float) * clusters * dims);
    for (size_t i = 0; i < clusters * dims; ++i) centers[i] = 5.0f * ko_next_gaussian(&rng);
    for (size_t i = 0; i < n; ++i) {
      const size_t c = i % clusters;
      for (size_t j = 0; j < dims; ++j)
        out[i * dims + j] = centers[c * dims + j] + ko_next_gaussian(&rng);
    }
    free(centers);
  }
  return 0;
}

/* ======================================================================== */
/* nndescent.cpp                                                             */
/* ======================================================================== */

/* init_random_graph nndescent.cpp:29-62 */
int ko_init_random_graph(const ko_dataset* ds, size_t k, uint64_t seed,
                         uint32_t* ids, float* dists, uint8_t* flags) {
  const size_t n = ds->n;
  if (k == 0 || k >= n) return -1;
  ko_entry* row = (ko_entry*)malloc(sizeof(ko_entry) * k);
  for (size_t r = 0; r < n; ++r) {
    ko_rng rng;
    ko_rng_init(&rng, ko_mix_seed(seed, r));
    size_t fill = 0;
    while (fill < k) {
      uint32_t id = (uint32_t)ko_next_below(&rng, n - 1);
      if (id >= r) ++id;
      int dup = 0;
      for (size_t j = 0; j < fill; ++j)
        if (row[j].id == id) {
          dup = 1;
          break;
        }
      if (dup) continue;
      row[fill].id = id;
      row[fill].dist = ko_row_distance(ds, r, id);
      row[fill].flag = 1;
      ++fill;
    }
    qsort(row, k, sizeof(ko_entry), entry_cmp);
    for (size_t j = 0; j < k; ++j) {
      ids[r * k + j] = row[j].id;
      dists[r * k + j] = row[j].dist;
      flags[r * k + j] = 1;
    }
  }
  free(row);
  return 0;
}

/* sample_neighbors nndescent.cpp:64-129 */
size_t ko_sample_neighbors(uint32_t* ids, uint8_t* flags, size_t n, size_t k,
                           double rho, uint64_t seed, size_t iter,
                           uint32_t* new_fwd, uint32_t* new_fwd_n,
                           uint32_t* old_fwd, uint32_t* old_fwd_n,
                           uint32_t* new_rev, uint32_t* new_rev_n,
                           uint32_t* old_rev, uint32_t* old_rev_n) {
  const size_t bound = (size_t)ceil(rho * (double)k);
  const uint64_t iter_seed = ko_mix_seed(seed, 0x5a3f1e00ULL + iter);
  uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * (k + 1));
  uint32_t* picks = (uint32_t*)malloc(sizeof(uint32_t) * (k + 1));
  /* forward pass :80-104 */
  for (size_t p = 0; p < n; ++p) {
    size_t np = 0, no = 0;
    for (size_t j = 0; j < k; ++j) {
      if (flags[p * k + j])
        pos[np++] = (uint32_t)j;
      else
        old_fwd[p * k + no++] = ids[p * k + j];
    }
    old_fwd_n[p] = (uint32_t)no;
    size_t take = np;
    if (np > bound) {
      ko_rng rng;
      ko_rng_init(&rng, ko_mix_seed(iter_seed, p));
      take = ko_sample_distinct(np, bound, &rng, picks);
      for (size_t i = 0; i < take; ++i) picks[i] = pos[picks[i]];
    } else {
      for (size_t i = 0; i < np; ++i) picks[i] = pos[i];
    }
    for (size_t i = 0; i < take; ++i) {
      new_fwd[p * bound + i] = ids[p * k + picks[i]];
      flags[p * k + picks[i]] = 0;
    }
    new_fwd_n[p] = (uint32_t)take;
  }
  /* serial transpose :108-113 -> CSR in ascending p order */
  size_t* cn = (size_t*)calloc(n + 1, sizeof(size_t));
  size_t* co = (size_t*)calloc(n + 1, sizeof(size_t));
  for (size_t p = 0; p < n; ++p) {
    for (size_t i = 0; i < new_fwd_n[p]; ++i) cn[new_fwd[p * bound + i] + 1]++;
    for (size_t i = 0; i < old_fwd_n[p]; ++i) co[old_fwd[p * k + i] + 1]++;
  }
  for (size_t v = 0; v < n; ++v) {
    cn[v + 1] += cn[v];
    co[v + 1] += co[v];
  }
  uint32_t* rn = (uint32_t*)malloc(sizeof(uint32_t) * (cn[n] + 1));
  uint32_t* ro = (uint32_t*)malloc(sizeof(uint32_t) * (co[n] + 1));
  size_t* wn = (size_t*)malloc(sizeof(size_t) * (n + 1));
  size_t* wo = (size_t*)malloc(sizeof(size_t) * (n + 1));
  memcpy(wn, cn, sizeof(size_t) * (n + 1));
  memcpy(wo, co, sizeof(size_t) * (n + 1));
  for (size_t p = 0; p < n; ++p) {
    for (size_t i = 0; i < new_fwd_n[p]; ++i) rn[wn[new_fwd[p * bound + i]]++] = (uint32_t)p;
    for (size_t i = 0; i < old_fwd_n[p]; ++i) ro[wo[old_fwd[p * k + i]]++] = (uint32_t)p;
  }
  /* reverse sampling :114-127, one rng shared by new_rev then old_rev */
  uint32_t* sp = (uint32_t*)malloc(sizeof(uint32_t) * (bound + 1));
  for (size_t p = 0; p < n; ++p) {
    ko_rng rng;
    ko_rng_init(&rng, ko_mix_seed(iter_seed, 0x8000000000000000ULL | (uint64_t)p));
    for (int which = 0; which < 2; ++which) {
      const uint32_t* list = which == 0 ? rn + cn[p] : ro + co[p];
      const size_t len = which == 0 ? cn[p + 1] - cn[p] : co[p + 1] - co[p];
      uint32_t* dst = which == 0 ? new_rev + p * bound : old_rev + p * bound;
      uint32_t* dn = which == 0 ? new_rev_n : old_rev_n;
      if (len > bound) {
        const size_t t = ko_sample_distinct(len, bound, &rng, sp);
        for (size_t i = 0; i < t; ++i) dst[i] = list[sp[i]];
        dn[p] = (uint32_t)t;
      } else {
        for (size_t i = 0; i < len; ++i) dst[i] = list[i];
        dn[p] = (uint32_t)len;
      }
    }
  }
  free(sp);
  free(rn);
  free(ro);
  free(wn);
  free(wo);
  free(cn);
  free(co);
  free(pos);
  free(picks);
  return bound;
}

static int list_has(const uint32_t* v, size_t n, uint32_t x) {
  for (size_t i = 0; i < n; ++i)
    if (v[i] == x) return 1;
  return 0;
}

/* build_join_lists nndescent.cpp:135-153 */
static void build_join_lists(size_t p, size_t bound, size_t k, const uint32_t* nf,
                             const uint32_t* nfn, const uint32_t* of, const uint32_t* ofn,
                             const uint32_t* nr, const uint32_t* nrn, const uint32_t* orv,
                             const uint32_t* orn, uint32_t* nl, size_t* nln, uint32_t* ol,
                             size_t* oln) {
  size_t a = 0, b = 0;
  for (size_t i = 0; i < nfn[p]; ++i)
    if (!list_has(nl, a, nf[p * bound + i])) nl[a++] = nf[p * bound + i];
  for (size_t i = 0; i < nrn[p]; ++i)
    if (!list_has(nl, a, nr[p * bound + i])) nl[a++] = nr[p * bound + i];
  for (size_t i = 0; i < ofn[p]; ++i) {
    const uint32_t id = of[p * k + i];
    if (!list_has(nl, a, id) && !list_has(ol, b, id)) ol[b++] = id;
  }
  for (size_t i = 0; i < orn[p]; ++i) {
    const uint32_t id = orv[p * bound + i];
    if (!list_has(nl, a, id) && !list_has(ol, b, id)) ol[b++] = id;
  }
  *nln = a;
  *oln = b;
}

typedef struct {
  size_t cap;
  ko_entry* slots;
  uint32_t* counts;
  float* worst;
} ko_cbuf;

/* CandidateBuffer::try_append nndescent.hpp:39-46 */
static void try_append(ko_cbuf* cb, uint32_t point, uint32_t id, float d) {
  if (d >= cb->worst[point]) return;
  const uint32_t slot = cb->counts[point]++;
  if (slot >= cb->cap) return;
  cb->slots[point * cb->cap + slot] = (ko_entry){id, d, 1};
}

/* nn_descent nndescent.cpp:225-259 (local_join :157-197, apply :199-223) */
long ko_nn_descent(const ko_dataset* ds, const ko_nnd_params* p, uint32_t* ids,
                   float* dists, uint8_t* flags, uint64_t* accepted_per_iter) {
  if (p->rho <= 0.0 || p->rho > 1.0) return -1;
  if (p->delta < 0.0) return -1;
  const size_t k = p->k;
  const size_t n = ds->n;
  const size_t cap = p->candidate_capacity ? p->candidate_capacity : 2 * k;
  if (cap < k) return -1;
  if (ko_init_random_graph(ds, k, p->seed, ids, dists, flags) != 0) return -1;
  ko_cbuf cb;
  cb.cap = cap;
  cb.slots = (ko_entry*)malloc(sizeof(ko_entry) * n * cap);
  cb.counts = (uint32_t*)calloc(n, sizeof(uint32_t));
  cb.worst = (float*)malloc(sizeof(float) * n);
  for (size_t i = 0; i < n; ++i) cb.worst[i] = dists[i * k + k - 1];
  const size_t bound = (size_t)ceil(p->rho * (double)k);
  uint32_t* nf = (uint32_t*)malloc(sizeof(uint32_t) * n * bound);
  uint32_t* of = (uint32_t*)malloc(sizeof(uint32_t) * n * k);
  uint32_t* nr = (uint32_t*)malloc(sizeof(uint32_t) * n * bound);
  uint32_t* orv = (uint32_t*)malloc(sizeof(uint32_t) * n * bound);
  uint32_t* nfn = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* ofn = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* nrn = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* orn = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* nl = (uint32_t*)malloc(sizeof(uint32_t) * (2 * bound + 1));
  uint32_t* ol = (uint32_t*)malloc(sizeof(uint32_t) * (k + bound + 1));
  ko_entry* row = (ko_entry*)malloc(sizeof(ko_entry) * k);
  const double threshold = p->delta * (double)k * (double)n;
  long iters = 0;
  for (size_t iter = 0; iter < p->max_iters; ++iter) {
    ko_sample_neighbors(ids, flags, n, k, p->rho, p->seed, iter, nf, nfn, of, ofn, nr,
                        nrn, orv, orn);
    /* local_join, serial p order */
    for (size_t q = 0; q < n; ++q) {
      size_t a, b;
      build_join_lists(q, bound, k, nf, nfn, of, ofn, nr, nrn, orv, orn, nl, &a, ol, &b);
      for (size_t i = 0; i < a; ++i) {
        for (size_t j = i + 1; j < a; ++j) {
          const float d = ko_row_distance(ds, nl[i], nl[j]);
          try_append(&cb, nl[i], nl[j], d);
          try_append(&cb, nl[j], nl[i], d);
        }
        for (size_t j = 0; j < b; ++j) {
          if (ol[j] == nl[i]) continue;
          const float d = ko_row_distance(ds, nl[i], ol[j]);
          try_append(&cb, nl[i], ol[j], d);
          try_append(&cb, ol[j], nl[i], d);
        }
      }
    }
    /* apply_candidates */
    uint64_t accepted = 0;
    for (size_t q = 0; q < n; ++q) {
      const size_t m = cb.counts[q] < cap ? cb.counts[q] : cap;
      if (m == 0) continue;
      for (size_t j = 0; j < k; ++j)
        row[j] = (ko_entry){ids[q * k + j], dists[q * k + j], flags[q * k + j]};
      size_t fill = k;
      for (size_t c = 0; c < m; ++c)
        if (ko_knn_insert(row, &fill, k, &cb.slots[q * cap + c])) ++accepted;
      for (size_t j = 0; j < k; ++j) {
        ids[q * k + j] = row[j].id;
        dists[q * k + j] = row[j].dist;
        flags[q * k + j] = row[j].flag;
      }
      cb.worst[q] = row[k - 1].dist;
      cb.counts[q] = 0;
    }
    if (accepted_per_iter) accepted_per_iter[iter] = accepted;
    iters = (long)iter + 1;
    if ((double)accepted < threshold) break;
  }
  free(cb.slots);
  free(cb.counts);
  free(cb.worst);
  free(nf);
  free(of);
  free(nr);
  free(orv);
  free(nfn);
  free(ofn);
  free(nrn);
  free(orn);
  free(nl);
  free(ol);
  free(row);
  return iters;
}

/* ======================================================================== */
/* graphopt.cpp:24-105                                                       */
/* ======================================================================== */

typedef struct {
  uint32_t id;
  float dist;
} ko_redge;

static int redge_cmp(const void* x, const void* y) {
  const ko_redge* a = (const ko_redge*)x;
  const ko_redge* b = (const ko_redge*)y;
  if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
  return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

int ko_optimize_graph(const uint32_t* ids, const float* dists, size_t n, size_t k,
                      const ko_dataset* ds, size_t out_degree, uint32_t* sg_ids) {
  if (out_degree == 0) out_degree = k;
  if (out_degree > k) return -1;
  if (n != ds->n) return -1;
  uint8_t* kept = (uint8_t*)calloc(n * k + 1, 1);
  uint32_t* kept_ids = (uint32_t*)malloc(sizeof(uint32_t) * (k + 1));
  /* pass 1 :35-58 */
  for (size_t u = 0; u < n; ++u) {
    size_t nk = 0;
    for (size_t j = 0; j < k; ++j) {
      const uint32_t w = ids[u * k + j];
      int detour = 0;
      for (size_t t = 0; t < nk; ++t) {
        if (ko_row_distance(ds, kept_ids[t], w) < dists[u * k + j]) {
          detour = 1;
          break;
        }
      }
      if (!detour) {
        kept[u * k + j] = 1;
        kept_ids[nk++] = w;
      }
    }
  }
  /* reverse aggregation :60-69 (serial, ascending u) */
  size_t* off = (size_t*)calloc(n + 1, sizeof(size_t));
  for (size_t u = 0; u < n; ++u)
    for (size_t j = 0; j < k; ++j)
      if (kept[u * k + j]) off[ids[u * k + j] + 1]++;
  for (size_t v = 0; v < n; ++v) off[v + 1] += off[v];
  ko_redge* rev = (ko_redge*)malloc(sizeof(ko_redge) * (off[n] + 1));
  size_t* w = (size_t*)malloc(sizeof(size_t) * (n + 1));
  memcpy(w, off, sizeof(size_t) * (n + 1));
  for (size_t u = 0; u < n; ++u)
    for (size_t j = 0; j < k; ++j)
      if (kept[u * k + j]) rev[w[ids[u * k + j]]++] = (ko_redge){(uint32_t)u, dists[u * k + j]};
  /* pass 2 :77-103 */
  uint32_t* row = (uint32_t*)malloc(sizeof(uint32_t) * (out_degree + 1));
  for (size_t u = 0; u < n; ++u) {
    size_t cnt = 0;
    const uint32_t* ir = ids + u * k;
    for (size_t j = 0; j < k && cnt < out_degree; ++j)
      if (kept[u * k + j]) row[cnt++] = ir[j];
    if (cnt < out_degree) {
      const size_t len = off[u + 1] - off[u];
      qsort(rev + off[u], len, sizeof(ko_redge), redge_cmp);
      for (size_t t = 0; t < len; ++t) {
        if (cnt >= out_degree) break;
        const uint32_t c = rev[off[u] + t].id;
        if (c != u && !list_has(row, cnt, c)) row[cnt++] = c;
      }
    }
    for (size_t j = 0; j < k && cnt < out_degree; ++j)
      if (!kept[u * k + j] && !list_has(row, cnt, ir[j])) row[cnt++] = ir[j];
    memcpy(sg_ids + u * out_degree, row, sizeof(uint32_t) * out_degree);
  }
  free(row);
  free(w);
  free(rev);
  free(off);
  free(kept_ids);
  free(kept);
  return 0;
}

/* ======================================================================== */
/* annsearch.cpp:50-129                                                      */
/* ======================================================================== */

typedef struct {
  uint32_t id;
  float dist;
  int expanded;
} ko_beam;

static int beam_closer(const ko_beam* a, const ko_beam* b) {
  if (a->dist != b->dist) return a->dist < b->dist;
  return a->id < b->id;
}

/* beam_insert annsearch.cpp:26-31 */
static void beam_insert(ko_beam* beam, size_t* size, size_t width, ko_beam e) {
  if (*size == width && !beam_closer(&e, &beam[*size - 1])) return;
  /* upper_bound: first element with e < elem */
  size_t pos = 0;
  while (pos < *size && !beam_closer(&e, &beam[pos])) ++pos;
  for (size_t i = *size; i > pos; --i) beam[i] = beam[i - 1];
  beam[pos] = e;
  ++*size;
  if (*size > width) --*size;
}

int ko_ann_search(const ko_dataset* q, const uint32_t* sg_ids, size_t sg_n,
                  size_t deg, const ko_dataset* v, const ko_search_params* p,
                  uint32_t* out_ids, float* out_dists, uint32_t* hops_out,
                  uint32_t* scored_out) {
  if (q->dims != v->dims || q->elem != v->elem || q->metric != v->metric) return -1;
  if (sg_n != v->n) return -1;
  if (p->k_s == 0 || p->k_s > v->n) return -1;
  if (p->k_s > p->beam_width) return -1;
  const size_t nq = q->n;
  const size_t n = v->n;
  const size_t width = p->beam_width;
  const size_t max_hops = p->max_hops ? p->max_hops : p->beam_width * 4;
  size_t entries = p->num_entry_points > p->k_s ? p->num_entry_points : p->k_s;
  if (entries > n) entries = n;
  memset(out_ids, 0, sizeof(uint32_t) * nq * p->k_s);
  memset(out_dists, 0, sizeof(float) * nq * p->k_s);
  uint32_t* stamp = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
  ko_beam* beam = (ko_beam*)malloc(sizeof(ko_beam) * (width + 2));
  uint32_t* starts = (uint32_t*)malloc(sizeof(uint32_t) * (entries + 1));
  uint32_t epoch = 0;
  for (size_t qi = 0; qi < nq; ++qi) {
    ++epoch;
    size_t bs = 0;
    uint32_t scored = 0;
    ko_rng rng;
    ko_rng_init(&rng, ko_mix_seed(p->seed, 0xa11ce000ULL + qi));
    const size_t ns = ko_sample_distinct(n, entries, &rng, starts);
    for (size_t s = 0; s < ns; ++s) {
      const uint32_t id = starts[s];
      stamp[id] = epoch;
      ko_beam e = {id, ko_cross_distance(q, qi, v, id), 0};
      ++scored;
      beam_insert(beam, &bs, width, e);
    }
    size_t hops = 0;
    while (hops < max_hops) {
      size_t idx = bs;
      for (size_t i = 0; i < bs; ++i)
        if (!beam[i].expanded) {
          idx = i;
          break;
        }
      if (idx == bs) break;
      beam[idx].expanded = 1;
      const uint32_t u = beam[idx].id;
      for (size_t t = 0; t < deg; ++t) {
        const uint32_t nb = sg_ids[u * deg + t];
        if (stamp[nb] == epoch) continue;
        stamp[nb] = epoch;
        ko_beam e = {nb, ko_cross_distance(q, qi, v, nb), 0};
        ++scored;
        beam_insert(beam, &bs, width, e);
      }
      ++hops;
    }
    if (hops_out) hops_out[qi] = (uint32_t)hops;
    if (scored_out) scored_out[qi] = scored;
    const size_t out = p->k_s < bs ? p->k_s : bs;
    for (size_t i = 0; i < out; ++i) {
      out_ids[qi * p->k_s + i] = beam[i].id;
      out_dists[qi * p->k_s + i] = beam[i].dist;
    }
  }
  free(stamp);
  free(beam);
  free(starts);
  return 0;
}

/* ======================================================================== */
/* refine.cpp                                                                */
/* ======================================================================== */

static int is_pow2(size_t v) { return v != 0 && (v & (v - 1)) == 0; }
static size_t log2_exact(size_t v) {
  size_t l = 0;
  while (((size_t)1 << l) < v) ++l;
  return l;
}

/* partition_dataset refine.cpp:86-126 (ids + offsets; rows gathered by caller) */
int ko_partition(size_t n, size_t ranks, uint64_t seed, uint32_t* to_external,
                 uint64_t* offsets) {
  if (ranks == 0 || ranks > n) return -1;
  for (size_t i = 0; i < n; ++i) to_external[i] = (uint32_t)i;
  if (ranks > 1) {
    ko_rng rng;
    ko_rng_init(&rng, ko_mix_seed(seed, 0x9a71710ULL));
    ko_shuffle_u32(to_external, n, &rng);
  }
  const size_t base = n / ranks, extra = n % ranks;
  offsets[0] = 0;
  for (size_t r = 0; r < ranks; ++r) offsets[r + 1] = offsets[r] + base + (r < extra ? 1 : 0);
  return 0;
}

/* tree_levels refine.cpp:128-132 */
long ko_tree_levels(size_t ranks, size_t groups) {
  if (!is_pow2(ranks) || !is_pow2(groups) || groups > ranks) return -1;
  return (long)log2_exact(ranks / groups);
}

/* tree_schedule refine.cpp:134-149 */
long ko_tree_schedule(size_t ranks, size_t groups, size_t rank, size_t level,
                      size_t* group_hi, size_t* partners) {
  const long levels = ko_tree_levels(ranks, groups);
  if (levels < 0 || rank >= ranks || (long)level >= levels) return -1;
  const size_t size = (size_t)1 << level;
  const size_t block = rank / size;
  const size_t lo = block * size;
  *group_hi = lo + size;
  const size_t plo = (block ^ 1U) * size;
  for (size_t i = 0; i < size; ++i) partners[i] = plo + i;
  return (long)lo;
}

/* translate_to_external refine.cpp:395-416 */
void ko_translate_to_external(const uint32_t* to_external, size_t n, size_t k,
                              const uint32_t* in_ids, const float* in_d,
                              uint32_t* out_ids, float* out_d) {
  ko_entry* row = (ko_entry*)malloc(sizeof(ko_entry) * (k + 1));
  for (size_t r = 0; r < n; ++r) {
    for (size_t j = 0; j < k; ++j)
      row[j] = (ko_entry){to_external[in_ids[r * k + j]], in_d[r * k + j], 0};
    qsort(row, k, sizeof(ko_entry), entry_cmp);
    const size_t dst = to_external[r];
    for (size_t j = 0; j < k; ++j) {
      out_ids[dst * k + j] = row[j].id;
      out_d[dst * k + j] = row[j].dist;
    }
  }
  free(row);
}

/* merge_results_into refine.cpp:49-60 over rows [0, nrows) of g */
static void merge_results_into(uint32_t* gids, float* gd, size_t nrows, size_t k,
                               const uint32_t* rids, const float* rd, size_t ks,
                               size_t id_base) {
  ko_entry* a = (ko_entry*)malloc(sizeof(ko_entry) * (k + 1));
  ko_entry* b = (ko_entry*)malloc(sizeof(ko_entry) * (ks + 1));
  ko_entry* o = (ko_entry*)malloc(sizeof(ko_entry) * (k + 1));
  for (size_t r = 0; r < nrows; ++r) {
    for (size_t j = 0; j < k; ++j) a[j] = (ko_entry){gids[r * k + j], gd[r * k + j], 0};
    for (size_t j = 0; j < ks; ++j)
      b[j] = (ko_entry){(uint32_t)(rids[r * ks + j] + id_base), rd[r * ks + j], 0};
    const size_t c = ko_merge_rows(a, k, b, ks, k, o);
    (void)c; /* always k: the graph row alone has k distinct ids */
    for (size_t j = 0; j < k; ++j) {
      gids[r * k + j] = o[j].id;
      gd[r * k + j] = o[j].dist;
    }
  }
  free(a);
  free(b);
  free(o);
}

typedef struct {
  size_t n;
  size_t dims;
  int elem;
  int metric;
  size_t esz;
} shape_t;

static ko_dataset view_rows(const ko_dataset* ds, size_t lo, size_t cnt) {
  const size_t esz = ds->elem == 0 ? 4 : 1;
  ko_dataset v = *ds;
  v.data = (const uint8_t*)ds->data + lo * ds->dims * esz;
  v.n = cnt;
  return v;
}

/* effective_groups refine.cpp:160-183 */
static size_t effective_groups(const uint64_t* offsets, size_t p, size_t dims,
                               size_t esz, const ko_refine_config* cfg, size_t od) {
  if (p == 1) return 1;
  int skip = cfg->skip_tree_phase;
  if (!skip && cfg->max_concat_bytes != 0) {
    const size_t gsz = p / cfg->groups;
    size_t span = 0;
    for (size_t g = 0; g < cfg->groups; ++g) {
      const size_t s = offsets[(g + 1) * gsz] - offsets[g * gsz];
      if (s > span) span = s;
    }
    const size_t est = span * (dims * esz + cfg->k * 8 + od * 4);
    if (est > cfg->max_concat_bytes) skip = 1;
  }
  return skip ? p : cfg->groups;
}

/* The refinement body of build_distributed refine.cpp:536-549 run in
 * lockstep.  `data_perm` holds all rows in internal-id (shuffled) order, so a
 * rank's dataset / a contiguous span of ranks is a row range of it (exactly
 * the rank-order concatenations at refine.cpp:201-206, 270-285, 323-330). */
static int refine_lockstep(const ko_dataset* data_perm, const ko_refine_config* cfg,
                           const uint64_t* offsets, uint32_t* gids, float* gd,
                           int mode) {
  const size_t p = cfg->ranks;
  const size_t k = cfg->k;
  const size_t od = cfg->out_degree ? cfg->out_degree : k;
  const size_t esz = data_perm->elem == 0 ? 4 : 1;
  ko_search_params sp = cfg->search;
  sp.k_s = cfg->k_s ? cfg->k_s : k;
  const size_t ks = sp.k_s;
  const size_t n = data_perm->n;
  size_t maxb = 0;
  for (size_t r = 0; r < p; ++r)
    if (offsets[r + 1] - offsets[r] > maxb) maxb = offsets[r + 1] - offsets[r];
  uint32_t* rid = (uint32_t*)malloc(sizeof(uint32_t) * maxb * ks + 4);
  float* rdd = (float*)malloc(sizeof(float) * maxb * ks + 4);
  uint32_t* sgall = (uint32_t*)malloc(sizeof(uint32_t) * n * od + 4);
  uint32_t* pub_ids = (uint32_t*)malloc(sizeof(uint32_t) * n * k + 4);
  float* pub_d = (float*)malloc(sizeof(float) * n * k + 4);
  uint32_t* tmp_ids = (uint32_t*)malloc(sizeof(uint32_t) * n * k + 4);

  if (mode == 1) {
    /* all_to_all_refine refine.cpp:473-502: each rank's own optimized graph */
    for (size_t i = 0; i < p; ++i) {
      const size_t lo = offsets[i], cnt = offsets[i + 1] - lo;
      for (size_t t = 0; t < cnt * k; ++t) tmp_ids[t] = gids[lo * k + t] - (uint32_t)lo;
      ko_dataset dv = view_rows(data_perm, lo, cnt);
      ko_optimize_graph(tmp_ids, gd + lo * k, cnt, k, &dv, od, sgall + lo * od);
    }
    for (size_t i = 0; i < p; ++i) {
      const size_t lo = offsets[i], cnt = offsets[i + 1] - lo;
      ko_dataset local = view_rows(data_perm, lo, cnt);
      for (size_t step = 1; step < p; ++step) {
        const size_t j = (i + step) % p;
        const size_t jlo = offsets[j], jcnt = offsets[j + 1] - jlo;
        ko_dataset vec = view_rows(data_perm, jlo, jcnt);
        ko_ann_search(&local, sgall + jlo * od, jcnt, od, &vec, &sp, rid, rdd, NULL, NULL);
        merge_results_into(gids + lo * k, gd + lo * k, cnt, k, rid, rdd, ks, jlo);
      }
    }
    goto done;
  }
  {
    const size_t groups = effective_groups(offsets, p, data_perm->dims, esz, cfg, od);
    const long levels = ko_tree_levels(p, groups);
    /* publish graph (epoch 0) + barrier */
    memcpy(pub_ids, gids, sizeof(uint32_t) * n * k);
    memcpy(pub_d, gd, sizeof(float) * n * k);
    size_t* partners = (size_t*)malloc(sizeof(size_t) * (p + 1));
    for (long level = 0; level < levels; ++level) {
      for (size_t i = 0; i < p; ++i) {
        size_t ghi;
        const long glo = ko_tree_schedule(p, groups, i, (size_t)level, &ghi, partners);
        (void)glo;
        const size_t size = (size_t)1 << level;
        const size_t base = offsets[partners[0]];
        const size_t cnt = offsets[partners[size - 1] + 1] - base;
        /* pulled graph rows of the partner block, shifted by -base */
        for (size_t t = 0; t < cnt * k; ++t) tmp_ids[t] = pub_ids[base * k + t] - (uint32_t)base;
        ko_dataset pulled = view_rows(data_perm, base, cnt);
        uint32_t* sg = sgall; /* scratch */
        ko_optimize_graph(tmp_ids, pub_d + base * k, cnt, k, &pulled, od, sg);
        const size_t lo = offsets[i], lcnt = offsets[i + 1] - lo;
        ko_dataset local = view_rows(data_perm, lo, lcnt);
        ko_ann_search(&local, sg, cnt, od, &pulled, &sp, rid, rdd, NULL, NULL);
        merge_results_into(gids + lo * k, gd + lo * k, lcnt, k, rid, rdd, ks, base);
      }
      /* publish (staged) + barrier: snapshot swaps in */
      memcpy(pub_ids, gids, sizeof(uint32_t) * n * k);
      memcpy(pub_d, gd, sizeof(float) * n * k);
    }
    free(partners);
    /* grouped merge refine.cpp:256-293; every member computes the same
     * search graph over its group span (byte-identical, test_refine.cpp:244) */
    const size_t gsz = p / groups;
    for (size_t g = 0; g < groups; ++g) {
      const size_t glo = offsets[g * gsz], ghi = offsets[(g + 1) * gsz];
      const size_t cnt = ghi - glo;
      for (size_t t = 0; t < cnt * k; ++t) tmp_ids[t] = pub_ids[glo * k + t] - (uint32_t)glo;
      ko_dataset span = view_rows(data_perm, glo, cnt);
      ko_optimize_graph(tmp_ids, pub_d + glo * k, cnt, k, &span, od, sgall + glo * od);
    }
    /* flat refine refine.cpp:300-351 */
    if (groups > 1) {
      for (size_t i = 0; i < p; ++i) {
        const size_t my_group = i / gsz;
        const size_t lo = offsets[i], lcnt = offsets[i + 1] - lo;
        ko_dataset local = view_rows(data_perm, lo, lcnt);
        for (size_t step = 1; step < groups; ++step) {
          const size_t grp = (my_group + step) % groups;
          const size_t glo = offsets[grp * gsz], cnt = offsets[(grp + 1) * gsz] - glo;
          ko_dataset vec = view_rows(data_perm, glo, cnt);
          ko_ann_search(&local, sgall + glo * od, cnt, od, &vec, &sp, rid, rdd, NULL, NULL);
          merge_results_into(gids + lo * k, gd + lo * k, lcnt, k, rid, rdd, ks, glo);
        }
      }
    }
  }
done:
  free(rid);
  free(rdd);
  free(sgall);
  free(pub_ids);
  free(pub_d);
  free(tmp_ids);
  return 0;
}

/* validate_config refine.cpp:359-378 */
static int validate_config(const uint64_t* offsets, const ko_refine_config* cfg) {
  const size_t p = cfg->ranks;
  if (!is_pow2(p)) return -1;
  if (p > 1 && (!is_pow2(cfg->groups) || cfg->groups < 2 || cfg->groups > p)) return -1;
  size_t minb = offsets[1] - offsets[0];
  for (size_t r = 1; r < p; ++r)
    if (offsets[r + 1] - offsets[r] < minb) minb = offsets[r + 1] - offsets[r];
  if (cfg->k >= minb) return -1;
  const size_t ks = cfg->k_s ? cfg->k_s : cfg->k;
  if (ks > minb) return -1;
  const size_t od = cfg->out_degree ? cfg->out_degree : cfg->k;
  if (od > cfg->k) return -1;
  return 0;
}

static void* gather_rows(const ko_dataset* ds, const uint32_t* to_external) {
  const size_t esz = ds->elem == 0 ? 4 : 1;
  const size_t rb = ds->dims * esz;
  uint8_t* out = (uint8_t*)malloc(ds->n * rb + 4);
  for (size_t i = 0; i < ds->n; ++i)
    memcpy(out + i * rb, (const uint8_t*)ds->data + (size_t)to_external[i] * rb, rb);
  return out;
}

int ko_refine_from_local(const ko_dataset* ds, const ko_refine_config* cfg,
                         const uint32_t* to_external, const uint64_t* offsets,
                         uint32_t* ids, float* dists, int mode) {
  if (validate_config(offsets, cfg) != 0) return -1;
  void* perm = gather_rows(ds, to_external);
  ko_dataset dp = *ds;
  dp.data = perm;
  const int rc = refine_lockstep(&dp, cfg, offsets, ids, dists, mode);
  free(perm);
  return rc;
}

int ko_build_distributed(const ko_dataset* ds, const ko_refine_config* cfg,
                         uint32_t* out_ids, float* out_d) {
  const size_t n = ds->n, p = cfg->ranks, k = cfg->k;
  if (p == 0 || p > n) return -1;
  uint32_t* to_ext = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint64_t* offsets = (uint64_t*)malloc(sizeof(uint64_t) * (p + 1));
  ko_partition(n, p, cfg->seed, to_ext, offsets);
  if (validate_config(offsets, cfg) != 0) {
    free(to_ext);
    free(offsets);
    return -1;
  }
  void* perm = gather_rows(ds, to_ext);
  ko_dataset dp = *ds;
  dp.data = perm;
  uint32_t* gids = (uint32_t*)malloc(sizeof(uint32_t) * n * k);
  float* gd = (float*)malloc(sizeof(float) * n * k);
  uint8_t* fl = (uint8_t*)malloc(n * k);
  /* local_build_rank refine.cpp:380-390 */
  int rc = 0;
  for (size_t r = 0; r < p; ++r) {
    const size_t lo = offsets[r], cnt = offsets[r + 1] - lo;
    ko_dataset local = view_rows(&dp, lo, cnt);
    ko_nnd_params np = cfg->nn;
    np.k = k;
    np.seed = p == 1 ? cfg->nn.seed : ko_mix_seed(cfg->nn.seed, r);
    if (ko_nn_descent(&local, &np, gids + lo * k, gd + lo * k, fl + lo * k, NULL) < 0) {
      rc = -1;
      break;
    }
    for (size_t t = 0; t < cnt * k; ++t) gids[lo * k + t] += (uint32_t)lo;
  }
  if (rc == 0 && p > 1) rc = refine_lockstep(&dp, cfg, offsets, gids, gd, 0);
  if (rc == 0) ko_translate_to_external(to_ext, n, k, gids, gd, out_ids, out_d);
  free(gids);
  free(gd);
  free(fl);
  free(perm);
  free(to_ext);
  free(offsets);
  return rc;
}

/* ======================================================================== */
/* evalio.cpp:125-192                                                        */
/* ======================================================================== */

int ko_brute_force_rows(const ko_dataset* ds, const uint64_t* rows, size_t q,
                        size_t k, uint32_t* ids, float* dists) {
  if (k >= ds->n) return -1;
  ko_entry* row = (ko_entry*)malloc(sizeof(ko_entry) * (k + 1));
  for (size_t t = 0; t < q; ++t) {
    const size_t r = (size_t)rows[t];
    size_t fill = 0;
    for (size_t j = 0; j < ds->n; ++j) {
      if (j == r) continue;
      ko_entry c = {(uint32_t)j, ko_row_distance(ds, r, j), 0};
      ko_knn_insert(row, &fill, k, &c);
    }
    for (size_t j = 0; j < k; ++j) {
      ids[t * k + j] = row[j].id;
      dists[t * k + j] = row[j].dist;
    }
  }
  free(row);
  return 0;
}

double ko_recall_rows(const uint32_t* test_ids, size_t test_k, const uint32_t* truth_ids,
                      size_t truth_k, size_t q, size_t k_eval) {
  size_t hits = 0;
  for (size_t r = 0; r < q; ++r) {
    const uint32_t* t = test_ids + r * test_k;
    const uint32_t* g = truth_ids + r * truth_k;
    for (size_t i = 0; i < k_eval; ++i)
      for (size_t j = 0; j < k_eval; ++j)
        if (t[i] == g[j]) {
          ++hits;
          break;
        }
  }
  return (double)hits / (double)(q * k_eval);
}
