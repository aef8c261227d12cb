/*
 * qvmc_oracle.c — CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * Restates, in plain C and in the reference's own order of operations:
 *   HamiltonianIndex::from_terms       proj/src/hamiltonian.cpp:63-117
 *   HamiltonianIndex::group_element    proj/src/hamiltonian.cpp:186-194
 *   HamiltonianIndex::matrix_element   proj/src/hamiltonian.cpp:178-184
 *   loop_over_terms / loop_over_batch  proj/src/coupling.cpp:62-102
 *   PerSource::flatten (canonical)     proj/src/coupling.cpp:37-58
 *   local_energies                     proj/src/energy.cpp:13-48
 *   variational_energy                 proj/src/energy.cpp:50-78
 * Pinned against the reference's KATs and against oracle/_ref by
 * tests/test_oracle.py. Only tests/, smoke() and bench.py's cpu_baseline may
 * use it; the product never does.
 */
#include "qvmc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* qo_last_error(void) { return g_err; }
void qo_free(void* p) { free(p); }

/* ---------------------------------------------------------------- hashing */

static uint64_t mix64(uint64_t h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdULL;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ULL;
  h ^= h >> 33;
  return h;
}

static uint64_t hash_words(const uint64_t* w, int n) {
  uint64_t h = 0x9e3779b97f4a7c15ULL;
  for (int i = 0; i < n; ++i) h = mix64(h ^ (w[i] + 0x9e3779b97f4a7c15ULL + (h << 6)));
  return h;
}

static int eq_words(const uint64_t* a, const uint64_t* b, int n) {
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return 0;
  return 1;
}

/* Open-addressing map from a word key (stored externally at
 * store[idx*kw]) to idx. */
typedef struct {
  int64_t cap; /* power of two */
  int64_t* slot;
  const uint64_t* const* store;
  int kw;
} wmap;

static int wmap_init(wmap* m, int64_t expect, const uint64_t* const* store, int kw) {
  int64_t cap = 16;
  while (cap < 2 * expect + 2) cap <<= 1;
  m->cap = cap;
  m->slot = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
  if (!m->slot) return -1;
  for (int64_t i = 0; i < cap; ++i) m->slot[i] = -1;
  m->store = store;
  m->kw = kw;
  return 0;
}

static void wmap_free(wmap* m) { free(m->slot); }

/* Returns existing idx for key, or -1 if absent. */
static int64_t wmap_find(const wmap* m, const uint64_t* key) {
  int64_t s = (int64_t)(hash_words(key, m->kw) & (uint64_t)(m->cap - 1));
  for (;;) {
    const int64_t v = m->slot[s];
    if (v < 0) return -1;
    if (eq_words(*m->store + v * m->kw, key, m->kw)) return v;
    s = (s + 1) & (m->cap - 1);
  }
}

/* Inserts idx (key read from the store); returns the existing idx if the key
 * is already present, else -1. */
static int64_t wmap_insert(wmap* m, int64_t idx) {
  const uint64_t* key = *m->store + idx * m->kw;
  int64_t s = (int64_t)(hash_words(key, m->kw) & (uint64_t)(m->cap - 1));
  for (;;) {
    const int64_t v = m->slot[s];
    if (v < 0) {
      m->slot[s] = idx;
      return -1;
    }
    if (eq_words(*m->store + v * m->kw, key, m->kw)) return v;
    s = (s + 1) & (m->cap - 1);
  }
}

static int and_popc(const uint64_t* a, const uint64_t* b, int n) {
  int c = 0;
  for (int i = 0; i < n; ++i) c += __builtin_popcountll(a[i] & b[i]);
  return c;
}

/* ------------------------------------------------------------ the index */

struct qo_index {
  int n_qubits, kw;
  int64_t n_terms, n_xy, diag;
  uint64_t* xy;     /* [n_xy][kw] first-occurrence order */
  int64_t* off;     /* [n_xy+1] */
  double* coeff;    /* [n_terms] grouped */
  uint64_t* yz;     /* [n_terms][kw] */
  uint8_t* yw;      /* [n_terms] */
  wmap xy_map;
  const uint64_t* xy_store;
};

void qo_index_free(qo_index* h) {
  if (!h) return;
  wmap_free(&h->xy_map);
  free(h->xy);
  free(h->off);
  free(h->coeff);
  free(h->yz);
  free(h->yw);
  free(h);
}

qo_index* qo_index_from_terms(int n_qubits, int kw, int64_t n_raw, const double* coeff, const uint64_t* xw,
                              const uint64_t* yw, const uint64_t* zw) {
  if (n_qubits < 1 || n_qubits > 256 || kw != (n_qubits + 63) / 64) {
    snprintf(g_err, sizeof g_err, "invalid_argument: qubit count out of range");
    return NULL;
  }
  const int tail = n_qubits % 64;
  const uint64_t tail_mask = tail ? ((1ULL << tail) - 1) : ~0ULL;
  for (int64_t t = 0; t < n_raw; ++t)
    for (int w = 0; w < kw; ++w) {
      const uint64_t a = xw[t * kw + w], b = yw[t * kw + w], c = zw[t * kw + w];
      if ((a & b) | (a & c) | (b & c)) {
        snprintf(g_err, sizeof g_err, "invalid_argument: term %lld has overlapping Pauli masks", (long long)t);
        return NULL;
      }
      if (w == kw - 1 && ((a | b | c) & ~tail_mask)) {
        snprintf(g_err, sizeof g_err, "invalid_argument: term %lld has bits beyond qubit count", (long long)t);
        return NULL;
      }
    }

  /* merge duplicate (x,y,z) strings, first-occurrence order (hamiltonian.cpp:68-85) */
  const int k3 = 3 * kw;
  uint64_t* mkey = (uint64_t*)malloc((size_t)(n_raw ? n_raw : 1) * k3 * sizeof(uint64_t));
  double* mcoef = (double*)malloc((size_t)(n_raw ? n_raw : 1) * sizeof(double));
  const uint64_t* store = mkey;
  wmap seen;
  wmap_init(&seen, n_raw, &store, k3);
  int64_t n_merged = 0;
  for (int64_t t = 0; t < n_raw; ++t) {
    uint64_t* k = mkey + n_merged * k3;
    memcpy(k, xw + t * kw, kw * 8);
    memcpy(k + kw, yw + t * kw, kw * 8);
    memcpy(k + 2 * kw, zw + t * kw, kw * 8);
    const int64_t prev = wmap_insert(&seen, n_merged);
    if (prev < 0) {
      mcoef[n_merged] = coeff[t];
      ++n_merged;
    } else {
      mcoef[prev] += coeff[t];
    }
  }
  wmap_free(&seen);

  /* group survivors by xy = x|y in first-occurrence order (hamiltonian.cpp:88-112) */
  qo_index* h = (qo_index*)calloc(1, sizeof(qo_index));
  h->n_qubits = n_qubits;
  h->kw = kw;
  uint64_t* xy_all = (uint64_t*)malloc((size_t)(n_merged ? n_merged : 1) * kw * 8);
  int64_t* grp = (int64_t*)malloc((size_t)(n_merged ? n_merged : 1) * 8);
  h->xy = (uint64_t*)malloc((size_t)(n_merged ? n_merged : 1) * kw * 8);
  h->xy_store = h->xy;
  wmap_init(&h->xy_map, n_merged, &h->xy_store, kw);
  int64_t n_xy = 0, n_keep = 0;
  for (int64_t i = 0; i < n_merged; ++i) {
    grp[i] = -1;
    if (fabs(mcoef[i]) < 1e-12) continue; /* kDropThreshold, hamiltonian.cpp:14,93 */
    const uint64_t* k = mkey + i * k3;
    for (int w = 0; w < kw; ++w) h->xy[n_xy * kw + w] = k[w] | k[kw + w];
    int64_t g = wmap_insert(&h->xy_map, n_xy);
    if (g < 0) g = n_xy++;
    grp[i] = g;
    ++n_keep;
  }
  (void)xy_all;
  free(xy_all);
  h->n_xy = n_xy;
  h->n_terms = n_keep;
  h->off = (int64_t*)calloc((size_t)n_xy + 1, 8);
  for (int64_t i = 0; i < n_merged; ++i)
    if (grp[i] >= 0) h->off[grp[i] + 1]++;
  for (int64_t g = 0; g < n_xy; ++g) h->off[g + 1] += h->off[g];
  int64_t* fill = (int64_t*)malloc((size_t)(n_xy ? n_xy : 1) * 8);
  for (int64_t g = 0; g < n_xy; ++g) fill[g] = h->off[g];
  h->coeff = (double*)malloc((size_t)(n_keep ? n_keep : 1) * 8);
  h->yz = (uint64_t*)malloc((size_t)(n_keep ? n_keep : 1) * kw * 8);
  h->yw = (uint8_t*)malloc((size_t)(n_keep ? n_keep : 1));
  for (int64_t i = 0; i < n_merged; ++i) {
    if (grp[i] < 0) continue;
    const int64_t t = fill[grp[i]]++;
    const uint64_t* k = mkey + i * k3;
    h->coeff[t] = mcoef[i];
    int yc = 0;
    for (int w = 0; w < kw; ++w) {
      h->yz[t * kw + w] = k[kw + w] | k[2 * kw + w];
      yc += __builtin_popcountll(k[kw + w]);
    }
    h->yw[t] = (uint8_t)yc;
  }
  free(fill);
  free(grp);
  free(mkey);
  free(mcoef);
  /* diagonal index (hamiltonian.cpp:114-115) */
  uint64_t zero[4] = {0, 0, 0, 0};
  h->diag = wmap_find(&h->xy_map, zero);
  return h;
}

void qo_index_info(const qo_index* h, int64_t* n_terms, int64_t* n_xy, int64_t* diag) {
  *n_terms = h->n_terms;
  *n_xy = h->n_xy;
  *diag = h->diag;
}

void qo_index_export(const qo_index* h, uint64_t* xy_words, int64_t* off, double* coeff, uint64_t* yz, uint8_t* yw) {
  if (xy_words) memcpy(xy_words, h->xy, (size_t)h->n_xy * h->kw * 8);
  if (off) memcpy(off, h->off, (size_t)(h->n_xy + 1) * 8);
  if (coeff) memcpy(coeff, h->coeff, (size_t)h->n_terms * 8);
  if (yz) memcpy(yz, h->yz, (size_t)h->n_terms * h->kw * 8);
  if (yw) memcpy(yw, h->yw, (size_t)h->n_terms);
}

/* ------------------------------------------------------ matrix elements */

/* i^q table (hamiltonian.cpp:19-20) */
static const double kQre[4] = {1.0, 0.0, -1.0, 0.0};
static const double kQim[4] = {0.0, 1.0, 0.0, -1.0};

void qo_group_element(const qo_index* h, const uint64_t* xp, int64_t g, double* out2) {
  double re = 0.0, im = 0.0;
  for (int64_t t = h->off[g]; t < h->off[g + 1]; ++t) {
    const int q = (h->yw[t] + 2 * and_popc(xp, h->yz + t * h->kw, h->kw)) & 3;
    re += h->coeff[t] * kQre[q];
    im += h->coeff[t] * kQim[q];
  }
  out2[0] = re;
  out2[1] = im;
}

void qo_matrix_element(const qo_index* h, const uint64_t* x, const uint64_t* xp, double* out2) {
  uint64_t m[4];
  for (int w = 0; w < h->kw; ++w) m[w] = x[w] ^ xp[w];
  const int64_t g = wmap_find(&h->xy_map, m);
  if (g < 0) {
    out2[0] = out2[1] = 0.0;
    return;
  }
  qo_group_element(h, xp, g, out2);
}

/* ------------------------------------------------------- coupled pairs */

static int cmp_pair(const void* a, const void* b) {
  const uint32_t* p = (const uint32_t*)a;
  const uint32_t* q = (const uint32_t*)b;
  return (p[1] > q[1]) - (p[1] < q[1]);
}

typedef struct {
  uint32_t* e;
  int64_t n, cap;
} vec3;

static void vec3_push(vec3* v, uint32_t a, uint32_t b, uint32_t c) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 1024;
    v->e = (uint32_t*)realloc(v->e, (size_t)v->cap * 12);
  }
  v->e[3 * v->n] = a;
  v->e[3 * v->n + 1] = b;
  v->e[3 * v->n + 2] = c;
  v->n++;
}

int64_t qo_pairs(const qo_index* h, int64_t n_unq, const uint64_t* keys, int backend, uint32_t** out3,
                 uint64_t* ops) {
  const int kw = h->kw;
  const uint64_t* store = keys;
  wmap members;
  wmap_init(&members, n_unq, &store, kw);
  for (int64_t i = 0; i < n_unq; ++i)
    if (wmap_insert(&members, i) >= 0) {
      wmap_free(&members);
      snprintf(g_err, sizeof g_err, "invalid_argument: duplicate basis vector at %lld", (long long)i);
      return -1;
    }
  vec3 v = {NULL, 0, 0};
  *ops = 0;
  uint64_t c[4];
  for (int64_t i = 0; i < n_unq; ++i) {
    const int64_t row0 = v.n;
    const uint64_t* x = keys + i * kw;
    if (backend == 0) {
      /* coupling.cpp:72-80: every flip mask, membership test */
      for (int64_t g = 0; g < h->n_xy; ++g) {
        for (int w = 0; w < kw; ++w) c[w] = x[w] ^ h->xy[g * kw + w];
        const int64_t j = wmap_find(&members, c);
        if (j >= 0) vec3_push(&v, (uint32_t)i, (uint32_t)j, (uint32_t)g);
      }
      *ops += (uint64_t)h->n_xy;
    } else {
      /* coupling.cpp:90-98: every partner, flip-mask lookup */
      for (int64_t j = 0; j < n_unq; ++j) {
        for (int w = 0; w < kw; ++w) c[w] = x[w] ^ keys[j * kw + w];
        const int64_t g = wmap_find(&h->xy_map, c);
        if (g >= 0) vec3_push(&v, (uint32_t)i, (uint32_t)j, (uint32_t)g);
      }
      *ops += (uint64_t)n_unq;
    }
    /* canonical order inside the row: by x' (coupling.cpp:49-52) */
    qsort(v.e + 3 * row0, (size_t)(v.n - row0), 12, cmp_pair);
  }
  wmap_free(&members);
  *out3 = v.e ? v.e : (uint32_t*)malloc(12);
  return v.n;
}

/* ------------------------------------------------------- local energies */

static void accumulate(const qo_index* h, const uint64_t* keys, const double* la, const double* ph, int64_t i,
                       int64_t j, int64_t g, double* sr, double* si) {
  double e2[2];
  qo_group_element(h, keys + j * h->kw, g, e2);
  const double dlog = la[j] - la[i];
  const double dphase = ph[j] - ph[i];
  const double a = exp(dlog);
  /* h * exp(dlog + 0i) * (cos + i sin)  (energy.cpp:38-43) */
  const double hr = e2[0] * a, hi = e2[1] * a;
  const double c = cos(dphase), s = sin(dphase);
  *sr += hr * c - hi * s;
  *si += hr * s + hi * c;
}

int qo_local_energies(const qo_index* h, int64_t n_unq, const uint64_t* keys, const double* la, const double* ph,
                      int64_t n_pairs, const uint32_t* p3, double* out) {
  int64_t* rb = (int64_t*)malloc((size_t)(n_unq ? n_unq : 1) * 8);
  int64_t* re = (int64_t*)malloc((size_t)(n_unq ? n_unq : 1) * 8);
  for (int64_t i = 0; i < n_unq; ++i) rb[i] = re[i] = 0;
  /* runs from the canonical order (energy.cpp:19-28) */
  int64_t b = 0;
  while (b < n_pairs) {
    int64_t e = b;
    const uint32_t x = p3[3 * b];
    while (e < n_pairs && p3[3 * e] == x) ++e;
    rb[x] = b;
    re[x] = e;
    b = e;
  }
  int status = 0;
  for (int64_t i = 0; i < n_unq; ++i) {
    if (isinf(la[i])) {
      snprintf(g_err, sizeof g_err, "logic_error: local_energies: sampled state has zero amplitude");
      status = -2;
      break;
    }
    double sr = 0.0, si = 0.0;
    for (int64_t e = rb[i]; e < re[i]; ++e) accumulate(h, keys, la, ph, i, p3[3 * e + 1], p3[3 * e + 2], &sr, &si);
    out[2 * i] = sr;
    out[2 * i + 1] = si;
  }
  free(rb);
  free(re);
  return status;
}

int qo_variational_energy(int64_t n, const double* lp, double norm, double log_norm, const double* eloc, double* out5,
                          double* weights) {
  if (!(norm > 0.0)) {
    snprintf(g_err, sizeof g_err, "runtime_error: variational_energy: sampled norm is zero");
    return -3;
  }
  double mr = 0.0, mi = 0.0, ipr = 0.0, sw = 0.0, se2 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double w = exp(lp[i] - log_norm);
    if (weights) weights[i] = w;
    mr += w * eloc[2 * i];
    mi += w * eloc[2 * i + 1];
    ipr += w * w;
    sw += w;
    se2 += w * (eloc[2 * i] * eloc[2 * i] + eloc[2 * i + 1] * eloc[2 * i + 1]);
  }
  out5[0] = mr;
  out5[1] = mi;
  out5[2] = ipr;
  out5[3] = sw;
  out5[4] = se2;
  const double ae = fabs(mr);
  if (fabs(mi) > 1e-6 * (ae > 1.0 ? ae : 1.0)) {
    snprintf(g_err, sizeof g_err, "runtime_error: variational_energy: imaginary residual %g", mi);
    return -4;
  }
  return 0;
}

/* --------------------------------------------- per-row E_loc (threaded) */

typedef struct {
  const qo_index* h;
  const wmap* members;
  const uint64_t* keys;
  const double *la, *ph;
  int64_t r0, r1, base;
  double* out;
  double* scale;
  int64_t visited;
  int status;
} rows_job;

static void* rows_worker(void* arg) {
  rows_job* J = (rows_job*)arg;
  const qo_index* h = J->h;
  const int kw = h->kw;
  uint32_t* hit = (uint32_t*)malloc((size_t)(h->n_xy ? h->n_xy : 1) * 12);
  uint64_t c[4];
  for (int64_t i = J->r0; i < J->r1; ++i) {
    if (isinf(J->la[i])) {
      J->status = -2;
      break;
    }
    const uint64_t* x = J->keys + i * kw;
    int64_t nh = 0;
    for (int64_t g = 0; g < h->n_xy; ++g) {
      for (int w = 0; w < kw; ++w) c[w] = x[w] ^ h->xy[g * kw + w];
      const int64_t j = wmap_find(J->members, c);
      if (j >= 0) {
        hit[3 * nh] = (uint32_t)i;
        hit[3 * nh + 1] = (uint32_t)j;
        hit[3 * nh + 2] = (uint32_t)g;
        ++nh;
      }
    }
    qsort(hit, (size_t)nh, 12, cmp_pair);
    double sr = 0.0, si = 0.0, sc = 0.0;
    for (int64_t e = 0; e < nh; ++e) {
      const int64_t j = hit[3 * e + 1], g = hit[3 * e + 2];
      accumulate(h, J->keys, J->la, J->ph, i, j, g, &sr, &si);
      if (J->scale) {
        double ga = 0.0;
        for (int64_t t = h->off[g]; t < h->off[g + 1]; ++t) ga += fabs(h->coeff[t]);
        sc += ga * exp(J->la[j] - J->la[i]);
      }
    }
    J->out[2 * (i - J->base)] = sr;
    J->out[2 * (i - J->base) + 1] = si;
    if (J->scale) J->scale[i - J->base] = sc;
    J->visited += nh;
  }
  free(hit);
  return NULL;
}

int64_t qo_eloc_rows(const qo_index* h, int64_t n_unq, const uint64_t* keys, const double* la, const double* ph,
                     int64_t r0, int64_t r1, int threads, double* out, double* scale) {
  const uint64_t* store = keys;
  wmap members;
  wmap_init(&members, n_unq, &store, h->kw);
  for (int64_t i = 0; i < n_unq; ++i)
    if (wmap_insert(&members, i) >= 0) {
      wmap_free(&members);
      snprintf(g_err, sizeof g_err, "invalid_argument: duplicate basis vector at %lld", (long long)i);
      return -1;
    }
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  rows_job jobs[256];
  pthread_t tid[256];
  const int64_t n = r1 - r0;
  const int64_t chunk = (n + threads - 1) / threads;
  int used = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t a = r0 + t * chunk, b = a + chunk < r1 ? a + chunk : r1;
    if (a >= b) break;
    jobs[t] = (rows_job){h, &members, keys, la, ph, a, b, r0, out, scale, 0, 0};
    pthread_create(&tid[t], NULL, rows_worker, &jobs[t]);
    ++used;
  }
  int64_t visited = 0;
  int status = 0;
  for (int t = 0; t < used; ++t) {
    pthread_join(tid[t], NULL);
    visited += jobs[t].visited;
    if (jobs[t].status) status = jobs[t].status;
  }
  wmap_free(&members);
  if (status) {
    snprintf(g_err, sizeof g_err, "logic_error: local_energies: sampled state has zero amplitude");
    return status;
  }
  return visited;
}

/* ------------------------------------ listed rows vs the whole sample set */

/* The rows of a row LIST against the whole sample set: per row the
 * LoopOverTerms candidate loop (coupling.cpp:72-80) over every flip mask,
 * the row's pairs in canonical order (coupling.cpp:49-52), and optionally
 * its E_loc (energy.cpp:35-44) and absolute-sum scale. One members map for
 * the whole call (the row-range variant above rebuilds nothing per row
 * either, but takes contiguous ranges only). */
typedef struct {
  const qo_index* h;
  const wmap* members;
  const uint64_t* keys;
  const double *la, *ph;
  const int64_t* rows;
  int64_t k0, k1;
  uint32_t** row_pairs; /* per listed row, malloc'd canonical triples */
  int64_t* counts;
  double* out;
  double* scale;
  int status;
} list_job;

static void* list_worker(void* arg) {
  list_job* J = (list_job*)arg;
  const qo_index* h = J->h;
  const int kw = h->kw;
  uint64_t c[4];
  for (int64_t k = J->k0; k < J->k1; ++k) {
    const int64_t i = J->rows[k];
    const uint64_t* x = J->keys + i * kw;
    vec3 v = {NULL, 0, 0};
    for (int64_t g = 0; g < h->n_xy; ++g) {
      for (int w = 0; w < kw; ++w) c[w] = x[w] ^ h->xy[g * kw + w];
      const int64_t j = wmap_find(J->members, c);
      if (j >= 0) vec3_push(&v, (uint32_t)i, (uint32_t)j, (uint32_t)g);
    }
    if (v.n) qsort(v.e, (size_t)v.n, 12, cmp_pair);
    J->row_pairs[k] = v.e;
    J->counts[k] = v.n;
    if (J->out) {
      if (isinf(J->la[i])) {
        J->status = -2;
        continue;
      }
      double sr = 0.0, si = 0.0, sc = 0.0;
      for (int64_t e = 0; e < v.n; ++e) {
        const int64_t j = v.e[3 * e + 1], g = v.e[3 * e + 2];
        accumulate(h, J->keys, J->la, J->ph, i, j, g, &sr, &si);
        double ga = 0.0;
        for (int64_t t = h->off[g]; t < h->off[g + 1]; ++t) ga += fabs(h->coeff[t]);
        sc += ga * exp(J->la[j] - J->la[i]);
      }
      J->out[2 * k] = sr;
      J->out[2 * k + 1] = si;
      if (J->scale) J->scale[k] = sc;
    }
  }
  return NULL;
}

int64_t qo_rows_list(const qo_index* h, int64_t n_unq, const uint64_t* keys, const double* la, const double* ph,
                     int64_t n_rows, const int64_t* rows, int threads, uint32_t** out3, int64_t* out_counts,
                     double* out_eloc, double* out_scale) {
  for (int64_t k = 0; k < n_rows; ++k)
    if (rows[k] < 0 || rows[k] >= n_unq) {
      snprintf(g_err, sizeof g_err, "invalid_argument: row %lld out of range", (long long)rows[k]);
      return -1;
    }
  const uint64_t* store = keys;
  wmap members;
  wmap_init(&members, n_unq, &store, h->kw);
  for (int64_t i = 0; i < n_unq; ++i)
    if (wmap_insert(&members, i) >= 0) {
      wmap_free(&members);
      snprintf(g_err, sizeof g_err, "invalid_argument: duplicate basis vector at %lld", (long long)i);
      return -1;
    }
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  uint32_t** rp = (uint32_t**)calloc((size_t)(n_rows ? n_rows : 1), sizeof(uint32_t*));
  list_job jobs[256];
  pthread_t tid[256];
  const int64_t chunk = (n_rows + threads - 1) / threads;
  int used = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t a = t * chunk, b = a + chunk < n_rows ? a + chunk : n_rows;
    if (a >= b) break;
    jobs[t] = (list_job){h, &members, keys, la, ph, rows, a, b, rp, out_counts, out_eloc, out_scale, 0};
    pthread_create(&tid[t], NULL, list_worker, &jobs[t]);
    ++used;
  }
  int status = 0;
  for (int t = 0; t < used; ++t) {
    pthread_join(tid[t], NULL);
    if (jobs[t].status) status = jobs[t].status;
  }
  wmap_free(&members);
  int64_t total = 0;
  for (int64_t k = 0; k < n_rows; ++k) total += out_counts[k];
  uint32_t* all = (uint32_t*)malloc((size_t)(total ? total : 1) * 12);
  int64_t at = 0;
  for (int64_t k = 0; k < n_rows; ++k) {
    if (out_counts[k]) memcpy(all + 3 * at, rp[k], (size_t)out_counts[k] * 12);
    at += out_counts[k];
    free(rp[k]);
  }
  free(rp);
  *out3 = all;
  if (status) {
    snprintf(g_err, sizeof g_err, "logic_error: local_energies: sampled state has zero amplitude");
    return status;
  }
  return total;
}
