/*
 * gm_oracle.c -- CPU restatement of the reference FastGM path.
 *
 * TEST INFRASTRUCTURE ONLY (see gm_oracle.h).  Built with
 * -ffp-contract=off and without fast-math so every double operation is
 * the same IEEE operation CPython performs; log() is glibc's.
 */
#define _GNU_SOURCE
#include "gm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* randgen.py:46-58 */
#define K_ELEM 0x9E3779B97F4A7C15ULL
#define K_STEP 0xC2B2AE3D27D4EB4FULL
#define K_RETRY 0xD6E8FEB86659FD93ULL
#define M1 0xBF58476D1CE4E5B9ULL
#define M2 0x94D049BB133111EBULL
#define INV_2_53 0x1p-53
#define INV_2_54 0x1p-54

uint64_t gmo_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * M1;
  x = (x ^ (x >> 27)) * M2;
  return x ^ (x >> 31);
}

uint64_t gmo_fingerprint(uint64_t global_seed, uint64_t stream_salt) {
  return gmo_mix64(global_seed + gmo_mix64(stream_salt));
}

uint64_t gmo_derive_seed(uint64_t master, uint64_t index) {
  return gmo_mix64(master + (index + 1) * K_ELEM);
}

static inline double u_from_bits(uint64_t x) {
  /* randgen.py:119: (x >> 11) * 2**-53 + 2**-54; the product is exact, the
   * add rounds to nearest even (can give exactly 1.0). */
  double a = (double)(x >> 11) * INV_2_53;
  return a + INV_2_54;
}

double gmo_uniform_open(uint64_t global_seed, uint64_t element, uint64_t step) {
  return u_from_bits(gmo_mix64(global_seed + element * K_ELEM + step * K_STEP));
}

/* The keyed uniforms u_i = uniform_open(seed, i0 + i, 1) and glibc's
 * log(u_i) (what math.log returns, randgen.py:186): the checker of the
 * device log. */
void gmo_log_uniforms(uint64_t seed, int64_t i0, int64_t n, double *u_out, double *log_out) {
  for (int64_t i = 0; i < n; ++i) {
    const double u = gmo_uniform_open(seed, (uint64_t)(i0 + i), 1);
    u_out[i] = u;
    log_out[i] = log(u);
  }
}

/* 2**64 mod m, for m >= 1 */
static inline uint64_t pow64_mod(uint64_t m) { return (UINT64_MAX % m + 1) % m; }

uint64_t gmo_rand_int_between(uint64_t perm_seed, uint64_t element,
                              uint64_t step, uint64_t lo, uint64_t hi) {
  uint64_t m = hi - lo + 1;
  uint64_t r = pow64_mod(m);
  uint64_t base = perm_seed + element * K_ELEM + step * K_STEP;
  for (uint64_t attempt = 0;; ++attempt) {
    uint64_t x = gmo_mix64(base + attempt * K_RETRY);
    /* limit = 2**64 - r; r == 0 means no rejection */
    if (r == 0 || x < (uint64_t)0 - r) return lo + x % m;
  }
}

/* ---- LazyPermutation (randgen.py:146-155): sparse map position->value,
 * missing slot i reads i+1.  Open addressing, keys are position+1. */
typedef struct {
  uint32_t *key;
  uint32_t *val;
  uint32_t cap; /* power of two or 0 */
  uint32_t used;
} permmap;

static void pm_free(permmap *p) {
  free(p->key);
  free(p->val);
  p->key = p->val = NULL;
  p->cap = p->used = 0;
}

static int pm_grow(permmap *p) {
  uint32_t ncap = p->cap ? p->cap * 2 : 16;
  uint32_t *nk = (uint32_t *)calloc(ncap, sizeof(uint32_t));
  uint32_t *nv = (uint32_t *)malloc(ncap * sizeof(uint32_t));
  if (!nk || !nv) {
    free(nk);
    free(nv);
    return -1;
  }
  for (uint32_t i = 0; i < p->cap; ++i) {
    if (!p->key[i]) continue;
    uint32_t h = (p->key[i] * 0x9E3779B1u) & (ncap - 1);
    while (nk[h]) h = (h + 1) & (ncap - 1);
    nk[h] = p->key[i];
    nv[h] = p->val[i];
  }
  free(p->key);
  free(p->val);
  p->key = nk;
  p->val = nv;
  p->cap = ncap;
  return 0;
}

static inline uint32_t pm_get(const permmap *p, uint32_t pos) {
  if (p->cap) {
    uint32_t key = pos + 1;
    uint32_t h = (key * 0x9E3779B1u) & (p->cap - 1);
    while (p->key[h]) {
      if (p->key[h] == key) return p->val[h];
      h = (h + 1) & (p->cap - 1);
    }
  }
  return pos + 1;
}

static inline int pm_set(permmap *p, uint32_t pos, uint32_t v) {
  if ((p->used + 1) * 2 > p->cap && pm_grow(p)) return -1;
  uint32_t key = pos + 1;
  uint32_t h = (key * 0x9E3779B1u) & (p->cap - 1);
  while (p->key[h]) {
    if (p->key[h] == key) {
      p->val[h] = v;
      return 0;
    }
    h = (h + 1) & (p->cap - 1);
  }
  p->key[h] = key;
  p->val[h] = v;
  p->used++;
  return 0;
}

/* randgen.py:158-207, emitting order statistics z0+1..z1.  perm is either
 * a dense 1..k array (dense != NULL) or a permmap.  Returns b. */
static double run_queue(uint64_t useed, uint64_t pseed, uint64_t element,
                        double weight, int32_t k, int32_t z0, int32_t z1,
                        double b, uint32_t *dense, permmap *pm,
                        double *out_t, int32_t *out_s, int *oom) {
  uint64_t ubase = useed + element * K_ELEM;
  uint64_t pbase = pseed + element * K_ELEM;
  int idx = 0;
  for (int32_t z = z0 + 1; z <= z1; ++z) {
    uint64_t x = gmo_mix64(ubase + (uint64_t)z * K_STEP);
    double u = u_from_bits(x);
    double denom = weight * (double)(k - z + 1);
    double inc = -log(u) / denom;
    b = b + inc;
    uint64_t m = (uint64_t)(k - z + 1);
    uint64_t r = pow64_mod(m);
    uint64_t g = gmo_mix64(pbase + (uint64_t)z * K_STEP);
    uint64_t attempt = 0;
    while (r != 0 && g >= (uint64_t)0 - r) {
      ++attempt;
      g = gmo_mix64(pbase + (uint64_t)z * K_STEP + attempt * K_RETRY);
    }
    uint32_t j = (uint32_t)((uint64_t)z + g % m);
    uint32_t zi = (uint32_t)z - 1, ji = j - 1;
    uint32_t vz, vj;
    if (dense) {
      vz = dense[zi];
      vj = dense[ji];
      dense[zi] = vj;
      dense[ji] = vz;
    } else {
      vz = pm_get(pm, zi);
      vj = pm_get(pm, ji);
      if (pm_set(pm, zi, vj) || pm_set(pm, ji, vz)) *oom = 1;
    }
    out_t[idx] = b;
    out_s[idx] = (int32_t)vj; /* perm[zi] after the swap */
    ++idx;
  }
  return b;
}

void gmo_run_queue_full(uint64_t global_seed, uint64_t perm_seed,
                        uint64_t element, double weight, int32_t k,
                        double *times, int32_t *servers) {
  uint32_t *dense = (uint32_t *)malloc((size_t)k * sizeof(uint32_t));
  for (int32_t i = 0; i < k; ++i) dense[i] = (uint32_t)i + 1;
  int oom = 0;
  run_queue(global_seed, perm_seed, element, weight, k, 0, k, 0.0, dense, NULL,
            times, servers, &oom);
  free(dense);
}

/* ---- CPython math.fsum: Shewchuk partials + exact final rounding. */
double gmo_fsum(const double *x, int64_t n) {
  int64_t cap = 32, np = 0;
  double *p = (double *)malloc((size_t)cap * sizeof(double));
  for (int64_t t = 0; t < n; ++t) {
    double xv = x[t];
    int64_t i = 0;
    for (int64_t j = 0; j < np; ++j) {
      double y = p[j];
      if (fabs(xv) < fabs(y)) {
        double tmp = xv;
        xv = y;
        y = tmp;
      }
      double hi = xv + y;
      double lo = y - (hi - xv);
      if (lo != 0.0) p[i++] = lo;
      xv = hi;
    }
    np = i;
    if (np == cap) {
      cap *= 2;
      p = (double *)realloc(p, (size_t)cap * sizeof(double));
    }
    p[np++] = xv;
  }
  double hi = 0.0, lo = 0.0;
  int64_t m = np;
  if (m > 0) {
    hi = p[--m];
    while (m > 0) {
      double xv = hi;
      double y = p[--m];
      hi = xv + y;
      double yr = hi - xv;
      lo = y - yr;
      if (lo != 0.0) break;
    }
    if (m > 0 && ((lo < 0.0 && p[m - 1] < 0.0) || (lo > 0.0 && p[m - 1] > 0.0))) {
      double y = lo * 2.0;
      double xv = hi + y;
      double yr = xv - hi;
      if (y == yr) hi = xv;
    }
  }
  free(p);
  return hi;
}

static int check_weights(const double *w, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    double v = w[i];
    if (!isfinite(v) || v <= 0.0 || v < 1e-300) return GMO_INVALID_WEIGHT;
  }
  return GMO_OK;
}

/* sketch.py:183-209 */
int gmo_sketch_naive(const uint64_t *ids, const double *w, int64_t n,
                     int32_t k, uint64_t global_seed, uint64_t stream_salt,
                     double *y, uint64_t *s, int64_t *emitted) {
  if (k < 1) return GMO_INVALID_PARAMETER;
  if (n == 0) return GMO_EMPTY_VECTOR;
  if (check_weights(w, n)) return GMO_INVALID_WEIGHT;
  uint64_t pseed = global_seed ^ stream_salt;
  double *times = (double *)malloc((size_t)k * sizeof(double));
  int32_t *servers = (int32_t *)malloc((size_t)k * sizeof(int32_t));
  uint32_t *dense = (uint32_t *)malloc((size_t)k * sizeof(uint32_t));
  unsigned char *set = (unsigned char *)calloc((size_t)k, 1);
  if (!times || !servers || !dense || !set) return GMO_NO_MEMORY;
  int oom = 0;
  for (int64_t e = 0; e < n; ++e) {
    for (int32_t i = 0; i < k; ++i) dense[i] = (uint32_t)i + 1;
    run_queue(global_seed, pseed, ids[e], w[e], k, 0, k, 0.0, dense, NULL,
              times, servers, &oom);
    for (int32_t idx = 0; idx < k; ++idx) {
      double t = times[idx];
      int32_t c = servers[idx] - 1;
      if (!set[c] || t < y[c]) {
        set[c] = 1;
        y[c] = t;
        s[c] = ids[e];
      }
    }
  }
  free(times);
  free(servers);
  free(dense);
  free(set);
  if (emitted) *emitted = n * (int64_t)k;
  return GMO_OK;
}

static int32_t argmax_first(const double *y, int32_t k) {
  int32_t best = 0;
  for (int32_t j = 1; j < k; ++j)
    if (y[j] > y[best]) best = j;
  return best;
}

/* sketch.py:218-311 */
int gmo_sketch_fast(const uint64_t *ids, const double *w, int64_t n,
                    int32_t k, int64_t delta, uint64_t global_seed,
                    uint64_t stream_salt, double *y, uint64_t *s,
                    int64_t *emitted) {
  if (k < 1) return GMO_INVALID_PARAMETER;
  if (delta <= 0) delta = k;
  if (n == 0) return GMO_EMPTY_VECTOR;
  if (check_weights(w, n)) return GMO_INVALID_WEIGHT;
  uint64_t pseed = global_seed ^ stream_salt;
  double weight_sum = gmo_fsum(w, n);
  int32_t *zs = (int32_t *)calloc((size_t)n, sizeof(int32_t));
  double *bs = (double *)calloc((size_t)n, sizeof(double));
  permmap *perms = (permmap *)calloc((size_t)n, sizeof(permmap));
  double *times = (double *)malloc((size_t)k * sizeof(double));
  int32_t *servers = (int32_t *)malloc((size_t)k * sizeof(int32_t));
  unsigned char *set = (unsigned char *)calloc((size_t)k, 1);
  if (!zs || !bs || !perms || !times || !servers || !set) return GMO_NO_MEMORY;
  int64_t emit = 0;
  int32_t unset = k;
  int64_t R = 0;
  int oom = 0;
  while (unset) {
    R += delta;
    for (int64_t idx = 0; idx < n; ++idx) {
      double weight = w[idx];
      double tf = ceil((double)R * weight / weight_sum);
      int32_t target = tf > (double)k ? k : (int32_t)tf;
      int32_t z = zs[idx];
      if (z >= target) continue;
      bs[idx] = run_queue(global_seed, pseed, ids[idx], weight, k, z, target,
                          bs[idx], NULL, &perms[idx], times, servers, &oom);
      int32_t span = target - z;
      emit += span;
      for (int32_t t = 0; t < span; ++t) {
        double tv = times[t];
        int32_t c = servers[t] - 1;
        if (!set[c]) {
          set[c] = 1;
          y[c] = tv;
          s[c] = ids[idx];
          --unset;
        } else if (tv < y[c]) {
          y[c] = tv;
          s[c] = ids[idx];
        }
      }
      zs[idx] = target;
    }
  }
  int32_t jstar = argmax_first(y, k);
  double one_t;
  int32_t one_s;
  for (int64_t idx = 0; idx < n; ++idx) {
    int32_t z = zs[idx];
    if (z >= k) continue;
    double weight = w[idx];
    double b = bs[idx];
    while (z < k) {
      b = run_queue(global_seed, pseed, ids[idx], weight, k, z, z + 1, b, NULL,
                    &perms[idx], &one_t, &one_s, &oom);
      ++z;
      ++emit;
      if (one_t > y[jstar]) break;
      int32_t c = one_s - 1;
      if (one_t < y[c]) {
        y[c] = one_t;
        s[c] = ids[idx];
        if (c == jstar) jstar = argmax_first(y, k);
      }
    }
    zs[idx] = z;
    bs[idx] = b;
    pm_free(&perms[idx]);
  }
  for (int64_t idx = 0; idx < n; ++idx) pm_free(&perms[idx]);
  free(zs);
  free(bs);
  free(perms);
  free(times);
  free(servers);
  free(set);
  if (emitted) *emitted = emit;
  return oom ? GMO_NO_MEMORY : GMO_OK;
}

/* ---- id -> weight map for stream dedup (stream.py:67-78) */
typedef struct {
  uint64_t *key;
  double *val;
  unsigned char *used;
  uint64_t cap, count;
} wmap;

static inline uint64_t wm_hash(uint64_t key) { return gmo_mix64(key ^ 0x5bd1e995ULL); }

static int wm_grow(wmap *m) {
  uint64_t ncap = m->cap ? m->cap * 2 : 64;
  uint64_t *nk = (uint64_t *)malloc(ncap * sizeof(uint64_t));
  double *nv = (double *)malloc(ncap * sizeof(double));
  unsigned char *nu = (unsigned char *)calloc(ncap, 1);
  if (!nk || !nv || !nu) return -1;
  for (uint64_t i = 0; i < m->cap; ++i) {
    if (!m->used[i]) continue;
    uint64_t h = wm_hash(m->key[i]) & (ncap - 1);
    while (nu[h]) h = (h + 1) & (ncap - 1);
    nu[h] = 1;
    nk[h] = m->key[i];
    nv[h] = m->val[i];
  }
  free(m->key);
  free(m->val);
  free(m->used);
  m->key = nk;
  m->val = nv;
  m->used = nu;
  m->cap = ncap;
  return 0;
}

/* returns pointer to stored weight or NULL (and inserts w when absent) */
static double *wm_find_or_insert(wmap *m, uint64_t key, double w, int *inserted, int *oom) {
  if ((m->count + 1) * 2 > m->cap && wm_grow(m)) {
    *oom = 1;
    return NULL;
  }
  uint64_t h = wm_hash(key) & (m->cap - 1);
  while (m->used[h]) {
    if (m->key[h] == key) {
      *inserted = 0;
      return &m->val[h];
    }
    h = (h + 1) & (m->cap - 1);
  }
  m->used[h] = 1;
  m->key[h] = key;
  m->val[h] = w;
  m->count++;
  *inserted = 1;
  return &m->val[h];
}

/* stream.py:58-153 */
int gmo_sketch_stream(const uint64_t *ids, const double *w, int64_t n,
                      int32_t k, uint64_t global_seed, uint64_t stream_salt,
                      int skip_duplicates, double *y, uint64_t *s,
                      int64_t *emitted, int64_t *err_index) {
  if (k < 1) return GMO_INVALID_PARAMETER;
  uint64_t pseed = global_seed ^ stream_salt;
  wmap wm;
  memset(&wm, 0, sizeof(wm));
  unsigned char *set = (unsigned char *)calloc((size_t)k, 1);
  uint32_t *dense = (uint32_t *)malloc((size_t)k * sizeof(uint32_t));
  uint32_t *touched = (uint32_t *)malloc((size_t)k * 2 * sizeof(uint32_t));
  if (!set || !dense || !touched) return GMO_NO_MEMORY;
  for (int32_t i = 0; i < k; ++i) dense[i] = (uint32_t)i + 1;
  int32_t unset = k, jstar = 0;
  int prune = 0, oom = 0, rc = GMO_OK;
  int64_t emit = 0;
  for (int64_t it = 0; it < n; ++it) {
    uint64_t element = ids[it];
    double weight = w[it];
    if (!isfinite(weight) || weight <= 0.0 || weight < 1e-300) {
      rc = GMO_INVALID_WEIGHT;
      if (err_index) *err_index = it;
      break;
    }
    int inserted = 0;
    double *known = wm_find_or_insert(&wm, element, weight, &inserted, &oom);
    if (oom) {
      rc = GMO_NO_MEMORY;
      break;
    }
    if (!inserted) {
      if (*known != weight) {
        rc = GMO_INCONSISTENT_WEIGHT;
        if (err_index) *err_index = it;
        break;
      }
      if (skip_duplicates) continue;
    }
    /* one element at a time: a dense permutation restored after use */
    double b = 0.0, t;
    int32_t z = 0, c, ntouch = 0;
    uint64_t ubase = global_seed + element * K_ELEM;
    uint64_t pbase = pseed + element * K_ELEM;
    while (z < k) {
      /* inline run_queue(z -> z+1) so touched slots can be restored */
      ++z;
      uint64_t x = gmo_mix64(ubase + (uint64_t)z * K_STEP);
      double u = u_from_bits(x);
      double denom = weight * (double)(k - z + 1);
      b = b + (-log(u) / denom);
      uint64_t m = (uint64_t)(k - z + 1);
      uint64_t r = pow64_mod(m);
      uint64_t g = gmo_mix64(pbase + (uint64_t)z * K_STEP);
      uint64_t attempt = 0;
      while (r != 0 && g >= (uint64_t)0 - r) {
        ++attempt;
        g = gmo_mix64(pbase + (uint64_t)z * K_STEP + attempt * K_RETRY);
      }
      uint32_t j = (uint32_t)((uint64_t)z + g % m);
      uint32_t zi = (uint32_t)z - 1, ji = j - 1;
      uint32_t vz = dense[zi], vj = dense[ji];
      dense[zi] = vj;
      dense[ji] = vz;
      touched[ntouch++] = zi;
      touched[ntouch++] = ji;
      ++emit;
      t = b;
      c = (int32_t)vj - 1;
      if (!prune) {
        if (!set[c]) {
          set[c] = 1;
          y[c] = t;
          s[c] = element;
          if (--unset == 0) {
            prune = 1;
            jstar = argmax_first(y, k);
          }
        } else if (t < y[c]) {
          y[c] = t;
          s[c] = element;
        }
      }
      if (prune) {
        if (t > y[jstar]) break;
        if (t < y[c]) {
          y[c] = t;
          s[c] = element;
          if (c == jstar) jstar = argmax_first(y, k);
        }
      }
    }
    for (int32_t q = 0; q < ntouch; ++q) dense[touched[q]] = touched[q] + 1;
  }
  if (rc == GMO_OK && unset > 0) rc = GMO_INCOMPLETE;
  free(wm.key);
  free(wm.val);
  free(wm.used);
  free(set);
  free(dense);
  free(touched);
  if (emitted) *emitted = emit;
  return rc;
}

/* ---- batched CSR on host threads (the CPU baseline) */
typedef struct {
  const uint64_t *ids;
  const double *w;
  const int64_t *offsets;
  int64_t n_vec;
  int32_t k;
  uint64_t seed, salt;
  int mode;
  double *y;
  uint64_t *s;
  int64_t *emitted;
  int64_t next; /* atomic work counter */
  int rc;
} csr_job;

typedef struct {
  uint64_t id;
  double w;
} item;

static int item_cmp(const void *a, const void *b) {
  uint64_t x = ((const item *)a)->id, y = ((const item *)b)->id;
  return x < y ? -1 : x > y;
}

static void *csr_worker(void *arg) {
  csr_job *job = (csr_job *)arg;
  uint64_t *ids = NULL;
  double *ws = NULL;
  item *items = NULL;
  int64_t cap = 0;
  for (;;) {
    int64_t v = __atomic_fetch_add(&job->next, 1, __ATOMIC_RELAXED);
    if (v >= job->n_vec) break;
    int64_t lo = job->offsets[v], hi = job->offsets[v + 1], n = hi - lo;
    double *y = job->y + v * (int64_t)job->k;
    uint64_t *s = job->s + v * (int64_t)job->k;
    int64_t em = 0;
    int rc;
    if (job->mode == 0) {
      if (n > cap) {
        cap = n;
        ids = (uint64_t *)realloc(ids, (size_t)cap * sizeof(uint64_t));
        ws = (double *)realloc(ws, (size_t)cap * sizeof(double));
        items = (item *)realloc(items, (size_t)cap * sizeof(item));
      }
      for (int64_t i = 0; i < n; ++i) {
        items[i].id = job->ids[lo + i];
        items[i].w = job->w[lo + i];
      }
      qsort(items, (size_t)n, sizeof(item), item_cmp);
      for (int64_t i = 0; i < n; ++i) {
        ids[i] = items[i].id;
        ws[i] = items[i].w;
      }
      rc = gmo_sketch_fast(ids, ws, n, job->k, job->k, job->seed, job->salt, y, s, &em);
    } else {
      rc = gmo_sketch_stream(job->ids + lo, job->w + lo, n, job->k, job->seed,
                             job->salt, 1, y, s, &em, NULL);
    }
    if (job->emitted) job->emitted[v] = em;
    if (rc) __atomic_store_n(&job->rc, rc, __ATOMIC_RELAXED);
  }
  free(ids);
  free(ws);
  free(items);
  return NULL;
}

int gmo_sketch_csr(const uint64_t *ids, const double *w,
                   const int64_t *offsets, int64_t n_vec, int32_t k,
                   uint64_t global_seed, uint64_t stream_salt, int mode,
                   int threads, double *y, uint64_t *s, int64_t *emitted) {
  if (k < 1) return GMO_INVALID_PARAMETER;
  csr_job job = {ids, w, offsets, n_vec, k, global_seed, stream_salt, mode,
                 y, s, emitted, 0, GMO_OK};
  if (threads < 1) threads = 1;
  if (threads == 1) {
    csr_worker(&job);
    return job.rc;
  }
  pthread_t *th = (pthread_t *)malloc((size_t)threads * sizeof(pthread_t));
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, csr_worker, &job);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
  return job.rc;
}

/* estimate.py:103-125 */
void gmo_merge(const double *y_in, const uint64_t *s_in, int64_t n_sk,
               int32_t k, double *y_out, uint64_t *s_out) {
  memcpy(y_out, y_in, (size_t)k * sizeof(double));
  memcpy(s_out, s_in, (size_t)k * sizeof(uint64_t));
  for (int64_t r = 1; r < n_sk; ++r)
    for (int32_t j = 0; j < k; ++j) {
      double t = y_in[r * k + j];
      if (t < y_out[j]) {
        y_out[j] = t;
        s_out[j] = s_in[r * k + j];
      }
    }
}
