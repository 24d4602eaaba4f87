/*
 * graphmat_oracle.c -- CPU restatement of the reference superstep path.
 *
 * TEST INFRASTRUCTURE ONLY (see graphmat_oracle.h).  Compiled with
 * -ffp-contract=off so fp64 folds round exactly like the reference build
 * (FMA contraction breaks bitwise parity).
 */
#define _POSIX_C_SOURCE 200809L
#include "graphmat_oracle.h"

#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------ RNG */

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

static uint64_t splitmix_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t or_mix64(uint64_t x) {
  uint64_t s = x;
  return splitmix_next(&s);
}

/* Seeded bijection on [0, 2^scale): 4 rounds of add-const, multiply-by-odd and
 * xor-shift-right, all mod 2^scale (each step is invertible). */
typedef struct {
  uint64_t add[4], mul[4], mask;
  unsigned shift;
} perm_keys;

static void perm_init(perm_keys* pk, unsigned scale, uint64_t seed) {
  uint64_t st = seed ^ 0x7E57AB1E5EEDull;
  for (int r = 0; r < 4; ++r) {
    pk->add[r] = splitmix_next(&st);
    pk->mul[r] = splitmix_next(&st) | 1ull;
  }
  pk->mask = scale >= 64 ? ~0ull : ((1ull << scale) - 1ull);
  pk->shift = scale / 2 + 1;
}

static uint32_t perm_apply(const perm_keys* pk, uint32_t x) {
  uint64_t v = x;
  for (int r = 0; r < 4; ++r) {
    v = (v + pk->add[r]) & pk->mask;
    v = (v * pk->mul[r]) & pk->mask;
    v ^= v >> pk->shift;
  }
  return (uint32_t)v;
}

uint32_t or_permute(uint32_t x, unsigned scale, uint64_t seed) {
  perm_keys pk;
  perm_init(&pk, scale, seed);
  return perm_apply(&pk, x);
}

static uint64_t prob_threshold(double p) {
  if (p >= 1.0) return 1ull << 32;
  if (p <= 0.0) return 0;
  return (uint64_t)(p * 4294967296.0);
}

typedef struct {
  unsigned scale;
  uint64_t ta, tab, tabc, lo, hi;
  uint32_t key[2];
  int permute;
  const perm_keys* pk;
  uint32_t *src, *dst;
} rmat_job;

static void* rmat_worker(void* arg) {
  const rmat_job* j = (const rmat_job*)arg;
  const unsigned scale = j->scale;
  for (uint64_t t = j->lo; t < j->hi; ++t) {
    uint32_t s = 0, d = 0;
    for (unsigned l = 0; l < scale; l += 4) {
      const uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32), l >> 2, 0x524D4154u};
      uint32_t out[4];
      or_philox4x32_10(ctr, j->key, out);
      for (unsigned q = 0; q < 4 && l + q < scale; ++q) {
        const uint64_t r = out[q];
        const uint32_t bit = 1u << (scale - 1 - (l + q));
        if (r < j->ta) {
        } else if (r < j->tab) {
          d |= bit;
        } else if (r < j->tabc) {
          s |= bit;
        } else {
          s |= bit;
          d |= bit;
        }
      }
    }
    if (j->permute) {
      s = perm_apply(j->pk, s);
      d = perm_apply(j->pk, d);
    }
    j->src[t] = s;
    j->dst[t] = d;
  }
  return NULL;
}

/* Each tuple t is a pure function of (seed, t): the work is split across host
 * threads without changing the output. */
int64_t or_rmat_generate(unsigned scale, unsigned edge_factor, double a, double b, double c,
                         uint64_t seed, int permute, uint32_t* src, uint32_t* dst) {
  const uint64_t count = (uint64_t)edge_factor << scale;
  perm_keys pk;
  perm_init(&pk, scale, seed);
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  if (count < (1u << 16)) nt = 1;
  rmat_job jobs[64];
  pthread_t th[64];
  for (long i = 0; i < nt; ++i) {
    rmat_job* j = &jobs[i];
    j->scale = scale;
    j->ta = prob_threshold(a);
    j->tab = prob_threshold(a + b);
    j->tabc = prob_threshold(a + b + c);
    j->lo = count * (uint64_t)i / (uint64_t)nt;
    j->hi = count * (uint64_t)(i + 1) / (uint64_t)nt;
    j->key[0] = (uint32_t)seed;
    j->key[1] = (uint32_t)(seed >> 32);
    j->permute = permute;
    j->pk = &pk;
    j->src = src;
    j->dst = dst;
    if (nt > 1) pthread_create(&th[i], NULL, rmat_worker, j);
  }
  if (nt == 1)
    rmat_worker(&jobs[0]);
  else
    for (long i = 0; i < nt; ++i) pthread_join(th[i], NULL);
  return (int64_t)count;
}

uint8_t or_edge_weight(uint64_t seed, uint32_t src, uint32_t dst) {
  const uint64_t sw = or_mix64(seed ^ 0x57E16475ull);
  const uint64_t h = or_mix64(sw ^ (((uint64_t)src << 32) | dst));
  return (uint8_t)(1u + (uint32_t)((h >> 32) % 255u));
}

void or_edge_weights(uint64_t seed, int64_t m, const uint32_t* src, const uint32_t* dst,
                     uint8_t* w) {
  for (int64_t e = 0; e < m; ++e) w[e] = or_edge_weight(seed, src[e], dst[e]);
}

/* Cumulative rating pmf (0.05, 0.10, 0.29, 0.34, 0.22) as 32-bit thresholds. */
static const uint32_t kRatingThr[4] = {214748365u, 644245094u, 1889785610u, 3350074491u};

uint8_t or_rating(uint64_t seed, uint32_t user, uint32_t item) {
  const uint64_t sr = or_mix64(seed ^ 0x0DA7A5EEDull);
  const uint32_t h = (uint32_t)(or_mix64(sr ^ (((uint64_t)user << 32) | item)) >> 32);
  uint8_t r = 1;
  for (int i = 0; i < 4; ++i) r = (uint8_t)(r + (h >= kRatingThr[i]));
  return r;
}

void or_ratings(uint64_t seed, int64_t m, const uint32_t* src, const uint32_t* dst, uint8_t* r) {
  for (int64_t e = 0; e < m; ++e) r[e] = or_rating(seed, src[e], dst[e]);
}

int64_t or_bipartite_generate(uint32_t users, uint32_t items, double c_numerator, uint32_t cap,
                              uint64_t seed, uint32_t* src, uint32_t* dst) {
  /* Zipf(0.8) CDF over item ranks 1..items as 32-bit thresholds. */
  uint64_t* thr = (uint64_t*)malloc(sizeof(uint64_t) * (items ? items : 1));
  double total = 0.0;
  for (uint32_t j = 1; j <= items; ++j) total += pow((double)j, -0.8);
  double cum = 0.0;
  for (uint32_t j = 1; j <= items; ++j) {
    cum += pow((double)j, -0.8);
    thr[j - 1] = j == items ? (1ull << 32) : (uint64_t)(cum / total * 4294967296.0);
  }
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  int64_t out_n = 0;
  for (uint32_t u = 0; u < users; ++u) {
    double dd = floor(c_numerator / (double)(u + 1));
    if (dd < 1.0) dd = 1.0;
    if (dd > (double)cap) dd = (double)cap;
    const uint32_t deg = (uint32_t)dd;
    if (!src) {
      out_n += deg;
      continue;
    }
    uint32_t words[4] = {0, 0, 0, 0};
    for (uint32_t k = 0; k < deg; ++k) {
      if ((k & 3u) == 0) {
        const uint32_t ctr[4] = {u, k >> 2, 0, 0x42495054u};
        or_philox4x32_10(ctr, key, words);
      }
      const uint64_t r = words[k & 3u];
      uint32_t lo = 0, hi = items - 1; /* first j with r < thr[j] */
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (r < thr[mid])
          hi = mid;
        else
          lo = mid + 1;
      }
      src[out_n] = u;
      dst[out_n] = users + lo;
      ++out_n;
    }
  }
  free(thr);
  return out_n;
}

uint32_t or_pick_source(uint64_t seed, uint64_t n, const uint32_t* degree) {
  if (n == 0) return 0;
  const uint64_t base = or_mix64(seed ^ 0x50C0FFEEull);
  for (uint64_t i = 0; i < 1024; ++i) {
    const uint64_t cand = or_mix64(base + i) % n;
    if (degree[cand] > 0) return (uint32_t)cand;
  }
  for (uint64_t v = 0; v < n; ++v)
    if (degree[v] > 0) return (uint32_t)v;
  return 0;
}

/* ------------------------------------------------------------ preprocess */

/* Stable LSD radix sort of (key, payload) by key, 16-bit digits, skipping
 * digits that are constant across the input. */
static void radix_sort_kv(uint64_t* k, uint32_t* v, int64_t n) {
  if (n <= 1) return;
  uint64_t* k2 = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  uint32_t* v2 = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * 65536);
  uint64_t *ka = k, *kb = k2;
  uint32_t *va = v, *vb = v2;
  for (int shift = 0; shift < 64; shift += 16) {
    memset(cnt, 0, sizeof(int64_t) * 65536);
    for (int64_t i = 0; i < n; ++i) ++cnt[(ka[i] >> shift) & 0xFFFF];
    int trivial = 0;
    for (int d = 0; d < 65536; ++d)
      if (cnt[d] == n) trivial = 1;
    if (trivial) continue;
    int64_t run = 0;
    for (int d = 0; d < 65536; ++d) {
      const int64_t c = cnt[d];
      cnt[d] = run;
      run += c;
    }
    for (int64_t i = 0; i < n; ++i) {
      const int64_t pos = cnt[(ka[i] >> shift) & 0xFFFF]++;
      kb[pos] = ka[i];
      vb[pos] = va[i];
    }
    uint64_t* tk = ka;
    ka = kb;
    kb = tk;
    uint32_t* tv = va;
    va = vb;
    vb = tv;
  }
  if (ka != k) {
    memcpy(k, ka, sizeof(uint64_t) * (size_t)n);
    memcpy(v, va, sizeof(uint32_t) * (size_t)n);
  }
  free(k2);
  free(v2);
  free(cnt);
}

/* cleanup(): erase self loops, stable sort by (src,dst), unique keep-first
 * (src/io.cpp:192-196). */
static int64_t cleanup(int64_t m, uint32_t* src, uint32_t* dst, double* vals) {
  int64_t w = 0;
  for (int64_t e = 0; e < m; ++e) {
    if (src[e] == dst[e]) continue;
    src[w] = src[e];
    dst[w] = dst[e];
    if (vals) vals[w] = vals[e];
    ++w;
  }
  m = w;
  if (m == 0) return 0;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m);
  uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m);
  for (int64_t e = 0; e < m; ++e) {
    keys[e] = ((uint64_t)src[e] << 32) | dst[e];
    idx[e] = (uint32_t)e;
  }
  radix_sort_kv(keys, idx, m);
  double* nv = NULL;
  if (vals) {
    nv = (double*)malloc(sizeof(double) * (size_t)m);
    memcpy(nv, vals, sizeof(double) * (size_t)m);
  }
  int64_t out = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (i > 0 && keys[i] == keys[i - 1]) continue;
    src[out] = (uint32_t)(keys[i] >> 32);
    dst[out] = (uint32_t)keys[i];
    if (vals) vals[out] = nv[idx[i]];
    ++out;
  }
  free(keys);
  free(idx);
  free(nv);
  return out;
}

/* io::preprocess (src/io.cpp:184-222): cleanup, then SYMMETRIZE / DAGIFY append
 * the reversed edges after the originals and clean up again (stable: an
 * original (a, b) keeps its value over the reverse of (b, a)); DAGIFY then
 * drops src >= dst; BIPARTITE_CHECK rejects an edge whose source is some
 * edge's destination or whose destination is some edge's source. */
int64_t or_preprocess_checked(int64_t m, uint32_t* src, uint32_t* dst, double* vals, int mode,
                              int64_t* bad) {
  m = cleanup(m, src, dst, vals);
  if (mode == 1 || mode == 2) {
    for (int64_t e = 0; e < m; ++e) {
      src[m + e] = dst[e];
      dst[m + e] = src[e];
      if (vals) vals[m + e] = vals[e];
    }
    m = cleanup(2 * m, src, dst, vals);
    if (mode == 2) {
      int64_t w = 0;
      for (int64_t e = 0; e < m; ++e) {
        if (src[e] >= dst[e]) continue;
        src[w] = src[e];
        dst[w] = dst[e];
        if (vals) vals[w] = vals[e];
        ++w;
      }
      m = w;
    }
  } else if (mode == 3) {
    uint32_t mx = 0;
    for (int64_t e = 0; e < m; ++e) {
      if (src[e] > mx) mx = src[e];
      if (dst[e] > mx) mx = dst[e];
    }
    uint8_t* role = (uint8_t*)calloc((size_t)mx + 1, 1); /* bit 0 source, bit 1 destination */
    for (int64_t e = 0; e < m; ++e) {
      role[src[e]] |= 1;
      role[dst[e]] |= 2;
    }
    for (int64_t e = 0; e < m; ++e)
      if ((role[src[e]] & 2) || (role[dst[e]] & 1)) {
        if (bad) *bad = e;
        free(role);
        return -1;
      }
    free(role);
  }
  return m;
}

int64_t or_preprocess(int64_t m, uint32_t* src, uint32_t* dst, double* vals, int mode) {
  return or_preprocess_checked(m, src, dst, vals, mode, NULL);
}

/* triangle_count (algorithms/triangle_count.hpp:115-134): phase 1 gives every
 * vertex its ascending in-neighbour list (NeighborGatherProgram), phase 2 sends
 * each list along the out-edges and the receiver counts the ids shared with its
 * own list (ListIntersectProgram, a linear merge). */
int64_t or_triangle_count(uint64_t n, int64_t m, const uint32_t* src, const uint32_t* dst,
                          uint64_t* local, uint32_t* bad_src, uint32_t* bad_dst) {
  int found = 0;
  uint32_t bs = 0, bd = 0;
  for (int64_t e = 0; e < m; ++e)
    if (src[e] >= dst[e] &&
        (!found || src[e] < bs || (src[e] == bs && dst[e] < bd))) {
      found = 1;
      bs = src[e];
      bd = dst[e];
    }
  if (found) {
    if (bad_src) *bad_src = bs;
    if (bad_dst) *bad_dst = bd;
    return -1;
  }
  uint64_t* ptr = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n + 1));
  uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m ? m : 1));
  or_csr_build(n, m, dst, src, NULL, ptr, idx, NULL); /* rows = destinations */
  /* counting-sort CSR keeps input order: sort each list ascending */
  for (uint64_t v = 0; v < n; ++v) {
    uint32_t* a = idx + ptr[v];
    const uint64_t len = ptr[v + 1] - ptr[v];
    for (uint64_t i = 1; i < len; ++i) { /* insertion sort; lists are short in tests */
      const uint32_t x = a[i];
      uint64_t j = i;
      while (j > 0 && a[j - 1] > x) {
        a[j] = a[j - 1];
        --j;
      }
      a[j] = x;
    }
  }
  int64_t total = 0;
  for (uint64_t w = 0; w < n; ++w) {
    uint64_t cnt = 0;
    for (uint64_t k = ptr[w]; k < ptr[w + 1]; ++k) {
      const uint32_t v = idx[k];
      uint64_t a = ptr[v], ae = ptr[v + 1], b = ptr[w], be = ptr[w + 1];
      while (a < ae && b < be) {
        if (idx[a] < idx[b])
          ++a;
        else if (idx[b] < idx[a])
          ++b;
        else {
          ++cnt;
          ++a;
          ++b;
        }
      }
    }
    if (local) local[w] = cnt;
    total += (int64_t)cnt;
  }
  free(ptr);
  free(idx);
  return total;
}

void or_csr_build(uint64_t n, int64_t m, const uint32_t* row, const uint32_t* col,
                  const double* vals, uint64_t* ptr, uint32_t* idx, double* out_vals) {
  memset(ptr, 0, sizeof(uint64_t) * (size_t)(n + 1));
  for (int64_t e = 0; e < m; ++e) ++ptr[row[e] + 1];
  for (uint64_t v = 0; v < n; ++v) ptr[v + 1] += ptr[v];
  uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n ? n : 1));
  memcpy(fill, ptr, sizeof(uint64_t) * (size_t)n);
  for (int64_t e = 0; e < m; ++e) {
    const uint64_t pos = fill[row[e]]++;
    idx[pos] = col[e];
    if (vals && out_vals) out_vals[pos] = vals[e];
  }
  free(fill);
}

/* ------------------------------------------------------------- programs */

static void put_stats(or_stats* st, int64_t cap, int64_t it, int64_t active, int64_t msgs,
                      int64_t upd, double spmv_s, double total_s) {
  if (!st || it - 1 >= cap) return;
  or_stats* s = &st[it - 1];
  s->iteration = it;
  s->active_before = active;
  s->messages_generated = msgs;
  s->vertices_updated = upd;
  s->spmv_seconds = spmv_s;
  s->total_seconds = total_s;
}

/* BfsProgram (traversal.hpp:39-63) under run_distance_program (:95-115): the
 * frontier sends its level, receivers keep min(own, level+1); a receiver is
 * updated (and active next) iff its level dropped. Pushing over CSR(G) visits
 * the same (active source, destination) pairs as the pull over G^T. */
int64_t or_bfs(uint64_t n, const uint64_t* optr, const uint32_t* oidx, uint32_t root,
               int64_t max_iters, int32_t* level, or_stats* st, int64_t cap) {
  for (uint64_t v = 0; v < n; ++v) level[v] = -1;
  if (n == 0 || max_iters <= 0) return 0;
  level[root] = 0;
  uint32_t* fr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  uint32_t* nx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  int64_t nf = 1, it = 0;
  fr[0] = root;
  for (it = 1; it <= max_iters; ++it) {
    const double t0 = now_s();
    int64_t nn = 0;
    for (int64_t i = 0; i < nf; ++i) {
      const uint32_t u = fr[i];
      for (uint64_t e = optr[u]; e < optr[u + 1]; ++e) {
        const uint32_t v = oidx[e];
        if (level[v] < 0) {
          level[v] = (int32_t)it;
          nx[nn++] = v;
        }
      }
    }
    const double t1 = now_s();
    put_stats(st, cap, it, nf, nf, nn, t1 - t0, t1 - t0);
    uint32_t* t = fr;
    fr = nx;
    nx = t;
    nf = nn;
    if (nn == 0) break;
  }
  free(fr);
  free(nx);
  return it > max_iters ? max_iters : it;
}

/* SsspProgram (traversal.hpp:67-91): active vertices send their superstep-start
 * distance, receivers keep the min of (message + weight). */
int64_t or_sssp(uint64_t n, const uint64_t* optr, const uint32_t* oidx, const uint32_t* w,
                uint32_t root, int64_t max_iters, uint32_t* dist, or_stats* st, int64_t cap) {
  const uint64_t INF = 0xFFFFFFFFull;
  for (uint64_t v = 0; v < n; ++v) dist[v] = (uint32_t)INF;
  if (n == 0 || max_iters <= 0) return 0;
  dist[root] = 0;
  uint32_t* fr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  uint32_t* fx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n); /* message snapshot */
  uint32_t* touched = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  uint64_t* y = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  for (uint64_t v = 0; v < n; ++v) y[v] = ~0ull;
  int64_t nf = 1, it = 0;
  fr[0] = root;
  fx[0] = 0;
  for (it = 1; it <= max_iters; ++it) {
    const double t0 = now_s();
    int64_t nt = 0;
    for (int64_t i = 0; i < nf; ++i) {
      const uint32_t u = fr[i];
      const uint64_t xu = fx[i];
      for (uint64_t e = optr[u]; e < optr[u + 1]; ++e) {
        const uint32_t v = oidx[e];
        const uint64_t cand = xu + w[e];
        if (y[v] == ~0ull) touched[nt++] = v;
        if (cand < y[v]) y[v] = cand;
      }
    }
    const double t1 = now_s();
    int64_t nn = 0;
    for (int64_t i = 0; i < nt; ++i) {
      const uint32_t v = touched[i];
      if (y[v] < (uint64_t)dist[v]) {
        dist[v] = (uint32_t)y[v];
        fr[nn] = v; /* frontier array no longer read this superstep */
        fx[nn] = dist[v];
        ++nn;
      }
      y[v] = ~0ull;
    }
    const double t2 = now_s();
    put_stats(st, cap, it, nf, nf, nn, t1 - t0, t2 - t0);
    nf = nn;
    if (nn == 0) break;
  }
  free(fr);
  free(fx);
  free(touched);
  free(y);
  return it > max_iters ? max_iters : it;
}

int64_t or_sssp_f64(uint64_t n, const uint64_t* optr, const uint32_t* oidx, const double* w,
                    uint32_t root, int64_t max_iters, double* dist, or_stats* st, int64_t cap) {
  for (uint64_t v = 0; v < n; ++v) dist[v] = INFINITY;
  if (n == 0 || max_iters <= 0) return 0;
  dist[root] = 0.0;
  uint32_t* fr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  double* fx = (double*)malloc(sizeof(double) * (size_t)n);
  uint32_t* touched = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  uint8_t* yv = (uint8_t*)calloc((size_t)n, 1);
  int64_t nf = 1, it = 0;
  fr[0] = root;
  fx[0] = 0.0;
  for (it = 1; it <= max_iters; ++it) {
    const double t0 = now_s();
    int64_t nt = 0;
    for (int64_t i = 0; i < nf; ++i) {
      const uint32_t u = fr[i];
      for (uint64_t e = optr[u]; e < optr[u + 1]; ++e) {
        const uint32_t v = oidx[e];
        const double cand = fx[i] + w[e];
        if (!yv[v]) {
          yv[v] = 1;
          touched[nt++] = v;
          y[v] = INFINITY < cand ? INFINITY : cand; /* reduce(identity, r) */
        } else {
          y[v] = y[v] < cand ? y[v] : cand;
        }
      }
    }
    const double t1 = now_s();
    int64_t nn = 0;
    for (int64_t i = 0; i < nt; ++i) {
      const uint32_t v = touched[i];
      const double fresh = y[v] < dist[v] ? y[v] : dist[v];
      uint64_t a, b;
      memcpy(&a, &fresh, 8);
      memcpy(&b, &dist[v], 8);
      if (a != b) {
        dist[v] = fresh;
        fr[nn] = v;
        fx[nn] = fresh;
        ++nn;
      }
      yv[v] = 0;
    }
    const double t2 = now_s();
    put_stats(st, cap, it, nf, nf, nn, t1 - t0, t2 - t0);
    nf = nn;
    if (nn == 0) break;
  }
  free(fr);
  free(fx);
  free(touched);
  free(y);
  free(yv);
  return it > max_iters ? max_iters : it;
}

/* Normalised PageRank, restated through the engine phases: all vertices
 * active; non-dangling u sends rank/outdeg (pagerank.hpp:46-49 shape); each
 * receiver folds in ascending source order (engine.hpp:59-66); apply is
 * base + d*sum with base = (1-d)/N + d*D/N; un-messaged vertices take the
 * empty sum (collaborative_filtering.hpp:192-193 pattern). */
void or_pagerank_norm(uint64_t n, const uint64_t* iptr, const uint32_t* iidx,
                      const uint32_t* outdeg, double damping, int64_t iters, double* rank,
                      or_stats* st) {
  if (n == 0) return;
  const double nd = (double)n;
  for (uint64_t v = 0; v < n; ++v) rank[v] = 1.0 / nd;
  double* x = (double*)malloc(sizeof(double) * (size_t)n);
  double* fresh = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t it = 1; it <= iters; ++it) {
    const double t0 = now_s();
    double dangling = 0.0;
    int64_t msgs = 0;
    for (uint64_t u = 0; u < n; ++u) {
      if (outdeg[u] == 0) {
        dangling += rank[u];
      } else {
        x[u] = rank[u] / (double)outdeg[u];
        ++msgs;
      }
    }
    const double base = (1.0 - damping) / nd + damping * dangling / nd;
    const double t1 = now_s();
    int64_t upd = 0;
    for (uint64_t v = 0; v < n; ++v) {
      double sum = 0.0;
      int any = 0;
      for (uint64_t e = iptr[v]; e < iptr[v + 1]; ++e) {
        const uint32_t j = iidx[e];
        if (outdeg[j] == 0) continue;
        sum = any ? sum + x[j] : 0.0 + x[j];
        any = 1;
      }
      fresh[v] = base + damping * sum;
      if (any) {
        uint64_t a, b;
        memcpy(&a, &fresh[v], 8);
        memcpy(&b, &rank[v], 8);
        upd += a != b;
      }
    }
    const double t2 = now_s();
    memcpy(rank, fresh, sizeof(double) * (size_t)n);
    put_stats(st, iters, it, (int64_t)n, msgs, upd, t2 - t1, now_s() - t0);
  }
  free(x);
  free(fresh);
}

/* PageRankProgram (pagerank.hpp:36-63) + driver (:73-110), tolerance off. */
int64_t or_pagerank_ref(uint64_t n, const uint64_t* iptr, const uint32_t* iidx,
                        const uint32_t* outdeg, double r, int64_t iters, double* rank,
                        or_stats* st) {
  for (uint64_t v = 0; v < n; ++v) rank[v] = 1.0;
  if (n == 0) return 0;
  uint8_t* active = (uint8_t*)malloc((size_t)n);
  uint8_t* next = (uint8_t*)malloc((size_t)n);
  double* x = (double*)malloc(sizeof(double) * (size_t)n);
  double* fresh = (double*)malloc(sizeof(double) * (size_t)n);
  memset(active, 1, (size_t)n);
  int64_t it = 0;
  for (it = 1; it <= iters; ++it) {
    const double t0 = now_s();
    int64_t act = 0, msgs = 0;
    for (uint64_t u = 0; u < n; ++u) {
      act += active[u];
      if (active[u] && outdeg[u] > 0) {
        x[u] = rank[u] / (double)outdeg[u];
        ++msgs;
      }
    }
    const double t1 = now_s();
    int64_t upd = 0;
    memset(next, 0, (size_t)n);
    for (uint64_t v = 0; v < n; ++v) {
      double sum = 0.0;
      int any = 0;
      for (uint64_t e = iptr[v]; e < iptr[v + 1]; ++e) {
        const uint32_t j = iidx[e];
        if (!active[j] || outdeg[j] == 0) continue;
        sum = any ? sum + x[j] : 0.0 + x[j];
        any = 1;
      }
      fresh[v] = rank[v];
      if (!any) continue;
      const double f = r + (1.0 - r) * sum;
      uint64_t a, b;
      memcpy(&a, &f, 8);
      memcpy(&b, &rank[v], 8);
      if (a != b) {
        fresh[v] = f;
        next[v] = 1;
        ++upd;
      }
    }
    const double t2 = now_s();
    memcpy(rank, fresh, sizeof(double) * (size_t)n);
    uint8_t* t = active;
    active = next;
    next = t;
    put_stats(st, iters, it, act, msgs, upd, t2 - t1, now_s() - t0);
    if (upd == 0) break;
  }
  free(active);
  free(next);
  free(x);
  free(fresh);
  return it > iters ? iters : it;
}

/* One direction of CfGdProgram::process_message/reduce (collaborative_filtering.hpp:66-84)
 * folded over a CSR row in ascending source order. */
static int cf_fold_row(const uint64_t* ptr, const uint32_t* idx, const double* val, uint64_t v,
                       int64_t k, const double* f, double* acc, double* r) {
  int any = 0;
  const double* p = f + v * (uint64_t)k;
  for (uint64_t e = ptr[v]; e < ptr[v + 1]; ++e) {
    const double* q = f + (uint64_t)idx[e] * (uint64_t)k;
    double dot = 0.0;
    for (int64_t i = 0; i < k; ++i) dot += p[i] * q[i];
    const double err = val[e] - dot;
    for (int64_t i = 0; i < k; ++i) r[i] = err * q[i];
    for (int64_t i = 0; i < k; ++i) acc[i] = any ? acc[i] + r[i] : 0.0 + r[i];
    any = 1;
  }
  return any;
}

void or_cf_gd(uint64_t n, const uint64_t* tptr, const uint32_t* tidx, const double* tval,
              const uint64_t* fptr, const uint32_t* fidx, const double* fval, int64_t k,
              double gamma, double lambda, int64_t iters, double* factors,
              double* objective_trace, double* rmse_trace, int64_t* updated) {
  double* nf = (double*)malloc(sizeof(double) * (size_t)(n * (uint64_t)k + 1));
  double* yo = (double*)malloc(sizeof(double) * (size_t)k);
  double* yi = (double*)malloc(sizeof(double) * (size_t)k);
  double* r = (double*)malloc(sizeof(double) * (size_t)k);
  const int64_t m = n ? (int64_t)tptr[n] : 0;
  for (int64_t it = 0; it < iters; ++it) {
    int64_t upd = 0;
    for (uint64_t v = 0; v < n; ++v) {
      const int vo = cf_fold_row(tptr, tidx, tval, v, k, factors, yo, r);
      const int vi = cf_fold_row(fptr, fidx, fval, v, k, factors, yi, r);
      /* BOTH merge, out-route first (engine.hpp:118-126) */
      for (int64_t i = 0; i < k; ++i) {
        double s;
        if (vo && vi)
          s = yo[i] + yi[i];
        else if (vo)
          s = yo[i];
        else if (vi)
          s = yi[i];
        else
          s = 0.0;
        const double p = factors[v * (uint64_t)k + (uint64_t)i];
        nf[v * (uint64_t)k + (uint64_t)i] = p + gamma * (s - lambda * p);
      }
      /* apply_and_activate counts messaged vertices whose LatentVector changed
       * bitwise (engine.hpp:139-172, collaborative_filtering.hpp:29-35, 189) */
      if (vo || vi)
        upd += memcmp(nf + v * (uint64_t)k, factors + v * (uint64_t)k, sizeof(double) * (size_t)k) != 0;
    }
    if (updated) updated[it] = upd;
    memcpy(factors, nf, sizeof(double) * (size_t)(n * (uint64_t)k));
    /* cf_objective_value (collaborative_filtering.hpp:103-123): ratings grouped
     * by user (column of G^T), ascending. */
    double sq = 0.0, reg = 0.0;
    for (uint64_t u = 0; u < n; ++u) {
      for (uint64_t e = fptr[u]; e < fptr[u + 1]; ++e) {
        const uint64_t it2 = fidx[e];
        double dot = 0.0;
        for (int64_t d = 0; d < k; ++d)
          dot += factors[u * (uint64_t)k + (uint64_t)d] * factors[it2 * (uint64_t)k + (uint64_t)d];
        const double err = fval[e] - dot;
        sq += err * err;
      }
    }
    for (uint64_t v = 0; v < n * (uint64_t)k; ++v) reg += lambda * factors[v] * factors[v];
    if (objective_trace) objective_trace[it] = sq + reg;
    if (rmse_trace) rmse_trace[it] = m ? sqrt(sq / (double)m) : 0.0;
  }
  free(nf);
  free(yo);
  free(yi);
  free(r);
}

static int cf_fold_row_f32(const uint64_t* ptr, const uint32_t* idx, const double* val,
                           uint64_t v, int64_t k, const float* f, float* acc, float* r) {
  int any = 0;
  const float* p = f + v * (uint64_t)k;
  for (uint64_t e = ptr[v]; e < ptr[v + 1]; ++e) {
    const float* q = f + (uint64_t)idx[e] * (uint64_t)k;
    float dot = 0.0f;
    for (int64_t i = 0; i < k; ++i) dot += p[i] * q[i];
    const float err = (float)val[e] - dot;
    for (int64_t i = 0; i < k; ++i) r[i] = err * q[i];
    for (int64_t i = 0; i < k; ++i) acc[i] = any ? acc[i] + r[i] : r[i];
    any = 1;
  }
  return any;
}

void or_cf_gd_f32(uint64_t n, const uint64_t* tptr, const uint32_t* tidx, const double* tval,
                  const uint64_t* fptr, const uint32_t* fidx, const double* fval, int64_t k,
                  float gamma, float lambda, int64_t iters, float* factors,
                  double* rmse_trace, int64_t* updated) {
  float* nf = (float*)malloc(sizeof(float) * (size_t)(n * (uint64_t)k + 1));
  float* yo = (float*)malloc(sizeof(float) * (size_t)k);
  float* yi = (float*)malloc(sizeof(float) * (size_t)k);
  float* r = (float*)malloc(sizeof(float) * (size_t)k);
  const int64_t m = n ? (int64_t)tptr[n] : 0;
  for (int64_t it = 0; it < iters; ++it) {
    int64_t upd = 0;
    for (uint64_t v = 0; v < n; ++v) {
      const int vo = cf_fold_row_f32(tptr, tidx, tval, v, k, factors, yo, r);
      const int vi = cf_fold_row_f32(fptr, fidx, fval, v, k, factors, yi, r);
      for (int64_t i = 0; i < k; ++i) {
        float s = 0.0f;
        if (vo) s += yo[i];
        if (vi) s += yi[i];
        const float p = factors[v * (uint64_t)k + (uint64_t)i];
        nf[v * (uint64_t)k + (uint64_t)i] = p + gamma * (s - lambda * p);
      }
      if (vo || vi)
        upd += memcmp(nf + v * (uint64_t)k, factors + v * (uint64_t)k, sizeof(float) * (size_t)k) != 0;
    }
    if (updated) updated[it] = upd;
    memcpy(factors, nf, sizeof(float) * (size_t)(n * (uint64_t)k));
    double sq = 0.0;
    for (uint64_t u = 0; u < n; ++u) {
      for (uint64_t e = fptr[u]; e < fptr[u + 1]; ++e) {
        const uint64_t it2 = fidx[e];
        double dot = 0.0;
        for (int64_t d = 0; d < k; ++d)
          dot += (double)factors[u * (uint64_t)k + (uint64_t)d] *
                 (double)factors[it2 * (uint64_t)k + (uint64_t)d];
        const double err = fval[e] - dot;
        sq += err * err;
      }
    }
    if (rmse_trace) rmse_trace[it] = m ? sqrt(sq / (double)m) : 0.0;
  }
  free(nf);
  free(yo);
  free(yi);
  free(r);
}

void or_semiring_spmv(uint64_t n, const uint64_t* iptr, const uint32_t* iidx,
                      const int64_t* vals, const int64_t* x, const uint8_t* xvalid, int64_t* y,
                      uint8_t* yvalid) {
  for (uint64_t k = 0; k < n; ++k) {
    int64_t acc = 0;
    int any = 0;
    for (uint64_t e = iptr[k]; e < iptr[k + 1]; ++e) {
      const uint32_t j = iidx[e];
      if (!xvalid[j]) continue;
      acc += vals[e] * x[j];
      any = 1;
    }
    y[k] = any ? acc : 0;
    yvalid[k] = (uint8_t)any;
  }
}
