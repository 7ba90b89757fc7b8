/*
 * knnd_oracle.c — plain C restatement of the reference's per-round hot path.
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/ as the checker for the CUDA path,
 * by __graft_entry__.smoke() and by bench.py's CPU-baseline / reference arm.
 * Never linked into or called by the product package.
 *
 * Restates (paths relative to /root/reference/pkg/src/rankdescent/):
 *   oracle_transpose   descent.py:151-160  _transpose_csr (stable: sources
 *                                          ascending within each target)
 *   oracle_local_join  descent.py:230-242  _propose_scored, with the tallies of
 *                      descent.py:273-278 (comparisons += |U|, changed if the
 *                      row differs order-sensitively)
 *   oracle_fcc         descent.py:334-337  adjacency count of the sampled pairs
 *   oracle_sort_rows   descent.py:163-170  stable sort of each row by score
 *   oracle_exact_rows  evaluation.py:86-90 brute-force K smallest (score, id)
 * Scores follow similarity.py:101-106, D = xlogx[x] - sum_j log[y,j]*x[j], in
 * fp64 with a left-to-right sum (the reference's einsum order is numpy's own;
 * the two agree to ~1e-15 relative).  log and xlogx are passed in, computed
 * by numpy exactly as similarity.py:92-93 does.
 *
 * Anchors are independent (descent.py:282-288), so the loops run under
 * OpenMP with a per-thread scratch; results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* metric 0: KL (similarity.py:101-106), lg = log(points), xlogx = row entropies.
 * metric 1: squared Euclidean (similarity.py:135-140), pts = lg = the vectors,
 *           xlogx = their squared norms: max(sq[x] + sq[y] - 2 y.x, 0). */
static double score(const double *pts, const double *lg, const double *xlogx, int d, int64_t x, int64_t y,
                    int metric) {
  const double *px = pts + x * d, *ly = lg + y * d;
  double acc = 0.0;
  for (int j = 0; j < d; ++j) acc += ly[j] * px[j];
  if (metric == 1) {
    const double d2 = (xlogx[x] + xlogx[y]) - 2.0 * acc;
    return d2 > 0.0 ? d2 : 0.0;
  }
  return xlogx[x] - acc;
}

/* (score, id) strict order — core.py:83-90 */
static int key_lt(double sa, int64_t ia, double sb, int64_t ib) { return sa < sb || (sa == sb && ia < ib); }

/* LSD radix sort of uint32 keys, 8-bit digits */
static void radix_sort_u32(uint32_t *a, uint32_t *tmp, int64_t m) {
  uint32_t *src = a, *dst = tmp;
  for (int shift = 0; shift < 32; shift += 8) {
    int64_t cnt[257];
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < m; ++i) cnt[((src[i] >> shift) & 255u) + 1]++;
    if (cnt[1] == m) continue; /* every key has digit 0 here */
    for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
    for (int64_t i = 0; i < m; ++i) dst[cnt[(src[i] >> shift) & 255u]++] = src[i];
    uint32_t *t = src;
    src = dst;
    dst = t;
  }
  if (src != a) memcpy(a, src, (size_t)m * sizeof(uint32_t));
}

void oracle_transpose(const int32_t *F, int64_t n, int k, int64_t *indptr, int32_t *indices) {
  memset(indptr, 0, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t e = 0; e < n * k; ++e) indptr[F[e] + 1]++;
  for (int64_t t = 0; t < n; ++t) indptr[t + 1] += indptr[t];
  int64_t *cur = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  memcpy(cur, indptr, (size_t)n * sizeof(int64_t));
  for (int64_t e = 0; e < n * k; ++e) indices[cur[F[e]]++] = (int32_t)(e / k);
  free(cur);
}

typedef struct {
  uint32_t *ids, *tmp;
  double *s;
  int64_t cap;
} scratch_t;

static void scratch_fit(scratch_t *w, int64_t m) {
  if (m <= w->cap) return;
  free(w->ids);
  free(w->tmp);
  free(w->s);
  w->cap = m + m / 2 + 64;
  w->ids = (uint32_t *)malloc((size_t)w->cap * sizeof(uint32_t));
  w->tmp = (uint32_t *)malloc((size_t)w->cap * sizeof(uint32_t));
  w->s = (double *)malloc((size_t)w->cap * sizeof(double));
}

/* one anchor; returns |U|; writes the K best ids (and scores) */
static int64_t join_one(const double *pts, const double *lg, const double *xlogx, int d, int metric,
                        const int32_t *F, int k, const int64_t *indptr, const int32_t *indices, int64_t x,
                        scratch_t *w, int32_t *row, double *row_s) {
  const int64_t c0 = indptr[x], c = indptr[x + 1] - c0;
  const int64_t pre = (k + c) * (int64_t)(k + 1);
  scratch_fit(w, pre);
  int64_t m = 0;
  /* F(x), C(x), F(F(x)), F(C(x)) — descent.py:234 */
  for (int i = 0; i < k; ++i) w->ids[m++] = (uint32_t)F[x * k + i];
  for (int64_t i = 0; i < c; ++i) w->ids[m++] = (uint32_t)indices[c0 + i];
  for (int i = 0; i < k; ++i) {
    const int32_t *r = F + (int64_t)F[x * k + i] * k;
    for (int t = 0; t < k; ++t) w->ids[m++] = (uint32_t)r[t];
  }
  for (int64_t i = 0; i < c; ++i) {
    const int32_t *r = F + (int64_t)indices[c0 + i] * k;
    for (int t = 0; t < k; ++t) w->ids[m++] = (uint32_t)r[t];
  }
  /* np.unique, then drop x — descent.py:235-238 */
  radix_sort_u32(w->ids, w->tmp, m);
  int64_t u = 0;
  for (int64_t i = 0; i < m; ++i) {
    if ((int64_t)w->ids[i] == x) continue;
    if (u > 0 && w->ids[u - 1] == w->ids[i]) continue;
    w->ids[u++] = w->ids[i];
  }
  /* scores, then the K smallest (score, id) — descent.py:239-242 */
  int nb = 0;
  double bs[64];
  int64_t bi[64];
  for (int64_t i = 0; i < u; ++i) {
    const int64_t y = w->ids[i];
    const double s = score(pts, lg, xlogx, d, x, y, metric);
    if (nb == k && !key_lt(s, y, bs[k - 1], bi[k - 1])) continue;
    int p = nb < k ? nb++ : k - 1;
    while (p > 0 && key_lt(s, y, bs[p - 1], bi[p - 1])) {
      bs[p] = bs[p - 1];
      bi[p] = bi[p - 1];
      --p;
    }
    bs[p] = s;
    bi[p] = y;
  }
  for (int i = 0; i < nb; ++i) {
    row[i] = (int32_t)bi[i];
    if (row_s) row_s[i] = bs[i];
  }
  for (int i = nb; i < k; ++i) {
    row[i] = -1;
    if (row_s) row_s[i] = INFINITY;
  }
  return u;
}

/* anchors[0..na) -> out rows i*k..; tally[0] += sum |U|, tally[1] += changed */
int oracle_local_join(const double *pts, const double *lg, const double *xlogx, int64_t n, int d, int metric,
                      const int32_t *F, int k, const int64_t *indptr, const int32_t *indices, const int64_t *anchors,
                      int64_t na, int32_t *out, double *out_kl, int32_t *ucount, int64_t *tally, int nthreads) {
  (void)n;
  if (k < 1 || k > 64) return -1;
  int64_t comps = 0, changed = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads) reduction(+ : comps, changed)
#endif
  {
    scratch_t w = {0, 0, 0, 0};
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 256)
#endif
    for (int64_t a = 0; a < na; ++a) {
      const int64_t x = anchors[a];
      int32_t *row = out + a * k;
      int64_t u =
          join_one(pts, lg, xlogx, d, metric, F, k, indptr, indices, x, &w, row, out_kl ? out_kl + a * k : 0);
      if (ucount) ucount[a] = (int32_t)u;
      comps += u;
      int diff = 0;
      for (int i = 0; i < k; ++i) diff |= row[i] != F[x * k + i];
      changed += diff;
    }
    free(w.ids);
    free(w.tmp);
    free(w.s);
  }
  if (tally) {
    tally[0] += comps;
    tally[1] += changed;
  }
  return 0;
}

int32_t oracle_fcc(const int32_t *F, int64_t n, int k, const int64_t *xs, const int64_t *is, const int64_t *js,
                   int64_t S) {
  (void)n;
  int32_t cnt = 0;
  for (int64_t s = 0; s < S; ++s) {
    const int32_t y = F[xs[s] * k + is[s]], z = F[xs[s] * k + js[s]];
    int adj = 0;
    for (int t = 0; t < k; ++t) adj |= (F[(int64_t)z * k + t] == y) | (F[(int64_t)y * k + t] == z);
    cnt += adj;
  }
  return cnt;
}

/* stable sort of each row by score: insertion sort keyed (score, position) */
void oracle_sort_rows(const double *pts, const double *lg, const double *xlogx, int64_t n, int d, int metric, int k,
                      const int32_t *draws, int32_t *out, int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(static)
#endif
  for (int64_t x = 0; x < n; ++x) {
    double s[64];
    int32_t id[64];
    for (int i = 0; i < k; ++i) {
      const int32_t y = draws[x * k + i];
      const double v = score(pts, lg, xlogx, d, x, y, metric);
      int p = i;
      while (p > 0 && v < s[p - 1]) { /* strict: equal scores keep draw order */
        s[p] = s[p - 1];
        id[p] = id[p - 1];
        --p;
      }
      s[p] = v;
      id[p] = y;
    }
    memcpy(out + x * k, id, (size_t)k * sizeof(int32_t));
  }
}

/* brute-force exact K-NN rows for the given queries (anchor excluded) */
void oracle_exact_rows(const double *pts, const double *lg, const double *xlogx, int64_t n, int d, int metric, int k,
                       const int64_t *queries, int64_t q, int32_t *out, int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 4)
#endif
  for (int64_t a = 0; a < q; ++a) {
    const int64_t x = queries[a];
    double bs[64];
    int64_t bi[64];
    int nb = 0;
    for (int64_t y = 0; y < n; ++y) {
      if (y == x) continue;
      const double s = score(pts, lg, xlogx, d, x, y, metric);
      if (nb == k && !key_lt(s, y, bs[k - 1], bi[k - 1])) continue;
      int p = nb < k ? nb++ : k - 1;
      while (p > 0 && key_lt(s, y, bs[p - 1], bi[p - 1])) {
        bs[p] = bs[p - 1];
        bi[p] = bi[p - 1];
        --p;
      }
      bs[p] = s;
      bi[p] = y;
    }
    for (int i = 0; i < k; ++i) out[a * k + i] = (int32_t)bi[i];
  }
}
