/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see mprof_oracle.h).
 *
 * Multivariate joins of the reference: SiMPle (non-normalised, summed over
 * dimensions) and mSTOMP (k-dimensional z-normalised profiles for every k),
 * restated from their header contracts and SPEC.md prose. Never linked into
 * the product. Series are dim-major: x[dim * n + t].
 */
#include "mprof_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_REFRESH_ROWS 4096

static int64_t mi64(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t ma64(int64_t a, int64_t b) { return a > b ? a : b; }

/* ------------------------------------------------------------ raw (SiMPle) */

/* raw_norms (distance.hpp:36-42): per-window sums of squares, one dimension. */
void or_raw_norms(const double *x, int64_t n, int64_t w, double *out) {
  const int64_t L = n - w + 1;
  for (int64_t i = 0; i < L; ++i) {
    double s = 0.0;
    for (int64_t k = 0; k < w; ++k) s += x[i + k] * x[i + k];
    out[i] = s;
  }
}

/* raw_sq_term (distance.hpp:51-52): one dimension's squared contribution,
 * clamped at 0. */
double or_raw_sq_term(double sumsq_a, double sumsq_b, double qt) {
  const double v = sumsq_a + sumsq_b - 2.0 * qt;
  return v > 0.0 ? v : 0.0;
}

/* raw_distance_from_terms (distance.hpp:54-57): relative snap of rounding
 * residue to exactly 0. The reference leaves the threshold open; this build
 * fixes dsq <= 1e-12 * scale. */
double or_raw_distance_from_terms(double dsq_total, double scale) {
  if (dsq_total <= OR_RAW_SNAP * scale) return 0.0;
  return sqrt(dsq_total);
}

/* Direct raw distance between window i of A and window j of B over all dims:
 * sqrt(sum (a - b)^2) with the same snap against the summed energies. */
double or_raw_direct(const double *a, int64_t n_a, const double *b, int64_t n_b, int64_t dims,
                     int64_t w, int64_t i, int64_t j) {
  double d2 = 0.0, sc = 0.0;
  for (int64_t d = 0; d < dims; ++d) {
    const double *x = a + d * n_a + i, *y = b + d * n_b + j;
    for (int64_t t = 0; t < w; ++t) {
      const double e = x[t] - y[t];
      d2 += e * e;
      sc += x[t] * x[t] + y[t] * y[t];
    }
  }
  return or_raw_distance_from_terms(d2, sc);
}

/* raw_distance_profile (distance.hpp:44-49): distances from
 * one multivariate query (dims x w, dim-major) to every window of ts. */
int or_raw_distance_profile(const double *query, const double *ts, int64_t n, int64_t dims,
                            int64_t w, double *out) {
  if (w < 1 || w > n || dims < 1) return -1;
  const int64_t L = n - w + 1;
  double *dsq = calloc((size_t)L, sizeof(double)), *sc = calloc((size_t)L, sizeof(double));
  double *nt = malloc(sizeof(double) * L);
  for (int64_t d = 0; d < dims; ++d) {
    const double *q = query + d * w, *x = ts + d * n;
    double nq = 0.0;
    for (int64_t k = 0; k < w; ++k) nq += q[k] * q[k];
    or_raw_norms(x, n, w, nt);
    for (int64_t i = 0; i < L; ++i) {
      double qt = 0.0;
      for (int64_t k = 0; k < w; ++k) qt += q[k] * x[i + k];
      dsq[i] += or_raw_sq_term(nq, nt[i], qt);
      sc[i] += nq + nt[i];
    }
  }
  for (int64_t i = 0; i < L; ++i) out[i] = or_raw_distance_from_terms(dsq[i], sc[i]);
  free(dsq); free(sc); free(nt);
  return 0;
}

typedef struct {
  double *v, *l, *r; /* snapped squared distances: profile, left, right */
  int64_t *pi, *left, *right;
} sacc_t;

/*
 * simple (profile.hpp:96-100): STOMP-style iteration where
 * each cell is the non-normalised Euclidean distance summed over all dims
 * (raw_distance_profile semantics). Rows are query windows of B (self: A),
 * columns windows of A; per dim QT[i][j] = QT[i-1][j-1] - b[i-1] a[j-1] +
 * b[i+w-1] a[j+w-1], refreshed directly every 4096 rows; the cell value is
 * raw_distance_from_terms(sum_d raw_sq_term(..), sum_d energies); merge_min
 * with strict improvement. Self-joins apply the zone and also fill left /
 * right (as stomp); AB-joins use zone 0. n_workers contiguous
 * row chunks on the refresh grid, merged in fixed order.
 * Rows [row_begin, row_end) only when row_end > row_begin (timing samples).
 */
int or_simple_join(const double *a, int64_t n_a, const double *b, int64_t n_b, int64_t dims,
                   int64_t w, double ez_fraction, int n_workers, int64_t row_begin,
                   int64_t row_end, double *mp, int64_t *pi, int64_t *left, int64_t *right) {
  const int self = (b == NULL);
  if (self) { b = a; n_b = n_a; }
  if (dims < 1 || w < 4 || w > n_a || w > n_b) return -1;
  const int64_t zone = self ? or_zone_size(w, ez_fraction) : 0;
  if (zone < 0) return -1;
  const int64_t La = n_a - w + 1, Lb = n_b - w + 1;
  if (n_workers < 1) n_workers = 1;
  const int sample = row_end > row_begin;
  if (!sample) { row_begin = 0; row_end = Lb; }
  if (row_begin < 0 || row_end > Lb) return -1;

  double *na = malloc(sizeof(double) * dims * La), *nb = na;
  for (int64_t d = 0; d < dims; ++d) or_raw_norms(a + d * n_a, n_a, w, na + d * La);
  if (!self) {
    nb = malloc(sizeof(double) * dims * Lb);
    for (int64_t d = 0; d < dims; ++d) or_raw_norms(b + d * n_b, n_b, w, nb + d * Lb);
  }
  sacc_t *acc = calloc((size_t)n_workers, sizeof(sacc_t));

#pragma omp parallel num_threads(n_workers)
  {
#ifdef _OPENMP
    const int wk = omp_get_thread_num();
#else
    const int wk = 0;
#endif
    int64_t r0, r1;
    if (sample) {
      r0 = row_begin + (row_end - row_begin) * wk / n_workers;
      r1 = row_begin + (row_end - row_begin) * (wk + 1) / n_workers;
    } else {
      const int64_t g0 = row_begin / OR_REFRESH_ROWS;
      const int64_t nblk = (row_end - 1) / OR_REFRESH_ROWS - g0 + 1;
      const int64_t b0 = g0 + nblk * wk / n_workers, b1 = g0 + nblk * (wk + 1) / n_workers;
      r0 = ma64(row_begin, b0 * OR_REFRESH_ROWS);
      r1 = mi64(row_end, b1 * OR_REFRESH_ROWS);
    }
    sacc_t A;
    A.v = malloc(sizeof(double) * La); A.l = malloc(sizeof(double) * La);
    A.r = malloc(sizeof(double) * La);
    A.pi = malloc(sizeof(int64_t) * La); A.left = malloc(sizeof(int64_t) * La);
    A.right = malloc(sizeof(int64_t) * La);
    for (int64_t j = 0; j < La; ++j) {
      A.v[j] = A.l[j] = A.r[j] = INFINITY;
      A.pi[j] = A.left[j] = A.right[j] = -1;
    }
    double *qt = malloc(sizeof(double) * dims * La), *qn = malloc(sizeof(double) * dims * La);
    double *dsq = malloc(sizeof(double) * La), *sc = malloc(sizeof(double) * La);
    for (int64_t i = r0; i < r1; ++i) {
      for (int64_t d = 0; d < dims; ++d) {
        const double *ad = a + d * n_a, *bd = b + d * n_b;
        double *q = qt + d * La, *qq = qn + d * La;
        if (i == r0 || i % OR_REFRESH_ROWS == 0) {
          for (int64_t j = 0; j < La; ++j) {
            double s = 0.0;
            for (int64_t k = 0; k < w; ++k) s += bd[i + k] * ad[j + k];
            q[j] = s;
          }
        } else {
          const double bo = bd[i - 1], bn = bd[i + w - 1];
          for (int64_t j = La - 1; j >= 1; --j) qq[j] = q[j - 1] - bo * ad[j - 1] + bn * ad[j + w - 1];
          double s = 0.0;
          for (int64_t k = 0; k < w; ++k) s += bd[i + k] * ad[k];
          qq[0] = s;
          memcpy(q, qq, sizeof(double) * La);
        }
      }
      for (int64_t j = 0; j < La; ++j) { dsq[j] = 0.0; sc[j] = 0.0; }
      for (int64_t d = 0; d < dims; ++d) {
        const double nbi = nb[d * Lb + i];
        const double *q = qt + d * La, *nad = na + d * La;
        for (int64_t j = 0; j < La; ++j) {
          dsq[j] += or_raw_sq_term(nbi, nad[j], q[j]);
          sc[j] += nbi + nad[j];
        }
      }
      for (int64_t j = 0; j < La; ++j) {
        if (self && (j - i <= zone && i - j <= zone)) continue; /* apply_exclusion_zone */
        const double dv = or_raw_distance_from_terms(dsq[j], sc[j]);
        const double v = dv * dv;
        if (v < A.v[j]) { A.v[j] = v; A.pi[j] = i; }
        if (self) {
          if (j < i) { if (v < A.r[j]) { A.r[j] = v; A.right[j] = i; } }
          else if (v < A.l[j]) { A.l[j] = v; A.left[j] = i; }
        }
      }
    }
    free(qt); free(qn); free(dsq); free(sc);
    acc[wk] = A;
  }
  for (int64_t j = 0; j < La; ++j) {
    double v = INFINITY, l = INFINITY, r = INFINITY;
    int64_t p = -1, li = -1, ri = -1;
    for (int q = 0; q < n_workers; ++q) {
      if (acc[q].v[j] < v) { v = acc[q].v[j]; p = acc[q].pi[j]; }
      if (acc[q].l[j] < l) { l = acc[q].l[j]; li = acc[q].left[j]; }
      if (acc[q].r[j] < r) { r = acc[q].r[j]; ri = acc[q].right[j]; }
    }
    mp[j] = sqrt(v);
    pi[j] = p;
    if (left) left[j] = self ? li : -1;
    if (right) right[j] = self ? ri : -1;
  }
  for (int q = 0; q < n_workers; ++q) {
    free(acc[q].v); free(acc[q].l); free(acc[q].r);
    free(acc[q].pi); free(acc[q].left); free(acc[q].right);
  }
  free(acc);
  if (!self) free(nb);
  free(na);
  return 0;
}

/* Brute force SiMPle (oracle of the oracle): direct raw distances. */
int or_simple_brute(const double *a, int64_t n_a, const double *b, int64_t n_b, int64_t dims,
                    int64_t w, double ez_fraction, double *mp, int64_t *pi, int n_threads) {
  const int self = (b == NULL);
  if (self) { b = a; n_b = n_a; }
  if (dims < 1 || w < 4 || w > n_a || w > n_b) return -1;
  const int64_t zone = self ? or_zone_size(w, ez_fraction) : 0;
  const int64_t La = n_a - w + 1, Lb = n_b - w + 1;
  (void)n_threads;
#pragma omp parallel for schedule(dynamic, 16) num_threads(n_threads > 0 ? n_threads : 1)
  for (int64_t j = 0; j < La; ++j) {
    double best = INFINITY;
    int64_t bi = -1;
    for (int64_t i = 0; i < Lb; ++i) {
      if (self && (j - i <= zone && i - j <= zone)) continue;
      const double v = or_raw_direct(a, n_a, b, n_b, dims, w, j, i);
      if (v < best) { best = v; bi = i; }
    }
    mp[j] = best;
    pi[j] = bi;
  }
  return 0;
}

/* ------------------------------------------------------------------ mSTOMP */

/* Admissible dimension order: must dims (ascending index) then free dims
 * (ascending index), excluded dims dropped. Returns the count or -1 on a
 * parameter error (overlap, |exc| = d, invalid or repeated
 * dims). */
int64_t or_mstomp_dim_order(int64_t dims, const int64_t *must, int64_t n_must,
                            const int64_t *exc, int64_t n_exc, int64_t *order,
                            int64_t *n_must_out) {
  if (dims < 1) return -1;
  char *tag = calloc((size_t)dims, 1); /* 1 must, 2 exc */
  int64_t rc = 0;
  for (int64_t q = 0; q < n_must && rc == 0; ++q) {
    if (must[q] < 0 || must[q] >= dims || tag[must[q]]) rc = -1; else tag[must[q]] = 1;
  }
  for (int64_t q = 0; q < n_exc && rc == 0; ++q) {
    if (exc[q] < 0 || exc[q] >= dims || tag[exc[q]]) rc = -1; else tag[exc[q]] = 2;
  }
  if (rc == 0 && n_exc >= dims) rc = -1;
  int64_t c = 0;
  if (rc == 0) {
    for (int64_t d = 0; d < dims; ++d) if (tag[d] == 1) order[c++] = d;
    for (int64_t d = 0; d < dims; ++d) if (tag[d] == 0) order[c++] = d;
    if (n_must_out) *n_must_out = n_must;
  }
  free(tag);
  return rc == 0 ? c : -1;
}

/* Per-cell selection: sort the admissible per-dimension
 * distances ascending with the must dims forced to the front (ascending among
 * themselves), ties by position in `order` (stable); prefix means. slot[k] is
 * the dimension filling slot k, pk[k] the mean of the k+1 first. */
void or_mstomp_select(const double *dist, int64_t D, int64_t n_must, const int64_t *order,
                      int64_t *slot, double *pk) {
  int64_t idx[64];
  for (int64_t q = 0; q < D; ++q) idx[q] = q;
  /* stable insertion sort of [0, n_must) and [n_must, D) separately */
  for (int part = 0; part < 2; ++part) {
    const int64_t lo = part == 0 ? 0 : n_must, hi = part == 0 ? n_must : D;
    for (int64_t q = lo + 1; q < hi; ++q) {
      const int64_t v = idx[q];
      int64_t p = q - 1;
      while (p >= lo && dist[idx[p]] > dist[v]) { idx[p + 1] = idx[p]; --p; }
      idx[p + 1] = v;
    }
  }
  double s = 0.0;
  for (int64_t k = 0; k < D; ++k) {
    s += dist[idx[k]];
    pk[k] = s / (double)(k + 1);
    slot[k] = order[idx[k]];
  }
}

typedef struct {
  double *v;        /* [D][L] */
  int64_t *pi, *dim;
} macc_t;

/*
 * mstomp (profile.hpp:91-94): self-join. Per query
 * row i and admissible dimension, the z-normalised distance profile by the
 * STOMP recurrence (QT per dim, refreshed every 4096 rows, distance as in
 * or_stomp: znorm_dist_from_qt with the flat-window convention); per column j
 * the selection above, and row k (k < D) min-merges the mean of the k+1 first
 * with strict improvement, recording the dimension that filled slot k. Rows
 * k >= D repeat row D-1 with dim_order -1 (an exhausted selection). Near-zero
 * values are recomputed from direct distances at the chosen pair (as stomp's
 * near-zero convention). Outputs are dims x L (row k = (k+1)-dim profile).
 * Returns 0, -1 (bad window) or -2 (bad must / exc dims).
 */
int or_mstomp(const double *x, int64_t n, int64_t dims, int64_t w, double ez_fraction,
              const int64_t *must, int64_t n_must, const int64_t *exc, int64_t n_exc,
              int n_workers, int64_t row_begin, int64_t row_end, double *mp, int64_t *pi,
              int64_t *dim_order) {
  if (w < 4 || w > n) return -1;
  int64_t order[64], nm = 0;
  if (dims > 64) return -2;
  const int64_t D = or_mstomp_dim_order(dims, must, n_must, exc, n_exc, order, &nm);
  if (D < 1) return -2;
  const int64_t zone = or_zone_size(w, ez_fraction);
  if (zone < 0) return -1;
  const int64_t L = n - w + 1;
  if (n_workers < 1) n_workers = 1;
  const int sample = row_end > row_begin;
  if (!sample) { row_begin = 0; row_end = L; }
  if (row_begin < 0 || row_end > L) return -1;
  const double wd = (double)w;

  /* per admissible dim: globally centred copy, window means (centred), stds */
  double *xc = malloc(sizeof(double) * D * n), *mu = malloc(sizeof(double) * D * L);
  double *sd = malloc(sizeof(double) * D * L), *isd = malloc(sizeof(double) * D * L);
  double *mu_raw = malloc(sizeof(double) * L);
  for (int64_t q = 0; q < D; ++q) {
    const double *xd = x + order[q] * n;
    double g = 0.0;
    for (int64_t t = 0; t < n; ++t) g += xd[t];
    g /= (double)n;
    for (int64_t t = 0; t < n; ++t) xc[q * n + t] = xd[t] - g;
    or_rolling_mean_std(xd, n, w, mu_raw, sd + q * L, 1);
    for (int64_t j = 0; j < L; ++j) {
      mu[q * L + j] = mu_raw[j] - g;
      isd[q * L + j] = sd[q * L + j] == 0.0 ? 0.0 : 1.0 / sd[q * L + j];
    }
  }
  free(mu_raw);
  macc_t *acc = calloc((size_t)n_workers, sizeof(macc_t));

#pragma omp parallel num_threads(n_workers)
  {
#ifdef _OPENMP
    const int wk = omp_get_thread_num();
#else
    const int wk = 0;
#endif
    int64_t r0, r1;
    if (sample) {
      r0 = row_begin + (row_end - row_begin) * wk / n_workers;
      r1 = row_begin + (row_end - row_begin) * (wk + 1) / n_workers;
    } else {
      const int64_t g0 = row_begin / OR_REFRESH_ROWS;
      const int64_t nblk = (row_end - 1) / OR_REFRESH_ROWS - g0 + 1;
      const int64_t b0 = g0 + nblk * wk / n_workers, b1 = g0 + nblk * (wk + 1) / n_workers;
      r0 = ma64(row_begin, b0 * OR_REFRESH_ROWS);
      r1 = mi64(row_end, b1 * OR_REFRESH_ROWS);
    }
    macc_t A;
    A.v = malloc(sizeof(double) * D * L);
    A.pi = malloc(sizeof(int64_t) * D * L);
    A.dim = malloc(sizeof(int64_t) * D * L);
    for (int64_t e = 0; e < D * L; ++e) { A.v[e] = INFINITY; A.pi[e] = -1; A.dim[e] = -1; }
    double *qt = malloc(sizeof(double) * D * L), *qn = malloc(sizeof(double) * L);
    double dist[64], pk[64];
    int64_t slot[64];
    for (int64_t i = r0; i < r1; ++i) {
      for (int64_t q = 0; q < D; ++q) {
        const double *xd = xc + q * n;
        double *qq = qt + q * L;
        if (i == r0 || i % OR_REFRESH_ROWS == 0) {
          for (int64_t j = 0; j < L; ++j) {
            double s = 0.0;
            for (int64_t k = 0; k < w; ++k) s += xd[i + k] * xd[j + k];
            qq[j] = s;
          }
        } else {
          const double bo = xd[i - 1], bn = xd[i + w - 1];
          for (int64_t j = 1; j < L; ++j) qn[j] = qq[j - 1] - bo * xd[j - 1] + bn * xd[j + w - 1];
          double s = 0.0;
          for (int64_t k = 0; k < w; ++k) s += xd[i + k] * xd[k];
          qn[0] = s;
          memcpy(qq, qn, sizeof(double) * L);
        }
      }
      for (int64_t j = 0; j < L; ++j) {
        if (j - i <= zone && i - j <= zone) continue; /* apply_exclusion_zone */
        for (int64_t q = 0; q < D; ++q) {
          const double si = sd[q * L + i], sj = sd[q * L + j];
          double d2;
          if (si != 0.0 && sj != 0.0) {
            d2 = 2.0 * wd * (1.0 - (qt[q * L + j] - wd * mu[q * L + i] * mu[q * L + j]) /
                                       (wd * si) * isd[q * L + j]);
            d2 = d2 < 0.0 ? 0.0 : (d2 > 4.0 * wd ? 4.0 * wd : d2);
          } else {
            d2 = (si == 0.0 && sj == 0.0) ? 0.0 : wd; /* distance.hpp:14-15 */
          }
          dist[q] = sqrt(d2);
        }
        or_mstomp_select(dist, D, nm, order, slot, pk);
        for (int64_t k = 0; k < D; ++k) {
          const int64_t e = k * L + j;
          if (pk[k] < A.v[e]) { A.v[e] = pk[k]; A.pi[e] = i; A.dim[e] = slot[k]; }
        }
      }
    }
    free(qt); free(qn);
    acc[wk] = A;
  }
  double dist[64], pk[64];
  int64_t slot[64];
  for (int64_t k = 0; k < dims; ++k) {
    const int64_t kk = k < D ? k : D - 1;
    for (int64_t j = 0; j < L; ++j) {
      double v = INFINITY;
      int64_t p = -1, dm = -1;
      for (int q = 0; q < n_workers; ++q) {
        const int64_t e = kk * L + j;
        if (acc[q].v[e] < v) { v = acc[q].v[e]; p = acc[q].pi[e]; dm = acc[q].dim[e]; }
      }
      if (p >= 0 && v < 1e-3) { /* near-zero: direct distances at the chosen pair */
        for (int64_t q = 0; q < D; ++q) {
          const double *xd = x + order[q] * n;
          const double mi = mu[q * L + p], mj = mu[q * L + j];
          const double si = sd[q * L + p], sj = sd[q * L + j];
          double d2;
          if (si != 0.0 && sj != 0.0) {
            double gsh = xd[0] - xc[q * n]; /* undo the centring of mu */
            double s = 0.0;
            for (int64_t t = 0; t < w; ++t) {
              const double e = (xd[p + t] - (mi + gsh)) / si - (xd[j + t] - (mj + gsh)) / sj;
              s += e * e;
            }
            d2 = s > 4.0 * wd ? 4.0 * wd : s;
          } else {
            d2 = (si == 0.0 && sj == 0.0) ? 0.0 : wd;
          }
          dist[q] = sqrt(d2);
        }
        or_mstomp_select(dist, D, nm, order, slot, pk);
        v = pk[kk];
      }
      mp[k * L + j] = v;
      pi[k * L + j] = p;
      if (dim_order) dim_order[k * L + j] = k < D ? dm : -1;
    }
  }
  for (int q = 0; q < n_workers; ++q) { free(acc[q].v); free(acc[q].pi); free(acc[q].dim); }
  free(acc);
  free(xc); free(mu); free(sd); free(isd);
  return 0;
}
