/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see mprof_oracle.h).
 *
 * Restates the reference matrix-profile hot path on the CPU so that tests and
 * the bench's CPU baseline can check / time it. Never linked into the product.
 * Each function cites the reference contract it follows.
 */
#include "mprof_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_FLAT_REL 1e-10
#define OR_REFRESH_ROWS 4096 /* QT refreshed every 4096 rows */

static int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

/* distance.hpp:19-20; SPEC.md:110-118 (50*1/2 -> 25, 80*1/2 -> 40, 50*1/4 -> 13). */
int64_t or_zone_size(int64_t window, double fraction) {
  if (!(fraction >= 0.0)) return -1;
  return (int64_t)floor((double)window * fraction + 0.5);
}

/* rolling.hpp:21-23: flat if sd is below a threshold relative to |mean|. */
int or_is_flat_std(double sd, double mean) {
  double scale = fabs(mean) > 1.0 ? fabs(mean) : 1.0;
  return sd <= OR_FLAT_REL * scale;
}

/* rolling.hpp:25-29 / SPEC.md:70-78: population statistics per window. */
int or_rolling_mean_std(const double *ts, int64_t n, int64_t w, double *means, double *stds,
                        int n_threads) {
  if (w < 4 || w > n) return -1;
  const int64_t L = n - w + 1;
  (void)n_threads;
#pragma omp parallel for schedule(static) num_threads(n_threads > 0 ? n_threads : 1)
  for (int64_t i = 0; i < L; ++i) {
    const double *x = ts + i;
    double s = 0.0;
    for (int64_t k = 0; k < w; ++k) s += x[k];
    const double mu = s / (double)w;
    double ss = 0.0;
    for (int64_t k = 0; k < w; ++k) {
      const double d = x[k] - mu;
      ss += d * d;
    }
    double sd = sqrt(ss / (double)w);
    if (or_is_flat_std(sd, mu)) sd = 0.0; /* floor to exactly 0, rolling.hpp:26-28 */
    means[i] = mu;
    stds[i] = sd;
  }
  return 0;
}

/* distance.hpp:12-17 and SPEC.md "Flat-window convention" / "Distance clamping". */
double or_znorm_dist_from_qt(double qt, int64_t w, double mu_a, double sd_a, double mu_b,
                             double sd_b) {
  const int fa = sd_a == 0.0, fb = sd_b == 0.0;
  if (fa && fb) return 0.0;
  if (fa || fb) return sqrt((double)w);
  const double wd = (double)w;
  double d2 = 2.0 * wd * (1.0 - (qt - wd * mu_a * mu_b) / (wd * sd_a * sd_b));
  if (d2 < 0.0) d2 = 0.0;
  if (d2 > 4.0 * wd) d2 = 4.0 * wd;
  return sqrt(d2);
}

/* fft.hpp:64-66. */
int or_sliding_dot_direct(const double *q, int64_t w, const double *ts, int64_t n, double *out) {
  if (w < 1 || w > n) return -1;
  for (int64_t i = 0; i + w <= n; ++i) {
    double s = 0.0;
    for (int64_t k = 0; k < w; ++k) s += q[k] * ts[i + k];
    out[i] = s;
  }
  return 0;
}

/* apply_exclusion_zone_inplace (distance.hpp:22-24):
 * |i - center| <= zone -> +inf. */
void or_apply_exclusion_zone(double *dp, int64_t len, int64_t center, int64_t zone) {
  const int64_t lo = imax64(0, center - zone), hi = imin64(len - 1, center + zone);
  for (int64_t i = lo; i <= hi; ++i) dp[i] = INFINITY;
}

/* merge_min (profile.hpp:66-68). */
void or_merge_min(double *acc, int64_t *acc_idx, const double *dp, int64_t len,
                  int64_t source_index) {
  for (int64_t i = 0; i < len; ++i) {
    if (dp[i] < acc[i]) {
      acc[i] = dp[i];
      acc_idx[i] = source_index;
    }
  }
}

/* ---------------------------------------------------------------- brute force */

/* Direct z-normalised Euclidean distance between two windows (SPEC.md:185-193:
 * "direct per-window normalization"), with the flat-window convention. */
static double direct_dist(const double *x, double mx, double sx, const double *y, double my,
                          double sy, int64_t w) {
  const int fx = sx == 0.0, fy = sy == 0.0;
  if (fx && fy) return 0.0;
  if (fx || fy) return sqrt((double)w);
  const double ix = 1.0 / sx, iy = 1.0 / sy;
  double s = 0.0;
  for (int64_t k = 0; k < w; ++k) {
    const double d = (x[k] - mx) * ix - (y[k] - my) * iy;
    s += d * d;
  }
  if (s > 4.0 * (double)w) s = 4.0 * (double)w;
  return sqrt(s);
}

typedef struct {
  const double *a, *b;
  const double *ma, *sa, *mb, *sb;
  int64_t w, La, Lb, zone;
  int self;
} bf_ctx;

/* One profile position: distances from window i of a to every window of b
 * (b == a for self-join), exclusion zone |i-j| <= zone (distance.hpp:22-24),
 * min with the smallest index on ties (first in scan order). */
static void bf_row(const bf_ctx *c, int64_t i, double *mp, int64_t *pi, int64_t *left,
                   int64_t *right) {
  double best = INFINITY, bl = INFINITY, br = INFINITY;
  int64_t bi = -1, li = -1, ri = -1;
  for (int64_t j = 0; j < c->Lb; ++j) {
    if (c->self && llabs(i - j) <= c->zone) continue;
    const double d =
        direct_dist(c->a + i, c->ma[i], c->sa[i], c->b + j, c->mb[j], c->sb[j], c->w);
    if (d < best) { best = d; bi = j; }
    if (c->self) {
      if (j < i && d < bl) { bl = d; li = j; }
      if (j > i && d < br) { br = d; ri = j; }
    }
  }
  *mp = best;
  *pi = bi;
  if (left) *left = li;
  if (right) *right = ri;
}

static int bf_setup(bf_ctx *c, const double *a, int64_t n_a, const double *b, int64_t n_b,
                    int64_t w, double ez, int n_threads) {
  memset(c, 0, sizeof(*c));
  c->self = (b == NULL);
  if (c->self) { b = a; n_b = n_a; }
  if (w < 4 || w > n_a || w > n_b) return -1;
  c->a = a; c->b = b; c->w = w;
  c->La = n_a - w + 1; c->Lb = n_b - w + 1;
  c->zone = c->self ? or_zone_size(w, ez) : 0;
  if (c->zone < 0) return -1;
  double *ma = malloc(sizeof(double) * c->La), *sa = malloc(sizeof(double) * c->La);
  or_rolling_mean_std(a, n_a, w, ma, sa, n_threads);
  c->ma = ma; c->sa = sa;
  if (c->self) { c->mb = ma; c->sb = sa; }
  else {
    double *mb = malloc(sizeof(double) * c->Lb), *sb = malloc(sizeof(double) * c->Lb);
    or_rolling_mean_std(b, n_b, w, mb, sb, n_threads);
    c->mb = mb; c->sb = sb;
  }
  return 0;
}

static void bf_free(bf_ctx *c) {
  free((void *)c->ma); free((void *)c->sa);
  if (!c->self) { free((void *)c->mb); free((void *)c->sb); }
}

/* profile.hpp:70-73 */
int or_brute_force_mp(const double *a, int64_t n_a, const double *b, int64_t n_b, int64_t w,
                      double ez_fraction, double *mp, int64_t *pi, int64_t *left,
                      int64_t *right, int n_threads) {
  bf_ctx c;
  if (bf_setup(&c, a, n_a, b, n_b, w, ez_fraction, n_threads)) return -1;
#pragma omp parallel for schedule(dynamic, 16) num_threads(n_threads > 0 ? n_threads : 1)
  for (int64_t i = 0; i < c.La; ++i)
    bf_row(&c, i, mp + i, pi + i, left ? left + i : NULL, right ? right + i : NULL);
  bf_free(&c);
  return 0;
}

int or_brute_force_rows(const double *a, int64_t n_a, const double *b, int64_t n_b, int64_t w,
                        double ez_fraction, const int64_t *rows, int64_t n_rows, double *mp,
                        int64_t *pi, int64_t *left, int64_t *right, int n_threads) {
  bf_ctx c;
  if (bf_setup(&c, a, n_a, b, n_b, w, ez_fraction, n_threads)) return -1;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads > 0 ? n_threads : 1)
  for (int64_t r = 0; r < n_rows; ++r) {
    const int64_t i = rows[r];
    if (i < 0 || i >= c.La) { bad = 1; continue; }
    bf_row(&c, i, mp + r, pi + r, left ? left + r : NULL, right ? right + r : NULL);
  }
  bf_free(&c);
  return bad ? -1 : 0;
}

/* mass_distance_profile (distance.hpp:26-33): distances from a
 * query window to every window of ts; the FFT dot products are replaced by the
 * exact direct z-normalised distance (which is also what the reference's
 * near-zero recompute falls back to). query_index >= 0: |i - query_index| <=
 * zone -> +inf (self queries, apply_exclusion_zone semantics). */
int or_mass_distance_profile(const double *query, int64_t w, const double *ts, int64_t n,
                             int64_t query_index, int64_t zone, double *out, int n_threads) {
  if (w < 4 || w > n) return -1;
  const int64_t L = n - w + 1;
  double qm = 0.0;
  for (int64_t k = 0; k < w; ++k) qm += query[k];
  qm /= (double)w;
  double qss = 0.0;
  for (int64_t k = 0; k < w; ++k) qss += (query[k] - qm) * (query[k] - qm);
  double qsd = sqrt(qss / (double)w);
  if (or_is_flat_std(qsd, qm)) qsd = 0.0;
  double *mu = malloc(sizeof(double) * L), *sd = malloc(sizeof(double) * L);
  or_rolling_mean_std(ts, n, w, mu, sd, n_threads);
#pragma omp parallel for schedule(static) num_threads(n_threads > 0 ? n_threads : 1)
  for (int64_t i = 0; i < L; ++i) {
    if (query_index >= 0 && llabs(i - query_index) <= zone) { out[i] = INFINITY; continue; }
    out[i] = direct_dist(query, qm, qsd, ts + i, mu[i], sd[i], w);
  }
  free(mu); free(sd);
  return 0;
}

/* ---------------------------------------------------------------- STOMP */

/* Direct QT row: qt[j] = sum_k q[k] * t[j+k] for the (globally centred)
 * series (the reference's FFT seed row, fft.hpp:49-50, replaced by the exact
 * direct path fft.hpp:64-66). */
static void qt_row_direct(const double *q, const double *t, int64_t L, int64_t w, double *qt) {
  for (int64_t j = 0; j < L; ++j) {
    double s = 0.0;
    for (int64_t k = 0; k < w; ++k) s += q[k] * t[j + k];
    qt[j] = s;
  }
}

typedef struct {
  double *v2, *l2, *r2; /* squared distances: profile, left, right */
  int64_t *pi, *left, *right;
} acc_t;

/*
 * stomp (profile.hpp:80-83).
 * Rows are query windows of B (the "ts_b" of the recurrence),
 * columns are windows of A; each row's distance profile over A is min-merged
 * into the A-profile with source index = row (merge_min semantics, strict
 * improvement, so the lowest row wins ties). For a self-join B = A and the
 * zone excludes |i-j| <= zone. Both series are centred on their global means
 * before the QT recurrence (the rolling-stats header centres the same way,
 * rolling.hpp:24-27); the z-normalised distance is invariant to that shift.
 * Minima are taken on d^2 (monotone in d) and rooted once at the end.
 */
int or_stomp(const double *a, int64_t n_a, const double *b, int64_t n_b, int64_t w,
             double ez_fraction, int n_workers, int64_t row_begin, int64_t row_end, double *mp,
             int64_t *pi, int64_t *left, int64_t *right) {
  const int self = (b == NULL);
  if (self) { b = a; n_b = n_a; }
  if (w < 4 || w > n_a || w > n_b) return -1;
  const int64_t zone = self ? or_zone_size(w, ez_fraction) : 0;
  if (zone < 0) return -1;
  const int64_t La = n_a - w + 1, Lb = n_b - w + 1;
  if (n_workers < 1) n_workers = 1;
  const int sample = row_end > row_begin;
  if (!sample) { row_begin = 0; row_end = Lb; }
  if (row_begin < 0 || row_end > Lb) return -1;

  double ga = 0.0, gb = 0.0;
  for (int64_t t = 0; t < n_a; ++t) ga += a[t];
  ga /= (double)n_a;
  double *ac = malloc(sizeof(double) * n_a);
  for (int64_t t = 0; t < n_a; ++t) ac[t] = a[t] - ga;
  double *bc = ac;
  if (!self) {
    for (int64_t t = 0; t < n_b; ++t) gb += b[t];
    gb /= (double)n_b;
    bc = malloc(sizeof(double) * n_b);
    for (int64_t t = 0; t < n_b; ++t) bc[t] = b[t] - gb;
  }
  double *ma = malloc(sizeof(double) * La), *sa = malloc(sizeof(double) * La);
  or_rolling_mean_std(a, n_a, w, ma, sa, n_workers);
  for (int64_t j = 0; j < La; ++j) ma[j] -= ga;
  double *mb = ma, *sb = sa;
  if (!self) {
    mb = malloc(sizeof(double) * Lb); sb = malloc(sizeof(double) * Lb);
    or_rolling_mean_std(b, n_b, w, mb, sb, n_workers);
    for (int64_t i = 0; i < Lb; ++i) mb[i] -= gb;
  }
  double *isa = malloc(sizeof(double) * La);
  for (int64_t j = 0; j < La; ++j) isa[j] = sa[j] == 0.0 ? 0.0 : 1.0 / sa[j];

  acc_t *acc = calloc((size_t)n_workers, sizeof(acc_t));
  const double wd = (double)w;

#pragma omp parallel num_threads(n_workers)
  {
#ifdef _OPENMP
    const int wk = omp_get_thread_num();
#else
    const int wk = 0;
#endif
    /* Deterministic contiguous chunks. A full join cuts them on
     * the absolute 4096-row refresh grid so every row sees the same QT
     * arithmetic for any n_workers (bit-identical outputs). A
     * bounded row sample (timing only) splits rows evenly instead. */
    int64_t r0, r1;
    if (sample) {
      r0 = row_begin + (row_end - row_begin) * wk / n_workers;
      r1 = row_begin + (row_end - row_begin) * (wk + 1) / n_workers;
    } else {
      const int64_t g0 = row_begin / OR_REFRESH_ROWS;
      const int64_t nblk = (row_end - 1) / OR_REFRESH_ROWS - g0 + 1;
      const int64_t b0 = g0 + nblk * wk / n_workers, b1 = g0 + nblk * (wk + 1) / n_workers;
      r0 = imax64(row_begin, b0 * OR_REFRESH_ROWS);
      r1 = imin64(row_end, b1 * OR_REFRESH_ROWS);
    }
    acc_t A;
    A.v2 = malloc(sizeof(double) * La);
    A.l2 = malloc(sizeof(double) * La);
    A.r2 = malloc(sizeof(double) * La);
    A.pi = malloc(sizeof(int64_t) * La);
    A.left = malloc(sizeof(int64_t) * La);
    A.right = malloc(sizeof(int64_t) * La);
    for (int64_t j = 0; j < La; ++j) {
      A.v2[j] = INFINITY; A.l2[j] = INFINITY; A.r2[j] = INFINITY;
      A.pi[j] = -1; A.left[j] = -1; A.right[j] = -1;
    }
    double *qt = malloc(sizeof(double) * La), *qn = malloc(sizeof(double) * La);
    for (int64_t i = r0; i < r1; ++i) {
      if (i == r0 || i % OR_REFRESH_ROWS == 0) {
        qt_row_direct(bc + i, ac, La, w, qt);
      } else {
        /* QT[i][j] = QT[i-1][j-1] - tb[i-1] ta[j-1] + tb[i+w-1] ta[j+w-1] */
        const double bo = bc[i - 1], bn = bc[i + w - 1];
        for (int64_t j = 1; j < La; ++j) qn[j] = qt[j - 1] - bo * ac[j - 1] + bn * ac[j + w - 1];
        double s = 0.0;
        for (int64_t k = 0; k < w; ++k) s += bc[i + k] * ac[k];
        qn[0] = s;
        double *t = qt; qt = qn; qn = t;
      }
      const double mi = mb[i], si = sb[i];
      const int fi = si == 0.0;
      /* one fused pass per side: distance (distance.hpp:16 with the per-window
       * reciprocals hoisted), exclusion zone (distance.hpp:24) by the loop
       * bounds, merge_min into the profile and into left / right */
      const double inv_i = fi ? 0.0 : 1.0 / (wd * si), wmi = wd * mi, two_w = 2.0 * wd;
      const int64_t lo_ex = self ? imax64(0, i - zone) : La, hi_ex = self ? imin64(La - 1, i + zone) : -1;
      for (int part = 0; part < 2; ++part) {
        const int64_t j0 = part == 0 ? 0 : (self ? hi_ex + 1 : La);
        const int64_t j1 = part == 0 ? (self ? lo_ex : La) : La;
        double *side2 = part == 0 ? A.r2 : A.l2;   /* j < i: row i is a right neighbour of j */
        int64_t *sidei = part == 0 ? A.right : A.left;
        for (int64_t j = j0; j < j1; ++j) {
          double d2;
          if (!fi) {
            d2 = two_w * (1.0 - (qt[j] - wmi * ma[j]) * inv_i * isa[j]);
            d2 = d2 < 0.0 ? 0.0 : (d2 > 2.0 * two_w ? 2.0 * two_w : d2);
            if (isa[j] == 0.0) d2 = wd; /* exactly one flat -> sqrt(w) */
          } else {
            d2 = sa[j] == 0.0 ? 0.0 : wd;
          }
          if (d2 < A.v2[j]) { A.v2[j] = d2; A.pi[j] = i; }
          if (self && d2 < side2[j]) { side2[j] = d2; sidei[j] = i; }
        }
      }
    }
    free(qt); free(qn);
    acc[wk] = A;
  }
  /* Fixed-order merge: worker 0 first, strict improvement. */
  for (int64_t j = 0; j < La; ++j) {
    double v = INFINITY, l = INFINITY, r = INFINITY;
    int64_t p = -1, li = -1, ri = -1;
    for (int q = 0; q < n_workers; ++q) {
      if (acc[q].v2[j] < v) { v = acc[q].v2[j]; p = acc[q].pi[j]; }
      if (acc[q].l2[j] < l) { l = acc[q].l2[j]; li = acc[q].left[j]; }
      if (acc[q].r2[j] < r) { r = acc[q].r2[j]; ri = acc[q].right[j]; }
    }
    mp[j] = sqrt(v);
    pi[j] = p;
    /* Near-zero hits are recomputed directly so exact matches come out as 0
     * (the reference's convention for distance profiles, distance.hpp:30-33);
     * the QT formula cancels to ~sqrt(2w*eps) there. */
    if (p >= 0 && mp[j] < 1e-3) {
      mp[j] = direct_dist(a + j, ma[j] + ga, sa[j], b + p, mb[p] + (self ? ga : gb), sb[p], w);
    }
    if (left) left[j] = self ? li : -1;
    if (right) right[j] = self ? ri : -1;
  }
  for (int q = 0; q < n_workers; ++q) {
    free(acc[q].v2); free(acc[q].l2); free(acc[q].r2);
    free(acc[q].pi); free(acc[q].left); free(acc[q].right);
  }
  free(acc); free(isa);
  free(ac);
  if (!self) { free(bc); free(mb); free(sb); }
  free(ma); free(sa);
  return 0;
}

/* ---------------------------------------------------------------- SCRIMP */

/* splitmix64 for the seeded diagonal permutation ("deterministically
 * seeded random order"; the reference names mt19937_64 for data only). */
static uint64_t sm64(uint64_t *s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* SCRIMP's inner loop over an explicit list of diagonals: the
 * checker for partial (anytime) runs whose diagonal subset is known. Values
 * are the minima over those diagonals only; ties keep the smaller index. */
int or_scrimp_diagonals(const double *a, int64_t n_a, int64_t w, const int64_t *diags,
                        int64_t n_diags, double *mp, int64_t *pi, int n_threads) {
  if (w < 4 || w > n_a) return -1;
  const int64_t L = n_a - w + 1;
  double g = 0.0;
  for (int64_t t = 0; t < n_a; ++t) g += a[t];
  g /= (double)n_a;
  double *ac = malloc(sizeof(double) * n_a);
  for (int64_t t = 0; t < n_a; ++t) ac[t] = a[t] - g;
  double *mu = malloc(sizeof(double) * L), *sd = malloc(sizeof(double) * L);
  or_rolling_mean_std(a, n_a, w, mu, sd, n_threads);
  for (int64_t j = 0; j < L; ++j) mu[j] -= g;
  for (int64_t j = 0; j < L; ++j) { mp[j] = INFINITY; pi[j] = -1; }
  /* per-thread accumulators merged in fixed order (ties: smaller index) */
  if (n_threads < 1) n_threads = 1;
  double *bv = malloc(sizeof(double) * L * n_threads);
  int64_t *bi = malloc(sizeof(int64_t) * L * n_threads);
#pragma omp parallel num_threads(n_threads)
  {
#ifdef _OPENMP
    const int tid = omp_get_thread_num();
#else
    const int tid = 0;
#endif
    double *v = bv + (size_t)L * tid;
    int64_t *ix = bi + (size_t)L * tid;
    for (int64_t j = 0; j < L; ++j) { v[j] = INFINITY; ix[j] = -1; }
#pragma omp for schedule(dynamic, 8)
    for (int64_t q = 0; q < n_diags; ++q) {
      const int64_t k = diags[q];
      if (k <= 0 || k >= L) continue;
      double qt = 0.0;
      for (int64_t t = 0; t < w; ++t) qt += ac[t] * ac[k + t];
      for (int64_t i = 0; i + k < L; ++i) {
        const int64_t j = i + k;
        if (i > 0) qt = qt - ac[i - 1] * ac[j - 1] + ac[i + w - 1] * ac[j + w - 1];
        if (i > 0 && i % OR_REFRESH_ROWS == 0) {
          double sacc = 0.0;
          for (int64_t t = 0; t < w; ++t) sacc += ac[i + t] * ac[j + t];
          qt = sacc;
        }
        const double d = or_znorm_dist_from_qt(qt, w, mu[i], sd[i], mu[j], sd[j]);
        if (d < v[i] || (d == v[i] && j < ix[i])) { v[i] = d; ix[i] = j; }
        if (d < v[j] || (d == v[j] && i < ix[j])) { v[j] = d; ix[j] = i; }
      }
    }
  }
  for (int t = 0; t < n_threads; ++t)
    for (int64_t j = 0; j < L; ++j) {
      const double d = bv[(size_t)L * t + j];
      const int64_t x = bi[(size_t)L * t + j];
      if (d < mp[j] || (d == mp[j] && x >= 0 && x < pi[j])) { mp[j] = d; pi[j] = x; }
    }
  /* near-zero hits recomputed directly, as in or_stomp (exact repeats -> 0) */
  for (int64_t j = 0; j < L; ++j)
    if (pi[j] >= 0 && mp[j] < 1e-3)
      mp[j] = direct_dist(ac + j, mu[j], sd[j], ac + pi[j], mu[pi[j]], sd[pi[j]], w);
  free(bv); free(bi); free(mu); free(sd); free(ac);
  return 0;
}

/* scrimp (profile.hpp:85-89): each diagonal's first dot
 * product directly, then the O(1) update along the diagonal; each cell
 * min-merges into row i and row j. */
int or_scrimp(const double *a, int64_t n_a, int64_t w, double ez_fraction, int64_t s_size,
              uint64_t seed, double *mp, int64_t *pi, int64_t *left, int64_t *right,
              double *coverage) {
  if (w < 4 || w > n_a) return -1;
  const int64_t zone = or_zone_size(w, ez_fraction);
  if (zone < 0) return -1;
  const int64_t L = n_a - w + 1;
  double g = 0.0;
  for (int64_t t = 0; t < n_a; ++t) g += a[t];
  g /= (double)n_a;
  double *ac = malloc(sizeof(double) * n_a);
  for (int64_t t = 0; t < n_a; ++t) ac[t] = a[t] - g;
  double *mu = malloc(sizeof(double) * L), *sd = malloc(sizeof(double) * L);
  or_rolling_mean_std(a, n_a, w, mu, sd, 1);
  for (int64_t j = 0; j < L; ++j) mu[j] -= g;
  double *lv = malloc(sizeof(double) * L), *rv = malloc(sizeof(double) * L);
  for (int64_t j = 0; j < L; ++j) {
    mp[j] = INFINITY; pi[j] = -1; lv[j] = INFINITY; rv[j] = INFINITY;
    if (left) left[j] = -1;
    if (right) right[j] = -1;
  }
  const int64_t k0 = zone + 1;
  const int64_t nd = L > k0 ? L - k0 : 0;
  int64_t *order = malloc(sizeof(int64_t) * (nd > 0 ? nd : 1));
  for (int64_t q = 0; q < nd; ++q) order[q] = k0 + q;
  uint64_t st = seed;
  for (int64_t q = nd - 1; q > 0; --q) { /* Fisher-Yates */
    const int64_t r = (int64_t)(sm64(&st) % (uint64_t)(q + 1));
    const int64_t t = order[q]; order[q] = order[r]; order[r] = t;
  }
  const int64_t todo = (s_size <= 0 || s_size >= nd) ? nd : s_size;
  const double wd = (double)w;
  for (int64_t q = 0; q < todo; ++q) {
    const int64_t k = order[q];
    double qt = 0.0;
    for (int64_t t = 0; t < w; ++t) qt += ac[t] * ac[k + t];
    for (int64_t i = 0; i + k < L; ++i) {
      const int64_t j = i + k;
      if (i > 0) qt = qt - ac[i - 1] * ac[j - 1] + ac[i + w - 1] * ac[j + w - 1];
      if (i > 0 && i % OR_REFRESH_ROWS == 0) {
        double s = 0.0;
        for (int64_t t = 0; t < w; ++t) s += ac[i + t] * ac[j + t];
        qt = s;
      }
      const double d = or_znorm_dist_from_qt(qt, w, mu[i], sd[i], mu[j], sd[j]);
      (void)wd;
      /* row i gains neighbour j (right), row j gains neighbour i (left);
       * ties keep the smaller index */
      if (d < mp[i] || (d == mp[i] && j < pi[i])) { mp[i] = d; pi[i] = j; }
      if (d < mp[j] || (d == mp[j] && i < pi[j])) { mp[j] = d; pi[j] = i; }
      if (d < rv[i] || (d == rv[i] && right && j < right[i])) { rv[i] = d; if (right) right[i] = j; }
      if (d < lv[j] || (d == lv[j] && left && i < left[j])) { lv[j] = d; if (left) left[j] = i; }
    }
  }
  /* near-zero hits recomputed directly, as in or_stomp (exact repeats -> 0) */
  for (int64_t j = 0; j < L; ++j)
    if (pi[j] >= 0 && mp[j] < 1e-3)
      mp[j] = direct_dist(ac + j, mu[j], sd[j], ac + pi[j], mu[pi[j]], sd[pi[j]], w);
  const int full = todo == nd;
  if (!full) {
    if (left) for (int64_t j = 0; j < L; ++j) left[j] = -1;
    if (right) for (int64_t j = 0; j < L; ++j) right[j] = -1;
  }
  if (coverage) *coverage = nd > 0 ? (double)todo / (double)nd : 1.0;
  free(order); free(lv); free(rv); free(mu); free(sd); free(ac);
  return 0;
}
