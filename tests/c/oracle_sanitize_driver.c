/* TEST INFRASTRUCTURE: drives every oracle entry point on small seeded inputs
 * (edge cases included: window == n, zone >= L - 1, flat runs, AB with
 * n_b == window, single-row samples) so tests/test_oracle_sanitize.py can run
 * the oracle under AddressSanitizer + UndefinedBehaviorSanitizer. Prints a
 * checksum so the compiler cannot drop the work. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mprof_oracle.h"

static uint64_t st = 88172645463325252ULL;
static double rnd(void) {
  st ^= st << 13; st ^= st >> 7; st ^= st << 17;
  return (double)(st >> 11) / 9007199254740992.0 - 0.5;
}

static double sum_arr(const double *v, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += isfinite(v[i]) ? v[i] : 1.0;
  return s;
}

int main(void) {
  double acc = 0.0;
  const int64_t ns[] = {4, 9, 64, 300, 1000};
  const int64_t ws[] = {4, 4, 16, 50, 64};
  for (int c = 0; c < 5; ++c) {
    const int64_t n = ns[c], w = ws[c], L = n - w + 1;
    double *a = malloc(sizeof(double) * n), *b = malloc(sizeof(double) * (n + 7));
    double x = 0.0;
    for (int64_t i = 0; i < n; ++i) a[i] = (x += rnd());
    for (int64_t i = 0; i < n + 7; ++i) b[i] = rnd();
    if (n > 40) for (int64_t i = 10; i < 30; ++i) a[i] = 2.5;  /* flat run */
    double *mp = malloc(sizeof(double) * (L + 7)), *mu = malloc(sizeof(double) * L),
           *sd = malloc(sizeof(double) * L), *dp = malloc(sizeof(double) * (n + 7));
    int64_t *pi = malloc(sizeof(int64_t) * (L + 7)), *lf = malloc(sizeof(int64_t) * (L + 7)),
            *rt = malloc(sizeof(int64_t) * (L + 7));
    acc += (double)or_zone_size(w, 0.5) + or_is_flat_std(0.0, 1.0);
    or_rolling_mean_std(a, n, w, mu, sd, 2);
    acc += sum_arr(mu, L) + sum_arr(sd, L);
    acc += or_znorm_dist_from_qt(1.0, w, 0.1, 1.0, 0.2, 0.0);
    or_sliding_dot_direct(a, w, b, n, dp);
    acc += sum_arr(dp, n - w + 1);
    const double ezs[] = {0.0, 0.25, 0.5, 1e6};
    for (int e = 0; e < 4; ++e) {
      or_brute_force_mp(a, n, NULL, 0, w, ezs[e], mp, pi, lf, rt, 2);
      acc += sum_arr(mp, L);
      or_stomp(a, n, NULL, 0, w, ezs[e], 3, 0, 0, mp, pi, lf, rt);
      acc += sum_arr(mp, L);
      double cov = 0.0;
      or_scrimp(a, n, w, ezs[e], L / 3, 7, mp, pi, lf, rt, &cov);
      acc += sum_arr(mp, L) + cov;
    }
    or_stomp(a, n, b, w + (c % 3), w, 0.5, 2, 0, 0, mp, pi, NULL, NULL);  /* AB, short B */
    acc += sum_arr(mp, L);
    or_brute_force_mp(a, n, b, n + 7, w, 0.5, mp, pi, NULL, NULL, 1);
    acc += sum_arr(mp, L);
    const int64_t rows[] = {0, L - 1, L / 2};
    or_brute_force_rows(a, n, NULL, 0, w, 0.5, rows, 3, mp, pi, lf, rt, 2);
    acc += sum_arr(mp, 3);
    or_stomp(a, n, NULL, 0, w, 0.5, 2, 0, L > 1 ? 1 : L, mp, pi, lf, rt);
    or_mass_distance_profile(a, w, b, n + 7, 3, 2, dp, 2);
    acc += sum_arr(dp, n + 7 - w + 1);
    or_apply_exclusion_zone(dp, n + 7 - w + 1, 0, n + 100);
    const int64_t diags[] = {1, L > 2 ? L - 1 : 1};
    or_scrimp_diagonals(a, n, w, diags, L > 2 ? 2 : 1, mp, pi, 2);
    acc += sum_arr(mp, L);
    for (int64_t i = 0; i < L; ++i) mp[i] = INFINITY, pi[i] = -1;
    or_merge_min(mp, pi, mu, L, 5);
    acc += sum_arr(mp, L);
    /* multivariate: 3 dims */
    const int64_t d = 3;
    double *m3 = malloc(sizeof(double) * d * n), *o3 = malloc(sizeof(double) * d * L);
    int64_t *p3 = malloc(sizeof(int64_t) * d * L), *q3 = malloc(sizeof(int64_t) * d * L);
    for (int64_t i = 0; i < d * n; ++i) m3[i] = rnd();
    or_simple_join(m3, n, NULL, 0, d, w, 0.5, 2, 0, 0, o3, p3, lf, rt);
    acc += sum_arr(o3, L);
    or_simple_brute(m3, n, m3, n, d, w, 0.5, o3, p3, 2);
    acc += sum_arr(o3, L);
    const int64_t must[] = {1}, exc[] = {2};
    or_mstomp(m3, n, d, w, 0.5, must, 1, exc, 1, 2, 0, 0, o3, p3, q3);
    acc += sum_arr(o3, d * L);
    or_mstomp(m3, n, d, w, 0.5, NULL, 0, NULL, 0, 1, 0, 0, o3, p3, q3);
    acc += sum_arr(o3, d * L);
    free(m3); free(o3); free(p3); free(q3);
    free(a); free(b); free(mp); free(mu); free(sd); free(dp); free(pi); free(lf); free(rt);
  }
  printf("checksum %.6e\n", acc);
  return 0;
}
