/* Radius tables of the NATIVE source jumps (3D: Beta(2,2); 2D: the disk Green's law),
 * shared by the library and the C oracle, so both walk the same stream.
 *
 * The ball Green's function importance sampler draws the radius fraction t from
 * Beta(2,2), density 6 t (1 - t), CDF F(t) = 3 t^2 - 2 t^3 (greens.py:83-89: the
 * G-weighted radial law in 3D). The jump takes a 12-bit index k and uses
 *     t_k = E[t | k/N <= F(t) < (k+1)/N] = N [2 t^3 - 3/2 t^4]_{F^-1(k/N)}^{F^-1((k+1)/N)},
 * the conditional mean of its probability bin (N = 4096), with the exact quantile
 * F^-1(v) = 1/2 + sin(asin(2v - 1) / 3). Conditional means keep E[t] exact; E[t^2]
 * and E[t^3] differ from Beta(2,2)'s by -1.0e-8 and -1.5e-8 (tests/test_oracle_golden.py
 * test_beta22_table_moments). Entries are computed in double and rounded to float.
 */
#ifndef WOS_BETA_TABLE_H
#define WOS_BETA_TABLE_H

#include <math.h>

#define WOS_BETA_TABLE_BITS 12
#define WOS_BETA_TABLE_N (1 << WOS_BETA_TABLE_BITS)

static inline double wos_beta22_quantile(double v) {
  double s = 2.0 * v - 1.0;
  if (s > 1.0) s = 1.0;
  if (s < -1.0) s = -1.0;
  return 0.5 + sin(asin(s) / 3.0);
}

static inline void wos_beta22_table(float* out) {
  const double n = (double)WOS_BETA_TABLE_N;
  double ta = 0.0; /* F^-1(0) */
  for (int k = 0; k < WOS_BETA_TABLE_N; ++k) {
    const double tb = (k + 1 == WOS_BETA_TABLE_N) ? 1.0 : wos_beta22_quantile((k + 1) / n);
    /* n * integral of t dF over [ta, tb]: dF = 6 t (1 - t) dt */
    const double ga = 2.0 * ta * ta * ta - 1.5 * ta * ta * ta * ta;
    const double gb = 2.0 * tb * tb * tb - 1.5 * tb * tb * tb * tb;
    out[k] = (float)(n * (gb - ga));
    ta = tb;
  }
}

/* The 2D counterpart: the disk Green's function G(r) = ln(R/r) / (2 pi) makes the radius
 * fraction t = r/R of the importance-sampled source point follow p(t) = 4 t ln(1/t),
 * F(t) = t^2 (1 - 2 ln t) (greens.py:68-89: mass R^2/4). Entry k is again the
 * conditional mean of its 12-bit probability bin, N [4/9 t^3 (1 - 3 ln t)] between the
 * bin's quantiles (found by bisection in double; F has no closed-form inverse). */
static inline double wos_green2_cdf(double t) { return t <= 0.0 ? 0.0 : t * t * (1.0 - 2.0 * log(t)); }

static inline double wos_green2_quantile(double v) {
  double lo = 0.0, hi = 1.0;
  for (int it = 0; it < 200 && hi - lo > 1e-17; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (wos_green2_cdf(mid) < v) lo = mid;
    else hi = mid;
  }
  return 0.5 * (lo + hi);
}

static inline void wos_green2_table(float* out) {
  const double n = (double)WOS_BETA_TABLE_N;
  double ga = 0.0; /* antiderivative of t dF at t = 0 */
  for (int k = 0; k < WOS_BETA_TABLE_N; ++k) {
    const double tb = (k + 1 == WOS_BETA_TABLE_N) ? 1.0 : wos_green2_quantile((k + 1) / n);
    const double gb = (4.0 / 9.0) * tb * tb * tb * (1.0 - 3.0 * log(tb));
    out[k] = (float)(n * (gb - ga));
    ga = gb;
  }
}

#endif /* WOS_BETA_TABLE_H */
