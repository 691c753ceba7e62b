/*
 * wos_oracle.c — TEST INFRASTRUCTURE ONLY. Never linked into, loaded by, or
 * called from the product path (paper_2603_01193_b200/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs use it,
 * and only as the checker or the timed CPU baseline.
 *
 * A plain-C, fp64, scalar restatement of the reference's Walk-on-Spheres path
 * (arxiv 2603.01193, package `spherewalk`, read-only at /root/reference/pkg/src):
 *
 *   philox4x64 ........ rng.philox4x64            rng.py:57-82 (_mulhilo rng.py:44-54)
 *   u53 ............... rng.to_uniform            rng.py:100-102 (_kernels._u01 :85-87)
 *   nonzero_u ......... walker._redraw_zeros      walker.py:232-242 (_kernels._nonzero_u :90-102)
 *   ball_query ........ BallDomain.boundary_query geometry.py:196-206
 *   walk_ref_one ...... walker._poisson_generic   walker.py:257-314 (one row; the
 *                       vectorized loop's per-lane arithmetic in the same order)
 *   oracle_estimate ... estimator._estimate_block estimator.py:119-141 +
 *                       PointEstimate.from_values estimator.py:106-110 (two-pass)
 *
 * Box and polygon domains, and the sine / Gaussian / Fourier / arc-length /
 * quadratic problem terms, do not exist in the reference; they are the BASELINE
 * configs' problem data, passed to the reference through the duck-typed domain
 * protocol (dim, contains, boundary_query, bounding_radius) and Python callables
 * by tests/golden/make_golden.py, whose outputs pin this file
 * (tests/test_oracle_golden.py).
 *
 * oracle_walk_rows_native restates the product's NATIVE_F32 estimator
 * (Philox4x32-10 stream layout + Green's-function importance sampling) in fp64 so
 * the native kernel can be checked walk by walk, not only statistically.
 *
 * Build: oracle/Makefile -> oracle/_build/libwos_oracle.so
 */
#include "../include/wos_b200.h"
#include "../include/wos_beta_table.h"

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TWO_PI 6.283185307179586
/* NATIVE direction angles are 2 pi u - pi in [-pi, pi) (wos_walk.cuh dir_angle) */
#define PI 3.141592653589793
#define INV_TWO_PI (1.0 / TWO_PI)
#define INV_FOUR_PI (1.0 / (4.0 * 3.141592653589793))
#define PI 3.141592653589793

/* ------------------------------------------------------------------ */
/* Philox 4x64-10 (rng.py:31-41 constants, :76-81 round)               */
/* ------------------------------------------------------------------ */
static void philox4x64(const uint64_t c[4], uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
  for (int r = 0; r < 10; ++r) {
    unsigned __int128 p0 = (unsigned __int128)0xD2E7470EE14C6C93ull * x0;
    unsigned __int128 p1 = (unsigned __int128)0xCA5A826395121157ull * x2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t n0 = hi1 ^ x1 ^ k0, n2 = hi0 ^ x3 ^ k1;
    x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

void oracle_philox4x64(int64_t n, const uint64_t* ctr, uint64_t k0, uint64_t k1, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) philox4x64(ctr + 4 * i, k0, k1, out + 4 * i);
}

/* Philox 4x32-R (Random123 constants) — the NATIVE_F32 generator: R = 10 rounds by
 * default, 7 when WalkConfig.philox_rounds = 7 (oracle_set_philox_rounds). */
static int g_native_rounds = 10;
void oracle_set_philox_rounds(int r) { g_native_rounds = r; }

static void philox4x32_r(const uint32_t c[4], uint32_t k0, uint32_t k1, int rounds, uint32_t out[4]) {
  uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
  for (int r = 0; r < rounds; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * x0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ x1 ^ k0, n2 = hi0 ^ x3 ^ k1;
    x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* the NATIVE stream's block: g_native_rounds rounds */
static void philox4x32(const uint32_t c[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  philox4x32_r(c, k0, k1, g_native_rounds, out);
}

void oracle_philox4x32(int64_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out) {
  for (int64_t i = 0; i < n; ++i) philox4x32_r(ctr + 4 * i, k0, k1, 10, out + 4 * i);
}

void oracle_philox4x32_rounds(int64_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, int rounds,
                              uint32_t* out) {
  for (int64_t i = 0; i < n; ++i) philox4x32_r(ctr + 4 * i, k0, k1, rounds, out + 4 * i);
}

static double u53(uint64_t w) { return (double)(w >> 11) * 1.1102230246251565e-16; }

/* rejected zero uniform -> redraw at tag 1, 2, ... (walker.py:232-242) */
static double nonzero_u(double u, uint64_t draw, uint64_t pid, uint64_t tid, uint64_t k0,
                        uint64_t k1) {
  uint64_t tag = 1;
  while (u == 0.0) {
    uint64_t c[4] = {draw, pid, tid, tag}, w[4];
    philox4x64(c, k0, k1, w);
    u = u53(w[0]);
    tag += 1;
  }
  return u;
}

/* ------------------------------------------------------------------ */
/* Domains: distance to the boundary and the closest boundary point    */
/* ------------------------------------------------------------------ */
/* PolarDomain (geometry.py:83-153): table form [r0, c1, c2, stride, n, bx.., by..] */
static double polar_r(const double* P, double t) {
  return P[0] * (1.0 + P[1] * cos(4.0 * t) + P[2] * cos(8.0 * t)); /* _kernels.py:110-112 */
}
static double polar_curve_d2(const double* P, double t, double px, double py) {
  const double r = polar_r(P, t);
  const double dx = r * cos(t) - px, dy = r * sin(t) - py;
  return dx * dx + dy * dy;
}
/* the product's NATIVE form scans coarse to fine (wos_walk.cuh polar_query); the
 * drivers set this for native walks */
static int g_polar_native = 0;
static void polar_probe(const double* bx, const double* by, int n, int jj, double px, double py,
                        double* best, int* bj) {
  jj = jj < 0 ? jj + n : (jj >= n ? jj - n : jj);
  const double dx = bx[jj] - px, dy = by[jj] - py, d2 = dx * dx + dy * dy;
  if (d2 < *best) { *best = d2; *bj = jj; }
}
/* _kernels.polar_query_fast (_kernels.py:121-148, 185-219) */
static double polar_query(const double* P, double px, double py, double* qx, double* qy) {
  const int stride = (int)P[3], n = (int)P[4];
  const double *bx = P + 5, *by = P + 5 + n;
  double best = 1.0e300;
  int bj = 0;
  if (g_polar_native) {
    int st = stride > 1 ? stride : 8;
    for (int j = 0; j < n; j += st) polar_probe(bx, by, n, j, px, py, &best, &bj);
    while (st > 1) {
      const int f = st >= 8 ? st / 8 : 1, c = bj;
      for (int off = -st; off <= st; off += f)
        if (off != 0) polar_probe(bx, by, n, c + off, px, py, &best, &bj);
      st = f;
    }
  } else {
    for (int j = 0; j < n; j += stride) polar_probe(bx, by, n, j, px, py, &best, &bj);
    if (stride > 1) {
      const int lo = bj - stride;
      for (int off = 0; off <= 2 * stride; ++off) polar_probe(bx, by, n, lo + off, px, py, &best, &bj);
    }
  }
  const double h = TWO_PI / n, t0 = bj * h;
  const double fm = polar_curve_d2(P, t0 - h, px, py), fp = polar_curve_d2(P, t0 + h, px, py);
  const double denom = fm - 2.0 * best + fp;
  double shift = denom > 0.0 ? 0.5 * h * (fm - fp) / denom : 0.0;
  if (shift > h) shift = h;
  else if (shift < -h) shift = -h;
  const double tm = t0 + shift, r = polar_r(P, tm);
  const double cx = r * cos(tm), cy = r * sin(tm);
  const double dx = cx - px, dy = cy - py, dm = dx * dx + dy * dy;
  if (best < dm) { *qx = bx[bj]; *qy = by[bj]; return sqrt(best); }
  *qx = cx; *qy = cy;
  return sqrt(dm);
}

/* MeshDomain (geometry.py:259-323, 470-533): closest point on a triangle with its
 * feature region, the reference's operation order and region priority */
enum { R_A, R_B, R_C, R_AB, R_BC, R_CA, R_FACE };
static double dot3(const double* u, const double* v) { return u[0] * v[0] + u[1] * v[1] + u[2] * v[2]; }
static double clip01(double t) { return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t); }
static double sdiv(double n, double d) { return n / (d == 0.0 ? 1.0 : d); }
static int closest_tri(const double* p, const double* a, const double* b, const double* c, double* q) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  for (int i = 0; i < 3; ++i) {
    ab[i] = b[i] - a[i]; ac[i] = c[i] - a[i]; ap[i] = p[i] - a[i]; bp[i] = p[i] - b[i]; cp[i] = p[i] - c[i];
  }
  const double d1 = dot3(ab, ap), d2 = dot3(ac, ap), d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  const double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  const double vc = d1 * d4 - d3 * d2, vb = d5 * d2 - d1 * d6, va = d3 * d6 - d5 * d4;
  if (d1 <= 0.0 && d2 <= 0.0) { for (int i = 0; i < 3; ++i) q[i] = a[i]; return R_A; }
  if (d3 >= 0.0 && d4 <= d3) { for (int i = 0; i < 3; ++i) q[i] = b[i]; return R_B; }
  if (d6 >= 0.0 && d5 <= d6) { for (int i = 0; i < 3; ++i) q[i] = c[i]; return R_C; }
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    const double t = clip01(sdiv(d1, d1 - d3));
    for (int i = 0; i < 3; ++i) q[i] = a[i] + ab[i] * t;
    return R_AB;
  }
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    const double t = clip01(sdiv(d4 - d3, (d4 - d3) + (d5 - d6)));
    for (int i = 0; i < 3; ++i) q[i] = b[i] + (c[i] - b[i]) * t;
    return R_BC;
  }
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    const double t = clip01(sdiv(d2, d2 - d6));
    for (int i = 0; i < 3; ++i) q[i] = a[i] + ac[i] * t;
    return R_CA;
  }
  const double den = va + vb + vc, v = sdiv(vb, den), w = sdiv(vc, den);
  for (int i = 0; i < 3; ++i) q[i] = a[i] + ab[i] * v + ac[i] * w;
  return R_FACE;
}
/* brute-force nearest triangle (MeshDomain._closest_brute: first index attaining the minimum) */
static double mesh_nearest(const double* P, const double* x, double* q, int64_t* tri, int* reg) {
  const int64_t nv = (int64_t)P[0], nf = (int64_t)P[1];
  const double *V = P + 2, *F = P + 2 + 3 * nv;
  double best = INFINITY;
  for (int64_t t = 0; t < nf; ++t) {
    double qq[3];
    const int r = closest_tri(x, V + 3 * (int64_t)F[3 * t], V + 3 * (int64_t)F[3 * t + 1],
                              V + 3 * (int64_t)F[3 * t + 2], qq);
    const double df[3] = {qq[0] - x[0], qq[1] - x[1], qq[2] - x[2]};
    const double d2 = dot3(df, df);
    if (d2 < best) {
      best = d2; q[0] = qq[0]; q[1] = qq[1]; q[2] = qq[2]; *tri = t; *reg = r;
    }
  }
  return best;
}
/* MeshDomain._build_normals + _feature_normal (geometry.py:434-508) for one query */
static void mesh_feature_normal(const double* P, int64_t t, int reg, double* n) {
  const int64_t nv = (int64_t)P[0], nf = (int64_t)P[1];
  const double *V = P + 2, *F = P + 2 + 3 * nv;
  const int64_t id[3] = {(int64_t)F[3 * t], (int64_t)F[3 * t + 1], (int64_t)F[3 * t + 2]};
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t s = 0; s < nf; ++s) {
    const int64_t js[3] = {(int64_t)F[3 * s], (int64_t)F[3 * s + 1], (int64_t)F[3 * s + 2]};
    double e1[3], e2[3], fn[3];
    for (int c = 0; c < 3; ++c) { e1[c] = V[3 * js[1] + c] - V[3 * js[0] + c]; e2[c] = V[3 * js[2] + c] - V[3 * js[0] + c]; }
    fn[0] = e1[1] * e2[2] - e1[2] * e2[1];
    fn[1] = e1[2] * e2[0] - e1[0] * e2[2];
    fn[2] = e1[0] * e2[1] - e1[1] * e2[0];
    const double len = sqrt(fn[0] * fn[0] + fn[1] * fn[1] + fn[2] * fn[2]);
    for (int c = 0; c < 3; ++c) fn[c] /= len;
    if (reg == R_FACE) {
      if (s == t) { for (int c = 0; c < 3; ++c) n[c] = fn[c]; return; }
      continue;
    }
    if (reg <= R_C) { /* angle-weighted vertex normal */
      const int64_t vid = id[reg];
      for (int l = 0; l < 3; ++l) {
        if (js[l] != vid) continue;
        double a1[3], a2[3];
        for (int c = 0; c < 3; ++c) {
          a1[c] = V[3 * js[(l + 1) % 3] + c] - V[3 * js[l] + c];
          a2[c] = V[3 * js[(l + 2) % 3] + c] - V[3 * js[l] + c];
        }
        const double cs = dot3(a1, a2) / (sqrt(dot3(a1, a1)) * sqrt(dot3(a2, a2)));
        const double ang = acos(cs < -1.0 ? -1.0 : (cs > 1.0 ? 1.0 : cs));
        for (int c = 0; c < 3; ++c) acc[c] += ang * fn[c];
      }
    } else { /* edge normal: faces sharing the edge */
      const int l0 = reg == R_AB ? 0 : (reg == R_BC ? 1 : 2);
      const int64_t u = id[l0], w = id[(l0 + 1) % 3];
      for (int l = 0; l < 3; ++l) {
        const int64_t a = js[l], b = js[(l + 1) % 3];
        if ((a == u && b == w) || (a == w && b == u))
          for (int c = 0; c < 3; ++c) acc[c] += fn[c];
      }
    }
  }
  const double len = sqrt(dot3(acc, acc));
  for (int c = 0; c < 3; ++c) n[c] = acc[c] / (len == 0.0 ? 1.0 : len);
}

static double query(const wos_problem* pb, const double* x, double* q) {
  const int dim = pb->dim;
  const double* P = pb->dom;
  if (pb->dom_kind == WOS_DOM_POLAR) return polar_query(P, x[0], x[1], &q[0], &q[1]);
  if (pb->dom_kind == WOS_DOM_MESH) {
    int64_t t;
    int reg;
    return sqrt(mesh_nearest(P, x, q, &t, &reg));
  }
  if (pb->dom_kind == WOS_DOM_BALL) {
    /* geometry.py:196-206 */
    double u[3], s = 0.0;
    for (int i = 0; i < dim; ++i) { u[i] = x[i] - P[i]; s += u[i] * u[i]; }
    double rho = sqrt(s), R = P[dim];
    double d = fabs(R - rho);
    for (int i = 0; i < dim; ++i) {
      double dir = (rho == 0.0) ? (i == 0 ? 1.0 : 0.0) : u[i] / rho;
      q[i] = P[i] + R * dir;
    }
    return d;
  }
  if (pb->dom_kind == WOS_DOM_BOX) {
    /* min over faces; first nearest face wins (axis order, lower before upper) */
    double best = INFINITY;
    int axis = 0;
    double face = 0.0;
    for (int i = 0; i < dim; ++i) {
      double dl = x[i] - P[i], du = P[dim + i] - x[i];
      if (dl < best) { best = dl; axis = i; face = P[i]; }
      if (du < best) { best = du; axis = i; face = P[dim + i]; }
    }
    for (int i = 0; i < dim; ++i) q[i] = x[i];
    q[axis] = face;
    return best;
  }
  /* WOS_DOM_POLYGON */
  const int n = (int)P[0];
  const double* V = P + 1;
  double best = INFINITY, bx = 0.0, by = 0.0;
  for (int i = 0; i < n; ++i) {
    int j = (i + 1 == n) ? 0 : i + 1;
    double ax = V[2 * i], ay = V[2 * i + 1];
    double ex = V[2 * j] - ax, ey = V[2 * j + 1] - ay;
    double wx = x[0] - ax, wy = x[1] - ay;
    double t = (wx * ex + wy * ey) / (ex * ex + ey * ey);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    double cx = ax + t * ex, cy = ay + t * ey;
    double dx = x[0] - cx, dy = x[1] - cy;
    double d2 = dx * dx + dy * dy;
    if (d2 < best) { best = d2; bx = cx; by = cy; }
  }
  q[0] = bx; q[1] = by;
  return sqrt(best);
}

int oracle_contains(const wos_problem* pb, const double* x) {
  const int dim = pb->dim;
  const double* P = pb->dom;
  if (pb->dom_kind == WOS_DOM_MESH) { /* MeshDomain.signed_distance < 0 (geometry.py:510-525) */
    double q[3], n[3];
    int64_t t;
    int reg;
    mesh_nearest(P, x, q, &t, &reg);
    mesh_feature_normal(P, t, reg, n);
    return (x[0] - q[0]) * n[0] + (x[1] - q[1]) * n[1] + (x[2] - q[2]) * n[2] < 0.0;
  }
  if (pb->dom_kind == WOS_DOM_POLAR) { /* geometry.py:129-134 */
    const double th = atan2(x[1], x[0]);
    return hypot(x[0], x[1]) < polar_r(P, th);
  }
  if (pb->dom_kind == WOS_DOM_BALL) {
    double s = 0.0;
    for (int i = 0; i < dim; ++i) s += (x[i] - P[i]) * (x[i] - P[i]);
    return sqrt(s) < P[dim];
  }
  if (pb->dom_kind == WOS_DOM_BOX) {
    for (int i = 0; i < dim; ++i)
      if (!(x[i] > P[i] && x[i] < P[dim + i])) return 0;
    return 1;
  }
  const int n = (int)P[0];
  const double* V = P + 1;
  int inside = 0;
  for (int i = 0; i < n; ++i) {
    int j = (i + 1 == n) ? 0 : i + 1;
    double ax = V[2 * i], ay = V[2 * i + 1], bx = V[2 * j], by = V[2 * j + 1];
    if ((ay > x[1]) != (by > x[1])) {
      double xc = ax + (x[1] - ay) * (bx - ax) / (by - ay);
      if (x[0] < xc) inside = !inside;
    }
  }
  return inside;
}

/* ------------------------------------------------------------------ */
/* Problem terms                                                        */
/* ------------------------------------------------------------------ */
static double source(const wos_problem* pb, const double* y) {
  const int dim = pb->dim;
  const double* S = pb->src;
  switch (pb->src_kind) {
    case WOS_SRC_CONST:
      return S[0];
    case WOS_SRC_RBF2: { /* _kernels.py:248-259 */
      double d1x = y[0] - S[2], d1y = y[1] - S[3], d2x = y[0] - S[4], d2y = y[1] - S[5];
      return S[0] * exp(-(d1x * d1x + d1y * d1y)) + S[1] * exp(-(d2x * d2x + d2y * d2y));
    }
    case WOS_SRC_SINE: {
      const int K = (int)S[0];
      const double* a = S + 1;
      double sv[3][16];
      for (int i = 0; i < dim; ++i)
        for (int k = 0; k < K; ++k) sv[i][k] = sin((double)(k + 1) * PI * y[i]);
      double f = 0.0;
      if (dim == 2) {
        for (int k = 0; k < K; ++k)
          for (int l = 0; l < K; ++l) f += a[k * K + l] * sv[0][k] * sv[1][l];
      } else {
        for (int k = 0; k < K; ++k)
          for (int l = 0; l < K; ++l)
            for (int m = 0; m < K; ++m)
              f += a[(k * K + l) * K + m] * sv[0][k] * sv[1][l] * sv[2][m];
      }
      return f;
    }
    case WOS_SRC_GAUSS: {
      double r2 = 0.0;
      for (int i = 0; i < dim; ++i) r2 += (y[i] - S[2 + i]) * (y[i] - S[2 + i]);
      return S[0] * exp(-r2 / (2.0 * S[1] * S[1]));
    }
    default:
      return 0.0;
  }
}

static double boundary(const wos_problem* pb, const double* q) {
  const int dim = pb->dim;
  const double* B = pb->bnd;
  switch (pb->bnd_kind) {
    case WOS_BND_CONST:
      return B[0];
    case WOS_BND_LINEAR:
      if (dim == 2) return B[0] * q[0] + B[1] * q[1] + B[2];
      return B[0] * q[0] + B[1] * q[1] + B[2] * q[2] + B[3];
    case WOS_BND_FOURIER5: { /* _kernels.py:262-278 */
      double r = sqrt(q[0] * q[0] + q[1] * q[1]);
      double c = (r == 0.0) ? 1.0 : q[0] / r, s = (r == 0.0) ? 0.0 : q[1] / r;
      return B[0] + B[1] * c + B[2] * s + B[3] * (c * c - s * s) + B[4] * (2.0 * c * s);
    }
    case WOS_BND_FOURIER: {
      const int M = (int)B[0];
      double t = atan2(q[1], q[0]);
      double g = B[1];
      for (int m = 1; m <= M; ++m) g += B[1 + m] * cos(m * t) + B[1 + M + m] * sin(m * t);
      return g;
    }
    case WOS_BND_SQUARE_ARCSINE: {
      double x0 = B[0], y0 = B[1], side = B[2];
      const int M = (int)B[3];
      double u = (q[0] - x0) / side, v = (q[1] - y0) / side;
      /* nearest edge of the unit square in (u, v); CCW arc length in units of side */
      double db = fabs(v), dr = fabs(1.0 - u), dt = fabs(1.0 - v), dl = fabs(u);
      double s;
      if (db <= dr && db <= dt && db <= dl) s = u;
      else if (dr <= dt && dr <= dl) s = 1.0 + v;
      else if (dt <= dl) s = 2.0 + (1.0 - u);
      else s = 3.0 + (1.0 - v);
      double g = 0.0;
      for (int m = 1; m <= M; ++m) g += B[3 + m] * sin(TWO_PI * m * s / 4.0);
      return g;
    }
    case WOS_BND_QUADRATIC:
      return B[0] * q[0] * q[0] + B[1] * q[1] * q[1] + B[2] * q[0] * q[1] + B[3] * q[0] +
             B[4] * q[1] + B[5];
    default:
      return 0.0;
  }
}

/* ------------------------------------------------------------------ */
/* Delta tracking (walker.py:322-418, _kernels.py:476-558,             */
/* greens.py:100-193, pde.py:138-213)                                  */
/* ------------------------------------------------------------------ */
void oracle_native_keys(uint64_t seed, uint64_t ikey, uint32_t* k0, uint32_t* k1);
#define oracle_native_keys_fwd oracle_native_keys
static double u23(uint32_t w);
static double g_sigma_bar = 0.0; /* WalkConfig.sigma_bar for the screened walks */
static double g_majorant = -1.0; /* worst sigma' > sigma_bar met (walker.py:409-413) */
static pthread_mutex_t g_mu = PTHREAD_MUTEX_INITIALIZER;

void oracle_set_sigma_bar(double s) {
  g_sigma_bar = s;
  g_majorant = -1.0;
}
double oracle_majorant(void) { return g_majorant; }

/* pde._vc_log_alpha (pde.py:138-151): h, grad h, lap h with a = 4 pi phi, b = 3 pi phi */
static void vc_log_alpha(double phi, const double* x, double* h, double* g, double* lap) {
  const double a = 4.0 * PI * phi, b = 3.0 * PI * phi;
  const double ca = cos(a * x[0]), sa = sin(a * x[0]), cb = cos(b * x[1]), sb = sin(b * x[1]);
  *h = -x[1] * x[1] + ca * sb;
  g[0] = -a * sa * sb;
  g[1] = -2.0 * x[1] + b * ca * cb;
  g[2] = 0.0;
  *lap = -2.0 - (a * a + b * b) * ca * sb;
}
/* pde._vc_solution (pde.py:154-173) */
static void vc_solution(double phi, const double* x, double* u, double* gu, double* lu) {
  const double p = PI * phi;
  const double s1 = sin(p * x[0]), c1 = cos(p * x[0]);
  const double s2 = sin(2.0 * p * x[1]), c2 = cos(2.0 * p * x[1]);
  const double s3 = sin(3.0 * p * x[2]);
  *u = s1 * c2 + (1.0 - c1) * (1.0 - s2) + s3 * s3;
  if (gu) {
    gu[0] = p * c1 * c2 + p * s1 * (1.0 - s2);
    gu[1] = -2.0 * p * s1 * s2 - 2.0 * p * (1.0 - c1) * c2;
    gu[2] = 3.0 * p * sin(6.0 * p * x[2]);
    *lu = -p * p * s1 * c2 + p * p * c1 * (1.0 - s2) - 4.0 * p * p * s1 * c2 +
          4.0 * p * p * (1.0 - c1) * s2 + 18.0 * p * p * cos(6.0 * p * x[2]);
  }
}
/* pde._vc_sigma, _vc_sigma_prime, _vc_source(_prime), _vc_sqrt_alpha (pde.py:176-212) */
static void vc_coeffs(const double* P, const double* y, double* sp, double* fp) {
  double h, gh[3], lh, u, gu[3], lu;
  vc_log_alpha(P[0], y, &h, gh, &lh);
  const double sigma =
      P[1] + (P[2] - P[1]) * (1.0 + 0.5 * sin(2.0 * PI * y[0]) * cos(0.5 * PI * y[1]));
  *sp = sigma * exp(-h) + 0.5 * lh + 0.25 * (gh[0] * gh[0] + gh[1] * gh[1] + gh[2] * gh[2]);
  vc_solution(P[0], y, &u, gu, &lu);
  const double alpha = exp(h);
  const double f = -alpha * lu - alpha * (gh[0] * gu[0] + gh[1] * gu[1] + gh[2] * gu[2]) + sigma * u;
  *fp = f / exp(0.5 * h);
}
static double vc_solution_u(double phi, const double* x) {
  double u;
  vc_solution(phi, x, &u, NULL, NULL);
  return u;
}
static double vc_sqrt_alpha(double phi, const double* x) {
  double h, g[3], lap;
  vc_log_alpha(phi, x, &h, g, &lap);
  return exp(0.5 * h);
}
/* greens.radial_event_cdf / _kernels._radial_cdf */
static double radial_cdf(double q, double t) {
  if (q < 1.0e-4) return t * t * (3.0 - 2.0 * t);
  return (sinh(q) - q * t * cosh(q * (1.0 - t)) - sinh(q * (1.0 - t))) / (sinh(q) - q);
}
/* greens.invert_radial_event_cdf: fixed 64-step bisection */
static double invert_bisect(double q, double u) {
  double lo = 0.0, hi = 1.0;
  for (int it = 0; it < 64; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (radial_cdf(q, mid) < u) lo = mid;
    else hi = mid;
  }
  return 0.5 * (lo + hi);
}
static void note_majorant(double sp) {
  pthread_mutex_lock(&g_mu);
  if (sp > g_majorant) g_majorant = sp;
  pthread_mutex_unlock(&g_mu);
}

/* One delta-tracking walk. native = 0: the reference's Philox4x64 layout and the
 * 64-step bisection; const coefficients follow _kernels.walk_screened_ball3 (early
 * exit of a dead walk), the family follows walker._screened_generic. native = 1: the
 * product's NATIVE layout (one Philox4x32 block: x event, y direction z, z direction
 * phi, w radius) with the radial CDF inverted to convergence. */
static void walk_screened_one(const wos_problem* pb, const double* x0, uint64_t pid,
                              uint64_t tid, double sgn, uint64_t seed, double eps,
                              int64_t max_steps, int native, double* value, int64_t* steps,
                              uint8_t* hit) {
  const double sigma_bar = g_sigma_bar, sqrt_sig = sqrt(sigma_bar);
  const int vc = pb->src_kind == WOS_SRC_SCREENED_VC;
  const double* P = pb->src;
  const double sa0 = vc ? vc_sqrt_alpha(P[0], x0) : P[3];
  double x[3] = {x0[0], x0[1], x0[2]}, q[3], acc = 0.0, thr = 1.0;
  uint32_t k0n = 0, k1n = 0;
  if (native) oracle_native_keys_fwd(seed, pb->instance_key, &k0n, &k1n);
  const uint32_t c1 = (uint32_t)pid, c2 = (uint32_t)tid;
  const uint32_t c3 = (uint32_t)(tid >> 32) ^ ((uint32_t)(pid >> 32) * 0x85EBCA6Bu);
  for (int64_t step = 0;; ++step) {
    const double d = query(pb, x, q);
    const int shell = d < eps;
    if (shell || step >= max_steps) {
      const double g = vc ? vc_sqrt_alpha(P[0], q) * (vc_solution_u(P[0], q)) : pb->bnd[0];
      *value = (acc + thr * g) / sa0;
      *steps = step;
      *hit = (uint8_t)shell;
      return;
    }
    if (!vc && thr == 0.0 && P[2] == 0.0) { /* _kernels.py:533-538 */
      *value = acc / sa0;
      *steps = step;
      *hit = 1;
      return;
    }
    double qq = sqrt_sig * d;
    if (qq > 500.0) qq = 500.0;
    const double surf = qq < 1.0e-6 ? 1.0 - qq * qq / 6.0 : qq / sinh(qq);
    double ue, uz, uphi, ur;
    if (native) {
      uint32_t ca[4] = {c1, (uint32_t)(2 * step), c2, c3}, u[4];
      philox4x32(ca, k0n, k1n, u);
      ue = u23(u[0]);
      uz = u23(u[1]);
      uphi = u23(u[2]);
      ur = u23(u[3]) + 0x1p-24;
    } else {
      uint64_t c[4] = {2 * (uint64_t)step, pid, tid, 0}, w[4];
      philox4x64(c, seed, pb->instance_key, w);
      ue = u53(w[0]);
      uz = u53(w[1]);
      uphi = u53(w[2]);
      ur = u53(w[3]);
    }
    const double z = 2.0 * uz - 1.0; /* walker._sphere_dirs_3d */
    const double s = sqrt(fmax(0.0, 1.0 - z * z));
    const double phi = TWO_PI * uphi - (native ? PI : 0.0);
    const double dir[3] = {s * cos(phi), s * sin(phi), z};
    const int vol = ue >= surf;
    const double rad = vol ? d * invert_bisect(qq, ur) : d;
    for (int i = 0; i < 3; ++i) x[i] += sgn * rad * dir[i];
    if (vol) {
      double sp, fp = 0.0;
      int has_f = 1;
      if (vc) {
        vc_coeffs(P, x, &sp, &fp);
      } else {
        sp = P[0];
        fp = P[1];
        has_f = P[2] != 0.0;
      }
      if (sp > sigma_bar) note_majorant(sp);
      if (has_f) acc += thr * fp / sigma_bar;
      thr *= 1.0 - sp / sigma_bar;
    }
  }
}

/* ------------------------------------------------------------------ */
/* One reference-form trajectory (walker.py:257-314)                   */
/* ------------------------------------------------------------------ */
static void walk_ref_one(const wos_problem* pb, const double* x0, uint64_t pid, uint64_t tid,
                         double sgn, uint64_t seed, double eps, int64_t max_steps,
                         double* value, int64_t* steps, uint8_t* hit) {
  if (pb->src_kind == WOS_SRC_SCREENED_CONST || pb->src_kind == WOS_SRC_SCREENED_VC) {
    walk_screened_one(pb, x0, pid, tid, sgn, seed, eps, max_steps, 0, value, steps, hit);
    return;
  }
  const int dim = pb->dim;
  const int has_src = pb->src_kind != WOS_SRC_NONE;
  const uint64_t k0 = seed, k1 = pb->instance_key;
  double x[3] = {0, 0, 0}, q[3], acc = 0.0;
  for (int i = 0; i < dim; ++i) x[i] = x0[i];
  for (int64_t step = 0;; ++step) {
    double d = query(pb, x, q);
    int shell = d < eps;
    if (shell || step >= max_steps) { /* walker.py:275-281 */
      *value = acc + boundary(pb, q);
      *steps = step;
      *hit = (uint8_t)shell;
      return;
    }
    uint64_t draw = 2 * (uint64_t)step;
    uint64_t c[4] = {draw, pid, tid, 0}, w[4];
    philox4x64(c, k0, k1, w); /* walker.py:289 */
    double dir[3];
    if (dim == 2) {
      double theta = TWO_PI * u53(w[0]); /* _sphere_dirs_2d, walker.py:245-247 */
      dir[0] = cos(theta);
      dir[1] = sin(theta);
      if (has_src) { /* walker.py:292-298 */
        double u_rad = nonzero_u(u53(w[2]), draw, pid, tid, k0, k1);
        double rad = d * sqrt(u_rad);
        double phi = TWO_PI * u53(w[1]);
        double g[2] = {x[0] + sgn * rad * cos(phi), x[1] + sgn * rad * sin(phi)};
        double green = INV_TWO_PI * log(d / rad);
        acc -= PI * d * d * source(pb, g) * green;
      }
    } else {
      double z = 2.0 * u53(w[0]) - 1.0; /* _sphere_dirs_3d, walker.py:250-254 */
      double s = sqrt(fmax(0.0, 1.0 - z * z));
      double phi = TWO_PI * u53(w[1]);
      dir[0] = s * cos(phi);
      dir[1] = s * sin(phi);
      dir[2] = z;
      if (has_src) { /* walker.py:300-311 */
        uint64_t cb[4] = {draw + 1, pid, tid, 0}, wb[4];
        philox4x64(cb, k0, k1, wb);
        double u_rad = nonzero_u(u53(wb[0]), draw + 1, pid, tid, k0, k1);
        double rad = d * cbrt(u_rad);
        double vz = 2.0 * u53(w[2]) - 1.0;
        double vs = sqrt(fmax(0.0, 1.0 - vz * vz));
        double vphi = TWO_PI * u53(w[3]);
        double g[3] = {x[0] + sgn * rad * (vs * cos(vphi)), x[1] + sgn * rad * (vs * sin(vphi)),
                       x[2] + sgn * rad * vz};
        double green = INV_FOUR_PI * (1.0 / rad - 1.0 / d);
        double vol = (4.0 / 3.0) * PI * pow(d, 3.0);
        acc -= vol * source(pb, g) * green;
      }
    }
    for (int i = 0; i < dim; ++i) x[i] += sgn * d * dir[i]; /* walker.py:312 */
  }
}

/* ------------------------------------------------------------------ */
/* One NATIVE_F32-form trajectory, fp64 arithmetic                     */
/* ------------------------------------------------------------------ */
static double u23(uint32_t w) { return (double)(w >> 9) * (1.0 / 8388608.0); }

void oracle_native_keys(uint64_t seed, uint64_t ikey, uint32_t* k0, uint32_t* k1) {
  *k0 = (uint32_t)seed;
  *k1 = (uint32_t)(seed >> 32) ^ (uint32_t)ikey ^ ((uint32_t)(ikey >> 32) * 0x9E3779B9u);
}

/* a 13-bit field, midpoint-rounded: (b + 1/2) 2^-13 */
static double u13(uint32_t b) { return ((double)(b & 0x1FFFu) + 0.5) * (1.0 / 8192.0); }

/* the Beta(2,2) conditional-mean table of include/wos_beta_table.h, built once */
static float g_beta_tab[WOS_BETA_TABLE_N], g_green2_tab[WOS_BETA_TABLE_N];
static pthread_once_t g_beta_once = PTHREAD_ONCE_INIT;
static void build_tables(void) {
  wos_beta22_table(g_beta_tab);
  wos_green2_table(g_green2_tab);
}
static const float* beta_table(void) {
  pthread_once(&g_beta_once, build_tables);
  return g_beta_tab;
}
static const float* green2_table(void) {
  pthread_once(&g_beta_once, build_tables);
  return g_green2_tab;
}

void oracle_beta_table(float* out) {
  const float* t = beta_table();
  for (int k = 0; k < WOS_BETA_TABLE_N; ++k) out[k] = t[k];
}

void oracle_green2_table(float* out) {
  const float* t = green2_table();
  for (int k = 0; k < WOS_BETA_TABLE_N; ++k) out[k] = t[k];
}

static void walk_native_one(const wos_problem* pb, const double* x0, uint64_t pid, uint64_t tid,
                            double sgn, uint64_t seed, double eps, int64_t max_steps,
                            double* value, int64_t* steps, uint8_t* hit) {
  if (pb->src_kind == WOS_SRC_SCREENED_CONST || pb->src_kind == WOS_SRC_SCREENED_VC) {
    walk_screened_one(pb, x0, pid, tid, sgn, seed, eps, max_steps, 1, value, steps, hit);
    return;
  }
  const int dim = pb->dim;
  const int has_src = pb->src_kind != WOS_SRC_NONE;
  uint32_t k0, k1;
  oracle_native_keys(seed, pb->instance_key, &k0, &k1);
  const uint32_t c1 = (uint32_t)pid, c2 = (uint32_t)tid;
  const uint32_t c3 = (uint32_t)(tid >> 32) ^ ((uint32_t)(pid >> 32) * 0x85EBCA6Bu);
  double x[3] = {0, 0, 0}, q[3], acc = 0.0;
  for (int i = 0; i < dim; ++i) x[i] = x0[i];
  for (int64_t step = 0;; ++step) {
    double d = query(pb, x, q);
    int shell = d < eps;
    if (shell || step >= max_steps) {
      *value = acc + boundary(pb, q);
      *steps = step;
      *hit = (uint8_t)shell;
      return;
    }
    /* Philox4x32 blocks at counter (pid, 2*floor(s/per), tid, hi-words): a source-free
       jump needs one word (2D) or two (3D), a source jump two, so a block serves
       per = 4 / 2 / 2 consecutive jumps (wos_walk.cuh kPerBlock) */
    const int per = has_src ? 2 : (dim == 2 ? 4 : 2);
    const int sub = (int)(step % per);
    uint32_t u[4];
    {
      uint32_t ca[4] = {c1, (uint32_t)(2 * (step / per)), c2, c3};
      philox4x32(ca, k0, k1, u);
    }
    double dir[3];
    if (dim == 2 && !has_src) {
      double th = TWO_PI * u23(u[sub]) - PI;
      dir[0] = cos(th);
      dir[1] = sin(th);
    } else if (dim == 2) {
      /* layout v4 (wos_walk.cuh jump_source, 2D): words (u[0], u[1]) for an even step,
         (u[2], u[3]) for an odd one; theta = bits 19..31 and phi = bits 6..18 of the
         first word, the radius fraction from the disk Green's-law table at index
         (wb >> 26) | (wa & 63) << 6 */
      const uint32_t wa = u[2 * sub], wb = u[2 * sub + 1];
      double th = TWO_PI * u13(wa >> 19) - PI;
      dir[0] = cos(th);
      dir[1] = sin(th);
      double phi = TWO_PI * u13(wa >> 6) - PI;
      double r = d * (double)green2_table()[(wb >> 26) | ((wa & 0x3Fu) << 6)];
      double g[2] = {x[0] + sgn * r * cos(phi), x[1] + sgn * r * sin(phi)};
      acc -= (d * d * 0.25) * source(pb, g);
    } else if (!has_src) {
      double z = 2.0 * u23(u[2 * sub]) - 1.0;
      double s = sqrt(fmax(0.0, 1.0 - z * z));
      double phi = TWO_PI * u23(u[2 * sub + 1]) - PI;
      dir[0] = s * cos(phi);
      dir[1] = s * sin(phi);
      dir[2] = z;
    } else {
      /* layout v4 (wos_walk.cuh jump_source): 64 bits per jump, words (u[0], u[1]) for
         an even step, (u[2], u[3]) for an odd one; 13-bit midpoint-rounded direction
         fields (wa: z bits 6..18, phi bits 19..31; wb: z' bits 0..12, phi' bits 13..25)
         and a 12-bit index (wb >> 26) | (wa & 63) << 6 into the Beta(2,2)
         conditional-mean table */
      const uint32_t wa = u[2 * sub], wb = u[2 * sub + 1];
      double z = 2.0 * u13(wa >> 6) - 1.0;
      double s = sqrt(fmax(0.0, 1.0 - z * z));
      double phi = TWO_PI * u13(wa >> 19) - PI;
      dir[0] = s * cos(phi);
      dir[1] = s * sin(phi);
      dir[2] = z;
      double vz = 2.0 * u13(wb & 0x1FFFu) - 1.0;
      double vs = sqrt(fmax(0.0, 1.0 - vz * vz));
      double vphi = TWO_PI * u13(wb >> 13) - PI;
      double t = (double)beta_table()[(wb >> 26) | ((wa & 0x3Fu) << 6)];
      double r = d * t;
      double g[3] = {x[0] + sgn * r * (vs * cos(vphi)), x[1] + sgn * r * (vs * sin(vphi)),
                     x[2] + sgn * r * vz};
      acc -= (d * d * (1.0 / 6.0)) * source(pb, g);
    }
    for (int i = 0; i < dim; ++i) x[i] += sgn * d * dir[i];
  }
}

/* ------------------------------------------------------------------ */
/* Threaded drivers                                                     */
/* ------------------------------------------------------------------ */
typedef struct {
  const wos_problem* pb;
  int native;
  int64_t lo, hi;
  const double* pts;
  const uint64_t *pid, *tid;
  const double* sgn;
  uint64_t seed;
  double eps;
  int64_t max_steps;
  double* values;
  int64_t* steps;
  uint8_t* hits;
} rows_job;

static void* rows_worker(void* arg) {
  rows_job* j = (rows_job*)arg;
  const int dim = j->pb->dim;
  for (int64_t i = j->lo; i < j->hi; ++i) {
    if (j->native)
      walk_native_one(j->pb, j->pts + dim * i, j->pid[i], j->tid[i], j->sgn[i], j->seed, j->eps,
                      j->max_steps, j->values + i, j->steps + i, j->hits + i);
    else
      walk_ref_one(j->pb, j->pts + dim * i, j->pid[i], j->tid[i], j->sgn[i], j->seed, j->eps,
                   j->max_steps, j->values + i, j->steps + i, j->hits + i);
  }
  return NULL;
}

static int run_rows(const wos_problem* pb, int native, int64_t n, const double* pts,
                    const uint64_t* pid, const uint64_t* tid, const double* sgn, uint64_t seed,
                    double eps, int64_t max_steps, double* values, int64_t* steps, uint8_t* hits,
                    int nthreads) {
  g_polar_native = native;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  rows_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    rows_job j = {pb, native, n * t / nthreads, n * (t + 1) / nthreads, pts, pid, tid, sgn,
                  seed, eps, max_steps, values, steps, hits};
    jobs[t] = j;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, rows_worker, &jobs[t]);
  rows_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* walker.walk_poisson_values on the reference form (walker.py:181-229, generic path) */
int oracle_walk_rows(const wos_problem* pb, int64_t n, const double* pts, const uint64_t* pid,
                     const uint64_t* tid, const double* sgn, uint64_t seed, double eps,
                     int64_t max_steps, double* values, int64_t* steps, uint8_t* hits,
                     int nthreads) {
  return run_rows(pb, 0, n, pts, pid, tid, sgn, seed, eps, max_steps, values, steps, hits,
                  nthreads);
}

int oracle_walk_rows_native(const wos_problem* pb, int64_t n, const double* pts,
                            const uint64_t* pid, const uint64_t* tid, const double* sgn,
                            uint64_t seed, double eps, int64_t max_steps, double* values,
                            int64_t* steps, uint8_t* hits, int nthreads) {
  return run_rows(pb, 1, n, pts, pid, tid, sgn, seed, eps, max_steps, values, steps, hits,
                  nthreads);
}

typedef struct {
  const wos_problem* pbs;
  int native;
  int64_t lo, hi;
  const double* pts;
  const int64_t* pid;
  const int32_t* inst;
  int64_t L;
  uint64_t traj_start;
  int antithetic;
  uint64_t seed;
  double eps;
  int64_t max_steps;
  double *mean, *m2;
  uint64_t total_steps;
} est_job;

static void* est_worker(void* arg) {
  est_job* j = (est_job*)arg;
  const int64_t L = j->L;
  double* v = (double*)malloc(sizeof(double) * (size_t)L);
  uint64_t tot = 0;
  for (int64_t p = j->lo; p < j->hi; ++p) {
    const wos_problem* pb = j->pbs + (j->inst ? j->inst[p] : 0);
    const double* x0 = j->pts + pb->dim * p;
    for (int64_t r = 0; r < L; ++r) {
      uint64_t tid = j->antithetic ? j->traj_start + 2 * (uint64_t)(r / 2) : j->traj_start + (uint64_t)r;
      double sgn = (j->antithetic && (r & 1)) ? -1.0 : 1.0;
      int64_t st;
      uint8_t h;
      if (j->native)
        walk_native_one(pb, x0, (uint64_t)j->pid[p], tid, sgn, j->seed, j->eps, j->max_steps,
                        v + r, &st, &h);
      else
        walk_ref_one(pb, x0, (uint64_t)j->pid[p], tid, sgn, j->seed, j->eps, j->max_steps, v + r,
                     &st, &h);
      tot += (uint64_t)st;
    }
    int64_t n = L;
    if (j->antithetic) { /* estimator.py:137-139: pair means */
      n = L / 2;
      for (int64_t k = 0; k < n; ++k) v[k] = (v[2 * k] + v[2 * k + 1]) / 2.0;
    }
    double s = 0.0; /* PointEstimate.from_values, estimator.py:106-110 */
    for (int64_t k = 0; k < n; ++k) s += v[k];
    double mean = s / (double)n, m2 = 0.0;
    for (int64_t k = 0; k < n; ++k) m2 += (v[k] - mean) * (v[k] - mean);
    j->mean[p] = mean;
    j->m2[p] = m2;
  }
  free(v);
  j->total_steps = tot;
  return NULL;
}

/* estimator.estimate (estimator.py:144-181) over a multi-instance point list */
int oracle_estimate(const wos_problem* pbs, int native, int64_t P, const double* pts,
                    const int64_t* pid, const int32_t* inst, int64_t L, uint64_t traj_start,
                    int antithetic, uint64_t seed, double eps, int64_t max_steps, double* mean,
                    double* m2, uint64_t* total_steps, int nthreads) {
  g_polar_native = native;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  est_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    est_job j = {pbs, native, P * t / nthreads, P * (t + 1) / nthreads, pts, pid, inst, L,
                 traj_start, antithetic, seed, eps, max_steps, mean, m2, 0};
    jobs[t] = j;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, est_worker, &jobs[t]);
  est_worker(&jobs[0]);
  uint64_t tot = jobs[0].total_steps;
  for (int t = 1; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    tot += jobs[t].total_steps;
  }
  if (total_steps) *total_steps = tot;
  return 0;
}
