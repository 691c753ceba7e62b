// Persistent Walk-on-Spheres kernel for sm_100a.
//
// One template covers every (mode, dimension, domain, source) combination; the
// boundary term is a runtime switch because it runs once per walk.
//
// Execution model:
//   * persistent grid (SMs x resident CTAs), 8 warps per CTA;
//   * every warp owns a stream of walks ("items", point-major) that it pulls
//     from a global work counter in units of >= 128 walks;
//   * each lane carries one walk in registers (position, Green accumulator,
//     step, RNG counter words); when lanes finish (eps-shell hit or max_steps)
//     they are refilled with the next items of the warp's stream (lane refill),
//     so lanes do not idle while work remains; closed-form domains run the loop
//     jump-first (jump with the carried distance, query, finish at once);
//   * a finished walk with a non-constant boundary term is recorded at the next
//     refill together with the other finished lanes (deferred recording);
//   * ESTIMATE sink: walk values go to a per-warp shared-memory ring indexed by
//     the item's stream position; a unit (whole points for L <= 128, else a
//     128-walk chunk of one point) is reduced as soon as all its walks are done,
//     in fixed index order with fp64 warp-shuffle trees (two-pass mean / m2,
//     PointEstimate.from_values, estimator.py:106-110); chunks of long ensembles
//     are Chan-merged in chunk order by a second small kernel. The result does not
//     depend on which lane ran which walk, on the launch shape, or on the number
//     of GPUs;
//   * ROWS sink: per-walk (value, steps, hit) written straight to global memory
//     (walker.walk_poisson_values, walker.py:181-229).
//
// Numerics per mode:
//   REPLAY_F64 / REPLAY_F32 follow walker._poisson_generic (walker.py:257-314)
//   operation by operation, on Philox4x64 draws identical to the reference's.
//   NATIVE_F32 samples the source term from the ball Green's function (radius
//   fraction from a 12-bit table of the disk Green's law in 2D, of Beta(2,2) in 3D)
//   with weight r^2/(2 dim) (greens.py:83-89), uses MUFU sin/cos/sqrt/ex2, and
//   Philox4x32 blocks at counter (pid, 2 floor(step / jumps per block), tid,
//   hi-words) (10 rounds, or 7 with WalkConfig.philox_rounds = 7);
//   a source jump takes 64 bits (two jumps per block; jump_source below, with the
//   radius from a staged table; oracle/wos_oracle.c restates it);
//   source-free jumps share a block between 4 (2D) / 2 (3D) consecutive jumps
//   (kPerBlock; phase-locked amortised rounds on closed-form domains). Direction
//   angles are 2 pi u - pi (MUFU's accurate range). Single-instance NATIVE launches
//   (ONE) read the instance row and the Philox round keys from the kernel
//   parameters, kept in uniform registers; those with a constant boundary are
//   built without the deferral code (Spec BC), and box + monomial-sine ones walk
//   in scaled coordinates X = pi x (kScaled).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "wos_rng.cuh"
#include "wos_mesh.cuh"
#include "wos_types.h"

namespace wos {

#define WOS_FULL 0xffffffffu
#ifndef WOS_DEEP_STATS
#define WOS_DEEP_STATS 0
#endif
#ifndef WOS_DEEP_T
#define WOS_DEEP_T 8
#endif
#ifndef WOS_POLY_UNROLL4
#define WOS_POLY_UNROLL4 1
#endif
// polar / mesh walks keep the closest point of their last distance query for project()
#ifndef WOS_KEEP_CLOSEST
#define WOS_KEEP_CLOSEST 1
#endif
#ifndef WOS_KEEP_CLOSEST_MESH
#define WOS_KEEP_CLOSEST_MESH 1
#endif

// ------------------------------------------------------------------------
// math helpers
// ------------------------------------------------------------------------
__device__ __forceinline__ float fast_sqrt(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float fast_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// (w >> 9) | 1.0f  ->  [1, 2); u = f - 1 = (w >> 9) 2^-23 exactly (one LEA.HI)
__device__ __forceinline__ float f12(uint32_t w) { return __uint_as_float(0x3f800000u | (w >> 9)); }
// the same 23 bits with exponent 2^1: 2 f exactly, so z = 2u - 1 = f2(w) - 3 takes one FADD
__device__ __forceinline__ float f2x(uint32_t w) { return __uint_as_float(0x40000000u | (w >> 9)); }

constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 6.283185307179586;
constexpr double kInvTwoPi = 1.0 / 6.283185307179586;
constexpr double kInvFourPi = 1.0 / (4.0 * 3.141592653589793);
constexpr float kTwoPiF = 6.283185307179586f;
constexpr float kThreePiF = 9.42477796076938f;
// NATIVE direction angle 2 pi u - pi in [-pi, pi) from a 23-bit field f = 1 + u: the
// range on which MUFU.SIN/COS keep their 2^-21.4 bound (2^-20.4 on [0, 2 pi);
// tests/test_gpu_fastmath.py). Uniform in angle either way.
__device__ __forceinline__ float dir_angle(float f) { return fmaf(f, kTwoPiF, -kThreePiF); }
constexpr float kPiF = 3.141592653589793f;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void psincos(double a, double* s, double* c) { sincos(a, s, c); }
__device__ __forceinline__ void psincos(float a, float* s, float* c) { sincosf(a, s, c); }
__device__ __forceinline__ double psin(double a) { return sin(a); }
__device__ __forceinline__ float psin(float a) { return sinf(a); }
__device__ __forceinline__ double pcos(double a) { return cos(a); }
__device__ __forceinline__ float pcos(float a) { return cosf(a); }
__device__ __forceinline__ double psqrt(double a) { return sqrt(a); }
__device__ __forceinline__ float psqrt(float a) { return sqrtf(a); }
__device__ __forceinline__ double plog(double a) { return log(a); }
__device__ __forceinline__ float plog(float a) { return logf(a); }
__device__ __forceinline__ double pcbrt(double a) { return cbrt(a); }
__device__ __forceinline__ float pcbrt(float a) { return cbrtf(a); }
__device__ __forceinline__ double pexp(double a) { return exp(a); }
__device__ __forceinline__ float pexp(float a) { return expf(a); }
__device__ __forceinline__ double pmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ float pmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double pmax(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ float pmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double pabs(double a) { return fabs(a); }
__device__ __forceinline__ float pabs(float a) { return fabsf(a); }

// BC_: single-instance launch of a problem whose boundary value is a constant
// (a.bnd_c): the walk value is acc + g with no projection, so the kernel carries
// no deferred-recording code (it only costs registers and issue there)
// RND_: NATIVE Philox4x32 rounds fixed at compile time (the single-instance estimate
// kernels are built for 10 and for 7); 0 = read KArgs::philox_rounds at run time
template <int MODE_, int DIM_, int DOM_, int SRC_, int SK_, bool ONE_ = false, int SINK_ = SINK_ESTIMATE,
          bool BC_ = false, int RND_ = 0>
struct Spec {
  static constexpr int MODE = MODE_, DIM = DIM_, DOM = DOM_, SRC = SRC_, SK = SK_, SINK = SINK_;
  static constexpr int RND = RND_;
  static constexpr bool NATIVE = (MODE_ == MODE_NATIVE_F32);
  static constexpr bool ONE = ONE_;
  static constexpr bool BC = BC_;
  static_assert(!BC_ || ONE_, "constant-boundary kernels are single-instance launches");
  using Real = typename std::conditional<MODE_ == MODE_REPLAY_F64, double, float>::type;
  static_assert(!ONE_ || MODE_ == MODE_NATIVE_F32, "single-instance launches are NATIVE only");
};

// ------------------------------------------------------------------------
// the walker
// ------------------------------------------------------------------------
template <class S>
struct Walker {
  using Real = typename S::Real;
  static constexpr int DIM = S::DIM;
  static constexpr bool ONE = S::ONE;

  // (not for polygons, whose segment scan needs the registers, nor for the fp64-heavy
  // delta-tracking step, nor for the ROWS sink)
  static constexpr bool kHot = S::NATIVE && ONE && S::DOM != DOM_POLY && S::SINK == SINK_ESTIMATE &&
                               S::SRC != SRC_SCR_CONST && S::SRC != SRC_SCR_VC;
  static constexpr int kHotK = kHot ? 10 : 1;
  // Exit ring (single-instance source-free 2D estimate kernels with a non-constant
  // boundary: cfg1): a finishing walk stores its exit position (x, y) in its ring slot
  // (8 bytes) and the boundary term g(projection) is evaluated when the unit retires,
  // by all 32 lanes over the unit's slots, instead of by the few lanes that finished
  // since the last refill. Same finish_value() on the same position: identical values.
  static constexpr bool kExitRing = exit_ring_kernel(S::NATIVE, DIM, S::DOM, S::SRC, ONE,
                                                     S::SINK == SINK_ESTIMATE, S::BC);
  static constexpr int kRS = kExitRing ? 2 : 1;  // ring slot size in Reals
  // hot source coefficients: those the jump reads at compile-time offsets
  static constexpr int kHotSrcN =
      !kHot ? 0
      : S::SRC == SRC_CONST ? 1
      : S::SRC == SRC_RBF2 ? 6
      : S::SRC == SRC_GAUSS ? 2 + DIM
      : (S::SRC == SRC_SINE && (S::SK == 3 || S::SK == 4)) ? (DIM == 2 ? S::SK * S::SK : S::SK * S::SK * S::SK)
      : 0;
  static constexpr bool kHotSrc = kHotSrcN > 0;
  static constexpr int kHotC = kHot ? kSrcOff + kHotSrcN : 1;

  struct Lane {
    Real x[DIM];
    Real acc;
    Real sgn;
    const Real* row;  // this walk's instance row in the staged table (shared memory)
    int step;
    Real d;        // distance to the boundary at x (jump-first loop: carried to the next jump)
    uint32_t seq;  // ESTIMATE: byte offset of the walk's ring slot; ROWS: row index
    uint64_t pid, tid, ikey;   // REPLAY counters / key
    uint32_t c1, c2, c3;       // NATIVE kHot: counter words
    PhiloxPre pc;              // other NATIVE: the counter words folded through rounds 0-1
    uint32_t k1;               // NATIVE multi-instance: the instance key
    int32_t seg_off, n_seg, rec_off;
    int32_t seg_i;  // polygon: nearest segment found by the last distance query
    Real cq[DIM];   // polar / mesh: closest boundary point found by the last distance query
    uint32_t nseg = 0;  // NATIVE polygon: segment distances evaluated (work counter)
    Real thr;       // delta tracking: throughput (walker.py:365, _kernels.py:539)
    Real sa;        // delta tracking: sqrt(alpha) at the start point (walker.py:352-354)
    // single-instance NATIVE launches: the Philox round keys and the parameters the
    // jump reads, copied once from the constant bank through a shuffle so that ptxas
    // keeps them in (uniform) registers instead of reloading them every step
    uint32_t hk0[kHotK], hk1[kHotK];
    float hc[kHotC];
  };

  // instance parameters: constant bank (ONE) or the staged shared-memory row
  __device__ static __forceinline__ const Real* prow(const Lane& l, const KArgs& a) {
    if constexpr (ONE) return reinterpret_cast<const Real*>(a.cp);
    else return l.row;
  }
  __device__ static __forceinline__ Real domp(const Lane& l, const KArgs& a, int i) {
    if constexpr (kHot) return l.hc[kDomOff + i];  // i is a compile-time constant here
    else if constexpr (ONE) return (Real)a.cp[kDomOff + i];
    else return l.row[kDomOff + i];
  }

  // ---------------- domains ----------------
  // distance to the boundary (positive inside)
  __device__ static __forceinline__ Real dist(Lane& l, const KArgs& a, const float4* srec) {
    if constexpr (S::DOM == DOM_BALL || S::DOM == DOM_BOX || S::DOM == DOM_CUBE) return dist_at(l, a, l.x);
    else if constexpr (S::DOM == DOM_POLAR) {
      // (the closest point stays in the lane: a walk ends at the position of its last
      // query, so project() needs no second scan — run by the few lanes of a deferred batch)
      if constexpr (WOS_KEEP_CLOSEST) return polar_query(l, a, srec, l.x[0], l.x[1], &l.cq[0], &l.cq[1]);
      Real qx, qy;
      return polar_query(l, a, srec, l.x[0], l.x[1], &qx, &qy);
    } else if constexpr (S::DOM == DOM_MESH) {
      // MeshDomain.boundary_query (geometry.py:527-533): |p - closest|
      if constexpr (WOS_KEEP_CLOSEST_MESH) return psqrt(mesh_d2(l, a, l.cq));
      Real q[3];
      return psqrt(mesh_d2(l, a, q));
    } else {
      return poly_dist(l, a, srec);
    }
  }

  // closed-form domains: distance at any point x (the walk's, or a unit's start point)
  __device__ static __forceinline__ Real dist_at(const Lane& l, const KArgs& a, const Real* x) {
    if constexpr (S::DOM == DOM_BALL) {
      // geometry.py:196-206 / _kernels.py:329-339
      Real s = Real(0);
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        Real u = x[i] - domp(l, a, i);
        if constexpr (S::NATIVE) s = fmaf(u, u, s);
        else s = s + u * u;
      }
      if constexpr (S::NATIVE) return domp(l, a, 3) - fast_sqrt(s);
      else return pabs(domp(l, a, 3) - psqrt(s));
    } else if constexpr (S::DOM == DOM_CUBE) {
      // centred cube in X = pi (x - 1/2): h - max |X_i| (one FMNMX3 with |.| operands)
      Real m = fabsf(x[0]);
#pragma unroll
      for (int i = 1; i < DIM; ++i) m = fmaxf(m, fabsf(x[i]));
      return domp(l, a, 12) - m;
    } else {
      static_assert(S::DOM == DOM_BOX, "dist_at: closed-form domains only");
      if constexpr (S::NATIVE) {
        // min over axes of h_i - |x_i - c_i| (centre at [8, 11), half extent at [12, 15))
        Real d = domp(l, a, 12) - fabsf(x[0] - domp(l, a, 8));
#pragma unroll
        for (int i = 1; i < DIM; ++i) d = fminf(d, domp(l, a, 12 + i) - fabsf(x[i] - domp(l, a, 8 + i)));
        return d;
      } else {
        Real d = x[0] - domp(l, a, 0);
        d = pmin(d, domp(l, a, 4) - x[0]);
#pragma unroll
        for (int i = 1; i < DIM; ++i) {
          d = pmin(d, x[i] - domp(l, a, i));
          d = pmin(d, domp(l, a, 4 + i) - x[i]);
        }
        return d;
      }
    }
  }

  // polygon: min distance over segments; records the first nearest segment in l.seg_i
  // (the closest point is rebuilt from that one segment only at termination)
  // NATIVE records come in segment pairs (wos_capi.cu build): A_j = (x_2j, x_2j+1,
  // y_2j, y_2j+1), U_j = the same pairs of e_k/|e_k|^2, then A_j+1; one closing A
  // holds vertex 0 again. An odd polygon gets a zero-length last segment at vertex 0,
  // which never beats segment 0 (same end point). Both segments of a pair go through
  // packed FADD2/FMUL2/FFMA2 with the scalar seg_d2 operation order, so every
  // distance is bit-identical to seg_d2. The running minimum moves in blocks of 4
  // segments and remembers the first block attaining it (*bi_out = its first
  // segment); poly_project resolves the first nearest segment inside it.
  __device__ static __forceinline__ float seg_d2(float ax, float ay, float nx, float ny, float ux, float uy,
                                                 float px, float py) {
    const float ex = nx - ax, ey = ny - ay;
    const float wx = px - ax, wy = py - ay;
    const float t = __saturatef(fmaf(wx, ux, wy * uy));
    const float dx = fmaf(-t, ex, wx), dy = fmaf(-t, ey, wy);
    return fmaf(dx, dx, dy * dy);
  }

  __device__ static __forceinline__ float2 pair_d2(float4 A, float4 U, float4 An, float px, float py) {
    const float2 ex = make_float2(A.y - A.x, An.x - A.y), ey = make_float2(A.w - A.z, An.z - A.w);
    const float2 wx = __fadd2_rn(make_float2(px, px), make_float2(-A.x, -A.y));
    const float2 wy = __fadd2_rn(make_float2(py, py), make_float2(-A.z, -A.w));
    const float2 sy = __fmul2_rn(wy, make_float2(U.z, U.w));
    const float2 t = make_float2(__saturatef(fmaf(wx.x, U.x, sy.x)), __saturatef(fmaf(wx.y, U.y, sy.y)));
    const float2 nt = make_float2(-t.x, -t.y);
    const float2 dx = __ffma2_rn(nt, ex, wx), dy = __ffma2_rn(nt, ey, wy);
    return __ffma2_rn(dx, dx, __fmul2_rn(dy, dy));
  }

  // segment s of a paired record block: its distance (seg_d2 order) and, optionally,
  // the closest point
  __device__ static __forceinline__ float seg_at(const float4* rec, int s, float px, float py,
                                                 float* qx = nullptr, float* qy = nullptr) {
    const int j = s >> 1;
    const float4 A = __ldg(rec + 2 * j), U = __ldg(rec + 2 * j + 1), An = __ldg(rec + 2 * j + 2);
    const bool odd = s & 1;
    const float ax = odd ? A.y : A.x, ay = odd ? A.w : A.z;
    const float nx = odd ? An.x : A.y, ny = odd ? An.z : A.w;
    const float ux = odd ? U.y : U.x, uy = odd ? U.w : U.z;
    if (qx != nullptr) {
      const float ex = nx - ax, ey = ny - ay;
      const float wx = px - ax, wy = py - ay;
      const float t = __saturatef(fmaf(wx, ux, wy * uy));
      *qx = fmaf(t, ex, ax);
      *qy = fmaf(t, ey, ay);
    }
    return seg_d2(ax, ay, nx, ny, ux, uy, px, py);
  }

  template <class P>
  __device__ static __forceinline__ float poly_scan(const P rec, int n, float px, float py, int* bi_out) {
    float best = 3.0e38f;
    int bi = 0;
    float4 A = rec[0];
    const int m = (n + 1) >> 1;  // segment pairs
    const int m2 = m & ~1;
#pragma unroll 2
    for (int j = 0; j < m2; j += 2) {
      const float4 U0 = rec[2 * j + 1], A1 = rec[2 * j + 2], U1 = rec[2 * j + 3], A2 = rec[2 * j + 4];
      const float2 d01 = pair_d2(A, U0, A1, px, py), d23 = pair_d2(A1, U1, A2, px, py);
      const float mn = fminf(fminf(fminf(d01.x, d01.y), d23.x), d23.y);
      bi = mn < best ? 2 * j : bi;
      best = fminf(best, mn);
      A = A2;
    }
    if (m & 1) {  // last pair
      const int j = m - 1;
      const float2 d = pair_d2(A, rec[2 * j + 1], rec[2 * j + 2], px, py);
      const float mn = fminf(d.x, d.y);
      bi = mn < best ? 2 * j : bi;
      best = fminf(best, mn);
    }
    *bi_out = bi;
    return best;
  }

  // candidate-grid query (wos_capi.cu build_poly_grid): the cell's ascending list of
  // segment pairs; records the exact first nearest segment
  __device__ static __forceinline__ float poly_grid_scan(const float4* __restrict__ R, float4 H0, int G, int cells_off,
                                                         int idx_off, bool bytes8, const uint32_t* __restrict__ gw,
                                                         float px, float py, int* bi_out, uint32_t* n_pairs) {
    const int cx = min(max((int)((px - H0.x) * H0.z), 0), G - 1);
    const int cy = min(max((int)((py - H0.y) * H0.w), 0), G - 1);
    const uint16_t* idx = reinterpret_cast<const uint16_t*>(gw) + idx_off;
    float best = 3.0e38f;
    int bi = 0;
#if WOS_GRID_INLINE
    // the cell record carries its first pair indices (12 as bytes, or 4 as uint16):
    // most queries (near the boundary, where the walks spend their steps) need no
    // index load of their own
    const uint4 C = __ldg(reinterpret_cast<const uint4*>(gw + cells_off) + cy * G + cx);
    const uint32_t e = bytes8 ? (C.x & 0xFFFFu) : C.y;
    *n_pairs = e;
    const uint8_t* idx8 = reinterpret_cast<const uint8_t*>(idx);
#endif
    // The running minimum moves by pairs and remembers the first pair attaining it
    // (*bi_out = its first segment): poly_project rescans from there and takes the first
    // strictly nearest segment, which is the one the segment-by-segment scan records
    // (its pair's first segment wins a tie inside the pair, an earlier pair a tie between
    // pairs) — FMNMX, FSETP, FMNMX, SEL per pair instead of a compare and two selects
    // per segment.
    int bj = 0;
    auto eval = [&](int j) {
      const float2 d = pair_d2(__ldg(R + 2 * j), __ldg(R + 2 * j + 1), __ldg(R + 2 * j + 2), px, py);
      const float m = fminf(d.x, d.y);
      bj = m < best ? j : bj;
      best = fminf(best, m);
    };
#if WOS_GRID_INLINE
    if (bytes8) {
      // byte indices: the twelve inline ones four per word (one PRMT-class extract each,
      // no queue shifting), the rest from the index array
      const uint32_t e0 = min(e, 12u);
      uint32_t w = C.y, w1 = C.z, w2 = C.w;
#if !WOS_POLY_UNROLL4
      for (uint32_t k = 0; k < e0; ++k) {  // (the queue shifted by one byte per pair)
        eval((int)(w & 0xFFu));
        w = __funnelshift_r(w, w1, 8);
        w1 = __funnelshift_r(w1, w2, 8);
        w2 >>= 8;
      }
#else
      for (uint32_t k = 0; k < e0;) {
        eval((int)(w & 0xFFu));
        if (++k >= e0) break;
        eval((int)((w >> 8) & 0xFFu));
        if (++k >= e0) break;
        eval((int)((w >> 16) & 0xFFu));
        if (++k >= e0) break;
        eval((int)(w >> 24));
        ++k;
        w = w1;
        w1 = w2;
      }
#endif
      for (uint32_t k = 12; k < e; ++k) eval((int)__ldg(idx8 + (C.x >> 16) + (k - 12)));
    } else {
      const uint32_t e0 = min(e, 4u);
      for (uint32_t k = 0; k < e0; ++k) {
        const uint32_t wd = k < 2 ? C.z : C.w;
        eval((int)((k & 1) ? (wd >> 16) : (wd & 0xFFFFu)));
      }
      for (uint32_t k = 4; k < e; ++k) eval((int)__ldg(idx + C.x + (k - 4)));
    }
#else
    {
      const uint32_t* cell = gw + cells_off + cy * G + cx;
      const uint32_t b = __ldg(cell), e = __ldg(cell + 1);
      *n_pairs = e - b;
      for (uint32_t k = b; k < e; ++k) eval((int)__ldg(idx + k));
    }
#endif
    bi = 2 * bj;
    *bi_out = bi;
    return best;
  }

  __device__ static __forceinline__ Real poly_dist(Lane& l, const KArgs& a, const float4* srec) {
    if constexpr (S::NATIVE) {
      int bi;
      float best;
      const float4* R = (srec != nullptr ? srec : reinterpret_cast<const float4*>(a.segs)) + l.rec_off;
      const float4 H1 = R[-1];
      const int G = __float_as_int(H1.x);
      if (G > 0) {  // (sets with grids are never staged: R is global)
        uint32_t np;
        best = poly_grid_scan(R, R[-2], G, __float_as_int(H1.y), __float_as_int(H1.z), __float_as_int(H1.w) != 0,
                              reinterpret_cast<const uint32_t*>(a.nodes), l.x[0], l.x[1], &bi, &np);
#if WOS_DEEP_STATS == 1  // (measurement builds: the warp's longest list instead of the lane's)
        l.nseg += 2u * __reduce_max_sync(__activemask(), np);
#elif WOS_DEEP_STATS == 2  // pairs in lists longer than WOS_DEEP_T
        l.nseg += np > WOS_DEEP_T ? 2u * np : 0u;
#elif WOS_DEEP_STATS == 3  // queries with lists longer than WOS_DEEP_T
        l.nseg += np > WOS_DEEP_T ? 2u : 0u;
#elif WOS_DEEP_STATS == 4  // the warp's longest list among those of at most WOS_DEEP_T pairs
        l.nseg += 2u * __reduce_max_sync(__activemask(), np > WOS_DEEP_T ? 0u : np);
#else
        l.nseg += 2u * np;
#endif
      } else {  // R: shared memory when staged, else global
        best = poly_scan(R, l.n_seg, l.x[0], l.x[1], &bi);
        l.nseg += (uint32_t)(((l.n_seg + 1) >> 1) << 1);
      }
      l.seg_i = bi;
      return fast_sqrt(best);
    } else {
      // oracle/wos_oracle.c query(): t = clamp(w.e / e.e, 0, 1), c = a + t e
      const Real* seg = reinterpret_cast<const Real*>(a.segs) + 4 * (size_t)l.seg_off;
      const Real px = l.x[0], py = l.x[1];
      Real best = sizeof(Real) == 8 ? Real(1e300) : Real(3e38);
      int bi = 0;
      const int n = l.n_seg;
      for (int i = 0; i < n; ++i) {
        const Real ax = seg[4 * i], ay = seg[4 * i + 1], ex = seg[4 * i + 2], ey = seg[4 * i + 3];
        const Real wx = px - ax, wy = py - ay;
        Real t = (wx * ex + wy * ey) / (ex * ex + ey * ey);
        t = t < Real(0) ? Real(0) : (t > Real(1) ? Real(1) : t);
        const Real cx = ax + t * ex, cy = ay + t * ey;
        const Real dx = px - cx, dy = py - cy;
        const Real d2 = dx * dx + dy * dy;
        if (d2 < best) {
          best = d2;
          bi = i;
        }
      }
      l.seg_i = bi;
      return psqrt(best);
    }
  }

  // closest point on the segment recorded by the last distance query (NATIVE: the
  // first nearest segment of the recorded block of 4, or of the last pair)
  __device__ static __forceinline__ void poly_project(const Lane& l, const KArgs& a, Real* q) {
    const int i0 = l.seg_i;
    if constexpr (S::NATIVE) {
      const float4* rec = reinterpret_cast<const float4*>(a.segs) + l.rec_off;
      const int np = ((l.n_seg + 1) >> 1) << 1;  // segments incl. the odd polygon's pad
      int bi = i0;
      if (__float_as_int(__ldg(rec - 1).x) > 0) {
        // candidate grid: i0 is the first segment of the nearest pair; the second one wins
        // only if strictly nearer (pair_d2 = seg_d2 bit for bit); the closest point from
        // the same three records, in seg_at's operation order
        const int j = i0 >> 1;
        const float4 A = __ldg(rec + 2 * j), U = __ldg(rec + 2 * j + 1), An = __ldg(rec + 2 * j + 2);
        const float2 d = pair_d2(A, U, An, l.x[0], l.x[1]);
        const bool odd = d.y < d.x;
        const float ax = odd ? A.y : A.x, ay = odd ? A.w : A.z;
        const float nx = odd ? An.x : A.y, ny = odd ? An.z : A.w;
        const float ux = odd ? U.y : U.x, uy = odd ? U.w : U.z;
        const float ex = nx - ax, ey = ny - ay;
        const float wx = l.x[0] - ax, wy = l.x[1] - ay;
        const float t = __saturatef(fmaf(wx, ux, wy * uy));
        q[0] = fmaf(t, ex, ax);
        q[1] = fmaf(t, ey, ay);
        return;
      } else {  // block scan: the first nearest segment of the recorded block of 4
        const int i1 = min(i0 + 4, np);
        float best = 3.0e38f;
        for (int i = i0; i < i1; ++i) {
          const float d = seg_at(rec, i, l.x[0], l.x[1]);
          if (d < best) {
            best = d;
            bi = i;
          }
        }
      }
      float qx, qy;
      seg_at(rec, bi, l.x[0], l.x[1], &qx, &qy);
      q[0] = qx;
      q[1] = qy;
    } else {
      const int i = i0;
      const Real* seg = reinterpret_cast<const Real*>(a.segs) + 4 * (size_t)l.seg_off;
      const Real ax = seg[4 * i], ay = seg[4 * i + 1], ex = seg[4 * i + 2], ey = seg[4 * i + 3];
      const Real wx = l.x[0] - ax, wy = l.x[1] - ay;
      Real t = (wx * ex + wy * ey) / (ex * ex + ey * ey);
      t = t < Real(0) ? Real(0) : (t > Real(1) ? Real(1) : t);
      q[0] = ax + t * ex;
      q[1] = ay + t * ey;
    }
  }

  // closest boundary point at termination
  __device__ static __forceinline__ void project(const Lane& l, const KArgs& a, Real* q) {
    if constexpr (S::DOM == DOM_BALL && S::NATIVE) {
      // q = c + R u / |u| with one MUFU rsqrt (2^-22 relative: far below the Monte Carlo
      // error of g(q)); explicit FMAs: every kernel variant (estimate or rows sink,
      // single- or multi-instance) rounds the projection alike. |u| = 0 (or subnormal,
      // flushed): the +x axis point, as the reference (geometry.py:196-206)
      float s = 0.0f, u[DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        u[i] = l.x[i] - domp(l, a, i);
        s = fmaf(u[i], u[i], s);
      }
      float inv;
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(s));
      const bool zero = !(s > 0.0f) || !(inv < 3.0e38f);
      const float R = domp(l, a, 3);
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        const float dir = zero ? (i == 0 ? 1.0f : 0.0f) : u[i] * inv;
        q[i] = fmaf(R, dir, domp(l, a, i));
      }
    } else if constexpr (S::DOM == DOM_BALL) {
      Real s = Real(0), u[DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        u[i] = l.x[i] - domp(l, a, i);
        s = s + u[i] * u[i];
      }
      const Real rho = psqrt(s), R = domp(l, a, 3);
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        const Real dir = (rho == Real(0)) ? (i == 0 ? Real(1) : Real(0)) : u[i] / rho;
        q[i] = domp(l, a, i) + R * dir;
      }
    } else if constexpr (S::DOM == DOM_CUBE) {
      // (constant-boundary kernels only: their walk value needs no exit point)
#pragma unroll
      for (int i = 0; i < DIM; ++i) q[i] = l.x[i];
    } else if constexpr (S::DOM == DOM_BOX) {
      // first nearest face (axis order, lower before upper) — strict <
      Real best = l.x[0] - domp(l, a, 0), face = domp(l, a, 0);
      int axis = 0;
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        const Real dl = l.x[i] - domp(l, a, i), du = domp(l, a, 4 + i) - l.x[i];
        if (i > 0 && dl < best) {
          best = dl;
          axis = i;
          face = domp(l, a, i);
        }
        if (du < best) {
          best = du;
          axis = i;
          face = domp(l, a, 4 + i);
        }
      }
#pragma unroll
      for (int i = 0; i < DIM; ++i) q[i] = (i == axis) ? face : l.x[i];
    } else if constexpr (S::DOM == DOM_POLAR) {
      if constexpr (WOS_KEEP_CLOSEST) {
        q[0] = l.cq[0];
        q[1] = l.cq[1];
      } else {
        polar_query(l, a, nullptr, l.x[0], l.x[1], &q[0], &q[1]);
      }
    } else if constexpr (S::DOM == DOM_MESH) {
      if constexpr (WOS_KEEP_CLOSEST_MESH) {
#pragma unroll
        for (int i = 0; i < DIM; ++i) q[i] = l.cq[i];
      } else {
        Lane c = l;
        mesh_d2(c, a, q);
      }
    } else {
      poly_project(l, a, q);
    }
  }

  // ---------------- closed triangle meshes (geometry.MeshDomain) ----------------
  __device__ static __forceinline__ Real mesh_d2(Lane& l, const KArgs& a, Real* q) {
    int reg, tri;
    const Real d2 = mesh_nearest<Real>(reinterpret_cast<const MeshNode<Real>*>(a.nodes) + l.seg_off,
                                       reinterpret_cast<const Real*>(a.segs) + 9 * (size_t)l.rec_off,
                                       l.x, q, &reg, &tri, l.seg_i);
    l.seg_i = tri;  // next query starts from this triangle
    return d2;
  }

  // ---------------- polar star curves (geometry.PolarDomain) ----------------
  __device__ static __forceinline__ Real sq2(Real x, Real y) {
    if constexpr (S::NATIVE) return fmaf(x, x, y * y);
    else return x * x + y * y;
  }
  // r(t) = r0 (1 + c1 cos 4t + c2 cos 8t) (_kernels.polar_radius_nb, _kernels.py:110-112)
  __device__ static __forceinline__ Real polar_r(const Lane& l, const KArgs& a, Real t) {
    // NATIVE: explicit FMAs so every kernel variant rounds alike
    if constexpr (S::NATIVE)
      return domp(l, a, 0) * fmaf(domp(l, a, 2), __cosf(8.0f * t), fmaf(domp(l, a, 1), __cosf(4.0f * t), 1.0f));
    else
      return domp(l, a, 0) * (Real(1) + domp(l, a, 1) * pcos(Real(4) * t) + domp(l, a, 2) * pcos(Real(8) * t));
  }
  __device__ static __forceinline__ Real polar_curve_d2(const Lane& l, const KArgs& a, Real t, Real px,
                                                        Real py) {
    const Real r = polar_r(l, a, t);
    Real st, ct;
    if constexpr (S::NATIVE) __sincosf(t, &st, &ct);
    else psincos(t, &st, &ct);
    if constexpr (S::NATIVE) {
      const float dx = fmaf(r, ct, -px), dy = fmaf(r, st, -py);
      return fmaf(dx, dx, dy * dy);
    }
    const Real dx = r * ct - px, dy = r * st - py;
    return dx * dx + dy * dy;
  }
  // _kernels.polar_query_fast (_kernels.py:121-148, 185-219): strided scan of the curve
  // table plus a window around the winner, then one parabolic refinement of the squared
  // distance through the winner's neighbours; the table sample wins if it is closer.
  // `stab` is the table staged in shared memory (or null: read through L1).
  __device__ static __forceinline__ Real polar_query(const Lane& l, const KArgs& a, const float4* stab,
                                                     Real px, Real py, Real* qx, Real* qy) {
    using T2 = typename std::conditional<sizeof(Real) == 8, double2, float2>::type;
    const T2* tab = (stab ? reinterpret_cast<const T2*>(stab) : reinterpret_cast<const T2*>(a.segs)) +
                    l.seg_off;
    const int n = l.n_seg, stride = l.rec_off;
    Real best = Real(1e30);
    int bj = 0;
    auto probe = [&](int jj) {
      // window offsets stay within one table length: one conditional wrap, no modulo
      jj = jj < 0 ? jj + n : (jj >= n ? jj - n : jj);
      const T2 b = tab[jj];
      const Real d2 = sq2(b.x - px, b.y - py);
      if (d2 < best) {
        best = d2;
        bj = jj;
      }
    };
    if constexpr (S::NATIVE) {
      // NATIVE: coarse-to-fine scan, each level searching +-one coarse step around the
      // previous winner with an 8x finer stride (64 -> 8 -> 1, or 8 -> 1 for curves the
      // reference scans in full): 97 (or 529) table samples instead of 193 (or 4096);
      // every level stays inside the basin the coarser one found
      int s = stride > 1 ? stride : 8;
      for (int j = 0; j < n; j += s) probe(j);
      while (s > 1) {
        const int f = s >= 8 ? s / 8 : 1;
        const int c = bj;
        for (int off = -s; off <= s; off += f)
          if (off != 0) probe(c + off);
        s = f;
      }
    } else {
      for (int j = 0; j < n; j += stride) probe(j);
      if (stride > 1) {
        const int lo = bj - stride;
        for (int off = 0; off <= 2 * stride; ++off) probe(lo + off);
      }
    }
    const Real h = (Real)kTwoPi / (Real)n;
    const Real t0 = (Real)bj * h;
    const Real fm = polar_curve_d2(l, a, t0 - h, px, py);
    const Real fp = polar_curve_d2(l, a, t0 + h, px, py);
    const Real denom = (fm - Real(2) * best) + fp;
    Real shift = denom > Real(0) ? Real(0.5) * h * (fm - fp) / denom : Real(0);
    if (shift > h) shift = h;
    else if (shift < -h) shift = -h;
    const Real tm = t0 + shift;
    const Real r = polar_r(l, a, tm);
    Real st, ct;
    if constexpr (S::NATIVE) __sincosf(tm, &st, &ct);
    else psincos(tm, &st, &ct);
    const Real cx = r * ct, cy = r * st;
    const Real dx = cx - px, dy = cy - py;
    const Real dm = sq2(dx, dy);
    if (best < dm) {
      const T2 b = tab[bj];
      *qx = b.x;
      *qy = b.y;
      return psqrt(best);
    }
    *qx = cx;
    *qy = cy;
    return psqrt(dm);
  }

  // ---------------- problem terms ----------------
  template <int K>
  __device__ static __forceinline__ void sine_row(Real y, Real* s) {
    // s[k] = sin((k+1) pi y)
    if constexpr (S::NATIVE) {
      float s1, c1;
      __sincosf(kPiF * y, &s1, &c1);
      const float tc = c1 + c1;
      s[0] = s1;
      if constexpr (K > 1) s[1] = tc * s1;
#pragma unroll
      for (int k = 2; k < K; ++k) s[k] = fmaf(tc, s[k - 1], -s[k - 2]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) s[k] = sin((Real)(k + 1) * (Real)kPi * y);
    }
  }

  // NATIVE, K <= 4: sin(k pi y) = s U_{k-1}(c) with s = sin(pi y), c = cos(pi y), so the
  // series is s_x s_y (s_z) Q(c_x, c_y (, c_z)) with Q a polynomial whose monomial
  // coefficients the host precomputes (wos_capi.cu sine_monomial); nested Horner.
  static constexpr bool kMonomial = S::NATIVE && (S::SK == 3 || S::SK == 4);
  // Scaled coordinates (single-instance constant-boundary box kernels with a monomial
  // sine source): the walk runs in X = pi x (the host scales the box and eps), so the
  // source terms sin(k pi x) take MUFU arguments without the pi multiply (three fewer
  // FMUL per 3D jump); the Green weight carries 1/pi^2. The walk value acc + g needs no
  // exit point, so nothing is scaled back. wos_capi.cu launch_walk mirrors this test.
  static constexpr bool kScaled = WOS_SCALED_COORDS && kMonomial && ONE && S::BC &&
                                  (S::DOM == DOM_BOX || S::DOM == DOM_CUBE) && S::SINK == SINK_ESTIMATE;
  // Centred scaled coordinates (DOM_CUBE: a cube centred at 1/2, BASELINE cfg0 / cfg4):
  // X = pi (x - 1/2), so the distance is h - max_i |X_i| (FMNMX3 with |.| operands + one
  // FADD instead of 3 FADD + 3 FADD + FMNMX3 per 3D jump). The source keeps its form:
  // sin(pi x) = cos X and cos(pi x) = -sin X, so the kernel swaps the sincos outputs and
  // the host flips the sign of the odd-degree monomial coefficients (wos_capi.cu).
  static constexpr bool kCentered = S::DOM == DOM_CUBE;
  static_assert(!kCentered || kScaled, "DOM_CUBE kernels are scaled-coordinate kernels");
  static constexpr float kInvPi2F = 0.10132118364233778f;  // 1 / pi^2
  // a query point's coordinate in the walk's units (already-converted Real values pass)
  __device__ static __forceinline__ Real start_coord(double x) {
    if constexpr (kCentered) return (Real)(kPi * (x - 0.5));
    else if constexpr (kScaled) return (Real)(kPi * x);
    else return (Real)x;
  }
  __device__ static __forceinline__ Real start_coord(float x) { return x; }

  template <int K>
  __device__ static __forceinline__ Real sine_eval(const Real* __restrict__ a, const Real* y) {
    if constexpr (kMonomial) {
      float s[DIM], c[DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        if constexpr (kCentered) __sincosf(y[i], &c[i], &s[i]);  // s <- cos X, c <- sin X
        else __sincosf(kScaled ? y[i] : kPiF * y[i], &s[i], &c[i]);
      }
      // Independent Horner chains run two at a time as packed FFMA2 (fma.rn.f32x2,
      // elementwise fma.rn): the same operations in the same order as scalar fmaf, so
      // bit-identical to it, at half the issue slots.
      auto f2 = [](float x, float y) { return make_float2(x, y); };
      if constexpr (DIM == 2) {
        float hp[K];  // hp[p] = sum_r a[p][r] c1^r
#pragma unroll
        for (int p = 0; p + 1 < K; p += 2) {
          float2 h = f2(a[p * K + (K - 1)], a[(p + 1) * K + (K - 1)]);
#pragma unroll
          for (int r = K - 2; r >= 0; --r) h = __ffma2_rn(h, f2(c[1], c[1]), f2(a[p * K + r], a[(p + 1) * K + r]));
          hp[p] = h.x;
          hp[p + 1] = h.y;
        }
        if constexpr (K % 2) {
          float h = a[(K - 1) * K + (K - 1)];
#pragma unroll
          for (int r = K - 2; r >= 0; --r) h = fmaf(h, c[1], a[(K - 1) * K + r]);
          hp[K - 1] = h;
        }
        float q = hp[K - 1];
#pragma unroll
        for (int p = K - 2; p >= 0; --p) q = fmaf(q, c[0], hp[p]);
        return (s[0] * s[1]) * q;
      } else {
        auto A = [&](int p, int qd, int r) { return a[(p * K + qd) * K + r]; };
#ifndef WOS_ESTRIN_HEADS
#define WOS_ESTRIN_HEADS 1
#endif
        // K = 3 innermost chains as c2 A1 + c2^2 A2 (FMUL2 + FFMA2, coefficient pairs as
        // uniform operands) then + A0 (FADD2): no uniform->vector moves for the heads
        constexpr bool kEstrin = WOS_ESTRIN_HEADS && K == 3;
        const float c2sq = c[2] * c[2];
        auto chain2 = [&](float2 a0, float2 a1, float2 a2) {
          return __fadd2_rn(__ffma2_rn(f2(c[2], c[2]), a1, __fmul2_rn(f2(c2sq, c2sq), a2)), a0);
        };
        float mp[K];  // mp[p] = sum_qd c1^qd sum_r a[p][qd][r] c2^r
        // pairs of p: both chains of every level share the broadcast c2 / c1
#pragma unroll
        for (int p = 0; p + 1 < K; p += 2) {
          float2 hq[K];
#pragma unroll
          for (int qd = 0; qd < K; ++qd) {
            if constexpr (kEstrin) {
              hq[qd] = chain2(f2(A(p, qd, 0), A(p + 1, qd, 0)), f2(A(p, qd, 1), A(p + 1, qd, 1)),
                              f2(A(p, qd, 2), A(p + 1, qd, 2)));
            } else {
              float2 h = f2(A(p, qd, K - 1), A(p + 1, qd, K - 1));
#pragma unroll
              for (int r = K - 2; r >= 0; --r) h = __ffma2_rn(h, f2(c[2], c[2]), f2(A(p, qd, r), A(p + 1, qd, r)));
              hq[qd] = h;
            }
          }
          float2 m = hq[K - 1];
#pragma unroll
          for (int qd = K - 2; qd >= 0; --qd) m = __ffma2_rn(m, f2(c[1], c[1]), hq[qd]);
          mp[p] = m.x;
          mp[p + 1] = m.y;
        }
        if constexpr (K % 2) {  // the unpaired p: pairs of qd
          constexpr int p = K - 1;
          float hq[K];
#pragma unroll
          for (int qd = 0; qd + 1 < K; qd += 2) {
            float2 h;
            if constexpr (kEstrin) {
              h = chain2(f2(A(p, qd, 0), A(p, qd + 1, 0)), f2(A(p, qd, 1), A(p, qd + 1, 1)),
                         f2(A(p, qd, 2), A(p, qd + 1, 2)));
            } else {
              h = f2(A(p, qd, K - 1), A(p, qd + 1, K - 1));
#pragma unroll
              for (int r = K - 2; r >= 0; --r) h = __ffma2_rn(h, f2(c[2], c[2]), f2(A(p, qd, r), A(p, qd + 1, r)));
            }
            hq[qd] = h.x;
            hq[qd + 1] = h.y;
          }
          if constexpr (kEstrin) {
            hq[K - 1] = __fadd_rn(fmaf(c[2], A(p, K - 1, 1), __fmul_rn(c2sq, A(p, K - 1, 2))), A(p, K - 1, 0));
          } else {
            float h = A(p, K - 1, K - 1);
#pragma unroll
            for (int r = K - 2; r >= 0; --r) h = fmaf(h, c[2], A(p, K - 1, r));
            hq[K - 1] = h;
          }
          float m = hq[K - 1];
#pragma unroll
          for (int qd = K - 2; qd >= 0; --qd) m = fmaf(m, c[1], hq[qd]);
          mp[p] = m;
        }
        float q = mp[K - 1];
#pragma unroll
        for (int p = K - 2; p >= 0; --p) q = fmaf(q, c[0], mp[p]);
        return (s[0] * s[1] * s[2]) * q;
      }
    } else {
      Real sx[K], sy[K];
      sine_row<K>(y[0], sx);
      sine_row<K>(y[1], sy);
      if constexpr (DIM == 2) {
        Real f = Real(0);
        if constexpr (S::NATIVE && (K % 4) == 0) {
          // rows are 16-byte aligned (kSrcOff and the row stride are multiples of 4)
          // packed FFMA2: even / odd l accumulate in the two halves of a pair, and the
          // x factor scales both halves, so one horizontal add finishes the series
          const float4* a4 = reinterpret_cast<const float4*>(a);
          float2 fp = make_float2(0.f, 0.f);
#pragma unroll
          for (int k = 0; k < K; ++k) {
            float2 t = make_float2(0.f, 0.f);
#pragma unroll
            for (int l4 = 0; l4 < K / 4; ++l4) {
              const float4 c = a4[(k * K) / 4 + l4];
              t = __ffma2_rn(make_float2(c.x, c.y), make_float2(sy[4 * l4], sy[4 * l4 + 1]), t);
              t = __ffma2_rn(make_float2(c.z, c.w), make_float2(sy[4 * l4 + 2], sy[4 * l4 + 3]), t);
            }
            fp = __ffma2_rn(make_float2(sx[k], sx[k]), t, fp);
          }
          return fp.x + fp.y;
        } else {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            Real t = Real(0);
#pragma unroll
            for (int l = 0; l < K; ++l) t = t + a[k * K + l] * sy[l];
            f = f + sx[k] * t;
          }
          return f;
        }
      } else {
        Real sz[K];
        sine_row<K>(y[2], sz);
        Real f = Real(0);
#pragma unroll
        for (int i = 0; i < K; ++i) {
          Real u = Real(0);
#pragma unroll
          for (int j = 0; j < K; ++j) {
            Real t = Real(0);
#pragma unroll
            for (int k = 0; k < K; ++k) t = t + a[(i * K + j) * K + k] * sz[k];
            u = u + sy[j] * t;
          }
          f = f + sx[i] * u;
        }
        return f;
      }
    }
  }

  // runtime-K sine series (K <= 16), used when no specialisation matches
  __device__ static Real sine_eval_rt(const Real* __restrict__ a, const Real* y, int K) {
    Real f = Real(0);
    if constexpr (DIM == 2) {
      for (int k = 0; k < K; ++k) {
        const Real sk = sin((Real)(k + 1) * (Real)kPi * y[0]);
        Real t = Real(0);
        for (int l = 0; l < K; ++l) t = t + a[k * K + l] * sin((Real)(l + 1) * (Real)kPi * y[1]);
        f = f + sk * t;
      }
    } else {
      for (int i = 0; i < K; ++i) {
        const Real si = sin((Real)(i + 1) * (Real)kPi * y[0]);
        for (int j = 0; j < K; ++j) {
          const Real sj = sin((Real)(j + 1) * (Real)kPi * y[1]);
          Real t = Real(0);
          for (int k = 0; k < K; ++k)
            t = t + a[(i * K + j) * K + k] * sin((Real)(k + 1) * (Real)kPi * y[2]);
          f = f + si * sj * t;
        }
      }
    }
    return f;
  }

  __device__ static __forceinline__ Real source(const Lane& l, const KArgs& a, const Real* y) {
    const Real* P;
    if constexpr (kHotSrc) P = l.hc + kSrcOff;
    else P = prow(l, a) + kSrcOff;
    if constexpr (S::SRC == SRC_CONST) {
      return P[0];
    } else if constexpr (S::SRC == SRC_RBF2) {
      // _kernels.py:248-259
      const Real d1x = y[0] - P[2], d1y = y[1] - P[3], d2x = y[0] - P[4], d2y = y[1] - P[5];
      if constexpr (S::NATIVE)  // explicit FMAs: identical rounding in every kernel variant
        return fmaf(P[0], fast_ex2(-fmaf(d1x, d1x, d1y * d1y) * kLog2e),
                    P[1] * fast_ex2(-fmaf(d2x, d2x, d2y * d2y) * kLog2e));
      else
        return P[0] * pexp(-(d1x * d1x + d1y * d1y)) + P[1] * pexp(-(d2x * d2x + d2y * d2y));
    } else if constexpr (S::SRC == SRC_SINE) {
      if constexpr (S::SK > 0) return sine_eval<S::SK>(P, y);
      else return sine_eval_rt(P, y, a.sine_K);
    } else if constexpr (S::SRC == SRC_GAUSS) {
      Real r2 = Real(0);
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        const Real u = y[i] - P[2 + i];
        r2 = r2 + u * u;
      }
      // NATIVE table holds log2(e) / (2 sigma^2) at P[1]; REPLAY holds sigma
      if constexpr (S::NATIVE) return P[0] * fast_ex2(-r2 * P[1]);
      else return P[0] * pexp(-r2 / (Real(2) * P[1] * P[1]));
    } else {
      return Real(0);
    }
  }

  // Offset of the boundary parameters in an instance row, known at compile time when
  // the source kind fixes the source block's size (wos_capi.cu: bnd_off = kSrcOff + ns);
  // -1 = read KArgs::bnd_off. The kernel checks the host's value once at entry.
  static constexpr int kBndOff =
      S::SRC == SRC_NONE ? kSrcOff
      : S::SRC == SRC_CONST ? kSrcOff + 1
      : S::SRC == SRC_RBF2 ? kSrcOff + 6
      : S::SRC == SRC_GAUSS ? kSrcOff + 2 + DIM
      : (S::NATIVE && S::SRC == SRC_SINE && S::SK > 0) ? kSrcOff + (DIM == 2 ? S::SK * S::SK : S::SK * S::SK * S::SK)
      : -1;
  __device__ static __forceinline__ const Real* bnd_row(const Lane& l, const KArgs& a) {
    if constexpr (kBndOff >= 0) return prow(l, a) + kBndOff;
    else return prow(l, a) + a.bnd_off;
  }
  // NATIVE Fourier / arc-length series are evaluated to an order bucket (4, 8, else M);
  // the host pads the native rows with zero coefficients up to it (wos_capi.cu)
  __device__ static __forceinline__ int order_bucket(int M) { return M <= 4 ? 4 : (M <= 8 ? 8 : M); }

  __device__ static __forceinline__ Real boundary(const Lane& l, const KArgs& a, const Real* q) {
    const Real* B = bnd_row(l, a);
    switch (a.bnd_kind) {
      case BND_CONST:
        return B[0];
      case BND_LINEAR:
        // NATIVE terms use explicit FMAs so every kernel variant (single- / multi-instance)
        // rounds alike; REPLAY keeps the reference's unfused order
        if constexpr (S::NATIVE) {
          if constexpr (DIM == 2) return fmaf(B[1], q[1], fmaf(B[0], q[0], B[2]));
          else return fmaf(B[2], q[2], fmaf(B[1], q[1], fmaf(B[0], q[0], B[3])));
        }
        if constexpr (DIM == 2) return B[0] * q[0] + B[1] * q[1] + B[2];
        else return B[0] * q[0] + B[1] * q[1] + B[2] * q[2] + B[3];
      case BND_FOURIER5: {
        if constexpr (DIM == 2) {
          if constexpr (S::NATIVE) {
            const float r = sqrtf(fmaf(q[0], q[0], q[1] * q[1]));
            const float c = (r == 0.0f) ? 1.0f : q[0] / r;
            const float s = (r == 0.0f) ? 0.0f : q[1] / r;
            return fmaf(B[4], 2.0f * c * s,
                        fmaf(B[3], fmaf(c, c, -(s * s)), fmaf(B[2], s, fmaf(B[1], c, B[0]))));
          }
          const Real r = psqrt(q[0] * q[0] + q[1] * q[1]);
          const Real c = (r == Real(0)) ? Real(1) : q[0] / r;
          const Real s = (r == Real(0)) ? Real(0) : q[1] / r;
          return B[0] + B[1] * c + B[2] * s + B[3] * (c * c - s * s) + B[4] * (Real(2) * c * s);
        }
        return Real(0);
      }
      case BND_FOURIER: {
        if constexpr (DIM == 2) {
          const int M = a.bnd_M;
          Real g = B[1];
          if constexpr (S::NATIVE) {
            // (cos t, sin t) = q / |q| (t = polar angle), then the rotation recurrence;
            // orders up to 8 unrolled (coefficient offsets fixed at compile time)
            const float r2 = fmaf(q[0], q[0], q[1] * q[1]);
            float inv;
            asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(r2));
            const bool ok = r2 > 0.0f && inv < 3.0e38f;
            const float c1 = ok ? q[0] * inv : 1.0f, s1 = ok ? q[1] * inv : 0.0f;
            // native rows interleave the coefficient pairs: B[2m] = b_m, B[2m + 1] = c_m
            float cm = c1, sm = s1;
            auto term = [&](int m) {
              g = fmaf(B[2 * m], cm, fmaf(B[2 * m + 1], sm, g));
              const float cn = fmaf(cm, c1, -sm * s1);
              sm = fmaf(sm, c1, cm * s1);
              cm = cn;
            };
            const int Mb = order_bucket(M);
            if (Mb == 4) {
#pragma unroll
              for (int m = 1; m <= 4; ++m) term(m);
            } else if (Mb == 8) {
#pragma unroll
              for (int m = 1; m <= 8; ++m) term(m);
            } else {
              for (int m = 1; m <= Mb; ++m) term(m);
            }
          } else {
            const Real t = (Real)atan2((double)q[1], (double)q[0]);
            for (int m = 1; m <= M; ++m) {
              Real sm, cm;
              psincos((Real)m * t, &sm, &cm);
              g = g + B[1 + m] * cm + B[1 + M + m] * sm;
            }
          }
          return g;
        }
        return Real(0);
      }
      case BND_SQUARE_ARCSINE: {
        if constexpr (DIM == 2) {
          const Real x0 = B[0], y0 = B[1], side = B[2];
          const int M = a.bnd_M;
          Real u, v;
          if constexpr (S::NATIVE) {
            const float inv = __frcp_rn(side);
            u = (q[0] - x0) * inv;
            v = (q[1] - y0) * inv;
          } else {
            u = (q[0] - x0) / side;
            v = (q[1] - y0) / side;
          }
          const Real db = pabs(v), dr = pabs(Real(1) - u), dt = pabs(Real(1) - v), dl = pabs(u);
          Real s;
          if (db <= dr && db <= dt && db <= dl) s = u;
          else if (dr <= dt && dr <= dl) s = Real(1) + v;
          else if (dt <= dl) s = Real(2) + (Real(1) - u);
          else s = Real(3) + (Real(1) - v);
          Real g = Real(0);
          if constexpr (S::NATIVE) {
            // sin(m t), t = 2 pi s / 4, by the rotation recurrence from one sincos
            float s1, c1;
            __sincosf(kTwoPiF * s * 0.25f, &s1, &c1);
            float sm = s1, cm = c1;
            auto term = [&](int m) {
              g = fmaf(B[3 + m], sm, g);
              const float sn = fmaf(sm, c1, cm * s1);
              cm = fmaf(cm, c1, -sm * s1);
              sm = sn;
            };
            const int Mb = order_bucket(M);  // zero-padded rows (wos_capi.cu)
            if (Mb == 4) {
#pragma unroll
              for (int m = 1; m <= 4; ++m) term(m);
            } else if (Mb == 8) {
#pragma unroll
              for (int m = 1; m <= 8; ++m) term(m);
            } else {
              for (int m = 1; m <= Mb; ++m) term(m);
            }
          } else {
            for (int m = 1; m <= M; ++m) g = g + B[3 + m] * sin((Real)kTwoPi * (Real)m * s / Real(4));
          }
          return g;
        }
        return Real(0);
      }
      case BND_QUADRATIC:
        if constexpr (DIM == 2)
          return B[0] * q[0] * q[0] + B[1] * q[1] * q[1] + B[2] * q[0] * q[1] + B[3] * q[0] +
                 B[4] * q[1] + B[5];
        return Real(0);
      default:
        return Real(0);
    }
  }

  // ---------------- delta tracking (screened walks) ----------------
  // Transformed problem  Laplacian U - sigma' U = -f'  walked with a majorant sigma_bar
  // (walker.py:322-418, _kernels.py:476-558, greens.py:100-193). Row layouts:
  //   SRC_SCR_CONST [s', f', has_f', sqrt_alpha]     (ScreenedProblem.const_coeffs)
  //   SRC_SCR_VC    [phi, a_min, a_max, 4 pi phi, 3 pi phi, pi phi]   (pde.VcInstance)
  //   BND_VC        [phi, 4 pi phi, 3 pi phi, pi phi]
  static constexpr bool kScr = S::SRC == SRC_SCR_CONST || S::SRC == SRC_SCR_VC;
  // family coefficients: libm-accurate in REPLAY (the reference's numpy), MUFU fast math
  // in NATIVE (arguments stay below ~25 rad, where __sinf/__expf keep ~1e-6 absolute /
  // relative error, far under the Monte Carlo error)
  __device__ static __forceinline__ void tsincos(Real x, Real* s_, Real* c_) {
    if constexpr (S::NATIVE) __sincosf(x, s_, c_);
    else psincos(x, s_, c_);
  }
  __device__ static __forceinline__ Real tsin(Real x) {
    if constexpr (S::NATIVE) return __sinf(x);
    else return psin(x);
  }
  __device__ static __forceinline__ Real tcos(Real x) {
    if constexpr (S::NATIVE) return __cosf(x);
    else return pcos(x);
  }
  __device__ static __forceinline__ Real texp(Real x) {
    if constexpr (S::NATIVE) return __expf(x);
    else return pexp(x);
  }

  // h = log(alpha) = -x1^2 + cos(a x0) sin(b x1), its gradient and Laplacian (pde.py:138-151)
  __device__ static __forceinline__ void vc_log_alpha(Real a_, Real b_, const Real* x, Real* h,
                                                      Real* g, Real* lap) {
    Real sa_, ca_, sb_, cb_;
    tsincos(a_ * x[0], &sa_, &ca_);
    tsincos(b_ * x[1], &sb_, &cb_);
    *h = -x[1] * x[1] + ca_ * sb_;
    g[0] = -a_ * sa_ * sb_;
    g[1] = Real(-2) * x[1] + b_ * ca_ * cb_;
    g[2] = Real(0);
    *lap = Real(-2) - (a_ * a_ + b_ * b_) * ca_ * sb_;
  }
  // sigma(x) (pde.py:176-181)
  __device__ static __forceinline__ Real vc_sigma(Real amin, Real amax, const Real* x) {
    return amin + (amax - amin) * (Real(1) + Real(0.5) * tsin((Real)kTwoPi * x[0]) *
                                                  tcos((Real)(0.5 * kPi) * x[1]));
  }
  // manufactured solution u with gradient and Laplacian (pde.py:154-173)
  __device__ static __forceinline__ void vc_solution(Real p, const Real* x, Real* u, Real* gu,
                                                     Real* lu) {
    Real s1, c1, s2, c2;
    tsincos(p * x[0], &s1, &c1);
    tsincos(Real(2) * p * x[1], &s2, &c2);
    const Real s3 = tsin(Real(3) * p * x[2]);
    *u = s1 * c2 + (Real(1) - c1) * (Real(1) - s2) + s3 * s3;
    if (gu) {
      gu[0] = p * c1 * c2 + p * s1 * (Real(1) - s2);
      gu[1] = Real(-2) * p * s1 * s2 - Real(2) * p * (Real(1) - c1) * c2;
      gu[2] = Real(3) * p * tsin(Real(6) * p * x[2]);
      *lu = -p * p * s1 * c2 + p * p * c1 * (Real(1) - s2) - Real(4) * p * p * s1 * c2 +
            Real(4) * p * p * (Real(1) - c1) * s2 + Real(18) * p * p * tcos(Real(6) * p * x[2]);
    }
  }
  // sigma' = sigma e^-h + lap(h)/2 + |grad h|^2/4 and f' = f / sqrt(alpha) (pde.py:184-212)
  __device__ static __forceinline__ void vc_coeffs(const Real* P, const Real* y, Real* sp,
                                                   Real* fp) {
    Real h, gh[3], lh;
    vc_log_alpha(P[3], P[4], y, &h, gh, &lh);
    const Real sigma = vc_sigma(P[1], P[2], y);
    *sp = sigma * texp(-h) + Real(0.5) * lh + Real(0.25) * (gh[0] * gh[0] + gh[1] * gh[1] + gh[2] * gh[2]);
    Real u, gu[3], lu;
    vc_solution(P[5], y, &u, gu, &lu);
    const Real alpha = texp(h);
    const Real f = -alpha * lu - alpha * (gh[0] * gu[0] + gh[1] * gu[1] + gh[2] * gu[2]) + sigma * u;
    *fp = f / texp(Real(0.5) * h);
  }
  __device__ static __forceinline__ Real vc_sqrt_alpha(Real a_, Real b_, const Real* x) {
    Real h, g[3], lap;
    vc_log_alpha(a_, b_, x, &h, g, &lap);
    return texp(Real(0.5) * h);
  }
  // g' = sqrt(alpha) u at the exit point (pde.py:197-199)
  __device__ static __forceinline__ Real vc_boundary(const Real* B, const Real* q) {
    Real u;
    vc_solution(B[3], q, &u, nullptr, nullptr);
    return vc_sqrt_alpha(B[1], B[2], q) * u;
  }

  // fp64 volume-event radius-fraction CDF (greens.py:154-170, _kernels.py:491-495)
  __device__ static __forceinline__ double radial_cdf(double q, double t) {
    if (q < 1.0e-4) return t * t * (3.0 - 2.0 * t);
    return (sinh(q) - q * t * cosh(q * (1.0 - t)) - sinh(q * (1.0 - t))) / (sinh(q) - q);
  }
  // REPLAY: fixed 64-step bisection (greens.py:173-186, _kernels.py:498-511)
  __device__ static __forceinline__ double invert_radial_bisect(double q, double u) {
    double lo = 0.0, hi = 1.0;
    for (int it = 0; it < 64; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (radial_cdf(q, mid) < u) lo = mid;
      else hi = mid;
    }
    return 0.5 * (lo + hi);
  }
  // NATIVE fp32 inversion of the same CDF, stable over the whole q range:
  //  q < 1 : F = t^2 sum_k w_k p_k(t) / sum_k w_k, w_k = q^(2k-2) / (2k+1)!, the q-series of
  //          the hyperbolic form (p_k from expanding sinh/cosh; p_k(1) = 1), k <= 4;
  //  q >= 1: F = N / D scaled by 2 e^-q: D = 1 - e^-2q - 2q e^-q,
  //          N = A(x) - e^-2q + (1 - x) e^-(2q - x), x = q t, A(x) = 1 - (1 + x) e^-x
  //          (series for small x), pdf = q x (e^-x - e^-(2q - x)) / D.
  // Safeguarded Newton from the harmonic (q < 1) or Gamma(2) (q >= 1) quantile.
  __device__ static __forceinline__ float invert_radial_f32(float q, float u) {
    float lo = 0.0f, hi = 1.0f, t;
    // start: the harmonic quantile t = 1/2 - sin(asin(1 - 2u) / 3) for q < 3.5, else the
    // Gamma(2) quantile of x = q t (x = -ln(1 - u) + ln(1 + x), two fixed-point steps)
    if (q < 3.5f) {
      t = 0.5f - __sinf(asinf(1.0f - 2.0f * u) * (1.0f / 3.0f));
    } else {
      const float l1 = -__logf(1.0f - u);
      float x = l1 + __logf(1.0f + l1);
      x = l1 + __logf(1.0f + x);
      t = fminf(x / q, 0.999f);
    }
    // Newton until |F(t) - u| <= 1e-6 (fp32 resolution of u) or the step stalls
    if (q < 1.0f) {
      const float q2 = q * q;
      const float w1 = 1.0f / 6.0f, w2 = q2 * (1.0f / 120.0f), w3 = q2 * q2 * (1.0f / 5040.0f),
                  w4 = q2 * q2 * q2 * (1.0f / 362880.0f);
      const float iw = 1.0f / (w1 + w2 + w3 + w4);
      // combined polynomial P(t) = sum_j c_j t^j (degree 7), F = t^2 P(t)
      float c[8];
      c[0] = (3.0f * w1 + 10.0f * w2 + 21.0f * w3 + 36.0f * w4) * iw;
      c[1] = (-2.0f * w1 - 20.0f * w2 - 70.0f * w3 - 168.0f * w4) * iw;
      c[2] = (15.0f * w2 + 105.0f * w3 + 378.0f * w4) * iw;
      c[3] = (-4.0f * w2 - 84.0f * w3 - 504.0f * w4) * iw;
      c[4] = (35.0f * w3 + 420.0f * w4) * iw;
      c[5] = (-6.0f * w3 - 216.0f * w4) * iw;
      c[6] = (63.0f * w4) * iw;
      c[7] = (-8.0f * w4) * iw;
      for (int it = 0; it < 16; ++it) {
        float P = c[7], dP = 7.0f * c[7];
#pragma unroll
        for (int j = 6; j >= 0; --j) {
          P = fmaf(P, t, c[j]);
          if (j >= 1) dP = fmaf(dP, t, (float)j * c[j]);
        }
        const float F = t * t * P - u;
        if (fabsf(F) <= 1e-6f) break;
        if (F < 0.0f) lo = t;
        else hi = t;
        const float pdf = t * fmaf(t, dP, 2.0f * P);
        float tn = pdf > 0.0f ? t - F / pdf : 0.5f * (lo + hi);
        if (!(tn >= lo && tn <= hi)) tn = 0.5f * (lo + hi);
        const bool done = fabsf(tn - t) <= 2e-7f * fmaxf(t, 1e-3f);
        t = tn;
        if (done) break;
      }
      return t;
    }
    const float e2q = __expf(-2.0f * q);
    const float D = 1.0f - e2q - 2.0f * q * __expf(-q);
    for (int it = 0; it < 16; ++it) {
      const float x = q * t;
      const float ex = __expf(-x), e2 = __expf(x - 2.0f * q);
      float A;
      if (x < 0.25f) {  // 1 - (1 + x) e^-x = e^-x (x^2/2 + x^3/6 + x^4/24 + x^5/120 + x^6/720)
        A = ex * x * x * fmaf(x, fmaf(x, fmaf(x, fmaf(x, 1.0f / 720.0f, 1.0f / 120.0f), 1.0f / 24.0f), 1.0f / 6.0f), 0.5f);
      } else {
        A = fmaf(-(1.0f + x), ex, 1.0f);
      }
      const float F = (A - e2q + (1.0f - x) * e2) / D - u;
      if (fabsf(F) <= 1e-6f) break;
      if (F < 0.0f) lo = t;
      else hi = t;
      const float pdf = q * x * (ex - e2) / D;
      float tn = pdf > 0.0f ? t - F / pdf : 0.5f * (lo + hi);
      if (!(tn >= lo && tn <= hi)) tn = 0.5f * (lo + hi);
      const bool done = fabsf(tn - t) <= 2e-7f * fmaxf(t, 1e-3f);
      t = tn;
      if (done) break;
    }
    return t;
  }

  __device__ static __forceinline__ void note_majorant(const KArgs& a, double sp) {
    atomicMax(a.majorant, (unsigned long long)__double_as_longlong(sp));
  }
  // const-coefficient kernel path: a walk whose throughput died carries nothing more
  // (_kernels.py:533-538)
  __device__ static __forceinline__ bool dead(const Lane& l, const KArgs& a) {
    if constexpr (S::SRC == SRC_SCR_CONST) return l.thr == Real(0) && prow(l, a)[kSrcOff + 2] == Real(0);
    else return false;
  }

  // one delta-tracking step (walker.py:372-416; _kernels.py:539-557)
  __device__ static __forceinline__ void screened_event(Lane& l, const KArgs& a) {
    const Real* P = prow(l, a) + kSrcOff;
    Real sp, fp = Real(0);
    bool has_f = true;
    if constexpr (S::SRC == SRC_SCR_CONST) {
      sp = P[0];
      fp = P[1];
      has_f = P[2] != Real(0);
    } else {
      vc_coeffs(P, l.x, &sp, &fp);
    }
    if ((double)sp > a.sigma_bar) note_majorant(a, (double)sp);
    const Real sb = (Real)a.sigma_bar;
    if (has_f) l.acc = l.acc + l.thr * fp / sb;
    l.thr = l.thr * (Real(1) - sp / sb);
  }

  __device__ static __forceinline__ void advance_screened_replay(Lane& l, Real d, const KArgs& a) {
    uint64_t w[4];
    philox4x64(2ull * (uint64_t)l.step, l.pid, l.tid, 0ull, a.seed, l.ikey, w);
    double q = a.sqrt_sig * (double)d;
    if (q > 500.0) q = 500.0;
    const double surf = (q < 1.0e-6) ? 1.0 - q * q / 6.0 : q / sinh(q);
    const Real z = Real(2) * (Real)u01_53(w[1]) - Real(1);
    const Real s = psqrt(pmax(Real(0), Real(1) - z * z));
    const Real phi = (Real)kTwoPi * (Real)u01_53(w[2]);
    Real sph, cph;
    psincos(phi, &sph, &cph);
    const Real dir[3] = {s * cph, s * sph, z};
    const bool vol = u01_53(w[0]) >= surf;
    const Real rad = vol ? d * (Real)invert_radial_bisect(q, u01_53(w[3])) : d;
    const Real sr = l.sgn * rad;
#pragma unroll
    for (int i = 0; i < 3; ++i) l.x[i] = l.x[i] + sr * dir[i];
    if (vol) screened_event(l, a);
  }

  __device__ static __forceinline__ void advance_screened_native(Lane& l, float d, const KArgs& a) {
    const uint4 A = native_block(l, a);
    double q = a.sqrt_sig * (double)d;
    if (q > 500.0) q = 500.0;
    // surface probability q / sinh q in fp32 (it is compared with a 23-bit uniform):
    // series below 0.125, 2 q e^-q / (1 - e^-2q) above (no overflow up to q = 500)
    const float qf = (float)q;
    float surf;
    if (qf < 0.125f) {
      const float q2 = qf * qf;
      surf = fmaf(q2, fmaf(q2, fmaf(q2, -31.0f / 15120.0f, 7.0f / 360.0f), -1.0f / 6.0f), 1.0f);
    } else {
      const float e = __expf(-qf);
      surf = 2.0f * qf * e / fmaf(-e, e, 1.0f);
    }
    const float z = f2x(A.y) - 3.0f;
    const float sxy = fast_sqrt(fmaf(-z, z, 1.0f));
    float sph, cph;
    __sincosf(dir_angle(f12(A.z)), &sph, &cph);
    const bool vol = (f12(A.x) - 1.0f) >= surf;
    float rad = d;
    if (vol) rad = d * invert_radial_f32(qf, (f12(A.w) - 1.0f) + 0x1p-24f);
    const float sr = l.sgn * rad, srxy = sr * sxy;
    l.x[0] = fmaf(srxy, cph, l.x[0]);
    l.x[1] = fmaf(srxy, sph, l.x[1]);
    l.x[2] = fmaf(sr, z, l.x[2]);
    if (vol) screened_event(l, a);
  }

  // value at termination: acc + g(projection); constant g needs no projection
  __device__ static __forceinline__ Real finish_value(const Lane& l, const KArgs& a) {
    if constexpr (kScr) {
      // values = (acc + thr g'(q)) / sqrt_alpha(x0)  (walker.py:356-357,368-369)
      Real g;
      if constexpr (S::SRC == SRC_SCR_VC) {
        Real q[DIM];
        project(l, a, q);
        g = vc_boundary(bnd_row(l, a), q);
      } else {
        g = bnd_row(l, a)[0];
      }
      return (l.acc + l.thr * g) / l.sa;
    }
    if constexpr (S::BC) return l.acc + a.bnd_c;
    if constexpr (ONE) {
      if (a.bnd_kind == BND_CONST) return l.acc + a.bnd_c;
    }
    if (a.bnd_kind == BND_CONST) return l.acc + bnd_row(l, a)[0];
    Real q[DIM];
    project(l, a, q);
    return l.acc + boundary(l, a, q);
  }

  // ---------------- one jump ----------------
  // REPLAY: walker.py:284-313 operation by operation
  __device__ static __forceinline__ double nonzero_u(double u, uint64_t draw, const Lane& l,
                                                     const KArgs& a) {
    uint64_t tag = 1;
    while (u == 0.0) {  // walker.py:232-242, probability 2^-53 per draw
      uint64_t w[4];
      philox4x64(draw, l.pid, l.tid, tag, a.seed, l.ikey, w);
      u = u01_53(w[0]);
      tag += 1;
    }
    return u;
  }

  __device__ static __forceinline__ void advance_replay(Lane& l, Real d, const KArgs& a) {
    const uint64_t draw = 2ull * (uint64_t)l.step;
    uint64_t w[4];
    philox4x64(draw, l.pid, l.tid, 0ull, a.seed, l.ikey, w);
    Real dir[DIM];
    const Real sg = l.sgn;
    if constexpr (DIM == 2) {
      const Real theta = (Real)kTwoPi * (Real)u01_53(w[0]);
      psincos(theta, &dir[1], &dir[0]);
      if constexpr (S::SRC != SRC_NONE) {
        const Real u_rad = (Real)nonzero_u(u01_53(w[2]), draw, l, a);
        const Real rad = d * psqrt(u_rad);
        const Real phi = (Real)kTwoPi * (Real)u01_53(w[1]);
        Real sp, cp;
        psincos(phi, &sp, &cp);
        const Real g[2] = {l.x[0] + sg * rad * cp, l.x[1] + sg * rad * sp};
        const Real green = (Real)kInvTwoPi * plog(d / rad);
        l.acc -= (Real)kPi * d * d * source(l, a, g) * green;
      }
    } else {
      const Real z = Real(2) * (Real)u01_53(w[0]) - Real(1);
      const Real s = psqrt(pmax(Real(0), Real(1) - z * z));
      const Real phi = (Real)kTwoPi * (Real)u01_53(w[1]);
      Real sp, cp;
      psincos(phi, &sp, &cp);
      dir[0] = s * cp;
      dir[1] = s * sp;
      dir[2] = z;
      if constexpr (S::SRC != SRC_NONE) {
        uint64_t wb[4];
        philox4x64(draw + 1, l.pid, l.tid, 0ull, a.seed, l.ikey, wb);
        const Real u_rad = (Real)nonzero_u(u01_53(wb[0]), draw + 1, l, a);
        const Real rad = d * pcbrt(u_rad);
        const Real vz = Real(2) * (Real)u01_53(w[2]) - Real(1);
        const Real vs = psqrt(pmax(Real(0), Real(1) - vz * vz));
        const Real vphi = (Real)kTwoPi * (Real)u01_53(w[3]);
        Real vsp, vcp;
        psincos(vphi, &vsp, &vcp);
        const Real g[3] = {l.x[0] + sg * rad * (vs * vcp), l.x[1] + sg * rad * (vs * vsp),
                           l.x[2] + sg * rad * vz};
        const Real green = (Real)kInvFourPi * (Real(1) / rad - Real(1) / d);
        const Real vol = (Real)(4.0 / 3.0) * (Real)kPi * (d * d * d);
        l.acc -= vol * source(l, a, g) * green;
      }
    }
#pragma unroll
    for (int i = 0; i < DIM; ++i) l.x[i] += sg * d * dir[i];
  }

  // Source-free NATIVE walks need one uniform per jump in 2D and two in 3D, so a block
  // serves kPerBlock consecutive jumps: jump s takes word s % 4 (2D) / words
  // 2 (s % 2), 2 (s % 2) + 1 (3D) of the block at counter 2 floor(s / kPerBlock).
  // Kernels whose lanes run in phase lock (the amortised loop) draw each block once;
  // the others redraw it per jump and select the words (same stream).
  // The NATIVE 3D source jump (layout v4, below) also takes 64 bits: a block serves two
  // jumps, and its radius fraction comes from the shared-memory Beta(2,2) table
  static constexpr bool kBetaTab = S::NATIVE && S::SRC != SRC_NONE && !kScr;
  static constexpr int kPerBlock = (S::NATIVE && S::SRC == SRC_NONE) ? (DIM == 2 ? 4 : 2) : (kBetaTab ? 2 : 1);

  __device__ static __forceinline__ uint4 native_block(const Lane& l, const KArgs& a) {
    return native_block_at(l, a, 2u * ((uint32_t)l.step / (uint32_t)kPerBlock));
  }
  __device__ static __forceinline__ uint4 native_block_at(const Lane& l, const KArgs& a, uint32_t c0) {
    const int rounds = S::RND ? S::RND : a.philox_rounds;
// the hot kernels fold too since the jump-first loop made refills cheaper (cfg4 -0.7 %;
// it had cost +1.7 % with the test-first loop)
#ifndef WOS_MULTI_K0TAB
#define WOS_MULTI_K0TAB 1
#endif
#ifndef WOS_HOT_FOLD
#define WOS_HOT_FOLD 1
#endif
    if constexpr (kHot && WOS_HOT_FOLD) return philox4x32_rk_pre(c0, l.pc, l.hk0, l.hk1, rounds);
    else if constexpr (kHot) return philox4x32_rk(make_uint4(l.c1, c0, l.c2, l.c3), l.hk0, l.hk1, rounds);
    else if constexpr (ONE) return philox4x32_rk_pre(c0, l.pc, a.rk0, a.rk1, rounds);
    else if constexpr (WOS_MULTI_K0TAB) return philox4x32_pre_k0(c0, l.pc, a.rk0, l.k1, rounds);
    else return philox4x32_pre(c0, l.pc, a.nkey0, l.k1, rounds);
  }

  // the walk's fixed Philox counter words folded through rounds 0-2 (wos_rng.cuh): the
  // counter is (c1, block, c2, c3), c1 = low point id, c2 = low traj id, c3 = high words
  __device__ static __forceinline__ void set_counter(Lane& l, const KArgs& a, uint32_t c1, uint32_t c2,
                                                     uint32_t c3) {
    if constexpr (kHot && WOS_HOT_FOLD) {
      l.pc = philox_pre(c1, c2, c3, l.hk0[0], l.hk1[0], l.hk0[1], l.hk1[1], l.hk0[2], l.hk1[2]);
    } else if constexpr (kHot) {
      l.c1 = c1;
      l.c2 = c2;
      l.c3 = c3;
    }
    else if constexpr (ONE) l.pc = philox_pre(c1, c2, c3, a.rk0[0], a.rk1[0], a.rk0[1], a.rk1[1], a.rk0[2], a.rk1[2]);
    else
      l.pc = philox_pre(c1, c2, c3, a.nkey0, l.k1, a.nkey0 + 0x9E3779B9u, l.k1 + 0xBB67AE85u,
                        a.nkey0 + 2u * 0x9E3779B9u, l.k1 + 2u * 0xBB67AE85u);
  }

  // source-free NATIVE jumps from their words of the block (kPerBlock above)
  __device__ static __forceinline__ void move_native_2d(Lane& l, float d, uint32_t w) {
    float sth, cth;
    __sincosf(dir_angle(f12(w)), &sth, &cth);
    const float sd = l.sgn * d;
    l.x[0] = fmaf(sd, cth, l.x[0]);
    l.x[1] = fmaf(sd, sth, l.x[1]);
  }
  __device__ static __forceinline__ void move_native_3d(Lane& l, float d, uint32_t wz, uint32_t wphi) {
    const float z = f2x(wz) - 3.0f;
    const float sxy = fast_sqrt(fmaf(-z, z, 1.0f));
    float sph, cph;
    __sincosf(dir_angle(f12(wphi)), &sph, &cph);
    const float sd = l.sgn * d, sdxy = sd * sxy;
    l.x[0] = fmaf(sdxy, cph, l.x[0]);
    l.x[1] = fmaf(sdxy, sph, l.x[1]);
    l.x[2] = fmaf(sd, z, l.x[2]);
  }
  // the block's words for sub-jump k of an amortised round
  __device__ static __forceinline__ void move_native_word(Lane& l, float d, const uint4& B, int k,
                                                         const KArgs& a) {
    if constexpr (kBetaTab) {
      jump_source(l, d, a, k == 0 ? B.x : B.z, k == 0 ? B.y : B.w);
      return;
    }
    if constexpr (DIM == 2) move_native_2d(l, d, k == 0 ? B.x : k == 1 ? B.y : k == 2 ? B.z : B.w);
    else move_native_3d(l, d, k == 0 ? B.x : B.z, k == 0 ? B.y : B.w);
  }

  // NATIVE: Green's-function importance sampling, fp32 fast math, one Philox block
  __device__ static __forceinline__ void advance_native(Lane& l, float d, const KArgs& a) {
    const uint4 A = native_block(l, a);
    const float sd = l.sgn * d;
    if constexpr (DIM == 2 && S::SRC == SRC_NONE) {
      const uint32_t k = (uint32_t)l.step & 3u;
      move_native_2d(l, d, k == 0 ? A.x : k == 1 ? A.y : k == 2 ? A.z : A.w);
    } else if constexpr (S::SRC == SRC_NONE) {
      const bool odd = (l.step & 1) != 0;
      move_native_3d(l, d, odd ? A.z : A.x, odd ? A.w : A.y);
    } else {
      // source jumps (2D and 3D): two jumps per block, jump s takes words (x, y) for even
      // s, (z, w) for odd s
      const bool odd = (l.step & 1) != 0;
      jump_source(l, d, a, odd ? A.z : A.x, odd ? A.w : A.y);
    }
  }

  // NATIVE source jump, layout v4: 64 bits (two words) per jump, so one Philox4x32
  // block serves two jumps (kPerBlock = 2; phase-locked rounds in the hot loop):
  //   wa bits 0..5 -> radius index bits 6..11, 6..18 -> z (move), 19..31 -> phi (move)
  //   wb bits 0..12 -> z' (sample), 13..25 -> phi' (sample), 26..31 -> radius index
  //   bits 0..5
  // (2D: wa bits 6..18 -> phi (sample direction), 19..31 -> theta (move); wb only
  // lends its radius bits.) The radius index sits where one funnel shift of (wa:wb)
  // by 24 and one mask give its byte offset into the table (v3 took two shifts, two
  // masks and a merge per jump).
  // Direction fields are 13-bit, midpoint-rounded ((b + 1/2) 2^-13): the midpoint rule
  // on the periodic phi is spectrally accurate and on z errs by O(2^-26) of the
  // integrand's curvature — far below fp32 rounding of the walk value. The radius
  // fraction t ~ Beta(2,2) is the conditional mean of its 12-bit probability bin
  // (include/wos_beta_table.h: E[t] exact, E[t^2] -1.0e-8), read from the table the
  // kernel stages in shared memory. oracle/wos_oracle.c restates this layout.
  // (the mask and the shift go through inline PTX so that ptxas emits LOP3 + LEA / LEA.HI
  // rather than rewriting the add as an OR and needing a second LOP3 for the constant)
  __device__ static __forceinline__ float f13_lo(uint32_t w, uint32_t expo) {  // bits 0..12
    uint32_t m;
    asm("lop3.b32 %0, %1, 0x1fff, 0, 0xc0;" : "=r"(m) : "r"(w));
    return __uint_as_float((m << 10) + (expo | 0x200u));
  }
  __device__ static __forceinline__ float f13_mid6(uint32_t w, uint32_t expo) {  // bits 6..18
    uint32_t m;
    asm("lop3.b32 %0, %1, 0x7ffc0, 0, 0xc0;" : "=r"(m) : "r"(w));
    return __uint_as_float((m << 4) + (expo | 0x200u));
  }
  __device__ static __forceinline__ float f13_mid13(uint32_t w) {  // bits 13..25, in [1, 2)
    uint32_t r;
    asm("shf.r.clamp.b32 %0, %1, %2, 3;" : "=r"(r) : "r"(w & 0x3ffe000u), "r"(0u));
    return __uint_as_float(r + 0x3f800200u);
  }
  // byte offset of the radius-table entry: (wb >> 26) | (wa & 63) << 6, times 4
  __device__ static __forceinline__ uint32_t radius_off(uint32_t wa, uint32_t wb) {
    return __funnelshift_r(wb, wa, 24) & 0x3ffcu;
  }
  __device__ static __forceinline__ float f13_hi(uint32_t w) {  // bits 19..31
    uint32_t r;
    asm("shf.r.clamp.b32 %0, %1, %2, 9;" : "=r"(r) : "r"(w & 0xfff80000u), "r"(0u));
    return __uint_as_float(r + 0x3f800200u);
  }
  // The table's shared-memory address: the start of the dynamic window in
  // single-instance box / ball launches (nothing else is staged before it), else after
  // the instance table and the polygon records. It is read with ld.shared on that 32-bit offset, so no generic address of
  // the shared window has to be rebuilt inside the loop.
  static constexpr bool kBetaAtZero = ONE && (S::DOM == DOM_BOX || S::DOM == DOM_BALL || S::DOM == DOM_CUBE);
  // Polygon and mesh kernels read the table through L1 instead: their candidate-grid /
  // BVH records live in L1, and 16 KB of staged table per CTA shrinks L1 by 64 KB at 4
  // CTAs/SM (cfg3: twice the long-scoreboard stalls, +6 % time)
  static constexpr bool kBetaGlobal = S::DOM == DOM_POLY || S::DOM == DOM_MESH;
  __device__ static __forceinline__ uint32_t beta_tab_offset(const KArgs& a) {
    extern __shared__ __align__(16) unsigned char wos_smem_[];
    // the dynamic window's shared address (a link-time constant) plus what precedes it
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(wos_smem_);
    if constexpr (kBetaAtZero) return base;
    else return base + (uint32_t)(a.stage_bytes + a.seg_stage_bytes);
  }
  __device__ static __forceinline__ float beta_at(uint32_t off, uint32_t kbytes) {
    float t;
    asm("ld.shared.f32 %0, [%1];" : "=f"(t) : "r"(off + kbytes));
    return t;
  }
  __device__ static __forceinline__ void jump_source(Lane& l, float d, const KArgs& a, uint32_t wa,
                                                     uint32_t wb) {
    jump_source(l, d, a, wa, wb, beta_tab_offset(a));
  }
  __device__ static __forceinline__ void jump_source(Lane& l, float d, const KArgs& a, uint32_t wa,
                                                     uint32_t wb, uint32_t btab) {
    // (DOM_CUBE kernels run no antithetic walks — the launcher picks the scaled box
    // kernel for those — so their sign is +1 and the multiply goes)
    const float sd = kCentered ? d : l.sgn * d;
    auto radius_t = [&](uint32_t off) -> float {
      if constexpr (kBetaGlobal)
        return __ldg(reinterpret_cast<const float*>(reinterpret_cast<const unsigned char*>(a.beta_tab) + off));
      else return beta_at(btab, off);
    };
    if constexpr (DIM == 2) {
      // 2D: wa bits 19..31 -> theta (move), bits 0..12 -> phi (sample direction); the
      // radius index as in 3D, into the disk Green's-law table (wos_green2_table); wb's
      // other bits are not used
      float sth, cth;
      __sincosf(dir_angle(f13_hi(wa)), &sth, &cth);
      float sph, cph;
      __sincosf(dir_angle(f13_mid6(wa, 0x3f800000u)), &sph, &cph);
      const float sr = sd * radius_t(radius_off(wa, wb));
      const float g[2] = {fmaf(sr, cph, l.x[0]), fmaf(sr, sph, l.x[1])};
      // (scaled-coordinate kernels: the host folds the weight 1/4 pi^-2 into the coefficients)
      l.acc = fmaf(kScaled ? -(d * d) : -0.25f * d * d, source(l, a, g), l.acc);
      l.x[0] = fmaf(sd, cth, l.x[0]);
      l.x[1] = fmaf(sd, sth, l.x[1]);
      return;
    } else {
    // z = 2u - 1 is exact for u = f - 1, so fmaf(-z, z, 1) >= 0
    const float z = f13_mid6(wa, 0x40000000u) - 3.0f;
    const float sxy = fast_sqrt(fmaf(-z, z, 1.0f));
    float sph, cph;
    __sincosf(dir_angle(f13_hi(wa)), &sph, &cph);
    const float vz = f13_lo(wb, 0x40000000u) - 3.0f;
    const float vs = fast_sqrt(fmaf(-vz, vz, 1.0f));
    float vsp, vcp;
    __sincosf(dir_angle(f13_mid13(wb)), &vsp, &vcp);
    const float t = radius_t(radius_off(wa, wb));
    const float sr = sd * t;
    const float srv = sr * vs;
    // (x, y) pairs as packed FFMA2: elementwise fma.rn, identical to two fmaf
    const float2 xy = make_float2(l.x[0], l.x[1]);
    const float2 gxy = __ffma2_rn(make_float2(srv, srv), make_float2(vcp, vsp), xy);
    const float g[3] = {gxy.x, gxy.y, fmaf(sr, vz, l.x[2])};
    // (scaled-coordinate kernels: the host folds the weight 1/6 pi^-2 into the coefficients)
    l.acc = fmaf(kScaled ? -(d * d) : -(d * d) * (1.0f / 6.0f), source(l, a, g), l.acc);
    const float sdxy = sd * sxy;
    const float2 nxy = __ffma2_rn(make_float2(sdxy, sdxy), make_float2(cph, sph), xy);
    l.x[0] = nxy.x;
    l.x[1] = nxy.y;
    l.x[2] = fmaf(sd, z, l.x[2]);
    }
  }

  // ---------------- walk start ----------------
  // single-instance NATIVE start from precomputed counter words (same state as start)
  __device__ static __forceinline__ void start_native(Lane& l, const KArgs& a, const float* x0, float sgn,
                                                      uint32_t c1, uint32_t c2, uint32_t c3) {
#pragma unroll
    for (int i = 0; i < DIM; ++i) l.x[i] = x0[i];
    l.acc = 0.0f;
    l.sgn = sgn;
    l.step = 0;
    set_counter(l, a, c1, c2, c3);
  }

  template <class X>
  __device__ static __forceinline__ void start(Lane& l, const Real* table, const InstHdr* hdr,
                                               const KArgs& a, const X* x0, int inst,
                                               uint64_t pid, uint64_t tid, double sgn) {
#pragma unroll
    for (int i = 0; i < DIM; ++i) l.x[i] = start_coord(x0[i]);
    l.acc = Real(0);
    l.sgn = (Real)sgn;
    l.step = 0;
    if constexpr (!S::NATIVE) {
      l.pid = pid;
      l.tid = tid;
    }
    if constexpr (!ONE) {
      l.row = table + (size_t)inst * a.stride;
      const InstHdr h = hdr[inst];
      if constexpr (S::NATIVE) l.k1 = a.nkey1_seed ^ h.nkey1;
      else l.ikey = h.ikey;
      if constexpr (S::DOM == DOM_POLY || S::DOM == DOM_POLAR || S::DOM == DOM_MESH) {
        l.seg_off = h.seg_off;
        l.n_seg = h.n_seg;
        l.rec_off = h.rec_off;
      }
    } else if constexpr (S::DOM == DOM_POLY || S::DOM == DOM_POLAR || S::DOM == DOM_MESH) {
      const InstHdr h = hdr[0];
      l.seg_off = h.seg_off;
      l.n_seg = h.n_seg;
      l.rec_off = h.rec_off;
    }
    if constexpr (S::NATIVE)
      set_counter(l, a, (uint32_t)pid, (uint32_t)tid,
                  (uint32_t)(tid >> 32) ^ ((uint32_t)(pid >> 32) * 0x85EBCA6Bu));
    if constexpr (S::DOM == DOM_MESH) l.seg_i = -1;
    if constexpr (kScr) {
      l.thr = Real(1);
      const Real* P = prow(l, a) + kSrcOff;
      if constexpr (S::SRC == SRC_SCR_VC) l.sa = vc_sqrt_alpha(P[3], P[4], l.x);
      else l.sa = P[3];
    }
  }
};

// ------------------------------------------------------------------------
// warp-level helpers
// ------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(WOS_FULL, v, o);
  return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ------------------------------------------------------------------------
// the persistent kernel
// ------------------------------------------------------------------------
// Work units (also the ESTIMATE sink's retire blocks), fixed by L alone so that the
// reduction order never depends on the launch or on the number of GPUs:
//   L <= kChunk: U = ceil(kChunk / L) whole points (IU = U L walks); each point's L
//                values are reduced in the warp (two-pass, estimator.py:106-110) and
//                written to out_mean / out_m2;
//   L >  kChunk: one chunk of kChunk walks of one point (IU = kChunk; walks past L are
//                null items); the chunk's (mean, m2) goes to `partials` and
//                wos_merge_chunks Chan-merges each point's chunks in chunk order
//                (estimator.chan_merge, estimator.py:41-53).
// Each live unit has a shared-memory completion counter bumped by every finishing
// walk; at each refill the warp retires the completed units at the head of its
// stream, in order.
template <int RS = 1, class Real>
__device__ __forceinline__ double sample_at(const Real* ring, uint32_t base, uint32_t i, bool anti) {
  if (anti)
    return ((double)ring[((base + 2 * i) % kRing) * RS] + (double)ring[((base + 2 * i + 1) % kRing) * RS]) / 2.0;
  return (double)ring[((base + i) % kRing) * RS];
}

// two-pass moments of n samples starting at ring position `base`, warp-cooperative,
// fixed order (estimator.py:106-110)
template <int RS = 1, class Real>
__device__ __forceinline__ void warp_moments(const Real* ring, uint32_t base, uint32_t n, bool anti,
                                             int lane, double* mean, double* m2) {
  double sum = 0.0;
  for (uint32_t i = lane; i < n; i += 32) sum += sample_at<RS>(ring, base, i, anti);
  sum = warp_sum(sum);
  const double mu = sum / (double)n;
  double q = 0.0;
  for (uint32_t i = lane; i < n; i += 32) {
    const double v = sample_at<RS>(ring, base, i, anti);
    q += (v - mu) * (v - mu);
  }
  *mean = mu;
  *m2 = warp_sum(q);
}

template <class S>
__device__ __forceinline__ void wos_kernel_body(const KArgs& a) {
  using W = Walker<S>;
  using Real = typename S::Real;
  constexpr int DIM = S::DIM;
  constexpr bool est = S::SINK == SINK_ESTIMATE;
  constexpr bool kExitRing = W::kExitRing;
  constexpr int kRS = W::kRS;
  constexpr uint32_t kSlotBytes = (uint32_t)sizeof(Real) * kRS;  // bytes per ring slot
  extern __shared__ __align__(16) unsigned char smem[];

  // ---- stage the instance table into shared memory (multi-instance launches) ----
  Real* table = reinterpret_cast<Real*>(smem);
  if constexpr (!S::ONE) {
    const int n4 = a.stage_bytes / 16;
    const int4* src = reinterpret_cast<const int4*>(a.table);
    int4* dst = reinterpret_cast<int4*>(smem);
    for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
  }
  // ---- stage NATIVE polygon records after the table ----
  const float4* srec = nullptr;
  if constexpr ((S::NATIVE && S::DOM == DOM_POLY) || S::DOM == DOM_POLAR) {
    if (a.seg_stage_bytes > 0) {
      float4* dst = reinterpret_cast<float4*>(smem + a.stage_bytes);
      const float4* src = reinterpret_cast<const float4*>(a.segs);
      for (int i = threadIdx.x; i < a.seg_stage_bytes / 16; i += blockDim.x) dst[i] = src[i];
      srec = dst;
    }
  }
  // ---- stage the Beta(2,2) radius table (NATIVE 3D source jumps) after them ----
  if constexpr (W::kBetaTab && !W::kBetaGlobal) {
    float* dst = reinterpret_cast<float*>(smem + a.stage_bytes + a.seg_stage_bytes);
    for (int i = threadIdx.x; i < a.beta_stage_bytes / 4; i += blockDim.x) dst[i] = a.beta_tab[i];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (W::kBndOff >= 0) {
    // the compile-time boundary offset must be the host's (a mismatch would be a build
    // inconsistency): flag it through the watchdog and do nothing
    if (a.bnd_off != W::kBndOff) {
      if (threadIdx.x == 0) atomicExch(a.watchdog, 2u);
      return;
    }
  }
  // the warp's ring offset goes through a shuffle so that ptxas keeps it in a register
  // instead of re-deriving it from %tid and the launch constants every iteration
  const uint32_t woff = __shfl_sync(WOS_FULL, (uint32_t)(a.stage_bytes + a.seg_stage_bytes + a.beta_stage_bytes +
                                    warp * (kRing * kSlotBytes + kSlots * 4 + kUQ * 4)), 0);
  unsigned char* wbase = smem + woff;
  Real* ring = reinterpret_cast<Real*>(wbase);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(wbase + kRing * kSlotBytes);
  uint32_t* unitq = cnt + kSlots;
  if (lane < kSlots) cnt[lane] = 0u;
  __syncthreads();

  const bool anti = a.antithetic != 0;
  // antithetic pairs share a traj id (walk jr uses id jr & ~1) and walk jr & 1 is the
  // mirrored one: warp-uniform masks for the hot issue path
  const uint32_t anti_jmask = __shfl_sync(WOS_FULL, anti ? ~1u : ~0u, 0);
  const uint32_t anti_bit = __shfl_sync(WOS_FULL, anti ? 1u : 0u, 0);
  const uint32_t IU = a.IU, L = a.L, U = a.U;
  const bool split = a.n_chunks > 0;  // L > kChunk: units are chunks of one point
  const Real eps = sizeof(Real) == 8 ? (Real)a.eps : (Real)a.eps_f;

  // warp-uniform stream state
  uint32_t s_issue = 0, s_avail = 0, n_grabbed = 0;
  uint32_t r_seq = 0;    // first item of the next unit to retire
  uint32_t r_unit = 0;   // its index in this warp's stream
  bool exhausted = false;

  // fast refill path (ESTIMATE, one point per unit): warp-uniform cache of the unit's point
  const bool fast = est && (split || U == 1);
  uint32_t cu_k = 0xffffffffu;  // stream index of the cached unit (none yet)
  uint32_t cu_end = 0;          // stream position where the cached unit ends
  uint32_t cu_j0 = 0, cu_jend = 0;  // walk range [j0, jend) of the cached unit
  Real cu_x[DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i) cu_x[i] = Real(0);
  uint64_t cu_pid = 0;
  int cu_inst = 0;
  // single-instance NATIVE: Philox counter words of the cached unit's walk 0; walk
  // j0 + jj has c2 = cu_c2b + jj while cu_fastc (no 32-bit carry inside the unit)
  uint32_t cu_c1 = 0, cu_c2b = 0, cu_c3 = 0;
  PhiloxUnit cu_pu{0u, 0u, 0u};  // hot kernels: the unit's c2-free Philox fold
  bool cu_fastc = false;

  typename W::Lane l;
  if constexpr (W::kHot) {
    // Philox round keys and the jump's parameters go constant bank -> shared memory
    // (warp 0's ring, not yet in use) -> shuffle: loop-invariant registers that ptxas
    // cannot re-derive from the constant bank, so it keeps them in uniform registers
    // instead of re-issuing the constant loads every step
    uint32_t* hs = reinterpret_cast<uint32_t*>(smem + a.stage_bytes + a.seg_stage_bytes + a.beta_stage_bytes);
    for (int i = threadIdx.x; i < 20 + W::kHotC; i += blockDim.x)
      hs[i] = i < 10 ? a.rk0[i] : i < 20 ? a.rk1[i - 10] : __float_as_uint(a.cp[i - 20]);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      l.hk0[r] = __shfl_sync(WOS_FULL, hs[r], 0);
      l.hk1[r] = __shfl_sync(WOS_FULL, hs[10 + r], 0);
    }
#pragma unroll
    for (int i = 0; i < W::kHotC; ++i) l.hc[i] = __uint_as_float(__shfl_sync(WOS_FULL, hs[20 + i], 0));
    __syncthreads();
  }
  bool active = false;
  if constexpr (W::kExitRing) {  // (a lane without a walk reads as an ended walk: see the exit-ring round)
    l.d = Real(-1);
    l.step = 0;
    l.sgn = Real(1);
#pragma unroll
    for (int i = 0; i < DIM; ++i) l.x[i] = Real(0);
  }
  uint32_t blk = 0;          // byte offset of this lane's unit counter in cnt (ESTIMATE)
  unsigned idle = WOS_FULL;  // warp-uniform: lanes without a walk
  unsigned long long lane_steps = 0ull;
  uint32_t refills = 0;

  // in-order retirement of completed units (ESTIMATE sink)
  auto retire = [&]() {
    __syncwarp();
    while (r_seq + IU <= s_issue && cnt[r_unit % kSlots] == IU) {
      const uint32_t unit = unitq[r_unit % kUQ];
      if constexpr (kExitRing) {
        // the unit's slots hold exit positions: evaluate g(projection) for all of them,
        // 32 at a time, and leave each value in its slot's first word (a null item's
        // slot holds stale data; its value is computed and never read)
        for (uint32_t i = lane; i < IU; i += 32) {
          Real* slot = ring + ((r_seq + i) % kRing) * kRS;
          typename W::Lane t = l;
          t.x[0] = slot[0];
          t.x[1] = slot[1];
          t.acc = Real(0);
          slot[0] = W::finish_value(t, a);
        }
        __syncwarp();
      }
      if (split) {
        const uint32_t p = fast_div(unit, a.nc_mul, a.nc_shr);
        const uint32_t c = unit - p * a.n_chunks;
        const uint32_t valid = min((uint32_t)kChunk, L - c * kChunk);
        double mu, q;
        warp_moments<kRS>(ring, r_seq, anti ? valid / 2 : valid, anti, lane, &mu, &q);
        if (lane == 0) {
          a.partials[2 * (size_t)unit] = mu;
          a.partials[2 * (size_t)unit + 1] = q;
        }
      } else if (L <= 32) {
        // small L: lane per point, sequential fixed-order two-pass, coalesced stores
        const uint32_t ns = anti ? L / 2 : L;
        for (uint32_t pl = lane; pl < U; pl += 32) {
          const uint64_t p = (uint64_t)unit * U + pl;
          if (p < a.n_points) {
            const uint32_t base = r_seq + pl * L;
            double sum = 0.0;
            for (uint32_t i = 0; i < ns; ++i) sum += sample_at<kRS>(ring, base, i, anti);
            const double mu = sum / (double)ns;
            double q = 0.0;
            for (uint32_t i = 0; i < ns; ++i) {
              const double v = sample_at<kRS>(ring, base, i, anti);
              q += (v - mu) * (v - mu);
            }
            a.out_mean[p] = mu;
            a.out_m2[p] = q;
          }
        }
      } else {
        for (uint32_t pl = 0; pl < U; ++pl) {
          const uint64_t p = (uint64_t)unit * U + pl;
          if (p >= a.n_points) break;
          double mu, q;
          warp_moments<kRS>(ring, r_seq + pl * L, anti ? L / 2 : L, anti, lane, &mu, &q);
          if (lane == 0) {
            a.out_mean[p] = mu;
            a.out_m2[p] = q;
          }
        }
      }
      __syncwarp();
      if (lane == 0) cnt[r_unit % kSlots] = 0u;
      __syncwarp();
      r_seq += IU;
      ++r_unit;
    }
  };

  // Loop order. Jump-first (default): an iteration jumps with the distance carried
  // from the previous query, then queries the new position and records the walk at
  // once if it terminated; a new walk queries its start when it is issued (and is
  // recorded there with 0 steps if it starts in the shell). A walk of s jumps then
  // occupies s iterations of its lane instead of s + 1 (test-first: the terminating
  // query used an iteration of its own), so fewer lane slots of the jump block idle.
  // Termination semantics are unchanged: d < eps first (hit), then step >= max_steps,
  // the same state tested in the same order (walker.py:273-283).
  // Closed-form domains only: a polygon / polar / mesh query costs more than the jump,
  // and the extra divergent query of every issued walk outweighed the saved slots
  // (cfg3 +9 %; cfg4 -1.7 %, cfg2 -12 % with it).
#ifndef WOS_JUMP_FIRST
#define WOS_JUMP_FIRST 1
#endif
  constexpr bool kJumpFirst = WOS_JUMP_FIRST && (S::DOM == DOM_BALL || S::DOM == DOM_BOX || S::DOM == DOM_CUBE);
  // Polygons run jump-first in the cached-point refill only: there a unit's start
  // distance (and nearest segment) is queried once per unit, not per walk
#ifndef WOS_JUMP_FIRST_POLY
#define WOS_JUMP_FIRST_POLY 1
#endif
  constexpr bool kJumpFirstPoly = WOS_JUMP_FIRST_POLY && S::DOM == DOM_POLY && est;
  const bool jf = kJumpFirst || (kJumpFirstPoly && fast);
  // Amortised RNG (source-free NATIVE walks on closed-form domains): lanes are refilled
  // only between rounds of kPerBlock jumps, so every live lane enters a round at a step
  // that is a multiple of kPerBlock and one Philox block serves the whole round.
#ifndef WOS_AMORT_RNG
#define WOS_AMORT_RNG 1
#endif
  // NATIVE source jumps (two per block, layout v4) run the same rounds outside the hot
  // loop (multi-instance, non-constant-boundary and rows kernels): the round holds the
  // block only inside one iteration, so the second jump's words cost no registers across
  // iterations, and a jump no longer redraws the whole block for half of its words
  // (cfg2: a multi-instance Philox block with its per-round key adds is ~45 instructions).
  // (a lane whose walk ends after the first jump of a round idles for the second)
#ifndef WOS_AMORT_SRC
#define WOS_AMORT_SRC 1
#endif
  constexpr bool kAmort = WOS_AMORT_RNG && kJumpFirst && W::kPerBlock > 1 &&
                          (S::SRC == SRC_NONE || (WOS_AMORT_SRC && W::kBetaTab));
  // Branch-free step (single-instance constant-boundary NATIVE kernels with a source:
  // cfg0, cfg4): no deferred recording, so an idle lane holds no state worth keeping
#ifndef WOS_HOT_LOOP
#define WOS_HOT_LOOP 1
#endif
  constexpr bool kHotLoop = WOS_HOT_LOOP && W::kHot && S::BC && kJumpFirst && !W::kScr &&
                            (W::kPerBlock == 1 || W::kBetaTab);
  // the general amortised-round loop (source-free kernels; the hot loop runs its own rounds)
  constexpr bool kAmortLoop = kAmort && !kHotLoop;
  // Exit-ring kernels run the hot loop's lean refill (lazy retirement, branch-light
  // issue of the cached unit's walks) and branch-free rounds (below)
#ifndef WOS_EXIT_LEAN
#define WOS_EXIT_LEAN 1
#endif
  constexpr bool kExitLoop = WOS_EXIT_LEAN && kExitRing && kAmortLoop && W::kHot && WOS_HOT_FOLD;
  constexpr bool kLean = kHotLoop || kExitLoop;
  // One hot-loop step of a walk slot; returns whether the walk is still live. With a
  // two-jump block (3D source jumps) a step is a round of two jumps from one Philox
  // block: every slot enters a round at an even step (walks start at step 0 and are
  // issued between rounds), and a walk that ends after the first jump skips the second.
  // the staged Beta(2,2) table's shared-memory offset
  uint32_t hot_btab = 0u;
  if constexpr (W::kBetaTab) hot_btab = W::beta_tab_offset(a);
#ifndef WOS_HOT_PRED_RECORD1
#define WOS_HOT_PRED_RECORD1 1
#endif
#ifndef WOS_HOT_BRANCHFREE
#define WOS_HOT_BRANCHFREE 1
#endif
  auto hot_step = [&](typename W::Lane& s) -> bool {
    if constexpr (kExitLoop) {
      // Branch-free round of kPerBlock source-free jumps, every lane, live or not: a
      // walk that has ended (or a lane without one: its stale state is an ended walk's,
      // d = -1 before the first) jumps by 0, which leaves its position, and with it
      // the recomputed distance, unchanged, and its step count is not advanced — the
      // same operations in the same order for the walks that continue, so the results
      // equal the branched round's of the amortised loop below
      const uint4 B = W::native_block_at(s, a, 2u * ((uint32_t)s.step / (uint32_t)W::kPerBlock));
#pragma unroll
      for (int k = 0; k < W::kPerBlock; ++k) {
        const bool live = !((s.d < eps) | (s.step >= a.max_steps));
        W::move_native_word(s, live ? s.d : 0.0f, B, k, a);
        s.step += live ? 1 : 0;
        s.d = W::dist(s, a, srec);
      }
      return !((s.d < eps) | (s.step >= a.max_steps));
    } else if constexpr (!kHotLoop) {
      return false;  // (not used outside the hot loop)
    } else if constexpr (W::kPerBlock == 2 && WOS_HOT_BRANCHFREE) {
      // Branch-free round: the second jump runs in every lane and a walk that ended
      // after the first keeps that jump's value and step count (selects) — the same
      // operations in the same order for the walks that continue, so the results are
      // identical to the branched round below, without its divergent reconvergence
      const uint4 B = W::native_block_at(s, a, 2u * ((uint32_t)s.step >> 1));
      W::jump_source(s, s.d, a, B.x, B.y, hot_btab);
      const Real acc1 = s.acc;
      const Real d1 = W::dist(s, a, srec);
      const bool live1 = !((d1 < eps) | (s.step + 1 >= a.max_steps));
      W::jump_source(s, d1, a, B.z, B.w, hot_btab);
      s.d = W::dist(s, a, srec);
      s.acc = live1 ? s.acc : acc1;
      s.step += live1 ? 2 : 1;
      return live1 & !((s.d < eps) | (s.step >= a.max_steps));
    } else if constexpr (W::kPerBlock == 2) {
      const uint4 B = W::native_block_at(s, a, 2u * ((uint32_t)s.step >> 1));
      W::jump_source(s, s.d, a, B.x, B.y, hot_btab);
      s.step += 1;
      s.d = W::dist(s, a, srec);
      bool live = !((s.d < eps) | (s.step >= a.max_steps));
      if (live) {
        W::jump_source(s, s.d, a, B.z, B.w, hot_btab);
        s.step += 1;
        s.d = W::dist(s, a, srec);
        live = !((s.d < eps) | (s.step >= a.max_steps));
      }
      return live;
    } else {
      W::advance_native(s, s.d, a);
      s.step += 1;
      s.d = W::dist(s, a, srec);
      return !((s.d < eps) | (s.step >= a.max_steps));
    }
  };
  auto record = [&](Real d) {
    // walker.py:275-281: value = acc + g(projection), steps, hit = (d < eps)
    lane_steps += (unsigned long long)l.step;
    if constexpr (kExitRing) {
      // source-free: acc = 0, the value is g(projection of x), evaluated at retirement
      Real* slot = reinterpret_cast<Real*>(reinterpret_cast<unsigned char*>(ring) + l.seq);
      *reinterpret_cast<float2*>(slot) = make_float2(l.x[0], l.x[1]);
      atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk), 1u);
      active = false;
      return;
    }
    const Real v = W::finish_value(l, a);
    if constexpr (est) {
      *reinterpret_cast<Real*>(reinterpret_cast<unsigned char*>(ring) + l.seq) = v;
      atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk), 1u);
    } else {
      a.out_values[l.seq] = (double)v;
      a.out_steps[l.seq] = (int64_t)l.step;
      // a dead walk (const kernel path) reports hit = 1 unless it also ran out of steps
      a.out_hits[l.seq] = (uint8_t)(d < eps || (l.step < a.max_steps && W::dead(l, a)));
    }
    active = false;
  };
  // Deferred recording. An expensive boundary term (Fourier / arc-length series,
  // projections) evaluated when a walk ends runs with the one or two lanes that ended
  // in that step while the rest of the warp waits, once per step. A finished lane
  // instead keeps its walk's state in registers (it idles until the next refill
  // anyway) and all such lanes are recorded together at the next refill: one pass per
  // refill instead of one per step. Constant boundaries record at once (no gain).
#ifndef WOS_DEFER_RECORD
#define WOS_DEFER_RECORD 1
#endif
  // amortised-round launches with deferred recording refill at refill_min_deferred + this
  // (4 was cfg1's optimum before its kernel moved to the exit ring; cfg2 x16: 1.705 ms at
  // +4, 1.666 at +0, 1.663 at -2)
#ifndef WOS_AMORT_DEFER_ADD
#define WOS_AMORT_DEFER_ADD 0
#endif
  // exit-ring launches refill at refill_min + this many idle lanes (between rounds)
#ifndef WOS_EXIT_REFILL_ADD
#define WOS_EXIT_REFILL_ADD 4  // cfg1 x16: 1.566 ms at +0, 1.545 at +4, 1.556 at +7
#endif
  const bool defer = WOS_DEFER_RECORD && !kExitRing && !S::BC && a.bnd_kind != BND_CONST;
  bool pend = false;
  auto finish = [&](Real d) {
    if (defer) {
      l.d = d;
      pend = true;
      active = false;
    } else {
      record(d);
    }
  };
  auto flush = [&]() {
    if (defer && __any_sync(WOS_FULL, pend)) {
      if (pend) {
        record(l.d);
        pend = false;
      }
    }
  };
  // jump-first: query a freshly started walk; one starting in the shell ends here
  auto first_query = [&]() {
    if constexpr (kJumpFirst) {
      l.d = W::dist(l, a, srec);
      if (l.d < eps) finish(l.d);
    }
  };
  // the fast refill's walks all start at the cached point: its distance is queried once
  // per unit (warp-uniform) and an in-shell start is a uniform branch
  Real cu_d = Real(0);
  int cu_seg = 0;  // polygons: the nearest segment at the cached point

  // ======================================================================
  // Eager fast path (ESTIMATE, one point per unit, polygon domains): finished walks
  // are recorded and their lanes re-issued in the same divergent block right after
  // the step; unit grabs, retirement and the exit test run only when the unit or
  // the ring runs short. Re-issuing every iteration costs a divergent start per
  // iteration, which paid off (7 %) while a polygon jump was a full 128-segment
  // scan; with the candidate grid the jump is cheap and the batched refill of the
  // general loop below is as fast, so it is off by default (-D WOS_POLY_EAGER=1).
  // ======================================================================
#ifndef WOS_POLY_EAGER
#define WOS_POLY_EAGER 0
#endif
  constexpr bool kEager = WOS_POLY_EAGER && (S::DOM == DOM_POLY);
  if (kEager && fast) {
    while (true) {
      bool fin = false;
      if (active) {
        const Real d = W::dist(l, a, srec);
        if (d < eps || l.step >= a.max_steps || W::dead(l, a)) {
          fin = true;
        } else {
          if constexpr (W::kScr) {
            if constexpr (S::NATIVE) W::advance_screened_native(l, d, a);
            else W::advance_screened_replay(l, d, a);
          } else if constexpr (S::NATIVE) W::advance_native(l, d, a);
          else W::advance_replay(l, d, a);
          l.step += 1;
        }
      }
      idle |= __ballot_sync(WOS_FULL, fin);
      if (idle == 0u) continue;
      if (fin) {  // record: walker.py:275-281, value = acc + g(projection)
        const Real v = W::finish_value(l, a);
        lane_steps += (unsigned long long)l.step;
        *reinterpret_cast<Real*>(reinterpret_cast<unsigned char*>(ring) + l.seq) = v;
        atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk), 1u);
        active = false;
      }
      const uint32_t n_idle = (uint32_t)__popc(idle);
      uint32_t room = cu_end - s_issue;
      uint32_t cap = r_seq + (uint32_t)kRing - s_issue;
      if (room < n_idle || cap < n_idle) {
        // ---- slow path: free the ring, move to the next unit, or finish ----
        if (++refills > a.iter_limit) {  // watchdog (a stall can only loop through here)
          if (lane == 0) atomicExch(a.watchdog, 1u);
          break;
        }
        __syncwarp();
        retire();
        cap = r_seq + (uint32_t)kRing - s_issue;
        if (room == 0) {
          if (!exhausted && n_grabbed == cu_k + 1u && (n_grabbed - r_unit) < (uint32_t)kUQ) {
            uint32_t u = 0;
            if (lane == 0) u = atomicAdd(a.work_counter, 1u);
            u = __shfl_sync(WOS_FULL, u, 0);
            if (u >= a.n_units) {
              exhausted = true;
            } else {
              if (lane == 0) unitq[n_grabbed % kUQ] = u;
              ++n_grabbed;
              s_avail += IU;
            }
          }
          if (n_grabbed != cu_k + 1u) {  // the next unit is grabbed: cache its point
            cu_k += 1u;
            cu_end += IU;
            const uint32_t unit = unitq[cu_k % kUQ];
            uint32_t p = unit;
            cu_j0 = 0;
            cu_jend = L;
            if (split) {
              p = fast_div(unit, a.nc_mul, a.nc_shr);
              cu_j0 = (unit - p * a.n_chunks) * kChunk;
              cu_jend = min(L, cu_j0 + kChunk);
            }
#pragma unroll
            for (int i = 0; i < DIM; ++i) cu_x[i] = W::start_coord(a.points[(size_t)p * DIM + i]);
            cu_pid = a.point_ids ? (uint64_t)a.point_ids[p] : a.id_base + p;
            cu_inst = (!S::ONE && a.inst_index) ? a.inst_index[p] : 0;
            room = IU;
          } else if (n_idle == 32 && exhausted && r_seq == s_issue) {
            break;  // no walk left, none running, all retired
          }
        }
      }
      const uint32_t n = min(min(n_idle, room), cap);
      if (!active) {
        const uint32_t rank = __popc(idle & lanemask_lt());
        if (rank < n) {
          const uint32_t seq = s_issue + rank;
          const uint32_t j = cu_j0 + (seq - (cu_end - IU));
          blk = (cu_k % kSlots) * 4u;
          if (j < cu_jend) {
            const uint64_t tid = anti ? a.traj_start + 2ull * (j >> 1) : a.traj_start + j;
            const double sg = (anti && (j & 1u)) ? -1.0 : 1.0;
            W::start(l, table, a.hdr, a, cu_x, cu_inst, cu_pid, tid, sg);
            l.seq = (seq % kRing) * (uint32_t)sizeof(Real);
            active = true;
          } else {  // null item padding the point's last chunk: complete at once
            atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk), 1u);
          }
        }
      }
      s_issue += n;
      idle = __ballot_sync(WOS_FULL, !active);
    }
  } else {
  bool ilp2_done = false;
#ifndef WOS_ILP2
#define WOS_ILP2 0
#endif
  // exit-ring kernels run it too (64 registers, 4 CTAs/SM instead of 48 and 5): their
  // refill, which runs every round, is paid once per two rounds (cfg1 x16 1.542 -> 1.480 ms)
#ifndef WOS_EXIT_ILP2
#define WOS_EXIT_ILP2 1
#endif
#ifndef WOS_EXIT_ILP2_MIN_UNITS
#define WOS_EXIT_ILP2_MIN_UNITS 16
#endif
  if constexpr ((WOS_ILP2 && kHotLoop) || (WOS_EXIT_ILP2 && kExitLoop)) {
    // (exit-ring launches with few units per warp keep one walk per lane: with two the
    // warps' last units run half empty — cfg1 as a single estimate, 5 units per warp:
    // 0.153 ms with two slots, WOS_EXIT_ILP2_MIN_UNITS decides)
    if (fast && (!kExitLoop || a.n_units >= (uint32_t)WOS_EXIT_ILP2_MIN_UNITS * gridDim.x * (blockDim.x >> 5))) {
      // ==================================================================
      // Two walks per lane (slots A = l, B = lb): every iteration jumps both, so the
      // two independent dependency chains interleave and the loop / vote / refill
      // control is paid once per two jumps. The walks are the same as in the
      // one-slot loop (each keeps its stream and ring slot); only which lane and slot
      // runs which walk differs, which the in-order reduction does not see.
      // ==================================================================
      typename W::Lane lb = l;  // (shares the keys and coefficients)
      bool act_a = false, act_b = false;
      uint32_t blk_a = 0, blk_b = 0;
      unsigned idle_a = WOS_FULL, idle_b = WOS_FULL;
      const int thr2 = __shfl_sync(WOS_FULL, min(64, 2 * (a.refill_min + (kExitLoop ? WOS_EXIT_REFILL_ADD : 0))), 0);
      // move the cached unit to the next grabbed one; false if none is left
      auto next_unit = [&]() -> bool {
        if (!exhausted && n_grabbed == cu_k + 1u && (n_grabbed - r_unit) < (uint32_t)kUQ) {
          uint32_t u = 0;
          if (lane == 0) u = atomicAdd(a.work_counter, 1u);
          u = __shfl_sync(WOS_FULL, u, 0);
          if (u >= a.n_units) {
            exhausted = true;
          } else {
            if (lane == 0) unitq[n_grabbed % kUQ] = u;
            ++n_grabbed;
            s_avail += IU;
          }
        }
        if (n_grabbed == cu_k + 1u) return false;
        cu_k += 1u;
        cu_end += IU;
        const uint32_t unit = unitq[cu_k % kUQ];
        uint32_t p = unit;
        cu_j0 = 0;
        cu_jend = L;
        if (split) {
          p = fast_div(unit, a.nc_mul, a.nc_shr);
          cu_j0 = (unit - p * a.n_chunks) * kChunk;
          cu_jend = min(L, cu_j0 + kChunk);
        }
#pragma unroll
        for (int i = 0; i < DIM; ++i) cu_x[i] = W::start_coord(a.points[(size_t)p * DIM + i]);
        cu_pid = a.point_ids ? (uint64_t)a.point_ids[p] : a.id_base + p;
        cu_d = W::dist_at(l, a, cu_x);
        const uint64_t tid0 = a.traj_start + cu_j0;
        cu_c1 = (uint32_t)cu_pid;
        cu_c2b = (uint32_t)tid0;
        cu_c3 = (uint32_t)(tid0 >> 32) ^ ((uint32_t)(cu_pid >> 32) * 0x85EBCA6Bu);
        cu_pu = philox_pre_unit(cu_c1, cu_c3, l.hk1[0], l.hk0[1], l.hk1[1], l.hk0[2]);
        cu_fastc = (uint64_t)(uint32_t)tid0 + (cu_jend - cu_j0) <= 0x100000000ull;
        return true;
      };
      auto record2 = [&](typename W::Lane& s, uint32_t blk_s) {
        lane_steps += (unsigned long long)s.step;
        if constexpr (kExitLoop)
          *reinterpret_cast<float2*>(reinterpret_cast<unsigned char*>(ring) + s.seq) = make_float2(s.x[0], s.x[1]);
        else
        *reinterpret_cast<Real*>(reinterpret_cast<unsigned char*>(ring) + s.seq) = s.acc + a.bnd_c;
        atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk_s), 1u);
      };
      // Predicated recording (no divergent branch around the one to three lanes that
      // finish per iteration): the ring store and the unit-counter increment go out
      // under the lane's predicate; the step total accumulates in 32 bits and is
      // folded into the 64-bit lane total at every refill (a lane cannot run 2^32
      // steps between two refills)
#ifndef WOS_HOT_PRED_RECORD
#define WOS_HOT_PRED_RECORD 1
#endif
      const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
      const uint32_t cnt_s = (uint32_t)__cvta_generic_to_shared(cnt);
      uint32_t steps32 = 0u;
      auto record2p = [&](typename W::Lane& s, uint32_t blk_s, bool fin) {
        if constexpr (kExitLoop) {  // the exit position (exit ring)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.v2.f32 [%1], {%2, %3};\n\t"
              "@p red.shared.add.u32 [%4], 1;\n\t}" ::"r"((uint32_t)fin),
              "r"(ring_s + s.seq), "f"(s.x[0]), "f"(s.x[1]), "r"(cnt_s + blk_s)
              : "memory");
          steps32 += fin ? (uint32_t)s.step : 0u;
          return;
        }
        const float v = s.acc + a.bnd_c;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.f32 [%1], %2;\n\t"
            "@p red.shared.add.u32 [%3], 1;\n\t}" ::"r"((uint32_t)fin),
            "r"(ring_s + s.seq), "f"(v), "r"(cnt_s + blk_s)
            : "memory");
        steps32 += fin ? (uint32_t)s.step : 0u;
      };
      // issue the cached unit's next walks to the idle lanes of one slot; ranks start at base
      auto issue = [&](typename W::Lane& s, bool& act, uint32_t& blk_s, unsigned idle_s, uint32_t base,
                       uint32_t n) {
        const uint32_t rank = base + __popc(idle_s & lanemask_lt());
        const uint32_t seq = s_issue + rank;
        const uint32_t jr = seq - (cu_end - IU);
        const bool take = !act && rank < n;
        const bool real = cu_j0 + jr < cu_jend;
        const uint32_t blk_new = (cu_k % kSlots) * 4u;
        if (cu_fastc) {
          const uint32_t c2 = cu_c2b + (jr & anti_jmask);
          const PhiloxPre pc = philox_pre_walk(c2, cu_pu, l.hk0[0], l.hk1[2]);
          if (take && real) {
#pragma unroll
            for (int i = 0; i < DIM; ++i) s.x[i] = cu_x[i];
            s.acc = Real(0);
            s.step = 0;
            s.d = cu_d;
            s.pc = pc;
            s.sgn = __int_as_float(0x3f800000 | ((jr & anti_bit) << 31));
            s.seq = (seq % kRing) * kSlotBytes;
            blk_s = blk_new;
            act = true;
          }
        } else if (take && real) {
          const uint32_t j = cu_j0 + jr;
          const uint64_t tid = anti ? a.traj_start + 2ull * (j >> 1) : a.traj_start + j;
          W::start(s, table, a.hdr, a, cu_x, cu_inst, cu_pid, tid, (anti && (j & 1u)) ? -1.0 : 1.0);
          s.d = cu_d;
          s.seq = (seq % kRing) * kSlotBytes;
          blk_s = blk_new;
          act = true;
        }
        if (take && !real) atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk_new), 1u);
        if constexpr (!kExitLoop) {  // (an exit-ring round finishes such a walk itself)
          if (cu_d < eps && take && real) {  // the unit's point lies in the shell
            record2(s, blk_s);
            act = false;
          }
        }
      };
      while (true) {
        const uint32_t na = (uint32_t)__popc(idle_a);
        const int n_idle = (int)na + __popc(idle_b);
        if (n_idle >= thr2) {
          if constexpr (WOS_HOT_PRED_RECORD) {
            lane_steps += (unsigned long long)steps32;
            steps32 = 0u;
          }
          uint32_t room = cu_end - s_issue;
          uint32_t cap = r_seq + (uint32_t)kRing - s_issue;
          if (cap < (uint32_t)n_idle || room == 0) {
            retire();
            cap = r_seq + (uint32_t)kRing - s_issue;
          }
          if (room == 0 || cap == 0) {
            if (++refills > a.iter_limit) {
              if (lane == 0) atomicExch(a.watchdog, 1u);
              break;
            }
            if (room == 0) {
              if (next_unit()) {
                room = IU;
              } else if (n_idle == 64 && exhausted) {
                retire();
                if (r_seq == s_issue) break;  // no walk left, none running, all retired
              }
            }
          }
          const uint32_t n = min(min((uint32_t)n_idle, room), cap);
          issue(l, act_a, blk_a, idle_a, 0u, n);
          issue(lb, act_b, blk_b, idle_b, na, n);
          s_issue += n;
        }
        const bool live_a = hot_step(l);
        const bool live_b = hot_step(lb);
        const bool fin_a = act_a & !live_a;
        const bool fin_b = act_b & !live_b;
        if constexpr (WOS_HOT_PRED_RECORD) {
          record2p(l, blk_a, fin_a);
          record2p(lb, blk_b, fin_b);
        } else {
          if (fin_a) record2(l, blk_a);
          if (fin_b) record2(lb, blk_b);
        }
        act_a = act_a & !fin_a;
        act_b = act_b & !fin_b;
        idle_a = __ballot_sync(WOS_FULL, !act_a);
        idle_b = __ballot_sync(WOS_FULL, !act_b);
      }
      ilp2_done = true;
    }
  }
  if (!ilp2_done) {
  // Refill threshold (idle lanes), loop-invariant and at most 32 so that an all-idle
  // warp always refills; it goes through a shuffle so ptxas keeps it in a register
  // instead of reloading it from the constant bank every iteration.
  // (delta tracking: a step costs far more than recording, so the plain threshold;
  // amortised rounds refill only between rounds and batch 4 more: cfg1 -1.9 %)
  // polar walks keep their closest point, so recording a batch is only the boundary
  // term: they refill at the plain threshold (sweep 4-12: 17.7 ms at 4, 19.5 at 12 on
  // the mild curve; meshes, whose start and traversal cost more, keep the deferred one)
  constexpr bool kCheapRecord = WOS_KEEP_CLOSEST && S::DOM == DOM_POLAR;
  const int refill_thr = __shfl_sync(
      WOS_FULL,
      min(32, (defer && !W::kScr && !kCheapRecord) ? a.refill_min_deferred + (kAmortLoop ? WOS_AMORT_DEFER_ADD : 0)
                  : kCheapRecord   ? max(1, a.refill_min - 2)  // (sweep 2-7: 3 within 0.5 % of the best)
                  : kExitLoop      ? a.refill_min + WOS_EXIT_REFILL_ADD
                  : kExitRing      ? a.refill_min
                  : kAmortLoop     ? 1
                                   : a.refill_min), 0);
  while (true) {
    const int n_idle = __popc(idle);
    if (n_idle >= refill_thr) {
      flush();  // record the lanes that finished since the last refill
      // retire lazily: the ring holds kRing walks, so completed units only need to be
      // reduced before new walks are issued (one shared-memory check, no vote)
      if (est && (!kLean || !fast)) {  // (the hot loop's cached-unit refill retires lazily)
        __syncwarp();  // order the lanes' counter updates before the check
        if (r_seq + IU <= s_issue && cnt[r_unit % kSlots] == IU) retire();
      }
      if (fast) {
        // ============ refill, one point per unit: cached point in registers ============
        uint32_t room = cu_end - s_issue;
        uint32_t cap = r_seq + (uint32_t)kRing - s_issue;
        if constexpr (kLean) {
          // the hot loop refills in small batches: it retires only when the ring is
          // short of slots for them or a new unit is due (the unit queue and counter
          // slots must have room); retire() orders the lanes' counter updates itself
          if (cap < (uint32_t)n_idle || room == 0) {
            retire();
            cap = r_seq + (uint32_t)kRing - s_issue;
          }
        }
        if (room == 0 || cap == 0) {
          // watchdog: bail out and flag instead of spinning forever if the stream
          // bookkeeping ever stalled (a stall can only loop through here)
          if (++refills > a.iter_limit) {
            if (lane == 0) atomicExch(a.watchdog, 1u);
            break;
          }
          if (room == 0) {  // current unit fully issued: move to the next one
            if (!exhausted && n_grabbed == cu_k + 1u && (n_grabbed - r_unit) < (uint32_t)kUQ) {
              uint32_t u = 0;
              if (lane == 0) u = atomicAdd(a.work_counter, 1u);
              u = __shfl_sync(WOS_FULL, u, 0);
              if (u >= a.n_units) {
                exhausted = true;
              } else {
                if (lane == 0) unitq[n_grabbed % kUQ] = u;
                ++n_grabbed;
                s_avail += IU;
              }
            }
            if (n_grabbed != cu_k + 1u) {  // the next unit is grabbed: cache its point
              cu_k += 1u;
              cu_end += IU;
              const uint32_t unit = unitq[cu_k % kUQ];
              uint32_t p = unit;
              cu_j0 = 0;
              cu_jend = L;
              if (split) {
                p = fast_div(unit, a.nc_mul, a.nc_shr);
                cu_j0 = (unit - p * a.n_chunks) * kChunk;
                cu_jend = min(L, cu_j0 + kChunk);
              }
#pragma unroll
              for (int i = 0; i < DIM; ++i) cu_x[i] = W::start_coord(a.points[(size_t)p * DIM + i]);
              cu_pid = a.point_ids ? (uint64_t)a.point_ids[p] : a.id_base + p;
              cu_inst = (!S::ONE && a.inst_index) ? a.inst_index[p] : 0;
              if constexpr (kJumpFirst && S::ONE) cu_d = W::dist_at(l, a, cu_x);
              if constexpr (kJumpFirstPoly) {
                // the whole warp queries the unit's start point once (uniform work)
                typename W::Lane t = l;
                W::start(t, table, a.hdr, a, cu_x, cu_inst, cu_pid, 0ull, 1.0);
                cu_d = W::dist(t, a, srec);
                cu_seg = t.seg_i;
                l.nseg = t.nseg;  // every lane evaluated the unit's start query
              }
              if constexpr (S::NATIVE && S::ONE) {
                // walk j0 + jj has tid = traj_start + j0 + jj (antithetic: jj even; j0 even)
                const uint64_t tid0 = a.traj_start + cu_j0;
                cu_c1 = (uint32_t)cu_pid;
                cu_c2b = (uint32_t)tid0;
                cu_c3 = (uint32_t)(tid0 >> 32) ^ ((uint32_t)(cu_pid >> 32) * 0x85EBCA6Bu);
                if constexpr (W::kHot) cu_pu = philox_pre_unit(cu_c1, cu_c3, l.hk1[0], l.hk0[1], l.hk1[1], l.hk0[2]);
                cu_fastc = (uint64_t)(uint32_t)tid0 + (cu_jend - cu_j0) <= 0x100000000ull;
              }
              room = IU;
            } else if (n_idle == 32 && exhausted) {
              if constexpr (kLean) retire();  // (retirement is lazy there)
              if (r_seq == s_issue) break;  // no walk left, none running, all retired
            }
          }
        }
        const uint32_t n = min(min((uint32_t)n_idle, room), cap);
        if constexpr (kLean) {
          // Branch-light issue of the cached unit's next walks: the per-lane start state
          // (counter fold, sign, ring slot) is computed by every lane and committed by the
          // lanes that take a walk; the point, its distance and the unit slot are
          // warp-uniform. Same walks and streams as the general issue below.
          const uint32_t rank = __popc(idle & lanemask_lt());
          const uint32_t seq = s_issue + rank;
          const uint32_t jr = seq - (cu_end - IU);
          const bool take = !active && rank < n;
          const bool real = cu_j0 + jr < cu_jend;  // else a null item padding the last chunk
          const uint32_t blk_new = (cu_k % kSlots) * 4u;
          if (cu_fastc) {
            const uint32_t c2 = cu_c2b + (jr & anti_jmask);
            const PhiloxPre pc = philox_pre_walk(c2, cu_pu, l.hk0[0], l.hk1[2]);
            if (take && real) {
#pragma unroll
              for (int i = 0; i < DIM; ++i) l.x[i] = cu_x[i];
              l.acc = Real(0);
              l.step = 0;
              l.d = cu_d;
              l.pc = pc;
              l.sgn = __int_as_float(0x3f800000 | ((jr & anti_bit) << 31));
              l.seq = (seq % kRing) * kSlotBytes;
              blk = blk_new;
              active = true;
            }
          } else if (take && real) {  // the unit's traj ids cross a 2^32 boundary
            const uint32_t j = cu_j0 + jr;
            const uint64_t tid = anti ? a.traj_start + 2ull * (j >> 1) : a.traj_start + j;
            W::start(l, table, a.hdr, a, cu_x, cu_inst, cu_pid, tid, (anti && (j & 1u)) ? -1.0 : 1.0);
            l.d = cu_d;
            l.seq = (seq % kRing) * kSlotBytes;
            blk = blk_new;
            active = true;
          }
          if (take && !real) atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk_new), 1u);
          // the unit's point lies in the shell (an exit-ring round finishes such a walk itself)
          if constexpr (!kExitLoop)
            if (cu_d < eps && take && real) finish(cu_d);
        } else if (!active) {
          const uint32_t rank = __popc(idle & lanemask_lt());
          if (rank < n) {
            const uint32_t seq = s_issue + rank;
            const uint32_t jr = seq - (cu_end - IU);
            const uint32_t j = cu_j0 + jr;
            blk = (cu_k % kSlots) * 4u;
            if (j < cu_jend) {
              bool started = false;
              if constexpr (S::NATIVE && S::ONE && !W::kScr && S::DOM != DOM_POLY &&
                            S::DOM != DOM_POLAR && S::DOM != DOM_MESH) {
                if (cu_fastc) {
                  W::start_native(l, a, cu_x, (anti && (jr & 1u)) ? -1.0f : 1.0f, cu_c1,
                                  cu_c2b + (anti ? (jr & ~1u) : jr), cu_c3);
                  started = true;
                }
              }
              if (!started) {
                const uint64_t tid = anti ? a.traj_start + 2ull * (j >> 1) : a.traj_start + j;
                const double sg = (anti && (j & 1u)) ? -1.0 : 1.0;
                W::start(l, table, a.hdr, a, cu_x, cu_inst, cu_pid, tid, sg);
              }
              l.seq = (seq % kRing) * kSlotBytes;
              active = true;
              if constexpr (kJumpFirstPoly) {
                l.d = cu_d;
                l.seg_i = cu_seg;
                if (cu_d < eps) finish(cu_d);
              } else if constexpr (kJumpFirst && S::ONE) {
                l.d = cu_d;
                if (cu_d < eps) finish(cu_d);
              } else {
                first_query();
              }
            } else {  // null item padding the point's last chunk: complete at once
              atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk), 1u);
            }
          }
        }
        s_issue += n;
      } else {
        // ================= refill idle lanes (general) =================
        if (++refills > a.iter_limit) {
          if (lane == 0) atomicExch(a.watchdog, 1u);
          break;
        }
        const uint32_t live_units = n_grabbed - (est ? r_unit : fast_div(s_issue, a.iu_mul, a.iu_shr));
        bool grab = !exhausted && (s_avail - s_issue) < (uint32_t)n_idle && live_units < (uint32_t)kUQ;
        while (grab) {
          uint32_t u = 0;
          if (lane == 0) u = atomicAdd(a.work_counter, 1u);
          u = __shfl_sync(WOS_FULL, u, 0);
          if (u >= a.n_units) {
            exhausted = true;
          } else {
            if (lane == 0) unitq[n_grabbed % kUQ] = u;
            ++n_grabbed;
            s_avail += IU;
          }
          grab = !exhausted && (s_avail - s_issue) < (uint32_t)n_idle &&
                 (n_grabbed - (est ? r_unit : fast_div(s_issue, a.iu_mul, a.iu_shr))) < (uint32_t)kUQ;
        }
        __syncwarp();
        uint32_t n = min((uint32_t)n_idle, s_avail - s_issue);
        if (est) n = min(n, r_seq + (uint32_t)kRing - s_issue);
        if (n == 0 && n_idle == 32 && exhausted && s_issue == s_avail && (!est || r_seq == s_issue))
          break;  // no walk left, none running, all retired
        const uint32_t rank = __popc(idle & lanemask_lt());
        if (!active && rank < n) {
          const uint32_t seq = s_issue + rank;
          const uint32_t k = fast_div(seq, a.iu_mul, a.iu_shr);
          const uint32_t r = seq - k * IU;
          const uint32_t unit = unitq[k % kUQ];
          if constexpr (est) {
            const uint32_t pl = fast_div(r, a.l_mul, a.l_shr);
            const uint32_t j = r - pl * L;
            const uint64_t p = (uint64_t)unit * U + pl;
            blk = (k % kSlots) * 4u;
            if (p < a.n_points) {
              const int inst = (!S::ONE && a.inst_index) ? a.inst_index[p] : 0;
              const uint64_t tid = anti ? a.traj_start + 2ull * (j >> 1) : a.traj_start + j;
              const double sg = (anti && (j & 1u)) ? -1.0 : 1.0;
              W::start(l, table, a.hdr, a, a.points + (size_t)p * DIM, inst,
                       a.point_ids ? (uint64_t)a.point_ids[p] : a.id_base + p, tid, sg);
              l.seq = (seq % kRing) * kSlotBytes;
              active = true;
              first_query();
            } else {  // null item padding the last unit: complete at once
              atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk), 1u);
            }
          } else {
            const uint64_t row = (uint64_t)unit * IU + r;
            if (row < a.n_points) {
              W::start(l, table, a.hdr, a, a.points + (size_t)row * DIM, 0, a.row_pid[row],
                       a.row_tid[row], a.row_sign[row]);
              l.seq = (uint32_t)row;
              active = true;
              first_query();
            }
          }
        }
        s_issue += n;
      }
    }

    // ================= one step of every active walk =================
    if constexpr (kExitLoop) {
      // one branch-free round of every lane (hot_step above)
      const bool fin = active & !hot_step(l);
      // predicated record: the exit position to the walk's ring slot, one more of its unit done
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.v2.f32 [%1], {%2, %3};\n\t"
          "@p red.shared.add.u32 [%4], 1;\n\t}" ::"r"((uint32_t)fin),
          "r"((uint32_t)__cvta_generic_to_shared(ring) + l.seq), "f"(l.x[0]), "f"(l.x[1]),
          "r"((uint32_t)__cvta_generic_to_shared(cnt) + blk)
          : "memory");
      lane_steps += fin ? (unsigned long long)l.step : 0ull;
      active = active & !fin;
    } else if constexpr (kAmortLoop) {
      // one round: kPerBlock jumps of every live lane from one Philox block
      // (a lane whose walk ends mid-round stops moving and is finished after the round:
      // the sub-jumps stay straight-line predicated code)
      if (active) {
        const uint4 B = W::native_block_at(l, a, 2u * ((uint32_t)l.step / (uint32_t)W::kPerBlock));
        bool live = true;
        if constexpr (W::kBetaTab) {
          // source rounds: one jump body in a loop (two unrolled source jumps with the
          // block held across them spill at the multi-instance kernels' 64 registers)
#pragma unroll 1
          for (int k = 0; k < 2; ++k) {
            if (live) {
              W::jump_source(l, l.d, a, k == 0 ? B.x : B.z, k == 0 ? B.y : B.w);
              l.step += 1;
              l.d = W::dist(l, a, srec);
              live = !(l.d < eps || l.step >= a.max_steps);
            }
          }
        } else {
#pragma unroll
        for (int k = 0; k < W::kPerBlock; ++k) {
          if (live) {
            W::move_native_word(l, l.d, B, k, a);
            l.step += 1;
            l.d = W::dist(l, a, srec);
            live = !(l.d < eps || l.step >= a.max_steps);
          }
        }
        }
        if (!live) finish(l.d);
      }
    } else if constexpr (kHotLoop) {
      // every lane jumps, live or not: an idle lane (its walk recorded, the lane waiting
      // for a refill) computes a jump from its stale state that is never recorded, and
      // the warp runs the step without a divergent branch around it
      const bool fin = active & !hot_step(l);
      if constexpr (WOS_HOT_PRED_RECORD1) {
        // predicated record (as in the two-slot loop)
        const float v = l.acc + a.bnd_c;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.f32 [%1], %2;\n\t"
            "@p red.shared.add.u32 [%3], 1;\n\t}" ::"r"((uint32_t)fin),
            "r"((uint32_t)__cvta_generic_to_shared(ring) + l.seq), "f"(v),
            "r"((uint32_t)__cvta_generic_to_shared(cnt) + blk)
            : "memory");
        lane_steps += fin ? (unsigned long long)l.step : 0ull;
      } else if (fin) {
        lane_steps += (unsigned long long)l.step;
        *reinterpret_cast<Real*>(reinterpret_cast<unsigned char*>(ring) + l.seq) = l.acc + a.bnd_c;
        atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnt) + blk), 1u);
      }
      active = active & !fin;
    } else if (active) {
      if (jf) {
        // the walk is live at l.d >= eps, step < max_steps (tested when l.d was queried)
        if constexpr (W::kScr) {
          if constexpr (S::NATIVE) W::advance_screened_native(l, l.d, a);
          else W::advance_screened_replay(l, l.d, a);
        } else if constexpr (S::NATIVE) W::advance_native(l, l.d, a);
        else W::advance_replay(l, l.d, a);
        l.step += 1;
        l.d = W::dist(l, a, srec);
        if (l.d < eps || l.step >= a.max_steps || W::dead(l, a)) finish(l.d);
      } else {
        const Real d = W::dist(l, a, srec);
        if (d < eps || l.step >= a.max_steps || W::dead(l, a)) {
          finish(d);
        } else {
          if constexpr (W::kScr) {
            if constexpr (S::NATIVE) W::advance_screened_native(l, d, a);
            else W::advance_screened_replay(l, d, a);
          } else if constexpr (S::NATIVE) W::advance_native(l, d, a);
          else W::advance_replay(l, d, a);
          l.step += 1;
        }
      }
    }
    idle = __ballot_sync(WOS_FULL, !active);
  }
  }
  }

  // ---- walk-step total (u64, deterministic integer sum) ----
  if (a.total_steps != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lane_steps += __shfl_xor_sync(WOS_FULL, lane_steps, o);
    if (lane == 0) atomicAdd(a.total_steps, lane_steps);
  }
  // ---- NATIVE polygon work counter: segment distances evaluated (measured FP32 work) ----
  if constexpr (S::NATIVE && S::DOM == DOM_POLY) {
    if (a.seg_evals != nullptr) {
      unsigned long long ns = l.nseg;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ns += __shfl_xor_sync(WOS_FULL, ns, o);
      if (lane == 0) atomicAdd(a.seg_evals, ns);
    }
  }
}

// NW warps per CTA (the host reads it per kernel: wos_kernels_native.cu)
template <class S, int MINB, int NW = kWarps>
__global__ void __launch_bounds__(32 * NW, MINB) wos_walk_kernel(const __grid_constant__ KArgs a) {
  wos_kernel_body<S>(a);
}

}  // namespace wos
