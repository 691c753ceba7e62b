/*
 * wos_b200.h — C ABI of the B200-native Walk-on-Spheres (WoS) label estimator.
 *
 * This is the drop-in boundary for the reference's hot path
 * (arxiv 2603.01193, package `spherewalk`):
 *
 *   reference entry point                                   replaced by
 *   ------------------------------------------------------  ---------------------------
 *   walker.walk_poisson_values      (walker.py:181-229)     wos_walk_rows / _host
 *   _kernels.walk_plain_2d          (_kernels.py:286-367)   wos_walk_rows (2D rows)
 *   _kernels.walk_plain_ball3       (_kernels.py:375-468)   wos_walk_rows (3D rows)
 *   walker._poisson_generic         (walker.py:257-314)     wos_walk_rows (any spec)
 *   estimator.estimate              (estimator.py:144-181)  wos_estimate / _host
 *   estimator._estimate_block       (estimator.py:119-141)  wos_estimate (fused reduce)
 *   estimator.PointEstimate.from_values (estimator.py:106-110) fused per-point reduce
 *   rng.philox4x64                  (rng.py:57-82)          wos_philox4x64
 *   geometry.*.contains             (geometry.py:190-194)   wos_check_interior
 *   estimator.EstimateCache.update / cache_update (estimator.py:217-244,338-341)
 *                                                           wos_cache_fold
 *   surrogate.train label epoch     (surrogate.py:288-298)  wos_estimate_fold
 *
 * Entry points without a reference counterpart: wos_philox4x32 (the NATIVE stream's
 * generator, for KATs), wos_set_tuning / wos_set_refill_deferred (launch tuning; results
 * are bitwise independent of it), wos_probe_peaks (roofline denominators) and
 * wos_fastmath_probe (the fast-math error bound).
 *
 * Conventions (kept from the reference):
 *   - The reference solves  Laplacian(u) = f,  u = g on the boundary, and SUBTRACTS
 *     Green-weighted source samples (_kernels.py:307-311, walker.py:298). The kind
 *     codes below take f in that convention; a  -Laplacian(u) = f  problem passes -f.
 *   - Every trajectory is a pure function of (rng_seed, instance_key, point_id,
 *     traj_id, sign): results never depend on batch layout, launch shape or the
 *     number of GPUs (walker.py:11-14, test_estimator.py:147-154).
 *   - Kernels never raise; every entry point returns a wos_status and
 *     wos_last_error() holds a one-line message (the reference validates in Python,
 *     estimator.py:156-163, walker.py:139-145).
 *   - Output buffers are caller-owned. The *_host variants take host pointers and
 *     do the host<->device copies themselves; the others take device pointers and
 *     are ordered on the given CUDA stream (cudaStream_t passed as void*).
 *
 * No torch or CUDA types appear in these signatures.
 */
#ifndef WOS_B200_H
#define WOS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WOS_ABI_VERSION 4

/* ---- status codes ---------------------------------------------------- */
typedef enum wos_status {
  WOS_OK = 0,
  WOS_ERR_INVALID = 1,     /* bad argument (shape, size, parameter count)        */
  WOS_ERR_UNSUPPORTED = 2, /* domain/source/boundary kind not GPU-codeable       */
  WOS_ERR_CUDA = 3,        /* CUDA runtime error                                 */
  WOS_ERR_EXTERIOR = 4,    /* a start point lies outside the domain              */
  WOS_ERR_NOMEM = 5,
  WOS_ERR_MAJORANT = 6     /* delta tracking: sigma' exceeded sigma_bar (walker.py:51-52) */
} wos_status;

/* ---- numeric modes --------------------------------------------------- */
/* REPLAY_*: the reference's own estimator, draw for draw. Philox4x64-10 keyed
 *   (rng_seed, instance_key), counter (draw, point_id, traj_id, tag) exactly as
 *   walker.py:289,302 and _kernels.py:348,444; uniform-ball source sampling with
 *   |B| * G weights (walker.py:290-311).
 *   REPLAY_F64 runs the walk arithmetic in fp64, REPLAY_F32 rounds the uniforms to
 *   fp32 and runs the arithmetic in fp32.
 * NATIVE_F32: the production estimator. Philox4x32-10, Green's-function importance
 *   sampling of the source term (mass r^2/(2d): r^2/4 in 2D, r^2/6 in 3D,
 *   greens.py:83-89), fast-math sincos, fp32 walk state. Same expectation as the
 *   reference; statistically, not bitwise, equal.                             */
typedef enum wos_mode {
  WOS_MODE_REPLAY_F64 = 0,
  WOS_MODE_REPLAY_F32 = 1,
  WOS_MODE_NATIVE_F32 = 2
} wos_mode;

/* ---- domain kinds and parameter layouts (double[]) ------------------ */
/* WOS_DOM_BALL     disk (dim 2) or ball (dim 3):      [c_0..c_{dim-1}, R]
 *                  = geometry.BallDomain (geometry.py:172-238)
 * WOS_DOM_POLAR    2D star curve r(t) = r0 (1 + c1 cos 4t + c2 cos 8t) = geometry.PolarDomain
 *                  (geometry.py:83-153): [r0, c1, c2] (the library tabulates the curve at
 *                  4096 angles with its own libm) or [r0, c1, c2, stride, n, bx_0..bx_{n-1},
 *                  by_0..by_{n-1}] with the reference's own table (PolarDomain._bx/_by,
 *                  _stride) for bit-level replay. Distance and closest point follow
 *                  _kernels.polar_query_fast (strided table scan + window + one parabolic
 *                  refinement, _kernels.py:121-219); inside = |x| < r(atan2(y, x))
 * WOS_DOM_BOX      axis-aligned box:                   [lo_0..lo_{dim-1}, hi_0..hi_{dim-1}]
 *                  distance = min over faces, closest point = projection on the
 *                  first nearest face (axis order, lower face before upper face)
 * WOS_DOM_POLYGON  closed 2D polygon, n vertices:      [n, x_0, y_0, ..., x_{n-1}, y_{n-1}]
 *                  segments v_i -> v_{(i+1) mod n}; distance = min over segments,
 *                  closest point on the first nearest segment; inside = crossing
 *                  number (even-odd) test
 * WOS_DOM_MESH     closed, consistently oriented 3D triangle mesh = geometry.MeshDomain
 *                  (geometry.py:400-580): [nv, nf, v_0.x, v_0.y, v_0.z, ..., f_0.i, f_0.j,
 *                  f_0.k, ...] (face indices as doubles). The library builds a BVH;
 *                  distance / closest point = nearest triangle (closest_on_triangles,
 *                  geometry.py:259-323); inside = angle-weighted pseudo-normal test of
 *                  the closest feature (geometry.py:480-520)                      */
enum {
  WOS_DOM_BALL = 0,
  WOS_DOM_POLAR = 1,
  WOS_DOM_BOX = 2,
  WOS_DOM_POLYGON = 3,
  WOS_DOM_MESH = 4
};

/* ---- source kinds (f in the reference's  Laplacian(u) = f  convention) */
/* WOS_SRC_NONE     no source term
 * WOS_SRC_CONST    [c]                                   (_kernels.SRC_CONST)
 * WOS_SRC_RBF2     2D only: [a1, a2, c1x, c1y, c2x, c2y],
 *                  f = a1 exp(-|x-c1|^2) + a2 exp(-|x-c2|^2) (_kernels.py:248-259)
 * WOS_SRC_SINE     [K, a...] with K^dim coefficients in C order,
 *                  f = sum_{k_i=1..K} a_{k_0..} prod_i sin(k_i pi x_i)
 * WOS_SRC_GAUSS    [A, sigma, c_0..c_{dim-1}], f = A exp(-|x-c|^2 / (2 sigma^2)) */
enum {
  WOS_SRC_NONE = 0,
  WOS_SRC_CONST = 1,
  WOS_SRC_RBF2 = 2,
  WOS_SRC_SINE = 3,
  WOS_SRC_GAUSS = 4,
  WOS_SRC_SCREENED_CONST = 5,
  WOS_SRC_SCREENED_VC = 6
};

/* ---- delta tracking (walker.ScreenedProblem, walker.py:120-136, 322-418) ----
 * A screened problem is walked by delta tracking with the majorant
 * wos_walk_config.sigma_bar: each step exits to the sphere with probability
 * q / sinh q (q = sqrt(sigma_bar) d) or lands at a volume event drawn from the
 * screened Green's function, where the source deposits thr f'/sigma_bar and the
 * throughput thr picks up 1 - sigma'/sigma_bar (greens.py:100-193,
 * _kernels.py:476-558). The value is (acc + thr g'(exit)) / sqrt_alpha(start).
 * 3D ball or box domains. REPLAY_F64 follows the reference's Philox4x64 layout
 * (w0 event, w1/w2 direction, w3 radius; 64-step bisection of the radial CDF);
 * NATIVE_F32 uses one Philox4x32 block per step and Newton for the radial CDF.
 * WOS_SRC_SCREENED_CONST  [s', f', has_f' (0/1), sqrt_alpha], boundary WOS_BND_CONST [g']
 *                         = ScreenedProblem.const_coeffs (_kernels.walk_screened_ball3;
 *                         a walk whose throughput reaches 0 with has_f' = 0 stops, hit = 1)
 * WOS_SRC_SCREENED_VC     [phi, a_min, a_max], boundary WOS_BND_VC [phi]: the paper's
 *                         varying-coefficient family pde.VcInstance (pde.py:138-243):
 *                         sigma', f', g' = sqrt(alpha) u and sqrt(alpha) in closed form */

/* ---- boundary kinds (g evaluated at the projected exit point) -------- */
/* WOS_BND_CONST          [c]                                (_kernels.BND_CONST)
 * WOS_BND_FOURIER5       2D: [b0..b4], g = b0 + b1 c + b2 s + b3 (c^2-s^2) + b4 (2cs),
 *                        (c, s) = q/|q| ((1,0) at q = 0)   (_kernels.py:262-278)
 * WOS_BND_LINEAR         2D: [a, b, c] -> a x + b y + c;
 *                        3D: [a, b, c, d] -> a x + b y + c z + d (_kernels.py:270,439)
 * WOS_BND_FOURIER        2D: [M, b_0, b_1..b_M, c_1..c_M],
 *                        g = b_0 + sum_m b_m cos(m t) + c_m sin(m t), t = polar angle of q
 * WOS_BND_SQUARE_ARCSINE 2D: [x0, y0, side, M, c_1..c_M], s = counter-clockwise arc
 *                        length of q from corner (x0, y0) of the square
 *                        [x0, x0+side] x [y0, y0+side], g = sum_m c_m sin(2 pi m s / (4 side))
 * WOS_BND_QUADRATIC      2D: [axx, ayy, axy, ax, ay, a0],
 *                        g = axx x^2 + ayy y^2 + axy x y + ax x + ay y + a0
 * WOS_BND_VC             3D: [phi], g' = sqrt(alpha) u of the varying-coefficient
 *                        family (pde.py:197-199); only with WOS_SRC_SCREENED_VC    */
enum {
  WOS_BND_CONST = 0,
  WOS_BND_FOURIER5 = 1,
  WOS_BND_LINEAR = 2,
  WOS_BND_FOURIER = 3,
  WOS_BND_SQUARE_ARCSINE = 4,
  WOS_BND_QUADRATIC = 5,
  WOS_BND_VC = 6
};

/* One PDE instance: a walker.Problem (walker.py:102-116) reduced to its
 * (kind, params) specs (walker.py:160-171). Pointers are host pointers and are
 * only read during wos_problem_set_create.                                    */
typedef struct wos_problem {
  int32_t dim;       /* 2 or 3 */
  int32_t dom_kind;
  int32_t n_dom;
  const double* dom;
  int32_t src_kind;
  int32_t n_src;
  const double* src;
  int32_t bnd_kind;
  int32_t n_bnd;
  const double* bnd;
  uint64_t instance_key; /* Problem.instance_key: second Philox key word */
} wos_problem;

/* walker.WalkConfig (walker.py:55-79) after resolve_eps, plus the numeric mode. */
typedef struct wos_walk_config {
  double eps;          /* resolved eps_shell (> 0) */
  int64_t max_steps;   /* >= 1 */
  int32_t antithetic;  /* estimate only: mirrored pairs share a traj id */
  int32_t mode;        /* wos_mode */
  uint64_t rng_seed;   /* first Philox key word */
  double sigma_bar;    /* delta tracking majorant (WalkConfig.sigma_bar); ignored otherwise */
  int32_t philox_rounds; /* NATIVE_F32: Philox4x32 rounds per block, 10 (0 = default) or 7
                          * (opt-in, WalkConfig.philox_rounds); REPLAY modes ignore it */
  int32_t reserved;      /* 0 */
} wos_walk_config;

typedef struct wos_context wos_context;         /* per-device scratch + streams */
typedef struct wos_problem_set wos_problem_set; /* device-resident instance table */

/* ---- library / context ---------------------------------------------- */
int wos_abi_version(void);
const char* wos_last_error(void);
int wos_context_create(int32_t device, wos_context** out);
void wos_context_destroy(wos_context* ctx);

/* Upload n problems (same dim and kinds) as one device-resident table. */
int wos_problem_set_create(wos_context* ctx, const wos_problem* problems, int32_t n,
                           wos_problem_set** out);
void wos_problem_set_destroy(wos_problem_set* set);

/* ---- interior check (geometry.*.contains, estimator.py:156-159) --------
 * points: device [n, dim] fp64; inst_index: device [n] int32 or NULL (all 0).
 * Synchronous. *out_first_exterior = index of the first exterior point or -1. */
int wos_check_interior(wos_context* ctx, const wos_problem_set* set, int64_t n,
                       const double* points, const int32_t* inst_index,
                       int64_t* out_first_exterior, void* stream);

/* Same with host buffers (points [n, dim] fp64, inst_index [n] int32 or NULL). */
int wos_check_interior_host(wos_context* ctx, const wos_problem_set* set, int64_t n,
                            const double* points, const int32_t* inst_index,
                            int64_t* out_first_exterior);

/* ---- batch of independent trajectories (walker.walk_poisson_values) ----
 * Row i walks from points[i] under stream (point_ids[i], traj_ids[i], signs[i])
 * of problem 0 of the set. Device pointers, stream-ordered.
 * out_values: fp64 [n], out_steps: int64 [n], out_hits: uint8 [n]
 * (the (values, steps, hits) triple of _kernels.walk_plain_2d).            */
int wos_walk_rows(wos_context* ctx, const wos_problem_set* set, const wos_walk_config* cfg,
                  int64_t n, const double* points, const uint64_t* point_ids,
                  const uint64_t* traj_ids, const double* signs, double* out_values,
                  int64_t* out_steps, uint8_t* out_hits, void* stream);

/* Same with host buffers; synchronous. */
int wos_walk_rows_host(wos_context* ctx, const wos_problem_set* set,
                       const wos_walk_config* cfg, int64_t n, const double* points,
                       const uint64_t* point_ids, const uint64_t* traj_ids,
                       const double* signs, double* out_values, int64_t* out_steps,
                       uint8_t* out_hits);

/* ---- per-point ensemble estimate (estimator.estimate) ------------------
 * Point p (problem inst_index[p], or 0 if inst_index is NULL) runs L
 * trajectories with traj ids traj_start + j (antithetic: traj_start + 2*(j/2),
 * signs +1/-1, samples = pair means; estimator.py:119-141) and is reduced to
 * (mean, m2) with m2 = sum (v - mean)^2 over its n = L (or L/2) samples.
 * Device pointers: points [P, dim] fp64, point_ids [P] int64 or NULL (ids = 0..P-1,
 * estimator.py:165), inst_index [P] int32 or NULL, out_mean/out_m2 [P] fp64, out_total_steps: device uint64 accumulator
 * (added to, not overwritten) or NULL. Exterior start points and a watchdog trip
 * are flagged on the device without a sync; query them with wos_context_status().    */
int wos_estimate(wos_context* ctx, const wos_problem_set* set, const wos_walk_config* cfg,
                 int64_t n_points, const double* points, const int64_t* point_ids,
                 const int32_t* inst_index, int64_t L, uint64_t traj_start,
                 double* out_mean, double* out_m2, uint64_t* out_total_steps,
                 void* stream);

/* Same with host buffers (copies inside, synchronous; large calls are pipelined in
 * point chunks so host<->device copies overlap the walks). Returns WOS_ERR_EXTERIOR
 * (outputs undefined) if a start point is exterior; wos_context_exterior() then
 * reports its index. out_total_steps: host, may be NULL (overwritten, not added). */
int wos_estimate_host(wos_context* ctx, const wos_problem_set* set,
                      const wos_walk_config* cfg, int64_t n_points, const double* points,
                      const int64_t* point_ids, const int32_t* inst_index, int64_t L,
                      uint64_t traj_start, double* out_mean, double* out_m2,
                      uint64_t* out_total_steps);

/* Synchronizes `stream` and returns (then resets) the largest sigma' above sigma_bar
 * met by a delta-tracking volume event since the last call, or -1 if none. The
 * *_host entry points report it themselves as WOS_ERR_MAJORANT. */
int wos_context_majorant(wos_context* ctx, void* stream, double* out_worst_sigma_prime);

/* Synchronizes `stream` and returns the first exterior point index seen by
 * wos_estimate / wos_estimate_host since the last call (-1 if none), resetting it. */
int wos_context_exterior(wos_context* ctx, void* stream, int64_t* out_first_exterior);

/* Status of the last walking call on this context (device API error reporting).
 * Every walking entry point (wos_estimate, wos_walk_rows, wos_estimate_fold and the
 * *_host variants) clears the context's status block with one stream-ordered memset
 * before it walks, so the flags read here belong to that call; the device entry
 * points never synchronize on them. This synchronizes `stream`, returns and clears:
 *   *out_first_exterior     index of the first exterior start point, -1 if none
 *                           (estimator.py:156-159 raises ExteriorQueryError for it);
 *   *out_watchdog           non-zero if the walk kernel hit its iteration limit
 *                           (results of that call are invalid);
 *   *out_worst_sigma_prime  largest sigma' above sigma_bar met by a delta-tracking
 *                           volume event, -1 if none (walker.py:409-413).
 * Any output pointer may be NULL. The status is per context: calls interleaved on
 * several streams of one context share it. */
int wos_context_status(wos_context* ctx, void* stream, int64_t* out_first_exterior,
                       uint32_t* out_watchdog, double* out_worst_sigma_prime);

/* Measurement counters of this context (cumulative, never reset): *out_launches = the
 * kernels this library has launched on it (walk, interior check, chunk merge, cache
 * fold / targets); *out_seg_evals = segment distances evaluated by NATIVE polygon walks
 * (the measured work of a candidate-grid query; bench.py's cfg3 roofline). Synchronizes
 * `stream` first. Either pointer may be NULL. */
int wos_context_counters(wos_context* ctx, void* stream, uint64_t* out_launches,
                         uint64_t* out_seg_evals);

/* ---- epoch-averaged estimate cache (estimator.EstimateCache) -----------
 * replaces                                                      by
 *   EstimateCache.update / cache_update (estimator.py:217-244, 338-341)  wos_cache_fold
 *   EstimateCache.targets              (estimator.py:251-255)       wos_cache_targets
 *   training-label epoch: estimate(traj_start = epoch L) + cache_update
 *                                      (surrogate.py:288-298)       wos_estimate_fold
 * The cache is caller-owned device state over the frozen, sorted key set
 * (estimator.py:206-215): mean_sum, mean, m2 fp64 [n_keys], n int64 [n_keys].
 * Folding fresh estimate k into entry slot[k] (k itself if slot is NULL) does
 *   mean_sum += mean_k;  (n, mean, m2) <- chan_merge((n, mean, m2), (n_k, mean_k, m2_k))
 * in fp64 with the reference's operation order (estimator.py:41-53), so targets are
 * bit-identical to the reference cache fed the same estimates. n_k comes from
 * fresh_n [n_fresh] int64 (device) or, if fresh_n is NULL, fresh_n_all. Slots must
 * be distinct within one call. Device pointers, ordered on `stream`. */
int wos_cache_fold(wos_context* ctx, int64_t n_fresh, const int64_t* slot,
                   const double* fresh_mean, const double* fresh_m2, const int64_t* fresh_n,
                   int64_t fresh_n_all, double* mean_sum, int64_t* n, double* mean, double* m2,
                   void* stream);

/* out[k] = mean_sum[k] / epoch (epoch >= 1). */
int wos_cache_targets(wos_context* ctx, int64_t n_keys, const double* mean_sum, int64_t epoch,
                      double* out, void* stream);

/* One training-label epoch on the device: wos_estimate of the points (arguments as
 * there) folded straight into the cache entries slot[p] (NULL: p) with n = L (L/2
 * antithetic); the epoch's estimates never leave the device. */
int wos_estimate_fold(wos_context* ctx, const wos_problem_set* set, const wos_walk_config* cfg,
                      int64_t n_points, const double* points, const int64_t* point_ids,
                      const int32_t* inst_index, int64_t L, uint64_t traj_start,
                      const int64_t* slot, double* mean_sum, int64_t* n, double* mean,
                      double* m2, uint64_t* out_total_steps, void* stream);

/* ---- counter-based generators (known-answer tests) --------------------
 * Device pointers; ctr/out are [n, 4] words. */
int wos_philox4x64(wos_context* ctx, int64_t n, const uint64_t* ctr, uint64_t key0,
                   uint64_t key1, uint64_t* out, void* stream);
int wos_philox4x32(wos_context* ctx, int64_t n, const uint32_t* ctr, uint32_t key0,
                   uint32_t key1, uint32_t* out, void* stream);

/* Philox4x32-R for R in 1..16 (Random123 round function and key schedule): the KAT and
 * statistics hook of the NATIVE stream's opt-in 7-round variant (wos_walk_config
 * philox_rounds). Same arguments as wos_philox4x32 plus `rounds`. */
int wos_philox4x32_rounds(wos_context* ctx, int64_t n, const uint32_t* counters, uint32_t k0,
                          uint32_t k1, int32_t rounds, uint32_t* out, void* stream);

/* ---- launch tuning ---------------------------------------------------- */
/* refill_min: a warp refills idle lanes once at least this many are idle
 * (1..32, default 5). blocks_per_sm: persistent grid = SMs * blocks_per_sm (0 = auto). */
int wos_set_tuning(wos_context* ctx, int32_t refill_min, int32_t blocks_per_sm);
/* refill threshold of launches that defer recording finished walks to the refill
 * (non-constant boundary terms: recording pays once per refill, so larger batches
 * win; delta-tracking launches keep refill_min; 1..32, default 12). ABI version 3. */
int wos_set_refill_deferred(wos_context* ctx, int32_t refill_min);

/* ---- roofline probes ---------------------------------------------------
 * Measured on the device of ctx: MUFU (SFU) op/s and FP32 flop/s (FFMA = 2)
 * from dependent-chain-free microkernels timed with CUDA events, and the
 * effective SM clock implied by the FFMA rate (flop/s / (SMs * 256)).       */
int wos_probe_peaks(wos_context* ctx, double* out_sfu_ops_per_s, double* out_fp32_flops_per_s,
                    double* out_sm_clock_hz, int32_t* out_num_sms);

/* ---- fast-math error probe (ABI 3) -------------------------------------
 * The NATIVE kernels' fast-math primitives on device arrays x [n] fp32: __sincosf,
 * sqrt.approx(|x|), ex2.approx(x), so their error can be bounded against libm
 * (north-star: a fast-math path whose error is bounded against the reference).  */
int wos_fastmath_probe(wos_context* ctx, int64_t n, const float* x, float* out_sin, float* out_cos,
                       float* out_sqrt, float* out_ex2, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WOS_B200_H */
