// Shared host/device types of the WoS walker (launch arguments, instance headers).
#pragma once
#include <stdint.h>

namespace wos {

enum : int { DOM_BALL = 0, DOM_POLAR = 1, DOM_BOX = 2, DOM_POLY = 3, DOM_MESH = 4 };
// internal NATIVE kernel code (never a problem's domain): a cube centred at 1/2 walked in
// centred scaled coordinates X = pi (x - 1/2) (wos_walk.cuh Walker::kCentered)
enum : int { DOM_CUBE = 5 };
enum : int { SRC_NONE = 0, SRC_CONST = 1, SRC_RBF2 = 2, SRC_SINE = 3, SRC_GAUSS = 4 };
// delta-tracking (screened) walks: the "source" slot selects the transformed coefficients
enum : int { SRC_SCR_CONST = 5, SRC_SCR_VC = 6 };
enum : int {
  BND_CONST = 0,
  BND_FOURIER5 = 1,
  BND_LINEAR = 2,
  BND_FOURIER = 3,
  BND_SQUARE_ARCSINE = 4,
  BND_QUADRATIC = 5,
  BND_VC = 6  // varying-coefficient family: g' = sqrt(alpha) u_exact at the exit point
};
enum : int { MODE_REPLAY_F64 = 0, MODE_REPLAY_F32 = 1, MODE_NATIVE_F32 = 2 };
enum : int { SINK_ROWS = 0, SINK_ESTIMATE = 1 };

constexpr int kBlock = 256;       // threads per CTA (8 warps)
constexpr int kWarps = kBlock / 32;
// single-instance constant-boundary box kernels with a monomial sine source walk in
// X = pi x (wos_walk.cuh Walker::kScaled; the host scales box and eps to match)
#ifndef WOS_SCALED_COORDS
#define WOS_SCALED_COORDS 1
#endif
// cubes centred at 1/2 (BASELINE cfg0 / cfg4) walk in centred scaled coordinates
#ifndef WOS_CENTERED_CUBE
#define WOS_CENTERED_CUBE 1
#endif
// polygon candidate grids: 16-byte cell records with up to four pair indices inline
// (one dependent load fewer per query; wos_capi.cu build, wos_walk.cuh poly_grid_scan)
#ifndef WOS_GRID_INLINE
#define WOS_GRID_INLINE 1
#endif
#ifndef WOS_GRID_BYTES  // byte pair indices (12 inline) when a polygon has <= 256 pairs
#define WOS_GRID_BYTES 1
#endif
#ifndef WOS_RING
#define WOS_RING 512  // 1024 -> 512: cfg3 -2 %, cfg2 -3 % (more L1), others equal; 256 starves cfg4 (+17 %)
#endif
constexpr int kRing = WOS_RING;   // per-warp ring of walk values (estimate sink)
// Exit-ring kernels (wos_walk.cuh Walker::kExitRing) keep 8-byte ring slots; the host
// sizes their shared memory from the same predicate (wos_capi.cu pick_kernel).
#ifndef WOS_EXIT_RING
#define WOS_EXIT_RING 1
#endif
constexpr bool exit_ring_kernel(bool native, int dim, int dom, int src, bool one, bool est, bool bc) {
  return WOS_EXIT_RING && native && dim == 2 && (dom == DOM_BALL || dom == DOM_BOX) &&
         src == SRC_NONE && one && est && !bc;
}
constexpr int kSlots = 16;        // per-warp completion counters of live retire blocks
constexpr int kUQ = 16;           // per-warp queue of grabbed work units
#ifndef WOS_CHUNK
#define WOS_CHUNK 128
#endif
constexpr int kChunk = WOS_CHUNK; // L > kChunk: work units are kChunk-walk chunks of one point
constexpr int kUnitTarget = 128;  // L < 32: whole points per unit up to >= this many walks
constexpr int kCP = 256;          // floats of single-instance parameters held in the kernel params
constexpr int kDomOff = 0;        // table row: [0, 8) domain params
constexpr int kSrcOff = 16;       //            [16, 16 + ns) source params, then boundary params
// NATIVE box rows also hold the centre at [8, 11) and the half extent at [12, 15)

// Per-instance header (32 bytes), one per problem of a set.
struct InstHdr {
  uint64_t ikey;    // Problem.instance_key (REPLAY Philox4x64 key word 1)
  uint32_t nkey1;   // NATIVE key word 1 = (seed >> 32) ^ this (lo32(ikey) ^ hi32(ikey) * 0x9E3779B9)
  int32_t seg_off;  // polygon: first segment
  int32_t n_seg;    // polygon: segment count
  int32_t rec_off;  // polygon, NATIVE: first record of the n_seg + 1 vertex records
  int32_t pad[2];
};

// n / d for n < 2^31 with host-precomputed (mul, shr) (Granlund-Montgomery round-up)
__host__ __device__ inline uint32_t fast_div(uint32_t n, uint32_t mul, uint32_t shr) {
#ifdef __CUDA_ARCH__
  return (__umulhi(n, mul) + n) >> shr;
#else
  return (uint32_t)((((uint64_t)n * mul) >> 32) + n) >> shr;
#endif
}
inline void fast_div_init(uint32_t d, uint32_t* mul, uint32_t* shr) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  *shr = l;
  *mul = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
}

struct KArgs {
  // ---- problem set (device) ----
  const void* table;    // Real rows [n_inst][stride]
  const InstHdr* hdr;   // [n_inst]
  const void* segs;     // polygon segments / polar tables / mesh triangles (mode-specific layout)
  const void* nodes;    // mesh BVH nodes (MeshNode<Real>)
  int32_t n_inst;
  int32_t stride;       // Real elements per table row
  int32_t bnd_off;      // boundary params offset in a row
  int32_t stage_bytes;  // bytes of the table staged into shared memory (0 = read global)
  int32_t seg_stage_bytes;  // NATIVE polygon records staged after the table (0 = read global)
  int32_t sine_K;       // sine order (uniform over the set; padded)
  int32_t bnd_kind;
  int32_t bnd_M;        // Fourier / arc-length order (uniform over the set; padded)
  int32_t refill_min;   // refill idle lanes once this many are idle
  int32_t refill_min_deferred;  // ... in launches that defer recording finished walks
  float bnd_c;          // single-instance NATIVE launches: the BND_CONST boundary value
  // ---- walk config ----
  double eps;
  float eps_f;          // eps rounded to fp32 (NATIVE / REPLAY_F32 compare in fp32)
  int32_t max_steps;
  int32_t antithetic;
  uint64_t seed;        // REPLAY Philox4x64 key word 0
  uint32_t nkey0;       // NATIVE Philox4x32 key word 0 = lo32(seed)
  uint32_t nkey1_seed;  // hi32(seed), xored with InstHdr::nkey1
  int32_t sink;         // SINK_ROWS or SINK_ESTIMATE
  // ---- work decomposition ----
  uint32_t n_points;    // estimate: P; rows: n
  uint32_t L;           // estimate: walks per point; rows: 1
  uint32_t U;           // points per work unit
  uint32_t IU;          // items (walks) per work unit = U * L
  uint32_t n_units;
  uint32_t n_chunks;    // L > kChunk: chunks per point (ceil(L / kChunk)); else 0
  uint32_t nc_mul, nc_shr;  // magic numbers for n / n_chunks
  double* partials;     // L > kChunk: per-chunk (mean, m2), [P * n_chunks][2]
  uint32_t iu_mul, iu_shr;  // magic numbers: n / IU = (umulhi(n, mul) + n) >> shr, n < 2^31
  uint32_t l_mul, l_shr;    // same for n / L
  const double* points;        // [n, dim]
  const int64_t* point_ids;    // estimate; null = ids are id_base + index
  uint64_t id_base;
  const int32_t* inst_index;   // estimate, may be null
  uint64_t traj_start;
  const uint64_t* row_pid;     // rows
  const uint64_t* row_tid;
  const double* row_sign;
  // ---- outputs ----
  double* out_values;
  int64_t* out_steps;
  uint8_t* out_hits;
  double* out_mean;
  double* out_m2;
  unsigned long long* total_steps;
  unsigned int* work_counter;
  unsigned int* watchdog;      // set to 1 if a warp hit the iteration limit
  // ---- delta tracking (screened walks) ----
  double sigma_bar;            // absorption majorant (WalkConfig.sigma_bar)
  double sqrt_sig;             // sqrt(sigma_bar)
  unsigned long long* majorant;  // max violating sigma' seen (fp64 bits), 0 = none
  uint32_t iter_limit;         // max(2^27, 4 * max_steps) loop iterations per warp
  int32_t philox_rounds;       // NATIVE: Philox4x32 rounds per block (10, or 7 on request)
  unsigned long long* seg_evals;  // NATIVE polygons: segment distances evaluated (or null)
  const float* beta_tab;         // NATIVE 3D source jumps: Beta(2,2) table (wos_beta_table.h)
  int32_t beta_stage_bytes;      // its shared-memory bytes (0 when the kernel does not use it)
  // ---- single-instance NATIVE launches: the instance row and the Philox round
  // keys live in the kernel-parameter constant bank (FFMA / LOP3 c[] operands) ----
  uint32_t rk0[10];
  uint32_t rk1[10];
  alignas(16) float cp[kCP];
};

}  // namespace wos
