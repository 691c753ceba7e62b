// C ABI of libwos_b200.so (include/wos_b200.h): contexts, problem sets,
// launches of the persistent walk kernel, RNG known-answer kernels, interior
// check and the roofline probes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <mutex>
#include <thread>
#include "wos_beta_table.h"
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/wos_b200.h"
#include "wos_kernels.h"
#include "wos_rng.cuh"
#include "wos_types.h"
#include "wos_mesh.cuh"
#include <map>
#include <utility>

using namespace wos;

// ------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------
static thread_local char g_err[512] = "";

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(WOS_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),   \
                  __FILE__, __LINE__);                                                    \
  } while (0)

// ------------------------------------------------------------------------
// context and problem set
// ------------------------------------------------------------------------
constexpr int kCounterRing = 256;
constexpr size_t kStatusBytes = 32;
#ifndef WOS_CARVEOUT
#define WOS_CARVEOUT 1
#endif
#ifndef WOS_PIPE_CHUNKS
#define WOS_PIPE_CHUNKS 2  // cfg4 e2e/device: 1 chunk 95.0 %, 2 chunks 95.4 %, 3 93.4 %, 4 93.6 %, 8 89.5 %
// (three chunks with small first and last ones, -DWOS_PIPE_CHUNKS=3 -DWOS_PIPE_EDGE=8/16/32:
// 95.3 / 95.45 / 95.6 % against 95.35 % in the same call — within the noise, not adopted)
#endif
#ifndef WOS_PIPE_EDGE
#define WOS_PIPE_EDGE 0
#endif
constexpr int kPipeChunks = WOS_PIPE_CHUNKS;   // host pipeline: point chunks per call (at most)
constexpr int64_t kPipeMinWork = 1ll << 23;    // walks per chunk (at least)

struct wos_context {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;          // private stream of the *_host entry points
  cudaStream_t copy_stream = nullptr;     // host pipeline copies
  cudaStream_t stream2 = nullptr;         // host pipeline: odd chunks' walks (tails overlap)
  cudaEvent_t ev_copy[kPipeChunks] = {};
  cudaEvent_t ev_kernel[kPipeChunks] = {};
  cudaEvent_t ev_start = nullptr;
  unsigned int* d_counters = nullptr;     // work counters, one per launch slot
  std::atomic<unsigned> next_counter{0};
  // Device status block (one 32-byte allocation, reset by ONE stream-ordered memset at
  // the start of every walking entry point, so a flag always belongs to the call that
  // raised it; wos_context_status reads it): the first exterior point stored inverted
  // (atomicMax of ~index, 0 = none), the worst sigma' above sigma_bar (fp64 bits, 0 =
  // none), the kernel watchdog flag.
  unsigned long long* d_status = nullptr;
  unsigned long long* d_exterior = nullptr;  // = d_status + 0
  unsigned long long* d_majorant = nullptr;  // = d_status + 1
  unsigned int* d_watchdog = nullptr;        // = (unsigned*)(d_status + 2)
  unsigned long long* d_steps = nullptr;     // total-steps scratch of the *_host variants
  // measurement counters (wos_context_counters): kernels this library launched, and
  // the segment distances NATIVE polygon walks evaluated (the measured FP32 work of a
  // candidate-grid query)
  std::atomic<unsigned long long> n_launches{0};
  unsigned long long* d_perf = nullptr;
  float* d_beta_tab = nullptr;    // radius table of NATIVE 3D source jumps: Beta(2,2)
  float* d_green2_tab = nullptr;  // ... of NATIVE 2D source jumps: the disk Green's law
  // per-kernel launch attributes (dynamic shared memory set, occupancy at that size):
  // computed on the first launch of a (kernel, smem) pair instead of every launch
  std::unordered_map<const void*, std::pair<size_t, int>> launch_cache;
  std::mutex launch_mu;
  int64_t host_exterior = -1;
  void* d_scratch = nullptr;
  size_t scratch_bytes = 0;
  int refill_min = 5;  // measured optimum with the jump-first loop (4..6 within 1.5 %)
  int refill_min_deferred = 12;  // launches with deferred recording (8..16 within 3 % on cfg1-3)
  int blocks_per_sm = 0;
  std::mutex mu;  // serialises the *_host entry points' scratch
};

struct wos_problem_set {
  wos_context* ctx = nullptr;
  int n = 0, dim = 0, dom_kind = 0, src_kind = 0, bnd_kind = 0;
  int sine_K = 0;   // padded sine order of the tables
  int sine_K_native = 0, sk_native = 0;
  int bnd_M = 0;
  int stride = 0, bnd_off = 0;            // Real elements per row, boundary offset
  size_t bytes_d = 0, bytes_f = 0;        // padded table bytes
  double* d_table_d = nullptr;
  float* d_table_f = nullptr;             // REPLAY_F32 table (replay layout, float)
  float* d_table_n = nullptr;             // NATIVE table (native layout, float)
  InstHdr* d_hdr = nullptr;
  double* d_segs_d = nullptr;             // [nseg][ax, ay, ex, ey]
  float* d_segs_f = nullptr;              // REPLAY_F32: same, float
  float4* d_segs_n = nullptr;             // NATIVE: per polygon segment-pair records (poly_scan)
  size_t bytes_segs_n = 0;
  uint32_t* d_poly_grid = nullptr;        // NATIVE: polygon candidate grids (build_poly_grid)
  bool poly_grid = false;                 // some polygon of the set has a grid
  MeshNode<double>* d_mesh_nodes_d = nullptr;  // MESH: BVH nodes and leaf-ordered triangles
  MeshNode<float>* d_mesh_nodes_f = nullptr;
  double* d_mesh_tris_d = nullptr;
  float* d_mesh_tris_f = nullptr;
  double* d_mesh_fnorm = nullptr;         //       feature normals (21 per triangle), fp64
  double* d_polar_d = nullptr;            // POLAR: per instance n (bx, by) pairs, fp64
  float* d_polar_f = nullptr;             //        the same, fp32
  size_t bytes_polar_d = 0, bytes_polar_f = 0;
  std::vector<float> h_row_n;             // NATIVE row of problem 0 (single-instance launches)
  std::vector<float> h_row_n_scaled;      // ... with the box in X = pi x (scaled-coordinate kernels)
  std::vector<float> h_row_n_cube;        // ... a cube centred at 1/2 in X = pi (x - 1/2) (DOM_CUBE)
  bool cube = false;                      // problem 0's box is such a cube (and the source monomial)
  double scr_sprime_max = -1.0;           // SRC_SCR_CONST: largest s' of the set (majorant check)
  uint32_t h_nkey1 = 0;                   // its InstHdr::nkey1
};

int wos_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
int wos_context_device(const wos_context* c) { return c->device; }
void wos_context_count_launch(wos_context* c) { c->n_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" int wos_context_counters(wos_context* c, void* stream, uint64_t* out_launches,
                                    uint64_t* out_seg_evals) {
  if (!c) return fail(WOS_ERR_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  unsigned long long v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, c->d_perf, sizeof(v), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  if (out_launches) *out_launches = c->n_launches.load();
  if (out_seg_evals) *out_seg_evals = v;
  return WOS_OK;
}

extern "C" int wos_abi_version(void) { return WOS_ABI_VERSION; }
extern "C" const char* wos_last_error(void) { return g_err; }

extern "C" int wos_context_create(int32_t device, wos_context** out) {
  if (!out) return fail(WOS_ERR_INVALID, "null output pointer");
  int n = 0;
  CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(WOS_ERR_INVALID, "device %d out of range (%d)", device, n);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(WOS_ERR_UNSUPPORTED, "device %d is sm_%d%d; libwos_b200 is built for sm_100a",
                device, prop.major, prop.minor);
  // stream-ordered scratch (chunk partials) comes from the default pool: keep freed
  // memory cached so a per-call cudaMallocAsync never re-maps pages on the hot path
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  wos_context* c = new wos_context();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking);
  for (int i = 0; i < kPipeChunks && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&c->ev_copy[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_kernel[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_counters, sizeof(unsigned) * kCounterRing);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_status, kStatusBytes);
  if (e == cudaSuccess) e = cudaMemset(c->d_status, 0, kStatusBytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_steps, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_perf, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_beta_tab, sizeof(float) * WOS_BETA_TABLE_N);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_green2_tab, sizeof(float) * WOS_BETA_TABLE_N);
  if (e == cudaSuccess) {
    std::vector<float> bt(WOS_BETA_TABLE_N), gt(WOS_BETA_TABLE_N);
    wos_beta22_table(bt.data());
    wos_green2_table(gt.data());
    e = cudaMemcpy(c->d_beta_tab, bt.data(), sizeof(float) * WOS_BETA_TABLE_N, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(c->d_green2_tab, gt.data(), sizeof(float) * WOS_BETA_TABLE_N, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaMemset(c->d_perf, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) {
    c->d_exterior = c->d_status;
    c->d_majorant = c->d_status + 1;
    c->d_watchdog = reinterpret_cast<unsigned int*>(c->d_status + 2);
  }
  if (e != cudaSuccess) {
    delete c;
    return fail(WOS_ERR_CUDA, "context setup: %s", cudaGetErrorString(e));
  }
  *out = c;
  return WOS_OK;
}

extern "C" void wos_context_destroy(wos_context* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaFree(c->d_counters);
  cudaFree(c->d_status);
  cudaFree(c->d_steps);
  cudaFree(c->d_perf);
  cudaFree(c->d_beta_tab);
  cudaFree(c->d_green2_tab);
  cudaFree(c->d_scratch);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  for (int i = 0; i < kPipeChunks; ++i) {
    if (c->ev_copy[i]) cudaEventDestroy(c->ev_copy[i]);
    if (c->ev_kernel[i]) cudaEventDestroy(c->ev_kernel[i]);
  }
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  delete c;
}

extern "C" int wos_set_tuning(wos_context* c, int32_t refill_min, int32_t blocks_per_sm) {
  if (!c) return fail(WOS_ERR_INVALID, "null context");
  if (refill_min < 1 || refill_min > 32) return fail(WOS_ERR_INVALID, "refill_min must be 1..32");
  if (blocks_per_sm < 0 || blocks_per_sm > 32) return fail(WOS_ERR_INVALID, "blocks_per_sm must be 0..32");
  c->refill_min = refill_min;
  c->blocks_per_sm = blocks_per_sm;
  return WOS_OK;
}

extern "C" int wos_set_refill_deferred(wos_context* c, int32_t refill_min) {
  if (!c) return fail(WOS_ERR_INVALID, "null context");
  if (refill_min < 1 || refill_min > 32) return fail(WOS_ERR_INVALID, "refill_min must be 1..32");
  c->refill_min_deferred = refill_min;
  return WOS_OK;
}

static int need(int got, int want, const char* what) {
  if (got != want) return fail(WOS_ERR_INVALID, "%s expects %d parameters, got %d", what, want, got);
  return WOS_OK;
}

static int validate(const wos_problem& p) {
  if (p.dim != 2 && p.dim != 3) return fail(WOS_ERR_INVALID, "dim must be 2 or 3");
  int r;
  switch (p.dom_kind) {
    case WOS_DOM_BALL:
      if ((r = need(p.n_dom, p.dim + 1, "ball domain"))) return r;
      if (!(p.dom[p.dim] > 0.0)) return fail(WOS_ERR_INVALID, "ball radius must be positive");
      break;
    case WOS_DOM_BOX:
      if ((r = need(p.n_dom, 2 * p.dim, "box domain"))) return r;
      for (int i = 0; i < p.dim; ++i)
        if (!(p.dom[p.dim + i] > p.dom[i])) return fail(WOS_ERR_INVALID, "box must have positive extent");
      break;
    case WOS_DOM_POLYGON: {
      if (p.dim != 2) return fail(WOS_ERR_INVALID, "polygon domains are 2D");
      if (p.n_dom < 7) return fail(WOS_ERR_INVALID, "polygon needs >= 3 vertices");
      int nv = (int)p.dom[0];
      if (nv < 3 || p.n_dom != 1 + 2 * nv) return fail(WOS_ERR_INVALID, "polygon parameter count mismatch");
      break;
    }
    case WOS_DOM_MESH: {
      if (p.dim != 3) return fail(WOS_ERR_INVALID, "mesh domains are 3D");
      if (p.n_dom < 2) return fail(WOS_ERR_INVALID, "mesh needs [nv, nf, vertices, faces]");
      const int64_t nv = (int64_t)p.dom[0], nf = (int64_t)p.dom[1];
      if (nv < 4 || nf < 4) return fail(WOS_ERR_INVALID, "mesh needs >= 4 vertices and faces");
      if (p.n_dom != 2 + 3 * nv + 3 * nf) return fail(WOS_ERR_INVALID, "mesh parameter count mismatch");
      for (int64_t k = 0; k < 3 * nf; ++k) {
        const double f = p.dom[2 + 3 * nv + k];
        if (!(f >= 0.0 && f < (double)nv) || f != floor(f))
          return fail(WOS_ERR_INVALID, "face index out of range");
      }
      break;
    }
    case WOS_DOM_POLAR: {
      if (p.dim != 2) return fail(WOS_ERR_INVALID, "polar domains are 2D");
      if (p.n_dom != 3 && p.n_dom < 5) return fail(WOS_ERR_INVALID, "polar domain needs [r0, c1, c2(, stride, n, table)]");
      if (!(p.dom[0] > 0.0)) return fail(WOS_ERR_INVALID, "r0 must be positive");
      if (!(fabs(p.dom[1]) + fabs(p.dom[2]) < 1.0))
        return fail(WOS_ERR_INVALID, "|c1| + |c2| must be < 1 for a valid boundary");
      if (p.n_dom > 3) {
        const int st = (int)p.dom[3], nt = (int)p.dom[4];
        if (nt < 8 || nt > (1 << 16) || st < 1 || st > nt)
          return fail(WOS_ERR_INVALID, "polar table size / stride out of range");
        if (p.n_dom != 5 + 2 * nt) return fail(WOS_ERR_INVALID, "polar table parameter count mismatch");
      }
      break;
    }
    default:
      return fail(WOS_ERR_UNSUPPORTED, "unknown domain kind %d", p.dom_kind);
  }
  switch (p.src_kind) {
    case WOS_SRC_NONE:
      break;
    case WOS_SRC_CONST:
      if ((r = need(p.n_src, 1, "constant source"))) return r;
      break;
    case WOS_SRC_RBF2:
      if (p.dim != 2) return fail(WOS_ERR_UNSUPPORTED, "RBF2 source is 2D only");
      if ((r = need(p.n_src, 6, "RBF2 source"))) return r;
      break;
    case WOS_SRC_SINE: {
      if (p.n_src < 2) return fail(WOS_ERR_INVALID, "sine source needs [K, coeffs...]");
      int K = (int)p.src[0];
      if (K < 1 || K > 16) return fail(WOS_ERR_UNSUPPORTED, "sine order K must be 1..16");
      int nc = p.dim == 2 ? K * K : K * K * K;
      if ((r = need(p.n_src, 1 + nc, "sine source"))) return r;
      break;
    }
    case WOS_SRC_GAUSS:
      if ((r = need(p.n_src, 2 + p.dim, "Gaussian source"))) return r;
      if (!(p.src[1] > 0.0)) return fail(WOS_ERR_INVALID, "Gaussian sigma must be positive");
      break;
    case WOS_SRC_SCREENED_CONST:
      if (p.dim != 3) return fail(WOS_ERR_UNSUPPORTED, "delta tracking is 3D only (walker.py:322-418)");
      if ((r = need(p.n_src, 4, "screened constant coefficients"))) return r;
      if (p.bnd_kind != WOS_BND_CONST)
        return fail(WOS_ERR_INVALID, "screened constant coefficients take a constant boundary g'");
      if (!(p.src[3] > 0.0)) return fail(WOS_ERR_INVALID, "sqrt(alpha) must be positive");
      break;
    case WOS_SRC_SCREENED_VC:
      if (p.dim != 3) return fail(WOS_ERR_UNSUPPORTED, "delta tracking is 3D only (walker.py:322-418)");
      if ((r = need(p.n_src, 3, "varying-coefficient family"))) return r;
      if (p.bnd_kind != WOS_BND_VC)
        return fail(WOS_ERR_INVALID, "the varying-coefficient family takes the WOS_BND_VC boundary");
      break;
    default:
      return fail(WOS_ERR_UNSUPPORTED, "unknown source kind %d", p.src_kind);
  }
  if (p.dom_kind == WOS_DOM_POLYGON &&
      (p.src_kind == WOS_SRC_SCREENED_CONST || p.src_kind == WOS_SRC_SCREENED_VC))
    return fail(WOS_ERR_UNSUPPORTED, "delta tracking needs a 3D ball or box");
  switch (p.bnd_kind) {
    case WOS_BND_CONST:
      if ((r = need(p.n_bnd, 1, "constant boundary"))) return r;
      break;
    case WOS_BND_LINEAR:
      if ((r = need(p.n_bnd, p.dim + 1, "linear boundary"))) return r;
      break;
    case WOS_BND_FOURIER5:
      if (p.dim != 2) return fail(WOS_ERR_UNSUPPORTED, "FOURIER5 boundary is 2D only");
      if ((r = need(p.n_bnd, 5, "FOURIER5 boundary"))) return r;
      break;
    case WOS_BND_FOURIER: {
      if (p.dim != 2) return fail(WOS_ERR_UNSUPPORTED, "Fourier boundary is 2D only");
      if (p.n_bnd < 2) return fail(WOS_ERR_INVALID, "Fourier boundary needs [M, b0, ...]");
      int M = (int)p.bnd[0];
      if (M < 0 || M > 64) return fail(WOS_ERR_UNSUPPORTED, "Fourier order must be 0..64");
      if ((r = need(p.n_bnd, 2 + 2 * M, "Fourier boundary"))) return r;
      break;
    }
    case WOS_BND_SQUARE_ARCSINE: {
      if (p.dim != 2) return fail(WOS_ERR_UNSUPPORTED, "arc-length boundary is 2D only");
      if (p.n_bnd < 4) return fail(WOS_ERR_INVALID, "arc-length boundary needs [x0, y0, side, M, ...]");
      int M = (int)p.bnd[3];
      if (M < 0 || M > 64) return fail(WOS_ERR_UNSUPPORTED, "arc-length order must be 0..64");
      if ((r = need(p.n_bnd, 4 + M, "arc-length boundary"))) return r;
      break;
    }
    case WOS_BND_QUADRATIC:
      if (p.dim != 2) return fail(WOS_ERR_UNSUPPORTED, "quadratic boundary is 2D only");
      if ((r = need(p.n_bnd, 6, "quadratic boundary"))) return r;
      break;
    case WOS_BND_VC:
      if (p.src_kind != WOS_SRC_SCREENED_VC)
        return fail(WOS_ERR_INVALID, "WOS_BND_VC belongs to the varying-coefficient family");
      if ((r = need(p.n_bnd, 1, "varying-coefficient boundary"))) return r;
      if (p.bnd[0] != p.src[0])
        return fail(WOS_ERR_INVALID, "boundary and coefficients must share phi");
      break;
    default:
      return fail(WOS_ERR_UNSUPPORTED, "unknown boundary kind %d", p.bnd_kind);
  }
  return WOS_OK;
}

// ---- closed triangle meshes (geometry.MeshDomain, geometry.py:400-580) ----
// Feature normals as in MeshDomain._build_normals (geometry.py:434-468): unit face
// normals, angle-weighted vertex normals, edge normals from the two adjacent faces;
// a median-split BVH (largest box extent, leaves of <= 8 triangles, geometry.py:326-358)
// laid out depth first with the left child next to its parent.
// ---------------------------------------------------------------------------
// NATIVE polygon candidate grid. The polygon's bounding box is cut into G x G cells;
// each cell lists (ascending) the segment pairs that can hold the nearest segment of
// some point in the cell: pair j is listed when one of its segments comes within
// U + margin of the cell, U = min over segments of the largest corner distance (an
// upper bound of the boundary distance anywhere in the cell, the distance to a
// segment being convex). Unlisted segments are farther than the nearest one by more
// than the fp32 rounding of the query, so the listed minimum (and its first segment)
// is the full scan's. Walks spend most steps near the boundary, where lists are short.
// ---------------------------------------------------------------------------
static float bits_f32(int v) {
  float f;
  memcpy(&f, &v, sizeof(f));
  return f;
}

struct PolyGrid {
  int G = 0;
  double lo[2] = {0, 0}, ih[2] = {0, 0};
  std::vector<uint32_t> cells;  // G*G + 1 offsets into idx
  std::vector<uint16_t> idx;    // pair indices
};

static double seg_dist(double px, double py, double ax, double ay, double bx, double by) {
  const double ex = bx - ax, ey = by - ay, wx = px - ax, wy = py - ay;
  const double l2 = ex * ex + ey * ey;
  double t = l2 > 0 ? (wx * ex + wy * ey) / l2 : 0.0;
  t = t < 0 ? 0 : (t > 1 ? 1 : t);
  const double dx = wx - t * ex, dy = wy - t * ey;
  return sqrt(dx * dx + dy * dy);
}

// distance between segment ab and the box [x0, x1] x [y0, y1]
static double seg_box_dist(double ax, double ay, double bx, double by, double x0, double y0, double x1,
                           double y1) {
  // Liang-Barsky: does the segment meet the box?
  double t0 = 0.0, t1 = 1.0;
  const double dx = bx - ax, dy = by - ay;
  const double pp[4] = {-dx, dx, -dy, dy}, qq[4] = {ax - x0, x1 - ax, ay - y0, y1 - ay};
  bool hit = true;
  for (int k = 0; k < 4 && hit; ++k) {
    if (pp[k] == 0.0) {
      if (qq[k] < 0.0) hit = false;
    } else {
      const double r = qq[k] / pp[k];
      if (pp[k] < 0.0) t0 = std::max(t0, r);
      else t1 = std::min(t1, r);
      if (t0 > t1) hit = false;
    }
  }
  if (hit) return 0.0;
  auto pbox = [&](double px, double py) {
    const double ux = px < x0 ? x0 - px : (px > x1 ? px - x1 : 0.0);
    const double uy = py < y0 ? y0 - py : (py > y1 ? py - y1 : 0.0);
    return sqrt(ux * ux + uy * uy);
  };
  double d = std::min(pbox(ax, ay), pbox(bx, by));
  const double cx[4] = {x0, x1, x0, x1}, cy[4] = {y0, y0, y1, y1};
  for (int k = 0; k < 4; ++k) d = std::min(d, seg_dist(cx[k], cy[k], ax, ay, bx, by));
  return d;
}

// V: nv vertices; segments 0..np-1 with np = nv rounded up to even (the pad is the
// zero-length segment at vertex 0). The lists are refined down a quadtree: a child
// cell's candidates are a subset of its parent's (its U is no larger, its box
// distances no smaller), so each level only tests the parent's list.
static int np_pairs(int nv) { return (nv + 1) / 2; }  // segment pairs of an nv-gon

static void build_poly_grid(const double* V, int nv, PolyGrid* g) {
  const int np = nv + (nv & 1);
  g->G = 0;
  if (nv < 24) return;  // short polygons: the full scan is as cheap
#ifndef WOS_POLY_GRID_SCALE
#define WOS_POLY_GRID_SCALE 11.4
#endif
#ifndef WOS_POLY_GRID_MAX
#define WOS_POLY_GRID_MAX 128
#endif
  const double want = WOS_POLY_GRID_SCALE * sqrt((double)nv);
  int levels = 2;
  while ((1 << levels) < want && (1 << levels) < WOS_POLY_GRID_MAX) ++levels;
  const int G = 1 << levels;
  double lo[2] = {V[0], V[1]}, hi[2] = {V[0], V[1]};
  for (int k = 1; k < nv; ++k)
    for (int c = 0; c < 2; ++c) {
      lo[c] = std::min(lo[c], V[2 * k + c]);
      hi[c] = std::max(hi[c], V[2 * k + c]);
    }
  const double diag = hypot(hi[0] - lo[0], hi[1] - lo[1]);
  const double margin = 1e-5 * diag;
  for (int c = 0; c < 2; ++c) {
    const double pad = 1e-9 * diag;
    lo[c] -= pad;
    hi[c] += pad;
    g->lo[c] = lo[c];
    g->ih[c] = G / (hi[c] - lo[c]);
  }
  std::vector<double> SA(2 * np), SB(2 * np);
  for (int s = 0; s < np; ++s) {
    const int i = s < nv ? s : 0, j = s < nv ? (s + 1 == nv ? 0 : s + 1) : 0;
    SA[2 * s] = V[2 * i];
    SA[2 * s + 1] = V[2 * i + 1];
    SB[2 * s] = V[2 * j];
    SB[2 * s + 1] = V[2 * j + 1];
  }
  auto sd = [&](double px, double py, int s) {
    return seg_dist(px, py, SA[2 * s], SA[2 * s + 1], SB[2 * s], SB[2 * s + 1]);
  };
  // level l: (1 << l)^2 cells, row-major; cell c's candidate segments (ascending) are
  // data[off[c] .. off[c + 1])
  std::vector<uint32_t> off = {0u, (uint32_t)np}, noff;
  std::vector<int> data(np), ndata;
  for (int s = 0; s < np; ++s) data[s] = s;
  std::vector<double> dc;
  for (int l = 1; l <= levels; ++l) {
    const int n = 1 << l, pn = n >> 1;
    const double hx = (hi[0] - lo[0]) / n, hy = (hi[1] - lo[1]) / n;
    const double r = 0.5 * sqrt(hx * hx + hy * hy);
    noff.assign((size_t)n * n + 1, 0u);
    ndata.clear();
    for (int cy = 0; cy < n; ++cy)
      for (int cx = 0; cx < n; ++cx) {
        const size_t pc = (size_t)(cy >> 1) * pn + (cx >> 1);
        const int* C = data.data() + off[pc];
        const int nc = (int)(off[pc + 1] - off[pc]);
        const double x0 = lo[0] + cx * hx, y0 = lo[1] + cy * hy, x1 = x0 + hx, y1 = y0 + hy;
        const double qx[4] = {x0, x1, x0, x1}, qy[4] = {y0, y0, y1, y1};
        const double mx = 0.5 * (x0 + x1), my = 0.5 * (y0 + y1);
        double U = 1e300;
        dc.resize(nc);
        for (int k = 0; k < nc; ++k) {
          dc[k] = sd(mx, my, C[k]);
          if (dc[k] >= U) continue;  // convexity: its farthest corner cannot beat U
          double m = 0.0;
          for (int q = 0; q < 4; ++q) m = std::max(m, sd(qx[q], qy[q], C[k]));
          U = std::min(U, m);
        }
        for (int k = 0; k < nc; ++k) {
          if (dc[k] - r > U + margin) continue;  // box distance >= centre distance - r
          const int sg = C[k];
          if (seg_box_dist(SA[2 * sg], SA[2 * sg + 1], SB[2 * sg], SB[2 * sg + 1], x0, y0, x1, y1) <= U + margin)
            ndata.push_back(sg);
        }
        noff[(size_t)cy * n + cx + 1] = (uint32_t)ndata.size();
      }
    off.swap(noff);
    data.swap(ndata);
  }
  g->G = G;
  g->cells.assign((size_t)G * G + 1, 0);
  g->idx.clear();
  for (size_t c = 0; c < (size_t)G * G; ++c) {
    g->cells[c] = (uint32_t)g->idx.size();
    int last = -1;
    for (uint32_t k = off[c]; k < off[c + 1]; ++k) {
      const int sg = data[k];
      const int j = sg >> 1;
      if (j != last) g->idx.push_back((uint16_t)j);
      last = j;
    }
  }
  g->cells[(size_t)G * G] = (uint32_t)g->idx.size();
}

struct MeshBuild {
  std::vector<MeshNode<double>> nodes;
  std::vector<double> tris;   // leaf order, 9 per triangle
  std::vector<double> fnorm;  // leaf order, 21 per triangle
};

static int build_mesh(const wos_problem& p, MeshBuild* out) {
  const int64_t nv = (int64_t)p.dom[0], nf = (int64_t)p.dom[1];
  const double* V = p.dom + 2;
  const double* F = p.dom + 2 + 3 * nv;
  auto vtx = [&](int64_t i, int c) { return V[3 * i + c]; };
  std::vector<double> fn(3 * nf), vn(3 * nv, 0.0);
  std::map<std::pair<int64_t, int64_t>, std::array<double, 3>> en;
  for (int64_t t = 0; t < nf; ++t) {
    const int64_t id[3] = {(int64_t)F[3 * t], (int64_t)F[3 * t + 1], (int64_t)F[3 * t + 2]};
    double e1[3], e2[3], n[3];
    for (int c = 0; c < 3; ++c) {
      e1[c] = vtx(id[1], c) - vtx(id[0], c);
      e2[c] = vtx(id[2], c) - vtx(id[0], c);
    }
    n[0] = e1[1] * e2[2] - e1[2] * e2[1];
    n[1] = e1[2] * e2[0] - e1[0] * e2[2];
    n[2] = e1[0] * e2[1] - e1[1] * e2[0];
    const double len = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    if (len == 0.0) return fail(WOS_ERR_INVALID, "degenerate triangle in mesh");
    for (int c = 0; c < 3; ++c) fn[3 * t + c] = n[c] / len;
    for (int l = 0; l < 3; ++l) {
      double a1[3], a2[3];
      for (int c = 0; c < 3; ++c) {
        a1[c] = vtx(id[(l + 1) % 3], c) - vtx(id[l], c);
        a2[c] = vtx(id[(l + 2) % 3], c) - vtx(id[l], c);
      }
      const double dt = a1[0] * a2[0] + a1[1] * a2[1] + a1[2] * a2[2];
      const double ln = sqrt(a1[0] * a1[0] + a1[1] * a1[1] + a1[2] * a1[2]) *
                        sqrt(a2[0] * a2[0] + a2[1] * a2[1] + a2[2] * a2[2]);
      const double ang = acos(std::min(1.0, std::max(-1.0, dt / ln)));
      for (int c = 0; c < 3; ++c) vn[3 * id[l] + c] += ang * fn[3 * t + c];
    }
    for (int l = 0; l < 3; ++l) {
      int64_t u = id[l], w = id[(l + 1) % 3];
      auto key = u < w ? std::make_pair(u, w) : std::make_pair(w, u);
      auto it = en.find(key);
      if (it == en.end()) it = en.emplace(key, std::array<double, 3>{0.0, 0.0, 0.0}).first;
      for (int c = 0; c < 3; ++c) it->second[c] += fn[3 * t + c];
    }
  }
  auto unit = [](double* v) {
    const double l = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    const double d = l == 0.0 ? 1.0 : l;
    for (int c = 0; c < 3; ++c) v[c] /= d;
  };
  for (int64_t i = 0; i < nv; ++i) unit(&vn[3 * i]);
  for (auto& kv : en) unit(kv.second.data());
  // BVH over triangle boxes
  std::vector<double> lo(3 * nf), hi(3 * nf), cen(3 * nf);
  for (int64_t t = 0; t < nf; ++t)
    for (int c = 0; c < 3; ++c) {
      double mn = 1e300, mx = -1e300;
      for (int l = 0; l < 3; ++l) {
        const double v = vtx((int64_t)F[3 * t + l], c);
        mn = std::min(mn, v);
        mx = std::max(mx, v);
      }
      lo[3 * t + c] = mn;
      hi[3 * t + c] = mx;
      cen[3 * t + c] = 0.5 * (mn + mx);
    }
  std::vector<int64_t> order(nf);
  for (int64_t t = 0; t < nf; ++t) order[t] = t;
  out->nodes.clear();
  std::vector<int64_t> leaf_order;
  leaf_order.reserve(nf);
  // iterative DFS build: (start, stop, parent slot to patch with the right child)
  struct Job { int64_t start, stop; int64_t patch; };
  std::vector<Job> todo{{0, nf, -1}};
  while (!todo.empty()) {
    Job j = todo.back();
    todo.pop_back();
    const int idx = (int)out->nodes.size();
    if (j.patch >= 0) out->nodes[j.patch].right = idx;
    MeshNode<double> nd;
    for (int c = 0; c < 3; ++c) {
      nd.lo[c] = 1e300;
      nd.hi[c] = -1e300;
    }
    for (int64_t k = j.start; k < j.stop; ++k)
      for (int c = 0; c < 3; ++c) {
        nd.lo[c] = std::min(nd.lo[c], lo[3 * order[k] + c]);
        nd.hi[c] = std::max(nd.hi[c], hi[3 * order[k] + c]);
      }
    nd.right = -1;
    nd.first = 0;
    nd.count = 0;
    nd.pad = 0;
    if (j.stop - j.start <= 8) {
      nd.first = (int32_t)leaf_order.size();
      nd.count = (int32_t)(j.stop - j.start);
      for (int64_t k = j.start; k < j.stop; ++k) leaf_order.push_back(order[k]);
      out->nodes.push_back(nd);
      continue;
    }
    int axis = 0;
    for (int c = 1; c < 3; ++c)
      if (nd.hi[c] - nd.lo[c] > nd.hi[axis] - nd.lo[axis]) axis = c;
    const int64_t mid = j.start + (j.stop - j.start) / 2;
    std::nth_element(order.begin() + j.start, order.begin() + mid, order.begin() + j.stop,
                     [&](int64_t x, int64_t y) {
                       return cen[3 * x + axis] < cen[3 * y + axis] ||
                              (cen[3 * x + axis] == cen[3 * y + axis] && x < y);
                     });
    out->nodes.push_back(nd);
    // right subtree is built after the left one (it sits after it in DFS order)
    todo.push_back({mid, j.stop, (int64_t)idx});
    todo.push_back({j.start, mid, -1});
  }
  out->tris.resize(9 * (size_t)nf);
  out->fnorm.resize(21 * (size_t)nf);
  for (int64_t k = 0; k < nf; ++k) {
    const int64_t t = leaf_order[k];
    const int64_t id[3] = {(int64_t)F[3 * t], (int64_t)F[3 * t + 1], (int64_t)F[3 * t + 2]};
    for (int l = 0; l < 3; ++l)
      for (int c = 0; c < 3; ++c) out->tris[9 * k + 3 * l + c] = vtx(id[l], c);
    double* N = &out->fnorm[21 * k];
    for (int c = 0; c < 3; ++c) N[c] = fn[3 * t + c];
    for (int l = 0; l < 3; ++l)
      for (int c = 0; c < 3; ++c) N[3 + 3 * l + c] = vn[3 * id[l] + c];
    for (int l = 0; l < 3; ++l) {  // edges ab, bc, ca
      int64_t u = id[l], w = id[(l + 1) % 3];
      auto key = u < w ? std::make_pair(u, w) : std::make_pair(w, u);
      const auto& e = en[key];
      for (int c = 0; c < 3; ++c) N[12 + 3 * l + c] = e[c];
    }
  }
  return WOS_OK;
}

static int sine_native_order(int dim, int K, int* sk) {
  // specialised kernels exist for 2D K in {4, 8} and 3D K = 3; smaller K pads up
  if (dim == 2 && K <= 4) { *sk = 4; return 4; }
  if (dim == 2 && K <= 8) { *sk = 8; return 8; }
  if (dim == 3 && K <= 3) { *sk = 3; return 3; }
  *sk = 0;
  return K;
}

static size_t pad16(size_t b) { return (b + 15) & ~(size_t)15; }

// Monomial form of a sine series for the NATIVE K <= 4 kernels (wos_walk.cuh sine_eval):
// sin(k pi y) = s U_{k-1}(c), U Chebyshev polynomials of the second kind, so
// sum a_{i..} prod_d sin((i_d + 1) pi y_d) = prod_d s_d * sum b_{p..} prod_d c_d^{p_d}
// with b = a contracted with T[i][p] (monomial coefficients of U_i) along every axis.
static void sine_monomial(const double* a, int K, int dim, double* b) {
  double T[4][4] = {{1, 0, 0, 0}, {0, 2, 0, 0}, {-1, 0, 4, 0}, {0, -4, 0, 8}};
  if (dim == 2) {
    for (int p = 0; p < K; ++p)
      for (int q = 0; q < K; ++q) {
        double v = 0.0;
        for (int i = 0; i < K; ++i)
          for (int j = 0; j < K; ++j) v += a[i * K + j] * T[i][p] * T[j][q];
        b[p * K + q] = v;
      }
  } else {
    for (int p = 0; p < K; ++p)
      for (int q = 0; q < K; ++q)
        for (int r = 0; r < K; ++r) {
          double v = 0.0;
          for (int i = 0; i < K; ++i)
            for (int j = 0; j < K; ++j)
              for (int k = 0; k < K; ++k) v += a[(i * K + j) * K + k] * T[i][p] * T[j][q] * T[k][r];
          b[(p * K + q) * K + r] = v;
        }
  }
}

extern "C" int wos_problem_set_create(wos_context* ctx, const wos_problem* probs, int32_t n,
                                      wos_problem_set** out) {
  if (!ctx || !probs || !out) return fail(WOS_ERR_INVALID, "null argument");
  if (n < 1) return fail(WOS_ERR_INVALID, "need at least one problem");
  for (int i = 0; i < n; ++i) {
    int r = validate(probs[i]);
    if (r) return r;
    if (probs[i].dim != probs[0].dim || probs[i].dom_kind != probs[0].dom_kind ||
        probs[i].src_kind != probs[0].src_kind || probs[i].bnd_kind != probs[0].bnd_kind)
      return fail(WOS_ERR_INVALID, "a problem set needs one dimension and one domain/source/boundary kind");
  }
  const int dim = probs[0].dim;
  wos_problem_set* s = new wos_problem_set();
  s->ctx = ctx;
  s->n = n;
  s->dim = dim;
  s->dom_kind = probs[0].dom_kind;
  s->src_kind = probs[0].src_kind;
  s->bnd_kind = probs[0].bnd_kind;
  // uniform orders over the set (zero padding is exact)
  int K = 0, M = 0;
  for (int i = 0; i < n; ++i) {
    if (s->src_kind == WOS_SRC_SINE) K = std::max(K, (int)probs[i].src[0]);
    if (s->bnd_kind == WOS_BND_FOURIER) M = std::max(M, (int)probs[i].bnd[0]);
    if (s->bnd_kind == WOS_BND_SQUARE_ARCSINE) M = std::max(M, (int)probs[i].bnd[3]);
  }
  int sk = 0;
  int Kn = (s->src_kind == WOS_SRC_SINE) ? sine_native_order(dim, K, &sk) : 0;
  const int Kt = std::max(K, Kn);  // table order (native may pad higher)
  s->sine_K = K;
  s->sine_K_native = Kn;
  s->sk_native = sk;
  s->bnd_M = M;
  int ns = 0;
  switch (s->src_kind) {
    case WOS_SRC_CONST: ns = 1; break;
    case WOS_SRC_RBF2: ns = 6; break;
    case WOS_SRC_SINE: ns = dim == 2 ? Kt * Kt : Kt * Kt * Kt; break;
    case WOS_SRC_GAUSS: ns = 2 + dim; break;
    case WOS_SRC_SCREENED_CONST: ns = 4; break;
    case WOS_SRC_SCREENED_VC: ns = 6; break;
    default: ns = 0;
  }
  int nb = 0;
  // NATIVE series run to an order bucket (wos_walk.cuh order_bucket): the rows hold
  // zero coefficients up to it
  const int Mb = M <= 4 ? 4 : (M <= 8 ? 8 : M);
  switch (s->bnd_kind) {
    case WOS_BND_CONST: nb = 1; break;
    case WOS_BND_LINEAR: nb = dim + 1; break;
    case WOS_BND_FOURIER5: nb = 5; break;
    case WOS_BND_FOURIER: nb = 2 + 2 * Mb; break;
    case WOS_BND_SQUARE_ARCSINE: nb = 4 + Mb; break;
    case WOS_BND_QUADRATIC: nb = 6; break;
    case WOS_BND_VC: nb = 4; break;
  }
  s->bnd_off = kSrcOff + ns;
  s->stride = (kSrcOff + ns + nb + 3) & ~3;
  const int stride = s->stride;
  std::vector<double> td((size_t)n * stride, 0.0);   // replay layout
  std::vector<float> tn((size_t)n * stride, 0.0f);   // native layout
  std::vector<InstHdr> hd(n);
  std::vector<double> segd;
  std::vector<float4> segn;
  std::vector<uint32_t> pcells;  // NATIVE polygon candidate grids: cell offsets, pair lists
  std::vector<uint16_t> pidx;
  struct GridFix {
    size_t rec, cells, idx;
  };
  std::vector<GridFix> grid_fix;
  std::vector<PolyGrid> grids;  // NATIVE polygon candidate grids, built in parallel
  if (s->dom_kind == WOS_DOM_POLYGON) {
    grids.resize(n);
    const int nt = std::max(1, std::min(n, std::min(16, (int)std::thread::hardware_concurrency())));
    std::atomic<int> next{0};
    auto work = [&]() {
      for (int i = next++; i < n; i = next++) build_poly_grid(probs[i].dom + 1, (int)probs[i].dom[0], &grids[i]);
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
  }
  std::vector<double> polard;  // POLAR tables, (bx, by) pairs
  std::vector<MeshNode<double>> mnodes;  // MESH: all instances' BVHs, triangles, normals
  std::vector<double> mtris, mfnorm;
  for (int i = 0; i < n; ++i) {
    const wos_problem& p = probs[i];
    double* rd = td.data() + (size_t)i * stride;
    float* rn = tn.data() + (size_t)i * stride;
    memset(&hd[i], 0, sizeof(InstHdr));
    hd[i].ikey = p.instance_key;
    hd[i].nkey1 = (uint32_t)p.instance_key ^ ((uint32_t)(p.instance_key >> 32) * 0x9E3779B9u);
    // domain
    if (p.dom_kind == WOS_DOM_BALL) {
      for (int k = 0; k < dim; ++k) rd[k] = p.dom[k];
      rd[3] = p.dom[dim];
    } else if (p.dom_kind == WOS_DOM_MESH) {
      MeshBuild mb;
      const int r = build_mesh(p, &mb);
      if (r) {
        delete s;
        return r;
      }
      hd[i].seg_off = (int)mnodes.size();
      hd[i].n_seg = (int)mb.nodes.size();
      hd[i].rec_off = (int)(mtris.size() / 9);
      mnodes.insert(mnodes.end(), mb.nodes.begin(), mb.nodes.end());
      mtris.insert(mtris.end(), mb.tris.begin(), mb.tris.end());
      mfnorm.insert(mfnorm.end(), mb.fnorm.begin(), mb.fnorm.end());
    } else if (p.dom_kind == WOS_DOM_POLAR) {
      // geometry.py:97-112: the curve tabulated at n angles, strided scan for mild curves
      const double r0 = p.dom[0], c1 = p.dom[1], c2 = p.dom[2];
      rd[0] = r0;
      rd[1] = c1;
      rd[2] = c2;
      int nt = 4096, st = (fabs(c1) + fabs(c2) <= 0.45) ? 64 : 1;
      if (p.n_dom > 3) {
        st = (int)p.dom[3];
        nt = (int)p.dom[4];
      }
      hd[i].seg_off = (int)(polard.size() / 2);
      hd[i].n_seg = nt;
      hd[i].rec_off = st;
      for (int k = 0; k < nt; ++k) {
        if (p.n_dom > 3) {
          polard.push_back(p.dom[5 + k]);
          polard.push_back(p.dom[5 + nt + k]);
        } else {
          const double th = (double)k * (2.0 * M_PI / nt);
          const double r = r0 * (1.0 + c1 * cos(4.0 * th) + c2 * cos(8.0 * th));
          polard.push_back(r * cos(th));
          polard.push_back(r * sin(th));
        }
      }
    } else if (p.dom_kind == WOS_DOM_BOX) {
      for (int k = 0; k < dim; ++k) {
        rd[k] = p.dom[k];
        rd[4 + k] = p.dom[dim + k];
      }
    } else {
      const int nv = (int)p.dom[0];
      const double* V = p.dom + 1;
      hd[i].seg_off = (int)(segd.size() / 4);
      hd[i].n_seg = nv;
      std::vector<float> vx, vy, ux, uy;
      for (int k = 0; k < nv; ++k) {
        const int j = (k + 1 == nv) ? 0 : k + 1;
        const double ax = V[2 * k], ay = V[2 * k + 1];
        const double ex = V[2 * j] - ax, ey = V[2 * j + 1] - ay;
        segd.push_back(ax);
        segd.push_back(ay);
        segd.push_back(ex);
        segd.push_back(ey);
        const double l2 = ex * ex + ey * ey;
        vx.push_back((float)ax);
        vy.push_back((float)ay);
        ux.push_back((float)(ex / l2));
        uy.push_back((float)(ey / l2));
      }
      // NATIVE records in segment pairs (wos_walk.cuh poly_scan): two header records
      // (the candidate grid's box and offsets), then A_j = (x_2j, x_2j+1, y_2j, y_2j+1),
      // U_j = (u_2j, u_2j+1 by component), then a closing A at vertex 0. An odd
      // polygon gets a zero-length segment at vertex 0 (u = 0) as its pad.
      const PolyGrid& g = grids[i];
      segn.push_back(make_float4((float)g.lo[0], (float)g.lo[1], (float)g.ih[0], (float)g.ih[1]));
      grid_fix.push_back({segn.size(), pcells.size(), pidx.size()});
      segn.push_back(make_float4(bits_f32(g.G), 0.f, 0.f, 0.f));  // offsets patched below
#if WOS_GRID_INLINE
      // one 16-byte record per cell. Byte format (every pair index < 256, counts and the
      // overflow list < 65536): {count | overflow offset << 16, pairs 0-11 as bytes};
      // else the uint16 format {overflow offset, count, pairs 0-1, pairs 2-3}. The rest
      // of a cell's pairs go to the polygon's overflow list (bytes packed two per
      // uint16 slot in the byte format). Header record 1's w says which (1 = bytes).
      bool bytes8 = WOS_GRID_BYTES && g.G > 0 && (np_pairs(nv) <= 256);
      if (g.G > 0) {
        size_t over = 0;
        uint32_t maxn = 0;
        for (size_t c = 0; c + 1 < g.cells.size(); ++c) {
          const uint32_t n = g.cells[c + 1] - g.cells[c];
          maxn = std::max(maxn, n);
          over += n > 12 ? n - 12 : 0;
        }
        bytes8 = bytes8 && maxn < 65536 && over < 65536;
        const size_t pbase = pidx.size();
        std::vector<uint8_t> ov8;
        for (size_t c = 0; c + 1 < g.cells.size(); ++c) {
          const uint32_t b = g.cells[c], e = g.cells[c + 1], n = e - b;
          if (bytes8) {
            uint32_t w[3] = {0, 0, 0};
            for (uint32_t k = 0; k < n && k < 12; ++k) w[k >> 2] |= (uint32_t)g.idx[b + k] << (8 * (k & 3));
            pcells.push_back(n | ((uint32_t)ov8.size() << 16));
            pcells.push_back(w[0]);
            pcells.push_back(w[1]);
            pcells.push_back(w[2]);
            for (uint32_t k = 12; k < n; ++k) ov8.push_back((uint8_t)g.idx[b + k]);
          } else {
            uint32_t in[4] = {0, 0, 0, 0};
            for (uint32_t k = 0; k < n && k < 4; ++k) in[k] = g.idx[b + k];
            pcells.push_back((uint32_t)(pidx.size() - pbase));
            pcells.push_back(n);
            pcells.push_back(in[0] | (in[1] << 16));
            pcells.push_back(in[2] | (in[3] << 16));
            for (uint32_t k = 4; k < n; ++k) pidx.push_back(g.idx[b + k]);
          }
        }
        if (bytes8)
          for (size_t k = 0; k < ov8.size(); k += 2)
            pidx.push_back((uint16_t)(ov8[k] | ((k + 1 < ov8.size() ? ov8[k + 1] : 0) << 8)));
      }
      segn.back().w = bits_f32(bytes8 ? 1 : 0);
#else
      pcells.insert(pcells.end(), g.cells.begin(), g.cells.end());
      pidx.insert(pidx.end(), g.idx.begin(), g.idx.end());
#endif
      hd[i].rec_off = (int)segn.size();
      if (nv & 1) {
        vx.push_back((float)V[0]);
        vy.push_back((float)V[1]);
        ux.push_back(0.f);
        uy.push_back(0.f);
      }
      for (size_t k = 0; k < vx.size(); k += 2) {
        segn.push_back(make_float4(vx[k], vx[k + 1], vy[k], vy[k + 1]));
        segn.push_back(make_float4(ux[k], ux[k + 1], uy[k], uy[k + 1]));
      }
      segn.push_back(make_float4((float)V[0], 0.f, (float)V[1], 0.f));  // closing vertex
    }
    for (int k = 0; k < 8; ++k) rn[k] = (float)rd[k];
    if (p.dom_kind == WOS_DOM_BOX)  // NATIVE box distance: centre and half extent
      for (int k = 0; k < dim; ++k) {
        rn[8 + k] = (float)(0.5 * (p.dom[k] + p.dom[dim + k]));
        rn[12 + k] = (float)(0.5 * (p.dom[dim + k] - p.dom[k]));
      }
    // source
    double* sd = rd + kSrcOff;
    float* sn = rn + kSrcOff;
    switch (p.src_kind) {
      case WOS_SRC_CONST:
        sd[0] = p.src[0];
        break;
      case WOS_SRC_RBF2:
        for (int k = 0; k < 6; ++k) sd[k] = p.src[k];
        break;
      case WOS_SRC_SINE: {
        const int Ki = (int)p.src[0];
        const double* a = p.src + 1;
        std::vector<double> an((size_t)(dim == 2 ? Kn * Kn : Kn * Kn * Kn), 0.0);
        if (dim == 2) {
          for (int k = 0; k < Ki; ++k)
            for (int l = 0; l < Ki; ++l) {
              sd[k * K + l] = a[k * Ki + l];   // replay: order K
              an[k * Kn + l] = a[k * Ki + l];  // native: order Kn (zero-padded)
            }
        } else {
          for (int k = 0; k < Ki; ++k)
            for (int l = 0; l < Ki; ++l)
              for (int m = 0; m < Ki; ++m) {
                sd[(k * K + l) * K + m] = a[(k * Ki + l) * Ki + m];
                an[(k * Kn + l) * Kn + m] = a[(k * Ki + l) * Ki + m];
              }
        }
        if (sk == 3 || sk == 4) {  // monomial-Horner kernels
          std::vector<double> bm(an.size());
          sine_monomial(an.data(), Kn, dim, bm.data());
          for (size_t k = 0; k < bm.size(); ++k) sn[k] = (float)bm[k];
        } else {
          for (size_t k = 0; k < an.size(); ++k) sn[k] = (float)an[k];
        }
        break;
      }
      case WOS_SRC_GAUSS:
        for (int k = 0; k < 2 + dim; ++k) sd[k] = p.src[k];
        break;
      case WOS_SRC_SCREENED_CONST:
        for (int k = 0; k < 4; ++k) sd[k] = p.src[k];
        s->scr_sprime_max = std::max(s->scr_sprime_max, p.src[0]);
        break;
      case WOS_SRC_SCREENED_VC: {
        // pde.py:141-142,157: a = 4 pi phi, b = 3 pi phi, p = pi phi (Python's left-to-right products)
        const double phi = p.src[0];
        sd[0] = phi;
        sd[1] = p.src[1];
        sd[2] = p.src[2];
        sd[3] = (4.0 * M_PI) * phi;
        sd[4] = (3.0 * M_PI) * phi;
        sd[5] = M_PI * phi;
        break;
      }
    }
    if (p.src_kind != WOS_SRC_SINE)
      for (int k = 0; k < ns; ++k) sn[k] = (float)sd[k];
    if (p.src_kind == WOS_SRC_GAUSS) sn[1] = (float)(1.4426950408889634 / (2.0 * p.src[1] * p.src[1]));
    // boundary (orders padded to the set maximum)
    double* bd = rd + s->bnd_off;
    switch (p.bnd_kind) {
      case WOS_BND_FOURIER: {
        const int Mi = (int)p.bnd[0];
        bd[0] = M;
        bd[1] = p.bnd[1];
        for (int m = 1; m <= Mi; ++m) {
          bd[1 + m] = p.bnd[1 + m];
          bd[1 + M + m] = p.bnd[1 + Mi + m];
        }
        break;
      }
      case WOS_BND_SQUARE_ARCSINE: {
        const int Mi = (int)p.bnd[3];
        bd[0] = p.bnd[0];
        bd[1] = p.bnd[1];
        bd[2] = p.bnd[2];
        bd[3] = M;
        for (int m = 1; m <= Mi; ++m) bd[3 + m] = p.bnd[3 + m];
        break;
      }
      case WOS_BND_VC: {
        const double phi = p.bnd[0];
        bd[0] = phi;
        bd[1] = (4.0 * M_PI) * phi;
        bd[2] = (3.0 * M_PI) * phi;
        bd[3] = M_PI * phi;
        break;
      }
      default:
        for (int k = 0; k < p.n_bnd; ++k) bd[k] = p.bnd[k];
    }
    if (p.bnd_kind == WOS_BND_FOURIER) {
      // NATIVE row: [M, B1, b1, c1, b2, c2, ...] (pairs interleaved: offsets independent of M)
      const int Mi = (int)p.bnd[0];
      rn[s->bnd_off] = (float)Mb;
      rn[s->bnd_off + 1] = (float)p.bnd[1];
      for (int m = 1; m <= Mi; ++m) {
        rn[s->bnd_off + 2 * m] = (float)p.bnd[1 + m];
        rn[s->bnd_off + 2 * m + 1] = (float)p.bnd[1 + Mi + m];
      }
    } else {
      for (int k = 0; k < nb; ++k) rn[s->bnd_off + k] = (float)bd[k];
    }
  }
  s->h_row_n.assign(tn.begin(), tn.begin() + stride);
  s->h_row_n_scaled = s->h_row_n;
  if (s->dom_kind == WOS_DOM_BOX) {  // centre and half extent times pi, from the fp64 row
    for (int k = 0; k < s->dim; ++k) {
      s->h_row_n_scaled[8 + k] = (float)(M_PI * 0.5 * (td[k] + td[4 + k]));
      s->h_row_n_scaled[12 + k] = (float)(M_PI * 0.5 * (td[4 + k] - td[k]));
    }
    // the scaled-coordinate kernels (monomial sine sources) take the Green weight
    // 1 / (2 dim) pi^-2 folded into the source coefficients (wos_walk.cuh advance_native)
    if (s->src_kind == WOS_SRC_SINE && (s->sk_native == 3 || s->sk_native == 4)) {
      const double w = 1.0 / (2.0 * s->dim * M_PI * M_PI);
      for (int k = 0; k < ns; ++k)
        s->h_row_n_scaled[kSrcOff + k] = (float)((double)s->h_row_n[kSrcOff + k] * w);
      // a cube centred at 1/2: the centred scaled row (centre 0; the monomial coefficient
      // of c_0^p c_1^q (c_2^r) times (-1)^(p+q(+r)), since cos(pi x) = -sin X)
      bool cube = true;
      for (int k = 0; k < s->dim; ++k)
        cube = cube && td[k] + td[4 + k] == 1.0 && td[4 + k] - td[k] == td[4] - td[0];
      if (cube) {
        s->cube = true;
        s->h_row_n_cube = s->h_row_n_scaled;
        const int K = s->sk_native;
        for (int k = 0; k < s->dim; ++k) s->h_row_n_cube[8 + k] = 0.0f;
        for (int k = 0; k < ns; ++k) {
          const int deg = s->dim == 2 ? k / K + k % K : k / (K * K) + (k / K) % K + k % K;
          if (deg & 1) s->h_row_n_cube[kSrcOff + k] = -s->h_row_n_cube[kSrcOff + k];
        }
      }
    }
  }
  s->h_nkey1 = hd[0].nkey1;
  std::vector<float> tf(td.size());
  for (size_t k = 0; k < td.size(); ++k) tf[k] = (float)td[k];
  std::vector<float> segf(segd.size());
  for (size_t k = 0; k < segd.size(); ++k) segf[k] = (float)segd[k];

  s->bytes_d = pad16(td.size() * sizeof(double));
  s->bytes_f = pad16(tn.size() * sizeof(float));
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_table_d, s->bytes_d);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_table_f, s->bytes_f);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_table_n, s->bytes_f);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_hdr, sizeof(InstHdr) * n);
  if (e == cudaSuccess) e = cudaMemset(s->d_table_d, 0, s->bytes_d);
  if (e == cudaSuccess) e = cudaMemset(s->d_table_f, 0, s->bytes_f);
  if (e == cudaSuccess) e = cudaMemset(s->d_table_n, 0, s->bytes_f);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_table_d, td.data(), td.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_table_f, tf.data(), tf.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_table_n, tn.data(), tn.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_hdr, hd.data(), sizeof(InstHdr) * n, cudaMemcpyHostToDevice);
  if (!mnodes.empty()) {
    std::vector<MeshNode<float>> nf(mnodes.size());
    for (size_t k = 0; k < mnodes.size(); ++k) {
      for (int c = 0; c < 3; ++c) {
        // round the boxes outward so fp32 pruning never drops a closer triangle
        nf[k].lo[c] = nextafterf((float)mnodes[k].lo[c], -INFINITY);
        nf[k].hi[c] = nextafterf((float)mnodes[k].hi[c], INFINITY);
      }
      nf[k].right = mnodes[k].right;
      nf[k].first = mnodes[k].first;
      nf[k].count = mnodes[k].count;
      nf[k].pad = 0;
    }
    std::vector<float> tf(mtris.size());
    for (size_t k = 0; k < mtris.size(); ++k) tf[k] = (float)mtris[k];
    if (e == cudaSuccess) e = cudaMalloc(&s->d_mesh_nodes_d, mnodes.size() * sizeof(MeshNode<double>));
    if (e == cudaSuccess) e = cudaMalloc(&s->d_mesh_nodes_f, nf.size() * sizeof(MeshNode<float>));
    if (e == cudaSuccess) e = cudaMalloc(&s->d_mesh_tris_d, mtris.size() * 8);
    if (e == cudaSuccess) e = cudaMalloc(&s->d_mesh_tris_f, tf.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc(&s->d_mesh_fnorm, mfnorm.size() * 8);
    if (e == cudaSuccess)
      e = cudaMemcpy(s->d_mesh_nodes_d, mnodes.data(), mnodes.size() * sizeof(MeshNode<double>), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(s->d_mesh_nodes_f, nf.data(), nf.size() * sizeof(MeshNode<float>), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s->d_mesh_tris_d, mtris.data(), mtris.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s->d_mesh_tris_f, tf.data(), tf.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s->d_mesh_fnorm, mfnorm.data(), mfnorm.size() * 8, cudaMemcpyHostToDevice);
  }
  if (!polard.empty()) {
    std::vector<float> polarf(polard.size());
    for (size_t k = 0; k < polard.size(); ++k) polarf[k] = (float)polard[k];
    s->bytes_polar_d = polard.size() * 8;
    s->bytes_polar_f = polarf.size() * 4;
    if (e == cudaSuccess) e = cudaMalloc(&s->d_polar_d, s->bytes_polar_d);
    if (e == cudaSuccess) e = cudaMalloc(&s->d_polar_f, s->bytes_polar_f);
    if (e == cudaSuccess) e = cudaMemcpy(s->d_polar_d, polard.data(), s->bytes_polar_d, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s->d_polar_f, polarf.data(), s->bytes_polar_f, cudaMemcpyHostToDevice);
  }
  if (!segd.empty()) {
    // candidate grids: one buffer of 32-bit words, the cell offsets (rebased to the
    // polygon's list) then the uint16 pair lists; header record 1 = (G, cells, idx16)
    const size_t nw = pcells.size() + (pidx.size() + 1) / 2;
    std::vector<uint32_t> gbuf(std::max<size_t>(nw, 1), 0u);
    for (const PolyGrid& g : grids) s->poly_grid = s->poly_grid || g.G > 0;
    for (const GridFix& f : grid_fix) {
      float4& h1 = segn[f.rec];
      h1.y = bits_f32((int)f.cells);
      h1.z = bits_f32((int)(2 * pcells.size() + f.idx));
    }
    std::copy(pcells.begin(), pcells.end(), gbuf.begin());
    if (!pidx.empty()) memcpy(gbuf.data() + pcells.size(), pidx.data(), pidx.size() * 2);
    if (e == cudaSuccess) e = cudaMalloc(&s->d_poly_grid, gbuf.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(s->d_poly_grid, gbuf.data(), gbuf.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&s->d_segs_d, segd.size() * 8);
    if (e == cudaSuccess) e = cudaMalloc(&s->d_segs_f, segf.size() * 4);
    s->bytes_segs_n = segn.size() * sizeof(float4);
    if (e == cudaSuccess) e = cudaMalloc(&s->d_segs_n, segn.size() * sizeof(float4));
    if (e == cudaSuccess) e = cudaMemcpy(s->d_segs_d, segd.data(), segd.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(s->d_segs_f, segf.data(), segf.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(s->d_segs_n, segn.data(), segn.size() * sizeof(float4), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    wos_problem_set_destroy(s);
    return fail(WOS_ERR_CUDA, "problem set upload: %s", cudaGetErrorString(e));
  }
  *out = s;
  return WOS_OK;
}

extern "C" void wos_problem_set_destroy(wos_problem_set* s) {
  if (!s) return;
  cudaSetDevice(s->ctx->device);
  cudaFree(s->d_table_d);
  cudaFree(s->d_table_f);
  cudaFree(s->d_table_n);
  cudaFree(s->d_hdr);
  cudaFree(s->d_segs_d);
  cudaFree(s->d_segs_f);
  cudaFree(s->d_segs_n);
  cudaFree(s->d_poly_grid);
  cudaFree(s->d_polar_d);
  cudaFree(s->d_polar_f);
  cudaFree(s->d_mesh_nodes_d);
  cudaFree(s->d_mesh_nodes_f);
  cudaFree(s->d_mesh_tris_d);
  cudaFree(s->d_mesh_tris_f);
  cudaFree(s->d_mesh_fnorm);
  delete s;
}

// ------------------------------------------------------------------------
// interior check (geometry.*.contains; oracle_contains in oracle/wos_oracle.c)
// ------------------------------------------------------------------------
__global__ void wos_interior_kernel(int64_t n, const double* __restrict__ pts,
                                    const int32_t* __restrict__ inst, const double* __restrict__ table,
                                    int stride, const InstHdr* __restrict__ hdr,
                                    const double* __restrict__ segs, int dim, int dom_kind,
                                    unsigned long long* first, int64_t idx_base,
                                    const MeshNode<double>* __restrict__ mnodes,
                                    const double* __restrict__ mtris,
                                    const double* __restrict__ mfnorm) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int i = inst ? inst[p] : 0;
    const double* row = table + (size_t)i * stride;
    const double* x = pts + (size_t)p * dim;
    bool inside = true;
    if (dom_kind == WOS_DOM_BALL) {
      double s = 0.0;
      for (int k = 0; k < dim; ++k) s += (x[k] - row[k]) * (x[k] - row[k]);
      inside = sqrt(s) < row[3];
    } else if (dom_kind == WOS_DOM_BOX) {
      for (int k = 0; k < dim; ++k) inside = inside && (x[k] > row[k]) && (x[k] < row[4 + k]);
    } else if (dom_kind == WOS_DOM_MESH) {
      // MeshDomain.contains (geometry.py:510-525): the closest feature's pseudo-normal
      const InstHdr h = hdr[i];
      double q[3];
      int reg, tri;
      mesh_nearest<double>(mnodes + h.seg_off, mtris + 9 * (size_t)h.rec_off, x, q, &reg, &tri);
      const double* N = mfnorm + 21 * ((size_t)h.rec_off + tri);
      const double* nn = reg == MREG_FACE ? N : (reg <= MREG_C ? N + 3 + 3 * reg : N + 12 + 3 * (reg - MREG_AB));
      const double dot = (x[0] - q[0]) * nn[0] + (x[1] - q[1]) * nn[1] + (x[2] - q[2]) * nn[2];
      inside = dot < 0.0;
    } else if (dom_kind == WOS_DOM_POLAR) {
      // PolarDomain.contains (geometry.py:129-134): rho < r(atan2(y, x))
      const double th = atan2(x[1], x[0]);
      inside = hypot(x[0], x[1]) < row[0] * (1.0 + row[1] * cos(4.0 * th) + row[2] * cos(8.0 * th));
    } else {
      const InstHdr h = hdr[i];
      const double* S = segs + 4 * (size_t)h.seg_off;
      bool in = false;
      for (int k = 0; k < h.n_seg; ++k) {
        const double ax = S[4 * k], ay = S[4 * k + 1];
        const double bx = ax + S[4 * k + 2], by = ay + S[4 * k + 3];
        if ((ay > x[1]) != (by > x[1])) {
          const double xc = ax + (x[1] - ay) * (bx - ax) / (by - ay);
          if (x[0] < xc) in = !in;
        }
      }
      inside = in;
    }
    if (!inside) atomicMax(first, ~(unsigned long long)(idx_base + p));  // 0 = none
  }
}

static int launch_interior(wos_context* c, const wos_problem_set* s, int64_t n, const double* pts,
                           const int32_t* inst, cudaStream_t st, int64_t idx_base = 0) {
  if (n <= 0) return WOS_OK;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->num_sms * 8);
  wos_interior_kernel<<<blocks, 256, 0, st>>>(n, pts, inst, s->d_table_d, s->stride, s->d_hdr,
                                              s->d_segs_d, s->dim, s->dom_kind, c->d_exterior, idx_base,
                                              s->d_mesh_nodes_d, s->d_mesh_tris_d, s->d_mesh_fnorm);
  CUDA_TRY(cudaGetLastError());
  wos_context_count_launch(c);
  return WOS_OK;
}

static int check_watchdog(wos_context* c, cudaStream_t st) {
  unsigned int w = 0;
  CUDA_TRY(cudaMemcpyAsync(&w, c->d_watchdog, sizeof(w), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (w) {
    cudaMemsetAsync(c->d_watchdog, 0, sizeof(w), st);
    return fail(WOS_ERR_CUDA, w == 2u ? "walk kernel refused a boundary-parameter offset it was not built for"
                                      : "walk kernel watchdog tripped (iteration limit): results invalid");
  }
  return WOS_OK;
}

// delta tracking: report (and reset) a volume event whose sigma' exceeded sigma_bar
// (walker.py:409-413); the stream must already be synchronized
static int check_majorant(wos_context* c, const wos_walk_config* cfg, cudaStream_t st) {
  unsigned long long v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, c->d_majorant, sizeof(v), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (v) {
    CUDA_TRY(cudaMemsetAsync(c->d_majorant, 0, sizeof(v), st));
    double w;
    memcpy(&w, &v, sizeof(w));
    return fail(WOS_ERR_MAJORANT, "majorant violated: sigma'=%.17g > sigma_bar=%.17g", w,
                cfg->sigma_bar);
  }
  return WOS_OK;
}

extern "C" int wos_context_majorant(wos_context* c, void* stream, double* out) {
  if (!c || !out) return fail(WOS_ERR_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, c->d_majorant, sizeof(v), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemsetAsync(c->d_majorant, 0, sizeof(v), st));
  CUDA_TRY(cudaStreamSynchronize(st));
  double w = -1.0;
  if (v) memcpy(&w, &v, sizeof(w));
  *out = w;
  return WOS_OK;
}

static int read_exterior(wos_context* c, cudaStream_t st, int64_t* out) {
  unsigned long long v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, c->d_exterior, sizeof(v), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemsetAsync(c->d_exterior, 0, sizeof(v), st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *out = v ? (int64_t)~v : -1;
  return check_watchdog(c, st);
}

// one stream-ordered memset clears every status flag before a call walks
static int reset_status(wos_context* c, cudaStream_t st) {
  CUDA_TRY(cudaMemsetAsync(c->d_status, 0, kStatusBytes, st));
  return WOS_OK;
}

extern "C" int wos_context_status(wos_context* c, void* stream, int64_t* out_first_exterior,
                                  uint32_t* out_watchdog, double* out_worst_sigma_prime) {
  if (!c) return fail(WOS_ERR_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long h[kStatusBytes / 8];
  CUDA_TRY(cudaMemcpyAsync(h, c->d_status, kStatusBytes, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemsetAsync(c->d_status, 0, kStatusBytes, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  int64_t ext = h[0] ? (int64_t)~h[0] : -1;
  if (ext < 0) ext = c->host_exterior;
  c->host_exterior = -1;
  double w = -1.0;
  if (h[1]) memcpy(&w, &h[1], sizeof(w));
  if (out_first_exterior) *out_first_exterior = ext;
  if (out_watchdog) *out_watchdog = (uint32_t)(h[2] & 0xffffffffu);
  if (out_worst_sigma_prime) *out_worst_sigma_prime = w;
  return WOS_OK;
}

extern "C" int wos_check_interior(wos_context* c, const wos_problem_set* s, int64_t n,
                                  const double* points, const int32_t* inst_index,
                                  int64_t* out_first, void* stream) {
  if (!c || !s || !out_first) return fail(WOS_ERR_INVALID, "null argument");
  if (n < 0) return fail(WOS_ERR_INVALID, "negative point count");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int r = launch_interior(c, s, n, points, inst_index, st);
  if (r) return r;
  return read_exterior(c, st, out_first);
}

extern "C" int wos_context_exterior(wos_context* c, void* stream, int64_t* out) {
  if (!c || !out) return fail(WOS_ERR_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  int64_t v;
  int r = read_exterior(c, (cudaStream_t)stream, &v);
  if (r) return r;
  if (v < 0) v = c->host_exterior;
  c->host_exterior = -1;
  *out = v;
  return WOS_OK;
}

// ------------------------------------------------------------------------
// walk launches
// ------------------------------------------------------------------------
struct KernelInfo {
  const void* fn;
  size_t elem;  // sizeof(Real)
  bool one;     // single-instance NATIVE launch (parameters in the constant bank)
  bool cube;    // ... walking a cube centred at 1/2 in centred scaled coordinates (DOM_CUBE)
  int warps;    // warps per CTA the kernel is built for
};

static KernelInfo pick_kernel(const wos_problem_set* s, int mode, bool rows, int rounds, bool anti) {
  KernelInfo k{nullptr, 8, false, false, kWarps};
  const int dom = s->dom_kind == WOS_DOM_POLYGON ? DOM_POLY : s->dom_kind;
  if (mode == WOS_MODE_REPLAY_F64) {
    k.fn = get_kernel_replay_f64(s->dim, dom, s->src_kind, 0, rows);
    k.elem = 8;
  } else if (mode == WOS_MODE_REPLAY_F32) {
    k.fn = get_kernel_replay_f32(s->dim, dom, s->src_kind, 0, rows);
    k.elem = 4;
  } else {
    const int sk = s->src_kind == WOS_SRC_SINE ? s->sk_native : 0;
    k.one = (s->n == 1 && s->stride <= kCP);
    k.cube = WOS_CENTERED_CUBE && WOS_SCALED_COORDS && k.one && !rows && s->cube &&
             s->bnd_kind == WOS_BND_CONST && !anti;
    k.fn = get_kernel_native(s->dim, k.cube ? DOM_CUBE : dom, s->src_kind, sk, k.one, rows,
                             s->bnd_kind == WOS_BND_CONST, rounds, &k.warps);
    k.elem = 4;
    // exit-ring kernels keep (x, y) in 8-byte ring slots (wos_types.h exit_ring_kernel)
    if (exit_ring_kernel(true, s->dim, dom, s->src_kind, k.one, !rows, s->bnd_kind == WOS_BND_CONST)) k.elem = 8;
  }
  return k;
}

#ifndef WOS_SEG_STAGE_MAX
#define WOS_SEG_STAGE_MAX (96 * 1024)
#endif
static const size_t kSegStageMax = WOS_SEG_STAGE_MAX;  // polygon records staged per CTA at most

static size_t smem_bytes(size_t stage, size_t elem, int warps) {
  return stage + (size_t)warps * (kRing * elem + kSlots * 4 + kUQ * 4);
}

static int launch_walk(wos_context* c, const wos_problem_set* s, const wos_walk_config* cfg,
                       KArgs a, cudaStream_t st) {
  const int rounds = cfg->philox_rounds == 0 ? kPhiloxRoundsDefault : cfg->philox_rounds;
  if (cfg->mode == WOS_MODE_NATIVE_F32 && rounds != kPhiloxRoundsDefault && rounds != kPhiloxRoundsFast)
    return fail(WOS_ERR_INVALID, "philox_rounds must be %d or %d", kPhiloxRoundsDefault, kPhiloxRoundsFast);
  const KernelInfo k = pick_kernel(s, cfg->mode, a.sink == SINK_ROWS, rounds, cfg->antithetic != 0);
  bool scaled = false;  // the walk runs in X = pi x (see below)
  if (!k.fn)
    return fail(WOS_ERR_UNSUPPORTED, "no kernel for dim %d domain %d source %d mode %d", s->dim,
                s->dom_kind, s->src_kind, cfg->mode);
  if (cfg->mode == WOS_MODE_REPLAY_F64) {
    a.table = s->d_table_d;
    a.segs = s->d_segs_d;
    a.stage_bytes = (int)s->bytes_d;
    a.sine_K = s->sine_K;
  } else if (cfg->mode == WOS_MODE_REPLAY_F32) {
    a.table = s->d_table_f;
    a.segs = s->d_segs_f;
    a.stage_bytes = (int)s->bytes_f;
    a.sine_K = s->sine_K;
  } else {
    a.table = s->d_table_n;
    a.segs = s->d_segs_n;
    a.nodes = s->d_poly_grid;
    a.stage_bytes = (int)s->bytes_f;
    a.sine_K = s->sine_K_native;
    // polygon records go to shared memory when they fit and the set has no candidate
    // grids (grid queries touch a few records each: L1 serves them, and the freed
    // shared memory buys occupancy)
    if (s->bytes_segs_n > 0 && s->bytes_segs_n <= kSegStageMax && !s->poly_grid)
      a.seg_stage_bytes = (int)s->bytes_segs_n;
    if (k.one) {
      // instance row and Philox4x32 round keys ride in the kernel parameters
      a.stage_bytes = 0;
      // scaled-coordinate kernels (wos_walk.cuh Walker::kScaled: single-instance,
      // constant boundary, box, monomial sine source, estimate sink) walk in X = pi x
      scaled = WOS_SCALED_COORDS && a.sink == SINK_ESTIMATE && s->bnd_kind == WOS_BND_CONST &&
               s->dom_kind == WOS_DOM_BOX && s->src_kind == WOS_SRC_SINE &&
               (s->sk_native == 3 || s->sk_native == 4);
      memcpy(a.cp, (k.cube ? s->h_row_n_cube : scaled ? s->h_row_n_scaled : s->h_row_n).data(),
             sizeof(float) * s->stride);
      a.bnd_c = s->h_row_n[s->bnd_off];
      const uint32_t k0 = (uint32_t)cfg->rng_seed;
      const uint32_t k1 = (uint32_t)(cfg->rng_seed >> 32) ^ s->h_nkey1;
      for (int r = 0; r < 10; ++r) {
        a.rk0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
        a.rk1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
      }
    }
  }
  if (s->dom_kind == WOS_DOM_MESH) {
    const bool f64 = cfg->mode == WOS_MODE_REPLAY_F64;
    a.segs = f64 ? (const void*)s->d_mesh_tris_d : (const void*)s->d_mesh_tris_f;
    a.nodes = f64 ? (const void*)s->d_mesh_nodes_d : (const void*)s->d_mesh_nodes_f;
    a.seg_stage_bytes = 0;
  }
  if (s->dom_kind == WOS_DOM_POLAR) {
    // the curve table goes to shared memory when it fits (single-instance sets)
    const bool f64 = cfg->mode == WOS_MODE_REPLAY_F64;
    a.segs = f64 ? (const void*)s->d_polar_d : (const void*)s->d_polar_f;
    const size_t b = f64 ? s->bytes_polar_d : s->bytes_polar_f;
    a.seg_stage_bytes = (b + 15) / 16 * 16 <= kSegStageMax ? (int)((b + 15) / 16 * 16) : 0;
    if (a.seg_stage_bytes && b % 16) a.seg_stage_bytes = 0;  // staged as 16-byte words
  }
  a.hdr = s->d_hdr;
  a.n_inst = s->n;
  a.stride = s->stride;
  a.bnd_off = s->bnd_off;
  a.bnd_kind = s->bnd_kind;
  a.bnd_M = s->bnd_M;
  a.refill_min = c->refill_min;
  a.refill_min_deferred = c->refill_min_deferred;
  a.eps = cfg->eps;
  a.eps_f = (float)(scaled ? M_PI * cfg->eps : cfg->eps);
  a.max_steps = (int32_t)std::min<int64_t>(cfg->max_steps, 0x7fffffff);
  a.antithetic = cfg->antithetic ? 1 : 0;
  a.seed = cfg->rng_seed;
  a.nkey0 = (uint32_t)cfg->rng_seed;
  if (!k.one)  // multi-instance NATIVE kernels read the launch-uniform k0 schedule too
    for (int r = 0; r < 10; ++r) a.rk0[r] = a.nkey0 + (uint32_t)r * 0x9E3779B9u;
  a.nkey1_seed = (uint32_t)(cfg->rng_seed >> 32);
  if (s->src_kind == WOS_SRC_SCREENED_CONST || s->src_kind == WOS_SRC_SCREENED_VC) {
    // walker.py:324-325: delta tracking needs a positive majorant; the constant-coefficient
    // kernel path rejects s' > sigma_bar before walking (walker.py:336-340)
    if (!(cfg->sigma_bar > 0.0))
      return fail(WOS_ERR_INVALID, "delta tracking requires a positive sigma_bar");
    if (s->scr_sprime_max > cfg->sigma_bar) {
      return fail(WOS_ERR_MAJORANT, "majorant violated: sigma'=%.17g > sigma_bar=%.17g",
                  s->scr_sprime_max, cfg->sigma_bar);
    }
  }
  a.philox_rounds = rounds;
  a.sigma_bar = cfg->sigma_bar;
  a.sqrt_sig = sqrt(cfg->sigma_bar > 0.0 ? cfg->sigma_bar : 0.0);
  a.majorant = c->d_majorant;
  // NATIVE source jumps read their radius table from shared memory
  if (cfg->mode == WOS_MODE_NATIVE_F32 && s->src_kind != WOS_SRC_NONE &&
      s->src_kind != WOS_SRC_SCREENED_CONST && s->src_kind != WOS_SRC_SCREENED_VC) {
    a.beta_tab = s->dim == 3 ? c->d_beta_tab : c->d_green2_tab;
    // (polygon and mesh kernels read it through L1: wos_walk.cuh kBetaGlobal)
    if (s->dom_kind != WOS_DOM_POLYGON && s->dom_kind != WOS_DOM_MESH)
      a.beta_stage_bytes = (int)(sizeof(float) * WOS_BETA_TABLE_N);
  }
  const size_t smem =
      smem_bytes((size_t)a.stage_bytes + (size_t)a.seg_stage_bytes + (size_t)a.beta_stage_bytes, k.elem, k.warps);
  if (smem > 220 * 1024)
    return fail(WOS_ERR_UNSUPPORTED,
                "problem table too large for shared memory (%zu bytes); split the batch",
                (size_t)a.stage_bytes);
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> g(c->launch_mu);
    auto it = c->launch_cache.find(k.fn);
    if (it != c->launch_cache.end() && it->second.first == smem) {
      per_sm = it->second.second;
    } else {
      CUDA_TRY(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.fn, 32 * k.warps, smem));
#if WOS_CARVEOUT
      // the smallest shared-memory carve-out that still holds per_sm CTAs (plus the
      // 1 KB the runtime reserves per CTA): the rest of the 256 KB stays L1 for the
      // walks' global reads (polygon grids, BVH nodes, query points)
      if (per_sm > 0) {
        int smem_sm = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->device));
        const size_t need = (size_t)per_sm * (smem + 1024);
        const int pct = (int)std::min<size_t>(100, (need * 100 + smem_sm - 1) / smem_sm);
        CUDA_TRY(cudaFuncSetAttribute(k.fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        int per_sm2 = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k.fn, 32 * k.warps, smem));
        if (per_sm2 < per_sm)  // the carve-out rounding lost a CTA: let the driver choose
          CUDA_TRY(cudaFuncSetAttribute(k.fn, cudaFuncAttributePreferredSharedMemoryCarveout, -1));
      }
#endif
      c->launch_cache[k.fn] = std::make_pair(smem, per_sm);
    }
  }
  if (per_sm < 1) return fail(WOS_ERR_UNSUPPORTED, "kernel does not fit on an SM");
  if (c->blocks_per_sm > 0) per_sm = std::min(per_sm, c->blocks_per_sm);
  int64_t grid = (int64_t)c->num_sms * per_sm;
  grid = std::min<int64_t>(grid, ((int64_t)a.n_units + k.warps - 1) / k.warps);
  grid = std::max<int64_t>(grid, 1);
  unsigned slot = c->next_counter.fetch_add(1) % kCounterRing;
  a.work_counter = c->d_counters + slot;
  a.watchdog = c->d_watchdog;
  a.iter_limit = (uint32_t)std::min<int64_t>(0xffffffffll, std::max<int64_t>(1ll << 27, 4 * (int64_t)a.max_steps));
  CUDA_TRY(cudaMemsetAsync(a.work_counter, 0, sizeof(unsigned), st));
  void* args[] = {&a};
  a.seg_evals = c->d_perf;
  CUDA_TRY(cudaLaunchKernel(k.fn, dim3((unsigned)grid), dim3(32 * k.warps), args, smem, st));
  wos_context_count_launch(c);
  return WOS_OK;
}

// Chan-merge each point's chunk moments in chunk order (L > kChunk)
__global__ void wos_merge_chunks_kernel(uint32_t n_points, uint32_t L, uint32_t n_chunks, int anti,
                                        const double* __restrict__ partials, double* __restrict__ out_mean,
                                        double* __restrict__ out_m2) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n_points; p += gridDim.x * blockDim.x) {
    double n1 = 0.0, mean = 0.0, m2 = 0.0;
    for (uint32_t c = 0; c < n_chunks; ++c) {
      const uint32_t valid = min((uint32_t)kChunk, L - c * kChunk);
      const double n2 = (double)(anti ? valid / 2 : valid);
      const double mc = partials[2 * ((size_t)p * n_chunks + c)];
      const double qc = partials[2 * ((size_t)p * n_chunks + c) + 1];
      const double nn = n1 + n2;
      const double delta = mc - mean;
      mean = mean + delta * (n2 / nn);
      m2 = m2 + qc + delta * delta * (n1 * n2 / nn);
      n1 = nn;
    }
    out_mean[p] = mean;
    out_m2[p] = m2;
  }
}

static const int64_t kMaxItemsPerLaunch = (1ll << 31) - 4 * kRing;

extern "C" int wos_walk_rows(wos_context* c, const wos_problem_set* s, const wos_walk_config* cfg,
                             int64_t n, const double* points, const uint64_t* pid,
                             const uint64_t* tid, const double* signs, double* out_values,
                             int64_t* out_steps, uint8_t* out_hits, void* stream) {
  if (!c || !s || !cfg) return fail(WOS_ERR_INVALID, "null argument");
  if (n < 0) return fail(WOS_ERR_INVALID, "negative row count");
  if (!(cfg->eps > 0.0)) return fail(WOS_ERR_INVALID, "eps_shell must be positive");
  if (cfg->max_steps < 1) return fail(WOS_ERR_INVALID, "max_steps must be at least 1");
  if (n == 0) return WOS_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int r0 = reset_status(c, st);
  if (r0) return r0;
  for (int64_t off = 0; off < n; off += kMaxItemsPerLaunch) {
    const int64_t m = std::min<int64_t>(kMaxItemsPerLaunch, n - off);
    KArgs a;
    memset(&a, 0, sizeof(a));
    a.sink = SINK_ROWS;
    a.n_points = (uint32_t)m;
    a.L = 1;
    a.U = kUnitTarget;
    a.IU = kUnitTarget;
    a.n_units = (uint32_t)((m + kUnitTarget - 1) / kUnitTarget);
    a.n_chunks = 0;
    fast_div_init(a.IU, &a.iu_mul, &a.iu_shr);
    fast_div_init(1, &a.l_mul, &a.l_shr);
    fast_div_init(1, &a.nc_mul, &a.nc_shr);
    a.points = points + off * s->dim;
    a.row_pid = pid + off;
    a.row_tid = tid + off;
    a.row_sign = signs + off;
    a.out_values = out_values + off;
    a.out_steps = out_steps + off;
    a.out_hits = out_hits + off;
    int r = launch_walk(c, s, cfg, a, st);
    if (r) return r;
  }
  return WOS_OK;
}

// idx_base: index of points[0] in the caller's full point array (chunked host
// pipeline): offsets exterior-point reports and the default point ids.
static int estimate_impl(wos_context* c, const wos_problem_set* s, const wos_walk_config* cfg,
                         int64_t P, const double* points, const int64_t* point_ids,
                         const int32_t* inst_index, int64_t L, uint64_t traj_start,
                         double* out_mean, double* out_m2, uint64_t* out_total_steps,
                         cudaStream_t st, int64_t idx_base) {
  if (!c || !s || !cfg) return fail(WOS_ERR_INVALID, "null argument");
  if (P < 0) return fail(WOS_ERR_INVALID, "negative point count");
  if (L < 1) return fail(WOS_ERR_INVALID, "trajectory count must be at least 1");
  if (cfg->antithetic && (L % 2)) return fail(WOS_ERR_INVALID, "antithetic estimation needs an even trajectory count");
  if (!(cfg->eps > 0.0)) return fail(WOS_ERR_INVALID, "eps_shell must be positive");
  if (cfg->max_steps < 1) return fail(WOS_ERR_INVALID, "max_steps must be at least 1");
  if (L > kMaxItemsPerLaunch) return fail(WOS_ERR_UNSUPPORTED, "L too large");
  if (P == 0) return WOS_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  int r = launch_interior(c, s, P, points, inst_index, st, idx_base);
  if (r) return r;
  // L > kChunk: units are kChunk-walk chunks of one point, merged by wos_merge_chunks_kernel
  const bool split = L > kChunk;
  const int64_t n_chunks = split ? (L + kChunk - 1) / kChunk : 0;
  const int64_t items_per_point = split ? n_chunks * kChunk : L;
  const int64_t pts_per_launch = std::max<int64_t>(1, kMaxItemsPerLaunch / items_per_point);
  double* partials = nullptr;
  if (split) {
    const int64_t m_max = std::min<int64_t>(pts_per_launch, P);
    CUDA_TRY(cudaMallocAsync((void**)&partials, (size_t)m_max * n_chunks * 2 * sizeof(double), st));
  }
  for (int64_t off = 0; off < P; off += pts_per_launch) {
    const int64_t m = std::min<int64_t>(pts_per_launch, P - off);
    KArgs a;
    memset(&a, 0, sizeof(a));
    a.sink = SINK_ESTIMATE;
    a.n_points = (uint32_t)m;
    a.L = (uint32_t)L;
    if (split) {
      a.U = 1;
      a.IU = kChunk;
      a.n_chunks = (uint32_t)n_chunks;
      a.n_units = (uint32_t)(m * n_chunks);
      a.partials = partials;
    } else {
      // L >= 32: one point per unit (the cached-point fast refill path);
      // smaller L: whole points up to >= kUnitTarget walks per unit
      a.U = L >= 32 ? 1u : (uint32_t)((kUnitTarget + L - 1) / L);
      a.IU = a.U * a.L;
      a.n_units = (uint32_t)((m + a.U - 1) / a.U);
      a.n_chunks = 0;
    }
    fast_div_init(a.IU, &a.iu_mul, &a.iu_shr);
    fast_div_init(a.L, &a.l_mul, &a.l_shr);
    fast_div_init(std::max<uint32_t>(1u, a.n_chunks), &a.nc_mul, &a.nc_shr);
    a.points = points + off * s->dim;
    a.point_ids = point_ids ? point_ids + off : nullptr;
    a.id_base = (uint64_t)(idx_base + off);
    a.inst_index = inst_index ? inst_index + off : nullptr;
    a.traj_start = traj_start;
    a.out_mean = out_mean + off;
    a.out_m2 = out_m2 + off;
    a.total_steps = reinterpret_cast<unsigned long long*>(out_total_steps);
    r = launch_walk(c, s, cfg, a, st);
    if (r) {
      if (partials) cudaFreeAsync(partials, st);
      return r;
    }
    if (split) {
      const int blocks = (int)std::min<int64_t>((m + 255) / 256, (int64_t)c->num_sms * 8);
      wos_merge_chunks_kernel<<<blocks, 256, 0, st>>>((uint32_t)m, (uint32_t)L, (uint32_t)n_chunks,
                                                      cfg->antithetic ? 1 : 0, partials,
                                                      out_mean + off, out_m2 + off);
      CUDA_TRY(cudaGetLastError());
      wos_context_count_launch(c);
    }
  }
  if (partials) CUDA_TRY(cudaFreeAsync(partials, st));
  return WOS_OK;
}

extern "C" int wos_estimate(wos_context* c, const wos_problem_set* s, const wos_walk_config* cfg,
                            int64_t P, const double* points, const int64_t* point_ids,
                            const int32_t* inst_index, int64_t L, uint64_t traj_start,
                            double* out_mean, double* out_m2, uint64_t* out_total_steps,
                            void* stream) {
  if (c && s && cfg && P > 0) {
    CUDA_TRY(cudaSetDevice(c->device));
    int r = reset_status(c, (cudaStream_t)stream);
    if (r) return r;
  }
  return estimate_impl(c, s, cfg, P, points, point_ids, inst_index, L, traj_start, out_mean, out_m2,
                       out_total_steps, (cudaStream_t)stream, 0);
}

extern "C" int wos_estimate_fold(wos_context* c, const wos_problem_set* s,
                                 const wos_walk_config* cfg, int64_t P, const double* points,
                                 const int64_t* point_ids, const int32_t* inst_index, int64_t L,
                                 uint64_t traj_start, const int64_t* slot, double* mean_sum,
                                 int64_t* n, double* mean, double* m2, uint64_t* out_total_steps,
                                 void* stream) {
  if (!c || !cfg) return fail(WOS_ERR_INVALID, "wos_estimate_fold: null argument");
  if (P < 0) return fail(WOS_ERR_INVALID, "wos_estimate_fold: negative point count");
  if (P == 0) return WOS_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int r0 = reset_status(c, st);
  if (r0) return r0;
  // the epoch's fresh (mean, m2) live only in stream-ordered scratch
  double* fresh = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&fresh, 2 * (size_t)P * sizeof(double), st));
  int r = estimate_impl(c, s, cfg, P, points, point_ids, inst_index, L, traj_start, fresh,
                        fresh + P, out_total_steps, st, 0);
  if (r == WOS_OK)
    r = wos_cache_fold(c, P, slot, fresh, fresh + P, nullptr, cfg->antithetic ? L / 2 : L,
                       mean_sum, n, mean, m2, stream);
  cudaFreeAsync(fresh, st);
  return r;
}

// ---- host-buffer variants ------------------------------------------------
static int scratch(wos_context* c, size_t bytes, char** out) {
  if (bytes > c->scratch_bytes) {
    cudaFree(c->d_scratch);
    c->d_scratch = nullptr;
    c->scratch_bytes = 0;
    size_t want = std::max(bytes, (size_t)1 << 20);
    CUDA_TRY(cudaMalloc(&c->d_scratch, want));
    c->scratch_bytes = want;
  }
  *out = (char*)c->d_scratch;
  return WOS_OK;
}

static size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

extern "C" int wos_walk_rows_host(wos_context* c, const wos_problem_set* s,
                                  const wos_walk_config* cfg, int64_t n, const double* points,
                                  const uint64_t* pid, const uint64_t* tid, const double* signs,
                                  double* out_values, int64_t* out_steps, uint8_t* out_hits) {
  if (!c || !s || !cfg) return fail(WOS_ERR_INVALID, "null argument");
  if (n <= 0) return n < 0 ? fail(WOS_ERR_INVALID, "negative row count") : WOS_OK;
  std::lock_guard<std::mutex> g(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t bp = al(n * s->dim * 8), b8 = al(n * 8), b1 = al(n);
  char* base;
  int r = scratch(c, bp + 5 * b8 + b1, &base);
  if (r) return r;
  double* d_pts = (double*)base;
  uint64_t* d_pid = (uint64_t*)(base + bp);
  uint64_t* d_tid = (uint64_t*)(base + bp + b8);
  double* d_sgn = (double*)(base + bp + 2 * b8);
  double* d_val = (double*)(base + bp + 3 * b8);
  int64_t* d_stp = (int64_t*)(base + bp + 4 * b8);
  uint8_t* d_hit = (uint8_t*)(base + bp + 5 * b8);
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMemcpyAsync(d_pts, points, n * s->dim * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_pid, pid, n * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_tid, tid, n * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_sgn, signs, n * 8, cudaMemcpyHostToDevice, st));
  r = wos_walk_rows(c, s, cfg, n, d_pts, d_pid, d_tid, d_sgn, d_val, d_stp, d_hit, st);
  if (r) return r;
  CUDA_TRY(cudaMemcpyAsync(out_values, d_val, n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out_steps, d_stp, n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out_hits, d_hit, n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  r = check_watchdog(c, st);
  if (r) return r;
  return check_majorant(c, cfg, st);
}

extern "C" int wos_check_interior_host(wos_context* c, const wos_problem_set* s, int64_t n,
                                       const double* points, const int32_t* inst_index,
                                       int64_t* out_first) {
  if (!c || !s || !out_first) return fail(WOS_ERR_INVALID, "null argument");
  if (n <= 0) {
    *out_first = -1;
    return n < 0 ? fail(WOS_ERR_INVALID, "negative point count") : WOS_OK;
  }
  std::lock_guard<std::mutex> g(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t bp = al(n * s->dim * 8);
  char* base;
  int r = scratch(c, bp + al(n * 4), &base);
  if (r) return r;
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMemcpyAsync(base, points, n * s->dim * 8, cudaMemcpyHostToDevice, st));
  int32_t* d_inst = nullptr;
  if (inst_index) {
    d_inst = (int32_t*)(base + bp);
    CUDA_TRY(cudaMemcpyAsync(d_inst, inst_index, n * 4, cudaMemcpyHostToDevice, st));
  }
  r = launch_interior(c, s, n, (const double*)base, d_inst, st);
  if (r) return r;
  return read_exterior(c, st, out_first);
}

extern "C" int wos_estimate_host(wos_context* c, const wos_problem_set* s,
                                 const wos_walk_config* cfg, int64_t P, const double* points,
                                 const int64_t* point_ids, const int32_t* inst_index, int64_t L,
                                 uint64_t traj_start, double* out_mean, double* out_m2,
                                 uint64_t* out_total_steps) {
  if (!c || !s || !cfg) return fail(WOS_ERR_INVALID, "null argument");
  if (P <= 0) {
    if (out_total_steps) *out_total_steps = 0;
    return P < 0 ? fail(WOS_ERR_INVALID, "negative point count") : WOS_OK;
  }
  if (L < 1 || (cfg->antithetic && (L % 2)))  // same checks and messages as wos_estimate
    return estimate_impl(c, s, cfg, P, nullptr, nullptr, nullptr, L, traj_start, nullptr, nullptr,
                         nullptr, c->stream, 0);
  std::lock_guard<std::mutex> g(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t bp = al(P * s->dim * 8), b8 = al(P * 8), b4 = al(P * 4);
  char* base;
  int r = scratch(c, bp + 3 * b8 + b4, &base);
  if (r) return r;
  double* d_pts = (double*)base;
  int64_t* d_ids = point_ids ? (int64_t*)(base + bp) : nullptr;
  double* d_mean = (double*)(base + bp + b8);
  double* d_m2 = (double*)(base + bp + 2 * b8);
  int32_t* d_inst = inst_index ? (int32_t*)(base + bp + 3 * b8) : nullptr;
  const cudaStream_t cs = c->stream, xs = c->copy_stream, cs2 = c->stream2;
  CUDA_TRY(cudaMemsetAsync(c->d_steps, 0, sizeof(unsigned long long), cs));
  if ((r = reset_status(c, cs))) return r;
  CUDA_TRY(cudaEventRecord(c->ev_start, cs));
  CUDA_TRY(cudaStreamWaitEvent(cs2, c->ev_start, 0));
  // Software pipeline over point chunks: copies on `xs`, walks alternately on `cs` and
  // `cs2`, so the copies of chunk i+1 and the results of chunk i-1 overlap the walks
  // of chunk i, and chunk i+1's persistent grid fills the SMs chunk i's tail frees.
  const int64_t work = P * L;
  const int nch = (int)std::max<int64_t>(1, std::min<int64_t>(kPipeChunks, work / kPipeMinWork));
  int64_t lo[kPipeChunks + 1];
  for (int i = 0; i <= nch; ++i) lo[i] = P * i / nch;
#if WOS_PIPE_EDGE > 0
  // small first and last chunks (P / WOS_PIPE_EDGE points each): only their copies are
  // exposed, the middle chunks' overlap the walks
  if (nch >= 3) {
    const int64_t edge = P / WOS_PIPE_EDGE;
    lo[1] = edge;
    lo[nch - 1] = P - edge;
    for (int i = 2; i < nch - 1; ++i) lo[i] = edge + (P - 2 * edge) * (i - 1) / (nch - 2);
  }
#endif
  auto d2h = [&](int i) -> int {
    const int64_t o = lo[i], m = lo[i + 1] - lo[i];
    CUDA_TRY(cudaStreamWaitEvent(xs, c->ev_kernel[i], 0));
    CUDA_TRY(cudaMemcpyAsync(out_mean + o, d_mean + o, m * 8, cudaMemcpyDeviceToHost, xs));
    CUDA_TRY(cudaMemcpyAsync(out_m2 + o, d_m2 + o, m * 8, cudaMemcpyDeviceToHost, xs));
    return WOS_OK;
  };
  for (int i = 0; i < nch; ++i) {
    const int64_t o = lo[i], m = lo[i + 1] - lo[i];
    const cudaStream_t ks = (i & 1) ? cs2 : cs;
    CUDA_TRY(cudaMemcpyAsync(d_pts + o * s->dim, points + o * s->dim, m * s->dim * 8,
                             cudaMemcpyHostToDevice, xs));
    if (d_ids) CUDA_TRY(cudaMemcpyAsync(d_ids + o, point_ids + o, m * 8, cudaMemcpyHostToDevice, xs));
    if (d_inst) CUDA_TRY(cudaMemcpyAsync(d_inst + o, inst_index + o, m * 4, cudaMemcpyHostToDevice, xs));
    CUDA_TRY(cudaEventRecord(c->ev_copy[i], xs));
    CUDA_TRY(cudaStreamWaitEvent(ks, c->ev_copy[i], 0));
    r = estimate_impl(c, s, cfg, m, d_pts + o * s->dim, d_ids ? d_ids + o : nullptr,
                      d_inst ? d_inst + o : nullptr, L, traj_start, d_mean + o, d_m2 + o,
                      reinterpret_cast<uint64_t*>(c->d_steps), ks, o);
    if (r) return r;
    CUDA_TRY(cudaEventRecord(c->ev_kernel[i], ks));
    if (i > 0 && (r = d2h(i - 1))) return r;
  }
  if ((r = d2h(nch - 1))) return r;
  // join the second walk stream before reading the counters
  CUDA_TRY(cudaEventRecord(c->ev_start, cs2));
  CUDA_TRY(cudaStreamWaitEvent(cs, c->ev_start, 0));
  unsigned long long steps = 0, ext = 0;
  CUDA_TRY(cudaMemcpyAsync(&steps, c->d_steps, 8, cudaMemcpyDeviceToHost, cs));
  CUDA_TRY(cudaMemcpyAsync(&ext, c->d_exterior, 8, cudaMemcpyDeviceToHost, cs));
  CUDA_TRY(cudaMemsetAsync(c->d_exterior, 0, 8, cs));
  CUDA_TRY(cudaStreamSynchronize(cs));
  CUDA_TRY(cudaStreamSynchronize(xs));
  if (out_total_steps) *out_total_steps = steps;
  r = check_watchdog(c, cs);
  if (r) return r;
  r = check_majorant(c, cfg, cs);
  if (r) return r;
  if (ext != 0ull) {
    c->host_exterior = (int64_t)~ext;
    return fail(WOS_ERR_EXTERIOR, "exterior query: start point %lld", (long long)~ext);
  }
  return WOS_OK;
}

// ------------------------------------------------------------------------
// RNG known-answer kernels
// ------------------------------------------------------------------------
__global__ void philox64_kernel(int64_t n, const uint64_t* ctr, uint64_t k0, uint64_t k1, uint64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w[4];
    philox4x64(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3], k0, k1, w);
    for (int j = 0; j < 4; ++j) out[4 * i + j] = w[j];
  }
}
__global__ void philox32_kernel(int64_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, int rounds,
                                uint32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w =
        philox4x32(make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]), k0, k1, rounds);
    out[4 * i] = w.x;
    out[4 * i + 1] = w.y;
    out[4 * i + 2] = w.z;
    out[4 * i + 3] = w.w;
  }
}

extern "C" int wos_philox4x64(wos_context* c, int64_t n, const uint64_t* ctr, uint64_t k0, uint64_t k1,
                              uint64_t* out, void* stream) {
  if (!c) return fail(WOS_ERR_INVALID, "null context");
  if (n <= 0) return WOS_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 4096);
  philox64_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n, ctr, k0, k1, out);
  CUDA_TRY(cudaGetLastError());
  return WOS_OK;
}

extern "C" int wos_philox4x32(wos_context* c, int64_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1,
                              uint32_t* out, void* stream) {
  if (!c) return fail(WOS_ERR_INVALID, "null context");
  if (n <= 0) return WOS_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 4096);
  philox32_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n, ctr, k0, k1, kPhiloxRoundsDefault, out);
  CUDA_TRY(cudaGetLastError());
  return WOS_OK;
}

extern "C" int wos_philox4x32_rounds(wos_context* c, int64_t n, const uint32_t* ctr, uint32_t k0,
                                     uint32_t k1, int32_t rounds, uint32_t* out, void* stream) {
  if (!c) return fail(WOS_ERR_INVALID, "null context");
  if (rounds < 1 || rounds > 16) return fail(WOS_ERR_INVALID, "rounds must be in 1..16");
  if (n <= 0) return WOS_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 4096);
  philox32_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n, ctr, k0, k1, rounds, out);
  CUDA_TRY(cudaGetLastError());
  return WOS_OK;
}

// ------------------------------------------------------------------------
// roofline probes: MUFU and FFMA throughput
// ------------------------------------------------------------------------
constexpr int kProbeChains = 8;

__global__ void __launch_bounds__(256) probe_mufu_kernel(int iters, float seed, float* sink) {
  float v[kProbeChains];
#pragma unroll
  for (int j = 0; j < kProbeChains; ++j) v[j] = seed + 0.01f * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kProbeChains; ++j) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(v[j]));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kProbeChains; ++j) s += v[j];
  if (s == 1234.5f) sink[0] = s;
}

__global__ void __launch_bounds__(256) probe_ffma_kernel(int iters, float seed, float* sink) {
  float v[kProbeChains];
#pragma unroll
  for (int j = 0; j < kProbeChains; ++j) v[j] = seed + 0.01f * (threadIdx.x + j);
  const float a = 0.999f, b = 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kProbeChains; ++j) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[j]) : "f"(a), "f"(b));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kProbeChains; ++j) s += v[j];
  if (s == 1234.5f) sink[0] = s;
}

extern "C" int wos_fastmath_probe(wos_context* c, int64_t n, const float* x, float* out_sin, float* out_cos,
                                  float* out_sqrt, float* out_ex2, void* stream) {
  if (!c) return fail(WOS_ERR_INVALID, "null context");
  if (n < 0 || (n > 0 && (!x || !out_sin || !out_cos || !out_sqrt || !out_ex2)))
    return fail(WOS_ERR_INVALID, "bad fastmath probe arguments");
  CUDA_TRY(cudaSetDevice(wos_context_device(c)));
  const int err = launch_fastmath_probe(n, x, out_sin, out_cos, out_sqrt, out_ex2, stream);
  if (err) return fail(WOS_ERR_CUDA, "fastmath probe: %s", cudaGetErrorString((cudaError_t)err));
  return WOS_OK;
}

extern "C" int wos_probe_peaks(wos_context* c, double* sfu, double* fp32, double* clk, int32_t* nsm) {
  if (!c) return fail(WOS_ERR_INVALID, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  float* d_sink;
  CUDA_TRY(cudaMalloc(&d_sink, 16));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  cudaStream_t st = c->stream;
  const int blocks = c->num_sms * 8, threads = 256;
  double best_sfu = 0, best_fma = 0;
  for (int rep = 0; rep < 4; ++rep) {
    const int it_mufu = 4096, it_fma = 16384;
    CUDA_TRY(cudaEventRecord(e0, st));
    probe_mufu_kernel<<<blocks, threads, 0, st>>>(it_mufu, 1.5f, d_sink);
    CUDA_TRY(cudaEventRecord(e1, st));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    if (rep > 0) best_sfu = std::max(best_sfu, (double)blocks * threads * it_mufu * kProbeChains / (ms * 1e-3));
    CUDA_TRY(cudaEventRecord(e0, st));
    probe_ffma_kernel<<<blocks, threads, 0, st>>>(it_fma, 1.5f, d_sink);
    CUDA_TRY(cudaEventRecord(e1, st));
    CUDA_TRY(cudaEventSynchronize(e1));
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    if (rep > 0) best_fma = std::max(best_fma, 2.0 * blocks * threads * (double)it_fma * kProbeChains / (ms * 1e-3));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d_sink);
  if (sfu) *sfu = best_sfu;
  if (fp32) *fp32 = best_fma;
  if (clk) *clk = best_fma / ((double)c->num_sms * 256.0);
  if (nsm) *nsm = c->num_sms;
  return WOS_OK;
}
