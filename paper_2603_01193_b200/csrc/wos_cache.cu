// Epoch-averaged estimate cache on the device (estimator.EstimateCache,
// estimator.py:188-302) and the fused estimate -> cache fold of the
// training-label loop (surrogate.py:283-297).
//
// Compiled with --fmad=false: the fold must reproduce the reference's float64
// arithmetic operation by operation (Python never fuses a multiply-add), so an
// incremental, a resumed and a replayed run give bit-identical targets
// (test_estimator.py:196-222).
#include <cuda_runtime.h>

#include <cstdint>

#include "wos_b200.h"
#include "wos_kernels.h"

namespace wos {

// One epoch for entry s = slot[k] (or k): mean_sum += mean (estimator.py:232) and
// (n, mean, m2) <- chan_merge((n, mean, m2), (n_e, mean_e, m2_e)) (estimator.py:41-53,
// 233-243). n1 * n2 / n is Python's int-product / int true division: exact while the
// product stays below 2^53 (n1, n2 < 9.4e7 each), which the host checks.
__global__ void wos_cache_fold_kernel(int64_t n_fresh, const int64_t* __restrict__ slot,
                                      const double* __restrict__ fmean,
                                      const double* __restrict__ fm2,
                                      const int64_t* __restrict__ fn, int64_t fn_all,
                                      double* __restrict__ mean_sum, int64_t* __restrict__ n,
                                      double* __restrict__ mean, double* __restrict__ m2) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_fresh;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = slot ? slot[k] : k;
    const double em = fmean[k], em2 = fm2[k];
    const int64_t n2 = fn ? fn[k] : fn_all;
    mean_sum[s] = mean_sum[s] + em;
    const int64_t n1 = n[s];
    const int64_t nn = n1 + n2;
    if (nn == 0) {
      n[s] = 0;
      mean[s] = 0.0;
      m2[s] = 0.0;
      continue;
    }
    const double m1 = mean[s], m21 = m2[s];
    const double delta = em - m1;
    const double w2 = (double)n2 / (double)nn;
    const double w12 = (double)(n1 * n2) / (double)nn;
    mean[s] = m1 + delta * w2;
    m2[s] = (m21 + em2) + (delta * delta) * w12;
    n[s] = nn;
  }
}

// targets = mean_sum / epoch (estimator.py:251-255)
__global__ void wos_cache_targets_kernel(int64_t n_keys, const double* __restrict__ mean_sum,
                                         double epoch, double* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_keys;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = mean_sum[k] / epoch;
}

static int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace wos

using namespace wos;

extern "C" int wos_cache_fold(wos_context* ctx, int64_t n_fresh, const int64_t* slot,
                              const double* fresh_mean, const double* fresh_m2,
                              const int64_t* fresh_n, int64_t fresh_n_all, double* mean_sum,
                              int64_t* n, double* mean, double* m2, void* stream) {
  if (!ctx) return wos_fail(WOS_ERR_INVALID, "wos_cache_fold: null context");
  if (n_fresh < 0) return wos_fail(WOS_ERR_INVALID, "wos_cache_fold: negative key count");
  if (n_fresh == 0) return WOS_OK;
  if (!fresh_mean || !fresh_m2 || !mean_sum || !n || !mean || !m2)
    return wos_fail(WOS_ERR_INVALID, "wos_cache_fold: null buffer");
  if (!fresh_n && (fresh_n_all < 0 || fresh_n_all > (int64_t)94906265))
    return wos_fail(WOS_ERR_INVALID, "wos_cache_fold: sample count out of range");
  if (cudaSetDevice(wos_context_device(ctx)) != cudaSuccess)
    return wos_fail(WOS_ERR_CUDA, "wos_cache_fold: cudaSetDevice failed");
  wos_cache_fold_kernel<<<grid_for(n_fresh), 256, 0, (cudaStream_t)stream>>>(
      n_fresh, slot, fresh_mean, fresh_m2, fresh_n, fresh_n_all, mean_sum, n, mean, m2);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return wos_fail(WOS_ERR_CUDA, cudaGetErrorString(e));
  wos_context_count_launch(ctx);
  return WOS_OK;
}

extern "C" int wos_cache_targets(wos_context* ctx, int64_t n_keys, const double* mean_sum,
                                 int64_t epoch, double* out, void* stream) {
  if (!ctx) return wos_fail(WOS_ERR_INVALID, "wos_cache_targets: null context");
  if (n_keys < 0 || epoch < 1) return wos_fail(WOS_ERR_INVALID, "wos_cache_targets: empty cache");
  if (n_keys == 0) return WOS_OK;
  if (!mean_sum || !out) return wos_fail(WOS_ERR_INVALID, "wos_cache_targets: null buffer");
  if (cudaSetDevice(wos_context_device(ctx)) != cudaSuccess)
    return wos_fail(WOS_ERR_CUDA, "wos_cache_targets: cudaSetDevice failed");
  wos_cache_targets_kernel<<<grid_for(n_keys), 256, 0, (cudaStream_t)stream>>>(
      n_keys, mean_sum, (double)epoch, out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return wos_fail(WOS_ERR_CUDA, cudaGetErrorString(e));
  wos_context_count_launch(ctx);
  return WOS_OK;
}
