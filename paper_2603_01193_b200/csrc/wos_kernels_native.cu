// NATIVE_F32 kernel lookup (instantiations live in wos_kernels_native_{est,rows}.cu).
#include "wos_kernels.h"
#include "wos_walk.cuh"

namespace wos {
const void* get_kernel_native_est(int dim, int dom, int src, int sk, bool one);
const void* get_kernel_native_rows(int dim, int dom, int src, int sk, bool one);
const void* get_kernel_native_est_bc(int dim, int dom, int src, int sk, bool one);
const void* get_kernel_native_est_r7(int dim, int dom, int src, int sk, bool one);
const void* get_kernel_native_est_bc_r7(int dim, int dom, int src, int sk, bool one);

int get_kernel_native_est_warps();
int get_kernel_native_rows_warps();
int get_kernel_native_est_bc_warps();
int get_kernel_native_est_r7_warps();
int get_kernel_native_est_bc_r7_warps();

const void* get_kernel_native(int dim, int dom, int src, int sk, bool one, bool rows, bool bnd_const,
                              int rounds, int* warps) {
  if (rows) {
    *warps = get_kernel_native_rows_warps();
    return get_kernel_native_rows(dim, dom, src, sk, one);
  }
  if (one && rounds == kPhiloxRoundsFast) {
    *warps = bnd_const ? get_kernel_native_est_bc_r7_warps() : get_kernel_native_est_r7_warps();
    return bnd_const ? get_kernel_native_est_bc_r7(dim, dom, src, sk, one) : get_kernel_native_est_r7(dim, dom, src, sk, one);
  }
  if (one && bnd_const) {
    *warps = get_kernel_native_est_bc_warps();
    return get_kernel_native_est_bc(dim, dom, src, sk, one);
  }
  *warps = get_kernel_native_est_warps();
  return get_kernel_native_est(dim, dom, src, sk, one);
}
}  // namespace wos

namespace wos {
// The fast-math primitives of the NATIVE kernels, evaluated on given arguments so their
// error can be bounded against libm (wos_fastmath_probe, tests/test_gpu_fastmath.py).
__global__ void fastmath_probe_kernel(int64_t n, const float* __restrict__ x, float* __restrict__ s,
                                      float* __restrict__ c, float* __restrict__ q, float* __restrict__ e) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float si, co;
    __sincosf(x[i], &si, &co);
    s[i] = si;
    c[i] = co;
    q[i] = fast_sqrt(fabsf(x[i]));
    e[i] = fast_ex2(x[i]);
  }
}

int launch_fastmath_probe(int64_t n, const float* x, float* s, float* c, float* q, float* e, void* stream) {
  if (n <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  fastmath_probe_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, x, s, c, q, e);
  return (int)cudaGetLastError();
}
}  // namespace wos
