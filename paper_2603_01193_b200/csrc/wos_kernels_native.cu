// NATIVE_F32 kernel lookup (instantiations live in wos_kernels_native_{est,rows}.cu).
#include "wos_kernels.h"

namespace wos {
const void* get_kernel_native_est(int dim, int dom, int src, int sk, bool one);
const void* get_kernel_native_rows(int dim, int dom, int src, int sk, bool one);
const void* get_kernel_native_est_bc(int dim, int dom, int src, int sk, bool one);

const void* get_kernel_native(int dim, int dom, int src, int sk, bool one, bool rows, bool bnd_const) {
  if (rows) return get_kernel_native_rows(dim, dom, src, sk, one);
  if (one && bnd_const) return get_kernel_native_est_bc(dim, dom, src, sk, one);
  return get_kernel_native_est(dim, dom, src, sk, one);
}
}  // namespace wos
