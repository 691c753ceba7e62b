// NATIVE_F32 kernel lookup (instantiations live in wos_kernels_native_{est,rows}.cu).
#include "wos_kernels.h"

namespace wos {
const void* get_kernel_native_est(int dim, int dom, int src, int sk, bool one);
const void* get_kernel_native_rows(int dim, int dom, int src, int sk, bool one);

const void* get_kernel_native(int dim, int dom, int src, int sk, bool one, bool rows) {
  return rows ? get_kernel_native_rows(dim, dom, src, sk, one) : get_kernel_native_est(dim, dom, src, sk, one);
}
}  // namespace wos
