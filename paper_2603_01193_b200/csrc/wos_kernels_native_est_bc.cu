// NATIVE_F32 kernel instantiations, est sink, single-instance launches with a constant
// boundary (Spec BC; see wos_kernels_native.inc). Own unit for parallel compilation.
#include "wos_kernels.h"
#include "wos_walk.cuh"

#define WOS_SINK SINK_ESTIMATE
#define WOS_BC 1
#define WOS_FN get_kernel_native_est_bc
#include "wos_kernels_native.inc"
