// NATIVE_F32 kernel instantiations, est sink (see wos_kernels_native.inc).
#include "wos_kernels.h"
#include "wos_walk.cuh"

#define WOS_SINK SINK_ESTIMATE
#define WOS_FN get_kernel_native_est
#include "wos_kernels_native.inc"
