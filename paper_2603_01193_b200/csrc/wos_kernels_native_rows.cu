// NATIVE_F32 kernel instantiations, rows sink (see wos_kernels_native.inc).
#include "wos_kernels.h"
#include "wos_walk.cuh"

#define WOS_SINK SINK_ROWS
#define WOS_FN get_kernel_native_rows
#include "wos_kernels_native.inc"
