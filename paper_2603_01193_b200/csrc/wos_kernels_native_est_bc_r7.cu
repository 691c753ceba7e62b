// NATIVE_F32 single-instance estimate kernels built for the opt-in 7-round Philox
// stream (WalkConfig.philox_rounds = 7), constant boundary (Spec BC). Own unit for
// parallel compilation; see wos_kernels_native.inc.
#include "wos_kernels.h"
#include "wos_walk.cuh"

#define WOS_SINK SINK_ESTIMATE
#define WOS_BC 1
#define WOS_RND 7
#define WOS_ONE_ONLY 1
#define WOS_FN get_kernel_native_est_bc_r7
#include "wos_kernels_native.inc"
