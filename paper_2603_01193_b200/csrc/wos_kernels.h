// Kernel registry: one lookup per numeric mode (each compiled in its own unit).
#pragma once
#include <stdint.h>

namespace wos {
// Returns the __global__ entry for (dim, domain, source, sine order) or nullptr.
// rows = walk_poisson_values sink (per-walk outputs) instead of the per-point estimate
const void* get_kernel_replay_f64(int dim, int dom, int src, int sk, bool rows);
const void* get_kernel_replay_f32(int dim, int dom, int src, int sk, bool rows);
// one = single-instance launch (instance row + Philox keys in the kernel parameters);
// bnd_const = the boundary value is a constant (single-instance estimate kernels
// then drop the deferred-recording path); rounds = Philox4x32 rounds (10 or 7: the
// single-instance estimate kernels are compiled for each); *warps = the kernel's warps
// per CTA
const void* get_kernel_native(int dim, int dom, int src, int sk, bool one, bool rows, bool bnd_const,
                              int rounds, int* warps);
// fast-math primitives of the NATIVE kernels on given arguments (returns a cudaError_t)
int launch_fastmath_probe(int64_t n, const float* x, float* s, float* c, float* q, float* e, void* stream);
}  // namespace wos

// host helpers shared by the C-ABI units (defined in wos_capi.cu)
struct wos_context;
int wos_fail(int code, const char* fmt, ...);     // sets wos_last_error(), returns code
int wos_context_device(const wos_context* ctx);  // CUDA device ordinal of ctx
void wos_context_count_launch(wos_context* ctx); // one more kernel launched (wos_context_counters)
