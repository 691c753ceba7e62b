// Kernel registry: one lookup per numeric mode (each compiled in its own unit).
#pragma once

namespace wos {
// Returns the __global__ entry for (dim, domain, source, sine order) or nullptr.
const void* get_kernel_replay_f64(int dim, int dom, int src, int sk);
const void* get_kernel_replay_f32(int dim, int dom, int src, int sk);
// one = single-instance launch (instance row + Philox keys in the kernel parameters)
const void* get_kernel_native(int dim, int dom, int src, int sk, bool one);
}  // namespace wos
