// Kernel instantiations for MODE_REPLAY_F64 (see wos_walk.cuh).
#include "wos_kernels.h"
#include "wos_walk.cuh"

namespace wos {

// resident CTAs per SM the REPLAY_F64 kernels are built for. They are latency bound (fp64 libm
// chains, Philox4x64): at 1 CTA/SM (up to 255 registers, 100-156 used) cfg4 ran 252 ms with
// 40 % of the issue slots busy; 2 CTAs (128 registers, no spills) 158 ms; 3 (85 registers,
// up to 254 B of spills) 141 ms; 4 139 ms
#ifndef WOS_REPLAY_MINB
#define WOS_REPLAY_MINB 3
#endif

#define WOS_K(DIM, DOM, SRC, SK)                                                         \
  if (dim == DIM && dom == DOM && src == SRC && sk == SK)                                \
    return rows ? reinterpret_cast<const void*>(                                         \
                      &wos_walk_kernel<Spec<MODE_REPLAY_F64, DIM, DOM, SRC, SK, false, SINK_ROWS>, WOS_REPLAY_MINB>) \
                : reinterpret_cast<const void*>(                                         \
                      &wos_walk_kernel<Spec<MODE_REPLAY_F64, DIM, DOM, SRC, SK, false, SINK_ESTIMATE>, WOS_REPLAY_MINB>);

const void* get_kernel_replay_f64(int dim, int dom, int src, int sk, bool rows) {
  // 2D
  WOS_K(2, DOM_BALL, SRC_NONE, 0)
  WOS_K(2, DOM_BALL, SRC_CONST, 0)
  WOS_K(2, DOM_BALL, SRC_RBF2, 0)
  WOS_K(2, DOM_BALL, SRC_SINE, 0)
  WOS_K(2, DOM_BALL, SRC_GAUSS, 0)
  WOS_K(2, DOM_BOX, SRC_NONE, 0)
  WOS_K(2, DOM_BOX, SRC_CONST, 0)
  WOS_K(2, DOM_BOX, SRC_SINE, 0)
  WOS_K(2, DOM_BOX, SRC_GAUSS, 0)
  WOS_K(2, DOM_POLY, SRC_NONE, 0)
  WOS_K(2, DOM_POLY, SRC_CONST, 0)
  WOS_K(2, DOM_POLY, SRC_SINE, 0)
  WOS_K(2, DOM_POLY, SRC_GAUSS, 0)
  // polar star curves (geometry.PolarDomain; the linear family uses RBF2 + FOURIER5)
  WOS_K(2, DOM_POLAR, SRC_NONE, 0)
  WOS_K(2, DOM_POLAR, SRC_CONST, 0)
  WOS_K(2, DOM_POLAR, SRC_RBF2, 0)
  WOS_K(2, DOM_POLAR, SRC_GAUSS, 0)
  // 3D
  WOS_K(3, DOM_BALL, SRC_NONE, 0)
  WOS_K(3, DOM_BALL, SRC_CONST, 0)
  WOS_K(3, DOM_BALL, SRC_SINE, 0)
  WOS_K(3, DOM_BALL, SRC_GAUSS, 0)
  WOS_K(3, DOM_BOX, SRC_NONE, 0)
  WOS_K(3, DOM_BOX, SRC_CONST, 0)
  WOS_K(3, DOM_BOX, SRC_SINE, 0)
  WOS_K(3, DOM_BOX, SRC_GAUSS, 0)
  // closed triangle meshes (geometry.MeshDomain)
  WOS_K(3, DOM_MESH, SRC_NONE, 0)
  WOS_K(3, DOM_MESH, SRC_CONST, 0)
  WOS_K(3, DOM_MESH, SRC_GAUSS, 0)
  WOS_K(3, DOM_MESH, SRC_SCR_CONST, 0)
  WOS_K(3, DOM_MESH, SRC_SCR_VC, 0)
  // delta tracking (screened walks)
  WOS_K(3, DOM_BALL, SRC_SCR_CONST, 0)
  WOS_K(3, DOM_BALL, SRC_SCR_VC, 0)
  WOS_K(3, DOM_BOX, SRC_SCR_CONST, 0)
  WOS_K(3, DOM_BOX, SRC_SCR_VC, 0)
  return nullptr;
}

}  // namespace wos
