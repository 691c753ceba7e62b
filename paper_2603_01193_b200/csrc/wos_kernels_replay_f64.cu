// Kernel instantiations for MODE_REPLAY_F64 (see wos_walk.cuh).
#include "wos_kernels.h"
#include "wos_walk.cuh"

namespace wos {

#define WOS_K(DIM, DOM, SRC, SK)                                                         \
  if (dim == DIM && dom == DOM && src == SRC && sk == SK)                                \
    return rows ? reinterpret_cast<const void*>(                                         \
                      &wos_walk_kernel<Spec<MODE_REPLAY_F64, DIM, DOM, SRC, SK, false, SINK_ROWS>, 1>) \
                : reinterpret_cast<const void*>(                                         \
                      &wos_walk_kernel<Spec<MODE_REPLAY_F64, DIM, DOM, SRC, SK, false, SINK_ESTIMATE>, 1>);

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
