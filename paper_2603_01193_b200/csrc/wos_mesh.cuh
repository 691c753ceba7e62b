// Closed triangle meshes (geometry.MeshDomain, geometry.py:259-580): nearest point on
// a triangle with its feature region (closest_on_triangles, geometry.py:259-323), a
// bounding-volume-hierarchy nearest query, and the angle-weighted pseudo-normal
// inside test (geometry.py:480-520). Shared by the walk kernels (distance, exit
// point) and the interior check.
//
// Layout (built on the host, wos_capi.cu build_mesh): nodes in depth-first order,
// node k = {lo[3], hi[3]} + {right child or -1, first triangle, triangle count}; the
// left child of an inner node is k + 1. Triangles are stored in leaf order as
// {a, b, c} (9 Reals); the fp64 feature normals (face, vertices a/b/c, edges ab/bc/ca)
// follow the same order for the inside test.
#pragma once
#include <stdint.h>

namespace wos {

enum : int { MREG_A = 0, MREG_B = 1, MREG_C = 2, MREG_AB = 3, MREG_BC = 4, MREG_CA = 5, MREG_FACE = 6 };

template <class Real>
struct MeshNode {
  Real lo[3];
  Real hi[3];
  int32_t right;  // inner node: right child; leaf: -1
  int32_t first;  // leaf: first triangle (leaf order)
  int32_t count;  // leaf: triangle count
  int32_t pad;
};

template <class Real>
__device__ __forceinline__ Real mdot3(const Real* u, const Real* v) {
  return u[0] * v[0] + u[1] * v[1] + u[2] * v[2];  // explicit component sums (geometry.py:251-252)
}

// closest point on triangle (a, b, c) to p and its feature region, with the
// reference's operation order and region priority (A, B, C, AB, BC, CA, face)
template <class Real>
__device__ __forceinline__ int closest_on_triangle(const Real* p, const Real* a, const Real* b,
                                                   const Real* c, Real* q) {
  Real ab[3], ac[3], ap[3], bp[3], cp[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ab[i] = b[i] - a[i];
    ac[i] = c[i] - a[i];
    ap[i] = p[i] - a[i];
    bp[i] = p[i] - b[i];
    cp[i] = p[i] - c[i];
  }
  const Real d1 = mdot3(ab, ap), d2 = mdot3(ac, ap);
  const Real d3 = mdot3(ab, bp), d4 = mdot3(ac, bp);
  const Real d5 = mdot3(ab, cp), d6 = mdot3(ac, cp);
  const Real vc = d1 * d4 - d3 * d2;
  const Real vb = d5 * d2 - d1 * d6;
  const Real va = d3 * d6 - d5 * d4;
  const Real z = Real(0);
  if (d1 <= z && d2 <= z) {
#pragma unroll
    for (int i = 0; i < 3; ++i) q[i] = a[i];
    return MREG_A;
  }
  if (d3 >= z && d4 <= d3) {
#pragma unroll
    for (int i = 0; i < 3; ++i) q[i] = b[i];
    return MREG_B;
  }
  if (d6 >= z && d5 <= d6) {
#pragma unroll
    for (int i = 0; i < 3; ++i) q[i] = c[i];
    return MREG_C;
  }
  auto clip01 = [](Real t) { return t < Real(0) ? Real(0) : (t > Real(1) ? Real(1) : t); };
  auto sdiv = [](Real num, Real den) { return num / (den == Real(0) ? Real(1) : den); };
  if (vc <= z && d1 >= z && d3 <= z) {
    const Real t = clip01(sdiv(d1, d1 - d3));
#pragma unroll
    for (int i = 0; i < 3; ++i) q[i] = a[i] + ab[i] * t;
    return MREG_AB;
  }
  if (va <= z && (d4 - d3) >= z && (d5 - d6) >= z) {
    const Real t = clip01(sdiv(d4 - d3, (d4 - d3) + (d5 - d6)));
#pragma unroll
    for (int i = 0; i < 3; ++i) q[i] = b[i] + (c[i] - b[i]) * t;
    return MREG_BC;
  }
  if (vb <= z && d2 >= z && d6 <= z) {
    const Real t = clip01(sdiv(d2, d2 - d6));
#pragma unroll
    for (int i = 0; i < 3; ++i) q[i] = a[i] + ac[i] * t;
    return MREG_CA;
  }
  const Real denom = va + vb + vc;
  const Real v = sdiv(vb, denom), w = sdiv(vc, denom);
#pragma unroll
  for (int i = 0; i < 3; ++i) q[i] = a[i] + ab[i] * v + ac[i] * w;
  return MREG_FACE;
}

template <class Real>
__device__ __forceinline__ Real box_d2(const MeshNode<Real>& n, const Real* p) {
  Real s = Real(0);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const Real lo = n.lo[i] - p[i], hi = p[i] - n.hi[i];
    const Real d = (lo > Real(0) ? lo : Real(0)) + (hi > Real(0) ? hi : Real(0));
    s = s + d * d;
  }
  return s;
}

// Nearest triangle to p: squared distance, closest point, region and triangle (leaf
// order). Depth-first, nearer child first, pruned by the node boxes; a triangle
// replaces the best only when strictly closer.
// `hint` (or -1): a triangle to test first — a walk's previous nearest triangle is
// within 2d of the new position, so it bounds the search from the start and the
// traversal prunes almost every box.
template <class Real>
__device__ __forceinline__ Real mesh_nearest(const MeshNode<Real>* __restrict__ nodes,
                                             const Real* __restrict__ tris, const Real* p,
                                             Real* q_best, int* reg_best, int* tri_best,
                                             int hint = -1) {
  constexpr int kStack = 48;
  int stack[kStack];
  int sp = 0;
  int node = 0;
  Real best = Real(3.0e38);
  int breg = MREG_FACE, btri = 0;
  if (hint >= 0) {
    const Real* t = tris + 9 * (size_t)hint;
    breg = closest_on_triangle(p, t, t + 3, t + 6, q_best);
    Real df[3] = {q_best[0] - p[0], q_best[1] - p[1], q_best[2] - p[2]};
    best = mdot3(df, df);
    btri = hint;
  }
  while (true) {
    const MeshNode<Real> n = nodes[node];
    if (n.right < 0) {
      for (int k = 0; k < n.count; ++k) {
        const Real* t = tris + 9 * (size_t)(n.first + k);
        Real q[3];
        const int reg = closest_on_triangle(p, t, t + 3, t + 6, q);
        Real df[3] = {q[0] - p[0], q[1] - p[1], q[2] - p[2]};
        const Real d2 = mdot3(df, df);
        // strictly closer replaces; at a tie the lower leaf index wins, so the answer
        // does not depend on the hint
        if (d2 < best || (d2 == best && n.first + k < btri)) {
          best = d2;
          breg = reg;
          btri = n.first + k;
          q_best[0] = q[0];
          q_best[1] = q[1];
          q_best[2] = q[2];
        }
      }
    } else {
      const int l = node + 1, r = n.right;
      const Real dl = box_d2(nodes[l], p), dr = box_d2(nodes[r], p);
      const int nf = dl <= dr ? l : r, ff = dl <= dr ? r : l;
      const Real dn = dl <= dr ? dl : dr, dfar = dl <= dr ? dr : dl;
      // boxes at exactly the best distance are still visited (ties resolve by index)
      if (dfar <= best && sp < kStack) stack[sp++] = ff;
      if (dn <= best) {
        node = nf;
        continue;
      }
    }
    // pop the next node that can still hold a closer triangle
    bool found = false;
    while (sp > 0) {
      const int c = stack[--sp];
      if (box_d2(nodes[c], p) <= best) {
        node = c;
        found = true;
        break;
      }
    }
    if (!found) break;
  }
  *reg_best = breg;
  *tri_best = btri;
  return best;
}

}  // namespace wos
