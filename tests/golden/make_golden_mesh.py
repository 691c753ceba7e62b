"""Golden fixtures for closed triangle meshes, produced by the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_mesh.py

golden_mesh.npz: reference MeshDomain objects (geometry.make_icosphere with 2 and 4
subdivisions — brute-force and BVH nearest queries, geometry.py:470-497 — and
make_box_mesh), their vertices/faces, boundary_query and contains on probe points,
and walker.walk_poisson_values rows (generic path, walker.py:257-314) for a Poisson
problem with f = -1 and g = x + 2y - z + 0.5; plus delta-tracking rows of the
varying-coefficient family on the subdivision-2 sphere (walker._screened_generic).
"""

from __future__ import annotations

import os

import numpy as np

from spherewalk import _kernels, pde  # reference package
from spherewalk.geometry import make_box_mesh, make_icosphere
from spherewalk.walker import Problem, WalkConfig, walk_poisson_values, walk_screened_values

HERE = os.path.dirname(os.path.abspath(__file__))


def g_lin(q):
    q = np.asarray(q)
    return q[..., 0] + 2.0 * q[..., 1] - q[..., 2] + 0.5


def f_m1(p):
    return np.full(np.asarray(p).shape[0], -1.0)


def ball_points(rng, n, r):
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1)[:, None]
    return v * (r * rng.random(n) ** (1.0 / 3.0))[:, None]


def main():
    rng = np.random.default_rng(123)
    meshes = {"ico2": make_icosphere(2), "ico4": make_icosphere(4), "box": make_box_mesh(half_extent=0.7)}
    out = {"cases": np.array(list(meshes))}
    for name, dom in meshes.items():
        probe = ball_points(rng, 200, 1.3 if name != "box" else 1.2)
        d, q = dom.boundary_query(probe)
        prob = Problem(dom, boundary=g_lin, source=f_m1, instance_key=6,
                       boundary_spec=(_kernels.BND_LINEAR, (1.0, 2.0, -1.0, 0.5)),
                       source_spec=(_kernels.SRC_CONST, (-1.0,)))
        inside = dom.contains(probe)
        pts = probe[inside][:32]
        walks = 6
        p = np.repeat(pts, walks, axis=0)
        pid = np.repeat(np.arange(len(pts), dtype=np.int64) * 3 + 2, walks)
        tid = np.tile(np.arange(walks, dtype=np.int64) + 5, len(pts))
        sgn = np.where(rng.random(p.shape[0]) < 0.25, -1.0, 1.0)
        cfg = WalkConfig(rng_seed=17, max_steps=500)
        v, s, h = walk_poisson_values(prob, p, pid, tid, sgn, cfg)
        out.update({
            f"{name}_vertices": dom.vertices, f"{name}_faces": dom.faces,
            f"{name}_probe": probe, f"{name}_qd": d, f"{name}_qq": q, f"{name}_contains": inside,
            f"{name}_points": p, f"{name}_pid": pid, f"{name}_tid": tid, f"{name}_sgn": sgn,
            f"{name}_values": v, f"{name}_steps": s, f"{name}_hits": h,
            f"{name}_eps": np.array([cfg.resolve_eps(dom)]),
        })
        print(name, dom.faces.shape[0], "faces; walks", v.size, "mean steps", s.mean())
    # delta tracking on the coarse sphere
    dom = meshes["ico2"]
    phi, a_min, a_max = 0.91, 0.18, 1.05
    probes = ball_points(rng, 20000, 0.95)
    sb = max(1.1 * float(pde._vc_sigma_prime(phi, a_min, a_max, probes).max()), 0.01)
    inst = pde.VcInstance(phi, a_min, a_max, dom, sb, instance_key=4)
    pts = ball_points(rng, 24, 0.8)
    p = np.repeat(pts, 6, axis=0)
    pid = np.repeat(np.arange(24, dtype=np.int64), 6)
    tid = np.tile(np.arange(6, dtype=np.int64), 24)
    sgn = np.ones(p.shape[0])
    cfg = WalkConfig(rng_seed=21, max_steps=400, sigma_bar=sb)
    v, s, h = walk_screened_values(inst.problem, p, pid, tid, sgn, cfg)
    out.update({"vc_points": p, "vc_pid": pid, "vc_tid": tid, "vc_sgn": sgn, "vc_values": v,
                "vc_steps": s, "vc_hits": h, "vc_cfg": np.array([sb, cfg.resolve_eps(dom)]),
                "vc_params": np.array([phi, a_min, a_max])})
    print("vc on ico2: walks", v.size, "mean steps", s.mean())
    np.savez(os.path.join(HERE, "golden_mesh.npz"), **out)


if __name__ == "__main__":
    main()
