"""Golden fixtures for polar star-curve domains, produced by the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_polar.py

golden_polar.npz: for three linear-family instances (pde.LinearInstance: PolarDomain,
RBF2 source, FOURIER5 boundary — the paper's 2D family, pde.py:61-121) the walk rows
and the reference's (values, steps, hits) from walker.walk_poisson_values, which
routes these spec-coded problems to the compiled _kernels.walk_plain_2d with
polar_query_fast (walker.py:196-207). Case "strong" has |c1| + |c2| > 0.45, so the
reference scans the whole 4096-sample table (stride 1). Also the domain's own
boundary_query (golden-section refined) and contains on probe points.
"""

from __future__ import annotations

import os

import numpy as np

from spherewalk import pde  # reference package
from spherewalk.walker import WalkConfig, walk_poisson_values

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(31)
    insts = {
        "mild": pde.sample_linear_instance(rng, instance_key=3),
        "mild2": pde.sample_linear_instance(rng, instance_key=8),
        "strong": pde.LinearInstance(0.3, -0.25, (0.4, -0.7), ((0.1, 0.2), (-0.3, 0.05)),
                                     (0.2, -0.5, 0.3, 0.8, -0.1), instance_key=5),
    }
    out = {"cases": np.array(list(insts))}
    for name, inst in insts.items():
        dom = inst.domain
        lo, hi = dom.bounding_box()
        cand = lo + (hi - lo) * rng.random((4000, 2))
        pts = cand[dom.contains(cand)][:40]
        walks = 8
        p = np.repeat(pts, walks, axis=0)
        pid = np.repeat(np.arange(len(pts), dtype=np.int64) * 5 + 1, walks)
        tid = np.tile(np.arange(walks, dtype=np.int64) + 3, len(pts))
        sgn = np.where(rng.random(p.shape[0]) < 0.25, -1.0, 1.0)
        cfg = WalkConfig(rng_seed=99, max_steps=600)
        v, s, h = walk_poisson_values(inst.problem, p, pid, tid, sgn, cfg)
        probe = lo + (hi - lo) * rng.random((300, 2))
        d_ref, q_ref = dom.boundary_query(probe[dom.contains(probe)][:60])
        out.update({
            f"{name}_points": p, f"{name}_pid": pid, f"{name}_tid": tid, f"{name}_sgn": sgn,
            f"{name}_values": v, f"{name}_steps": s, f"{name}_hits": h,
            f"{name}_eps": np.array([cfg.resolve_eps(dom)]),
            f"{name}_shape": np.array([dom.r0, dom.c1, dom.c2, dom._stride, dom._bx.size]),
            f"{name}_bx": dom._bx, f"{name}_by": dom._by,
            f"{name}_src": np.array(inst.source_params), f"{name}_bnd": np.array(inst.b),
            f"{name}_ikey": np.array([inst.instance_key]),
            f"{name}_probe": probe, f"{name}_contains": dom.contains(probe),
            f"{name}_qprobe": probe[dom.contains(probe)][:60], f"{name}_qd": d_ref, f"{name}_qq": q_ref,
        })
        print(name, "stride", dom._stride, "walks", v.size, "mean steps", s.mean())
    np.savez(os.path.join(HERE, "golden_polar.npz"), **out)


if __name__ == "__main__":
    main()
