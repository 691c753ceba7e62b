"""Golden fixtures for delta tracking, produced by the REFERENCE's screened walker.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_screened.py

golden_screened.npz holds, per case, the spec record the product encodes, the
walk rows (points, point/traj ids, signs), sigma_bar and eps, and the reference's
(values, steps, hits) from walker.walk_screened_values (walker.py:322-357):

  const_ball   const_coeffs (0.7, 0.5, 1.0) on the unit ball: the compiled
               _kernels.walk_screened_ball3 path
  dead_ball    const_coeffs (2.0, None, 1.0) with sigma_bar = 2 and sqrt_alpha = 2:
               throughput dies at the first volume event (early exit, hit = 1)
  vc_ball      pde.VcInstance on the unit ball: the generic path
               (walker._screened_generic) with the family's closed-form callables
  vc_box       pde.VcInstance on the unit cube (a duck-typed box domain)
  violation    vc_ball with sigma_bar below the supremum of sigma': the reference
               raises MajorantViolationError (recorded as a flag)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from spherewalk import pde  # noqa: E402  (reference package)
from spherewalk.geometry import BallDomain  # noqa: E402
from spherewalk.walker import (  # noqa: E402
    MajorantViolationError,
    ScreenedProblem,
    WalkConfig,
    walk_screened_values,
)

from ref_adapters import RefBox  # noqa: E402

SRC_SCREENED_CONST, SRC_SCREENED_VC = 5, 6
BND_CONST, BND_VC = 0, 6
DOM_BALL, DOM_BOX = 0, 2


def rows(rng, pts, walks):
    P = pts.shape[0]
    p = np.repeat(pts, walks, axis=0)
    pid = np.repeat(np.arange(P, dtype=np.int64) * 7 + 3, walks)
    tid = np.tile(np.arange(walks, dtype=np.int64) + 11, P)
    sgn = np.where(rng.random(P * walks) < 0.25, -1.0, 1.0)
    return p, pid, tid, sgn


def ball_points(rng, n, r=0.9):
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1)[:, None]
    return v * (r * rng.random(n) ** (1.0 / 3.0))[:, None]


def vc_majorant(phi, a_min, a_max, pts):
    sup = float(pde._vc_sigma_prime(phi, a_min, a_max, pts).max())
    return max(1.1 * sup, 0.01)


def main():
    rng = np.random.default_rng(77)
    out = {}
    ball = BallDomain([0.0, 0.0, 0.0], 1.0)
    box = RefBox([0.0, 0.0, 0.0], [1.0, 1.0, 1.0])
    cases = []

    sp = ScreenedProblem(ball, None, None, const_coeffs=(0.7, 0.5, 1.0), instance_key=4)
    cases.append(("const_ball", sp, 2.0,
                  (3, DOM_BALL, (0.0, 0.0, 0.0, 1.0), SRC_SCREENED_CONST, (0.7, 0.5, 1.0, 1.0),
                   BND_CONST, (1.0,), 4), ball_points(rng, 48)))
    sp = ScreenedProblem(ball, None, None, sqrt_alpha=lambda p: np.full(p.shape[0], 2.0),
                         const_coeffs=(2.0, None, 1.0))
    cases.append(("dead_ball", sp, 2.0,
                  (3, DOM_BALL, (0.0, 0.0, 0.0, 1.0), SRC_SCREENED_CONST, (2.0, 0.0, 0.0, 2.0),
                   BND_CONST, (1.0,), 0), ball_points(rng, 32)))
    phi, a_min, a_max = 0.83, 0.21, 1.17
    sb = vc_majorant(phi, a_min, a_max, ball_points(rng, 20000, 1.0))
    inst = pde.VcInstance(phi, a_min, a_max, ball, sb, instance_key=9)
    cases.append(("vc_ball", inst.problem, sb,
                  (3, DOM_BALL, (0.0, 0.0, 0.0, 1.0), SRC_SCREENED_VC, (phi, a_min, a_max),
                   BND_VC, (phi,), 9), ball_points(rng, 48)))
    phi2, a2, b2 = 1.31, 0.12, 0.93
    sb2 = vc_majorant(phi2, a2, b2, rng.random((20000, 3)))
    inst2 = pde.VcInstance(phi2, a2, b2, box, sb2, instance_key=2)
    cases.append(("vc_box", inst2.problem, sb2,
                  (3, DOM_BOX, (0.0, 0.0, 0.0, 1.0, 1.0, 1.0), SRC_SCREENED_VC, (phi2, a2, b2),
                   BND_VC, (phi2,), 2), 0.05 + 0.9 * rng.random((40, 3))))

    names = []
    for name, prob, sigma_bar, rec, pts in cases:
        p, pid, tid, sgn = rows(rng, pts, 8)
        cfg = WalkConfig(sigma_bar=sigma_bar, rng_seed=1234, max_steps=400)
        eps = cfg.resolve_eps(prob.domain)
        v, s, h = walk_screened_values(prob, p, pid, tid, sgn, cfg)
        names.append(name)
        out[f"{name}_points"] = p
        out[f"{name}_pid"] = pid
        out[f"{name}_tid"] = tid
        out[f"{name}_sgn"] = sgn
        out[f"{name}_values"] = v
        out[f"{name}_steps"] = s
        out[f"{name}_hits"] = h
        out[f"{name}_cfg"] = np.array([sigma_bar, eps, 1234, 400], dtype=np.float64)
        dim, dk, dp, sk, spar, bk, bp, ikey = rec
        out[f"{name}_head"] = np.array([dim, dk, sk, bk, ikey], dtype=np.int64)
        out[f"{name}_dom"] = np.asarray(dp, np.float64)
        out[f"{name}_src"] = np.asarray(spar, np.float64)
        out[f"{name}_bnd"] = np.asarray(bp, np.float64)
        print(name, "walks", v.size, "mean steps", s.mean(), "hits", h.mean())
    # majorant violation: the same family with sigma_bar below sup sigma'
    viol = 0
    try:
        p, pid, tid, sgn = rows(rng, ball_points(rng, 16), 8)
        walk_screened_values(inst.problem, p, pid, tid, sgn,
                             WalkConfig(sigma_bar=0.2 * sb, rng_seed=5, max_steps=400))
    except MajorantViolationError:
        viol = 1
    out["violation_points"] = p
    out["violation_pid"] = pid
    out["violation_tid"] = tid
    out["violation_sgn"] = sgn
    out["violation_raised"] = np.array([viol])
    out["violation_sigma_bar"] = np.array([0.2 * sb])
    out["cases"] = np.array(names)
    np.savez(os.path.join(HERE, "golden_screened.npz"), **out)
    print("violation raised:", viol)


if __name__ == "__main__":
    main()
