"""Seeded fuzz over the kernel variants: dimension, domain, source, boundary, walks per
point (1, odd, chunked L > 128), antithetic pairs, single- and multi-instance sets.

Per case: the estimate sink (NATIVE) equals the two-pass moments of the ROWS sink's
walks on the same streams, and REPLAY estimates equal the oracle's reference form.
Covers the loop variants together (jump-first / test-first, amortised rounds,
deferred recording, constant-boundary kernels, chunk merge).
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

N_CASES = 40


def _case(seed):
    from paper_2603_01193_b200 import BallDomain, BoxDomain, Problem, specs, star_polygon

    rng = np.random.default_rng(seed)
    dim = int(rng.choice([2, 3]))
    dom_kind = rng.choice(["ball", "box", "poly"] if dim == 2 else ["ball", "box"])
    if dom_kind == "ball":
        dom = BallDomain(rng.uniform(-0.3, 0.3, dim), float(rng.uniform(0.5, 1.5)))
    elif dom_kind == "box":
        lo = rng.uniform(-0.5, 0.0, dim)
        dom = BoxDomain(lo, lo + rng.uniform(0.5, 1.5, dim))
    else:
        dom = star_polygon(rng.uniform(-0.08, 0.08, 4), rng.uniform(-0.08, 0.08, 4),
                           n_vertices=int(rng.choice([16, 40, 128])))
    src = rng.choice(["none", "const", "gauss"])
    bnd = rng.choice(["const", "linear"])
    n_inst = int(rng.choice([1, 1, 3]))
    probs = []
    for i in range(n_inst):
        ss = None
        if src == "const":
            ss = (specs.SRC_CONST, (float(rng.normal()),))
        elif src == "gauss":
            ss = specs.gauss_source(rng.uniform(-0.2, 0.2, dim), 0.3, float(rng.normal()))
        if bnd == "const":
            bs = (specs.BND_CONST, (float(rng.normal()),))
        else:
            bs = (specs.BND_LINEAR, tuple(rng.normal(size=dim + 1)))
        probs.append(Problem(dom, boundary_spec=bs, source_spec=ss, instance_key=int(rng.integers(0, 2**40))))
    L = int(rng.choice([1, 3, 8, 33, 128, 130, 300]))
    anti = bool(rng.random() < 0.3) and L % 2 == 0
    P = int(rng.choice([1, 7, 40]))
    lo, hi = dom.bounding_box()
    cand = lo + (hi - lo) * rng.random((60 * P + 60, dim))
    pts = cand[dom.contains(cand)][:P]
    inst = rng.integers(0, n_inst, pts.shape[0]).astype(np.int32) if n_inst > 1 else None
    ids = rng.permutation(10**6)[: pts.shape[0]].astype(np.int64)
    return probs, pts, ids, inst, L, anti, int(rng.integers(0, 2**32)), float(rng.choice([1e-3, 1e-2]))


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_estimate_sink_equals_rows(gpu, seed):
    from paper_2603_01193_b200 import WalkConfig, estimate_arrays, walk_poisson_values

    probs, pts, ids, inst, L, anti, rseed, eps = _case(seed)
    cfg = WalkConfig(eps_shell=eps, max_steps=400, antithetic=anti, rng_seed=rseed)
    t0 = 5 + seed
    mean, m2, n = estimate_arrays(probs, pts, L, cfg, inst_index=inst, point_ids=ids, traj_start=t0)
    P = pts.shape[0]
    ns = L // 2 if anti else L
    assert np.all(n == ns)
    # rows: per instance (walk_poisson_values takes one problem)
    inst_arr = np.zeros(P, np.int32) if inst is None else inst
    for k, prob in enumerate(probs):
        sel = np.flatnonzero(inst_arr == k)
        if sel.size == 0:
            continue
        rp = np.repeat(pts[sel], L, axis=0)
        rid = np.repeat(ids[sel], L)
        j = np.tile(np.arange(L), sel.size)
        tid = t0 + (2 * (j // 2) if anti else j)
        sgn = np.where(j % 2 == 1, -1.0, 1.0) if anti else np.ones(rp.shape[0])
        v, s, h = walk_poisson_values(prob, rp, rid, tid, sgn, cfg)
        v = v.reshape(sel.size, L)
        if anti:
            v = 0.5 * (v[:, 0::2] + v[:, 1::2])
        mu = v.mean(axis=1)
        np.testing.assert_allclose(mean[sel], mu, rtol=1e-11, atol=1e-13)
        np.testing.assert_allclose(m2[sel], ((v - mu[:, None]) ** 2).sum(axis=1), rtol=1e-8, atol=1e-11)


@pytest.mark.parametrize("seed", range(0, N_CASES, 3))
def test_fuzz_replay_estimate_equals_oracle(gpu, seed):
    from paper_2603_01193_b200 import WalkConfig, estimate_arrays

    probs, pts, ids, inst, L, anti, rseed, eps = _case(seed)
    cfg = WalkConfig(eps_shell=eps, max_steps=400, antithetic=anti, rng_seed=rseed, mode="replay")
    mean, m2, n = estimate_arrays(probs, pts, L, cfg, inst_index=inst, point_ids=ids, traj_start=3)
    mo, m2o, _ = O.estimate(probs, pts, L, seed=rseed, eps=eps, max_steps=400, point_ids=ids,
                            inst_index=inst, traj_start=3, antithetic=anti)
    np.testing.assert_allclose(mean, mo, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(m2, m2o, rtol=1e-6, atol=1e-12)
