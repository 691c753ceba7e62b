"""NATIVE source-free walks and the kernel paths the loop variants select.

Source-free NATIVE jumps draw one uniform (2D) or two (3D) per jump, so a Philox
block serves 4 / 2 consecutive jumps (wos_walk.cuh kPerBlock). Closed-form domains
run them in phase-locked rounds (one block per round); polygons, polar curves and
meshes redraw the block per jump and select the words. Both must give the walks the
oracle's restatement gives (oracle/wos_oracle.c walk_native_one). The estimate
sink is checked per kernel variant: single-instance constant boundary (Spec BC),
single-instance non-constant boundary (deferred recording), multi-instance.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _problem(dim, dom, bnd, ikey=5, scale=1.0):
    from paper_2603_01193_b200 import BallDomain, BoxDomain, PolygonDomain, Problem, specs, star_polygon

    if dom == "ball":
        d = BallDomain([0.1] * dim, 1.2)
    elif dom == "box":
        d = BoxDomain([0.0] * dim, [1.0] + [0.8] * (dim - 1))
    else:
        d = star_polygon([0.05, -0.03, 0.02, 0.04], [0.01, 0.06, -0.05, 0.02], n_vertices=48)
        assert isinstance(d, PolygonDomain)
    if bnd == "const":
        bs = (specs.BND_CONST, (0.75 * scale,))
    else:
        bs = (specs.BND_LINEAR, tuple(scale * c for c in [0.3, -0.7, 0.2][:dim]) + (0.1,))
    return Problem(d, boundary_spec=bs, instance_key=ikey)


def _points(dom, dim, n, seed=0):
    rng = np.random.default_rng(seed)
    lo, hi = dom.bounding_box()
    cand = lo + (hi - lo) * rng.random((8 * n, dim))
    return cand[dom.contains(cand)][:n]


CASES = [(2, "ball"), (2, "box"), (3, "ball"), (3, "box"), (2, "poly")]


@pytest.mark.parametrize("dim,dom", CASES)
@pytest.mark.parametrize("bnd", ["const", "linear"])
def test_sourcefree_rows_match_native_oracle(gpu, dim, dom, bnd):
    from paper_2603_01193_b200 import WalkConfig, walk_poisson_values

    prob = _problem(dim, dom, bnd)
    P, T = 48, 16
    pts = np.repeat(_points(prob.domain, dim, P), T, axis=0)
    pid = np.repeat(np.arange(P) * 7 + 3, T)
    tid = np.tile(np.arange(T) + 1000, P)
    sgn = np.ones(pts.shape[0])
    cfg = WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=11)
    v, s, h = walk_poisson_values(prob, pts, pid, tid, sgn, cfg)
    vo, so, ho = O.walk_rows(prob, pts, pid, tid, sgn, seed=11, eps=1e-3, max_steps=1000, native=True)
    same = s == so
    assert same.mean() >= 0.99, f"identical steps {same.mean():.4%}"
    assert np.array_equal(h[same], ho[same])
    err = np.abs(v[same] - vo[same]) / np.maximum(np.abs(vo[same]), 1.0)
    assert np.quantile(err, 0.99) < 1e-4


@pytest.mark.parametrize("dim,dom", CASES)
@pytest.mark.parametrize("bnd", ["const", "linear"])
def test_sourcefree_estimate_equals_rows(gpu, dim, dom, bnd):
    """Estimate sink (single-instance kernels: the BC variant for the constant
    boundary, deferred recording for the linear one; L > 128: chunks + Chan merge)
    against the per-point two-pass moments of the ROWS sink's walks (same streams)."""
    from paper_2603_01193_b200 import WalkConfig, estimate_arrays, walk_poisson_values

    prob = _problem(dim, dom, bnd)
    P, L, t0 = 40, 200, 17
    pts = _points(prob.domain, dim, P, seed=1)
    cfg = WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=4)
    mean, m2, n = estimate_arrays([prob], pts, L, cfg, traj_start=t0)
    assert np.all(n == L)
    v, _, _ = walk_poisson_values(prob, np.repeat(pts, L, axis=0), np.repeat(np.arange(P), L),
                                  np.tile(np.arange(L) + t0, P), np.ones(P * L), cfg)
    v = v.reshape(P, L)
    mu = v.mean(axis=1)
    np.testing.assert_allclose(mean, mu, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(m2, ((v - mu[:, None]) ** 2).sum(axis=1), rtol=1e-9, atol=1e-12)
    if bnd == "const":
        # every walk ends at g = 0.75: the mean is exact and the spread vanishes
        np.testing.assert_allclose(mean, 0.75, rtol=1e-7)


@pytest.mark.parametrize("dim,dom", CASES)
@pytest.mark.parametrize("bnd", ["const", "linear"])
def test_sourcefree_multi_instance_equals_single(gpu, dim, dom, bnd):
    """Multi-instance launches (no Spec BC, runtime boundary switch) give the same
    estimates as one launch per instance."""
    from paper_2603_01193_b200 import WalkConfig, estimate_arrays

    probs = [_problem(dim, dom, bnd, ikey=3), _problem(dim, dom, bnd, ikey=9, scale=-0.5)]
    pts = _points(probs[0].domain, dim, 40, seed=2)
    inst = np.arange(40) % 2
    cfg = WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=8)
    mean, m2, _ = estimate_arrays(probs, pts, 64, cfg, inst_index=inst)
    for k in (0, 1):
        sel = inst == k
        m1, q1, _ = estimate_arrays([probs[k]], pts[sel], 64, cfg, point_ids=np.flatnonzero(sel))
        np.testing.assert_allclose(mean[sel], m1, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("dim,dom", [(2, "ball"), (3, "box"), (2, "poly")])
def test_deferred_recording_is_tuning_invariant(gpu, dim, dom):
    """Deferred recording changes when a finished walk is recorded, never its value or
    its place in the per-point reduction: estimates are bitwise identical for any
    refill thresholds and launch shape."""
    from paper_2603_01193_b200 import WalkConfig, engine, estimate_arrays

    prob = _problem(dim, dom, "linear")
    pts = _points(prob.domain, dim, 64, seed=5)
    cfg = WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=2)
    ref = estimate_arrays([prob], pts, 300, cfg)
    ctx = engine.get_context(0)
    try:
        for rm, rmd, bps in ((5, 1, 0), (3, 32, 1), (17, 7, 2)):
            ctx.set_tuning(refill_min=rm, blocks_per_sm=bps, refill_min_deferred=rmd)
            got = estimate_arrays([prob], pts, 300, cfg)
            assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    finally:
        ctx.set_tuning()


def _exit_ring_problem(dom, bnd):
    from paper_2603_01193_b200 import BallDomain, BoxDomain, Problem, specs

    d = BallDomain([0.1, -0.2], 1.2) if dom == "ball" else BoxDomain([0.0, -0.1], [1.0, 0.7])
    if bnd == "fourier":
        M = 8
        rng = np.random.default_rng(3)
        bs = (specs.BND_FOURIER, (float(M), 0.2) + tuple(rng.normal(size=2 * M) / (1 + np.arange(2 * M) % M)))
    else:
        bs = (specs.BND_LINEAR, (0.3, -0.7, 0.1))
    return Problem(d, boundary_spec=bs, instance_key=21)


@pytest.mark.parametrize("dom,bnd", [("ball", "fourier"), ("ball", "linear"), ("box", "linear")])
@pytest.mark.parametrize("L", [4, 64, 300])
@pytest.mark.parametrize("anti", [False, True])
@pytest.mark.parametrize("max_steps", [3, 1000])
def test_exit_ring_estimate_equals_rows(gpu, dom, bnd, L, anti, max_steps):
    """Exit-ring kernels (single-instance source-free 2D, non-constant boundary: a
    finished walk leaves its exit position in the ring and g(projection) is evaluated
    when its unit retires; branch-free rounds) against the ROWS sink's walks of the same
    streams: whole-point units (L = 4: 32 points per unit, L = 64: the cached-point
    refill), chunks (L = 300), antithetic pairs, walks cut at max_steps, and start
    points inside the shell (recorded with 0 steps)."""
    from paper_2603_01193_b200 import WalkConfig, estimate_arrays, walk_poisson_values

    prob = _exit_ring_problem(dom, bnd)
    P, t0 = 70, 6
    pts = _points(prob.domain, 2, P - 6, seed=7)
    # six more points inside the shell (distance < eps from the boundary)
    if dom == "ball":
        th = np.linspace(0.3, 5.5, 6)
        shell = np.array([0.1, -0.2]) + (1.2 - 4e-4) * np.stack([np.cos(th), np.sin(th)], axis=1)
    else:
        shell = np.stack([np.linspace(0.1, 0.9, 6), np.full(6, 0.7 - 3e-4)], axis=1)
    pts = np.concatenate([pts[:30], shell, pts[30:]])
    cfg = WalkConfig(eps_shell=1e-3, max_steps=max_steps, rng_seed=4, antithetic=anti)
    mean, m2, n = estimate_arrays([prob], pts, L, cfg, traj_start=t0)
    j = np.arange(L)
    tid = t0 + (2 * (j >> 1) if anti else j)
    sgn = np.where(anti & (j % 2 == 1), -1.0, 1.0)
    rows_cfg = WalkConfig(eps_shell=1e-3, max_steps=max_steps, rng_seed=4)
    v, s, _ = walk_poisson_values(prob, np.repeat(pts, L, axis=0), np.repeat(np.arange(P), L),
                                  np.tile(tid, P), np.tile(sgn, P), rows_cfg)
    v = v.reshape(P, L)
    if anti:
        v = 0.5 * (v[:, 0::2] + v[:, 1::2])
    assert np.all(n == v.shape[1])
    mu = v.mean(axis=1)
    np.testing.assert_allclose(mean, mu, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(m2, ((v - mu[:, None]) ** 2).sum(axis=1), rtol=1e-9, atol=1e-12)
    s = s.reshape(P, L)
    assert np.all(s[30:36] == 0) and s.max() <= max_steps
    if max_steps == 3:
        assert (s == 3).mean() > 0.3  # most walks are cut


@pytest.mark.parametrize("anti,rounds", [(False, 10), (True, 10), (False, 7)])
def test_exit_ring_two_slot_loop_equals_one_slot_and_rows(gpu, anti, rounds):
    """Exit-ring launches with at least 16 units per warp run two walks per lane
    (wos_walk.cuh WOS_EXIT_ILP2); smaller ones keep one. With one CTA per SM a 20,000
    point estimate is above the threshold, with the default grid below it: both must
    give the same bits, and the ROWS sink's walks of the same streams the same moments."""
    from paper_2603_01193_b200 import WalkConfig, engine, estimate_arrays, walk_poisson_values

    prob = _exit_ring_problem("ball", "fourier")
    P, L, t0 = 20000, 32, 3
    pts = _points(prob.domain, 2, P, seed=11)
    assert pts.shape[0] == P
    # (rounds = 7: the single-instance estimate kernels compiled for the opt-in stream)
    cfg = WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=9, antithetic=anti, philox_rounds=rounds)
    ctx = engine.get_context(0)
    one = estimate_arrays([prob], pts, L, cfg, traj_start=t0)
    try:
        ctx.set_tuning(blocks_per_sm=1)
        two = estimate_arrays([prob], pts, L, cfg, traj_start=t0)
    finally:
        ctx.set_tuning()
    assert np.array_equal(one[0], two[0]) and np.array_equal(one[1], two[1])
    sel = np.arange(0, P, 41)
    j = np.arange(L)
    tid = t0 + (2 * (j >> 1) if anti else j)
    sgn = np.where(anti & (j % 2 == 1), -1.0, 1.0)
    rows_cfg = WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=9, philox_rounds=rounds)
    v, _, _ = walk_poisson_values(prob, np.repeat(pts[sel], L, axis=0), np.repeat(sel, L),
                                  np.tile(tid, sel.size), np.tile(sgn, sel.size), rows_cfg)
    v = v.reshape(sel.size, L)
    if anti:
        v = 0.5 * (v[:, 0::2] + v[:, 1::2])
    mu = v.mean(axis=1)
    np.testing.assert_allclose(two[0][sel], mu, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(two[1][sel], ((v - mu[:, None]) ** 2).sum(axis=1), rtol=1e-9, atol=1e-12)
