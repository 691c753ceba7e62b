"""Delta-tracking (screened) walks on the GPU.

REPLAY rows follow the reference walk for walk (golden_screened.npz from
walker.walk_screened_values); NATIVE rows follow the native oracle; both forms
reproduce the closed-form centre values of constant screened problems
(test_walker.py:262-313), the reduction to the plain walker, the manufactured
solution of the varying-coefficient family, and the reference's errors.
"""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O
from test_oracle_screened import case_record

pytestmark = pytest.mark.gpu

CASES = ["const_ball", "dead_ball", "vc_ball", "vc_box"]


def _problem(z, name):
    from paper_2603_01193_b200 import BallDomain, BoxDomain, ScreenedProblem

    dim, dk, dp, sk, sp, bk, bp, ikey = case_record(z, name)
    dom = BallDomain(dp[:3], dp[3]) if dk == 0 else BoxDomain(dp[:3], dp[3:])
    if sk == 6:
        return ScreenedProblem(dom, vc_params=sp, instance_key=ikey)
    fprime = sp[1] if sp[2] else None
    return ScreenedProblem(dom, sqrt_alpha=sp[3], const_coeffs=(sp[0], fprime, bp[0]),
                           instance_key=ikey)


def _cfg(z, name, mode):
    from paper_2603_01193_b200 import WalkConfig

    sb, eps, seed, ms = z[f"{name}_cfg"]
    return WalkConfig(eps_shell=eps, max_steps=int(ms), sigma_bar=sb, rng_seed=int(seed), mode=mode)


@pytest.mark.parametrize("name", CASES)
def test_replay_rows_match_reference(gpu, name):
    from paper_2603_01193_b200 import walk_screened_values

    z = load_golden("golden_screened.npz")
    v, s, h = walk_screened_values(_problem(z, name), z[f"{name}_points"], z[f"{name}_pid"],
                                   z[f"{name}_tid"], z[f"{name}_sgn"], _cfg(z, name, "replay"))
    same = s == z[f"{name}_steps"]
    assert same.mean() >= 0.995, f"identical steps {same.mean():.3%}"
    assert np.array_equal(h[same], z[f"{name}_hits"][same])
    ref = z[f"{name}_values"]
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref**2)))
    assert np.max(np.abs(v[same] - ref[same]) / scale[same]) < 1e-9


@pytest.mark.parametrize("name", CASES)
def test_native_rows_match_native_oracle(gpu, name):
    from paper_2603_01193_b200 import walk_screened_values

    z = load_golden("golden_screened.npz")
    sb, eps, seed, ms = z[f"{name}_cfg"]
    args = (z[f"{name}_points"], z[f"{name}_pid"], z[f"{name}_tid"], z[f"{name}_sgn"])
    v, s, h = walk_screened_values(_problem(z, name), *args, _cfg(z, name, "native"))
    vo, so, ho = O.walk_rows(case_record(z, name), *args, seed=int(seed), eps=eps,
                             max_steps=int(ms), native=True, sigma_bar=sb)
    same = s == so
    assert same.mean() >= 0.97, f"identical steps {same.mean():.3%}"
    rms = np.sqrt(np.mean(vo**2)) + 1e-30
    err = np.abs(v[same] - vo[same]) / np.maximum(np.abs(vo[same]), rms)
    assert np.quantile(err, 0.99) < 1e-3


def screened_center_value(R, s_prime, f_prime, g_prime):
    """Centre value of Laplacian U - s'U = -f' on a ball, U = g' (test_walker.py:262-267)."""
    if s_prime == 0.0:
        return g_prime + f_prime * R * R / 6.0
    q = math.sqrt(s_prime) * R
    return f_prime / s_prime + (g_prime - f_prime / s_prime) * q / math.sinh(q)


@pytest.mark.parametrize("mode", ["replay", "native"])
@pytest.mark.parametrize("coeffs,sigma_bar", [((1.0, None, 1.0), 1.0), ((0.7, 0.5, 1.0), 2.0),
                                              ((0.0, 2.0, 0.5), 0.5)])
def test_constant_centre_values(gpu, mode, coeffs, sigma_bar):
    from paper_2603_01193_b200 import BallDomain, ScreenedProblem, WalkConfig, estimate

    sp = ScreenedProblem(BallDomain([0.0, 0.0, 0.0], 1.0), const_coeffs=coeffs)
    L = 200_000
    (e,) = estimate(sp, [[0.0, 0.0, 0.0]], L, WalkConfig(sigma_bar=sigma_bar, rng_seed=41, mode=mode))
    want = screened_center_value(1.0, coeffs[0], coeffs[1] or 0.0, coeffs[2])
    assert e.n_samples == L
    assert abs(e.mean - want) < 4.0 * e.std_error, (e.mean, want, e.std_error)


@pytest.mark.parametrize("mode", ["replay", "native"])
def test_throughput_dies_at_full_absorption(gpu, mode):
    """sigma' == sigma_bar: every sample is exactly 0 or g' (test_walker.py:278-284)."""
    from paper_2603_01193_b200 import BallDomain, ScreenedProblem, WalkConfig, walk_screened_values

    sp = ScreenedProblem(BallDomain([0.0, 0.0, 0.0], 1.0), const_coeffs=(2.0, None, 1.0))
    n = 5000
    v, s, h = walk_screened_values(sp, np.tile([0.2, 0.0, 0.0], (n, 1)), np.zeros(n, np.int64),
                                   np.arange(n), np.ones(n), WalkConfig(sigma_bar=2.0, rng_seed=43,
                                                                        mode=mode))
    assert set(np.unique(v)) <= {0.0, 1.0}
    assert 0.0 in v and 1.0 in v
    assert h.all()


@pytest.mark.parametrize("mode", ["replay", "native"])
def test_reduction_to_plain_walker(gpu, mode):
    """alpha = 1, sigma = 0: delta tracking with f' = -f equals the plain walker (test_walker.py:286-296)."""
    from paper_2603_01193_b200 import (BallDomain, Problem, ScreenedProblem, WalkConfig, estimate,
                                       specs)

    ball = BallDomain([0.0, 0.0, 0.0], 1.0)
    sp = ScreenedProblem(ball, const_coeffs=(0.0, -1.0, 0.0))
    plain = Problem(ball, boundary_spec=specs.const_boundary(0.0), source_spec=specs.const_source(1.0))
    (ed,) = estimate(sp, [[0.1, 0.0, 0.2]], 200_000, WalkConfig(sigma_bar=0.5, rng_seed=47, mode=mode))
    (ep,) = estimate(plain, [[0.1, 0.0, 0.2]], 200_000, WalkConfig(rng_seed=48, mode=mode))
    assert abs(ed.mean - ep.mean) < 4.0 * math.hypot(ed.std_error, ep.std_error)


@pytest.mark.parametrize("mode", ["replay", "native"])
@pytest.mark.parametrize("name", ["vc_ball", "vc_box"])
def test_vc_family_manufactured_solution(gpu, mode, name):
    """The family solves div(alpha grad u) - sigma u = -f with known u (pde.py:154-173)."""
    from paper_2603_01193_b200 import estimate_arrays

    z = load_golden("golden_screened.npz")
    prob = _problem(z, name)
    pts = z[f"{name}_points"][::8][:12]
    L = 8192 if mode == "native" else 2048
    mean, m2, n = estimate_arrays([prob], pts, L, _cfg(z, name, mode))
    se = np.sqrt(m2 / (n - 1) / n)
    phi = prob.vc_params[0]
    u = O_vc_solution(phi, pts)
    zsc = (mean - u) / se
    assert np.max(np.abs(zsc)) < 4.5, zsc
    assert np.sqrt(np.mean(zsc**2)) < 1.6


def O_vc_solution(phi, x):
    # pde._vc_solution (pde.py:154-173), the manufactured exact solution
    p = math.pi * phi
    return (np.sin(p * x[:, 0]) * np.cos(2 * p * x[:, 1])
            + (1 - np.cos(p * x[:, 0])) * (1 - np.sin(2 * p * x[:, 1])) + np.sin(3 * p * x[:, 2]) ** 2)


@pytest.mark.parametrize("mode", ["replay", "native"])
def test_majorant_violation(gpu, mode):
    from paper_2603_01193_b200 import (BallDomain, MajorantViolationError, ScreenedProblem,
                                       WalkConfig, estimate, walk_screened_values)

    ball = BallDomain([0.0, 0.0, 0.0], 1.0)
    with pytest.raises(MajorantViolationError):  # test_walker.py:315-318 (const, up front)
        walk_screened_values(ScreenedProblem(ball, const_coeffs=(3.0, None, 1.0)),
                             [[0.0, 0.0, 0.0]], [0], [0], [1.0], WalkConfig(sigma_bar=1.0, mode=mode))
    z = load_golden("golden_screened.npz")
    prob = _problem(z, "vc_ball")
    cfg = WalkConfig(sigma_bar=float(z["violation_sigma_bar"][0]), rng_seed=5, max_steps=400,
                     mode=mode)
    with pytest.raises(MajorantViolationError):  # discovered at volume events (walker.py:409-413)
        walk_screened_values(prob, z["violation_points"], z["violation_pid"], z["violation_tid"],
                             z["violation_sgn"], cfg)
    with pytest.raises(MajorantViolationError):
        estimate(prob, z["violation_points"][:4], 64, cfg)
    # the context is clean afterwards
    v, _, _ = walk_screened_values(prob, z["vc_ball_points"][:8], np.arange(8), np.arange(8),
                                   np.ones(8), _cfg(z, "vc_ball", mode))
    assert np.isfinite(v).all()


def test_sigma_bar_required(gpu):
    from paper_2603_01193_b200 import (BallDomain, ScreenedProblem, WalkConfig, estimate,
                                       walk_screened_delta)

    sp = ScreenedProblem(BallDomain([0.0, 0.0, 0.0], 1.0), const_coeffs=(0.0, None, 1.0))
    with pytest.raises(ValueError):
        walk_screened_delta(sp, [0.0, 0.0, 0.0], WalkConfig())
    with pytest.raises(ValueError):
        estimate(sp, [[0.0, 0.0, 0.0]], 4, WalkConfig())


@pytest.mark.parametrize("mode", ["replay", "native"])
def test_sqrt_alpha_rescales_start(gpu, mode):
    """test_walker.py:328-336: values are divided by sqrt(alpha) at the start point."""
    from paper_2603_01193_b200 import BallDomain, ScreenedProblem, WalkConfig, walk_screened_values

    sp = ScreenedProblem(BallDomain([0.0, 0.0, 0.0], 1.0), sqrt_alpha=2.0,
                         const_coeffs=(0.0, None, 1.0))
    v, _, _ = walk_screened_values(sp, np.tile([0.1, 0.0, 0.0], (100, 1)), np.zeros(100, np.int64),
                                   np.arange(100), np.ones(100), WalkConfig(sigma_bar=0.5, rng_seed=59,
                                                                            mode=mode))
    assert np.all(v == 0.5)


def test_screened_estimate_is_layout_invariant(gpu):
    from paper_2603_01193_b200 import estimate_arrays

    z = load_golden("golden_screened.npz")
    prob = _problem(z, "vc_ball")
    pts = z["vc_ball_points"][::8]
    cfg = _cfg(z, "vc_ball", "native")
    a = estimate_arrays([prob], pts, 300, cfg, point_ids=np.arange(len(pts)))
    perm = np.random.default_rng(0).permutation(len(pts))
    b = estimate_arrays([prob], pts[perm], 300, cfg, point_ids=perm)
    assert np.array_equal(a[0][perm], b[0]) and np.array_equal(a[1][perm], b[1])


def test_screened_label_epochs(gpu):
    """The label cache drives delta tracking too; a violating epoch leaves it untouched."""
    from paper_2603_01193_b200 import EstimateCache, MajorantViolationError, WalkConfig

    z = load_golden("golden_screened.npz")
    prob = _problem(z, "vc_ball")
    pts = z["vc_ball_points"][::8]
    cache = EstimateCache()
    t1 = cache.label_epoch(prob, pts, 64, _cfg(z, "vc_ball", "native"), j=9)
    t2 = cache.label_epoch(prob, pts, 64, _cfg(z, "vc_ball", "native"), j=9)
    assert t2.shape == (len(pts),) and cache.epoch == 2
    bad = WalkConfig(sigma_bar=float(z["violation_sigma_bar"][0]), rng_seed=5, max_steps=400)
    with pytest.raises(MajorantViolationError):
        cache.label_epoch(prob, pts, 64, bad, j=9)
    assert cache.epoch == 2
    assert np.array_equal(cache.targets(), t2.cpu().numpy())
    del t1
