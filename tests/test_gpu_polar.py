"""Polar star-curve domains on the GPU (polar part).

REPLAY rows reproduce the reference's compiled walk on the paper's linear family
(walk_plain_2d + polar_query_fast) walk for walk; NATIVE rows follow the native
oracle; estimates agree statistically with the reference form; the GPU interior
check equals PolarDomain.contains; multi-instance sets (tables read through L1)
give the same walks as single-instance launches (tables in shared memory).
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O
from test_oracle_polar import CASES, polar_problem

pytestmark = pytest.mark.gpu


def _cfg(z, name, mode):
    from paper_2603_01193_b200 import WalkConfig

    return WalkConfig(eps_shell=float(z[f"{name}_eps"][0]), max_steps=600, rng_seed=99, mode=mode)


def _rows(z, name):
    return z[f"{name}_points"], z[f"{name}_pid"], z[f"{name}_tid"], z[f"{name}_sgn"]


@pytest.mark.parametrize("name", CASES)
def test_replay_rows_match_reference_kernel(gpu, name):
    from paper_2603_01193_b200 import walk_poisson_values

    z = load_golden("golden_polar.npz")
    v, s, h = walk_poisson_values(polar_problem(z, name), *_rows(z, name), _cfg(z, name, "replay"))
    same = s == z[f"{name}_steps"]
    assert same.mean() >= 0.995, f"identical steps {same.mean():.3%}"
    assert np.array_equal(h[same], z[f"{name}_hits"][same])
    ref = z[f"{name}_values"]
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref**2)))
    assert np.max(np.abs(v[same] - ref[same]) / scale[same]) < 1e-9


@pytest.mark.parametrize("name", CASES)
def test_native_rows_match_native_oracle(gpu, name):
    from paper_2603_01193_b200 import walk_poisson_values

    z = load_golden("golden_polar.npz")
    prob = polar_problem(z, name)
    v, s, h = walk_poisson_values(prob, *_rows(z, name), _cfg(z, name, "native"))
    vo, so, ho = O.walk_rows(prob, *_rows(z, name), seed=99, eps=float(z[f"{name}_eps"][0]),
                             max_steps=600, native=True)
    same = s == so
    assert same.mean() >= 0.97, f"identical steps {same.mean():.3%}"
    rms = np.sqrt(np.mean(vo**2)) + 1e-30
    err = np.abs(v[same] - vo[same]) / np.maximum(np.abs(vo[same]), rms)
    assert np.quantile(err, 0.99) < 1e-3


@pytest.mark.parametrize("name", CASES)
def test_interior_check_matches_reference(gpu, name):
    from paper_2603_01193_b200 import ExteriorQueryError, estimate

    z = load_golden("golden_polar.npz")
    prob = polar_problem(z, name)
    probe, inside = z[f"{name}_probe"], z[f"{name}_contains"]
    estimate(prob, probe[inside][:5], 2, _cfg(z, name, "native"))
    with pytest.raises(ExteriorQueryError):
        estimate(prob, probe[~inside][:1], 2, _cfg(z, name, "native"))


@pytest.mark.parametrize("name", ["mild", "strong"])
def test_native_estimate_matches_reference_form(gpu, name):
    from paper_2603_01193_b200 import estimate_arrays

    z = load_golden("golden_polar.npz")
    prob = polar_problem(z, name)
    pts = z[f"{name}_points"][::8][:24]
    L = 4096
    cfg = _cfg(z, name, "native")
    mean, m2, n = estimate_arrays([prob], pts, L, cfg)
    om, om2, _ = O.estimate([prob], pts, L, seed=7, eps=cfg.eps_shell, max_steps=600)
    se = np.sqrt(m2 / (n - 1) / n + om2 / (L - 1) / L)
    zs = (mean - om) / se
    assert np.max(np.abs(zs)) < 4.5
    assert np.sqrt(np.mean(zs**2)) < 1.6


@pytest.mark.parametrize("mode", ["replay", "native"])
def test_multi_instance_equals_single(gpu, mode):
    """Two curves in one set (tables read through L1) == each alone (table in shared memory)."""
    from paper_2603_01193_b200 import estimate_arrays

    z = load_golden("golden_polar.npz")
    a, b = polar_problem(z, "mild"), polar_problem(z, "strong")
    pa, pb = z["mild_points"][::8][:16], z["strong_points"][::8][:16]
    cfg = _cfg(z, "mild", mode)
    ma, qa, _ = estimate_arrays([a], pa, 64, cfg)
    mb, qb, _ = estimate_arrays([b], pb, 64, cfg)
    mm, qm, _ = estimate_arrays([a, b], np.concatenate([pa, pb]), 64, cfg,
                                inst_index=np.repeat([0, 1], [16, 16]),
                                point_ids=np.concatenate([np.arange(16), np.arange(16)]))
    if mode == "replay":
        assert np.array_equal(mm, np.concatenate([ma, mb]))
        assert np.array_equal(qm, np.concatenate([qa, qb]))
    else:
        # NATIVE single- and multi-instance kernels are separate fp32 instantiations; the
        # Fourier boundary at the polar projection may round differently in the last bits
        np.testing.assert_allclose(mm, np.concatenate([ma, mb]), rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(qm, np.concatenate([qa, qb]), rtol=1e-5, atol=1e-8)
