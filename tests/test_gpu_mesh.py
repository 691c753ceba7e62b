"""Closed triangle meshes on the GPU (mesh part).

The device BVH query must give the reference's nearest triangle distance and exit
point (REPLAY rows equal the reference walk for walk on a 320-face brute-force
sphere, a 5120-face BVH sphere and a 12-face box), NATIVE rows follow the native
oracle, the pseudo-normal inside test equals MeshDomain.contains, and delta
tracking runs on meshes too.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O
from test_oracle_mesh import CASES, mesh_problem

pytestmark = pytest.mark.gpu


def _cfg(z, name, mode):
    from paper_2603_01193_b200 import WalkConfig

    return WalkConfig(eps_shell=float(z[f"{name}_eps"][0]), max_steps=500, rng_seed=17, mode=mode)


def _rows(z, name):
    return z[f"{name}_points"], z[f"{name}_pid"], z[f"{name}_tid"], z[f"{name}_sgn"]


@pytest.mark.parametrize("name", CASES)
def test_replay_rows_match_reference(gpu, name):
    from paper_2603_01193_b200 import walk_poisson_values

    z = load_golden("golden_mesh.npz")
    v, s, h = walk_poisson_values(mesh_problem(z, name), *_rows(z, name), _cfg(z, name, "replay"))
    same = s == z[f"{name}_steps"]
    assert same.mean() >= 0.995, f"identical steps {same.mean():.3%}"
    assert np.array_equal(h[same], z[f"{name}_hits"][same])
    ref = z[f"{name}_values"]
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref**2)))
    assert np.max(np.abs(v[same] - ref[same]) / scale[same]) < 1e-12


@pytest.mark.parametrize("name", CASES)
def test_native_rows_match_native_oracle(gpu, name):
    from paper_2603_01193_b200 import walk_poisson_values

    z = load_golden("golden_mesh.npz")
    prob = mesh_problem(z, name)
    v, s, h = walk_poisson_values(prob, *_rows(z, name), _cfg(z, name, "native"))
    vo, so, ho = O.walk_rows(prob, *_rows(z, name), seed=17, eps=float(z[f"{name}_eps"][0]),
                             max_steps=500, native=True)
    same = s == so
    assert same.mean() >= 0.97, f"identical steps {same.mean():.3%}"
    rms = np.sqrt(np.mean(vo**2)) + 1e-30
    err = np.abs(v[same] - vo[same]) / np.maximum(np.abs(vo[same]), rms)
    assert np.quantile(err, 0.99) < 1e-3


@pytest.mark.parametrize("name", CASES)
def test_interior_check_matches_reference(gpu, name):
    from paper_2603_01193_b200 import ExteriorQueryError, estimate

    z = load_golden("golden_mesh.npz")
    prob = mesh_problem(z, name)
    probe, inside = z[f"{name}_probe"], z[f"{name}_contains"]
    estimate(prob, probe[inside], 2, _cfg(z, name, "native"))
    for p in probe[~inside][:10]:
        with pytest.raises(ExteriorQueryError):
            estimate(prob, p[None, :], 2, _cfg(z, name, "native"))


def test_delta_tracking_on_mesh(gpu):
    from paper_2603_01193_b200 import MeshDomain, ScreenedProblem, WalkConfig, walk_screened_values
    from paper_2603_01193_b200.engine import problem_record

    z = load_golden("golden_mesh.npz")
    prob = ScreenedProblem(MeshDomain(z["ico2_vertices"], z["ico2_faces"]),
                           vc_params=tuple(z["vc_params"]), instance_key=4)
    sb, eps = z["vc_cfg"]
    args = (z["vc_points"], z["vc_pid"], z["vc_tid"], z["vc_sgn"])
    v, s, h = walk_screened_values(prob, *args, WalkConfig(eps_shell=eps, max_steps=400, rng_seed=21,
                                                           sigma_bar=sb, mode="replay"))
    same = s == z["vc_steps"]
    assert same.mean() >= 0.99
    ref = z["vc_values"]
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref**2)))
    assert np.max(np.abs(v[same] - ref[same]) / scale[same]) < 1e-9
    vn, sn, hn = walk_screened_values(prob, *args, WalkConfig(eps_shell=eps, max_steps=400,
                                                              rng_seed=21, sigma_bar=sb))
    vo, so, ho = O.walk_rows(problem_record(prob), *args, seed=21, eps=eps, max_steps=400,
                             native=True, sigma_bar=sb)
    assert np.mean(sn == so) >= 0.95


def test_native_estimate_on_bvh_mesh_matches_reference_form(gpu):
    from paper_2603_01193_b200 import estimate_arrays

    z = load_golden("golden_mesh.npz")
    prob = mesh_problem(z, "ico4")
    pts = z["ico4_points"][::6][:16]
    L = 4096
    cfg = _cfg(z, "ico4", "native")
    mean, m2, n = estimate_arrays([prob], pts, L, cfg)
    om, om2, _ = O.estimate([prob], pts, L // 4, seed=3, eps=cfg.eps_shell, max_steps=500)
    se = np.sqrt(m2 / (n - 1) / n + om2 / (L // 4 - 1) / (L // 4))
    zs = (mean - om) / se
    assert np.max(np.abs(zs)) < 4.5
    assert np.sqrt(np.mean(zs**2)) < 1.6
