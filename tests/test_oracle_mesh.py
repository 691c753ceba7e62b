"""Closed triangle meshes: oracle vs the reference (CPU).

golden_mesh.npz holds reference MeshDomain queries (brute force and BVH), inside
tests, and walks (plain Poisson and the varying-coefficient delta-tracking family)
on icospheres and a box mesh (tests/golden/make_golden_mesh.py).
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O

CASES = ["ico2", "ico4", "box"]


def mesh_problem(z, name):
    from paper_2603_01193_b200 import MeshDomain, Problem

    dom = MeshDomain(z[f"{name}_vertices"], z[f"{name}_faces"])
    return Problem(dom, boundary_spec=(2, (1.0, 2.0, -1.0, 0.5)), source_spec=(1, (-1.0,)),
                   instance_key=6)


@pytest.mark.parametrize("name", CASES)
def test_mesh_oracle_walks_match_reference(name):
    z = load_golden("golden_mesh.npz")
    prob = mesh_problem(z, name)
    v, s, h = O.walk_rows(prob, z[f"{name}_points"], z[f"{name}_pid"], z[f"{name}_tid"],
                          z[f"{name}_sgn"], seed=17, eps=float(z[f"{name}_eps"][0]), max_steps=500)
    same = s == z[f"{name}_steps"]
    assert same.mean() >= 0.995, f"identical steps {same.mean():.3%}"
    assert np.array_equal(h[same], z[f"{name}_hits"][same])
    ref = z[f"{name}_values"]
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref**2)))
    assert np.max(np.abs(v[same] - ref[same]) / scale[same]) < 1e-12


@pytest.mark.parametrize("name", CASES)
def test_mesh_oracle_contains(name):
    z = load_golden("golden_mesh.npz")
    got = O.contains(mesh_problem(z, name), z[f"{name}_probe"])
    assert np.array_equal(got, z[f"{name}_contains"])


def test_mesh_oracle_delta_tracking_matches_reference():
    from paper_2603_01193_b200 import MeshDomain, ScreenedProblem
    from paper_2603_01193_b200.engine import problem_record

    z = load_golden("golden_mesh.npz")
    dom = MeshDomain(z["ico2_vertices"], z["ico2_faces"])
    prob = ScreenedProblem(dom, vc_params=tuple(z["vc_params"]), instance_key=4)
    sb, eps = z["vc_cfg"]
    v, s, h = O.walk_rows(problem_record(prob), z["vc_points"], z["vc_pid"], z["vc_tid"],
                          z["vc_sgn"], seed=21, eps=eps, max_steps=400, sigma_bar=sb)
    same = s == z["vc_steps"]
    assert same.mean() >= 0.99, f"identical steps {same.mean():.3%}"
    ref = z["vc_values"]
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref**2)))
    assert np.max(np.abs(v[same] - ref[same]) / scale[same]) < 1e-9
