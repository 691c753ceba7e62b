"""Polar star-curve domains: oracle vs the reference (CPU).

golden_polar.npz holds the reference's compiled walk (walk_plain_2d with
polar_query_fast) on the paper's linear family, including a strong curve scanned
with stride 1 (tests/golden/make_golden_polar.py).
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O

CASES = ["mild", "mild2", "strong"]


def polar_problem(z, name):
    from paper_2603_01193_b200 import PolarDomain, Problem

    r0, c1, c2, stride, n = z[f"{name}_shape"]
    dom = PolarDomain(r0, c1, c2, table_size=int(n))
    return Problem(dom, boundary_spec=(1, tuple(z[f"{name}_bnd"])),
                   source_spec=(2, tuple(z[f"{name}_src"])), instance_key=int(z[f"{name}_ikey"][0]))


@pytest.mark.parametrize("name", CASES)
def test_product_table_equals_reference_table(name):
    """PolarDomain tabulates the curve with numpy exactly as the reference does."""
    z = load_golden("golden_polar.npz")
    dom = polar_problem(z, name).domain
    assert np.array_equal(dom._bx, z[f"{name}_bx"]) and np.array_equal(dom._by, z[f"{name}_by"])
    assert dom._stride == int(z[f"{name}_shape"][3])
    probe = z[f"{name}_probe"]
    assert np.array_equal(dom.contains(probe), z[f"{name}_contains"])


@pytest.mark.parametrize("name", CASES)
def test_polar_oracle_matches_reference_kernel(name):
    z = load_golden("golden_polar.npz")
    prob = polar_problem(z, name)
    v, s, h = O.walk_rows(prob, z[f"{name}_points"], z[f"{name}_pid"], z[f"{name}_tid"],
                          z[f"{name}_sgn"], seed=99, eps=float(z[f"{name}_eps"][0]), max_steps=600)
    same = s == z[f"{name}_steps"]
    assert same.mean() >= 0.995, f"identical steps {same.mean():.3%}"
    assert np.array_equal(h[same], z[f"{name}_hits"][same])
    ref = z[f"{name}_values"]
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref**2)))
    assert np.max(np.abs(v[same] - ref[same]) / scale[same]) < 1e-9


@pytest.mark.parametrize("name", CASES)
def test_polar_oracle_contains(name):
    z = load_golden("golden_polar.npz")
    got = O.contains(polar_problem(z, name), z[f"{name}_probe"])
    assert np.array_equal(got, z[f"{name}_contains"])
