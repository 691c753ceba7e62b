"""Delta-tracking oracle (wos_oracle.c walk_screened_one) vs the reference (CPU).

golden_screened.npz comes from the reference's walker.walk_screened_values on the
compiled constant-coefficient ball kernel, its dead-walk early exit, and the generic
path with the paper's varying-coefficient family on a ball and a box
(tests/golden/make_golden_screened.py).
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O


def case_record(z, name):
    h = z[f"{name}_head"]
    return (int(h[0]), int(h[1]), tuple(z[f"{name}_dom"]), int(h[2]), tuple(z[f"{name}_src"]),
            int(h[3]), tuple(z[f"{name}_bnd"]), int(h[4]))


@pytest.mark.parametrize("name", ["const_ball", "dead_ball", "vc_ball", "vc_box"])
def test_screened_oracle_matches_reference(name):
    z = load_golden("golden_screened.npz")
    rec = case_record(z, name)
    sigma_bar, eps, seed, max_steps = z[f"{name}_cfg"]
    v, s, h = O.walk_rows(rec, z[f"{name}_points"], z[f"{name}_pid"], z[f"{name}_tid"],
                          z[f"{name}_sgn"], seed=int(seed), eps=eps, max_steps=int(max_steps),
                          sigma_bar=sigma_bar)
    assert O.majorant() < 0.0
    same = s == z[f"{name}_steps"]
    assert same.mean() >= 0.995, f"identical steps {same.mean():.3%}"
    assert np.array_equal(h[same], z[f"{name}_hits"][same])
    ref = z[f"{name}_values"]
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref**2)))
    assert np.max(np.abs(v[same] - ref[same]) / scale[same]) < 1e-9


def test_screened_oracle_reports_majorant_violation():
    z = load_golden("golden_screened.npz")
    assert int(z["violation_raised"][0]) == 1
    rec = case_record(z, "vc_ball")
    O.walk_rows(rec, z["violation_points"], z["violation_pid"], z["violation_tid"],
                z["violation_sgn"], seed=5, eps=1e-3, max_steps=400,
                sigma_bar=float(z["violation_sigma_bar"][0]))
    assert O.majorant() > float(z["violation_sigma_bar"][0])


def test_screened_records_encode_like_the_product():
    """The product's problem_record gives the golden records for the mirror's problems."""
    from paper_2603_01193_b200 import BallDomain, BoxDomain, ScreenedProblem
    from paper_2603_01193_b200.engine import problem_record

    z = load_golden("golden_screened.npz")
    ball = BallDomain([0.0, 0.0, 0.0], 1.0)
    assert problem_record(ScreenedProblem(ball, const_coeffs=(0.7, 0.5, 1.0), instance_key=4)) == \
        case_record(z, "const_ball")
    assert problem_record(ScreenedProblem(ball, sqrt_alpha=2.0, const_coeffs=(2.0, None, 1.0))) == \
        case_record(z, "dead_ball")
    phi, a_min, a_max = z["vc_ball_src"]
    assert problem_record(ScreenedProblem(ball, vc_params=(phi, a_min, a_max), instance_key=9)) == \
        case_record(z, "vc_ball")
    phi, a_min, a_max = z["vc_box_src"]
    box = BoxDomain([0.0, 0.0, 0.0], [1.0, 1.0, 1.0])
    assert problem_record(ScreenedProblem(box, vc_params=(phi, a_min, a_max), instance_key=2)) == \
        case_record(z, "vc_box")
