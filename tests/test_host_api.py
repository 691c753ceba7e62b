"""Host-side logic of the drop-in API (no GPU): configs, specs, validation, moments.

Mirrors the reference's own host-side checks (walker.py:55-79, estimator.py:41-110,
geometry.py:172-238) and pins the synthetic BASELINE inputs.
"""

import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_01193_b200 import (BallDomain, BoxDomain, PointEstimate, PolygonDomain, Problem,
                                   WalkConfig, chan_merge, configs, specs)
from paper_2603_01193_b200.engine import UnsupportedProblemError, mode_code, problem_record
from paper_2603_01193_b200.geometry import UnsupportedDomainError, domain_spec


class TestWalkConfig:
    def test_defaults_match_reference(self):
        c = WalkConfig()
        assert (c.eps_shell, c.max_steps, c.antithetic, c.sigma_bar, c.rng_seed) == (None, 1000, False, None, 0)

    def test_validation(self):
        with pytest.raises(ValueError):
            WalkConfig(eps_shell=0.0)
        with pytest.raises(ValueError):
            WalkConfig(max_steps=0)
        with pytest.raises(ValueError):
            WalkConfig(mode="fast")

    def test_eps_default_scales_with_domain(self):
        big = BallDomain([0.0, 0.0], 100.0)
        assert WalkConfig().resolve_eps(big) == pytest.approx(0.1)
        assert WalkConfig(eps_shell=1e-4).resolve_eps(big) == 1e-4

    def test_modes(self):
        assert mode_code("replay") == 0 and mode_code("replay_f32") == 1 and mode_code("native") == 2


class TestPointEstimate:
    def test_from_values_two_pass(self):
        v = np.random.default_rng(0).lognormal(size=500)
        e = PointEstimate.from_values(v)
        assert e.mean == pytest.approx(v.mean(), rel=1e-14)
        assert e.variance == pytest.approx(v.var(ddof=1), rel=1e-12)

    def test_single_sample_nan(self):
        e = PointEstimate.from_values([2.5])
        assert math.isnan(e.variance) and math.isnan(e.std_error)

    def test_chan_merge_matches_pooled(self):
        rng = np.random.default_rng(2)
        a, b = rng.normal(size=300), rng.normal(loc=5.0, size=700)
        ea, eb = PointEstimate.from_values(a), PointEstimate.from_values(b)
        n, m, m2 = chan_merge(ea.n_samples, ea.mean, ea.m2, eb.n_samples, eb.mean, eb.m2)
        both = np.concatenate([a, b])
        assert n == 1000
        assert m == pytest.approx(both.mean(), rel=1e-12)
        assert m2 / (n - 1) == pytest.approx(both.var(ddof=1), rel=1e-12)
        assert chan_merge(0, 0.0, 0.0, 3, 1.5, 0.2) == (3, 1.5, 0.2)


class TestSpecs:
    def test_reference_kind_codes(self):
        # _kernels.py:34-46
        assert (specs.SRC_NONE, specs.SRC_CONST, specs.SRC_RBF2) == (0, 1, 2)
        assert (specs.BND_CONST, specs.BND_FOURIER5, specs.BND_LINEAR) == (0, 1, 2)
        assert (specs.DOM_BALL, specs.DOM_POLAR) == (0, 1)

    def test_sine_negation(self):
        a = np.arange(9.0).reshape(3, 3)
        kind, params = specs.sine_source(a, negate=True)
        assert kind == specs.SRC_SINE and params[0] == 3.0
        np.testing.assert_array_equal(params[1:], -a.ravel())

    def test_problem_record_requires_specs(self):
        with pytest.raises(UnsupportedProblemError):
            problem_record(Problem(BoxDomain([0, 0], [1, 1]), boundary=lambda q: q[:, 0]))
        with pytest.raises(UnsupportedProblemError):
            problem_record(Problem(BoxDomain([0, 0], [1, 1]), boundary_spec=specs.const_boundary(0.0),
                                   source=lambda y: y[:, 0]))

    def test_reference_ball_domain_is_accepted(self):
        class BallDomain:  # duck-typed like spherewalk.geometry.BallDomain
            center = np.array([0.1, 0.2])
            radius = 2.0
        kind, params, dim = domain_spec(BallDomain())
        assert (kind, dim) == (specs.DOM_BALL, 2) and params == (0.1, 0.2, 2.0)

    def test_polar_domain_rejected(self):
        class PolarDomain:
            dim = 2
        with pytest.raises(UnsupportedDomainError):
            domain_spec(PolarDomain())

    def test_problem_unwraps_holder(self):
        import types

        p = Problem(BoxDomain([0, 0], [1, 1]), boundary_spec=specs.const_boundary(1.0))
        assert problem_record(types.SimpleNamespace(problem=p)) == problem_record(p)


class TestGeometry:
    def test_contains_matches_oracle(self):
        rng = np.random.default_rng(3)
        pts = rng.uniform(-1.5, 1.5, size=(400, 2))
        for dom in (BoxDomain([-1, -0.5], [1, 0.5]), BallDomain([0.1, 0.0], 1.0),
                    configs.build(3).problems[5].domain):
            rec = (2, dom.spec()[0], dom.spec()[1], 0, (), 0, (0.0,), 0)
            np.testing.assert_array_equal(dom.contains(pts), O.contains(rec, pts))

    def test_polygon_sampling_is_interior(self):
        poly = configs.build(3).problems[0].domain
        pts = poly.sample_interior(500, np.random.default_rng(0))
        assert poly.contains(pts).all()


class TestConfigPins:
    def test_sizes(self):
        expect = {0: (1024, 256, 1), 1: (3160, 1024, 1), 2: (262144, 4, 64), 3: (262144, 64, 32),
                  4: (262144, 256, 1)}
        for i, (P, L, n) in expect.items():
            w = configs.build(i)
            assert (w.n_points, w.L, len(w.problems)) == (P, L, n)
            assert w.points.shape == (P, w.dim)

    def test_points_are_interior(self):
        for i in range(5):
            w = configs.build(i)
            for j, prob in enumerate(w.problems[:4]):
                sel = w.inst_index == j
                assert prob.domain.contains(w.points[sel]).all()

    def test_reproducible(self):
        a, b = configs.build(3), configs.build(3)
        np.testing.assert_array_equal(a.points, b.points)
        assert problem_record(a.problems[7]) == problem_record(b.problems[7])

    def test_source_sign_convention(self):
        # BASELINE states -Lap u = f; the reference (and the spec) take Lap u = f_ref = -f
        w = configs.build(0)
        a = w.meta["a"]
        rec = problem_record(w.problems[0])
        np.testing.assert_array_equal(np.asarray(rec[4][1:]), -a.ravel())

    def test_analytic_solution_solves_the_pde(self):
        # -Lap u = f for the manufactured cfg0/cfg4 solutions (finite differences)
        for i in (0, 4):
            w = configs.build(i)
            x = w.points[:50]
            h = 1e-4
            lap = np.zeros(len(x))
            for d in range(w.dim):
                e = np.zeros(w.dim)
                e[d] = h
                lap += (w.analytic(x + e) - 2 * w.analytic(x) + w.analytic(x - e)) / h**2
            f = configs.sine_series(w.meta["a"], x)
            np.testing.assert_allclose(-lap, f, rtol=1e-4, atol=1e-6)


def test_welford_matches_two_pass():
    """estimator.py:56-83 (the reference's test_estimator.py:67-73)."""
    from paper_2603_01193_b200 import WelfordAccumulator

    v = np.random.default_rng(1).lognormal(mean=2.0, sigma=1.5, size=10_000)
    acc = WelfordAccumulator()
    acc.extend(v)
    assert acc.n == v.size
    assert acc.mean == pytest.approx(v.mean(), rel=1e-10)
    assert acc.variance == pytest.approx(v.var(ddof=1), rel=1e-10)
    one = WelfordAccumulator()
    one.push(2.5)
    assert one.mean == 2.5 and np.isnan(one.variance)


def test_welford_merge_matches_pooled():
    """The reference's test_estimator.py:75-85: merging equals pooling the samples."""
    from paper_2603_01193_b200 import WelfordAccumulator

    rng = np.random.default_rng(2)
    a, b = rng.normal(size=300), rng.normal(loc=5.0, size=700)
    left, right = WelfordAccumulator(), WelfordAccumulator()
    left.extend(a)
    right.extend(b)
    left.merge(right)
    both = np.concatenate([a, b])
    assert left.n == 1000
    assert left.mean == pytest.approx(both.mean(), rel=1e-12)
    assert left.variance == pytest.approx(both.var(ddof=1), rel=1e-12)
    empty = WelfordAccumulator()
    empty.merge(left)
    assert (empty.n, empty.mean, empty.m2) == (left.n, left.mean, left.m2)


def test_problem_set_cache_is_lru_and_never_closes_a_held_set(monkeypatch):
    """eviction drops only the cache's reference (no close() under a caller)
    and a hit moves the entry to the most-recently-used end."""
    from paper_2603_01193_b200 import engine

    closed = []

    class FakeSet:
        def __init__(self, ctx, problems):
            self.problems = problems

        def close(self):
            closed.append(self)

    monkeypatch.setattr(engine, "ProblemSet", FakeSet)
    monkeypatch.setattr(engine, "_psets", {})
    monkeypatch.setattr(engine, "_PSET_CACHE_MAX", 2)
    monkeypatch.setattr(engine, "problem_record", lambda p: p)
    ctx = object()
    a = engine.problem_set(ctx, ["a"])
    engine.problem_set(ctx, ["b"])
    assert engine.problem_set(ctx, ["a"]) is a  # hit: "a" becomes most recent
    engine.problem_set(ctx, ["c"])  # evicts "b", not "a"
    assert engine.problem_set(ctx, ["a"]) is a
    assert [k[1] for k in engine._psets] == [("c",), ("a",)]
    assert closed == []
