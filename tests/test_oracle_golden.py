"""Pin the CPU oracle (oracle/wos_oracle.c) to the reference's own outputs.

Golden fixtures were produced by running the reference package itself
(tests/golden/make_golden.py): Philox words from rng.philox4x64, uniform draws
captured from live reference walks, per-walk (values, steps, hits) from
walker.walk_poisson_values on every BASELINE config, estimator.estimate
moments, and the reference's numba kernels on spec-coded disk/ball problems.
"""

import numpy as np
import pytest

from conftest import GOLDEN, golden_records, load_golden
from oracle import oracle as O

CFGS = [0, 1, 2, 3, 4]


def test_philox4x64_random123_kat():
    for ctr, key, want in O.PHILOX4X64_KAT:
        assert O.philox4x64_int(ctr, key) == list(want)
        assert [int(w) for w in O.philox4x64([ctr], *key)[0]] == list(want)


def test_philox4x32_random123_kat():
    for ctr, key, want in O.PHILOX4X32_KAT:
        assert O.philox4x32_int(ctr, key) == list(want)
        assert [int(w) for w in O.philox4x32([ctr], *key)[0]] == list(want)


def test_philox4x64_matches_reference_words():
    z = load_golden("golden_rng.npz")
    for c, k, w in zip(z["ctr"], z["key"], z["words"]):
        assert O.philox4x64_int(c, k) == [int(v) for v in w]
        got = O.philox4x64([c], int(k[0]), int(k[1]))[0]
        assert np.array_equal(got, w)


def test_philox4x64_numpy_cross_check():
    # numpy's Philox block at counter c equals the reference's at c + 1 (test_rng.py:29-39)
    z = load_golden("golden_rng.npz")
    k0, k1 = (int(v) for v in z["np_key"])
    for blk in range(4):
        assert O.philox4x64_int((blk + 1, 0, 0, 0), (k0, k1)) == [int(v) for v in z["np_raw"][blk]]


def test_captured_reference_draws():
    z = load_golden("golden_capture.npz")
    for k0, k1 in {(int(a), int(b)) for a, b in z["key"]}:
        m = (z["key"][:, 0] == k0) & (z["key"][:, 1] == k1)
        got = O.philox4x64(z["ctr"][m], k0, k1)
        assert np.array_equal(got, z["words"][m])


@pytest.mark.parametrize("cfg", CFGS)
def test_oracle_rows_match_reference(cfg):
    z = load_golden(f"golden_cfg{cfg}.npz")
    recs = golden_records(z)
    seed, eps, ms = int(z["seed"][0]), float(z["eps"][0]), int(z["max_steps"][0])
    for inst in np.unique(z["inst"]):
        m = z["inst"] == inst
        v, s, h = O.walk_rows(recs[inst], z["points"][m], z["pid"][m], z["tid"][m], z["sign"][m],
                              seed=seed, eps=eps, max_steps=ms)
        assert np.array_equal(s, z["steps"][m])
        assert np.array_equal(h, z["hits"][m])
        np.testing.assert_allclose(v, z["values"][m], rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("cfg", CFGS)
def test_oracle_truncated_walks(cfg):
    z = load_golden(f"golden_cfg{cfg}.npz")
    rec = golden_records(z)[int(z["t_inst"][0])]
    v, s, h = O.walk_rows(rec, z["t_points"], z["t_pid"], z["t_tid"], z["t_sign"],
                          seed=int(z["seed"][0]), eps=float(z["eps"][0]), max_steps=3)
    assert np.array_equal(s, z["t_steps"])
    assert np.array_equal(h, z["t_hits"])
    assert (z["t_hits"] == 0).any()  # the fixture exercises the max_steps exit
    np.testing.assert_allclose(v, z["t_values"], rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("cfg", [0, 1, 4])
@pytest.mark.parametrize("anti", [False, True])
def test_oracle_estimate_matches_reference(cfg, anti):
    from paper_2603_01193_b200 import configs

    w = configs.build(cfg)
    z = load_golden("golden_estimate.npz")
    tag = f"cfg{cfg}_{'anti' if anti else 'plain'}"
    sel = z[tag + "_sel"]
    L = int(z[tag + "_L"][0])
    mean, m2, _ = O.estimate(w.problems, w.points[sel], L, seed=w.cfg.rng_seed, eps=w.cfg.eps_shell,
                             max_steps=w.cfg.max_steps, point_ids=w.point_ids[sel], traj_start=5,
                             antithetic=anti)
    np.testing.assert_allclose(mean, z[tag + "_mean"], rtol=1e-9, atol=1e-14)
    np.testing.assert_allclose(m2, z[tag + "_m2"], rtol=1e-7, atol=1e-14)


def _refkernel_record(z, name):
    from paper_2603_01193_b200 import specs

    dim = int(z[name + "_dim"][0])
    src = z[name + "_src"]
    bnd = z[name + "_bnd"]
    dom = (0.0,) * dim + (1.0,)
    sk = specs.SRC_NONE if src[0] < 0 else int(src[0])
    sp = () if src[0] < 0 else tuple(src[1:])
    return (dim, specs.DOM_BALL, dom, sk, sp, int(bnd[0]), tuple(bnd[1:]), 3)


def test_oracle_matches_reference_numba_kernels():
    z = load_golden("golden_refkernels.npz")
    for name in z["names"]:
        name = str(name)
        rec = _refkernel_record(z, name)
        v, s, h = O.walk_rows(rec, z[name + "_points"], z[name + "_pid"], z[name + "_tid"],
                              z[name + "_sign"], seed=11, eps=float(z[name + "_eps"][0]), max_steps=1000)
        assert np.array_equal(s, z[name + "_steps"]), name
        np.testing.assert_allclose(v, z[name + "_values"], rtol=1e-10, atol=1e-13, err_msg=name)


def test_golden_records_match_config_builders():
    """The pinned synthetic configs still produce the problems the fixtures were made from."""
    from paper_2603_01193_b200 import configs
    from paper_2603_01193_b200.engine import problem_record

    for cfg in CFGS:
        z = load_golden(f"golden_cfg{cfg}.npz")
        recs = golden_records(z)
        w = configs.build(cfg)
        for i, r in enumerate(recs):
            mine = problem_record(w.problems[i])
            assert mine[:2] == r[:2] and mine[3] == r[3] and mine[5] == r[5] and mine[7] == r[7]
            np.testing.assert_array_equal(mine[2], r[2])
            np.testing.assert_array_equal(mine[4], r[4])
            np.testing.assert_array_equal(mine[6], r[6])


def test_philox4x32_rounds_restatement():
    """The C oracle's Philox4x32-R (the NATIVE stream's 10- and opt-in 7-round blocks)
    equals the exact-integer restatement for every round count."""
    rng = np.random.default_rng(9)
    ctr = rng.integers(0, 2**32, size=(64, 4), dtype=np.uint64).astype(np.uint32)
    for rounds in (1, 2, 7, 10, 13):
        got = O.philox4x32(ctr, 0x1234, 0xFEDC, rounds=rounds)
        for i in range(64):
            assert [int(v) for v in got[i]] == O.philox4x32_int(ctr[i], (0x1234, 0xFEDC), rounds=rounds)
    assert O.philox4x32_int((0, 0, 0, 0), (0, 0), rounds=10) == list(O.PHILOX4X32_KAT[0][2])


def test_beta22_table_moments():
    """The 3D source jump's radius fraction: the conditional mean of a 12-bit Beta(2,2)
    probability bin (include/wos_beta_table.h). Every entry lies inside its bin's
    quantile interval; the table keeps E[t] = 1/2 (to fp32 rounding) and misses Beta(2,2)'s
    E[t^2] = 3/10 and E[t^3] = 1/5 by about -1.0e-8 and -1.5e-8."""
    t = O.beta_table().astype(np.float64)
    assert t.size == 4096 and np.all(np.diff(t) > 0)
    v = np.arange(4097) / 4096.0
    q = 0.5 + np.sin(np.arcsin(2 * v - 1) / 3)
    assert np.all(t >= q[:-1]) and np.all(t <= q[1:])
    assert np.allclose(3 * q**2 - 2 * q**3, v, atol=1e-15)  # the quantile is exact
    assert abs(t.mean() - 0.5) < 1e-10
    assert -2e-8 < (t * t).mean() - 0.3 < 0
    assert -3e-8 < (t**3).mean() - 0.2 < 0


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_oracle_rows_match_large_reference_sets(cfg):
    """The C oracle (reference form, fp64) against the reference's own walks on 40,960
    rows per config (golden_large_cfg{i}.npz; inputs re-derived by large_rows.py)."""
    import sys

    sys.path.insert(0, GOLDEN)
    from large_rows import large_rows

    from paper_2603_01193_b200 import configs

    w = configs.build(cfg)
    z = load_golden(f"golden_large_cfg{cfg}.npz")
    inst, pts, pid, tid, sgn = large_rows(w, cfg)
    assert pts.shape[0] == z["values"].size >= 40960
    for k in np.unique(inst):
        m = inst == k
        v, s, h = O.walk_rows(w.problems[k], pts[m], pid[m], tid[m], sgn[m], seed=w.cfg.rng_seed,
                              eps=w.cfg.eps_shell, max_steps=w.cfg.max_steps)
        assert np.array_equal(s, z["steps"][m])
        assert np.array_equal(h, z["hits"][m])
        np.testing.assert_allclose(v, z["values"][m], rtol=1e-12, atol=1e-15)


def test_green2_table_moments():
    """The 2D source jump's radius fraction: conditional means of 12-bit bins of the disk
    Green's law p(t) = 4 t ln(1/t) (include/wos_beta_table.h). Entries lie in their bins,
    E[t] = 4/9 to fp32 rounding, E[t^2] = 1/4 - 9.5e-9."""
    t = O.green2_table().astype(np.float64)
    assert t.size == 4096 and np.all(np.diff(t) > 0)
    F = lambda x: np.where(x > 0, x * x * (1 - 2 * np.log(np.maximum(x, 1e-300))), 0.0)  # noqa: E731
    k = np.arange(4096)
    assert np.all(F(t) >= k / 4096 - 1e-7) and np.all(F(t) <= (k + 1) / 4096 + 1e-7)
    assert abs(t.mean() - 4 / 9) < 1e-9
    assert -2e-8 < (t * t).mean() - 0.25 < 0
