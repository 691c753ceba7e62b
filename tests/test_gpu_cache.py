"""Device-resident estimate cache (wos_cache_fold / wos_estimate_fold) on the GPU.

Mirrors the reference's TestEstimateCache (test_estimator.py:166-300): targets are
bit-identical to the reference cache fed the same estimates (golden_cache.npz and
the CPU oracle), incremental == replayed == resumed runs bit for bit, pooled
variance equals the one-shot estimate's, and the epoch average is unbiased with
variance ~ 1/k.
"""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle.cache_oracle import OracleCache

pytestmark = pytest.mark.gpu


def _poisson():
    from paper_2603_01193_b200 import BallDomain, Problem, specs

    # test_estimator.py:40-46: unit disk, f = 1, g = 0
    return Problem(BallDomain([0.0, 0.0], 1.0), boundary_spec=specs.const_boundary(0.0),
                   source_spec=specs.const_source(1.0))


PTS = np.array([[0.1, 0.2], [0.3, -0.1], [0.0, 0.0]])
KEYS = [(7, 0), (7, 1), (7, 2)]


def _cfg(seed, mode="native"):
    from paper_2603_01193_b200 import WalkConfig

    return WalkConfig(rng_seed=seed, mode=mode)


def test_fold_matches_reference_golden_every_epoch(gpu):
    from paper_2603_01193_b200.cache import EstimateCache

    z = load_golden("golden_cache.npz")
    cache = EstimateCache()
    for t in range(int(z["n_epochs"][0])):
        cache.update_arrays(z[f"e{t}_keys"], z[f"e{t}_mean"], z[f"e{t}_m2"], z[f"e{t}_n"])
        ms, n, mean, m2 = cache.host_state()
        assert np.array_equal(cache.key_array, z["keys_sorted"])
        assert np.array_equal(ms, z[f"e{t}_mean_sum"])
        assert np.array_equal(n, z[f"e{t}_cn"])
        assert np.array_equal(mean, z[f"e{t}_cmean"])
        assert np.array_equal(m2, z[f"e{t}_cm2"])
        assert np.array_equal(cache.targets(), z[f"e{t}_targets"])


def test_dict_interface_and_swec_bytes(gpu, tmp_path):
    from paper_2603_01193_b200 import PointEstimate
    from paper_2603_01193_b200.cache import EstimateCache, cache_update

    z = load_golden("golden_cache.npz")
    cache = EstimateCache()
    for t in range(int(z["n_epochs"][0])):
        fresh = {(int(k[0]), int(k[1])): PointEstimate(float(a), float(b), int(c))
                 for k, a, b, c in zip(z[f"e{t}_keys"], z[f"e{t}_mean"], z[f"e{t}_m2"],
                                       z[f"e{t}_n"])}
        cache_update(cache, fresh)
    p = tmp_path / "c.bin"
    cache.save(p)
    assert p.read_bytes() == z["swec"].tobytes()
    c = tmp_path / "c.csv"
    cache.export_csv(c, {k: (0.125 * k[1], -0.5 + k[0] / 3.0) for k in cache.keys})
    assert c.read_bytes() == z["csv"].tobytes()


def test_load_reference_file_and_continue(gpu, tmp_path):
    from paper_2603_01193_b200.cache import EstimateCache

    z = load_golden("golden_cache.npz")
    p = tmp_path / "ref.bin"
    p.write_bytes(z["swec"].tobytes())
    cache = EstimateCache.load(p)
    oc = OracleCache()
    for t in range(int(z["n_epochs"][0])):
        oc.update({(int(k[0]), int(k[1])): (a, b, c) for k, a, b, c in
                   zip(z[f"e{t}_keys"], z[f"e{t}_mean"], z[f"e{t}_m2"], z[f"e{t}_n"])})
    rng = np.random.default_rng(5)
    for _ in range(3):
        ks = np.array(oc.keys)[rng.permutation(len(oc.keys))]
        mean, m2 = rng.normal(size=len(ks)), rng.random(len(ks))
        n = rng.integers(1, 500, len(ks))
        cache.update_arrays(ks, mean, m2, n)
        oc.update({(int(k[0]), int(k[1])): (a, b, int(c)) for k, a, b, c in zip(ks, mean, m2, n)})
    assert cache.epoch == oc.epoch
    assert np.array_equal(cache.targets(), oc.targets())
    _, ms, cn, cm, c2 = oc.arrays()
    for a, b in zip(cache.host_state(), (ms, cn, cm, c2)):
        assert np.array_equal(a, b)


def test_first_update_is_identity(gpu):
    from paper_2603_01193_b200 import PointEstimate
    from paper_2603_01193_b200.cache import EstimateCache, cache_update

    cache = EstimateCache()
    cache_update(cache, {(0, 0): PointEstimate(1.25, 0.5, 10)})
    assert cache.epoch == 1
    assert cache.target((0, 0)) == 1.25
    assert cache.estimates()[(0, 0)].n_samples == 10


def test_second_update_averages(gpu):
    from paper_2603_01193_b200 import PointEstimate
    from paper_2603_01193_b200.cache import EstimateCache, cache_update

    cache = EstimateCache()
    cache_update(cache, {(0, 0): PointEstimate(1.0, 0.0, 4)})
    cache_update(cache, {(0, 0): PointEstimate(2.0, 0.0, 4)})
    assert cache.target((0, 0)) == (1.0 + 2.0) / 2.0
    assert cache.estimates()[(0, 0)].n_samples == 8


def test_key_mismatch_rejected(gpu):
    from paper_2603_01193_b200 import PointEstimate
    from paper_2603_01193_b200.cache import CacheShapeError, EstimateCache, cache_update

    cache = EstimateCache()
    cache_update(cache, {(0, 0): PointEstimate(1.0, 0.0, 4), (0, 1): PointEstimate(2.0, 0.0, 4)})
    with pytest.raises(CacheShapeError, match="cache shape mismatch"):
        cache_update(cache, {(0, 0): PointEstimate(1.0, 0.0, 4)})
    with pytest.raises(CacheShapeError, match="cache shape mismatch"):
        cache_update(cache, {(0, 0): PointEstimate(1.0, 0.0, 4), (9, 9): PointEstimate(2.0, 0.0, 4)})
    assert cache.epoch == 1


def _label_run(cache, cfg, L, k, first_epoch=0, pts=PTS, keys=KEYS):
    for _ in range(k):
        cache.label_epoch(_poisson(), pts, L, cfg, keys=keys)
    return cache


@pytest.mark.parametrize("mode", ["native", "replay"])
def test_label_epochs_replay_bit_equality(gpu, mode):
    """k device epochs == the oracle folding k separate estimate calls (test_estimator.py:196-208)."""
    from paper_2603_01193_b200 import estimate_arrays
    from paper_2603_01193_b200.cache import EstimateCache

    cfg = _cfg(101, mode)
    L, k = 20, 5
    cache = _label_run(EstimateCache(), cfg, L, k)
    assert cache.epoch == k
    oc = OracleCache()
    for t in range(k):
        mean, m2, n = estimate_arrays(_poisson(), PTS, L, cfg, traj_start=t * L,
                                      point_ids=[0, 1, 2])
        oc.update({key: (a, b, int(c)) for key, a, b, c in zip(KEYS, mean, m2, n)})
    assert np.array_equal(cache.targets(), oc.targets())
    for key in KEYS:
        assert cache.estimates()[key].n_samples == k * L


def test_label_epochs_resume_bit_equality(gpu, tmp_path):
    """save / load between epochs changes nothing (test_estimator.py:210-222)."""
    from paper_2603_01193_b200.cache import EstimateCache

    cfg = _cfg(102)
    straight = _label_run(EstimateCache(), cfg, 16, 6)
    part = _label_run(EstimateCache(), cfg, 16, 2)
    path = tmp_path / "cache.bin"
    part.save(path)
    resumed = EstimateCache.load(path)
    _label_run(resumed, cfg, 16, 4)
    assert resumed.epoch == straight.epoch
    assert np.array_equal(resumed.targets(), straight.targets())
    a, b = resumed.estimates(), straight.estimates()
    for key in KEYS:
        assert a[key] == b[key]
    p2 = tmp_path / "straight.bin"
    straight.save(p2)
    resumed.save(path)
    assert path.read_bytes() == p2.read_bytes()


def test_pooled_variance_matches_direct(gpu):
    """Chan-merged m2 over epochs == one-shot m2 (test_estimator.py:230-238)."""
    from paper_2603_01193_b200 import estimate
    from paper_2603_01193_b200.cache import EstimateCache

    cfg = _cfg(103)
    cache = _label_run(EstimateCache(), cfg, 25, 4, pts=PTS[:1], keys=[(0, 0)])
    merged = cache.estimates()[(0, 0)]
    (direct,) = estimate(_poisson(), PTS[:1], 100, cfg, point_ids=[0])
    assert merged.n_samples == direct.n_samples
    assert merged.m2 == pytest.approx(direct.m2, rel=1e-12)
    assert merged.variance == pytest.approx(direct.variance, rel=1e-12)


# the reference tests sit at the disk centre, where the native (Green's-function
# importance-sampled) estimator is exact with zero variance: run them in replay mode
# (the reference's estimator) there, and in native mode at an off-centre point
@pytest.mark.parametrize("mode,pt", [("replay", 2), ("native", 1)])
def test_unbiased_across_epoch_counts(gpu, mode, pt):
    """test_estimator.py:240-248 (disjoint trajectory windows)."""
    from paper_2603_01193_b200 import estimate_arrays
    from paper_2603_01193_b200.cache import EstimateCache

    cfg = _cfg(104, mode)
    P = PTS[pt:pt + 1]
    one = _label_run(EstimateCache(), cfg, 200, 1, pts=P, keys=[(0, 0)])
    fifty = EstimateCache()
    # skip ten epochs' windows so the long run shares no trajectory with `one`
    for t in range(10):
        mean, m2, n = estimate_arrays(_poisson(), P, 200, cfg, traj_start=t * 200,
                                      point_ids=[0])
        fifty.update_arrays([(0, 0)], mean, m2, n)
    _label_run(fifty, cfg, 200, 50, pts=P, keys=[(0, 0)])
    e1, e50 = one.estimates()[(0, 0)], fifty.estimates()[(0, 0)]
    gap = abs(e1.mean - e50.mean)
    assert gap < 3.0 * math.hypot(e1.std_error, e50.std_error)


@pytest.mark.parametrize("mode,pt", [("replay", 2), ("native", 1)])
def test_variance_decays_with_epochs(gpu, mode, pt):
    """var(target after k epochs) ~ 1/k across replicas (test_estimator.py:250-272).

    The replicas are keys of one cache (distinct point ids), so every epoch is one
    label_epoch call.
    """
    from paper_2603_01193_b200.cache import EstimateCache

    cfg = _cfg(105, mode)
    reps = 4000
    pts = np.repeat(PTS[pt:pt + 1], reps, axis=0)
    keys = [(0, r) for r in range(reps)]
    cache = EstimateCache()
    collected = {}
    for _ in range(16):
        tg = cache.label_epoch(_poisson(), pts, 4, cfg, keys=keys)
        if cache.epoch in (1, 4, 16):
            collected[cache.epoch] = tg.cpu().numpy()
    var = {k: np.var(v, ddof=1) for k, v in collected.items()}
    for k in (4, 16):
        ratio = var[1] / var[k]
        assert k / 1.3 <= ratio <= k * 1.3


def test_exterior_point_raises_before_touching_cache(gpu):
    from paper_2603_01193_b200 import ExteriorQueryError
    from paper_2603_01193_b200.cache import EstimateCache

    cache = _label_run(EstimateCache(), _cfg(106), 8, 1)
    before = cache.targets()
    bad = PTS.copy()
    bad[1] = [2.0, 0.0]
    with pytest.raises(ExteriorQueryError):
        cache.label_epoch(_poisson(), bad, 8, _cfg(106), keys=KEYS)
    assert cache.epoch == 1
    assert np.array_equal(cache.targets(), before)


def test_label_epoch_targets_stay_on_device(gpu):
    import torch

    from paper_2603_01193_b200 import configs
    from paper_2603_01193_b200.cache import EstimateCache

    w = configs.build(4).subset(np.arange(0, 262144, 97))
    pts = torch.as_tensor(w.points, device="cuda")
    cache = EstimateCache()
    t1 = cache.label_epoch(w.problems[0], pts, 32, w.cfg, j=4)
    t2 = cache.label_epoch(w.problems[0], pts, 32, w.cfg, j=4)
    assert t1.is_cuda and t2.is_cuda and t2.shape == (w.n_points,)
    # the two-epoch target is the average of two independent 32-walk means
    assert torch.isfinite(t2).all()
    e = cache.estimates()
    assert e[(4, 0)].n_samples == 64
