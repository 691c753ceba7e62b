"""North-star check 2 at full size (slow): NATIVE (GPU, the production kernels) against the
reference form (the pinned C oracle, estimator.estimate semantics, estimator.py:144-181)
on EVERY query point of a BASELINE config at its configured walks per point.

The per-point z uses each arm's own sample SEs; walk values are skewed and small-L sample
SEs are noisy, so the test bounds the distribution rather than single points:
rms z near 1, the global mean difference within 4 pooled SEs, and the z of 64-point bin
means (64 L walks per bin; cfg2's L = 4 makes per-point SEs Student-t with 3 dof) near
N(0, 1). profiles/check2_full.py prints the same statistics for all five configs
(profiles/r2c_check2_full.txt).
"""

import dataclasses

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _check2(c, seed_shift=0):
    from paper_2603_01193_b200 import configs, estimate_arrays

    w = configs.build(c)
    multi = len(w.problems) > 1
    inst = w.inst_index if multi else None
    L = w.L
    s0 = w.cfg.rng_seed + seed_shift
    cfg = dataclasses.replace(w.cfg, rng_seed=s0)
    m, v, _ = estimate_arrays(w.problems, w.points, L, cfg, point_ids=w.point_ids, inst_index=inst)
    om, ov, _ = O.estimate(w.problems, w.points, L, seed=s0 + 1, eps=w.cfg.eps_shell,
                           max_steps=w.cfg.max_steps, point_ids=w.point_ids, inst_index=inst,
                           nthreads=O.default_threads())
    se2 = lambda var: var / (L - 1) / L  # noqa: E731
    floor = 1e-6 * np.maximum(1.0, np.abs(om))
    z = (m - om) / np.sqrt(se2(v) + se2(ov) + floor**2)
    g = np.sum(m - om) / np.sqrt(np.sum(se2(v) + se2(ov)))
    zb = []
    for k in range(len(w.problems)):
        idx = np.flatnonzero(w.inst_index == k)
        for b in range(0, idx.size - 63, 64):
            s = idx[b:b + 64]
            var = (np.sum(v[s] / (L - 1)) + np.sum(ov[s] / (L - 1))) / L / 64**2
            zb.append((m[s].mean() - om[s].mean()) / np.sqrt(var))
    return z, g, np.asarray(zb)


@pytest.mark.parametrize("c", [0, 1, 2, 4])
def test_check2_full_size(gpu, c):
    z, g, zb = _check2(c)
    rms = float(np.sqrt(np.mean(z**2)))
    rms_b = float(np.sqrt(np.mean(zb**2)))
    if c != 2:  # cfg2 (L = 4): per-point z are t-distributed with 3 dof, bins carry the check
        assert 0.9 < rms < 1.15, rms
    assert abs(g) < 4.0, g
    # rms of n near-normal bin z: sd ~ 1/sqrt(2 n) (cfg0 has only 16 bins)
    assert abs(rms_b - 1.0) < max(0.15, 4.0 / np.sqrt(2 * zb.size)), (rms_b, zb.size)
    # 64-point bins are near-normal: |z| > 5 has probability 6e-7 per bin
    assert np.max(np.abs(zb)) < 5.5, np.max(np.abs(zb))
