"""Golden fixtures for the estimate cache, produced by the REFERENCE's EstimateCache.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cache.py

Writes golden_cache.npz: per epoch the fresh (key, mean, m2, n) inputs in the
(shuffled) order they were folded, the reference state after every epoch
(mean_sum, n, mean, m2 over the sorted keys, and targets), the SWEC file bytes
of the final state (estimator.py:270-280) and the CSV export bytes
(estimator.py:304-335).
"""

from __future__ import annotations

import os
import tempfile

import numpy as np

from spherewalk.estimator import EstimateCache, PointEstimate, cache_update  # reference

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(2026)
    keys = [(j, i) for j in (0, 3, 7) for i in range(23)]
    epochs = 6
    out = {"n_epochs": np.array([epochs])}
    cache = EstimateCache()
    for t in range(epochs):
        order = rng.permutation(len(keys))
        ks = np.array([keys[k] for k in order], dtype=np.int64)
        mean = rng.normal(0.0, 1.0, len(keys)) * 10.0 ** rng.integers(-6, 3, len(keys))
        m2 = np.abs(rng.normal(0.0, 1.0, len(keys))) * 10.0 ** rng.integers(-8, 2, len(keys))
        n = rng.choice([1, 2, 4, 64, 256, 1000, 4096], size=len(keys)).astype(np.int64)
        fresh = {tuple(int(v) for v in k): PointEstimate(float(a), float(b), int(c))
                 for k, a, b, c in zip(ks, mean, m2, n)}
        cache_update(cache, fresh)
        out[f"e{t}_keys"] = ks
        out[f"e{t}_mean"] = mean
        out[f"e{t}_m2"] = m2
        out[f"e{t}_n"] = n
        out[f"e{t}_targets"] = cache.targets().copy()
        out[f"e{t}_mean_sum"] = cache._mean_sum.copy()
        out[f"e{t}_cn"] = cache._n.copy()
        out[f"e{t}_cmean"] = cache._mean.copy()
        out[f"e{t}_cm2"] = cache._m2.copy()
    out["keys_sorted"] = np.array(cache.keys, dtype=np.int64)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "c.bin")
        cache.save(p)
        out["swec"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
        coords = {k: (0.125 * k[1], -0.5 + k[0] / 3.0) for k in cache.keys}
        c = os.path.join(d, "c.csv")
        cache.export_csv(c, coords)
        out["csv"] = np.frombuffer(open(c, "rb").read(), dtype=np.uint8)
    np.savez(os.path.join(HERE, "golden_cache.npz"), **out)
    print("wrote golden_cache.npz", len(keys), "keys", epochs, "epochs")


if __name__ == "__main__":
    main()
