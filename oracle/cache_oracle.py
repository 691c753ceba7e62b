"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's EstimateCache.

Only tests/ (and the CPU legs of bench.py / smoke()) may import this module; the
product's cache is paper_2603_01193_b200/cache.py on the GPU. Each step follows
the reference (spherewalk/estimator.py) line for line in plain Python floats, so
it is pinned bit-for-bit against golden states and SWEC bytes produced by the
reference itself (tests/golden/make_golden_cache.py).
"""

from __future__ import annotations

import struct

import numpy as np

SWEC_MAGIC = b"SWEC"
SWEC_HEADER = struct.Struct("<IQQ")
SWEC_ENTRY = np.dtype(
    [("j", "<i8"), ("i", "<i8"), ("mean_sum", "<f8"), ("n", "<i8"), ("mean", "<f8"), ("m2", "<f8")]
)


def chan_merge(n1, mean1, m21, n2, mean2, m22):
    """estimator.py:41-53 (Python ints and floats)."""
    n = n1 + n2
    if n == 0:
        return 0, 0.0, 0.0
    delta = mean2 - mean1
    mean = mean1 + delta * (n2 / n)
    m2 = m21 + m22 + delta * delta * (n1 * n2 / n)
    return n, mean, m2


class OracleCache:
    """estimator.py:188-302: dict of per-key [mean_sum, n, mean, m2] over sorted keys."""

    def __init__(self):
        self.epoch = 0
        self.keys = []
        self.state = {}

    def update(self, fresh):
        """estimator.py:217-244. fresh: {(j, i): (mean, m2, n)}."""
        if self.epoch == 0 and not self.state:
            self.keys = sorted(fresh.keys())  # _adopt, estimator.py:206-215
            self.state = {k: [0.0, 0, 0.0, 0.0] for k in self.keys}
        elif set(fresh.keys()) != set(self.state.keys()):
            raise KeyError("cache shape mismatch")
        for key, (mean, m2, n) in fresh.items():
            s = self.state[key]
            s[0] += float(mean)
            s[1], s[2], s[3] = chan_merge(int(s[1]), float(s[2]), float(s[3]), int(n), float(mean),
                                          float(m2))
        self.epoch += 1

    def targets(self):
        """estimator.py:251-255."""
        if self.epoch == 0:
            return np.empty(0)
        return np.array([self.state[k][0] for k in self.keys]) / self.epoch

    def arrays(self):
        """(keys (n, 2), mean_sum, n, mean, m2) in key order."""
        ks = np.array(self.keys, dtype=np.int64).reshape(-1, 2)
        cols = list(zip(*[self.state[k] for k in self.keys])) if self.keys else [[], [], [], []]
        return (ks, np.array(cols[0], dtype=np.float64), np.array(cols[1], dtype=np.int64),
                np.array(cols[2], dtype=np.float64), np.array(cols[3], dtype=np.float64))

    def swec_bytes(self):
        """estimator.py:270-280."""
        ks, ms, n, mean, m2 = self.arrays()
        body = np.empty(ks.shape[0], dtype=SWEC_ENTRY)
        body["j"], body["i"] = ks[:, 0], ks[:, 1]
        body["mean_sum"], body["n"], body["mean"], body["m2"] = ms, n, mean, m2
        return SWEC_MAGIC + SWEC_HEADER.pack(1, self.epoch, ks.shape[0]) + body.tobytes()
