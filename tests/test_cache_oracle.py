"""Estimate-cache oracle and host codec vs the reference's own outputs (CPU).

golden_cache.npz was produced by the reference's EstimateCache
(tests/golden/make_golden_cache.py): the oracle must reproduce every epoch's
state bit for bit, and the product's SWEC/CSV host code must reproduce the
reference's file bytes (estimator.py:270-335).
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle.cache_oracle import OracleCache
from paper_2603_01193_b200 import cache as C
from paper_2603_01193_b200.estimator import PointEstimate


def _epochs(z):
    for t in range(int(z["n_epochs"][0])):
        yield t, z[f"e{t}_keys"], z[f"e{t}_mean"], z[f"e{t}_m2"], z[f"e{t}_n"]


def test_oracle_matches_reference_every_epoch():
    z = load_golden("golden_cache.npz")
    oc = OracleCache()
    for t, ks, mean, m2, n in _epochs(z):
        oc.update({(int(k[0]), int(k[1])): (a, b, c) for k, a, b, c in zip(ks, mean, m2, n)})
        keys, ms, cn, cm, c2 = oc.arrays()
        assert np.array_equal(keys, z["keys_sorted"])
        assert np.array_equal(ms, z[f"e{t}_mean_sum"])
        assert np.array_equal(cn, z[f"e{t}_cn"])
        assert np.array_equal(cm, z[f"e{t}_cmean"])
        assert np.array_equal(c2, z[f"e{t}_cm2"])
        assert np.array_equal(oc.targets(), z[f"e{t}_targets"])
    assert oc.swec_bytes() == z["swec"].tobytes()


def test_host_swec_codec_matches_reference_bytes(tmp_path):
    z = load_golden("golden_cache.npz")
    last = int(z["n_epochs"][0]) - 1
    p = tmp_path / "c.bin"
    C.write_swec(p, last + 1, z["keys_sorted"], z[f"e{last}_mean_sum"], z[f"e{last}_cn"],
                 z[f"e{last}_cmean"], z[f"e{last}_cm2"])
    assert p.read_bytes() == z["swec"].tobytes()
    epoch, keys, body = C.read_swec(p)
    assert epoch == last + 1
    assert np.array_equal(keys, z["keys_sorted"])
    assert np.array_equal(body["m2"], z[f"e{last}_cm2"])


def test_host_csv_export_matches_reference_bytes(tmp_path):
    z = load_golden("golden_cache.npz")
    last = int(z["n_epochs"][0]) - 1
    epoch = last + 1
    rows = []
    for k, (j, i) in enumerate(z["keys_sorted"]):
        est = PointEstimate(float(z[f"e{last}_mean_sum"][k] / epoch), float(z[f"e{last}_cm2"][k]),
                            int(z[f"e{last}_cn"][k]))
        rows.append((int(j), (0.125 * int(i), -0.5 + int(j) / 3.0), est))
    p = tmp_path / "c.csv"
    C.export_csv(p, rows)
    assert p.read_bytes() == z["csv"].tobytes()


@pytest.mark.parametrize("blob,msg", [
    (b"not a cache", "not an estimate cache"),
    (b"SWEC\x02\x00\x00\x00" + b"\x00" * 16, "unsupported cache version"),
    (b"SWEC\x01\x00", "truncated"),
    (b"SWEC\x01\x00\x00\x00" + (1).to_bytes(8, "little") + (3).to_bytes(8, "little") + b"\x00" * 8,
     "truncated"),
])
def test_swec_reader_validates(tmp_path, blob, msg):
    p = tmp_path / "bad.bin"
    p.write_bytes(blob)
    with pytest.raises(ValueError, match=msg):
        C.read_swec(p)


def test_empty_cache_file_roundtrip(tmp_path):
    p = tmp_path / "e.bin"
    C.write_swec(p, 0, np.empty((0, 2), np.int64), [], [], [], [])
    assert p.read_bytes() == OracleCache().swec_bytes()
    epoch, keys, body = C.read_swec(p)
    assert epoch == 0 and keys.shape == (0, 2) and body.size == 0


def test_device_cache_fails_loudly_without_cuda():
    import torch

    from paper_2603_01193_b200 import _lib
    from paper_2603_01193_b200.cache import EstimateCache

    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    cache = EstimateCache()
    with pytest.raises(_lib.WosUnavailableError):
        cache.update_arrays([(0, 0)], [1.0], [0.0], 4)
    assert cache.epoch == 0
