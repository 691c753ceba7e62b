"""pytest configuration: the `gpu` marker and repo-root imports.

`-m "not gpu"` runs here (no GPU): oracle vs golden fixtures, host logic, the
C-ABI library's exports, gloo multi-process sharding. `-m gpu` runs on a B200
and calls the CUDA path through the C ABI.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libwos_b200.so")
    config.addinivalue_line("markers", "slow: full-size statistical checks (minutes; GPU plus host oracle)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_records(z):
    """Spec records stored in a golden_cfg*.npz."""
    recs = []
    for i in range(int(z["n_records"][0])):
        h = z[f"rec{i}_head"]
        recs.append((int(h[0]), int(h[1]), tuple(float(v) for v in z[f"rec{i}_dom"]), int(h[2]),
                     tuple(float(v) for v in z[f"rec{i}_src"]), int(h[3]),
                     tuple(float(v) for v in z[f"rec{i}_bnd"]), int(z[f"rec{i}_ikey"][0])))
    return recs


class RecordProblem:
    """A Problem-like object built from a spec record (for the GPU API)."""

    def __init__(self, rec):
        from paper_2603_01193_b200 import geometry, specs

        dim, dk, dp, sk, sp, bk, bp, ikey = rec
        if dk == specs.DOM_BOX:
            self.domain = geometry.BoxDomain(dp[:dim], dp[dim:])
        elif dk == specs.DOM_BALL:
            self.domain = geometry.BallDomain(dp[:dim], dp[dim])
        else:
            n = int(dp[0])
            self.domain = geometry.PolygonDomain(np.asarray(dp[1:]).reshape(n, 2))
        self.source = None
        self.boundary = None
        self.source_spec = None if sk == specs.SRC_NONE else (sk, sp)
        self.boundary_spec = (bk, bp)
        self.instance_key = ikey


@pytest.fixture(scope="session")
def gpu():
    """Skip-free GPU guard: a GPU test must fail loudly if CUDA or the library is missing."""
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2603_01193_b200 import _lib, engine

    _lib.load_library()
    return engine.get_context(0)
