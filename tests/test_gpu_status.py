"""Device-API error reporting (wos_status): errors belong to the call that raised them.

The device entry points (wos_estimate / estimate_tensors) never synchronize; an
exterior start point (estimator.py:156-159) or a watchdog trip is flagged in the
context's status block, which every walking call clears first (one stream-ordered
memset). estimate_tensors(check=True) reads it and raises the reference's error.
"""

import numpy as np
import pytest
import torch

from paper_2603_01193_b200 import configs, engine
from paper_2603_01193_b200.geometry import ExteriorQueryError
from paper_2603_01193_b200.estimator import estimate_arrays, estimate_tensors

pytestmark = pytest.mark.gpu


def _tensors(w, pts):
    dev = torch.device("cuda", 0)
    return (torch.from_numpy(np.ascontiguousarray(pts)).to(dev),
            torch.arange(pts.shape[0], dtype=torch.int64, device=dev))


def test_exterior_point_raises_on_the_call_that_saw_it(gpu):
    w = configs.build(4)
    ctx = engine.get_context(0)
    pset = engine.ProblemSet(ctx, w.problems)
    eps = w.cfg.resolve_eps(w.problems[0].domain)
    bad = w.points[:64].copy()
    bad[37] = (0.5, 1.5, 0.5)
    bad[50] = (-0.1, 0.5, 0.5)
    p, i = _tensors(w, bad)
    with pytest.raises(ExteriorQueryError, match=r"\[0.5, 1.5, 0.5\]"):
        estimate_tensors(pset, p, i, 16, w.cfg, eps=eps, check=True)
    # the flag was consumed: a clean call after it reports nothing
    p, i = _tensors(w, w.points[:64])
    m, _ = estimate_tensors(pset, p, i, 16, w.cfg, eps=eps, check=True)
    assert torch.isfinite(m).all()


def test_unchecked_flag_does_not_leak_into_the_next_call(gpu):
    """An unchecked call with an exterior point leaves its flag set; the next call clears
    the status block before it walks, so neither it nor a later wos_estimate_host / interior
    check reports the stale index (it used to name a point of another array)."""
    w = configs.build(4)
    ctx = engine.get_context(0)
    pset = engine.ProblemSet(ctx, w.problems)
    eps = w.cfg.resolve_eps(w.problems[0].domain)
    bad = w.points[:64].copy()
    bad[3] = (2.0, 2.0, 2.0)
    p, i = _tensors(w, bad)
    estimate_tensors(pset, p, i, 16, w.cfg, eps=eps)  # no check: flag stays on the device
    p, i = _tensors(w, w.points[64:80])
    estimate_tensors(pset, p, i, 16, w.cfg, eps=eps)
    assert ctx.status(torch.cuda.current_stream(0)) == (-1, 0, -1.0)
    estimate_tensors(pset, *_tensors(w, bad), 16, w.cfg, eps=eps)
    mean, _, _ = estimate_arrays(w.problems, w.points[:8], 16, w.cfg)  # host path
    assert np.isfinite(mean).all()


def test_status_reports_the_first_exterior_index(gpu):
    w = configs.build(4)
    ctx = engine.get_context(0)
    pset = engine.ProblemSet(ctx, w.problems)
    bad = w.points[:300].copy()
    for k in (250, 120, 299):
        bad[k] = (1.0 + 0.01 * k, 0.5, 0.5)
    p, i = _tensors(w, bad)
    estimate_tensors(pset, p, i, 8, w.cfg, eps=1e-3)
    first, wd, sp = ctx.status(torch.cuda.current_stream(0))
    assert (first, wd, sp) == (120, 0, -1.0)
