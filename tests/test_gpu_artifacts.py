"""Row f4 on the GPU: solve / bench artifacts of the GPU path vs the reference CLI's.

The same configs the reference CLI ran (tests/golden/make_golden_artifacts.py) go
through ``artifacts.solve`` / ``artifacts.bench`` in REPLAY mode: the stamp line is
byte-identical (with the reference's program name and version), ids and points are
the same strings, means match the reference's to rounding (REPLAY_F64 tolerance)
and sample counts are equal. Re-running gives byte-identical files.
"""

import csv
import io
import json

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

Z = load_golden("golden_artifacts.npz")
SOLVES = sorted({k.split("__")[0] for k in Z.files if k.startswith("solve_")})


def _rows(text):
    lines = text.splitlines()
    return lines[0], list(csv.reader(io.StringIO("\n".join(lines[1:]))))


@pytest.mark.parametrize("name", SOLVES)
def test_solve_replay_matches_reference_cli(gpu, tmp_path, name):
    from paper_2603_01193_b200 import artifacts

    cfg = json.loads(str(Z[f"{name}__config"]))
    ref_stamp, ref_rows = _rows(bytes(Z[f"{name}__csv"]).decode())
    out = tmp_path / f"{name}.csv"
    path, summ = artifacts.solve(dict(cfg, output=str(out)), mode="replay", program="spherewalk", version="0.1.0")
    stamp, rows = _rows(path.read_text())
    assert stamp == ref_stamp
    assert rows[0] == ref_rows[0]
    assert len(rows) == len(ref_rows)
    dim = len(rows[0]) - 4
    for r, q in zip(rows[1:], ref_rows[1:]):
        assert r[: 1 + dim] == q[: 1 + dim]  # id and coordinates, same strings
        assert r[-1] == q[-1]  # n_samples
        assert abs(float(r[-3]) - float(q[-3])) <= 1e-12 * max(1.0, abs(float(q[-3])))
        rv, qv = float(r[-2]), float(q[-2])
        assert abs(rv - qv) <= 1e-9 * max(1e-12, abs(qv))
    s = json.loads(summ.read_text())
    ref = json.loads(bytes(Z[f"{name}__summary"]).decode())
    for key in ("header", "command", "n_points", "trajectories", "antithetic"):
        assert s[key] == ref[key]
    assert abs(s["mean_min"] - ref["mean_min"]) <= 1e-12 * max(1.0, abs(ref["mean_min"]))
    # determinism: a second run writes the same bytes (the GPU path's analogue of
    # the reference's worker-count invariance, test_acceptance.py:355-391)
    out2 = tmp_path / f"{name}_2.csv"
    artifacts.solve(dict(cfg, output=str(out2)), mode="replay", program="spherewalk", version="0.1.0")
    assert out2.read_bytes() == path.read_bytes()


def test_solve_native_is_deterministic_and_close(gpu, tmp_path):
    from paper_2603_01193_b200 import artifacts

    name = "solve_disk_grid"
    cfg = json.loads(str(Z[f"{name}__config"]))
    cfg = dict(cfg, trajectories=4096)
    a, _ = artifacts.solve(dict(cfg, output=str(tmp_path / "a.csv")))
    b, _ = artifacts.solve(dict(cfg, output=str(tmp_path / "b.csv")))
    assert a.read_bytes() == b.read_bytes()
    _, ids, pts, ests = artifacts.read_solve_csv(a)
    # Laplacian u = 1 on the unit disk, u = 0 on the circle: u = (r^2 - 1) / 4
    exact = (np.sum(pts * pts, axis=1) - 1.0) / 4.0
    mean = np.array([e.mean for e in ests])
    se = np.array([e.std_error for e in ests])
    # at the disk centre the first jump lands on the circle and the Green-weighted
    # constant source is exact: zero variance, exact mean
    zero = se == 0.0
    np.testing.assert_allclose(mean[zero], exact[zero], rtol=1e-6)
    assert np.all(np.abs(mean[~zero] - exact[~zero]) < 5.0 * se[~zero])


def test_bench_replay_matches_reference_cli(gpu, tmp_path):
    from paper_2603_01193_b200 import artifacts

    name = "bench_disk"
    cfg = json.loads(str(Z[f"{name}__config"]))
    ref_stamp, ref_rows = _rows(bytes(Z[f"{name}__csv"]).decode())
    path, summ = artifacts.bench(dict(cfg, output=str(tmp_path / "b.csv")), mode="replay",
                                 program="spherewalk", version="0.1.0")
    stamp, rows = _rows(path.read_text())
    assert stamp == ref_stamp and rows[0] == ref_rows[0]
    for r, q in zip(rows[1:], ref_rows[1:]):
        assert r[:2] == q[:2]
        for j in (2, 3, 4):
            assert abs(float(r[j]) - float(q[j])) <= 1e-10 * max(1e-12, abs(float(q[j])))
    s = json.loads(summ.read_text())
    assert s["header"] == ref_stamp and s["replicas"] == cfg["replicas"]


def test_solve_bytes_invariant_to_workers(gpu, tmp_path):
    """The reference's criterion 12 (test_acceptance.py:355-391): CSV bytes after the run
    stamp are identical for workers 1/4/8 (strided point shards, here all on cuda:0)
    and the stamps differ only in their workers field."""
    from paper_2603_01193_b200 import artifacts

    cfg = json.loads(str(Z["solve_disk_grid__config"]))
    bodies, stamps = {}, {}
    for workers in (1, 4, 8):
        out = tmp_path / f"w{workers}.csv"
        artifacts.solve(dict(cfg, workers=workers, output=str(out)))
        stamps[workers], bodies[workers] = out.read_bytes().split(b"\n", 1)
    assert bodies[1] == bodies[4] == bodies[8]
    assert len({h.replace(b"workers=%d" % w, b"workers=*") for w, h in stamps.items()}) == 1
