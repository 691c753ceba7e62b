"""Row f4: solve / bench artifacts byte-compatible with the reference CLI (CPU tests).

Golden files come from the reference CLI itself (tests/golden/make_golden_artifacts.py):
fed the reference's own estimates, the writers here must reproduce its CSV and
summary bytes, and the config hash / run stamp / grid points must match.
"""

import json

import numpy as np
import pytest

from conftest import load_golden
from paper_2603_01193_b200 import artifacts
from paper_2603_01193_b200.estimator import PointEstimate

Z = load_golden("golden_artifacts.npz")
CASES = sorted({k.split("__")[0] for k in Z.files})
SOLVES = [c for c in CASES if str(Z[f"{c}__command"]) == "solve"]


def case(name):
    cfg = json.loads(str(Z[f"{name}__config"]))
    csv_bytes = bytes(Z[f"{name}__csv"])
    summary = json.loads(bytes(Z[f"{name}__summary"]).decode())
    return cfg, csv_bytes, summary


def calls(name):
    for i in range(int(Z[f"{name}__calls"])):
        yield {k: Z[f"{name}__c{i}_{k}"] for k in ("points", "ids", "L", "traj_start", "mean", "m2", "n")}


def effective(name):
    cfg, _, _ = case(name)
    return artifacts.RunConfig.load(str(Z[f"{name}__command"]), dict(cfg, output="x.csv"))


@pytest.mark.parametrize("name", CASES)
def test_run_stamp_matches_reference(name):
    _, csv_bytes, summary = case(name)
    stamp = effective(name).stamp(program="spherewalk", version="0.1.0")
    assert csv_bytes.split(b"\n", 1)[0].decode() == stamp == summary["header"]
    ours = effective(name).stamp()
    assert ours.startswith("# wos-b200 ") and ours.split(" ", 3)[3] == stamp.split(" ", 3)[3]


@pytest.mark.parametrize("name", SOLVES)
def test_grid_points_match_reference(name):
    cfg, _, _ = case(name)
    prob = artifacts.problem_from_spec(cfg["problem"])
    pts, ids = artifacts.query_points(artifacts.RunConfig.load("solve", cfg), prob.domain)
    (c,) = list(calls(name))
    np.testing.assert_array_equal(pts, c["points"])
    np.testing.assert_array_equal(ids, c["ids"])


@pytest.mark.parametrize("name", SOLVES)
@pytest.mark.parametrize("as_arrays", [False, True])
def test_solve_csv_bytes_from_reference_estimates(tmp_path, name, as_arrays):
    _, csv_bytes, _ = case(name)
    (c,) = list(calls(name))
    stamp = effective(name).stamp(program="spherewalk", version="0.1.0")
    if as_arrays:
        res = (c["mean"], c["m2"], c["n"])
    else:
        res = [PointEstimate(float(a), float(b), int(n)) for a, b, n in zip(c["mean"], c["m2"], c["n"])]
    out = tmp_path / "s.csv"
    artifacts.write_solve_csv(out, stamp, c["ids"], c["points"], res)
    assert out.read_bytes() == csv_bytes
    stamp2, ids, pts, ests = artifacts.read_solve_csv(out)
    assert stamp2 == stamp
    np.testing.assert_array_equal(ids, c["ids"])
    np.testing.assert_array_equal(pts, c["points"])
    np.testing.assert_array_equal([e.mean for e in ests], c["mean"])


@pytest.mark.parametrize("name", SOLVES)
def test_solve_summary_bytes(tmp_path, name):
    _, _, summary = case(name)
    out = tmp_path / "s.csv"
    payload = dict(summary, output=str(out))
    path = artifacts.write_summary(out, payload)
    assert path.name == "s.summary.json"
    ref = json.dumps(payload, indent=2, sort_keys=True) + "\n"
    assert path.read_text() == ref
    (c,) = list(calls(name))
    assert summary["n_points"] == len(c["mean"])
    assert summary["mean_min"] == float(np.min(c["mean"])) and summary["mean_max"] == float(np.max(c["mean"]))


def test_bench_rows_from_reference_means(tmp_path):
    name = "bench_disk"
    cfg, csv_bytes, summary = case(name)
    by_L = {}
    for c in calls(name):
        by_L.setdefault(int(c["L"]), []).append((int(c["traj_start"]), c["mean"]))
    lines = csv_bytes.decode().splitlines()
    rows = []
    assert lines[1] == "trajectories,replicas,mean,replica_variance,variance_times_l,seconds_per_replica"
    for line, srow, L in zip(lines[2:], summary["rows"], cfg["trajectory_counts"]):
        reps = sorted(by_L[L])
        assert [t for t, _ in reps] == [k * L for k in range(cfg["replicas"])]
        wall = float(line.split(",")[-1]) * cfg["replicas"]
        row, s = artifacts.bench_stats(L, np.stack([m for _, m in reps]), wall)
        assert ",".join(repr(v) for v in row[:5]) == ",".join(line.split(",")[:5])
        assert s == srow
        rows.append(row[:5] + [float(line.split(",")[-1])])
    out = tmp_path / "b.csv"
    artifacts.write_bench_csv(out, lines[0], rows)
    assert out.read_bytes() == csv_bytes


def test_config_errors(monkeypatch):
    load = artifacts.RunConfig.load
    with pytest.raises(artifacts.UsageError, match="unknown config field"):
        load("solve", {"trajectoriez": 3})
    with pytest.raises(artifacts.UsageError, match="unknown config field"):
        load("solve", {"replicas": 3})  # a bench-only field
    rc = load("solve", {})
    with pytest.raises(artifacts.UsageError, match="exactly one of 'problem' or 'instance'"):
        artifacts.run_problem(rc)
    rc.values["instance"] = {"family": "linear"}
    with pytest.raises(artifacts.UsageError, match="out of scope"):
        artifacts.run_problem(rc)
    with pytest.raises(artifacts.UsageError, match="bad domain config"):
        artifacts.problem_from_spec({"domain": {"kind": "torus"}})
    monkeypatch.setenv(artifacts.WORKERS_ENV, "3")
    assert load("solve", {}).workers == 3
    assert load("solve", {"workers": 2}).workers == 2
    monkeypatch.setenv(artifacts.WORKERS_ENV, "x")
    with pytest.raises(artifacts.UsageError, match="not an integer"):
        load("solve", {})
    with pytest.raises(artifacts.UsageError, match="at least 1"):
        load("solve", {"workers": 0})
    monkeypatch.delenv(artifacts.WORKERS_ENV)
    assert load("bench", {}).workers == 1 and load("bench", {})["output"] == "bench.csv"
    prob = artifacts.problem_from_spec({"domain": {"kind": "ball", "center": [0, 0], "radius": 1.0}})
    with pytest.raises(artifacts.UsageError, match="no interior points"):
        artifacts.query_points(load("solve", {"grid": {"lo": [2, 2], "hi": [3, 3], "shape": [2, 2]}}), prob.domain)
    with pytest.raises(artifacts.UsageError, match="dimension 2"):
        artifacts.query_points(load("solve", {"points": [[0, 0, 0]]}), prob.domain)
    with pytest.raises(artifacts.UsageError, match="exactly one of 'points' or 'grid'"):
        artifacts.query_points(load("solve", {}), prob.domain)


def test_runtime_keys_do_not_change_the_hash():
    load = artifacts.RunConfig.load
    a = load("solve", {"seed": 4, "workers": 1, "output": "a.csv"})
    b = load("solve", {"seed": 4, "workers": 8, "output": "b.csv"})
    assert a.identity_hash() == b.identity_hash()
    assert a.identity_hash() != load("solve", {"seed": 5}).identity_hash()
    assert a.identity_hash() != load("bench", {"seed": 4}).identity_hash()
