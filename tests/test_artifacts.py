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
    defaults = artifacts.SOLVE_DEFAULTS if str(Z[f"{name}__command"]) == "solve" else artifacts.BENCH_DEFAULTS
    eff = artifacts.effective_config(defaults, dict(cfg, output="x.csv"))
    artifacts.resolve_workers(eff)
    return eff


@pytest.mark.parametrize("name", CASES)
def test_run_stamp_matches_reference(name):
    _, csv_bytes, summary = case(name)
    stamp = artifacts.run_stamp(effective(name), program="spherewalk", version="0.1.0")
    assert csv_bytes.split(b"\n", 1)[0].decode() == stamp == summary["header"]
    ours = artifacts.run_stamp(effective(name))
    assert ours.startswith("# wos-b200 ") and ours.split(" ", 3)[3] == stamp.split(" ", 3)[3]


@pytest.mark.parametrize("name", SOLVES)
def test_grid_points_match_reference(name):
    cfg, _, _ = case(name)
    prob = artifacts.build_problem(cfg["problem"])
    pts, ids = artifacts.build_points(cfg, prob.domain, "solve")
    (c,) = list(calls(name))
    np.testing.assert_array_equal(pts, c["points"])
    np.testing.assert_array_equal(ids, c["ids"])


@pytest.mark.parametrize("name", SOLVES)
@pytest.mark.parametrize("as_arrays", [False, True])
def test_solve_csv_bytes_from_reference_estimates(tmp_path, name, as_arrays):
    _, csv_bytes, _ = case(name)
    (c,) = list(calls(name))
    stamp = artifacts.run_stamp(effective(name), program="spherewalk", version="0.1.0")
    if as_arrays:
        res = (c["mean"], c["m2"], c["n"])
    else:
        res = [PointEstimate(float(a), float(b), int(n)) for a, b, n in zip(c["mean"], c["m2"], c["n"])]
    out = tmp_path / "s.csv"
    artifacts.write_estimate_csv(out, stamp, c["ids"], c["points"], res)
    assert out.read_bytes() == csv_bytes
    stamp2, ids, pts, ests = artifacts.read_estimate_csv(out)
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
    assert lines[1] == "trajectories,replicas,mean,replica_variance,variance_times_l,seconds_per_replica"
    for line, srow, L in zip(lines[2:], summary["rows"], cfg["trajectory_counts"]):
        reps = sorted(by_L[L])
        assert [t for t, _ in reps] == [k * L for k in range(cfg["replicas"])]
        wall = float(line.split(",")[-1]) * cfg["replicas"]
        row, s = artifacts.bench_row(L, np.stack([m for _, m in reps]), wall)
        assert ",".join(str(v) for v in row[:5]) == ",".join(line.split(",")[:5])
        assert s == srow
    out = tmp_path / "b.csv"
    rows = [line.split(",") for line in lines[2:]]
    artifacts.write_bench_csv(out, lines[0], rows)
    assert out.read_bytes() == csv_bytes


def test_config_errors(monkeypatch):
    with pytest.raises(artifacts.UsageError, match="unknown config field"):
        artifacts.effective_config(artifacts.SOLVE_DEFAULTS, {"trajectoriez": 3})
    eff = artifacts.effective_config(artifacts.SOLVE_DEFAULTS, {})
    with pytest.raises(artifacts.UsageError, match="exactly one of 'problem' or 'instance'"):
        artifacts.build_instance(eff, "solve")
    eff["instance"] = {"family": "linear"}
    with pytest.raises(artifacts.UsageError, match="out of scope"):
        artifacts.build_instance(eff, "solve")
    with pytest.raises(artifacts.UsageError, match="bad domain config"):
        artifacts.build_problem({"domain": {"kind": "torus"}})
    monkeypatch.setenv(artifacts.ENV_WORKERS, "3")
    eff = artifacts.effective_config(artifacts.SOLVE_DEFAULTS, {})
    assert artifacts.resolve_workers(eff) == 3 and eff["workers"] == 3
    monkeypatch.setenv(artifacts.ENV_WORKERS, "x")
    with pytest.raises(artifacts.UsageError, match="not an integer"):
        artifacts.resolve_workers(artifacts.effective_config(artifacts.SOLVE_DEFAULTS, {}))
    with pytest.raises(artifacts.UsageError, match="at least 1"):
        artifacts.resolve_workers({"workers": 0})
    prob = artifacts.build_problem({"domain": {"kind": "ball", "center": [0, 0], "radius": 1.0}})
    with pytest.raises(artifacts.UsageError, match="no interior points"):
        artifacts.build_points({"grid": {"lo": [2, 2], "hi": [3, 3], "shape": [2, 2]}}, prob.domain, "solve")
    with pytest.raises(artifacts.UsageError, match="dimension 2"):
        artifacts.build_points({"points": [[0, 0, 0]]}, prob.domain, "solve")
    with pytest.raises(artifacts.UsageError, match="exactly one of 'points' or 'grid'"):
        artifacts.build_points({}, prob.domain, "solve")


def test_runtime_keys_do_not_change_the_hash():
    a = artifacts.effective_config(artifacts.SOLVE_DEFAULTS, {"seed": 4, "workers": 1, "output": "a.csv"})
    b = artifacts.effective_config(artifacts.SOLVE_DEFAULTS, {"seed": 4, "workers": 8, "output": "b.csv"})
    assert artifacts.config_hash(a) == artifacts.config_hash(b)
    c = artifacts.effective_config(artifacts.SOLVE_DEFAULTS, {"seed": 5})
    assert artifacts.config_hash(a) != artifacts.config_hash(c)
