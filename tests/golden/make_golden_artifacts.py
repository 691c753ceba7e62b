"""Golden run artifacts from the REFERENCE CLI.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_artifacts.py

Runs ``spherewalk.cli.main(["solve" | "bench", config.json])`` (cli.py:289-327,
630-679) on small configs and stores, per case: the config, the CSV and
summary bytes the reference wrote, and the PointEstimates it computed (captured by
wrapping ``spherewalk.cli.estimate``), so the CPU tests can feed the same estimates
to ``artifacts.write_estimate_csv`` and compare bytes, and the GPU tests can run
the same config through the GPU path in REPLAY mode.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import tempfile

import numpy as np

import spherewalk.cli as cli  # reference package

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    "solve_disk_grid": ("solve", {
        "problem": {"domain": {"kind": "ball", "center": [0.0, 0.0], "radius": 1.0}, "g": 0.0, "f": 1.0},
        "grid": {"lo": [-0.7, -0.7], "hi": [0.7, 0.7], "shape": [5, 5]},
        "trajectories": 32, "seed": 11, "workers": 1,
    }),
    "solve_ball3_points_anti": ("solve", {
        "problem": {"domain": {"kind": "ball", "center": [0.1, 0.0, -0.2], "radius": 1.5}, "g": 1.5,
                    "f": -2.0, "instance_key": 7},
        "points": [[0.0, 0.0, 0.0], [0.5, -0.3, 0.2], [1.0, 0.4, -0.5], [-0.9, 0.1, 0.3]],
        "trajectories": 16, "antithetic": True, "eps_shell": 1e-3, "max_steps": 500, "seed": 3,
        "workers": 1,
    }),
    "solve_polar_grid": ("solve", {
        "problem": {"domain": {"kind": "polar", "r0": 1.0, "c1": 0.1, "c2": -0.05}, "g": 2.0},
        "grid": {"lo": [-1.0, -1.0], "hi": [1.0, 1.0], "shape": [7, 6]},
        "trajectories": 8, "seed": 5, "workers": 1,
    }),
    "bench_disk": ("bench", {
        "problem": {"domain": {"kind": "ball", "center": [0.0, 0.0], "radius": 1.0}, "g": 0.5, "f": 1.0},
        "points": [[0.0, 0.0], [0.3, 0.2], [-0.5, 0.4]],
        "trajectory_counts": [4, 16], "replicas": 5, "seed": 2, "workers": 1,
    }),
}


def main():
    captured = []
    real = cli.estimate

    def capture(problem, points, L, walk, **kw):
        res = real(problem, points, L, walk, **kw)
        captured.append((np.asarray(points, dtype=np.float64), np.asarray(kw.get("point_ids")), int(L),
                         int(kw.get("traj_start", 0)), res))
        return res

    cli.estimate = capture
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, (command, cfg) in CASES.items():
            captured.clear()
            csv_path = os.path.join(tmp, name + ".csv")
            cfg_path = os.path.join(tmp, name + ".json")
            with open(cfg_path, "w") as fh:
                json.dump(dict(cfg, output=csv_path), fh)
            with contextlib.redirect_stdout(io.StringIO()):
                assert cli.main([command, cfg_path]) == 0
            out[f"{name}__command"] = np.array(command)
            out[f"{name}__config"] = np.array(json.dumps(cfg))
            out[f"{name}__csv"] = np.frombuffer(open(csv_path, "rb").read(), dtype=np.uint8)
            summ = os.path.join(tmp, name + ".summary.json")
            out[f"{name}__summary"] = np.frombuffer(open(summ, "rb").read(), dtype=np.uint8)
            out[f"{name}__calls"] = np.array(len(captured))
            for i, (pts, ids, L, ts, res) in enumerate(captured):
                out[f"{name}__c{i}_points"] = pts
                out[f"{name}__c{i}_ids"] = ids.astype(np.int64)
                out[f"{name}__c{i}_L"] = np.array(L)
                out[f"{name}__c{i}_traj_start"] = np.array(ts)
                out[f"{name}__c{i}_mean"] = np.array([r.mean for r in res])
                out[f"{name}__c{i}_m2"] = np.array([r.m2 for r in res])
                out[f"{name}__c{i}_n"] = np.array([r.n_samples for r in res], dtype=np.int64)
    cli.estimate = real
    np.savez_compressed(os.path.join(HERE, "golden_artifacts.npz"), **out)
    print("wrote golden_artifacts.npz:", ", ".join(CASES))


if __name__ == "__main__":
    main()
