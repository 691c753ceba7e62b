"""Run artifacts of the label estimator in the reference CLI's file formats (row f4).

Downstream A/B tooling of the reference diffs the files ``spherewalk solve`` and
``spherewalk bench`` write (``cli.py:267-278, 630-679``; its acceptance criterion,
``test_acceptance.py:355-391``). This module produces those files from estimates
computed on the GPU. Only the bytes are the contract, so only these pieces follow
the reference exactly:

* the identity hash: sha256 of ``json.dumps(cfg, sort_keys=True, separators=(",", ":"))``
  over the effective config (command defaults overlaid with the user's keys) minus
  the runtime keys ``workers, output, history, summary`` — 12 hex digits
  (``cli.py:54,153-156``); the defaults are therefore the reference's values;
* the stamp line ``# <program> <version> seed=<s> workers=<w> config=<hash>``
  (``cli.py:159-163``), written with ``\\n``; table rows end in ``\\r\\n`` (the csv
  module's dialect the reference writes with);
* the solve table ``instance_id, x0.., mean, variance, n_samples`` and the bench
  table ``trajectories, replicas, mean, replica_variance, variance_times_l,
  seconds_per_replica``, floats as Python ``repr``; ``variance`` = m2 / (n - 1),
  nan below two samples (``estimator.py:98-103``);
* lattice query points: ``np.linspace`` per axis, C order, the flat lattice index
  as the point id, exterior lattice points dropped (``cli.py:216-251``);
* ``<output>.summary.json``: ``json.dump(indent=2, sort_keys=True)`` plus a newline.

Everything else (how a config is validated and resolved, the problem and point
builders) is this package's own. ``workers`` is the number of strided point shards
of ``estimate`` (shard i on GPU i mod n_gpus): the files are identical for any
value. Configs name a ``problem`` (domain plus constant g and f); the reference's
``instance`` configs build ``pde.py`` families, which are out of scope
(DESIGN.md section 8), and are rejected with ``UsageError``. There is no argument
parser: ``solve`` / ``bench`` take the config mapping.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import specs
from .estimator import PointEstimate, estimate_arrays
from .geometry import BallDomain, BoxDomain, MeshDomain, PolarDomain, PolygonDomain
from .walker import Problem, WalkConfig

PROGRAM = "wos-b200"
WORKERS_ENV = "SPHEREWALK_WORKERS"  # the reference's worker-count variable (cli.py:50)
_NOT_HASHED = frozenset({"workers", "output", "history", "summary"})
_BOTH = ("solve", "bench")

# field -> (default, commands accepting it); output defaults to "<command>.csv".
# The defaults enter the identity hash, so they are the reference's.
_FIELDS = {
    "problem": (None, _BOTH),
    "instance": (None, _BOTH),
    "points": (None, _BOTH),
    "grid": (None, _BOTH),
    "trajectories": (100, ("solve",)),
    "trajectory_counts": ((1, 10, 100), ("bench",)),
    "replicas": (100, ("bench",)),
    "antithetic": (False, _BOTH),
    "eps_shell": (None, _BOTH),
    "max_steps": (1000, _BOTH),
    "sigma_bar": (None, _BOTH),
    "seed": (0, _BOTH),
    "workers": (None, _BOTH),
    "output": (None, _BOTH),
}
_SOLVE_COLUMNS_TAIL = ("mean", "variance", "n_samples")
_BENCH_COLUMNS = ("trajectories", "replicas", "mean", "replica_variance", "variance_times_l",
                  "seconds_per_replica")


class UsageError(Exception):
    """Bad config content (the reference CLI exits with status 1 on these)."""


def _package_version():
    from . import __version__

    return __version__


def _jsonable(v):
    """Defaults are stored immutable; the hash and the files see JSON values."""
    return list(v) if isinstance(v, tuple) else v


# ---------------------------------------------------------------------------
# config
# ---------------------------------------------------------------------------


@dataclass
class RunConfig:
    """A command's effective configuration: defaults + the user's keys, workers resolved."""

    command: str
    values: dict = field(default_factory=dict)

    @classmethod
    def load(cls, command: str, user: dict, environ=None) -> "RunConfig":
        if command not in _BOTH:
            raise UsageError(f"unknown command {command!r}")
        allowed = sorted(k for k, (_, cmds) in _FIELDS.items() if command in cmds)
        extra = sorted(set(user) - set(allowed))
        if extra:
            raise UsageError(f"unknown config field(s): {', '.join(extra)}; allowed: {', '.join(allowed)}")
        values = {k: _jsonable(_FIELDS[k][0]) for k in allowed}
        values["output"] = f"{command}.csv"
        # JSON round trip: a private copy with exactly the types the hash will see
        values.update(json.loads(json.dumps(user)))
        rc = cls(command, values)
        rc.values["workers"] = rc._workers(os.environ if environ is None else environ)
        return rc

    def _workers(self, environ) -> int:
        w = self.values.get("workers")
        source = "workers"
        if w is None:
            w, source = environ.get(WORKERS_ENV, 1), WORKERS_ENV
        try:
            w = int(w)
        except (TypeError, ValueError):
            raise UsageError(f"{source}={w!r} is not an integer") from None
        if w < 1:
            raise UsageError("workers must be at least 1")
        return w

    def __getitem__(self, key):
        return self.values[key]

    @property
    def workers(self) -> int:
        return self.values["workers"]

    def identity_hash(self) -> str:
        """12 hex digits identifying the run's content (runtime keys excluded)."""
        core = {k: v for k, v in self.values.items() if k not in _NOT_HASHED}
        text = json.dumps(core, sort_keys=True, separators=(",", ":"))
        return hashlib.sha256(text.encode()).hexdigest()[:12]

    def stamp(self, program: str = PROGRAM, version: str | None = None) -> str:
        """The first line of every artifact."""
        v = _package_version() if version is None else version
        return (f"# {program} {v} seed={int(self.values.get('seed') or 0)} "
                f"workers={self.workers} config={self.identity_hash()}")

    def walk_config(self, mode: str = "native") -> WalkConfig:
        return WalkConfig(eps_shell=self.values["eps_shell"], max_steps=int(self.values["max_steps"]),
                          antithetic=bool(self.values["antithetic"]), sigma_bar=self.values["sigma_bar"],
                          rng_seed=int(self.values["seed"]), mode=mode)


# ---------------------------------------------------------------------------
# problems and query points
# ---------------------------------------------------------------------------

_DOMAINS = {
    "ball": lambda d: BallDomain(d.get("center", [0.0, 0.0, 0.0]), d.get("radius", 1.0)),
    "polar": lambda d: PolarDomain(r0=d.get("r0", 1.0), c1=d.get("c1", 0.0), c2=d.get("c2", 0.0)),
    "mesh": lambda d: MeshDomain(np.array(d["vertices"]), np.array(d["faces"])),
    "box": lambda d: BoxDomain(d["lo"], d["hi"]),
    "polygon": lambda d: PolygonDomain(np.asarray(d["vertices"], dtype=np.float64)),
}


def domain_from_spec(d):
    """Domain descriptor -> domain: the reference's ball / polar / mesh kinds
    (geometry.py:686-704; meshes as inline vertices + faces) plus box and polygon."""
    if not isinstance(d, dict):
        raise UsageError("domain must be an object")
    make = _DOMAINS.get(d.get("kind"))
    if make is None:
        raise ValueError(f"unknown domain kind: {d.get('kind')!r}")
    if d.get("kind") == "mesh" and "path" in d:
        raise UsageError("OBJ mesh files are not loaded here; pass vertices and faces")
    return make(d)


def problem_from_spec(spec) -> Problem:
    """{"domain": ..., "g": const, "f": const or absent, "instance_key": int} -> Problem."""
    if not isinstance(spec, dict) or spec.get("domain") is None:
        raise UsageError("problem config needs 'domain'")
    try:
        dom = domain_from_spec(spec["domain"])
    except (ValueError, KeyError, TypeError) as exc:
        raise UsageError(f"bad domain config: {exc}") from exc
    src = spec.get("f")
    return Problem(dom, instance_key=int(spec.get("instance_key", 0)),
                   boundary_spec=(specs.BND_CONST, (float(spec.get("g", 0.0)),)),
                   source_spec=None if src is None else (specs.SRC_CONST, (float(src),)))


def run_problem(rc: RunConfig) -> Problem:
    has_p, has_i = rc["problem"] is not None, rc["instance"] is not None
    if has_p == has_i:
        raise UsageError(f"{rc.command} config needs exactly one of 'problem' or 'instance'")
    if has_i:
        raise UsageError("'instance' configs build pde.py problem families, which are out of scope; "
                         "use 'problem' or the Python API")
    return problem_from_spec(rc["problem"])


def query_points(rc: RunConfig, domain):
    """(points, ids): explicit rows with ids 0..n-1, or the interior points of a lattice
    with their flat lattice indices as ids."""
    rows, grid = rc["points"], rc["grid"]
    if (rows is None) == (grid is None):
        raise UsageError(f"{rc.command} config needs exactly one of 'points' or 'grid'")
    dim = domain.dim
    if rows is not None:
        pts = np.atleast_2d(np.asarray(rows, dtype=np.float64))
        if pts.ndim != 2 or pts.shape[1] != dim:
            raise UsageError(f"points must be rows of dimension {dim}")
        return pts, np.arange(len(pts))
    missing = [k for k in ("lo", "hi", "shape") if grid.get(k) is None]
    if missing:
        raise UsageError(f"grid config needs {missing[0]!r}")
    lo, hi = np.asarray(grid["lo"], dtype=np.float64), np.asarray(grid["hi"], dtype=np.float64)
    shape = tuple(int(n) for n in grid["shape"])
    if lo.shape != (dim,) or hi.shape != (dim,) or len(shape) != dim:
        raise UsageError(f"grid lo/hi/shape must all have dimension {dim}")
    if min(shape) < 1:
        raise UsageError("grid shape entries must be positive")
    lattice = np.stack(np.meshgrid(*(np.linspace(a, b, n) for a, b, n in zip(lo, hi, shape)), indexing="ij"),
                       axis=-1).reshape(-1, dim)
    if not hasattr(domain, "contains"):
        raise UsageError(f"grid filtering needs {type(domain).__name__}.contains; pass 'points'")
    keep = np.flatnonzero(np.atleast_1d(domain.contains(lattice)))
    if keep.size == 0:
        raise UsageError("grid contains no interior points")
    return lattice[keep], keep


# ---------------------------------------------------------------------------
# files
# ---------------------------------------------------------------------------


def _cell(v) -> str:
    return str(v) if isinstance(v, (int, np.integer, str)) else repr(float(v))


def write_table(path, stamp: str, columns, rows) -> Path:
    """Stamp line, then a header row and data rows in the csv module's excel dialect
    (comma separated, CRLF); cells are ints, strings or repr floats (never quoted)."""
    lines = [",".join(columns)] + [",".join(_cell(v) for v in r) for r in rows]
    with open(path, "w", newline="") as fh:
        fh.write(stamp + "\n")
        fh.write("".join(line + "\r\n" for line in lines))
    return Path(path)


def _sample_variance(m2, n):
    return float(m2) / (int(n) - 1) if int(n) >= 2 else math.nan


def solve_rows(ids, points, estimates):
    """Rows of the solve table; ``estimates`` = PointEstimates or a (mean, m2, n) triple."""
    if isinstance(estimates, tuple) and len(estimates) == 3:
        mean, m2, n = (np.asarray(a).tolist() for a in estimates)
        var = [_sample_variance(b, c) for b, c in zip(m2, n)]
    else:
        mean = [e.mean for e in estimates]
        var = [e.variance for e in estimates]
        n = [e.n_samples for e in estimates]
    pts = np.asarray(points, dtype=np.float64).tolist()
    return [[int(i), *map(float, p), float(mu), float(v), int(k)]
            for i, p, mu, v, k in zip(np.asarray(ids).tolist(), pts, mean, var, n)]


def write_solve_csv(path, stamp, ids, points, estimates) -> Path:
    dim = np.asarray(points).reshape(len(ids), -1).shape[1]
    cols = ["instance_id"] + [f"x{d}" for d in range(dim)] + list(_SOLVE_COLUMNS_TAIL)
    return write_table(path, stamp, cols, solve_rows(ids, points, estimates))


def read_solve_csv(path):
    """(stamp, ids, points, [PointEstimate]) back from a solve table."""
    stamp, _, body = Path(path).read_bytes().decode().partition("\n")
    rows = [r.split(",") for r in body.split("\r\n") if r]
    dim = len(rows[0]) - 4
    data = rows[1:]
    ids = np.array([int(r[0]) for r in data], dtype=np.int64)
    pts = np.array([[float(c) for c in r[1:1 + dim]] for r in data], dtype=np.float64).reshape(-1, dim)
    ests = [PointEstimate(float(r[-3]), 0.0 if int(r[-1]) < 2 else float(r[-2]) * (int(r[-1]) - 1), int(r[-1]))
            for r in data]
    return stamp, ids, pts, ests


def bench_stats(L, replica_means, seconds):
    """One bench row from the (replicas, points) matrix of replica means: the replica
    variance per point (ddof 1) averaged over points, times L (the 1/L variance law),
    and wall seconds per replica. Returns (row, summary record)."""
    m = np.asarray(replica_means, dtype=np.float64)
    r = m.shape[0]
    v = float(np.mean(np.var(m, axis=0, ddof=1)))
    row = [int(L), int(r), float(np.mean(m)), v, v * L, seconds / r]
    return row, {"trajectories": int(L), "replica_variance": v, "variance_times_l": v * L}


def write_bench_csv(path, stamp, rows) -> Path:
    return write_table(path, stamp, _BENCH_COLUMNS, rows)


def write_summary(csv_path, payload) -> Path:
    """``<csv stem>.summary.json`` beside the table."""
    out = Path(csv_path).with_suffix(".summary.json")
    out.write_text(json.dumps(payload, indent=2, sort_keys=True) + "\n")
    return out


# ---------------------------------------------------------------------------
# commands
# ---------------------------------------------------------------------------


def solve(user_cfg, *, mode="native", program=PROGRAM, version=None, verbose=False):
    """Estimate every query point on the GPU and write the solve table and summary.
    Returns (table path, summary path)."""
    rc = RunConfig.load("solve", user_cfg)
    prob = run_problem(rc)
    pts, ids = query_points(rc, prob.domain)
    L = int(rc["trajectories"])
    walk = rc.walk_config(mode)
    stamp = rc.stamp(program, version)
    t0 = time.perf_counter()
    est = estimate_arrays([prob], pts, L, walk, point_ids=ids, workers=rc.workers)
    wall = time.perf_counter() - t0
    table = write_solve_csv(rc["output"], stamp, ids, pts, est)
    summary = write_summary(table, {
        "header": stamp, "command": "solve", "output": str(rc["output"]), "n_points": len(pts),
        "trajectories": L, "antithetic": walk.antithetic, "mean_min": float(np.min(est[0])),
        "mean_max": float(np.max(est[0])), "wall_seconds": round(wall, 3),
    })
    if verbose:
        print(stamp)
        print(f"wrote {table} ({len(pts)} points x {L} trajectories) and {summary}")
    return table, summary


def bench(user_cfg, *, mode="native", program=PROGRAM, version=None, verbose=False):
    """Replica variance per trajectory count; replica k uses trajectory window
    [k L, (k + 1) L). Writes the bench table and summary; returns their paths."""
    rc = RunConfig.load("bench", user_cfg)
    prob = run_problem(rc)
    pts, ids = query_points(rc, prob.domain)
    counts = [int(L) for L in rc["trajectory_counts"]]
    reps = int(rc["replicas"])
    if reps < 2 or not counts:
        raise UsageError("bench needs at least 2 replicas and one trajectory count")
    walk = rc.walk_config(mode)
    stamp = rc.stamp(program, version)
    rows, records = [], []
    for L in counts:
        t0 = time.perf_counter()
        means = np.stack([estimate_arrays([prob], pts, L, walk, point_ids=ids, traj_start=k * L,
                                          workers=rc.workers)[0] for k in range(reps)])
        row, rec = bench_stats(L, means, time.perf_counter() - t0)
        rows.append(row)
        records.append(rec)
    table = write_bench_csv(rc["output"], stamp, rows)
    summary = write_summary(table, {"header": stamp, "command": "bench", "output": str(rc["output"]),
                                    "n_points": len(pts), "replicas": reps, "rows": records})
    if verbose:
        print(stamp)
        print(f"wrote {table} and {summary}")
    return table, summary
