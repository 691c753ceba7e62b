"""Run artifacts of the label estimator: the reference CLI's solve / bench file formats.

SURVEY.md 8(f) row f4. The reference's ``spherewalk solve`` and ``spherewalk bench``
(``cli.py:267-327, 613-679``) write a CSV behind a one-line run stamp plus a
``.summary.json``; downstream A/B tooling diffs those files. This module writes the
same artifacts from estimates computed by the GPU path, byte for byte in the
reference's format:

* run stamp ``# <program> <version> seed=<s> workers=<w> config=<hash12>``
  (``cli.py:159-163``); the hash is sha256 over the sorted, compact JSON of the
  config without its runtime keys (``cli.py:54,153-156``), so the same config file
  hashes the same here and in the reference;
* solve CSV columns ``instance_id, x0.., mean, variance, n_samples`` with Python
  ``repr`` floats (``cli.py:267-278``); ``variance`` is ``m2/(n-1)`` (nan below two
  samples, ``estimator.py:98-103``);
* bench CSV columns ``trajectories, replicas, mean, replica_variance,
  variance_times_l, seconds_per_replica`` (``cli.py:630-679``);
* ``<output>.summary.json``: ``json.dump(indent=2, sort_keys=True)`` + newline
  (``cli.py:166-171``).

``workers`` maps to the number of GPUs, as in ``estimate``. Configs name a
``problem`` (domain + constant g / f, ``cli.py:194-213``); the reference's
``instance`` configs build problem families from ``pde.py``, which is out of scope
 and raises ``UsageError``. The command-line parser itself is
not rebuilt: ``solve(cfg)`` / ``bench(cfg)`` take the config dict the reference's
``main`` would have assembled.
"""

from __future__ import annotations

import copy
import csv
import hashlib
import json
import math
import os
import time
from pathlib import Path

import numpy as np

from . import specs
from .estimator import PointEstimate, estimate_arrays
from .geometry import BallDomain, BoxDomain, MeshDomain, PolarDomain, PolygonDomain
from .walker import Problem, WalkConfig

ENV_WORKERS = "SPHEREWALK_WORKERS"  # cli.py:50
RUNTIME_KEYS = ("workers", "output", "history", "summary")  # cli.py:54
PROGRAM = "wos-b200"

SOLVE_DEFAULTS = {  # cli.py:285-298
    "problem": None,
    "instance": None,
    "points": None,
    "grid": None,
    "trajectories": 100,
    "antithetic": False,
    "eps_shell": None,
    "max_steps": 1000,
    "sigma_bar": None,
    "seed": 0,
    "workers": None,
    "output": "solve.csv",
}

BENCH_DEFAULTS = {  # cli.py:613-627
    "problem": None,
    "instance": None,
    "points": None,
    "grid": None,
    "trajectory_counts": [1, 10, 100],
    "replicas": 100,
    "antithetic": False,
    "eps_shell": None,
    "max_steps": 1000,
    "sigma_bar": None,
    "seed": 0,
    "workers": None,
    "output": "bench.csv",
}


class UsageError(Exception):
    """Bad config content (the reference's cli.UsageError, exit code 1)."""


def _version():
    from . import __version__

    return __version__


# ---------------------------------------------------------------------------
# config plumbing
# ---------------------------------------------------------------------------


def _merge(base, layer):
    for key, value in layer.items():
        if isinstance(value, dict) and isinstance(base.get(key), dict):
            _merge(base[key], value)
        else:
            base[key] = value
    return base


def effective_config(defaults, cfg):
    """``defaults`` overlaid with ``cfg``; unknown keys raise (cli.py:118-132)."""
    unknown = set(cfg) - set(defaults)
    if unknown:
        raise UsageError(
            f"unknown config field(s): {', '.join(sorted(unknown))}; "
            f"allowed: {', '.join(sorted(defaults))}"
        )
    return _merge(copy.deepcopy(defaults), copy.deepcopy(cfg))


def resolve_workers(cfg) -> int:
    """``workers`` from the config, else $SPHEREWALK_WORKERS, else 1 (cli.py:135-150)."""
    workers = cfg.get("workers")
    if workers is None:
        env = os.environ.get(ENV_WORKERS)
        if env is not None:
            try:
                workers = int(env)
            except ValueError:
                raise UsageError(f"{ENV_WORKERS}={env!r} is not an integer") from None
        else:
            workers = 1
    workers = int(workers)
    if workers < 1:
        raise UsageError("workers must be at least 1")
    cfg["workers"] = workers
    return workers


def config_hash(cfg) -> str:
    """12 hex digits of sha256 over the config minus runtime keys (cli.py:153-156)."""
    trimmed = {k: v for k, v in cfg.items() if k not in RUNTIME_KEYS}
    blob = json.dumps(trimmed, sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(blob.encode()).hexdigest()[:12]


def run_stamp(cfg, program=PROGRAM, version=None) -> str:
    """The first line of every artifact (cli.py:159-163)."""
    version = _version() if version is None else version
    return (
        f"# {program} {version} seed={int(cfg.get('seed', 0))} "
        f"workers={cfg['workers']} config={config_hash(cfg)}"
    )


def write_summary(output, payload) -> Path:
    """``<output>.summary.json`` next to the CSV (cli.py:166-171)."""
    path = Path(output).with_suffix(".summary.json")
    with open(path, "w") as fh:
        json.dump(payload, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return path


# ---------------------------------------------------------------------------
# problems and points
# ---------------------------------------------------------------------------


def domain_from_config(d):
    """Domain descriptors of geometry.domain_from_config (geometry.py:686-704) plus
    this package's ``box`` (lo, hi) and ``polygon`` (vertices)."""
    if not isinstance(d, dict):
        raise UsageError("domain must be an object")
    kind = d.get("kind")
    if kind == "ball":
        return BallDomain(d.get("center", [0.0, 0.0, 0.0]), d.get("radius", 1.0))
    if kind == "polar":
        return PolarDomain(r0=d.get("r0", 1.0), c1=d.get("c1", 0.0), c2=d.get("c2", 0.0))
    if kind == "mesh":
        if "path" in d:
            raise UsageError("OBJ mesh files are not loaded here; pass vertices and faces")
        return MeshDomain(np.array(d["vertices"]), np.array(d["faces"]))
    if kind == "box":
        return BoxDomain(d["lo"], d["hi"])
    if kind == "polygon":
        return PolygonDomain(np.asarray(d["vertices"], dtype=np.float64))
    raise ValueError(f"unknown domain kind: {kind!r}")


def build_problem(spec) -> Problem:
    """Constant-data problem from {"domain", "g", "f", "instance_key"} (cli.py:194-213)."""
    if not isinstance(spec, dict):
        raise UsageError("problem must be an object")
    if spec.get("domain") is None:
        raise UsageError("problem config needs 'domain'")
    try:
        domain = domain_from_config(spec["domain"])
    except (ValueError, KeyError, TypeError) as exc:
        raise UsageError(f"bad domain config: {exc}") from exc
    g = float(spec.get("g", 0.0))
    f = spec.get("f")
    return Problem(
        domain,
        instance_key=int(spec.get("instance_key", 0)),
        boundary_spec=(specs.BND_CONST, (g,)),
        source_spec=None if f is None else (specs.SRC_CONST, (float(f),)),
    )


def build_instance(cfg, command) -> Problem:
    problem, instance = cfg.get("problem"), cfg.get("instance")
    if (problem is None) == (instance is None):
        raise UsageError(f"{command} config needs exactly one of 'problem' or 'instance'")
    if instance is not None:
        raise UsageError("'instance' configs build pde.py problem families, which are out of scope; "
                         "use 'problem' or the Python API")
    return build_problem(problem)


def _contains(domain, pts):
    if not hasattr(domain, "contains"):
        raise UsageError(f"grid filtering needs {type(domain).__name__}.contains; pass 'points'")
    return np.atleast_1d(domain.contains(pts))


def build_points(cfg, domain, command):
    """Explicit points (ids 0..n-1), or a linspace lattice filtered to the interior
    keeping the lattice ids (cli.py:216-251)."""
    points, grid = cfg.get("points"), cfg.get("grid")
    if (points is None) == (grid is None):
        raise UsageError(f"{command} config needs exactly one of 'points' or 'grid'")
    dim = domain.dim
    if points is not None:
        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim == 1:
            pts = pts[None, :]
        if pts.ndim != 2 or pts.shape[1] != dim:
            raise UsageError(f"points must be rows of dimension {dim}")
        return pts, np.arange(pts.shape[0])
    for key in ("lo", "hi", "shape"):
        if grid.get(key) is None:
            raise UsageError(f"grid config needs {key!r}")
    lo = np.asarray(grid["lo"], dtype=np.float64)
    hi = np.asarray(grid["hi"], dtype=np.float64)
    shape = [int(n) for n in grid["shape"]]
    if not (lo.shape == hi.shape == (dim,)) or len(shape) != dim:
        raise UsageError(f"grid lo/hi/shape must all have dimension {dim}")
    if any(n < 1 for n in shape):
        raise UsageError("grid shape entries must be positive")
    axes = [np.linspace(lo[a], hi[a], shape[a]) for a in range(dim)]
    mesh = np.meshgrid(*axes, indexing="ij")
    pts = np.column_stack([m.ravel() for m in mesh])
    ids = np.arange(pts.shape[0])
    inside = _contains(domain, pts)
    if not inside.any():
        raise UsageError("grid contains no interior points")
    return pts[inside], ids[inside]


def walk_config(cfg, mode="native") -> WalkConfig:
    """WalkConfig from the config keys (cli.py:254-264) and the numeric mode."""
    return WalkConfig(
        eps_shell=cfg.get("eps_shell"),
        max_steps=int(cfg.get("max_steps", 1000)),
        antithetic=bool(cfg.get("antithetic", False)),
        sigma_bar=cfg.get("sigma_bar"),
        rng_seed=int(cfg.get("seed", 0)),
        mode=mode,
    )


# ---------------------------------------------------------------------------
# writers
# ---------------------------------------------------------------------------


def _variance(m2, n):
    return float(m2) / (int(n) - 1) if n >= 2 else math.nan


def write_estimate_csv(path, header, ids, points, results):
    """The solve CSV (cli.py:267-278). ``results`` is a list of PointEstimate or a
    (mean, m2, n) triple of arrays."""
    if isinstance(results, tuple) and len(results) == 3:
        mean, m2, n = (np.asarray(a) for a in results)
        var = [_variance(b, c) for b, c in zip(m2.tolist(), n.tolist())]
        mean, n = mean.tolist(), n.tolist()
    else:
        mean = [r.mean for r in results]
        var = [r.variance for r in results]
        n = [r.n_samples for r in results]
    pts = np.asarray(points, dtype=np.float64)
    dim = pts.shape[1]
    with open(path, "w", newline="") as fh:
        fh.write(header + "\n")
        w = csv.writer(fh)
        w.writerow(["instance_id"] + [f"x{d}" for d in range(dim)] + ["mean", "variance", "n_samples"])
        for pid, pt, mu, v, k in zip(np.asarray(ids).tolist(), pts.tolist(), mean, var, n):
            w.writerow([int(pid)] + [repr(float(c)) for c in pt] + [repr(float(mu)), repr(float(v)), int(k)])


def write_bench_csv(path, header, rows):
    """The bench CSV (cli.py:662-668); rows = [L, replicas, mean, var, var L, s/replica]."""
    with open(path, "w", newline="") as fh:
        fh.write(header + "\n")
        w = csv.writer(fh)
        w.writerow(
            ["trajectories", "replicas", "mean", "replica_variance", "variance_times_l", "seconds_per_replica"]
        )
        w.writerows(rows)


def bench_row(L, means, wall):
    """One bench row from the (replicas, points) matrix of replica means (cli.py:645-659)."""
    means = np.asarray(means, dtype=np.float64)
    replicas = means.shape[0]
    var = float(means.var(axis=0, ddof=1).mean())
    row = [int(L), replicas, repr(float(means.mean())), repr(var), repr(var * L), repr(wall / replicas)]
    return row, {"trajectories": int(L), "replica_variance": var, "variance_times_l": var * L}


# ---------------------------------------------------------------------------
# commands
# ---------------------------------------------------------------------------


def solve(cfg, *, mode="native", program=PROGRAM, version=None, verbose=False):
    """``spherewalk solve`` on the GPU path (cli.py:289-327): estimate every point,
    write the CSV and its summary. Returns (csv path, summary path)."""
    cfg = effective_config(SOLVE_DEFAULTS, cfg)
    workers = resolve_workers(cfg)
    problem = build_instance(cfg, "solve")
    points, ids = build_points(cfg, problem.domain, "solve")
    L = int(cfg.get("trajectories", 100))
    walk = walk_config(cfg, mode)
    header = run_stamp(cfg, program, version)
    t0 = time.perf_counter()
    mean, m2, n = estimate_arrays([problem], points, L, walk, point_ids=ids, workers=workers)
    wall = time.perf_counter() - t0
    out = cfg["output"]
    write_estimate_csv(out, header, ids, points, (mean, m2, n))
    summary = write_summary(
        out,
        {
            "header": header,
            "command": "solve",
            "output": str(out),
            "n_points": int(points.shape[0]),
            "trajectories": L,
            "antithetic": walk.antithetic,
            "mean_min": float(np.min(mean)),
            "mean_max": float(np.max(mean)),
            "wall_seconds": round(wall, 3),
        },
    )
    if verbose:
        print(header)
        print(f"wrote {out} ({points.shape[0]} points x {L} trajectories) and {summary}")
    return Path(out), summary


def bench(cfg, *, mode="native", program=PROGRAM, version=None, verbose=False):
    """``spherewalk bench`` on the GPU path (cli.py:630-679): replica variance per
    trajectory count, replica k on trajectory window [k L, (k+1) L)."""
    cfg = effective_config(BENCH_DEFAULTS, cfg)
    workers = resolve_workers(cfg)
    problem = build_instance(cfg, "bench")
    points, ids = build_points(cfg, problem.domain, "bench")
    counts = [int(L) for L in cfg["trajectory_counts"]]
    replicas = int(cfg["replicas"])
    if replicas < 2 or not counts:
        raise UsageError("bench needs at least 2 replicas and one trajectory count")
    walk = walk_config(cfg, mode)
    header = run_stamp(cfg, program, version)
    rows, summary_rows = [], []
    for L in counts:
        t0 = time.perf_counter()
        means = np.empty((replicas, points.shape[0]))
        for k in range(replicas):
            means[k] = estimate_arrays([problem], points, L, walk, point_ids=ids, traj_start=k * L,
                                       workers=workers)[0]
        row, srow = bench_row(L, means, time.perf_counter() - t0)
        rows.append(row)
        summary_rows.append(srow)
    out = cfg["output"]
    write_bench_csv(out, header, rows)
    summary = write_summary(
        out,
        {
            "header": header,
            "command": "bench",
            "output": str(out),
            "n_points": int(points.shape[0]),
            "replicas": replicas,
            "rows": summary_rows,
        },
    )
    if verbose:
        print(header)
        print(f"wrote {out} and {summary}")
    return Path(out), summary


def read_estimate_csv(path):
    """Parse a solve CSV: (stamp line, ids, points, list of PointEstimate)."""
    with open(path, newline="") as fh:
        stamp = fh.readline().rstrip("\n")
        rows = list(csv.reader(fh))
    cols = rows[0]
    dim = len(cols) - 4
    ids = np.array([int(r[0]) for r in rows[1:]], dtype=np.int64)
    pts = np.array([[float(c) for c in r[1:1 + dim]] for r in rows[1:]], dtype=np.float64).reshape(-1, dim)
    ests = []
    for r in rows[1:]:
        n = int(r[-1])
        var = float(r[-2])
        ests.append(PointEstimate(float(r[-3]), 0.0 if n < 2 else var * (n - 1), n))
    return stamp, ids, pts, ests
