"""Walk-on-spheres trajectories on the GPU — drop-in for ``spherewalk.walker``.

Same names, arguments, return values and errors as the reference
(``walker.py:55-116, 181-229, 426-462``); the walk itself runs in the sm_100a
kernels of libwos_b200.so. Problems must be spec-coded (``boundary_spec`` /
``source_spec`` plus a Ball/Box/Polygon domain); others raise
``UnsupportedProblemError`` instead of falling back to a CPU path.

``WalkConfig`` gains one field, ``mode``:

* ``"replay"`` (= ``"replay_f64"``): the reference's own estimator and Philox4x64
  draws, fp64 arithmetic — walk-for-walk equal to ``spherewalk`` within rounding.
* ``"replay_f32"``: the same draws, fp32 arithmetic.
* ``"native"``: the production estimator (Philox4x32, Green's-function importance
  sampling, fp32 fast math) — statistically equal, much faster. Default.
"""

from __future__ import annotations

from ctypes import byref, c_int64
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import (
    problem_set,
    UnsupportedProblemError,
    get_context,
    mode_code,
    raise_exterior,
    walk_config_struct,
)
from .geometry import ExteriorQueryError

__all__ = [
    "MajorantViolationError",
    "ScreenedProblem",
    "walk_screened_delta",
    "walk_screened_values",
    "WalkConfig",
    "TrajectoryResult",
    "TrajectoryStream",
    "Problem",
    "UnsupportedProblemError",
    "TERM_BOUNDARY",
    "TERM_MAX_STEPS",
    "walk_poisson",
    "walk_poisson_antithetic",
    "walk_poisson_values",
]

TERM_BOUNDARY = "boundary"
TERM_MAX_STEPS = "max_steps"


@dataclass(frozen=True)
class WalkConfig:
    """Knobs shared by every walker (walker.py:55-79) plus the numeric mode."""

    eps_shell: float | None = None
    max_steps: int = 1000
    antithetic: bool = False
    sigma_bar: float | None = None
    rng_seed: int = 0
    mode: str = "native"
    # NATIVE mode: Philox4x32 rounds per block. 10 (Random123's default) is the
    # production stream; 7 (the fewest rounds Random123 reports Crush-resistant) is an
    # opt-in faster stream. REPLAY modes ignore it.
    philox_rounds: int = 10

    def __post_init__(self):
        if self.eps_shell is not None and self.eps_shell <= 0.0:
            raise ValueError("eps_shell must be positive")
        if self.max_steps < 1:
            raise ValueError("max_steps must be at least 1")
        if self.philox_rounds not in (7, 10):
            raise ValueError("philox_rounds must be 10 or 7")
        mode_code(self.mode)

    def resolve_eps(self, domain) -> float:
        if self.eps_shell is not None:
            return self.eps_shell
        return 1.0e-3 * domain.bounding_radius()


@dataclass(frozen=True)
class TrajectoryResult:
    value: float
    steps_taken: int
    terminated_by: str


@dataclass(frozen=True)
class TrajectoryStream:
    """Which substream of the seed a trajectory draws from (walker.py:89-99)."""

    point_id: int = 0
    traj_id: int = 0
    sign: float = 1.0


@dataclass(frozen=True)
class Problem:
    """A Poisson problem: domain, boundary g, optional source f (walker.py:102-116).

    ``boundary``/``source`` callables are accepted for signature compatibility
    but the GPU walker reads only the ``*_spec`` codes.
    """

    domain: object
    boundary: object = None
    source: object = None
    instance_key: int = 0
    boundary_spec: tuple | None = None
    source_spec: tuple | None = None


class MajorantViolationError(RuntimeError):
    """sigma' exceeded the delta-tracking majorant sigma_bar (walker.py:51-52)."""


@dataclass(frozen=True)
class ScreenedProblem:
    """Transformed screened problem for delta tracking (walker.py:120-136).

    The GPU walker reads the coefficient codes: ``const_coeffs = (s', f' or None, g')``
    (the reference's compiled form; ``sqrt_alpha`` then None or a number), or
    ``vc_params = (phi, a_min, a_max)`` for the paper's varying-coefficient family
    (pde.VcInstance, pde.py:138-243: sigma', f', g' and sqrt(alpha) in closed form).
    The callable fields are kept for signature compatibility only.
    """

    domain: object
    sigma_prime: object = None
    boundary_prime: object = None
    source_prime: object = None
    sqrt_alpha: object = None
    instance_key: int = 0
    const_coeffs: tuple | None = None
    vc_params: tuple | None = None


def check_screened(status: int) -> None:
    """_lib.check with WOS_ERR_MAJORANT mapped to MajorantViolationError."""
    if status == _lib.WOS_ERR_MAJORANT:
        raise MajorantViolationError(_lib.last_error())
    _lib.check(status)


def _cfg_of(cfg):
    return cfg if cfg is not None else WalkConfig()


def _streams_as_arrays(point_ids, traj_ids, signs, n):
    # walker.py:139-145
    pid = np.ascontiguousarray(np.asarray(point_ids).astype(np.int64).astype(np.uint64))
    tid = np.ascontiguousarray(np.asarray(traj_ids).astype(np.int64).astype(np.uint64))
    sgn = np.ascontiguousarray(np.asarray(signs, dtype=np.float64))
    if not (pid.shape == tid.shape == sgn.shape == (n,)):
        raise ValueError("stream arrays must match the number of start points")
    return pid, tid, sgn


def walk_poisson_values(inst, points, point_ids, traj_ids, signs, cfg):
    """Values, step counts, and boundary-hit flags for a batch of walks.

    One row per trajectory: points[i] walked under stream
    (point_ids[i], traj_ids[i], signs[i]) — walker.py:181-229. Returns
    (values float64 (n,), steps int64 (n,), hits uint8 (n,)).
    """
    inst = getattr(inst, "problem", inst)
    cfg = _cfg_of(cfg)
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    if pts.ndim != 2:
        raise ValueError("points must be an (n, d) array")
    n = pts.shape[0]
    pid, tid, sgn = _streams_as_arrays(point_ids, traj_ids, signs, n)
    ctx = get_context()
    pset = problem_set(ctx, [inst])
    if pts.shape[1] != pset.dim:
        raise ValueError(f"expected points of dimension {pset.dim}, got shape {pts.shape}")
    wc = walk_config_struct(cfg.resolve_eps(inst.domain), cfg.max_steps, False, cfg.mode, cfg.rng_seed,
                            philox_rounds=cfg.philox_rounds)
    values = np.empty(n, dtype=np.float64)
    steps = np.empty(n, dtype=np.int64)
    hits = np.empty(n, dtype=np.uint8)
    if n:
        _lib.check(
            ctx._lib.wos_walk_rows_host(
                ctx.handle, pset.handle, byref(wc), n, pts.ctypes.data, pid.ctypes.data,
                tid.ctypes.data, sgn.ctypes.data, values.ctypes.data, steps.ctypes.data,
                hits.ctypes.data,
            )
        )
    return values, steps, hits


def walk_screened_values(inst, points, point_ids, traj_ids, signs, cfg):
    """Batch interface of the delta-tracking walker, one row per walk (walker.py:322-357).

    Returns (values, steps, hits) like ``walk_poisson_values``; values are already
    divided by sqrt(alpha) at the start point.
    """
    inst = getattr(inst, "problem", inst)
    cfg = _cfg_of(cfg)
    if cfg.sigma_bar is None or cfg.sigma_bar <= 0.0:
        raise ValueError("delta tracking requires a positive cfg.sigma_bar")
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    if pts.ndim != 2:
        raise ValueError("points must be an (n, d) array")
    n = pts.shape[0]
    pid, tid, sgn = _streams_as_arrays(point_ids, traj_ids, signs, n)
    ctx = get_context()
    pset = problem_set(ctx, [inst])
    if pts.shape[1] != pset.dim:
        raise ValueError(f"expected points of dimension {pset.dim}, got shape {pts.shape}")
    wc = walk_config_struct(cfg.resolve_eps(inst.domain), cfg.max_steps, False, cfg.mode,
                            cfg.rng_seed, cfg.sigma_bar, philox_rounds=cfg.philox_rounds)
    values = np.empty(n, dtype=np.float64)
    steps = np.empty(n, dtype=np.int64)
    hits = np.empty(n, dtype=np.uint8)
    if n:
        check_screened(
            ctx._lib.wos_walk_rows_host(
                ctx.handle, pset.handle, byref(wc), n, pts.ctypes.data, pid.ctypes.data,
                tid.ctypes.data, sgn.ctypes.data, values.ctypes.data, steps.ctypes.data,
                hits.ctypes.data,
            )
        )
    return values, steps, hits


def walk_screened_delta(inst, xi, cfg, stream: TrajectoryStream | None = None) -> TrajectoryResult:
    """One delta-tracking trajectory from the interior point xi (walker.py:465-475)."""
    inst = getattr(inst, "problem", inst)
    cfg = _cfg_of(cfg)
    if cfg.sigma_bar is None or cfg.sigma_bar <= 0.0:
        raise ValueError("delta tracking requires a positive cfg.sigma_bar")
    _require_interior(inst, xi)
    s = stream or TrajectoryStream()
    out = walk_screened_values(
        inst, np.asarray(xi, dtype=np.float64)[None, :], [s.point_id], [s.traj_id], [s.sign], cfg
    )
    return _as_result(*out)


def _require_interior(inst, xi):
    """walker.py:426-428, evaluated on the GPU (wos_check_interior)."""
    ctx = get_context()
    pset = problem_set(ctx, [inst])
    pts = np.ascontiguousarray(np.asarray(xi, dtype=np.float64).reshape(1, -1))
    if pts.shape[1] != pset.dim:
        raise ValueError(f"expected a point of dimension {pset.dim}")
    first = c_int64(-1)
    _lib.check(
        ctx._lib.wos_check_interior_host(ctx.handle, pset.handle, 1, pts.ctypes.data, None, byref(first))
    )
    raise_exterior(pts, first.value)


def _as_result(values, steps, hits, i=0):
    term = TERM_BOUNDARY if hits[i] else TERM_MAX_STEPS
    return TrajectoryResult(float(values[i]), int(steps[i]), term)


def walk_poisson(inst, xi, cfg, stream: TrajectoryStream | None = None) -> TrajectoryResult:
    """One walk-on-spheres trajectory from the interior point xi (walker.py:436-444)."""
    inst = getattr(inst, "problem", inst)
    _require_interior(inst, xi)
    s = stream or TrajectoryStream()
    out = walk_poisson_values(
        inst, np.asarray(xi, dtype=np.float64)[None, :], [s.point_id], [s.traj_id], [s.sign], cfg
    )
    return _as_result(*out)


def walk_poisson_antithetic(inst, xi, cfg, stream: TrajectoryStream | None = None):
    """A mirrored pair of trajectories sharing one random stream (walker.py:447-462)."""
    inst = getattr(inst, "problem", inst)
    _require_interior(inst, xi)
    s = stream or TrajectoryStream()
    p = np.asarray(xi, dtype=np.float64)[None, :].repeat(2, axis=0)
    out = walk_poisson_values(inst, p, [s.point_id] * 2, [s.traj_id] * 2, [1.0, -1.0], cfg)
    return _as_result(*out, i=0), _as_result(*out, i=1)


__all__ += ["ExteriorQueryError"]
