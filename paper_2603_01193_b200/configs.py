"""The five BASELINE.json synthetic configurations, with every unstated choice pinned.

All inputs are seeded synthetic data (no dataset exists for this path). Each
builder returns a ``Workload``: problems in the reference's  Laplacian(u) = f
convention (BASELINE states  -Laplacian(u) = f, so source coefficients are
negated; SURVEY.md section 0 finding 2), the concatenated query points, their
point ids and instance index, L, and the WalkConfig.

PINs:
  * coefficients and points come from ``np.random.default_rng(config index)``,
    drawn in the order written below;
  * grids are cell centres, point ids are flat lattice indices (C order, like
    cli._build_points, cli.py:223-251);
  * cfg1 keeps lattice points with r < 0.99 (3160 points);
  * cfg2's boundary is  g = sum_{m=1..4} c_m sin(2 pi m s / 4), s = CCW arc length
    from (0, 0); instance j has instance_key j and point ids 0..4095;
  * cfg3's 128 vertices sit at t_j = 2 pi j / 128; c is area-uniform in the disk
    of radius 0.3; points by rejection from the polygon's bounding box;
  * rng_seed = 0 for every config; replicas vary traj_start.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import specs
from .geometry import BallDomain, BoxDomain, PolygonDomain, star_polygon
from .walker import Problem, WalkConfig

__all__ = ["Workload", "build", "CONFIG_NAMES", "n_configs"]

CONFIG_NAMES = {
    0: "cfg0_square_sine_poisson",
    1: "cfg1_disk_fourier_laplace",
    2: "cfg2_square_batch64_weak_labels",
    3: "cfg3_star_polygons32_gauss",
    4: "cfg4_cube_sine_poisson_3d",
}


@dataclass
class Workload:
    index: int
    name: str
    dim: int
    problems: list
    points: np.ndarray  # (P, dim) float64, all instances concatenated
    point_ids: np.ndarray  # (P,) int64
    inst_index: np.ndarray  # (P,) int32
    L: int
    cfg: WalkConfig
    analytic: object = None  # callable(points (P, dim)) -> (P,) or None
    meta: dict = field(default_factory=dict)

    @property
    def n_points(self) -> int:
        return int(self.points.shape[0])

    @property
    def n_walks(self) -> int:
        return self.n_points * self.L

    def subset(self, idx):
        idx = np.asarray(idx)
        return Workload(
            self.index, self.name, self.dim, self.problems, self.points[idx], self.point_ids[idx],
            self.inst_index[idx], self.L, self.cfg, self.analytic, dict(self.meta),
        )

    def replicate(self, R: int):
        """R independent label replicas of every point in one batch.

        Replica r of point p gets point id r * (max id + 1) + id, i.e. its own Philox
        streams: R independent estimates of the same labels (small
        configs are measured with replicas per launch).
        """
        if R <= 1:
            return self
        span = int(self.point_ids.max()) + 1
        ids = np.concatenate([self.point_ids + r * span for r in range(R)])
        return Workload(
            self.index, self.name, self.dim, self.problems, np.tile(self.points, (R, 1)), ids,
            np.tile(self.inst_index, R), self.L, self.cfg, self.analytic,
            dict(self.meta, replicas=R),
        )

    def with_mode(self, mode: str):
        c = self.cfg
        cfg = WalkConfig(c.eps_shell, c.max_steps, c.antithetic, c.sigma_bar, c.rng_seed, mode)
        return Workload(
            self.index, self.name, self.dim, self.problems, self.points, self.point_ids,
            self.inst_index, self.L, cfg, self.analytic, dict(self.meta),
        )


def n_configs() -> int:
    return len(CONFIG_NAMES)


def _cell_centres(n, lo, hi, dim):
    ax = lo + (np.arange(n) + 0.5) * ((hi - lo) / n)
    mesh = np.meshgrid(*([ax] * dim), indexing="ij")
    return np.column_stack([m.ravel() for m in mesh])


def sine_series(a, pts):
    """sum a_{k..} prod sin(k pi x) for a (K,)*dim coefficient array."""
    K = a.shape[0]
    dim = a.ndim
    k = np.arange(1, K + 1)
    S = [np.sin(np.pi * np.outer(pts[:, i], k)) for i in range(dim)]
    if dim == 2:
        return np.einsum("kl,pk,pl->p", a, S[0], S[1])
    return np.einsum("ijk,pi,pj,pk->p", a, S[0], S[1], S[2])


def _cfg0(scale: float = 1.0):
    rng = np.random.default_rng(0)
    K = 4
    k = np.arange(1, K + 1)
    denom = k[:, None] ** 2 + k[None, :] ** 2
    a = rng.standard_normal((K, K)) / denom
    n = 32
    pts = _cell_centres(n, 0.0, 1.0, 2)
    dom = BoxDomain([0.0, 0.0], [1.0, 1.0])
    prob = Problem(
        dom, boundary_spec=specs.const_boundary(0.0), source_spec=specs.sine_source(a, negate=True)
    )
    P = pts.shape[0]
    u_coef = a / (np.pi**2 * denom)
    return Workload(
        0, CONFIG_NAMES[0], 2, [prob], pts, np.arange(P, dtype=np.int64), np.zeros(P, np.int32),
        256, WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=0),
        analytic=lambda p: sine_series(u_coef, p), meta={"a": a},
    )


def _cfg1(scale: float = 1.0):
    rng = np.random.default_rng(1)
    M = 8
    m = np.arange(1, M + 1)
    b = rng.standard_normal(M) / m
    c = rng.standard_normal(M) / m
    n = 64
    grid = _cell_centres(n, -1.0, 1.0, 2)
    ids = np.arange(grid.shape[0], dtype=np.int64)
    keep = np.hypot(grid[:, 0], grid[:, 1]) < 0.99
    pts, ids = grid[keep], ids[keep]
    dom = BallDomain([0.0, 0.0], 1.0)
    prob = Problem(dom, boundary_spec=specs.fourier_boundary(b, c))

    def analytic(p):
        r = np.hypot(p[:, 0], p[:, 1])
        t = np.arctan2(p[:, 1], p[:, 0])
        return sum(r**mm * (b[mm - 1] * np.cos(mm * t) + c[mm - 1] * np.sin(mm * t)) for mm in m)

    return Workload(
        1, CONFIG_NAMES[1], 2, [prob], pts, ids, np.zeros(pts.shape[0], np.int32), 1024,
        WalkConfig(eps_shell=1e-4, max_steps=2000, rng_seed=0), analytic=analytic,
        meta={"b": b, "c": c},
    )


def _cfg2(scale: float = 1.0):
    rng = np.random.default_rng(2)
    n_inst = 64
    K = 8
    npts = 4096
    k = np.arange(1, K + 1)
    denom = (k[:, None] ** 2 + k[None, :] ** 2) ** 1.5
    dom = BoxDomain([0.0, 0.0], [1.0, 1.0])
    problems, pts, ids, inst, coeffs = [], [], [], [], []
    for j in range(n_inst):
        a = rng.standard_normal((K, K)) / denom
        cm = rng.normal(0.0, 0.1, size=4)
        p = rng.uniform(0.0, 1.0, size=(npts, 2))
        problems.append(
            Problem(
                dom, instance_key=j,
                boundary_spec=specs.square_arcsine_boundary(cm, (0.0, 0.0), 1.0),
                source_spec=specs.sine_source(a, negate=True),
            )
        )
        coeffs.append((a, cm))
        pts.append(p)
        ids.append(np.arange(npts, dtype=np.int64))
        inst.append(np.full(npts, j, np.int32))
    return Workload(
        2, CONFIG_NAMES[2], 2, problems, np.concatenate(pts), np.concatenate(ids),
        np.concatenate(inst), 4, WalkConfig(eps_shell=1e-3, max_steps=500, rng_seed=0),
        meta={"coeffs": coeffs},
    )


def _cfg3(scale: float = 1.0):
    rng = np.random.default_rng(3)
    n_dom = 32
    npts = 8192
    problems, pts, ids, inst, meta = [], [], [], [], []
    for j in range(n_dom):
        alpha = rng.uniform(-0.08, 0.08, size=4)
        beta = rng.uniform(-0.08, 0.08, size=4)
        rc = 0.3 * math.sqrt(rng.uniform())
        tc = 2.0 * math.pi * rng.uniform()
        center = (rc * math.cos(tc), rc * math.sin(tc))
        poly = star_polygon(alpha, beta, 128)
        p = poly.sample_interior(npts, rng)
        problems.append(
            Problem(
                poly, instance_key=j,
                boundary_spec=specs.quadratic_boundary(axx=1.0, ayy=-1.0),
                source_spec=specs.gauss_source(center, 0.2, 1.0, negate=True),
            )
        )
        meta.append({"alpha": alpha, "beta": beta, "center": center})
        pts.append(p)
        ids.append(np.arange(npts, dtype=np.int64))
        inst.append(np.full(npts, j, np.int32))
    return Workload(
        3, CONFIG_NAMES[3], 2, problems, np.concatenate(pts), np.concatenate(ids),
        np.concatenate(inst), 64, WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=0),
        meta={"polygons": meta},
    )


def _cfg4(scale: float = 1.0):
    rng = np.random.default_rng(4)
    K = 3
    k = np.arange(1, K + 1)
    denom = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    a = rng.standard_normal((K, K, K)) / denom
    n = 64
    pts = _cell_centres(n, 0.0, 1.0, 3)
    dom = BoxDomain([0.0, 0.0, 0.0], [1.0, 1.0, 1.0])
    prob = Problem(
        dom, boundary_spec=specs.const_boundary(0.0), source_spec=specs.sine_source(a, negate=True)
    )
    P = pts.shape[0]
    u_coef = a / (np.pi**2 * denom)
    return Workload(
        4, CONFIG_NAMES[4], 3, [prob], pts, np.arange(P, dtype=np.int64), np.zeros(P, np.int32),
        256, WalkConfig(eps_shell=1e-3, max_steps=1000, rng_seed=0),
        analytic=lambda p: sine_series(u_coef, p), meta={"a": a},
    )


_BUILDERS = {0: _cfg0, 1: _cfg1, 2: _cfg2, 3: _cfg3, 4: _cfg4}


def build(index: int, mode: str = "native") -> Workload:
    """Workload for BASELINE config ``index`` (0..4) in the given walk mode."""
    w = _BUILDERS[int(index)]()
    return w.with_mode(mode)
