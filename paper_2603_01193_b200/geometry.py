"""Domain descriptors for the GPU walker.

A domain is reduced to ``(dom_kind, params)`` (layouts in include/wos_b200.h).
``BallDomain`` keeps the reference's constructor and attribute names
(``geometry.py:172-238``) so reference code constructing it runs unchanged;
the reference's own ``BallDomain`` objects are accepted too (duck-typed on
``center``/``radius``). ``BoxDomain`` and ``PolygonDomain`` are new: the
reference has neither a 2D box nor a polygon (finding 3).

Host ``contains`` is plain numpy and is only meant for generating synthetic
inputs (rejection sampling); the estimator validates start points on the GPU
(``wos_check_interior``).
"""

from __future__ import annotations

import math

import numpy as np

from . import specs

__all__ = [
    "ExteriorQueryError",
    "UnsupportedDomainError",
    "BallDomain",
    "BoxDomain",
    "MeshDomain",
    "PolarDomain",
    "PolygonDomain",
    "mesh_params",
    "polar_params",
    "star_polygon",
    "domain_spec",
]


class ExteriorQueryError(ValueError):
    """A point-local query was made outside the domain (geometry.py:40-41)."""


class UnsupportedDomainError(TypeError):
    """The domain has no GPU encoding."""


def _as_points(x, dim):
    pts = np.asarray(x, dtype=np.float64)
    single = pts.ndim == 1
    if single:
        pts = pts[None, :]
    if pts.ndim != 2 or pts.shape[1] != dim:
        raise ValueError(f"expected points of dimension {dim}, got shape {pts.shape}")
    return pts, single


class BallDomain:
    """Disk (2D) or ball (3D); same constructor as the reference (geometry.py:175-183)."""

    def __init__(self, center, radius):
        self.center = np.asarray(center, dtype=np.float64)
        if self.center.ndim != 1 or self.center.shape[0] not in (2, 3):
            raise ValueError("center must be a 2- or 3-vector")
        if radius <= 0.0:
            raise ValueError("radius must be positive")
        self.radius = float(radius)
        self.dim = self.center.shape[0]

    def bounding_radius(self):
        return self.radius

    def bounding_box(self):
        return self.center - self.radius, self.center + self.radius

    def contains(self, x):
        pts, single = _as_points(x, self.dim)
        inside = np.linalg.norm(pts - self.center, axis=1) < self.radius
        return bool(inside[0]) if single else inside

    def spec(self):
        return specs.DOM_BALL, tuple(self.center.tolist()) + (self.radius,)

    def __repr__(self):
        return f"BallDomain(center={self.center.tolist()}, radius={self.radius})"


class BoxDomain:
    """Axis-aligned box [lo, hi] in 2D or 3D."""

    def __init__(self, lo, hi):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        if self.lo.shape != self.hi.shape or self.lo.ndim != 1 or self.lo.shape[0] not in (2, 3):
            raise ValueError("lo/hi must be matching 2- or 3-vectors")
        if np.any(self.hi <= self.lo):
            raise ValueError("box must have positive extent")
        self.dim = self.lo.shape[0]

    def bounding_radius(self):
        return float(0.5 * np.linalg.norm(self.hi - self.lo))

    def bounding_box(self):
        return self.lo.copy(), self.hi.copy()

    def contains(self, x):
        pts, single = _as_points(x, self.dim)
        inside = np.all((pts > self.lo) & (pts < self.hi), axis=1)
        return bool(inside[0]) if single else inside

    def spec(self):
        return specs.DOM_BOX, tuple(self.lo.tolist()) + tuple(self.hi.tolist())

    def __repr__(self):
        return f"BoxDomain(lo={self.lo.tolist()}, hi={self.hi.tolist()})"


class PolygonDomain:
    """Closed simple 2D polygon with vertices in order (segments v_i -> v_{i+1})."""

    dim = 2

    def __init__(self, vertices):
        v = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64))
        if v.ndim != 2 or v.shape[1] != 2 or v.shape[0] < 3:
            raise ValueError("polygon needs an (n >= 3, 2) vertex array")
        self.vertices = v

    def bounding_box(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    def bounding_radius(self):
        lo, hi = self.bounding_box()
        c = 0.5 * (lo + hi)
        return float(np.max(np.hypot(*(self.vertices - c).T)))

    def contains(self, x):
        """Crossing-number test (even-odd rule)."""
        pts, single = _as_points(x, 2)
        a = self.vertices
        b = np.roll(a, -1, axis=0)
        px = pts[:, 0:1]
        py = pts[:, 1:2]
        cond = (a[None, :, 1] > py) != (b[None, :, 1] > py)
        with np.errstate(divide="ignore", invalid="ignore"):
            xc = a[None, :, 0] + (py - a[None, :, 1]) * (b[None, :, 0] - a[None, :, 0]) / (
                b[None, :, 1] - a[None, :, 1]
            )
        crossings = np.sum(cond & (px < xc), axis=1)
        inside = (crossings % 2) == 1
        return bool(inside[0]) if single else inside

    def sample_interior(self, n, rng):
        """Uniform interior points by rejection from the bounding box."""
        lo, hi = self.bounding_box()
        out = np.empty((n, 2))
        filled = 0
        while filled < n:
            cand = rng.uniform(lo, hi, size=(max(4096, 2 * (n - filled)), 2))
            hits = cand[self.contains(cand)]
            take = min(hits.shape[0], n - filled)
            out[filled : filled + take] = hits[:take]
            filled += take
        return out

    def spec(self):
        return specs.DOM_POLYGON, (float(self.vertices.shape[0]),) + tuple(self.vertices.ravel().tolist())

    def __repr__(self):
        return f"PolygonDomain(n={self.vertices.shape[0]})"


class PolarDomain:
    """Star-shaped 2D domain r(t) = r0 (1 + c1 cos 4t + c2 cos 8t) (geometry.py:83-153).

    Same constructor, table and scan stride as the reference: the curve is tabulated
    at ``table_size`` angles with numpy (so the GPU replays the reference's table bit
    for bit) and mild curves (|c1| + |c2| <= 0.45) are scanned with stride 64.
    """

    dim = 2
    _FAST_SCAN_LIMIT = 0.45

    def __init__(self, r0=1.0, c1=0.0, c2=0.0, *, table_size=4096):
        if r0 <= 0.0:
            raise ValueError("r0 must be positive")
        if abs(c1) + abs(c2) >= 1.0:
            raise ValueError("|c1| + |c2| must be < 1 for a valid boundary")
        self.r0, self.c1, self.c2 = float(r0), float(c1), float(c2)
        self.table_size = int(table_size)
        theta = np.arange(self.table_size) * (2.0 * np.pi / self.table_size)
        r = self.radius(theta)
        self._bx = np.ascontiguousarray(r * np.cos(theta))
        self._by = np.ascontiguousarray(r * np.sin(theta))
        self._stride = 64 if abs(c1) + abs(c2) <= self._FAST_SCAN_LIMIT else 1
        self._lo = np.array([self._bx.min(), self._by.min()])
        self._hi = np.array([self._bx.max(), self._by.max()])

    def radius(self, theta):
        theta = np.asarray(theta, dtype=np.float64)
        return self.r0 * (1.0 + self.c1 * np.cos(4.0 * theta) + self.c2 * np.cos(8.0 * theta))

    def bounding_box(self):
        return self._lo.copy(), self._hi.copy()

    def bounding_radius(self):
        center = 0.5 * (self._lo + self._hi)
        return float(np.hypot(self._bx - center[0], self._by - center[1]).max())

    def contains(self, x):
        pts, single = _as_points(x, 2)
        inside = np.hypot(pts[:, 0], pts[:, 1]) < self.radius(np.arctan2(pts[:, 1], pts[:, 0]))
        return bool(inside[0]) if single else inside

    def spec(self):
        return specs.DOM_POLAR, polar_params(self)

    def __repr__(self):
        return f"PolarDomain(r0={self.r0}, c1={self.c1}, c2={self.c2})"


class MeshDomain:
    """Closed, consistently oriented triangle mesh (3D), geometry.MeshDomain (geometry.py:400-580).

    Same constructor as the reference. Distances, closest points and the inside test
    (angle-weighted pseudo-normal of the closest feature) run on the GPU over a BVH the
    library builds (WOS_DOM_MESH); start points are validated there by ``estimate``.
    """

    dim = 3

    def __init__(self, vertices, faces):
        v = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64))
        f = np.ascontiguousarray(np.asarray(faces, dtype=np.int64))
        if v.ndim != 2 or v.shape[1] != 3:
            raise ValueError("vertices must be (n, 3)")
        if f.ndim != 2 or f.shape[1] != 3:
            raise ValueError("faces must be (m, 3) triangles")
        if f.min() < 0 or f.max() >= v.shape[0]:
            raise ValueError("face index out of range")
        tri = v[f]
        if np.any(np.linalg.norm(np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]), axis=1) == 0.0):
            raise ValueError("degenerate triangle in mesh")
        self.vertices = v
        self.faces = f
        self._lo = v.min(axis=0)
        self._hi = v.max(axis=0)

    def bounding_box(self):
        return self._lo.copy(), self._hi.copy()

    def bounding_radius(self):
        center = 0.5 * (self._lo + self._hi)
        return float(np.linalg.norm(self.vertices - center, axis=1).max())

    def spec(self):
        return specs.DOM_MESH, mesh_params(self)

    def __repr__(self):
        return f"MeshDomain({self.vertices.shape[0]} vertices, {self.faces.shape[0]} faces)"


def mesh_params(dom):
    """[nv, nf, vertices..., faces...] of a MeshDomain (ours or the reference's)."""
    v = np.asarray(dom.vertices, dtype=np.float64)
    f = np.asarray(dom.faces, dtype=np.int64)
    return (float(v.shape[0]), float(f.shape[0])) + tuple(v.ravel().tolist()) + tuple(
        f.astype(np.float64).ravel().tolist())


def polar_params(dom):
    """[r0, c1, c2, stride, n, bx..., by...] of a PolarDomain (ours or the reference's)."""
    return ((float(dom.r0), float(dom.c1), float(dom.c2), float(dom._stride), float(dom._bx.size))
            + tuple(np.asarray(dom._bx, np.float64).tolist()) + tuple(np.asarray(dom._by, np.float64).tolist()))


def star_polygon(alpha, beta, n_vertices=128, r0=1.0):
    """Star-shaped polygon r(t) = r0 (1 + sum_m alpha_m cos(m t) + beta_m sin(m t)), m = 2.., at
    t_j = 2 pi j / n (BASELINE config 3)."""
    t = 2.0 * math.pi * np.arange(n_vertices) / n_vertices
    r = np.full(n_vertices, 1.0)
    for i, (a, b) in enumerate(zip(alpha, beta)):
        m = i + 2
        r += a * np.cos(m * t) + b * np.sin(m * t)
    r *= r0
    return PolygonDomain(np.column_stack([r * np.cos(t), r * np.sin(t)]))


def domain_spec(dom):
    """(dom_kind, params, dim) for our domains and the reference's BallDomain."""
    if hasattr(dom, "spec"):
        kind, params = dom.spec()
        return kind, params, int(dom.dim)
    name = type(dom).__name__
    if name == "BallDomain" and hasattr(dom, "center") and hasattr(dom, "radius"):
        c = np.asarray(dom.center, dtype=np.float64)
        return specs.DOM_BALL, tuple(c.tolist()) + (float(dom.radius),), int(c.shape[0])
    if name == "PolarDomain" and hasattr(dom, "_bx") and hasattr(dom, "r0"):
        return specs.DOM_POLAR, polar_params(dom), 2
    if name == "MeshDomain" and hasattr(dom, "vertices") and hasattr(dom, "faces"):
        return specs.DOM_MESH, mesh_params(dom), 3
    raise UnsupportedDomainError(
        f"{name} has no GPU encoding (supported: BallDomain, BoxDomain, PolygonDomain, PolarDomain, "
        "MeshDomain)"
    )
