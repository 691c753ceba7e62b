"""GPU distance queries vs closed forms and brute force (reference test_geometry.py).

The walk API exposes the device query through the exit point: with an eps shell
larger than the domain every walk stops at step 0 and returns g at the projection
of its start point, so linear g = x_i recovers the closest boundary point q and the
distance |p - q| (walker.py:275-281). Mirrors test_geometry.py:60-80 (polar
distance vs brute force, oscillating curve near the centre), :201-242 (cube signed
distance in closed form, BVH == brute force) and test_walker.py:170-176 (harmonic
linear data on a mesh).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def projections(domain, pts, mode):
    from paper_2603_01193_b200 import Problem, WalkConfig, walk_poisson_values

    pts = np.asarray(pts, dtype=np.float64)
    dim = pts.shape[1]
    n = pts.shape[0]
    q = np.empty_like(pts)
    for i in range(dim):
        coeffs = [0.0] * (dim + 1)
        coeffs[i] = 1.0
        prob = Problem(domain, boundary_spec=(2, tuple(coeffs)))
        v, s, h = walk_poisson_values(prob, pts, np.zeros(n, np.int64), np.arange(n), np.ones(n),
                                      WalkConfig(eps_shell=100.0, max_steps=1, mode=mode))
        assert np.all(s == 0) and np.all(h == 1)
        q[:, i] = v
    return q, np.linalg.norm(pts - q, axis=1)


def brute_polar_distance(dom, p, n=200_000):
    t = np.linspace(0.0, 2.0 * np.pi, n, endpoint=False)
    r = dom.radius(t)
    d = np.hypot(r * np.cos(t) - p[0], r * np.sin(t) - p[1])
    k = int(np.argmin(d))
    # refine the dense winner on a fine local grid
    tt = np.linspace(t[k] - 2 * np.pi / n, t[k] + 2 * np.pi / n, 2001)
    rr = dom.radius(tt)
    return float(np.min(np.hypot(rr * np.cos(tt) - p[0], rr * np.sin(tt) - p[1])))


@pytest.mark.parametrize("mode,tol", [("replay", 1e-6), ("native", 2e-5)])
def test_polar_distance_matches_brute_force(gpu, mode, tol):
    from paper_2603_01193_b200 import PolarDomain

    dom = PolarDomain(1.0, 0.18, -0.12)
    rng = np.random.default_rng(42)
    lo, hi = dom.bounding_box()
    cand = lo + (hi - lo) * rng.random((400, 2))
    pts = cand[dom.contains(cand)][:40]
    _, d = projections(dom, pts, mode)
    want = np.array([brute_polar_distance(dom, p) for p in pts])
    assert np.max(np.abs(d - want)) < tol * dom.r0


@pytest.mark.parametrize("mode,tol", [("replay", 1e-6), ("native", 2e-5)])
def test_polar_distance_near_centre_of_oscillating_curve(gpu, mode, tol):
    from paper_2603_01193_b200 import PolarDomain

    dom = PolarDomain(1.0, 0.2, 0.2)
    pts = np.array([[0.0, 0.0], [1e-3, -2e-3], [0.05, 0.02]])
    _, d = projections(dom, pts, mode)
    want = np.array([brute_polar_distance(dom, p) for p in pts])
    assert np.max(np.abs(d - want)) < tol


@pytest.mark.parametrize("mode,tol", [("replay", 1e-12), ("native", 1e-6)])
def test_cube_mesh_distance_closed_form(gpu, mode, tol):
    from paper_2603_01193_b200 import MeshDomain

    corners = np.array([[sx, sy, sz] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)], float)
    faces = np.array([[0, 1, 3], [0, 3, 2], [4, 6, 7], [4, 7, 5], [0, 4, 5], [0, 5, 1],
                      [2, 3, 7], [2, 7, 6], [0, 2, 6], [0, 6, 4], [1, 5, 7], [1, 7, 3]])
    mesh = MeshDomain(corners, faces)
    pts = np.random.default_rng(9).uniform(-0.99, 0.99, size=(300, 3))
    _, d = projections(mesh, pts, mode)
    want = -np.max(np.abs(pts) - 1.0, axis=1)  # interior distance to the cube surface
    assert np.max(np.abs(d - want)) < tol


def _icosphere(sub):
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
         (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    v = [np.array(p, float) / np.linalg.norm(p) for p in v]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
         (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(sub):
        mid = {}

        def m(i, j):
            k = (min(i, j), max(i, j))
            if k not in mid:
                p = v[i] + v[j]
                v.append(p / np.linalg.norm(p))
                mid[k] = len(v) - 1
            return mid[k]

        nf = []
        for i, j, k in f:
            a, b, c = m(i, j), m(j, k), m(k, i)
            nf += [(i, a, c), (j, b, a), (k, c, b), (a, b, c)]
        f = nf
    return np.array(v), np.array(f)


def test_mesh_bvh_equals_brute_force(gpu):
    """The device BVH distance equals the oracle's brute-force scan bit for bit."""
    from oracle import oracle as O
    from paper_2603_01193_b200 import MeshDomain, Problem

    V, F = _icosphere(3)
    mesh = MeshDomain(V, F)
    rng = np.random.default_rng(17)
    v = rng.normal(size=(200, 3))
    pts = v / np.linalg.norm(v, axis=1)[:, None] * (0.95 * rng.random(200) ** (1 / 3))[:, None]
    q, d = projections(mesh, pts, "replay")
    prob = Problem(mesh, boundary_spec=(2, (1.0, 0.0, 0.0, 0.0)))
    vo, _, _ = O.walk_rows(prob, pts, np.zeros(200, np.int64), np.arange(200), np.ones(200), seed=0,
                           eps=100.0, max_steps=1)
    assert np.allclose(q[:, 0], vo, rtol=0, atol=1e-12)
    # inscribed sphere: the surface sits slightly inside the unit sphere
    assert np.all(d <= 1.0 - np.linalg.norm(pts, axis=1) + 1e-12)
    assert np.max(np.abs(d - (1.0 - np.linalg.norm(pts, axis=1)))) < 6e-3


@pytest.mark.parametrize("mode", ["replay", "native"])
def test_mesh_walk_harmonic_linear(gpu, mode):
    """g = x0 is harmonic, so the estimate equals it inside the cube (test_walker.py:170-176)."""
    from paper_2603_01193_b200 import MeshDomain, Problem, WalkConfig, estimate

    corners = np.array([[sx, sy, sz] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)], float)
    faces = np.array([[0, 1, 3], [0, 3, 2], [4, 6, 7], [4, 7, 5], [0, 4, 5], [0, 5, 1],
                      [2, 3, 7], [2, 7, 6], [0, 2, 6], [0, 6, 4], [1, 5, 7], [1, 7, 3]])
    prob = Problem(MeshDomain(corners, faces), boundary_spec=(2, (1.0, 0.0, 0.0, 0.0)))
    (e,) = estimate(prob, [[0.25, 0.1, -0.4]], 20_000, WalkConfig(rng_seed=6, mode=mode))
    assert abs(e.mean - 0.25) < 4.0 * e.std_error


def _brute_polygon(V, p):
    """fp64 full scan: distance, closest point and FIRST nearest segment (the reference's
    min over segments, geometry.py polygon adapter / oracle query())."""
    A = V
    B = np.roll(V, -1, axis=0)
    E = B - A
    W = p[None, :] - A
    t = np.clip((W * E).sum(1) / (E * E).sum(1), 0.0, 1.0)
    C = A + t[:, None] * E
    d = np.hypot(*(p[None, :] - C).T)
    k = int(np.argmin(d))
    return d[k], C[k]


def _comb_polygon(n=20):
    """A concave comb: the unit square with n deep notches cut from the top edge, so
    cell candidate lists mix near and far teeth."""
    v = [(0.0, 0.0), (1.0, 0.0), (1.0, 1.0)]
    for k in range(n - 1, -1, -1):
        xa, xb = (k + 0.7) / n, (k + 0.3) / n
        v += [(xa, 1.0), (xa, 0.35), (xb, 0.35), (xb, 1.0)]
    v.append((0.0, 1.0))
    return np.array(v)


@pytest.mark.parametrize("mode,tol", [("replay", 1e-12), ("native", 3e-6)])
@pytest.mark.parametrize("shape", ["star128", "star97", "comb"])
def test_polygon_distance_candidate_grid(gpu, mode, tol, shape):
    """Polygons with >= 24 vertices answer NATIVE queries through the candidate grid
    (wos_capi.cu build_poly_grid): distance and closest point equal the full fp64 scan
    (odd vertex counts add a zero-length pad segment; the comb is strongly concave)."""
    from paper_2603_01193_b200 import PolygonDomain, star_polygon

    if shape == "star128":
        dom = star_polygon([0.07, -0.05, 0.04, 0.03], [0.02, 0.06, -0.04, 0.02], 128)
    elif shape == "star97":
        dom = star_polygon([0.3, -0.2, 0.1, 0.05], [0.1, 0.2, -0.1, 0.05], 97)
    else:
        dom = PolygonDomain(_comb_polygon())
    V = np.asarray(dom.vertices, float)
    assert len(V) >= 24
    rng = np.random.default_rng(5)
    lo, hi = V.min(0), V.max(0)
    cand = lo + (hi - lo) * rng.random((6000, 2))
    pts = cand[dom.contains(cand)][:300]
    # and points hugging the boundary (where walks spend their steps)
    mid = 0.5 * (V + np.roll(V, -1, axis=0))
    cen = V.mean(0)
    near = mid + 1e-3 * (cen - mid) / np.linalg.norm(cen - mid, axis=1)[:, None]
    pts = np.vstack([pts, near[dom.contains(near)][:100]])
    q, d = projections(dom, pts, mode)
    for p, qi, di in zip(pts, q, d):
        want_d, want_q = _brute_polygon(V, p)
        assert abs(di - want_d) <= tol * max(1.0, want_d), (p, di, want_d)
        # the closest point is on the boundary at the minimum distance
        assert abs(np.hypot(*(p - qi)) - want_d) <= 10 * tol
