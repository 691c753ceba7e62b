"""Express the BASELINE configs through the REFERENCE's own API (fixture generation only).

The reference package has no box, polygon, sine, Gaussian, Fourier-M, arc-length
or quadratic problem terms (finding 3). Its generic walk
path (walker.py:257-314) accepts any duck-typed domain with ``dim``,
``contains``, ``boundary_query`` and ``bounding_radius`` and any callables for
g and f, so these picklable adapters carry the configs' problem data into it.
Their arithmetic follows the parameter layouts of include/wos_b200.h; the
source callables return f in the reference's  Laplacian(u) = f  convention
(the spec params already hold -f).

Used only by tests/golden/make_golden.py, in this container, where
/root/reference is importable.
"""

from __future__ import annotations

import numpy as np

SRC_NONE, SRC_CONST, SRC_RBF2, SRC_SINE, SRC_GAUSS = 0, 1, 2, 3, 4
BND_CONST, BND_FOURIER5, BND_LINEAR, BND_FOURIER, BND_SQUARE_ARCSINE, BND_QUADRATIC = 0, 1, 2, 3, 4, 5
DOM_BALL, DOM_POLAR, DOM_BOX, DOM_POLYGON = 0, 1, 2, 3


def _pts(x, dim):
    p = np.asarray(x, dtype=np.float64)
    single = p.ndim == 1
    if single:
        p = p[None, :]
    return np.ascontiguousarray(p), single


class RefBox:
    def __init__(self, lo, hi):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.dim = self.lo.shape[0]

    def bounding_radius(self):
        return float(0.5 * np.linalg.norm(self.hi - self.lo))

    def contains(self, x):
        p, single = _pts(x, self.dim)
        inside = np.all((p > self.lo) & (p < self.hi), axis=1)
        return bool(inside[0]) if single else inside

    def boundary_query(self, x):
        p, single = _pts(x, self.dim)
        n = p.shape[0]
        cand = np.empty((n, 2 * self.dim))
        for i in range(self.dim):
            cand[:, 2 * i] = p[:, i] - self.lo[i]
            cand[:, 2 * i + 1] = self.hi[i] - p[:, i]
        k = np.argmin(cand, axis=1)  # first nearest face wins
        d = cand[np.arange(n), k]
        axis = k // 2
        face = np.where(k % 2 == 0, self.lo[axis], self.hi[axis])
        q = p.copy()
        q[np.arange(n), axis] = face
        if single:
            return float(d[0]), q[0]
        return d, q


class RefPolygon:
    dim = 2

    def __init__(self, vertices):
        self.v = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64))
        self.e = np.roll(self.v, -1, axis=0) - self.v

    def bounding_radius(self):
        lo, hi = self.v.min(axis=0), self.v.max(axis=0)
        c = 0.5 * (lo + hi)
        return float(np.max(np.hypot(*(self.v - c).T)))

    def contains(self, x):
        p, single = _pts(x, 2)
        a = self.v
        b = np.roll(a, -1, axis=0)
        py = p[:, 1:2]
        cond = (a[None, :, 1] > py) != (b[None, :, 1] > py)
        with np.errstate(divide="ignore", invalid="ignore"):
            xc = a[None, :, 0] + (py - a[None, :, 1]) * (b[None, :, 0] - a[None, :, 0]) / (
                b[None, :, 1] - a[None, :, 1])
        inside = (np.sum(cond & (p[:, 0:1] < xc), axis=1) % 2) == 1
        return bool(inside[0]) if single else inside

    def boundary_query(self, x):
        p, single = _pts(x, 2)
        ax, ay = self.v[:, 0][None, :], self.v[:, 1][None, :]
        ex, ey = self.e[:, 0][None, :], self.e[:, 1][None, :]
        wx = p[:, 0:1] - ax
        wy = p[:, 1:2] - ay
        t = np.clip((wx * ex + wy * ey) / (ex * ex + ey * ey), 0.0, 1.0)
        cx = ax + t * ex
        cy = ay + t * ey
        dx = p[:, 0:1] - cx
        dy = p[:, 1:2] - cy
        d2 = dx * dx + dy * dy
        k = np.argmin(d2, axis=1)
        r = np.arange(p.shape[0])
        d = np.sqrt(d2[r, k])
        q = np.column_stack([cx[r, k], cy[r, k]])
        if single:
            return float(d[0]), q[0]
        return d, q


class RefSource:
    def __init__(self, kind, params, dim):
        self.kind = int(kind)
        self.p = np.asarray(params, dtype=np.float64)
        self.dim = dim

    def __call__(self, y):
        y = np.asarray(y, dtype=np.float64)
        P = self.p
        if self.kind == SRC_CONST:
            return np.full(y.shape[0], P[0])
        if self.kind == SRC_SINE:
            K = int(P[0])
            a = P[1:].reshape((K,) * self.dim)
            k = np.arange(1, K + 1)
            S = [np.sin(np.outer(y[:, i], k) * np.pi) for i in range(self.dim)]
            if self.dim == 2:
                return np.einsum("kl,pk,pl->p", a, S[0], S[1])
            return np.einsum("ijk,pi,pj,pk->p", a, S[0], S[1], S[2])
        if self.kind == SRC_GAUSS:
            c = P[2 : 2 + self.dim]
            r2 = np.sum((y - c) ** 2, axis=1)
            return P[0] * np.exp(-r2 / (2.0 * P[1] * P[1]))
        raise ValueError(self.kind)


class RefBoundary:
    def __init__(self, kind, params, dim):
        self.kind = int(kind)
        self.p = np.asarray(params, dtype=np.float64)
        self.dim = dim

    def __call__(self, q):
        q = np.asarray(q, dtype=np.float64)
        B = self.p
        if self.kind == BND_CONST:
            return np.full(q.shape[0], B[0])
        if self.kind == BND_FOURIER:
            M = int(B[0])
            t = np.arctan2(q[:, 1], q[:, 0])
            g = np.full(q.shape[0], B[1])
            for m in range(1, M + 1):
                g = g + B[1 + m] * np.cos(m * t) + B[1 + M + m] * np.sin(m * t)
            return g
        if self.kind == BND_SQUARE_ARCSINE:
            x0, y0, side, M = B[0], B[1], B[2], int(B[3])
            u = (q[:, 0] - x0) / side
            v = (q[:, 1] - y0) / side
            db, dr, dt, dl = np.abs(v), np.abs(1.0 - u), np.abs(1.0 - v), np.abs(u)
            s = np.where(
                (db <= dr) & (db <= dt) & (db <= dl), u,
                np.where((dr <= dt) & (dr <= dl), 1.0 + v,
                         np.where(dt <= dl, 2.0 + (1.0 - u), 3.0 + (1.0 - v))))
            g = np.zeros(q.shape[0])
            for m in range(1, M + 1):
                g = g + B[3 + m] * np.sin(2.0 * np.pi * m * s / 4.0)
            return g
        if self.kind == BND_QUADRATIC:
            x, y = q[:, 0], q[:, 1]
            return B[0] * x * x + B[1] * y * y + B[2] * x * y + B[3] * x + B[4] * y + B[5]
        raise ValueError(self.kind)


def ref_problem(record, Problem, BallDomain):
    """Reference walker.Problem for one of our spec records (generic path: no specs)."""
    dim, dk, dp, sk, sp, bk, bp, ikey = record
    if dk == DOM_BOX:
        dom = RefBox(dp[:dim], dp[dim:])
    elif dk == DOM_POLYGON:
        n = int(dp[0])
        dom = RefPolygon(np.asarray(dp[1:], dtype=np.float64).reshape(n, 2))
    elif dk == DOM_BALL:
        dom = BallDomain(dp[:dim], dp[dim])
    else:
        raise ValueError(dk)
    src = None if sk == SRC_NONE else RefSource(sk, sp, dim)
    return Problem(dom, boundary=RefBoundary(bk, bp, dim), source=src, instance_key=int(ikey))
