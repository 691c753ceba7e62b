"""(kind, params) codes for domains, sources and boundaries.

Mirrors the reference's spec-coded problem terms (``_kernels.py:34-46``,
``walker.py:108-116,160-178``): a problem is GPU-codeable when its domain,
boundary and source reduce to a kind code plus a flat float64 parameter list.
The numeric values match the reference where the kinds overlap (SRC_NONE/CONST/
RBF2, BND_CONST/FOURIER5/LINEAR), so a reference ``Problem`` built with
``_kernels`` codes runs unchanged. Parameter layouts are documented in
``include/wos_b200.h``.

The reference solves  Laplacian(u) = f  and subtracts source samples; all
source params here are in that convention. Builders taking ``f`` for a
``-Laplacian(u) = f`` problem say so and negate.
"""

from __future__ import annotations

import numpy as np

# source kinds (_kernels.py:34-37 for the first three)
SRC_NONE = 0
SRC_CONST = 1
SRC_RBF2 = 2
SRC_SINE = 3
SRC_GAUSS = 4
# delta tracking: transformed coefficients of a ScreenedProblem (walker.py:120-136)
SRC_SCREENED_CONST = 5
SRC_SCREENED_VC = 6

# boundary kinds (_kernels.py:39-42 for the first three)
BND_CONST = 0
BND_FOURIER5 = 1
BND_LINEAR = 2
BND_FOURIER = 3
BND_SQUARE_ARCSINE = 4
BND_QUADRATIC = 5
BND_VC = 6

# domain kinds (_kernels.py:44-46: DOM_DISK = 0, DOM_POLAR = 1)
DOM_BALL = 0
DOM_POLAR = 1
DOM_BOX = 2
DOM_POLYGON = 3
DOM_MESH = 4

SRC_NAMES = {SRC_NONE: "none", SRC_CONST: "const", SRC_RBF2: "rbf2", SRC_SINE: "sine", SRC_GAUSS: "gauss",
             SRC_SCREENED_CONST: "screened_const", SRC_SCREENED_VC: "screened_vc"}
BND_NAMES = {
    BND_CONST: "const",
    BND_FOURIER5: "fourier5",
    BND_LINEAR: "linear",
    BND_FOURIER: "fourier",
    BND_SQUARE_ARCSINE: "square_arcsine",
    BND_QUADRATIC: "quadratic",
    BND_VC: "vc",
}


def _flat(values) -> tuple:
    return tuple(float(v) for v in np.asarray(values, dtype=np.float64).ravel())


def sine_source(coeffs, *, negate: bool = False):
    """f = sum a_{k..} prod_i sin(k_i pi x_i), k_i = 1..K; coeffs has shape (K,)*dim.

    ``negate=True`` turns the coefficients of a  -Laplacian(u) = f  problem into the
    reference's  Laplacian(u) = f  convention.
    """
    a = np.asarray(coeffs, dtype=np.float64)
    K = a.shape[0]
    if a.ndim not in (2, 3) or any(s != K for s in a.shape):
        raise ValueError("sine coefficients must be a (K, K) or (K, K, K) array")
    if negate:
        a = -a
    return (SRC_SINE, (float(K),) + _flat(a))


def gauss_source(center, sigma, amplitude=1.0, *, negate: bool = False):
    """f = A exp(-|x - c|^2 / (2 sigma^2))."""
    A = -float(amplitude) if negate else float(amplitude)
    return (SRC_GAUSS, (A, float(sigma)) + _flat(center))


def const_source(c):
    return (SRC_CONST, (float(c),))


def const_boundary(c):
    return (BND_CONST, (float(c),))


def linear_boundary(coeffs):
    return (BND_LINEAR, _flat(coeffs))


def fourier_boundary(b, c, b0=0.0):
    """g(t) = b0 + sum_{m=1..M} b_m cos(m t) + c_m sin(m t), t = polar angle of q."""
    b = np.asarray(b, dtype=np.float64).ravel()
    c = np.asarray(c, dtype=np.float64).ravel()
    if b.shape != c.shape:
        raise ValueError("Fourier cosine and sine coefficient counts differ")
    return (BND_FOURIER, (float(b.size), float(b0)) + _flat(b) + _flat(c))


def square_arcsine_boundary(coeffs, lo=(0.0, 0.0), side=1.0):
    """g = sum_m c_m sin(2 pi m s / (4 side)), s = CCW arc length from corner ``lo``."""
    c = np.asarray(coeffs, dtype=np.float64).ravel()
    return (BND_SQUARE_ARCSINE, (float(lo[0]), float(lo[1]), float(side), float(c.size)) + _flat(c))


def quadratic_boundary(axx=0.0, ayy=0.0, axy=0.0, ax=0.0, ay=0.0, a0=0.0):
    return (BND_QUADRATIC, (float(axx), float(ayy), float(axy), float(ax), float(ay), float(a0)))


def normalize(spec):
    """(kind, params) -> (int kind, tuple of floats)."""
    kind, params = spec
    return int(kind), _flat(params) if len(np.atleast_1d(params)) else ()
