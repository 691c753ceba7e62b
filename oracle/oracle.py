"""TEST INFRASTRUCTURE ONLY — Python handle on the CPU oracle (oracle/wos_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; the product package never does. See wos_oracle.c for the
reference file:line each routine restates.

Also holds the exact-integer Philox restatements used as known-answer
references (the method of the reference's own tests/test_rng.py:11-26).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libwos_oracle.so")

MASK64 = (1 << 64) - 1
MASK32 = (1 << 32) - 1


class _Problem(ctypes.Structure):
    _fields_ = [
        ("dim", c_int32),
        ("dom_kind", c_int32),
        ("n_dom", c_int32),
        ("dom", POINTER(c_double)),
        ("src_kind", c_int32),
        ("n_src", c_int32),
        ("src", POINTER(c_double)),
        ("bnd_kind", c_int32),
        ("n_bnd", c_int32),
        ("bnd", POINTER(c_double)),
        ("instance_key", c_uint64),
    ]


_lib = None


def build():
    """Compile the oracle with its Makefile (gcc; seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = c_void_p
        L.oracle_walk_rows.argtypes = [P, c_int64, P, P, P, P, c_uint64, c_double, c_int64, P, P, P, c_int]
        L.oracle_walk_rows_native.argtypes = L.oracle_walk_rows.argtypes
        L.oracle_estimate.argtypes = [
            P, c_int, c_int64, P, P, P, c_int64, c_uint64, c_int, c_uint64, c_double, c_int64, P, P,
            P, c_int,
        ]
        L.oracle_philox4x64.argtypes = [c_int64, P, c_uint64, c_uint64, P]
        L.oracle_philox4x32.argtypes = [c_int64, P, c_uint32, c_uint32, P]
        L.oracle_philox4x32_rounds.argtypes = [c_int64, P, c_uint32, c_uint32, c_int, P]
        L.oracle_set_philox_rounds.argtypes = [c_int]
        L.oracle_beta_table.argtypes = [P]
        L.oracle_green2_table.argtypes = [P]
        L.oracle_contains.argtypes = [P, P]
        L.oracle_contains.restype = c_int
        L.oracle_set_sigma_bar.argtypes = [c_double]
        L.oracle_majorant.restype = c_double
        _lib = L
    return _lib


def _record(problem):
    """Problem (ours or reference-shaped) or record tuple -> record tuple."""
    if isinstance(problem, tuple) and len(problem) == 8:
        return problem
    from paper_2603_01193_b200.engine import problem_record  # pure Python, no GPU

    return problem_record(problem)


class _Problems:
    """ctypes array of oracle problems keeping their parameter buffers alive."""

    def __init__(self, problems):
        recs = [_record(p) for p in problems]
        self.dim = recs[0][0]
        self.keep = []
        self.arr = (_Problem * len(recs))()
        dbl = POINTER(c_double)
        for i, (dim, dk, dp, sk, sp, bk, bp, ikey) in enumerate(recs):
            d = np.ascontiguousarray(np.asarray(dp or (0.0,), np.float64))
            s = np.ascontiguousarray(np.asarray(sp or (0.0,), np.float64))
            b = np.ascontiguousarray(np.asarray(bp or (0.0,), np.float64))
            self.keep += [d, s, b]
            self.arr[i] = _Problem(
                dim, dk, len(dp), d.ctypes.data_as(dbl), sk, len(sp), s.ctypes.data_as(dbl), bk,
                len(bp), b.ctypes.data_as(dbl), int(ikey) & MASK64,
            )

    @property
    def ptr(self):
        return ctypes.addressof(self.arr)


def default_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def walk_rows(problem, points, point_ids, traj_ids, signs, *, seed, eps, max_steps, native=False,
              nthreads=None, sigma_bar=0.0, philox_rounds=10):
    """(values, steps, hits) like walker.walk_poisson_values (reference form by default).

    Screened problems walk by delta tracking with majorant ``sigma_bar``
    (walker.walk_screened_values); ``majorant()`` then reports a violation.
    """
    lib = load()
    lib.oracle_set_sigma_bar(float(sigma_bar))
    lib.oracle_set_philox_rounds(int(philox_rounds))
    pr = _Problems([problem])
    pts = np.ascontiguousarray(np.asarray(points, np.float64))
    n = pts.shape[0]
    pid = np.ascontiguousarray(np.asarray(point_ids).astype(np.int64).astype(np.uint64))
    tid = np.ascontiguousarray(np.asarray(traj_ids).astype(np.int64).astype(np.uint64))
    sgn = np.ascontiguousarray(np.asarray(signs, np.float64))
    values = np.empty(n)
    steps = np.empty(n, np.int64)
    hits = np.empty(n, np.uint8)
    fn = lib.oracle_walk_rows_native if native else lib.oracle_walk_rows
    fn(pr.ptr, n, pts.ctypes.data, pid.ctypes.data, tid.ctypes.data, sgn.ctypes.data,
       int(seed) & MASK64, float(eps), int(max_steps), values.ctypes.data, steps.ctypes.data,
       hits.ctypes.data, int(nthreads or default_threads()))
    return values, steps, hits


def estimate(problems, points, L, *, seed, eps, max_steps, point_ids=None, inst_index=None,
             traj_start=0, antithetic=False, native=False, nthreads=None, sigma_bar=0.0,
             philox_rounds=10):
    """(mean, m2, total_steps) like estimator.estimate (two-pass moments per point)."""
    lib = load()
    lib.oracle_set_sigma_bar(float(sigma_bar))
    lib.oracle_set_philox_rounds(int(philox_rounds))
    if not isinstance(problems, (list, tuple)) or (isinstance(problems, tuple) and len(problems) == 8
                                                   and isinstance(problems[0], int)):
        problems = [problems]
    pr = _Problems(problems)
    pts = np.ascontiguousarray(np.asarray(points, np.float64))
    P = pts.shape[0]
    pid = np.ascontiguousarray(np.arange(P, dtype=np.int64) if point_ids is None
                               else np.asarray(point_ids).astype(np.int64))
    inst = None if inst_index is None else np.ascontiguousarray(np.asarray(inst_index, np.int32))
    mean = np.empty(P)
    m2 = np.empty(P)
    tot = c_uint64(0)
    lib.oracle_estimate(pr.ptr, int(native), P, pts.ctypes.data, pid.ctypes.data,
                        None if inst is None else inst.ctypes.data, int(L), int(traj_start) & MASK64,
                        int(bool(antithetic)), int(seed) & MASK64, float(eps), int(max_steps),
                        mean.ctypes.data, m2.ctypes.data, ctypes.addressof(tot),
                        int(nthreads or default_threads()))
    return mean, m2, tot.value


def majorant():
    """Largest sigma' above sigma_bar met by the last screened call, or -1."""
    return float(load().oracle_majorant())


def contains(problem, points):
    lib = load()
    pr = _Problems([problem])
    pts = np.ascontiguousarray(np.asarray(points, np.float64))
    d = pr.dim
    return np.array([bool(lib.oracle_contains(pr.ptr, pts[i].ctypes.data)) for i in range(pts.shape[0])])


def philox4x64(ctr, k0, k1):
    lib = load()
    c = np.ascontiguousarray(np.asarray(ctr, np.uint64).reshape(-1, 4))
    out = np.empty_like(c)
    lib.oracle_philox4x64(c.shape[0], c.ctypes.data, int(k0) & MASK64, int(k1) & MASK64, out.ctypes.data)
    return out


def philox4x32(ctr, k0, k1, rounds=10):
    lib = load()
    c = np.ascontiguousarray(np.asarray(ctr, np.uint32).reshape(-1, 4))
    out = np.empty_like(c)
    lib.oracle_philox4x32_rounds(c.shape[0], c.ctypes.data, int(k0) & MASK32, int(k1) & MASK32,
                                 int(rounds), out.ctypes.data)
    return out


def native_keys(seed, ikey):
    """Philox4x32 key of the NATIVE_F32 stream (wos_oracle.c oracle_native_keys)."""
    seed &= MASK64
    ikey &= MASK64
    k0 = seed & MASK32
    k1 = ((seed >> 32) ^ (ikey & MASK32) ^ (((ikey >> 32) * 0x9E3779B9) & MASK32)) & MASK32
    return k0, k1


# ---- exact-integer restatements (test_rng.py:11-26 method) ------------------

def philox4x64_int(counter, key):
    x = [int(v) & MASK64 for v in counter]
    k0, k1 = (int(v) & MASK64 for v in key)
    for _ in range(10):
        p0 = 0xD2E7470EE14C6C93 * x[0]
        p1 = 0xCA5A826395121157 * x[2]
        x = [(p1 >> 64) ^ x[1] ^ k0, p1 & MASK64, (p0 >> 64) ^ x[3] ^ k1, p0 & MASK64]
        k0 = (k0 + 0x9E3779B97F4A7C15) & MASK64
        k1 = (k1 + 0xBB67AE8584CAA73B) & MASK64
    return x


def philox4x32_int(counter, key, rounds=10):
    x = [int(v) & MASK32 for v in counter]
    k0, k1 = (int(v) & MASK32 for v in key)
    for _ in range(rounds):
        p0 = 0xD2511F53 * x[0]
        p1 = 0xCD9E8D57 * x[2]
        x = [((p1 >> 32) ^ x[1] ^ k0) & MASK32, p1 & MASK32, ((p0 >> 32) ^ x[3] ^ k1) & MASK32,
             p0 & MASK32]
        k0 = (k0 + 0x9E3779B9) & MASK32
        k1 = (k1 + 0xBB67AE85) & MASK32
    return x


# Random123 published known-answer vectors (kat_vectors), 10 rounds.
PHILOX4X64_KAT = [
    ((0, 0, 0, 0), (0, 0),
     (0x16554D9ECA36314C, 0xDB20FE9D672D0FDC, 0xD7E772CEE186176B, 0x7E68B68AEC7BA23B)),
    ((MASK64,) * 4, (MASK64,) * 2,
     (0x87B092C3013FE90B, 0x438C3C67BE8D0224, 0x9CC7D7C69CD777B6, 0xA09CAEBF594F0BA0)),
    ((0x243F6A8885A308D3, 0x13198A2E03707344, 0xA4093822299F31D0, 0x082EFA98EC4E6C89),
     (0x452821E638D01377, 0xBE5466CF34E90C6C),
     (0xA528F45403E61D95, 0x38C72DBD566E9788, 0xA5A1610E72FD18B5, 0x57BD43B5E52B7FE6)),
]
PHILOX4X32_KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((MASK32,) * 4, (MASK32,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def beta_table():
    """The NATIVE 3D source jump's Beta(2,2) conditional-mean table (include/wos_beta_table.h)."""
    out = np.empty(4096, dtype=np.float32)
    load().oracle_beta_table(out.ctypes.data)
    return out


def green2_table():
    """The NATIVE 2D source jump's disk Green's-law radius table (include/wos_beta_table.h)."""
    out = np.empty(4096, dtype=np.float32)
    load().oracle_green2_table(out.ctypes.data)
    return out


def median3_grid_moments(bits):
    """Exact (E[t], E[t^2]) of t = the median of three iid uniform ``bits``-bit integers,
    midpoint-rounded to (k + 1/2) 2^-bits: the NATIVE 3D source jump's Beta(2,2) radius
    fraction (wos_walk.cuh f_top12 / umed3). P(med <= k) = 3 F^2 - 2 F^3 with
    F = (k + 1) 2^-bits; exact rational arithmetic."""
    from fractions import Fraction

    n = 1 << bits
    e1 = e2 = Fraction(0)
    prev = Fraction(0)
    for k in range(n):
        F = Fraction(k + 1, n)
        G = 3 * F * F - 2 * F * F * F
        t = Fraction(2 * k + 1, 2 * n)
        e1 += t * (G - prev)
        e2 += t * t * (G - prev)
        prev = G
    return float(e1), float(e2)
