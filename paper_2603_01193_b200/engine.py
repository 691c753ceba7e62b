"""Device contexts and problem sets: the thin host layer over the C ABI.

One ``wos_context`` per CUDA device (persistent scratch, launch tuning), and
one device-resident ``wos_problem_set`` per list of problems. Everything that
computes runs in libwos_b200.so on the GPU; this module only marshals.
"""

from __future__ import annotations

import ctypes
import threading
from ctypes import byref, c_double, c_int32, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

from . import _lib, specs
from .geometry import ExteriorQueryError, domain_spec

__all__ = [
    "UnsupportedProblemError",
    "problem_record",
    "Context",
    "ProblemSet",
    "get_context",
    "problem_set",
    "is_screened",
    "mode_code",
]


class UnsupportedProblemError(ValueError):
    """The problem cannot be encoded for the GPU walker (no CPU fallback)."""


_MODES = {
    "replay": _lib.MODE_REPLAY_F64,
    "replay_f64": _lib.MODE_REPLAY_F64,
    "replay_f32": _lib.MODE_REPLAY_F32,
    "native": _lib.MODE_NATIVE_F32,
    "native_f32": _lib.MODE_NATIVE_F32,
}


def mode_code(mode) -> int:
    if isinstance(mode, int):
        return mode
    try:
        return _MODES[mode]
    except KeyError:
        raise ValueError(f"unknown walk mode {mode!r}; expected one of {sorted(_MODES)}") from None


def _screened_record(inst, dom_kind, dom_params, dim):
    """Spec record of a delta-tracking problem (walker.py:120-136).

    Constant coefficients come from ``const_coeffs = (s', f' or None, g')`` (the
    reference's compiled form, walker.py:331-347); the paper's varying-coefficient
    family (pde.VcInstance) from ``vc_params = (phi, a_min, a_max)``. ``sqrt_alpha``
    must be None or a number for constant coefficients (it is implied for the family).
    """
    if dim != 3:
        raise UnsupportedProblemError("delta tracking is 3D only (walker.py:322-418)")
    ikey = int(getattr(inst, "instance_key", 0)) & ((1 << 64) - 1)
    vc = getattr(inst, "vc_params", None)
    if vc is not None:
        phi, a_min, a_max = (float(v) for v in vc)
        return (dim, dom_kind, tuple(dom_params), specs.SRC_SCREENED_VC, (phi, a_min, a_max),
                specs.BND_VC, (phi,), ikey)
    cc = getattr(inst, "const_coeffs", None)
    if cc is None:
        raise UnsupportedProblemError(
            "screened problem without const_coeffs or vc_params: callable coefficients have "
            "no GPU encoding (no CPU fallback)"
        )
    sprime, fprime, gprime = cc
    sa = getattr(inst, "sqrt_alpha", None)
    if sa is None:
        sa = 1.0
    elif callable(sa):
        raise UnsupportedProblemError("a callable sqrt_alpha has no GPU encoding; pass a number")
    return (dim, dom_kind, tuple(dom_params), specs.SRC_SCREENED_CONST,
            (float(sprime), 0.0 if fprime is None else float(fprime),
             0.0 if fprime is None else 1.0, float(sa)),
            specs.BND_CONST, (float(gprime),), ikey)


def is_screened(inst) -> bool:
    inst = getattr(inst, "problem", inst)
    return hasattr(inst, "sigma_prime") or hasattr(inst, "const_coeffs") or hasattr(inst, "vc_params")


def problem_record(inst):
    """Reduce a Problem (ours or the reference's) to a plain spec record.

    Mirrors ``walker._specs_for_kernel`` (walker.py:160-171): the boundary must
    carry a ``boundary_spec``; a present source must carry a ``source_spec``.
    Screened (delta-tracking) problems reduce to their coefficient specs.
    """
    inst = getattr(inst, "problem", inst)
    dom = inst.domain
    dom_kind, dom_params, dim = domain_spec(dom)
    if is_screened(inst):
        return _screened_record(inst, dom_kind, dom_params, dim)
    bspec = getattr(inst, "boundary_spec", None)
    if bspec is None:
        raise UnsupportedProblemError(
            "problem has no boundary_spec; the GPU walker needs (kind, params) problem "
            "terms (walker.py:160-171) and has no callable/CPU fallback"
        )
    sspec = getattr(inst, "source_spec", None)
    if sspec is None:
        if getattr(inst, "source", None) is not None:
            raise UnsupportedProblemError(
                "problem has a source callable but no source_spec; not GPU-codeable"
            )
        sspec = (specs.SRC_NONE, ())
    skind, sparams = specs.normalize(sspec)
    bkind, bparams = specs.normalize(bspec)
    ikey = int(getattr(inst, "instance_key", 0)) & ((1 << 64) - 1)
    return (dim, dom_kind, tuple(dom_params), skind, tuple(sparams), bkind, tuple(bparams), ikey)


class Context:
    """A wos_context bound to one CUDA device."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        self._lib = _lib.lib()
        h = c_void_p()
        _lib.check(self._lib.wos_context_create(self.device, byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            self._lib.wos_context_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def set_tuning(self, refill_min: int = 5, blocks_per_sm: int = 0, refill_min_deferred: int = 12):
        _lib.check(self._lib.wos_set_tuning(self.handle, int(refill_min), int(blocks_per_sm)))
        _lib.check(self._lib.wos_set_refill_deferred(self.handle, int(refill_min_deferred)))

    def probe_peaks(self):
        sfu, fp32, clk = c_double(), c_double(), c_double()
        nsm = c_int32()
        _lib.check(
            self._lib.wos_probe_peaks(self.handle, byref(sfu), byref(fp32), byref(clk), byref(nsm))
        )
        return {
            "sfu_ops_per_s": sfu.value,
            "fp32_flops_per_s": fp32.value,
            "sm_clock_hz": clk.value,
            "num_sms": nsm.value,
        }

    def status(self, stream=None):
        """(first exterior index or -1, watchdog flag, worst sigma' above sigma_bar or -1)
        of the last walking call on this context; synchronizes ``stream`` and clears."""
        first, wd, sp = c_int64(-1), c_uint32(0), c_double(-1.0)
        _lib.check(self._lib.wos_context_status(self.handle, _stream_ptr(stream), byref(first), byref(wd),
                                        byref(sp)))
        return first.value, int(wd.value), sp.value

    def counters(self, stream=None):
        """(kernels launched by the library on this context, NATIVE polygon segment
        distances evaluated), cumulative; synchronizes ``stream``."""
        launches, segs = c_uint64(0), c_uint64(0)
        _lib.check(self._lib.wos_context_counters(self.handle, _stream_ptr(stream), byref(launches),
                                                  byref(segs)))
        return int(launches.value), int(segs.value)

    def exterior(self, stream=None) -> int:
        first = c_int64(-1)
        _lib.check(self._lib.wos_context_exterior(self.handle, _stream_ptr(stream), byref(first)))
        return first.value


_ctx_lock = threading.Lock()
_contexts: dict[int, Context] = {}


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover
        pass
    return 0


def get_context(device: int | None = None) -> Context:
    dev = _current_device() if device is None else int(device)
    with _ctx_lock:
        ctx = _contexts.get(dev)
        if ctx is None:
            ctx = Context(dev)
            _contexts[dev] = ctx
        return ctx


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return c_void_p(stream)
    return c_void_p(int(getattr(stream, "cuda_stream", stream)))


class ProblemSet:
    """Device-resident table of problem instances (same dim and kinds)."""

    def __init__(self, ctx: Context, problems):
        recs = [problem_record(p) for p in problems]
        if not recs:
            raise ValueError("need at least one problem")
        head = recs[0]
        for r in recs[1:]:
            if (r[0], r[1], r[3], r[5]) != (head[0], head[1], head[3], head[5]):
                raise UnsupportedProblemError(
                    "a problem set needs one dimension and one domain/source/boundary kind"
                )
        self.ctx = ctx
        self.dim = head[0]
        self.records = recs
        arrs = []
        structs = (_lib.WosProblem * len(recs))()
        for i, (dim, dk, dp, sk, sp, bk, bp, ikey) in enumerate(recs):
            d = np.ascontiguousarray(np.asarray(dp if dp else (0.0,), dtype=np.float64))
            s = np.ascontiguousarray(np.asarray(sp if sp else (0.0,), dtype=np.float64))
            b = np.ascontiguousarray(np.asarray(bp if bp else (0.0,), dtype=np.float64))
            arrs += [d, s, b]
            dbl = ctypes.POINTER(ctypes.c_double)
            structs[i] = _lib.WosProblem(
                dim, dk, len(dp), d.ctypes.data_as(dbl), sk, len(sp), s.ctypes.data_as(dbl),
                bk, len(bp), b.ctypes.data_as(dbl), ikey,
            )
        h = c_void_p()
        _lib.check(ctx._lib.wos_problem_set_create(ctx.handle, structs, len(recs), byref(h)))
        self.handle = h

    def __len__(self):
        return len(self.records)

    def close(self):
        if self.handle:
            self.ctx._lib.wos_problem_set_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


_pset_lock = threading.Lock()
_psets: "dict[tuple, ProblemSet]" = {}
_PSET_CACHE_MAX = 64


def problem_set(ctx: Context, problems) -> ProblemSet:
    """Device problem set for ``problems``, reused across calls with the same specs.

    Keyed by the problems' spec records (and the context), so a training loop that
    estimates the same instance every epoch uploads its table once.
    """
    recs = tuple(problem_record(p) for p in problems)
    key = (id(ctx), recs)
    with _pset_lock:
        ps = _psets.pop(key, None)
        if ps is None:
            ps = ProblemSet(ctx, problems)
        _psets[key] = ps  # most recently used last
        while len(_psets) > _PSET_CACHE_MAX:
            # least recently used: drop the cache's reference only; the set frees its
            # device tables (ProblemSet.__del__) once no caller or thread still holds it
            _psets.pop(next(iter(_psets)))
        return ps


def walk_config_struct(eps: float, max_steps: int, antithetic: bool, mode, seed: int,
                       sigma_bar=None, philox_rounds: int = 10):
    return _lib.WosWalkConfig(
        float(eps), int(max_steps), int(bool(antithetic)), mode_code(mode),
        int(seed) & ((1 << 64) - 1), 0.0 if sigma_bar is None else float(sigma_bar),
        int(philox_rounds), 0,
    )


def raise_exterior(points, first: int):
    if first >= 0:
        pt = np.asarray(points)[first]
        raise ExteriorQueryError(f"exterior query: start point {np.atleast_1d(pt).tolist()}")
