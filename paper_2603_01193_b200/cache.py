"""Device-resident epoch-averaged estimate cache — drop-in for ``spherewalk.estimator.EstimateCache``.

The reference keeps, per key (instance j, point i), the running sum of epoch means
plus Chan-pooled moments, and serves ``mean_sum / epoch`` as the training target
(estimator.py:188-302). Here the four per-key arrays live in HBM as torch tensors
and every fold runs on the GPU (``wos_cache_fold``, fp64 with the reference's
operation order, so targets are bit-identical to the reference fed the same
estimates). ``label_epoch`` is the training-label loop body of
``surrogate.train`` (surrogate.py:288-298): the epoch's walks are estimated and
folded into the cache in one stream-ordered call (``wos_estimate_fold``) and the
targets stay on the device for the consumer.

The on-disk format is the reference's SWEC v1 (estimator.py:26-38, 270-302), so
caches move between the two implementations byte for byte.
"""

from __future__ import annotations

import csv
import struct
from ctypes import byref, c_double, c_int64

import numpy as np

from . import _lib
from .engine import (
    _stream_ptr,
    get_context,
    is_screened,
    problem_set,
    raise_exterior,
    walk_config_struct,
)
from .estimator import PointEstimate
from .walker import MajorantViolationError, check_screened

__all__ = [
    "CacheShapeError",
    "EstimateCache",
    "cache_update",
    "export_csv",
    "read_swec",
    "write_swec",
]

# SWEC v1 (estimator.py:26-38): magic, <IQQ (version, epoch, count), then count
# little-endian records (j i8, i i8, mean_sum f8, n i8, mean f8, m2 f8), sorted by (j, i)
SWEC_MAGIC = b"SWEC"
SWEC_VERSION = 1
_SWEC_HEADER = struct.Struct("<IQQ")
SWEC_ENTRY = np.dtype(
    [("j", "<i8"), ("i", "<i8"), ("mean_sum", "<f8"), ("n", "<i8"), ("mean", "<f8"), ("m2", "<f8")]
)

# n1 * n2 must stay exact in fp64 for the device fold (see wos_cache.cu)
_MAX_FOLD_N = 1 << 53


class CacheShapeError(RuntimeError):
    """Update keys do not match the cache's frozen key set (estimator.py:184-185)."""


def write_swec(path, epoch, keys, mean_sum, n, mean, m2):
    """Write the SWEC v1 file of a cache state (estimator.py:270-280)."""
    keys = np.asarray(keys, dtype=np.int64).reshape(-1, 2)
    body = np.empty(keys.shape[0], dtype=SWEC_ENTRY)
    body["j"] = keys[:, 0]
    body["i"] = keys[:, 1]
    body["mean_sum"] = mean_sum
    body["n"] = n
    body["mean"] = mean
    body["m2"] = m2
    with open(path, "wb") as fh:
        fh.write(SWEC_MAGIC)
        fh.write(_SWEC_HEADER.pack(SWEC_VERSION, int(epoch), body.shape[0]))
        fh.write(body.tobytes())


def read_swec(path):
    """Parse a SWEC v1 file -> (epoch, keys (n, 2) int64, body record array) (estimator.py:282-302)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[: len(SWEC_MAGIC)] != SWEC_MAGIC:
        raise ValueError("not an estimate cache file")
    if len(blob) < len(SWEC_MAGIC) + _SWEC_HEADER.size:
        raise ValueError("truncated estimate cache file")
    version, epoch, count = _SWEC_HEADER.unpack_from(blob, len(SWEC_MAGIC))
    if version != SWEC_VERSION:
        raise ValueError(f"unsupported cache version {version}")
    off = len(SWEC_MAGIC) + _SWEC_HEADER.size
    if len(blob) < off + count * SWEC_ENTRY.itemsize:
        raise ValueError("truncated estimate cache file")
    body = np.frombuffer(blob, dtype=SWEC_ENTRY, count=count, offset=off)
    keys = np.stack([body["j"], body["i"]], axis=1).astype(np.int64)
    return int(epoch), keys, body


def _key_arrays(keys):
    k = np.asarray(list(keys) if not isinstance(keys, np.ndarray) else keys, dtype=np.int64)
    return k.reshape(-1, 2)


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise _lib.WosUnavailableError("EstimateCache keeps its state on a CUDA device; none is visible")
    return torch


class EstimateCache:
    """Running average of per-epoch ensemble means, keyed by (j, i), held in HBM.

    Same contract as the reference (estimator.py:188-200): the first update freezes
    the (sorted) key set; later updates must cover exactly the same keys; after k
    epochs of L walks every entry holds n = k L and its target is the plain average
    of its k epoch means. ``device`` selects the CUDA device (default: current).
    """

    def __init__(self, device=None):
        self.epoch = 0
        self._device = device
        self._keys = np.empty((0, 2), dtype=np.int64)
        self._index = None  # (j, i) -> slot, built lazily for the dict interface
        self._state = None  # device tensors: mean_sum, n, mean, m2
        self._last_order = None  # (query keys, slot tensor or None) of the last update

    # ---------------- keys ----------------
    def __len__(self):
        return int(self._keys.shape[0])

    @property
    def keys(self) -> list[tuple[int, int]]:
        return [(int(j), int(i)) for j, i in self._keys]

    @property
    def key_array(self) -> np.ndarray:
        """The frozen keys, (n, 2) int64, in target order."""
        return self._keys

    def _ctx(self):
        torch = _torch()
        dev = torch.cuda.current_device() if self._device is None else int(self._device)
        self._device = dev
        return get_context(dev), torch

    def _adopt(self, keys):
        """Freeze the key set (estimator.py:206-215): sorted (j, i), zeroed moments."""
        ctx, torch = self._ctx()
        q = _key_arrays(keys)
        order = np.lexsort((q[:, 1], q[:, 0]))
        ks = q[order]
        if ks.shape[0] > 1 and np.any(np.all(ks[1:] == ks[:-1], axis=1)):
            raise ValueError("duplicate cache keys")
        self._keys = ks
        self._index = None
        z = ks.shape[0]
        dev = torch.device("cuda", ctx.device)
        self._state = (
            torch.zeros(z, dtype=torch.float64, device=dev),
            torch.zeros(z, dtype=torch.int64, device=dev),
            torch.zeros(z, dtype=torch.float64, device=dev),
            torch.zeros(z, dtype=torch.float64, device=dev),
        )

    def _slots(self, keys):
        """Slot of each update key in the frozen order, or None for the identity.

        Raises CacheShapeError unless the update keys are exactly the cache's key set
        (estimator.py:219-224).
        """
        q = _key_arrays(keys)
        last = self._last_order
        if last is not None and last[0].shape == q.shape and np.array_equal(last[0], q):
            return last[1]
        if q.shape[0] == self._keys.shape[0] and np.array_equal(q, self._keys):
            slots = None
        else:
            order = np.lexsort((q[:, 1], q[:, 0]))
            if q.shape[0] != self._keys.shape[0] or not np.array_equal(q[order], self._keys):
                raise CacheShapeError(
                    "cache shape mismatch: update covers "
                    f"{q.shape[0]} keys, cache holds {self._keys.shape[0]}"
                )
            s = np.empty(q.shape[0], dtype=np.int64)
            s[order] = np.arange(q.shape[0], dtype=np.int64)
            torch = _torch()
            slots = torch.from_numpy(s).to(torch.device("cuda", self._device))
        self._last_order = (q.copy(), slots)
        return slots

    def _begin(self, keys):
        if self.epoch == 0 and self._state is None:
            self._adopt(keys)
        return self._slots(keys)

    # ---------------- updates ----------------
    def update(self, fresh):
        """Fold one epoch of fresh per-key PointEstimates (estimator.py:217-244)."""
        keys = list(fresh.keys())
        ests = list(fresh.values())
        self.update_arrays(
            keys,
            np.array([e.mean for e in ests], dtype=np.float64),
            np.array([e.m2 for e in ests], dtype=np.float64),
            np.array([e.n_samples for e in ests], dtype=np.int64),
        )

    def update_arrays(self, keys, mean, m2, n):
        """Fold one epoch given per-key arrays (host numpy or CUDA tensors).

        ``keys`` (m, 2) int64 on the host; ``mean``/``m2`` fp64 and ``n`` int64 (or a
        scalar count shared by every key) aligned with ``keys``.
        """
        if self.epoch > 0 and self._state is None:  # loaded empty cache
            raise CacheShapeError("cache shape mismatch: update covers keys, cache holds 0")
        slots = self._begin(keys)
        ctx, torch = self._ctx()
        dev = torch.device("cuda", ctx.device)
        m = len(self)
        fm = torch.as_tensor(mean, dtype=torch.float64).to(dev).contiguous()
        fq = torch.as_tensor(m2, dtype=torch.float64).to(dev).contiguous()
        if np.ndim(n) == 0:
            nn = int(n)
            if not 0 <= nn < _MAX_FOLD_N:
                raise ValueError("sample count out of range")
            fn, fn_all = None, nn
        else:
            fn = torch.as_tensor(n, dtype=torch.int64).to(dev).contiguous()
            fn_all = 0
        if fm.numel() != m or fq.numel() != m or (fn is not None and fn.numel() != m):
            raise ValueError("estimate arrays must have one entry per key")
        ms, cn, cm, c2 = self._state
        stream = torch.cuda.current_stream(dev)
        _lib.check(
            ctx._lib.wos_cache_fold(
                ctx.handle, m, None if slots is None else slots.data_ptr(), fm.data_ptr(),
                fq.data_ptr(), None if fn is None else fn.data_ptr(), fn_all, ms.data_ptr(),
                cn.data_ptr(), cm.data_ptr(), c2.data_ptr(), _stream_ptr(stream),
            )
        )
        self.epoch += 1

    def label_epoch(self, problem, points, L, cfg, *, j=0, keys=None, point_ids=None,
                    total_steps=None):
        """One training-label epoch on the GPU (surrogate.py:288-298).

        Estimates ``points`` with L fresh walks each, trajectory window
        ``traj_start = epoch * L`` (estimate's point_ids default 0..N-1), folds the
        estimates into the cache on the device, and returns the targets as a CUDA
        fp64 tensor aligned with ``key_array``. ``keys`` default to (j, i), i < N.
        """
        ctx, torch = self._ctx()
        dev = torch.device("cuda", ctx.device)
        problem = getattr(problem, "problem", problem)
        pts = torch.as_tensor(points, dtype=torch.float64).to(dev).contiguous()
        if pts.ndim == 1:
            pts = pts[None, :]
        P = pts.shape[0]
        if keys is None:
            keys = np.stack([np.full(P, int(j), np.int64), np.arange(P, dtype=np.int64)], axis=1)
        if len(_key_arrays(keys)) != P:
            raise ValueError("need one key per point")
        if L < 1 or (cfg.antithetic and L % 2):
            raise ValueError("trajectory count must be at least 1 (even when antithetic)")
        pset = problem_set(ctx, [problem])
        if pts.shape[1] != pset.dim:
            raise ValueError(f"expected points of dimension {pset.dim}, got {tuple(pts.shape)}")
        stream = torch.cuda.current_stream(dev)
        # the reference checks the interior before touching the cache (estimator.py:156-159)
        first = c_int64(-1)
        _lib.check(ctx._lib.wos_check_interior(ctx.handle, pset.handle, P, pts.data_ptr(), None,
                                               byref(first), _stream_ptr(stream)))
        raise_exterior(pts.cpu().numpy(), first.value)
        slots = self._begin(keys)
        pids = None
        if point_ids is not None:
            pids = torch.as_tensor(np.asarray(point_ids, dtype=np.int64)).to(dev).contiguous()
        screened = is_screened(problem)
        if screened and (cfg.sigma_bar is None or cfg.sigma_bar <= 0.0):
            raise ValueError("delta tracking requires a positive cfg.sigma_bar")
        wc = walk_config_struct(cfg.resolve_eps(problem.domain), cfg.max_steps, cfg.antithetic,
                                cfg.mode, cfg.rng_seed, cfg.sigma_bar, philox_rounds=cfg.philox_rounds)
        ms, cn, cm, c2 = self._state
        if total_steps is None:
            total_steps = torch.zeros(1, dtype=torch.int64, device=dev)
        if screened:
            # a majorant violation surfaces only after the walks: estimate into scratch,
            # check, then fold, so a failing epoch leaves the cache untouched (the
            # reference raises inside estimate, before cache_update)
            mean = torch.empty(P, dtype=torch.float64, device=dev)
            m2 = torch.empty(P, dtype=torch.float64, device=dev)
            check_screened(ctx._lib.wos_estimate(
                ctx.handle, pset.handle, byref(wc), P, pts.data_ptr(),
                None if pids is None else pids.data_ptr(), None, int(L),
                (self.epoch * int(L)) & ((1 << 64) - 1), mean.data_ptr(), m2.data_ptr(),
                total_steps.data_ptr(), _stream_ptr(stream)))
            worst = c_double(-1.0)
            _lib.check(ctx._lib.wos_context_majorant(ctx.handle, _stream_ptr(stream), byref(worst)))
            if worst.value >= 0.0:
                raise MajorantViolationError(
                    f"majorant violated: sigma'={worst.value!r} > sigma_bar={cfg.sigma_bar!r}")
            _lib.check(ctx._lib.wos_cache_fold(
                ctx.handle, P, None if slots is None else slots.data_ptr(), mean.data_ptr(),
                m2.data_ptr(), None, L // 2 if cfg.antithetic else L, ms.data_ptr(), cn.data_ptr(),
                cm.data_ptr(), c2.data_ptr(), _stream_ptr(stream)))
            self.epoch += 1
            return self.targets_tensor()
        _lib.check(
            ctx._lib.wos_estimate_fold(
                ctx.handle, pset.handle, byref(wc), P, pts.data_ptr(),
                None if pids is None else pids.data_ptr(), None, int(L),
                (self.epoch * int(L)) & ((1 << 64) - 1),
                None if slots is None else slots.data_ptr(), ms.data_ptr(), cn.data_ptr(),
                cm.data_ptr(), c2.data_ptr(), total_steps.data_ptr(), _stream_ptr(stream),
            )
        )
        self.epoch += 1
        return self.targets_tensor()

    # ---------------- reads ----------------
    def targets_tensor(self):
        """Device fp64 tensor of all targets (mean_sum / epoch), key_array order."""
        ctx, torch = self._ctx()
        if self.epoch == 0 or self._state is None:
            return torch.empty(0, dtype=torch.float64, device=torch.device("cuda", ctx.device))
        ms = self._state[0]
        out = torch.empty_like(ms)
        stream = torch.cuda.current_stream(ms.device)
        _lib.check(
            ctx._lib.wos_cache_targets(ctx.handle, ms.numel(), ms.data_ptr(), int(self.epoch),
                                       out.data_ptr(), _stream_ptr(stream))
        )
        return out

    def targets(self) -> np.ndarray:
        """All targets, aligned with the sorted key order of ``keys`` (estimator.py:251-255)."""
        if self.epoch == 0:
            return np.empty(0)
        return self.targets_tensor().cpu().numpy()

    def target(self, key) -> float:
        """Average of this key's epoch means so far (estimator.py:245-249)."""
        if self.epoch == 0:
            raise KeyError("cache is empty")
        if self._index is None:
            self._index = {(int(j), int(i)): k for k, (j, i) in enumerate(self._keys)}
        k = self._index[tuple(int(v) for v in key)]
        return float(self._state[0][k].item() / self.epoch)

    def host_state(self):
        """(mean_sum, n, mean, m2) as host arrays (one device->host copy each)."""
        if self._state is None:
            z = len(self)
            return np.zeros(z), np.zeros(z, np.int64), np.zeros(z), np.zeros(z)
        return tuple(t.cpu().numpy() for t in self._state)

    def estimates(self) -> dict:
        """Per-key PointEstimate(target, pooled m2, n) (estimator.py:257-268)."""
        ms, n, _, m2 = self.host_state()
        out = {}
        for k, (j, i) in enumerate(self._keys):
            out[(int(j), int(i))] = PointEstimate(
                float(ms[k] / self.epoch) if self.epoch else 0.0, float(m2[k]), int(n[k])
            )
        return out

    # ---------------- persistence ----------------
    def save(self, path):
        ms, n, mean, m2 = self.host_state()
        write_swec(path, self.epoch, self._keys, ms, n, mean, m2)

    @classmethod
    def load(cls, path, device=None) -> "EstimateCache":
        epoch, keys, body = read_swec(path)
        cache = cls(device)
        cache.epoch = epoch
        cache._keys = keys
        if keys.shape[0]:
            ctx, torch = cache._ctx()
            dev = torch.device("cuda", ctx.device)
            cache._state = tuple(
                torch.from_numpy(np.ascontiguousarray(body[f])).to(dev)
                for f in ("mean_sum", "n", "mean", "m2")
            )
            cache._state = (cache._state[0], cache._state[1].to(torch.int64), cache._state[2],
                            cache._state[3])
        return cache

    def export_csv(self, path, coords):
        """One row per key: instance id, coordinates, moments (estimator.py:304-313)."""
        rows = []
        for key, est in sorted(self.estimates().items()):
            rows.append((key[0], coords[key], est))
        export_csv(path, rows)


def cache_update(cache: EstimateCache, fresh) -> EstimateCache:
    """Fold one epoch of fresh estimates into the cache and return it (estimator.py:338-341)."""
    cache.update(fresh)
    return cache


def export_csv(path, rows):
    """Write (instance_id, coords, PointEstimate) rows as CSV (estimator.py:316-335).

    Floats are rendered with repr so identical estimates give identical bytes.
    """
    rows = list(rows)
    dim = len(rows[0][1]) if rows else 0
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["instance_id"] + [f"x{d}" for d in range(dim)] + ["mean", "variance", "n_samples"])
        for instance_id, coords, est in rows:
            w.writerow(
                [int(instance_id)]
                + [repr(float(c)) for c in coords]
                + [repr(float(est.mean)), repr(float(est.variance)), int(est.n_samples)]
            )
