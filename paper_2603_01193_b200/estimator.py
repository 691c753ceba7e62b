"""Per-point ensemble estimates on the GPU — drop-in for ``spherewalk.estimator.estimate``.

``estimate`` keeps the reference signature and semantics (``estimator.py:144-181``):
L trajectories per point (traj ids ``traj_start + j``; antithetic pairs share an
id and their pair means are the samples), reduced to ``PointEstimate(mean, m2,
n_samples)``. The walks and the per-point reduction run fused in one persistent
sm_100a kernel; ``workers`` > 1 splits the points into that many strided shards
(point p -> shard p mod workers), shard i on GPU i mod n_gpus (threads, one context
per device). Results are bit-identical for any worker
count, batch layout or point order, like the reference's.

``estimate_arrays`` returns numpy arrays instead of a list of dataclasses and
takes multi-instance batches (one problem per point via ``inst_index``).
``estimate_tensors`` is the device-resident variant (torch tensors in and out,
stream-ordered, no host copies) used for benchmarking and multi-GPU sharding.
"""

from __future__ import annotations

import math
from ctypes import byref, c_int64, c_uint64
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import get_context, is_screened, problem_set, raise_exterior, walk_config_struct
from .geometry import ExteriorQueryError
from .walker import check_screened

__all__ = [
    "PointEstimate",
    "WelfordAccumulator",
    "chan_merge",
    "estimate",
    "estimate_arrays",
    "estimate_tensors",
    "check_status",
    "ExteriorQueryError",
]


def chan_merge(n1, mean1, m21, n2, mean2, m22):
    """Pool two (count, mean, squared-deviation sum) triples (estimator.py:41-53)."""
    n = n1 + n2
    if n == 0:
        return 0, 0.0, 0.0
    delta = mean2 - mean1
    mean = mean1 + delta * (n2 / n)
    m2 = m21 + m22 + delta * delta * (n1 * n2 / n)
    return n, mean, m2


class WelfordAccumulator:
    """Streaming (count, mean, m2) of a sequence of samples: the reference estimator
    module's one-pass accumulator (estimator.py:56-83), for host-side consumers of
    walk values. ``push`` is Welford's update; ``merge`` pools another accumulator
    with ``chan_merge``; ``variance`` is m2 / (n - 1), nan below two samples."""

    __slots__ = ("n", "mean", "m2")

    def __init__(self):
        self.n, self.mean, self.m2 = 0, 0.0, 0.0

    def push(self, x):
        x = float(x)
        self.n += 1
        d = x - self.mean
        self.mean += d / self.n
        self.m2 += d * (x - self.mean)

    def extend(self, values):
        for x in np.asarray(values, dtype=np.float64).ravel().tolist():
            self.push(x)

    def merge(self, other):
        self.n, self.mean, self.m2 = chan_merge(self.n, self.mean, self.m2, other.n, other.mean, other.m2)

    @property
    def variance(self):
        return self.m2 / (self.n - 1) if self.n >= 2 else math.nan


@dataclass(frozen=True)
class PointEstimate:
    """Moments of a finite trajectory ensemble at one query point (estimator.py:86-110)."""

    mean: float
    m2: float
    n_samples: int

    @property
    def variance(self) -> float:
        if self.n_samples >= 2:
            return self.m2 / (self.n_samples - 1)
        return math.nan

    @property
    def std_error(self) -> float:
        v = self.variance
        return math.sqrt(v / self.n_samples) if v == v else math.nan

    @classmethod
    def from_values(cls, values) -> "PointEstimate":
        v = np.asarray(values, dtype=np.float64)
        mean = float(v.mean())
        m2 = float(np.square(v - mean).sum())
        return cls(mean, m2, int(v.size))


def _validate_counts(L, antithetic):
    if L < 1:
        raise ValueError("trajectory count must be at least 1")
    if antithetic and L % 2:
        raise ValueError("antithetic estimation needs an even trajectory count")


def _estimate_one_device(device, problems, pts, pids, inst, L, cfg, eps, traj_start):
    ctx = get_context(device)
    pset = problem_set(ctx, problems)
    if pts.shape[1] != pset.dim:
        raise ValueError(f"expected points of dimension {pset.dim}, got shape {pts.shape}")
    P = pts.shape[0]
    wc = walk_config_struct(eps, cfg.max_steps, cfg.antithetic, cfg.mode, cfg.rng_seed,
                            cfg.sigma_bar, philox_rounds=cfg.philox_rounds)
    mean = np.empty(P, dtype=np.float64)
    m2 = np.empty(P, dtype=np.float64)
    steps = c_uint64(0)
    status = ctx._lib.wos_estimate_host(
        ctx.handle, pset.handle, byref(wc), P, pts.ctypes.data, None if pids is None else pids.ctypes.data,
        None if inst is None else inst.ctypes.data, int(L), int(traj_start) & ((1 << 64) - 1),
        mean.ctypes.data, m2.ctypes.data, byref(steps),
    )
    if status == _lib.WOS_ERR_EXTERIOR:
        return None, None, ctx.exterior(), 0
    check_screened(status)
    return mean, m2, -1, steps.value


def _device_count():
    try:
        import torch

        return max(1, torch.cuda.device_count())
    except Exception:  # pragma: no cover
        return 1


def _estimate_shards(problems, pts, pids, inst, L, cfg, eps, traj_start, n_shards):
    """Strided shards (point p -> shard p mod n_shards, distributed.shard_indices), shard i
    on device i mod n_gpus, reassembled in point order. An exception raised in a shard
    (exterior point, majorant violation, CUDA error) is re-raised here, as the reference's
    ``fut.result()`` does (estimator.py:176-181)."""
    from concurrent.futures import ThreadPoolExecutor

    from .distributed import shard_indices

    P = pts.shape[0]
    ndev = _device_count()
    if pids is None:
        pids = np.arange(P, dtype=np.int64)
    shards = [shard_indices(P, i, n_shards) for i in range(n_shards)]

    def run(i):
        idx = shards[i]
        return _estimate_one_device(
            i % ndev, problems, np.ascontiguousarray(pts[idx]), np.ascontiguousarray(pids[idx]),
            None if inst is None else np.ascontiguousarray(inst[idx]), L, cfg, eps, traj_start,
        )

    with ThreadPoolExecutor(max_workers=min(n_shards, ndev)) as ex:
        futs = [ex.submit(run, i) for i in range(n_shards)]
        results = [f.result() for f in futs]
    # the reference reports the first exterior point in point order (estimator.py:156-159)
    firsts = [int(idx[first]) for (_, _, first, _), idx in zip(results, shards) if first >= 0]
    if firsts:
        raise_exterior(pts, min(firsts))
    mean = np.empty(P, dtype=np.float64)
    m2 = np.empty(P, dtype=np.float64)
    for (m, v, _, _), idx in zip(results, shards):
        mean[idx] = m
        m2[idx] = v
    return mean, m2, sum(r[3] for r in results)


def estimate_arrays(problems, points, L, cfg, *, inst_index=None, point_ids=None, traj_start=0,
                    workers=1, return_steps=False):
    """Per-point (mean, m2, n_samples) arrays for a batch of problem instances.

    ``problems`` is one Problem or a list; ``inst_index[p]`` selects point p's
    problem (default all 0). ``point_ids`` default to ``arange(P)``.
    """
    if not isinstance(problems, (list, tuple)):
        problems = [problems]
    problems = [getattr(p, "problem", p) for p in problems]
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    if pts.ndim == 1:
        pts = pts[None, :]
    P = pts.shape[0]
    # point_ids=None: ids 0..P-1 (estimator.py:165), generated on the device (no copy)
    pids = None if point_ids is None else np.ascontiguousarray(np.asarray(point_ids).astype(np.int64))
    if pids is not None and pids.shape != (P,):
        raise ValueError("point_ids must have one entry per point")
    inst = None
    if inst_index is not None:
        inst = np.ascontiguousarray(np.asarray(inst_index, dtype=np.int32))
        if inst.shape != (P,) or (P and (inst.min() < 0 or inst.max() >= len(problems))):
            raise ValueError("inst_index must map every point to a problem")
    eps = cfg.resolve_eps(problems[0].domain)
    if is_screened(problems[0]) and (cfg.sigma_bar is None or cfg.sigma_bar <= 0.0):
        raise ValueError("delta tracking requires a positive cfg.sigma_bar")
    if L < 1 or (cfg.antithetic and L % 2):
        # the reference checks the interior first (estimator.py:156-163)
        ctx = get_context()
        pset = problem_set(ctx, problems)
        first = c_int64(-1)
        _lib.check(ctx._lib.wos_check_interior_host(
            ctx.handle, pset.handle, P, pts.ctypes.data, None if inst is None else inst.ctypes.data,
            byref(first)))
        raise_exterior(pts, first.value)
        _validate_counts(L, cfg.antithetic)
    n_samples = L // 2 if cfg.antithetic else L
    # workers = strided point shards (the reference's process fan-out, estimator.py:166-181:
    # here shard i runs on GPU i mod n_gpus); results are bit-identical for any count
    n_shards = min(max(1, int(workers)), max(P, 1))
    if n_shards <= 1:
        mean, m2, first, steps = _estimate_one_device(None, problems, pts, pids, inst, L, cfg, eps, traj_start)
        raise_exterior(pts, first)
    else:
        mean, m2, steps = _estimate_shards(problems, pts, pids, inst, L, cfg, eps, traj_start, n_shards)
    n = np.full(P, n_samples, dtype=np.int64)
    if return_steps:
        return mean, m2, n, steps
    return mean, m2, n


def estimate(inst, points, L, cfg, *, workers=1, traj_start=0, point_ids=None):
    """Estimate the solution at each point from L fresh trajectories (estimator.py:144-181).

    Returns one PointEstimate per point. With cfg.antithetic the L trajectories
    form L/2 mirrored pairs and the pair means are the samples.
    """
    inst = getattr(inst, "problem", inst)
    mean, m2, n = estimate_arrays(
        [inst], points, L, cfg, point_ids=point_ids, traj_start=traj_start, workers=workers
    )
    return [PointEstimate(float(a), float(b), int(c)) for a, b, c in zip(mean, m2, n)]


def estimate_tensors(pset, points, point_ids, L, cfg, *, inst_index=None, traj_start=0,
                     out_mean=None, out_m2=None, total_steps=None, stream=None, eps=None,
                     check=False):
    """Device-resident estimate: torch CUDA tensors in/out, ordered on ``stream``.

    points float64 (P, dim), point_ids int64 (P,), inst_index int32 (P,) or None,
    total_steps: uint64-compatible int64 tensor (1,) accumulated on the device.

    The call never synchronizes: an exterior start point, a majorant violation or a
    kernel watchdog trip is flagged on the device (the context's status block, cleared
    at the start of every call). ``check=True`` synchronizes ``stream`` after the launch
    and raises what the reference would (ExteriorQueryError naming the point,
    estimator.py:156-159; MajorantViolationError, walker.py:409-413) or a RuntimeError
    for a watchdog trip; otherwise ``pset.ctx.status(stream)`` reads the flags later.
    """
    import torch

    ctx = pset.ctx
    P = points.shape[0]
    if out_mean is None:
        out_mean = torch.empty(P, dtype=torch.float64, device=points.device)
    if out_m2 is None:
        out_m2 = torch.empty(P, dtype=torch.float64, device=points.device)
    if stream is None:
        stream = torch.cuda.current_stream(points.device)
    e = eps if eps is not None else cfg.eps_shell
    wc = walk_config_struct(e, cfg.max_steps, cfg.antithetic, cfg.mode, cfg.rng_seed, cfg.sigma_bar,
                            philox_rounds=cfg.philox_rounds)
    _lib.check(
        ctx._lib.wos_estimate(
            ctx.handle, pset.handle, byref(wc), P, points.data_ptr(), point_ids.data_ptr(),
            None if inst_index is None else inst_index.data_ptr(), int(L),
            int(traj_start) & ((1 << 64) - 1), out_mean.data_ptr(), out_m2.data_ptr(),
            None if total_steps is None else total_steps.data_ptr(), stream.cuda_stream,
        )
    )
    if check:
        check_status(ctx, stream, points, cfg)
    return out_mean, out_m2


def check_status(ctx, stream, points, cfg):
    """Raise the error the last walking call on ``ctx`` flagged on the device, if any."""
    from .walker import MajorantViolationError

    first, watchdog, worst = ctx.status(stream)
    if watchdog:
        raise RuntimeError("walk kernel watchdog tripped (iteration limit): results invalid")
    if worst >= 0.0:
        raise MajorantViolationError(
            f"majorant violated: sigma'={worst!r} > sigma_bar={cfg.sigma_bar!r}")
    if first >= 0:
        pt = points[first].detach().cpu().numpy() if hasattr(points, "detach") else np.asarray(points)[first]
        raise_exterior(np.asarray(pt)[None, :], 0)
