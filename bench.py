"""Benchmark of the B200 WoS label estimator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One "step" = one full pass of the estimator over the workload: every query
point of the config runs its L walks and is reduced to (mean, m2). Default
workload: BASELINE config 4 (unit cube, 3x3x3 sine source, 64^3 = 262,144 cell
centres x 256 walks, eps 1e-3, max 1000 steps, NATIVE_F32) — the config BASELINE
names for 1/2/4/8-GPU scaling. Under torchrun each rank takes a strided
(round-robin) shard of the points, runs its walks locally and the shards'
(mean, m2) are all-gathered over NCCL: the only collective.

Metric: walk-steps/s (whole job), plus walks/s. Timing: CUDA events on the
launching stream around each step, L2 flushed (256 MiB write) before every step
outside the timed window, max over ranks. The CPU baseline is the oracle
(oracle/wos_oracle.c, a C restatement of the reference's path) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic work per walk-step / per walk (native form):
# (F_step, S_step, F_walk, S_walk) in FP32 flops (FFMA = 2) and SFU ops
WORK = {
    0: (71, 9, 9, 0),
    1: (13, 3, 87, 1),
    2: (187, 9, 31, 2),
    3: (2072, 7, 4232, 2),
    4: (125, 12, 12, 0),
}


def _ncu_traffic(workload):
    """DRAM bytes (read + write) per launch of the walk kernel from the committed ncu capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[workload]
        return d["dram_bytes_read"] + d["dram_bytes_write"]
    except (OSError, KeyError, ValueError):
        return None


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {
            "sm_mhz": float(np.median(sm)) if sm else None,
            "sm_max_mhz": float(max(smax)) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def cpu_baseline(w, budget_s=12.0, nthreads=None):
    """Oracle (reference-form C port) on the host cores over a bounded, strided sample."""
    from oracle import oracle as O

    nthreads = nthreads or O.default_threads()
    O.load()
    n = 64
    t_used = 0.0
    while True:
        idx = np.arange(0, w.n_points, max(1, w.n_points // n))[:n]
        sub = w.subset(idx)
        t0 = time.perf_counter()
        _, _, steps = O.estimate(sub.problems, sub.points, w.L, seed=w.cfg.rng_seed, eps=w.cfg.eps_shell,
                                 max_steps=w.cfg.max_steps, point_ids=sub.point_ids,
                                 inst_index=sub.inst_index, nthreads=nthreads)
        dt = time.perf_counter() - t0
        t_used += dt
        if dt >= budget_s * 0.5 or n >= w.n_points or t_used > budget_s * 2:
            break
        n = min(w.n_points, int(n * max(2.0, min(16.0, budget_s * 0.6 / max(dt, 1e-3)))))
    return {
        "value": steps / dt,
        "unit": "walk-steps/s",
        "cores": nthreads,
        "kind": "port",
        "walks_per_s": sub.n_points * w.L / dt,
        "sample": f"{sub.n_points} of {w.n_points} points (strided) x {w.L} walks, reference form "
                  f"(Philox4x64, uniform-ball source, fp64), {steps} walk-steps in {dt:.2f}s",
    }


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (oracle port) on the host cores, rank 0 only."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2603_01193_b200 import configs

    w = configs.build(args.config, mode="replay")
    nthreads = O.default_threads()
    # a bounded strided sample per step, sized to ~1 s of host work
    n = max(32, min(w.n_points, 2048 if args.config in (4, 3) else 8192))
    idx = np.arange(0, w.n_points, max(1, w.n_points // n))[:n]
    sub = w.subset(idx)

    def one(step):
        t0 = time.perf_counter()
        _, _, s = O.estimate(sub.problems, sub.points, w.L, seed=w.cfg.rng_seed, eps=w.cfg.eps_shell,
                             max_steps=w.cfg.max_steps, point_ids=sub.point_ids,
                             inst_index=sub.inst_index, traj_start=step * w.L, nthreads=nthreads)
        return time.perf_counter() - t0, s

    for i in range(args.warmup):
        one(i)
    tot_t, tot_s = 0.0, 0
    for i in range(args.steps):
        dt, s = one(args.warmup + i)
        tot_t += dt
        tot_s += s
    val = tot_s / tot_t
    walks = sub.n_points * w.L * args.steps / tot_t
    sample = (f"{sub.n_points} of {w.n_points} points (strided) x {w.L} walks per step, "
              f"reference form (Philox4x64, uniform-ball source, fp64) via oracle/wos_oracle.c")
    line = {
        "impl": "reference",
        "metric": "walk-steps/s",
        "value": val,
        "unit": "walk-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE config, pinned seeds)",
        "walks_per_s": walks,
        "config": {"workload": w.name, "walks_per_point": w.L, "sample_points": int(sub.n_points)},
        "cpu_baseline": {"value": val, "unit": "walk-steps/s", "cores": nthreads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": val, "unit": "walk-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", default="native")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", type=int, default=1,
                    help="independent label replicas per point per step (small configs)")
    ap.add_argument("--refill-min", type=int, default=None)
    ap.add_argument("--refill-min-deferred", type=int, default=None)
    ap.add_argument("--blocks-per-sm", type=int, default=None)
    args = ap.parse_args()

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", rank)

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2603_01193_b200 import _lib, configs, engine
    from paper_2603_01193_b200.distributed import gather_estimates, shard_indices
    from paper_2603_01193_b200.estimator import estimate_tensors

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    w = configs.build(args.config, mode=args.mode).replicate(args.replicas)
    idx = shard_indices(w.n_points, rank, world)
    shard = w.subset(idx)
    ctx = engine.get_context(local)
    if args.refill_min or args.blocks_per_sm or args.refill_min_deferred:
        ctx.set_tuning(args.refill_min or 5, args.blocks_per_sm or 0, args.refill_min_deferred or 12)
    pset = engine.ProblemSet(ctx, w.problems)
    pts = torch.from_numpy(np.ascontiguousarray(shard.points)).to(dev)
    ids = torch.from_numpy(np.ascontiguousarray(shard.point_ids)).to(dev)
    inst = torch.from_numpy(np.ascontiguousarray(shard.inst_index)).to(dev) if len(w.problems) > 1 else None
    steps_acc = torch.zeros(1, dtype=torch.int64, device=dev)
    mean = torch.empty(shard.n_points, dtype=torch.float64, device=dev)
    m2 = torch.empty_like(mean)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    eps = w.cfg.resolve_eps(w.problems[0].domain)

    def step(i, acc=None):
        estimate_tensors(pset, pts, ids, w.L, w.cfg, inst_index=inst, traj_start=i * w.L,
                         out_mean=mean, out_m2=m2, total_steps=acc, stream=stream, eps=eps)
        if world > 1:
            gather_estimates(mean, m2, w.n_points, rank, world)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        step(args.warmup + i, steps_acc)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    tot_steps = steps_acc.clone()
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_steps, op=dist.ReduceOp.SUM)
    ms = float(t.item())
    S = int(tot_steps.item())
    n_walks = w.n_walks * args.steps
    value = S / (ms * 1e-3)
    walks_per_s = n_walks / (ms * 1e-3)

    # ---- roofline of the dominant kernel (the persistent walk kernel) ----
    F_step, S_step, F_walk, S_walk = WORK[args.config]
    t_launch = ms * 1e-3 / args.steps
    # per-rank algorithmic work per launch; the slowest rank defines t_launch
    S_rank = S / args.steps / world
    Nw_rank = w.n_walks / world
    sfu_ach = (S_rank * S_step + Nw_rank * S_walk) / t_launch
    fp32_ach = (S_rank * F_step + Nw_rank * F_walk) / t_launch
    peaks = ctx.probe_peaks() if rank == 0 else None

    # ---- e2e through the C-ABI with host buffers (H2D + kernel + D2H per step) ----
    def pinned(a):
        # page-locked host buffers (the contract's pinned host memory): the library's
        # chunked pipeline overlaps their copies with the walks
        t = torch.empty(a.shape, dtype=torch.from_numpy(np.empty(0, a.dtype)).dtype).pin_memory()
        out = t.numpy()
        out[...] = a
        return out, t

    host_pts, _keep_pts = pinned(np.ascontiguousarray(shard.points))
    # default ids (0..P-1, the reference's estimate() default) are generated on the device
    host_ids, _keep_ids = (None, None) if world == 1 and args.replicas == 1 and np.array_equal(
        shard.point_ids, np.arange(shard.n_points)) else pinned(np.ascontiguousarray(shard.point_ids))
    host_inst, _keep_inst = pinned(np.ascontiguousarray(shard.inst_index)) if inst is not None else (None, None)
    out_mean, _keep_mean = pinned(np.empty(shard.n_points))
    out_m2, _keep_m2 = pinned(np.empty(shard.n_points))
    from ctypes import byref, c_uint64

    wc = engine.walk_config_struct(eps, w.cfg.max_steps, w.cfg.antithetic, w.cfg.mode, w.cfg.rng_seed)
    e2e_steps = c_uint64(0)

    def e2e_once(i):
        _lib.check(ctx._lib.wos_estimate_host(
            ctx.handle, pset.handle, byref(wc), shard.n_points, host_pts.ctypes.data,
            None if host_ids is None else host_ids.ctypes.data,
            None if host_inst is None else host_inst.ctypes.data, w.L,
            i * w.L, out_mean.ctypes.data, out_m2.ctypes.data, byref(e2e_steps)))
        return e2e_steps.value

    e2e_once(0)
    n_e2e = max(3, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_S = 0
    for i in range(n_e2e):
        e2e_S += e2e_once(1000 + i)
    e2e_t = time.perf_counter() - t0
    te = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
    se = torch.tensor([e2e_S], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        dist.all_reduce(se, op=dist.ReduceOp.SUM)
    e2e_value = int(se.item()) / float(te.item())
    h2d = host_pts.nbytes + (0 if host_ids is None else host_ids.nbytes) + \
        (0 if host_inst is None else host_inst.nbytes)
    d2h = out_mean.nbytes + out_m2.nbytes + 16

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(configs.build(args.config, mode="replay").replicate(args.replicas))
        sfu_peak = peaks["sfu_ops_per_s"]
        fp32_peak = peaks["fp32_flops_per_s"]
        fr_sfu = sfu_ach / sfu_peak
        fr_fp32 = fp32_ach / fp32_peak
        bound = "sfu" if fr_sfu >= fr_fp32 else "fp32"
        line = {
            "metric": "walk-steps/s",
            "value": value,
            "unit": "walk-steps/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32" if args.mode.startswith("native") else ("f64" if args.mode.startswith("replay") and not args.mode.endswith("f32") else "f32"),
            "data": "synthetic (BASELINE config, pinned seeds; no dataset exists for this path)",
            "walks_per_s": walks_per_s,
            "walk_steps_per_step": S / args.steps,
            "mean_steps_per_walk": S / n_walks,
            "config": {
                "workload": w.name,
                "points": w.n_points,
                "walks_per_point": w.L,
                "instances": len(w.problems),
                "replicas": args.replicas,
                "eps": w.cfg.eps_shell,
                "max_steps": w.cfg.max_steps,
                "mode": args.mode,
                "parallelism": f"dp{world} strided point shards + NCCL all-gather of (mean, m2)",
                "l2": "flushed (256 MiB write) before every timed step, outside the events",
                "traj_windows": "step i uses traj ids [i*L, (i+1)*L)",
            },
            "roofline": {
                "bound": bound,
                "achieved": sfu_ach if bound == "sfu" else fp32_ach,
                "peak": sfu_peak if bound == "sfu" else fp32_peak,
                "unit": "SFU op/s" if bound == "sfu" else "FP32 flop/s",
                "frac": fr_sfu if bound == "sfu" else fr_fp32,
                "traffic": _ncu_traffic(w.name),
                "sfu": {"achieved": sfu_ach, "peak_measured": sfu_peak, "frac": fr_sfu,
                        "per_step": S_step, "per_walk": S_walk},
                "fp32": {"achieved": fp32_ach, "peak_measured": fp32_peak, "frac": fr_fp32,
                         "per_step": F_step, "per_walk": F_walk},
                "peak_source": "measured in this run by wos_probe_peaks (MUFU rsqrt / FFMA microkernels)",
                "sm_clock_mhz_probe": peaks["sm_clock_hz"] / 1e6,
            },
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "walk-steps/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "wos_estimate_host (C ABI, pinned host buffers; copies inside, pipelined in point chunks)"},
            "gpu_launches": 2 * args.steps,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
