"""Benchmark of the B200 WoS label estimator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
                    [--mode native|replay|replay_f32] [--philox-rounds 10|7]

One "step" = one full pass of the estimator over the workload: every query
point of the config runs its L walks and is reduced to (mean, m2). Default
workload: BASELINE config 4 (unit cube, 3x3x3 sine source, 64^3 = 262,144 cell
centres x 256 walks, eps 1e-3, max 1000 steps, NATIVE_F32) — the config BASELINE
names for 1/2/4/8-GPU scaling. Under torchrun each rank takes a strided
(round-robin) shard of the points, runs its walks locally and the shards'
(mean, m2) are all-gathered over NCCL: the only collective.

Metric: walk-steps/s (whole job), plus walks/s. Timing: CUDA events on the
launching stream around each step, L2 flushed (256 MiB write) before every step
outside the timed window, max over ranks. On rank 0 at N = 1 the line also
carries: the cfg4 reference form on the GPU (REPLAY_F64, the reference's
estimator draw for draw, fp64), per-config sub-records for cfg0-cfg3 (one
estimate's latency and replica-batched throughput, each with its roofline), and
the CPU baseline: the oracle (oracle/wos_oracle.c, a C restatement of the
reference's path) on the host cores over a seeded random sample of the points.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic work per walk-step / per walk (native form):
# (F_step, S_step, F_walk, S_walk) in FP32 flops (FFMA = 2) and SFU ops.
# cfg3 is measured instead (see work()): its candidate-grid query evaluates a
# varying number of segments, counted in the kernel.
WORK = {
    0: (71, 9, 9, 0),
    1: (13, 3, 87, 1),
    2: (187, 9, 31, 2),
    3: (None, 7, 87, 2),
    4: (125, 12, 12, 0),
}
SEG_FLOPS = 16        # one point-to-segment distance (128 segments x 16)
CFG3_STEP_FLOPS = 24  # the rest of a cfg3 jump: Gaussian f 6 + move, sample, tests 18
SFU_PER_SM_CLK = 16   # MUFU ops per SM per clock (sin/cos/sqrt/rsqrt/ex2/lg2/rcp)
FP32_PER_SM_CLK = 256  # 128 FP32 lanes x 2 flops (FFMA)
LABEL_BYTES = 16      # per point written by the estimate: mean, m2 (fp64)
DEFAULT_REPLICAS = {0: 64, 1: 16, 2: 16, 3: 1, 4: 1}


def work(cfg_index, steps, walks, seg_evals=0):
    """(FP32 flops, SFU ops) of `steps` walk-steps and `walks` walks of config cfg_index."""
    F_step, S_step, F_walk, S_walk = WORK[cfg_index]
    if F_step is None:  # measured: segment distances counted by the kernel
        fp32 = SEG_FLOPS * seg_evals + CFG3_STEP_FLOPS * steps + F_walk * walks
    else:
        fp32 = F_step * steps + F_walk * walks
    return fp32, S_step * steps + S_walk * walks


def _ncu_traffic(workload):
    """DRAM bytes (read + write) per launch of the walk kernel from the committed ncu capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[workload]
        return d["dram_bytes_read"] + d["dram_bytes_write"], d.get("source")
    except (OSError, KeyError, ValueError):
        return None, None


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


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


def sample_points(w, n, seed=12345):
    """A seeded random sample of n points (sorted): representative of the whole config,
    unlike a fixed stride (every 128th point of cfg4's C-order 64^3 grid is one face
    plane)."""
    n = min(n, w.n_points)
    return np.sort(np.random.default_rng(seed).permutation(w.n_points)[:n])


def _oracle_sample(w, n, traj_start, nthreads):
    from oracle import oracle as O

    sub = w.subset(sample_points(w, n))
    t0 = time.perf_counter()
    _, _, steps = O.estimate(sub.problems, sub.points, w.L, seed=w.cfg.rng_seed, eps=w.cfg.eps_shell,
                             max_steps=w.cfg.max_steps, point_ids=sub.point_ids, inst_index=sub.inst_index,
                             traj_start=traj_start, nthreads=nthreads)
    return time.perf_counter() - t0, steps, sub.n_points


def cpu_baseline(w, budget_s=12.0, nthreads=None, full_steps_per_walk=None):
    """Oracle (reference-form C port) on the host cores over a bounded seeded sample."""
    from oracle import oracle as O

    nthreads = nthreads or O.default_threads()
    O.load()
    n, t_used = 64, 0.0
    while True:
        dt, steps, m = _oracle_sample(w, n, 0, nthreads)
        t_used += dt
        if dt >= budget_s * 0.5 or n >= w.n_points or t_used > budget_s * 2:
            break
        n = min(w.n_points, int(n * max(2.0, min(16.0, budget_s * 0.6 / max(dt, 1e-3)))))
    out = {
        "value": steps / dt,
        "unit": "walk-steps/s",
        "cores": nthreads,
        "cpu_model": cpu_model(),
        "kind": "port",
        "walks_per_s": m * w.L / dt,
        "sample": f"{m} of {w.n_points} points (seeded random sample) x {w.L} walks, reference form "
                  f"(Philox4x64, uniform-ball source, fp64), {steps} walk-steps in {dt:.2f}s",
        "sample_mean_steps_per_walk": steps / (m * w.L),
    }
    if full_steps_per_walk is not None:
        out["full_config_mean_steps_per_walk"] = full_steps_per_walk
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (oracle port) on the host cores, rank 0 only."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2603_01193_b200 import configs

    w = configs.build(args.config, mode="replay")
    nthreads = O.default_threads()
    # a bounded seeded sample per step, sized to ~1 s of host work
    n = max(32, min(w.n_points, 2048 if args.config in (4, 3) else 8192))
    for i in range(args.warmup):
        _oracle_sample(w, n, i * w.L, nthreads)
    tot_t, tot_s = 0.0, 0
    for i in range(args.steps):
        dt, s, m = _oracle_sample(w, n, (args.warmup + i) * w.L, nthreads)
        tot_t += dt
        tot_s += s
    val = tot_s / tot_t
    walks = m * w.L * args.steps / tot_t
    sample = (f"{m} of {w.n_points} points (seeded random sample) x {w.L} walks per step, "
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
        "mean_steps_per_walk": tot_s / (m * w.L * args.steps),
        "config": {"workload": w.name, "walks_per_point": w.L, "sample_points": int(m)},
        "cpu_baseline": {"value": val, "unit": "walk-steps/s", "cores": nthreads, "cpu_model": cpu_model(),
                         "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": "walk-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def roofline(cfg_index, steps, walks, seconds, seg_evals, peaks, n_sm, clk_hz):
    """Fractions of the FP32 / SFU issue roofline for `steps` walk-steps and `walks` walks in
    `seconds` of one GPU: against the nominal peak (n_SM x {16 MUFU, 256 flop} x clock)
    and against the probes measured in this run."""
    fp32, sfu = work(cfg_index, steps, walks, seg_evals)
    a_sfu, a_fp32 = sfu / seconds, fp32 / seconds
    nom_sfu, nom_fp32 = n_sm * SFU_PER_SM_CLK * clk_hz, n_sm * FP32_PER_SM_CLK * clk_hz
    fr_sfu, fr_fp32 = a_sfu / nom_sfu, a_fp32 / nom_fp32
    bound = "sfu" if fr_sfu >= fr_fp32 else "fp32"
    out = {
        "bound": bound,
        "achieved": a_sfu if bound == "sfu" else a_fp32,
        "peak": nom_sfu if bound == "sfu" else nom_fp32,
        "unit": "SFU op/s" if bound == "sfu" else "FP32 flop/s",
        "frac": fr_sfu if bound == "sfu" else fr_fp32,
        "peak_source": f"nominal: {n_sm} SMs x {SFU_PER_SM_CLK} MUFU (or {FP32_PER_SM_CLK} flop) per clock "
                       f"x {clk_hz / 1e6:.0f} MHz (max SM clock)",
        "sfu": {"achieved": a_sfu, "peak_nominal": nom_sfu, "frac": fr_sfu},
        "fp32": {"achieved": a_fp32, "peak_nominal": nom_fp32, "frac": fr_fp32},
    }
    if peaks:
        out["sfu"].update(peak_probe=peaks["sfu_ops_per_s"], frac_probe=a_sfu / peaks["sfu_ops_per_s"])
        out["fp32"].update(peak_probe=peaks["fp32_flops_per_s"], frac_probe=a_fp32 / peaks["fp32_flops_per_s"])
    F_step, S_step, F_walk, S_walk = WORK[cfg_index]
    out["work"] = {"S_step": S_step, "S_walk": S_walk, "F_walk": F_walk}
    if F_step is None:
        out["work"].update(F_step="measured", seg_evals=seg_evals,
                           segments_per_step=seg_evals / max(steps, 1),
                           F_rule=f"{SEG_FLOPS} x segment distances + {CFG3_STEP_FLOPS} x steps + "
                                  f"{F_walk} x walks")
    else:
        out["work"]["F_step"] = F_step
    return out


def _time_estimates(step_fn, stream, n, flush=None):
    """CUDA-event times (s) of n calls of step_fn(i) on `stream`."""
    import torch

    times = []
    for i in range(n):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step_fn(i)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    return times


def config_record(ctx, cfg_index, replicas, peaks, n_sm, clk_hz, flush, philox_rounds, reps=5):
    """One BASELINE config on this GPU: a single estimate's latency (median of reps
    launches, inputs resident) and replica-batched throughput (R independent label
    replicas per launch, SURVEY.md 8(d) protocol items (i) and (ii))."""
    import torch

    from paper_2603_01193_b200 import configs, engine
    from paper_2603_01193_b200.estimator import estimate_tensors

    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    out = {}
    for label, R in (("single", 1), ("replicas", replicas)):
        w = configs.build(cfg_index).replicate(R)
        cfg = dataclasses.replace(w.cfg, philox_rounds=philox_rounds)
        pset = engine.ProblemSet(ctx, w.problems)
        pts = torch.from_numpy(np.ascontiguousarray(w.points)).to(dev)
        ids = torch.from_numpy(np.ascontiguousarray(w.point_ids)).to(dev)
        inst = torch.from_numpy(np.ascontiguousarray(w.inst_index)).to(dev) if len(w.problems) > 1 else None
        eps = cfg.resolve_eps(w.problems[0].domain)
        acc = torch.zeros(1, dtype=torch.int64, device=dev)

        def one(i, acc_=None):
            estimate_tensors(pset, pts, ids, w.L, cfg, inst_index=inst, traj_start=(100 + i) * w.L,
                             total_steps=acc_, stream=stream, eps=eps)

        for i in range(2):
            one(i)
        _, seg0 = ctx.counters(stream)
        t = _time_estimates(lambda i: one(i, acc), stream, reps, flush)
        _, seg1 = ctx.counters(stream)
        S = int(acc.item()) / reps
        t_med = float(np.median(t))
        rec = {
            "replicas": R,
            "points": w.n_points,
            "walks_per_point": w.L,
            "ms": 1e3 * t_med,
            "walk_steps_per_s": S / t_med,
            "walks_per_s": w.n_walks / t_med,
            "mean_steps_per_walk": S / w.n_walks,
            "roofline": roofline(cfg_index, S, w.n_walks, t_med, (seg1 - seg0) / reps, peaks, n_sm, clk_hz),
        }
        out[label] = rec
        pset.close()
    return {"workload": configs.CONFIG_NAMES[cfg_index], "mode": "native",
            "timing": f"CUDA events, median of {reps} launches, L2 flushed before each", **out}


def replay_f64_record(ctx, cfg_index, flush, reps=2):
    """The reference's estimator on the GPU (REPLAY_F64: Philox4x64, uniform-ball source,
    fp64, draw for draw the reference's) over the full config: the like-for-like fp64
    throughput and the full config's reference-form steps per walk."""
    import torch

    from paper_2603_01193_b200 import configs, engine
    from paper_2603_01193_b200.estimator import estimate_tensors

    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    w = configs.build(cfg_index, mode="replay")
    pset = engine.ProblemSet(ctx, w.problems)
    pts = torch.from_numpy(np.ascontiguousarray(w.points)).to(dev)
    ids = torch.from_numpy(np.ascontiguousarray(w.point_ids)).to(dev)
    inst = torch.from_numpy(np.ascontiguousarray(w.inst_index)).to(dev) if len(w.problems) > 1 else None
    eps = w.cfg.resolve_eps(w.problems[0].domain)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    estimate_tensors(pset, pts, ids, w.L, w.cfg, inst_index=inst, stream=stream, eps=eps)
    t = _time_estimates(lambda i: estimate_tensors(pset, pts, ids, w.L, w.cfg, inst_index=inst,
                                                   traj_start=(1 + i) * w.L, total_steps=acc,
                                                   stream=stream, eps=eps), stream, reps, flush)
    S = int(acc.item()) / reps
    ts = float(np.mean(t))
    pset.close()
    return {"workload": w.name, "mode": "replay_f64",
            "what": "the reference's estimator draw for draw (Philox4x64, uniform-ball source, fp64)",
            "ms": 1e3 * ts, "walk_steps_per_s": S / ts, "walks_per_s": w.n_walks / ts,
            "mean_steps_per_walk": S / w.n_walks, "dtype": "f64"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", default="native")
    ap.add_argument("--philox-rounds", type=int, default=10, choices=[10, 7],
                    help="NATIVE Philox4x32 rounds (10: production stream; 7: opt-in)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the per-config sub-records and the REPLAY_F64 line")
    ap.add_argument("--replicas", type=int, default=None,
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

    # WOS_BENCH_BACKEND / WOS_BENCH_DEVICE exist only to exercise the multi-rank code path
    # on a one-GPU box (gloo, every rank on one device; each rank's kernels independent):
    # the measured configuration is NCCL with one GPU per rank
    backend = os.environ.get("WOS_BENCH_BACKEND", "nccl")
    dev_index = _env_int("WOS_BENCH_DEVICE", local)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    replicas = args.replicas or 1
    w = configs.build(args.config, mode=args.mode).replicate(replicas)
    w.cfg = dataclasses.replace(w.cfg, philox_rounds=args.philox_rounds)
    idx = shard_indices(w.n_points, rank, world)
    shard = w.subset(idx)
    ctx = engine.get_context(dev_index)
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
    # the first exterior point / watchdog / majorant flags of the warm-up: all clear
    first, watchdog, _ = ctx.status(stream)
    if first >= 0 or watchdog:
        raise RuntimeError(f"estimate flagged an error during warm-up: exterior {first}, watchdog {watchdog}")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(dev_index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0, seg0 = ctx.counters(stream)
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
    launches1, seg1 = ctx.counters(stream)
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

    # ---- roofline of the dominant kernel (the persistent walk kernel), per rank ----
    t_launch = ms * 1e-3 / args.steps
    peaks = ctx.probe_peaks() if rank == 0 else None
    n_sm = peaks["num_sms"] if peaks else torch.cuda.get_device_properties(dev).multi_processor_count
    clk_max_mhz = clk.get("sm_max_mhz") or _measured_peaks().get("sm_max_mhz") or 1965.0
    clk_hz = clk_max_mhz * 1e6
    rl = roofline(args.config, S / args.steps / world, w.n_walks / world, t_launch,
                  (seg1 - seg0) / args.steps, peaks, n_sm, clk_hz)
    traffic, traffic_src = _ncu_traffic(w.name)
    rl["traffic"] = traffic
    rl["traffic_source"] = traffic_src or "none committed"
    # the labels the estimate writes (mean, m2 per point): bytes per launch and the
    # bandwidth they take over the kernel, against the measured HBM copy bandwidth
    hbm = _measured_peaks().get("hbm_gbs")
    label_bytes = LABEL_BYTES * shard.n_points
    label = {"bytes_per_step": label_bytes, "gbs": label_bytes / t_launch / 1e9,
             "hbm_peak_gbs": hbm, "frac_of_hbm": (label_bytes / t_launch / 1e9 / hbm) if hbm else None,
             "note": "written by the fused in-kernel reduction as units retire; HBM is not the bound"}

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
    host_ids, _keep_ids = (None, None) if world == 1 and replicas == 1 and np.array_equal(
        shard.point_ids, np.arange(shard.n_points)) else pinned(np.ascontiguousarray(shard.point_ids))
    host_inst, _keep_inst = pinned(np.ascontiguousarray(shard.inst_index)) if inst is not None else (None, None)
    out_mean, _keep_mean = pinned(np.empty(shard.n_points))
    out_m2, _keep_m2 = pinned(np.empty(shard.n_points))
    from ctypes import byref, c_uint64

    wc = engine.walk_config_struct(eps, w.cfg.max_steps, w.cfg.antithetic, w.cfg.mode, w.cfg.rng_seed,
                                   philox_rounds=w.cfg.philox_rounds)
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
        extras = {}
        full_spw = None
        if world == 1 and not args.no_extras and args.mode == "native":
            # the same workload on the other NATIVE stream (10 <-> 7 Philox rounds), timed
            # the same way, so both streams' numbers come from one run
            alt = 7 if args.philox_rounds == 10 else 10
            cfg_alt = dataclasses.replace(w.cfg, philox_rounds=alt)
            acc_alt = torch.zeros(1, dtype=torch.int64, device=dev)
            n_alt = min(args.steps, 10)
            # warm-up launches first: the other stream's kernel is a different instantiation,
            # and its first launch pays the lazy module load
            for i in range(max(args.warmup, 3)):
                estimate_tensors(pset, pts, ids, w.L, cfg_alt, inst_index=inst,
                                 traj_start=(400 + i) * w.L, out_mean=mean, out_m2=m2,
                                 stream=stream, eps=eps)
            torch.cuda.synchronize()
            t_alt = _time_estimates(
                lambda i: estimate_tensors(pset, pts, ids, w.L, cfg_alt, inst_index=inst,
                                           traj_start=(500 + i) * w.L, out_mean=mean, out_m2=m2,
                                           total_steps=acc_alt, stream=stream, eps=eps),
                stream, n_alt, flush)
            S_alt = int(acc_alt.item()) / n_alt
            ta = float(np.sum(t_alt)) / n_alt
            extras["other_stream"] = {
                "philox_rounds": alt, "ms_per_step": 1e3 * ta, "value": S_alt / ta,
                "unit": "walk-steps/s", "walks_per_s": w.n_walks / ta,
                "roofline": roofline(args.config, S_alt, w.n_walks, ta, 0, peaks, n_sm, clk_hz),
                "timing": f"CUDA events, {n_alt} estimates, L2 flushed before each"}
        if world == 1 and not args.no_extras:
            if args.config == 4 and args.mode == "native":
                extras["replay_f64"] = replay_f64_record(ctx, 4, flush)
                full_spw = extras["replay_f64"]["mean_steps_per_walk"]
            extras["configs"] = {
                f"cfg{c}": config_record(ctx, c, DEFAULT_REPLICAS[c], peaks, n_sm, clk_hz, flush,
                                         args.philox_rounds)
                for c in (0, 1, 2, 3) if c != args.config
            }
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(configs.build(args.config, mode="replay").replicate(replicas),
                               full_steps_per_walk=full_spw)
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
            "dtype": "f32" if args.mode.startswith("native") or args.mode.endswith("f32") else "f64",
            "data": "synthetic (BASELINE config, pinned seeds; no dataset exists for this path)",
            "walks_per_s": walks_per_s,
            "walk_steps_per_step": S / args.steps,
            "mean_steps_per_walk": S / n_walks,
            "config": {
                "workload": w.name,
                "points": w.n_points,
                "walks_per_point": w.L,
                "instances": len(w.problems),
                "replicas": replicas,
                "eps": w.cfg.eps_shell,
                "max_steps": w.cfg.max_steps,
                "mode": args.mode,
                "philox_rounds": args.philox_rounds,
                "parallelism": f"dp{world} strided point shards + NCCL all-gather of (mean, m2)",
                "l2": "flushed (256 MiB write) before every timed step, outside the events",
                "traj_windows": "step i uses traj ids [i*L, (i+1)*L)",
            },
            "roofline": rl,
            "label_writeout": label,
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "walk-steps/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "wos_estimate_host (C ABI, pinned host buffers; copies inside, pipelined in point chunks)"},
            # kernels the library launched in the timed region (its own launch counter):
            # per step the interior check, the walk kernel and (L > 128) the chunk merge
            "gpu_launches": int(launches1 - launches0),
        }
        line.update(extras)
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
