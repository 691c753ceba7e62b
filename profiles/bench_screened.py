"""Delta-tracking throughput on one GPU vs the CPU oracle (row f2 evidence).

    python profiles/bench_screened.py > profiles/<tag>_screened.txt

Workload: the paper's varying-coefficient family (pde.VcInstance) on the unit ball
and on the unit cube, 65,536 interior points x 256 walks, eps 1e-3, NATIVE and
REPLAY forms; CUDA-event time of estimate_tensors after warm-up. The CPU line runs
the oracle's reference-form walk (fp64, all host threads) on a strided sample.
"""

import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from oracle import oracle as O  # noqa: E402  (CPU baseline only)
from paper_2603_01193_b200 import BallDomain, BoxDomain, ScreenedProblem, WalkConfig, engine  # noqa: E402
from paper_2603_01193_b200.estimator import estimate_tensors  # noqa: E402


def vc_sigma_prime(phi, a_min, a_max, y):
    # pde._vc_sigma_prime (pde.py:184-189), for the majorant only
    a, b = 4 * math.pi * phi, 3 * math.pi * phi
    x0, x1 = y[:, 0], y[:, 1]
    ca, sa, cb, sb = np.cos(a * x0), np.sin(a * x0), np.cos(b * x1), np.sin(b * x1)
    h = -x1 * x1 + ca * sb
    g0, g1 = -a * sa * sb, -2 * x1 + b * ca * cb
    lap = -2 - (a * a + b * b) * ca * sb
    sigma = a_min + (a_max - a_min) * (1 + 0.5 * np.sin(2 * math.pi * x0) * np.cos(0.5 * math.pi * x1))
    return sigma * np.exp(-h) + 0.5 * lap + 0.25 * (g0 * g0 + g1 * g1)


def main():
    rng = np.random.default_rng(0)
    phi, a_min, a_max = 0.83, 0.21, 1.17
    P, L = 65536, 256
    ctx = engine.get_context(0)
    for dname in ("ball", "cube"):
        if dname == "ball":
            dom = BallDomain([0.0, 0.0, 0.0], 1.0)
            v = rng.normal(size=(P, 3))
            pts = v / np.linalg.norm(v, axis=1)[:, None] * (0.95 * rng.random(P) ** (1 / 3))[:, None]
            probe = pts
        else:
            dom = BoxDomain([0.0, 0.0, 0.0], [1.0, 1.0, 1.0])
            pts = 0.02 + 0.96 * rng.random((P, 3))
            probe = rng.random((20000, 3))
        sb = max(1.1 * float(vc_sigma_prime(phi, a_min, a_max, probe).max()), 0.01)
        prob = ScreenedProblem(dom, vc_params=(phi, a_min, a_max))
        pset = engine.problem_set(ctx, [prob])
        dpts = torch.as_tensor(pts, device="cuda")
        ids = torch.arange(P, dtype=torch.int64, device="cuda")
        for mode in ("native", "replay"):
            cfg = WalkConfig(eps_shell=1e-3, sigma_bar=sb, rng_seed=0, mode=mode)
            steps = torch.zeros(1, dtype=torch.int64, device="cuda")
            for w in range(2):
                estimate_tensors(pset, dpts, ids, L, cfg, traj_start=w * L, total_steps=steps)
            torch.cuda.synchronize()
            steps.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for r in range(reps):
                estimate_tensors(pset, dpts, ids, L, cfg, traj_start=(10 + r) * L, total_steps=steps)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            st = int(steps.item()) / reps
            print(f"{dname:5s} {mode:7s} sigma_bar {sb:8.3f}  {ms:9.3f} ms/estimate  "
                  f"{st / (ms * 1e-3):.3e} walk-steps/s  {P * L / (ms * 1e-3):.3e} walks/s  "
                  f"mean steps {st / (P * L):.2f}")
        # CPU: the oracle's reference form on a strided sample, all host threads
        idx = np.arange(0, P, 256)
        t0 = time.perf_counter()
        _, _, tot = O.estimate([engine.problem_record(prob)], pts[idx], L, seed=0, eps=1e-3,
                               max_steps=1000, point_ids=idx, sigma_bar=sb)
        dt = time.perf_counter() - t0
        print(f"{dname:5s} cpu-oracle reference form, {O.default_threads()} threads, {len(idx)} points "
              f"x {L}: {tot / dt:.3e} walk-steps/s")


if __name__ == "__main__":
    main()
