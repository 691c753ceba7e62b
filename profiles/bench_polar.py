"""Polar star-curve throughput on one GPU vs the CPU oracle (row f3 evidence).

    python profiles/bench_polar.py > profiles/<tag>_polar.txt

Workload: the paper's linear family (pde.LinearInstance: PolarDomain, RBF2 source,
FOURIER5 boundary), a mild curve (|c1| + |c2| <= 0.45: strided table scan) and a
strong one (full 4096-sample scan), 65,536 interior points x 256 walks, eps = the
reference default, NATIVE and REPLAY; CUDA-event time of estimate_tensors. The CPU
line runs the oracle's reference form (fp64, all host threads) on a strided sample.
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from oracle import oracle as O  # noqa: E402  (CPU baseline only)
from paper_2603_01193_b200 import PolarDomain, Problem, WalkConfig, engine  # noqa: E402
from paper_2603_01193_b200.estimator import estimate_tensors  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    P, L = 65536, 256
    ctx = engine.get_context(0)
    for name, (c1, c2) in (("mild", (0.12, -0.09)), ("strong", (0.3, -0.25))):
        dom = PolarDomain(1.0, c1, c2)
        lo, hi = dom.bounding_box()
        cand = lo + (hi - lo) * rng.random((4 * P, 2))
        pts = cand[dom.contains(cand)][:P]
        prob = Problem(dom, boundary_spec=(1, (0.2, -0.5, 0.3, 0.8, -0.1)),
                       source_spec=(2, (0.4, -0.7, 0.1, 0.2, -0.3, 0.05)), instance_key=3)
        pset = engine.problem_set(ctx, [prob])
        dpts = torch.as_tensor(pts, device="cuda")
        ids = torch.arange(P, dtype=torch.int64, device="cuda")
        eps = 1e-3 * dom.bounding_radius()
        for mode in ("native", "replay"):
            cfg = WalkConfig(eps_shell=eps, rng_seed=0, mode=mode)
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
            print(f"{name:6s} {mode:7s} stride {dom._stride:2d}  {ms:9.3f} ms/estimate  "
                  f"{st / (ms * 1e-3):.3e} walk-steps/s  {P * L / (ms * 1e-3):.3e} walks/s  "
                  f"mean steps {st / (P * L):.2f}")
        idx = np.arange(0, P, 512)
        t0 = time.perf_counter()
        _, _, tot = O.estimate([engine.problem_record(prob)], pts[idx], L, seed=0, eps=eps,
                               max_steps=1000, point_ids=idx)
        dt = time.perf_counter() - t0
        print(f"{name:6s} cpu-oracle reference form, {O.default_threads()} threads, {len(idx)} points "
              f"x {L}: {tot / dt:.3e} walk-steps/s")


if __name__ == "__main__":
    main()
