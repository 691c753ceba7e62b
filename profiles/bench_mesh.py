"""Triangle-mesh domain throughput on one GPU vs the CPU oracle (row f3 evidence).

    python profiles/bench_mesh.py > profiles/<tag>_mesh.txt

Workload: geodesic spheres with 320, 5,120 and 81,920 triangles (subdivided
icosahedra), Poisson problem f = -1, g linear, 65,536 interior points x 64 walks,
NATIVE and REPLAY; CUDA-event time of estimate_tensors. The CPU line runs the
oracle's reference form (brute-force nearest triangle, fp64, all host threads).
"""

import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from oracle import oracle as O  # noqa: E402  (CPU baseline only)
from paper_2603_01193_b200 import MeshDomain, Problem, WalkConfig, engine  # noqa: E402
from paper_2603_01193_b200.estimator import estimate_tensors  # noqa: E402


def icosphere(sub):
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
         (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    v = [np.array(p, float) / np.linalg.norm(p) for p in v]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
         (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(sub):
        mid = {}

        def m(i, j):
            k = (min(i, j), max(i, j))
            if k not in mid:
                p = v[i] + v[j]
                v.append(p / np.linalg.norm(p))
                mid[k] = len(v) - 1
            return mid[k]

        nf = []
        for i, j, k in f:
            a, b, c = m(i, j), m(j, k), m(k, i)
            nf += [(i, a, c), (j, b, a), (k, c, b), (a, b, c)]
        f = nf
    return np.array(v), np.array(f)


def main():
    rng = np.random.default_rng(0)
    P, L = 65536, 64
    ctx = engine.get_context(0)
    for sub in (2, 4, 6):
        V, F = icosphere(sub)
        dom = MeshDomain(V, F)
        prob = Problem(dom, boundary_spec=(2, (1.0, 2.0, -1.0, 0.5)), source_spec=(1, (-1.0,)))
        d = rng.normal(size=(P, 3))
        pts = d / np.linalg.norm(d, axis=1)[:, None] * (0.9 * rng.random(P) ** (1 / 3))[:, None]
        pset = engine.problem_set(ctx, [prob])
        dpts = torch.as_tensor(pts, device="cuda")
        ids = torch.arange(P, dtype=torch.int64, device="cuda")
        eps = 1e-3 * dom.bounding_radius()
        for mode in ("native", "replay"):
            cfg = WalkConfig(eps_shell=eps, rng_seed=0, mode=mode)
            steps = torch.zeros(1, dtype=torch.int64, device="cuda")
            estimate_tensors(pset, dpts, ids, L, cfg, total_steps=steps)
            torch.cuda.synchronize()
            steps.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for r in range(2):
                estimate_tensors(pset, dpts, ids, L, cfg, traj_start=(5 + r) * L, total_steps=steps)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 2
            st = int(steps.item()) / 2
            print(f"{F.shape[0]:6d} faces {mode:7s} {ms:9.3f} ms/estimate  {st / (ms * 1e-3):.3e} "
                  f"walk-steps/s  mean steps {st / (P * L):.2f}")
        idx = np.arange(0, P, 2048 if sub < 6 else 8192)
        t0 = time.perf_counter()
        _, _, tot = O.estimate([engine.problem_record(prob)], pts[idx], L, seed=0, eps=eps,
                               max_steps=1000, point_ids=idx)
        dt = time.perf_counter() - t0
        print(f"{F.shape[0]:6d} faces cpu-oracle (brute force), {O.default_threads()} threads, "
              f"{len(idx)} points x {L}: {tot / dt:.3e} walk-steps/s")


if __name__ == "__main__":
    main()
