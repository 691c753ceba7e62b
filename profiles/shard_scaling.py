"""Predicted strong scaling of cfg4 from one GPU: each rank of an N-GPU job walks the
strided shard p = r, r + N, ... (distributed.shard_indices). This times one such shard per
N on one B200 (CUDA events, L2 flushed, inputs resident) and reports N x t_1 / (N x t_N)
style efficiency t_1 / (N t_N) — the kernel-side part of the scaling (the NCCL all-gather
of (mean, m2) per step, 8 x 2 x 32768 doubles at N = 8, is not included).

    python profiles/shard_scaling.py > profiles/<tag>_shard_scaling.txt
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from paper_2603_01193_b200 import configs, engine  # noqa: E402
from paper_2603_01193_b200.distributed import shard_indices  # noqa: E402
from paper_2603_01193_b200.estimator import estimate_tensors  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    w = configs.build(4)
    ctx = engine.get_context(0)
    pset = engine.ProblemSet(ctx, w.problems)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    eps = w.cfg.resolve_eps(w.problems[0].domain)
    base = None
    for N in (1, 2, 4, 8):
        ts = []
        for r in ((0, N - 1) if N > 1 else (0,)):
            sh = w.subset(shard_indices(w.n_points, r, N))
            pts = torch.from_numpy(np.ascontiguousarray(sh.points)).to(dev)
            ids = torch.from_numpy(np.ascontiguousarray(sh.point_ids)).to(dev)
            mean = torch.empty(sh.n_points, dtype=torch.float64, device=dev)
            m2 = torch.empty_like(mean)
            for i in range(3):
                estimate_tensors(pset, pts, ids, w.L, w.cfg, traj_start=i * w.L, out_mean=mean, out_m2=m2,
                                 stream=stream, eps=eps)
            t = []
            for i in range(10):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                estimate_tensors(pset, pts, ids, w.L, w.cfg, traj_start=(10 + i) * w.L, out_mean=mean,
                                 out_m2=m2, stream=stream, eps=eps)
                b.record(stream)
                torch.cuda.synchronize()
                t.append(a.elapsed_time(b))
            ts.append(float(np.median(t)))
        tN = max(ts)  # the slowest rank sets the step
        if base is None:
            base = tN
        print(f"N={N}: shard of {w.n_points // N} points, ms per estimate (ranks 0 and N-1): "
              f"{', '.join(f'{x:.4f}' for x in ts)}; predicted speed-up {base / tN:.2f}x, "
              f"efficiency {base / (N * tN):.3f}")


if __name__ == "__main__":
    main()
