"""Large golden sets: 40,960 reference walks per BASELINE config, outputs only.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_large.py

Runs the REFERENCE's walker.walk_poisson_values (generic path, walker.py:257-314)
on the rows large_rows.py derives from the pinned configs, and stores per walk
(value f64, steps i32, hit u8) in golden_large_cfg{i}.npz. At this size the
north-star replay criterion ("identical step counts for >= 99.9 % of walks") and
the strict fp32 1e-5 rate are measured on tens of thousands of walks, not a
thousand (tests/test_gpu_replay_large.py, tests/test_oracle_golden.py).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from spherewalk import walker as W  # noqa: E402  (reference package)
from spherewalk.geometry import BallDomain as RefBall  # noqa: E402

from large_rows import large_rows  # noqa: E402
from paper_2603_01193_b200 import configs  # noqa: E402
from paper_2603_01193_b200.engine import problem_record  # noqa: E402
from ref_adapters import ref_problem  # noqa: E402


def main():
    for i in range(5):
        t0 = time.time()
        w = configs.build(i)
        c = w.cfg
        cfg = W.WalkConfig(eps_shell=c.eps_shell, max_steps=c.max_steps, rng_seed=c.rng_seed)
        inst, pts, pid, tid, sgn = large_rows(w, i)
        values = np.empty(pts.shape[0])
        steps = np.empty(pts.shape[0], np.int32)
        hits = np.empty(pts.shape[0], np.uint8)
        for k in np.unique(inst):
            m = inst == k
            prob = ref_problem(problem_record(w.problems[k]), W.Problem, RefBall)
            v, s, h = W.walk_poisson_values(prob, pts[m], pid[m], tid[m], sgn[m], cfg)
            values[m], steps[m], hits[m] = v, s, h
        np.savez_compressed(os.path.join(HERE, f"golden_large_cfg{i}.npz"), values=values, steps=steps,
                            hits=hits, seed=np.array([c.rng_seed], dtype=np.uint64))
        print(f"cfg{i}: {values.size} walks, mean steps {steps.mean():.2f}, hits {hits.mean():.4f}, "
              f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
