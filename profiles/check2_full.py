"""North-star check 2 at full size: NATIVE (GPU) vs the reference form, every point.

    python profiles/check2_full.py [--configs 0 1 2 3 4] [--rounds 10] > profiles/<tag>_check2_full.txt

For each BASELINE config, every query point at the configured walks per point:
  * NATIVE_F32 estimate on the GPU (the production kernel, seed s);
  * the reference form on the host cores: the C oracle (oracle/wos_oracle.c, pinned
    bit-for-bit to the reference's walks on 204,800 golden rows), independent seed s + 1
    (estimator.estimate semantics, estimator.py:144-181).
Per point z = (m_gpu - m_ref) / sqrt(se_gpu^2 + se_ref^2) (points starting inside the
eps-shell have zero variance in both arms; a 1e-6 floor keeps them finite). Reported:
rms z (~1), mean z (~0), the counts of |z| > 3 and |z| > 4 against their normal
expectations (2.7e-3 P and 6.3e-5 P, with binomial standard deviations). cfg2 runs
L = 4 walks per point, where per-point sample SEs follow Student-t with 3 dof, so it
is also scored on the means of 64-point bins of one instance (256 walks per bin).
"""

import argparse
import dataclasses
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2603_01193_b200 import configs, estimate_arrays  # noqa: E402


def zstats(z, label):
    P = z.size
    n3, n4 = int(np.sum(np.abs(z) > 3)), int(np.sum(np.abs(z) > 4))
    e3, e4 = 2.6998e-3 * P, 6.334e-5 * P
    print(f"  {label}: P={P} rms z {np.sqrt(np.mean(z**2)):.4f}  mean z {np.mean(z):+.4f}  "
          f"|z|>3: {n3} (expected {e3:.1f} +- {np.sqrt(e3):.1f})  |z|>4: {n4} "
          f"(expected {e4:.2f} +- {np.sqrt(e4):.2f})  max |z| {np.max(np.abs(z)):.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[0, 1, 2, 3, 4])
    ap.add_argument("--rounds", type=int, default=10)
    a = ap.parse_args()
    nthreads = O.default_threads()
    print(f"host threads for the reference form: {nthreads}; NATIVE Philox rounds: {a.rounds}")
    for c in a.configs:
        w = configs.build(c)
        cfg = dataclasses.replace(w.cfg, philox_rounds=a.rounds)
        multi = len(w.problems) > 1
        t0 = time.time()
        m, v, n = estimate_arrays(w.problems, w.points, w.L, cfg, point_ids=w.point_ids,
                                  inst_index=w.inst_index if multi else None)
        t1 = time.time()
        om, ov, steps = O.estimate(w.problems, w.points, w.L, seed=w.cfg.rng_seed + 1, eps=w.cfg.eps_shell,
                                   max_steps=w.cfg.max_steps, point_ids=w.point_ids,
                                   inst_index=w.inst_index if multi else None, nthreads=nthreads)
        t2 = time.time()
        L = w.L
        se1 = np.sqrt(v / (L - 1) / L)
        se2 = np.sqrt(ov / (L - 1) / L)
        floor = 1e-6 * np.maximum(1.0, np.abs(om))
        z = (m - om) / np.sqrt(se1**2 + se2**2 + floor**2)
        print(f"cfg{c} {w.name}: {w.n_points} points x {L} walks; GPU {t1 - t0:.1f}s, reference form "
              f"{t2 - t1:.1f}s ({steps / max(t2 - t1, 1e-9):.3g} walk-steps/s)")
        zstats(z, "per point")
        if c == 2:
            # 64-point bins within each instance: 256 walks per bin mean
            zb = []
            for k in range(len(w.problems)):
                idx = np.flatnonzero(w.inst_index == k)
                for b in range(0, idx.size - 63, 64):
                    s = idx[b:b + 64]
                    d = m[s].mean() - om[s].mean()
                    # variance of a bin mean = sum of the per-point variances / 64^2
                    var = (np.sum(v[s] / (L - 1)) + np.sum(ov[s] / (L - 1))) / L / 64**2
                    zb.append(d / np.sqrt(var))
            zstats(np.asarray(zb), "64-point bins")
        sys.stdout.flush()


if __name__ == "__main__":
    main()
