"""Full-size statistical validation of the GPU estimator against the closed forms.

    python profiles/validate_full.py > profiles/<tag>_full_validation.txt

For each BASELINE config with an analytic solution (cfg0, cfg1, cfg4), at the full
BASELINE size (every query point, the configured walks per point), NATIVE and REPLAY:

* per-point z = (mean - u(x)) / SE: rms z, mean z, max |z| and the count of |z| > 4;
* the rms error at L and at 16 L (16 independent trajectory windows pooled by the
  Chan merge): 1/sqrt(N) predicts a ratio of 4;
* the walk-weighted mean error relative to the rms SE (bias check).

The eps-shell bias of WoS is O(eps |grad u|) and walk values are skewed (per-point
sample SEs at small L are noisy), so rms z slightly above 1 is expected.
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from paper_2603_01193_b200 import configs, estimate_arrays  # noqa: E402


def merge(n1, m1, q1, n2, m2, q2):
    """Chan merge of per-point (count, mean, m2) arrays (estimator.chan_merge, vectorised)."""
    n = n1 + n2
    d = m2 - m1
    return n, m1 + d * (n2 / n), q1 + q2 + d * d * (n1 * n2 / n)


def run(cfg, mode, R=16):
    w = configs.build(cfg, mode=mode)
    exact = w.analytic(w.points)
    t0 = time.perf_counter()
    parts = []
    for r in range(R):
        parts.append(estimate_arrays(w.problems, w.points, w.L, w.cfg, point_ids=w.point_ids,
                                     traj_start=r * w.L))
    dt = time.perf_counter() - t0
    mean, m2, n = (np.asarray(a, dtype=np.float64) for a in parts[0])
    se = np.sqrt(m2 / (n - 1) / n)
    z = (mean - exact) / se
    err1 = float(np.sqrt(np.mean((mean - exact) ** 2)))
    N, M, Q = n.astype(np.float64), mean.copy(), m2.copy()
    for mu, q, k in parts[1:]:
        N, M, Q = merge(N, M, Q, np.asarray(k, np.float64), np.asarray(mu), np.asarray(q))
    seR = np.sqrt(Q / (N - 1) / N)
    zR = (M - exact) / seR
    errR = float(np.sqrt(np.mean((M - exact) ** 2)))
    print(f"cfg{cfg} {mode:6s} P={w.n_points} L={w.L}: rms z {np.sqrt(np.mean(z**2)):.3f}  mean z {np.mean(z):+.3f}"
          f"  max|z| {np.max(np.abs(z)):.2f}  #|z|>4 {int(np.sum(np.abs(z) > 4))}  |"
          f"  L x{R}: rms z {np.sqrt(np.mean(zR**2)):.3f}  mean z {np.mean(zR):+.3f}  max|z| {np.max(np.abs(zR)):.2f}"
          f"  |  rms err L {err1:.3e}, {R}L {errR:.3e}, ratio {err1 / errR:.2f} (1/sqrt(N): {np.sqrt(R):.1f})"
          f"  |  mean err / rms SE {np.mean(M - exact) / np.sqrt(np.mean(seR**2)):+.3f}  ({dt:.1f} s)", flush=True)


def main():
    for cfg in (0, 1, 4):
        for mode in ("native", "replay"):
            run(cfg, mode)


if __name__ == "__main__":
    main()
