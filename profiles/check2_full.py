"""North-star check 2 at full size: NATIVE (GPU) vs the reference form, every point.

    python profiles/check2_full.py [--configs 0 1 2 3 4] [--rounds 10] > profiles/<tag>_check2_full.txt

For each BASELINE config, every query point at the configured walks per point:
  * NATIVE_F32 estimate on the GPU (the production kernel), two independent runs
    (rng_seed s and s + 3);
  * the reference form on the host cores: the C oracle (oracle/wos_oracle.c, pinned
    bit-for-bit to the reference's walks on 204,800 golden rows), two independent runs
    (seeds s + 1 and s + 2) (estimator.estimate semantics, estimator.py:144-181).
Scores (points starting inside the eps-shell have zero variance in both arms; a
1e-6 floor keeps them finite):
  * z per point with the runs' own sample SEs: rms z (~1), mean z (~0), the counts of
    |z| > 3 and |z| > 4 against their normal expectations (2.7e-3 P and 6.3e-5 P);
  * the same z with the SEs taken from the OTHER run of each arm: walk values are
    skewed (the reference form's 1/r source weight most of all), so a run's sample SE
    is correlated with its own mean error and biases the mean of the self-SE z (cfg4:
    -0.11); independent SEs remove that correlation;
  * the global z: the mean difference over all points against its pooled SE (a
    systematic bias of the native estimator would show here).
  * z of 64-point bin means (consecutive points of one instance, SEs from the
    independent runs): a bin's SE sums 64 sample variances, so it is far less noisy
    than a point's — the check that also covers cfg2, whose L = 4 makes per-point SEs
    Student-t with 3 dof.
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
        multi = len(w.problems) > 1
        inst = w.inst_index if multi else None
        L = w.L

        def gpu(seed):
            cfg = dataclasses.replace(w.cfg, philox_rounds=a.rounds, rng_seed=seed)
            return estimate_arrays(w.problems, w.points, L, cfg, point_ids=w.point_ids, inst_index=inst)[:2]

        def ref(seed):
            om, ov, steps = O.estimate(w.problems, w.points, L, seed=seed, eps=w.cfg.eps_shell,
                                       max_steps=w.cfg.max_steps, point_ids=w.point_ids, inst_index=inst,
                                       nthreads=nthreads)
            return om, ov, steps

        s0 = w.cfg.rng_seed
        t0 = time.time()
        m, v = gpu(s0)
        _, v_b = gpu(s0 + 3)
        t1 = time.time()
        om, ov, steps = ref(s0 + 1)
        t2 = time.time()
        _, ov_b, _ = ref(s0 + 2)
        se = lambda var: np.sqrt(var / (L - 1) / L)  # noqa: E731
        floor = 1e-6 * np.maximum(1.0, np.abs(om))
        z = (m - om) / np.sqrt(se(v)**2 + se(ov)**2 + floor**2)
        z_ind = (m - om) / np.sqrt(se(v_b)**2 + se(ov_b)**2 + floor**2)
        g = np.sum(m - om) / np.sqrt(np.sum(se(v_b)**2 + se(ov_b)**2))
        print(f"cfg{c} {w.name}: {w.n_points} points x {L} walks; GPU 2 runs {t1 - t0:.1f}s, reference form "
              f"{t2 - t1:.1f}s per run ({steps / max(t2 - t1, 1e-9):.3g} walk-steps/s)")
        zstats(z, "per point, own SEs")
        zstats(z_ind, "per point, SEs of the independent runs")
        print(f"  global: mean difference {np.mean(m - om):+.3e} = {g:+.3f} pooled SE")
        # 64-point bins (consecutive points of one instance): 64 L walks per bin mean, whose
        # SE is a sum of 64 sample variances and so far less noisy than a point's
        zb = []
        for k in range(len(w.problems)):
            idx = np.flatnonzero(w.inst_index == k)
            for b in range(0, idx.size - 63, 64):
                s = idx[b:b + 64]
                d = m[s].mean() - om[s].mean()
                var = (np.sum(v_b[s] / (L - 1)) + np.sum(ov_b[s] / (L - 1))) / L / 64**2
                zb.append(d / np.sqrt(var))
        zstats(np.asarray(zb), "64-point bins, SEs of the independent runs")
        sys.stdout.flush()


if __name__ == "__main__":
    main()
