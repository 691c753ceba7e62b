"""North-star check 1 rates on the large golden sets (run on the GPU box).

    python profiles/replay_parity.py > profiles/<tag>_replay_parity.txt

For each config: REPLAY_F64 (must reproduce every reference walk) and REPLAY_F32
(identical step counts, strict and floored 1e-5 rates) over 40,960 reference walks.
"""

import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_gpu_replay_large import replay_rates  # noqa: E402

print("cfg  mode        walks  identical_steps  strict_1e-5  floored_1e-5  max|dv|/rms")
for cfg in range(5):
    for mode in ("replay", "replay_f32"):
        same, strict, floored, hits, worst, n = replay_rates(cfg, mode)
        print(f"{cfg:3d}  {mode:10s} {n:6d}  {same.mean():15.6f}  {strict.mean():11.6f}  "
              f"{floored.mean():12.6f}  {worst:.3e}")
        if mode == "replay_f32":
            print(f"     (walks with identical steps: strict {strict[same].mean():.6f}, floored "
                  f"{floored[same].mean():.6f}; differing steps: {int((~same).sum())} walks)")
