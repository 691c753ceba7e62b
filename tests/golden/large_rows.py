"""Input recipe of the large golden sets (tests/golden/golden_large_cfg{i}.npz).

The large sets store only the reference's OUTPUTS (per-walk value, step count,
hit flag); their inputs are re-derived here from the pinned BASELINE configs and
a fixed seed, by the generator (make_golden_large.py, in this container, against
the reference) and by the tests (on the GPU box) alike.

Rows: for each config, N_POINTS[i] query points drawn without replacement by
np.random.default_rng(7000 + i) (per instance for the multi-instance configs),
each with W trajectory ids 0..W-1 (all sign +1): 40,960
walks per config.
"""

from __future__ import annotations

import numpy as np

# (points per instance, instances, walks per point): 40,960 walks per config
# (cfg0: all 1,024 points x 40; cfg2: 16 instances x 80 points; cfg3: 8 polygons x 160)
PLAN = {0: (1024, None, 40), 1: (1280, None, 32), 2: (80, 16, 32), 3: (160, 8, 32), 4: (1280, None, 32)}


def large_rows(w, cfg_index):
    """(inst, points, point_ids, traj_ids, signs) of config cfg_index's large golden set."""
    n_pts, n_inst, n_walks = PLAN[cfg_index]
    rng = np.random.default_rng(7000 + cfg_index)
    insts = [None] if n_inst is None else list(range(n_inst))
    blocks = []
    for inst in insts:
        sel = np.arange(w.n_points) if inst is None else np.flatnonzero(w.inst_index == inst)
        pick = np.sort(rng.choice(sel, size=n_pts, replace=False))
        blocks.append((np.full(n_pts * n_walks, 0 if inst is None else inst, np.int32),
                       np.repeat(w.points[pick], n_walks, axis=0),
                       np.repeat(w.point_ids[pick], n_walks),
                       np.tile(np.arange(n_walks, dtype=np.int64), n_pts)))
    inst = np.concatenate([b[0] for b in blocks])
    pts = np.concatenate([b[1] for b in blocks])
    pid = np.concatenate([b[2] for b in blocks]).astype(np.int64)
    tid = np.concatenate([b[3] for b in blocks])
    return inst, pts, pid, tid, np.ones(pts.shape[0])
