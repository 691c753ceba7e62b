"""Per-walk difference of the NATIVE fp32 fast-math kernel vs the oracle's fp64 restatement of the
same native stream (BASELINE configs, 256 points x 64 walks each): profiles/r1e_native_error.txt."""
import sys, os, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
from oracle import oracle as O
from paper_2603_01193_b200 import configs, walk_poisson_values
for cfg in range(5):
    w = configs.build(cfg)
    sel = np.flatnonzero(w.inst_index == 0)[:256]
    T = 64
    pts = np.repeat(w.points[sel], T, axis=0); pid = np.repeat(w.point_ids[sel], T); tid = np.tile(np.arange(T), sel.size)
    sgn = np.ones(pts.shape[0])
    v, s, h = walk_poisson_values(w.problems[0], pts, pid, tid, sgn, w.cfg)
    vo, so, ho = O.walk_rows(w.problems[0], pts, pid, tid, sgn, seed=w.cfg.rng_seed, eps=w.cfg.eps_shell, max_steps=w.cfg.max_steps, native=True)
    m = s == so
    rms = np.sqrt(np.mean(vo**2))
    err = np.abs(v[m] - vo[m]) / rms
    bias = np.mean(v[m] - vo[m]) / rms
    print(f"cfg{cfg}: walks {len(v)} identical steps {m.mean():.5f}  |dv|/rms: median {np.median(err):.2e} p99 {np.quantile(err,0.99):.2e} max {err.max():.2e}  mean(dv)/rms {bias:+.2e}  rms {rms:.3e}")
