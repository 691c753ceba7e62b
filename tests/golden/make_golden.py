"""Generate the golden fixtures by running the REFERENCE (spherewalk) in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes small .npz files next to this script (committed; the GPU box has no
/root/reference):

* golden_rng.npz        Philox4x64-10 words from rng.philox4x64 (rng.py:57-82) on
                        the test_rng.py cases plus random counters, and numpy's
                        Philox cross-check (test_rng.py:29-54).
* golden_capture.npz    uniform draws CAPTURED from a live reference walk
                        (spherewalk.walker.philox4x64 wrapped while cfg0/cfg4 rows run):
                        counters, keys and the four words of every captured call.
* golden_cfg{i}.npz     per-walk (values, steps, hits) from
                        walker.walk_poisson_values (generic path, walker.py:257-314)
                        for rows of each BASELINE config, plus the spec records.
* golden_estimate.npz   estimator.estimate (estimator.py:144-181) means and m2.
* golden_refkernels.npz the reference's numba kernels (walk_plain_2d / walk_plain_ball3,
                        _kernels.py:286-468) on spec-coded disk/ball problems.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from spherewalk import _kernels, rng  # noqa: E402  (reference package)
from spherewalk import walker as W  # noqa: E402
from spherewalk.estimator import estimate as ref_estimate  # noqa: E402
from spherewalk.geometry import BallDomain as RefBall  # noqa: E402

from paper_2603_01193_b200 import configs  # noqa: E402
from paper_2603_01193_b200.engine import problem_record  # noqa: E402
from ref_adapters import ref_problem  # noqa: E402

MASK64 = (1 << 64) - 1


def records_array(recs):
    """Pack spec records into an object-free npz-friendly dict."""
    out = {}
    for i, (dim, dk, dp, sk, sp, bk, bp, ikey) in enumerate(recs):
        out[f"rec{i}_head"] = np.array([dim, dk, sk, bk], dtype=np.int64)
        out[f"rec{i}_dom"] = np.asarray(dp, dtype=np.float64)
        out[f"rec{i}_src"] = np.asarray(sp, dtype=np.float64)
        out[f"rec{i}_bnd"] = np.asarray(bp, dtype=np.float64)
        out[f"rec{i}_ikey"] = np.array([ikey], dtype=np.uint64)
    out["n_records"] = np.array([len(recs)])
    return out


def gen_rng():
    cases = [
        ((0, 0, 0, 0), (0, 0)),
        ((1, 2, 3, 4), (5, 6)),
        ((MASK64,) * 4, (MASK64, MASK64)),
        ((123456789, 0, 987654321, 17), (0xDEADBEEF, 42)),
    ]
    r = np.random.default_rng(12345)
    for _ in range(28):
        c = tuple(int(x) for x in r.integers(0, 2**63, size=4, dtype=np.int64))
        k = tuple(int(x) for x in r.integers(0, 2**63, size=2, dtype=np.int64))
        cases.append((c, k))
    ctr = np.array([c for c, _ in cases], dtype=np.uint64)
    key = np.array([k for _, k in cases], dtype=np.uint64)
    words = np.array([[int(w) for w in rng.philox4x64(*c, *k)] for c, k in cases], dtype=np.uint64)
    # numpy's Philox: its block at counter c equals the reference's at c + 1 (test_rng.py:29-39)
    npkey = (0x1234_5678_9ABC_DEF0, 0x0FED_CBA9_8765_4321)
    bg = np.random.Philox(counter=0, key=np.array(npkey, dtype=np.uint64))
    np_raw = bg.random_raw(16).reshape(4, 4)
    np.savez(os.path.join(HERE, "golden_rng.npz"), ctr=ctr, key=key, words=words,
             np_key=np.array(npkey, dtype=np.uint64), np_raw=np_raw)


def rows_for(w, n_pts, n_traj, rng_, instance=None):
    sel = np.arange(w.n_points) if instance is None else np.flatnonzero(w.inst_index == instance)
    pick = rng_.choice(sel, size=min(n_pts, sel.size), replace=False)
    pick.sort()
    pts = np.repeat(w.points[pick], n_traj, axis=0)
    pid = np.repeat(w.point_ids[pick], n_traj)
    tid = np.tile(np.arange(n_traj) // 2 * 2 + 7, pick.size)  # pairs share a traj id
    sign = np.tile(np.where(np.arange(n_traj) % 2 == 0, 1.0, -1.0), pick.size)
    return pts, pid, tid.astype(np.int64), sign


def run_ref_rows(rec, pts, pid, tid, sign, cfg):
    prob = ref_problem(rec, W.Problem, RefBall)
    return W.walk_poisson_values(prob, pts, pid, tid, sign, cfg)


def gen_configs():
    capture = []
    orig = W.philox4x64

    def recorder(c0, c1, c2, c3, k0, k1):
        out = orig(c0, c1, c2, c3, k0, k1)
        if sum(c[0].shape[0] for c in capture) < 4096:
            b = np.broadcast_arrays(*(np.asarray(c, dtype=np.uint64) for c in (c0, c1, c2, c3)))
            take = slice(0, None, 7)  # every 7th lane of the call keeps the fixture small
            capture.append((np.stack([np.ravel(x)[take] for x in b], axis=1), int(k0), int(k1),
                            np.stack([np.ravel(x)[take] for x in out], axis=1)))
        return out

    plan = {0: (48, 32, None), 1: (48, 32, None), 2: (24, 16, [0, 1, 2, 3]), 3: (16, 16, [0, 1, 2]),
            4: (32, 32, None)}
    for i in range(5):
        w = configs.build(i)
        recs = [problem_record(p) for p in w.problems]
        r_ = np.random.default_rng(100 + i)
        n_pts, n_traj, insts = plan[i]
        c = w.cfg
        cfg = W.WalkConfig(eps_shell=c.eps_shell, max_steps=c.max_steps, rng_seed=c.rng_seed)
        blocks = []
        for inst in insts or [None]:
            pts, pid, tid, sign = rows_for(w, n_pts, n_traj, r_, inst)
            rec = recs[0 if inst is None else inst]
            if i in (0, 4):
                W.philox4x64 = recorder
            try:
                v, s, h = run_ref_rows(rec, pts, pid, tid, sign, cfg)
            finally:
                W.philox4x64 = orig
            blocks.append((np.full(pts.shape[0], 0 if inst is None else inst, np.int32), pts, pid,
                           tid, sign, v, s, h))
        # max-steps truncation rows (hit = 0 semantics, walker.py:275-281)
        pts, pid, tid, sign = rows_for(w, 8, 8, r_, None if insts is None else insts[0])
        cfg_t = W.WalkConfig(eps_shell=c.eps_shell, max_steps=3, rng_seed=c.rng_seed)
        rec = recs[0 if insts is None else insts[0]]
        vt, st, ht = run_ref_rows(rec, pts, pid, tid, sign, cfg_t)
        cat = lambda k: np.concatenate([b[k] for b in blocks])  # noqa: E731
        np.savez(
            os.path.join(HERE, f"golden_cfg{i}.npz"),
            inst=cat(0), points=cat(1), pid=cat(2), tid=cat(3), sign=cat(4), values=cat(5),
            steps=cat(6), hits=cat(7), eps=np.array([c.eps_shell]), max_steps=np.array([c.max_steps]),
            seed=np.array([c.rng_seed], dtype=np.uint64),
            t_points=pts, t_pid=pid, t_tid=tid, t_sign=sign, t_values=vt, t_steps=st, t_hits=ht,
            t_inst=np.array([0 if insts is None else insts[0]]), t_max_steps=np.array([3]),
            **records_array(recs),
        )
        print(f"cfg{i}: {cat(5).size} rows, mean steps {cat(6).mean():.2f}, "
              f"hits {cat(7).mean():.3f}")
    ctr = np.concatenate([c[0] for c in capture])
    keys = np.concatenate([np.tile([[c[1], c[2]]], (c[0].shape[0], 1)) for c in capture]).astype(np.uint64)
    words = np.concatenate([c[3] for c in capture])
    np.savez(os.path.join(HERE, "golden_capture.npz"), ctr=ctr, key=keys, words=words)
    print(f"captured {ctr.shape[0]} Philox4x64 blocks from live reference walks")


def gen_estimate():
    out = {}
    for i, npts, L in ((0, 12, 32), (1, 8, 32), (4, 8, 32)):
        w = configs.build(i)
        rec = problem_record(w.problems[0])
        prob = ref_problem(rec, W.Problem, RefBall)
        sel = np.linspace(0, w.n_points - 1, npts).astype(int)
        for anti in (False, True):
            cfg = W.WalkConfig(eps_shell=w.cfg.eps_shell, max_steps=w.cfg.max_steps,
                               rng_seed=w.cfg.rng_seed, antithetic=anti)
            est = ref_estimate(prob, w.points[sel], L, cfg, traj_start=5, point_ids=w.point_ids[sel])
            tag = f"cfg{i}_{'anti' if anti else 'plain'}"
            out[tag + "_sel"] = sel
            out[tag + "_L"] = np.array([L])
            out[tag + "_mean"] = np.array([e.mean for e in est])
            out[tag + "_m2"] = np.array([e.m2 for e in est])
            out[tag + "_n"] = np.array([e.n_samples for e in est])
    np.savez(os.path.join(HERE, "golden_estimate.npz"), **out)


def gen_refkernels():
    """Reference numba kernels on spec-coded problems (the reference's compiled path)."""
    disk = RefBall([0.0, 0.0], 1.0)
    ball = RefBall([0.0, 0.0, 0.0], 1.0)
    cases = {
        "disk_const_src": (disk, (_kernels.SRC_CONST, (1.0,)), (_kernels.BND_CONST, (0.0,)), [0.3, -0.2]),
        "disk_rbf2_fourier5": (disk, (_kernels.SRC_RBF2, (0.7, -0.4, 0.2, 0.1, -0.3, 0.25)),
                               (_kernels.BND_FOURIER5, (0.1, 0.5, -0.2, 0.3, 0.05)), [-0.1, 0.4]),
        "disk_linear": (disk, None, (_kernels.BND_LINEAR, (0.5, 0.2, 0.3)), [0.2, 0.1]),
        "ball_const_src": (ball, (_kernels.SRC_CONST, (1.0,)), (_kernels.BND_CONST, (0.0,)), [0.1, 0.2, -0.3]),
        "ball_linear": (ball, (_kernels.SRC_CONST, (-2.0,)), (_kernels.BND_LINEAR, (0.3, -0.1, 0.2, 0.5)),
                        [0.0, 0.0, 0.0]),
    }
    out = {}
    n = 512
    for name, (dom, sspec, bspec, x0) in cases.items():
        prob = W.Problem(dom, boundary=lambda q: q[:, 0], source=None if sspec is None else (lambda y: y[:, 0]),
                         instance_key=3, boundary_spec=bspec, source_spec=sspec)
        cfg = W.WalkConfig(rng_seed=11, max_steps=1000)
        pts = np.tile(np.asarray(x0, dtype=np.float64), (n, 1))
        pid = np.full(n, 2)
        tid = np.arange(n) // 2
        sign = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
        v, s, h = W.walk_poisson_values(prob, pts, pid, tid, sign, cfg)
        out[name + "_points"] = pts
        out[name + "_pid"] = pid
        out[name + "_tid"] = tid
        out[name + "_sign"] = sign
        out[name + "_values"] = v
        out[name + "_steps"] = s
        out[name + "_hits"] = h
        out[name + "_dim"] = np.array([dom.dim])
        out[name + "_src"] = np.array([-1 if sspec is None else sspec[0]] + list(sspec[1] if sspec else []), dtype=np.float64)
        out[name + "_bnd"] = np.array([bspec[0]] + list(bspec[1]), dtype=np.float64)
        out[name + "_eps"] = np.array([cfg.resolve_eps(dom)])
    out["names"] = np.array(list(cases))
    np.savez(os.path.join(HERE, "golden_refkernels.npz"), **out)


if __name__ == "__main__":
    gen_rng()
    gen_configs()
    gen_estimate()
    gen_refkernels()
    print("golden fixtures written to", HERE)
