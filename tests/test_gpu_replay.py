"""Replay parity on the GPU: the CUDA path consumes the reference's own draws.

REPLAY_F64 regenerates the reference's Philox4x64 draws on the device (checked
bit-exactly against draws captured from live reference walks) and runs the
reference's estimator operation by operation: step counts must be identical
and values equal to rounding. REPLAY_F32 runs the same walks in fp32; the
north-star bar is identical steps for >= 99.9 % of walks and per-walk values
within 1e-5 relative (floored at the point's walk RMS).
"""

import numpy as np
import pytest

from conftest import RecordProblem, golden_records, load_golden

pytestmark = pytest.mark.gpu

CFGS = [0, 1, 2, 3, 4]


def _torch_dev(x, dtype=None):
    import torch

    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda:0")


def test_gpu_philox4x64_matches_reference(gpu):
    import torch

    from paper_2603_01193_b200 import _lib

    z = load_golden("golden_rng.npz")
    L = _lib.lib()
    for c, k, w in zip(z["ctr"], z["key"], z["words"]):
        ctr = _torch_dev(c.view(np.int64)[None, :])
        out = torch.empty_like(ctr)
        _lib.check(L.wos_philox4x64(gpu.handle, 1, ctr.data_ptr(), int(k[0]), int(k[1]), out.data_ptr(), None))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint64)[0], w)


def test_gpu_philox4x64_matches_captured_reference_draws(gpu):
    import torch

    from paper_2603_01193_b200 import _lib

    z = load_golden("golden_capture.npz")
    L = _lib.lib()
    for k0, k1 in {(int(a), int(b)) for a, b in z["key"]}:
        m = (z["key"][:, 0] == k0) & (z["key"][:, 1] == k1)
        ctr = _torch_dev(z["ctr"][m].view(np.int64))
        out = torch.empty_like(ctr)
        _lib.check(L.wos_philox4x64(gpu.handle, ctr.shape[0], ctr.data_ptr(), k0, k1, out.data_ptr(), None))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint64), z["words"][m])


def test_gpu_philox4x32_kat(gpu):
    import torch

    from oracle import oracle as O
    from paper_2603_01193_b200 import _lib

    L = _lib.lib()
    rng = np.random.default_rng(5)
    ctr = rng.integers(0, 2**32, size=(4096, 4), dtype=np.uint64).astype(np.uint32)
    for k0, k1 in [(0, 0), (0xDEADBEEF, 7), (0xFFFFFFFF, 0xFFFFFFFF)]:
        d = _torch_dev(ctr.view(np.int32))
        out = torch.empty_like(d)
        _lib.check(L.wos_philox4x32(gpu.handle, d.shape[0], d.data_ptr(), k0, k1, out.data_ptr(), None))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), O.philox4x32(ctr, k0, k1))
    for c, k, want in O.PHILOX4X32_KAT:
        d = _torch_dev(np.array([c], dtype=np.uint32).view(np.int32))
        out = torch.empty_like(d)
        _lib.check(L.wos_philox4x32(gpu.handle, 1, d.data_ptr(), k[0], k[1], out.data_ptr(), None))
        torch.cuda.synchronize()
        assert [int(v) for v in out.cpu().numpy().view(np.uint32)[0]] == list(want)


def _rows(z, prefix=""):
    return (z[prefix + "points"], z[prefix + "pid"], z[prefix + "tid"], z[prefix + "sign"])


@pytest.mark.parametrize("cfg", CFGS)
def test_replay_f64_rows_match_reference(gpu, cfg):
    from paper_2603_01193_b200 import WalkConfig, walk_poisson_values

    z = load_golden(f"golden_cfg{cfg}.npz")
    recs = golden_records(z)
    wc = WalkConfig(eps_shell=float(z["eps"][0]), max_steps=int(z["max_steps"][0]),
                    rng_seed=int(z["seed"][0]), mode="replay")
    for inst in np.unique(z["inst"]):
        m = z["inst"] == inst
        pts, pid, tid, sgn = (a[m] for a in _rows(z))
        v, s, h = walk_poisson_values(RecordProblem(recs[inst]), pts, pid, tid, sgn, wc)
        assert np.array_equal(s, z["steps"][m]), f"steps differ on {np.mean(s != z['steps'][m]):.4%}"
        assert np.array_equal(h, z["hits"][m])
        np.testing.assert_allclose(v, z["values"][m], rtol=1e-9, atol=1e-13)


@pytest.mark.parametrize("cfg", CFGS)
def test_replay_f64_truncated_rows(gpu, cfg):
    from paper_2603_01193_b200 import WalkConfig, walk_poisson_values

    z = load_golden(f"golden_cfg{cfg}.npz")
    rec = golden_records(z)[int(z["t_inst"][0])]
    wc = WalkConfig(eps_shell=float(z["eps"][0]), max_steps=3, rng_seed=int(z["seed"][0]), mode="replay")
    v, s, h = walk_poisson_values(RecordProblem(rec), *_rows(z, "t_"), wc)
    assert np.array_equal(s, z["t_steps"])
    assert np.array_equal(h, z["t_hits"])
    np.testing.assert_allclose(v, z["t_values"], rtol=1e-9, atol=1e-13)


@pytest.mark.parametrize("cfg", CFGS)
def test_replay_f32_rows_within_fp32_tolerance(gpu, cfg):
    """North-star check 1: identical steps >= 99.9 %, values within 1e-5 (floored)."""
    from paper_2603_01193_b200 import WalkConfig, walk_poisson_values

    z = load_golden(f"golden_cfg{cfg}.npz")
    recs = golden_records(z)
    wc = WalkConfig(eps_shell=float(z["eps"][0]), max_steps=int(z["max_steps"][0]),
                    rng_seed=int(z["seed"][0]), mode="replay_f32")
    same_steps, within = [], []
    for inst in np.unique(z["inst"]):
        m = z["inst"] == inst
        pts, pid, tid, sgn = (a[m] for a in _rows(z))
        v, s, _ = walk_poisson_values(RecordProblem(recs[inst]), pts, pid, tid, sgn, wc)
        ref = z["values"][m]
        same_steps.append(s == z["steps"][m])
        # floor: RMS of the walks of the same start point (relative error is ill-conditioned at 0)
        key = pid.astype(np.int64)
        rms = np.empty_like(ref)
        for p in np.unique(key):
            sel = key == p
            rms[sel] = np.sqrt(np.mean(ref[sel] ** 2))
        within.append(np.abs(v - ref) <= 1e-5 * np.maximum(np.abs(ref), rms) + 1e-12)
    same = np.concatenate(same_steps).mean()
    ok = np.concatenate(within).mean()
    assert same >= 0.999, f"identical step counts {same:.4%}"
    assert ok >= 0.99, f"within floored 1e-5: {ok:.4%}"


def test_replay_reference_numba_kernel_problems(gpu):
    """Spec-coded disk/ball problems the reference runs in walk_plain_2d / walk_plain_ball3."""
    from paper_2603_01193_b200 import WalkConfig, walk_poisson_values
    from test_oracle_golden import _refkernel_record

    z = load_golden("golden_refkernels.npz")
    for name in z["names"]:
        name = str(name)
        rec = _refkernel_record(z, name)
        wc = WalkConfig(eps_shell=float(z[name + "_eps"][0]), max_steps=1000, rng_seed=11, mode="replay")
        v, s, h = walk_poisson_values(RecordProblem(rec), z[name + "_points"], z[name + "_pid"],
                                      z[name + "_tid"], z[name + "_sign"], wc)
        assert np.array_equal(s, z[name + "_steps"]), name
        assert np.array_equal(h, z[name + "_hits"]), name
        np.testing.assert_allclose(v, z[name + "_values"], rtol=1e-9, atol=1e-12, err_msg=name)


@pytest.mark.parametrize("cfg", [0, 1, 4])
@pytest.mark.parametrize("anti", [False, True])
def test_replay_estimate_matches_reference(gpu, cfg, anti):
    from paper_2603_01193_b200 import configs, estimate_arrays

    w = configs.build(cfg, mode="replay")
    z = load_golden("golden_estimate.npz")
    tag = f"cfg{cfg}_{'anti' if anti else 'plain'}"
    sel = z[tag + "_sel"]
    L = int(z[tag + "_L"][0])
    from dataclasses import replace

    cfg_ = replace(w.cfg, antithetic=anti)
    mean, m2, n = estimate_arrays(w.problems, w.points[sel], L, cfg_, point_ids=w.point_ids[sel],
                                  traj_start=5)
    np.testing.assert_allclose(mean, z[tag + "_mean"], rtol=1e-9, atol=1e-14)
    np.testing.assert_allclose(m2, z[tag + "_m2"], rtol=1e-7, atol=1e-14)
    assert np.array_equal(n, z[tag + "_n"])
