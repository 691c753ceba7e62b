"""The sharded estimator on the CUDA kernel (north_star: points shard across GPUs).

The reference fans ``estimate`` out over a process pool and pins identical bits
for any worker count (pkg/tests/test_estimator.py:147-154, fan-out at
estimator.py:166-181). Here a shard is a strided slice of the points (point p ->
shard p mod N, distributed.shard_indices); this file runs N in {2, 3, 8} shards
through the real kernel on cuda:0 — one device stands in for N, each shard an
independent launch, no shard waits on another — and reassembles them with the
gather's own permutation (pack_shard / unpack_gathered), then runs a world-2 gloo
job whose ranks both walk on cuda:0. Every result must equal the unsharded
estimate bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_01193_b200 import configs, engine
from paper_2603_01193_b200.distributed import pack_shard, shard_indices, unpack_gathered
from paper_2603_01193_b200.estimator import estimate_arrays, estimate_tensors

pytestmark = pytest.mark.gpu


def _device_estimate(pset, w, idx, stream):
    dev = torch.device("cuda", 0)
    pts = torch.from_numpy(np.ascontiguousarray(w.points[idx])).to(dev)
    ids = torch.from_numpy(np.ascontiguousarray(w.point_ids[idx])).to(dev)
    inst = (torch.from_numpy(np.ascontiguousarray(w.inst_index[idx])).to(dev)
            if len(w.problems) > 1 else None)
    return estimate_tensors(pset, pts, ids, w.L, w.cfg, inst_index=inst, stream=stream,
                            eps=w.cfg.resolve_eps(w.problems[0].domain), check=True)


@pytest.mark.parametrize("cfg_index,n_points", [(4, None), (2, 65536)])
def test_strided_shards_on_the_kernel_equal_unsharded(gpu, cfg_index, n_points):
    """cfg4 (all 262,144 points x 256 walks) and cfg2 (64 instances, 4 walks) as 2, 3 and
    8 strided shards through estimate_tensors, reassembled with the all-gather's
    permutation: bitwise equal to the single launch."""
    w = configs.build(cfg_index)
    if n_points is not None:
        w = w.subset(np.arange(0, w.n_points, w.n_points // n_points)[:n_points])
    ctx = engine.get_context(0)
    pset = engine.ProblemSet(ctx, w.problems)
    stream = torch.cuda.current_stream(0)
    m_ref, v_ref = _device_estimate(pset, w, np.arange(w.n_points), stream)
    m_ref, v_ref = m_ref.cpu(), v_ref.cpu()
    assert torch.isfinite(m_ref).all()
    for world in (2, 3, 8):
        bufs = []
        for r in range(world):
            m, v = _device_estimate(pset, w, shard_indices(w.n_points, r, world), stream)
            bufs.append(pack_shard(m, v, w.n_points, world))
        gm, gv = unpack_gathered(torch.stack(bufs), w.n_points)
        assert torch.equal(gm.cpu(), m_ref), world
        assert torch.equal(gv.cpu(), v_ref), world


@pytest.mark.parametrize("workers", [2, 3, 8])
def test_estimate_workers_are_strided_shards(gpu, workers):
    """estimate_arrays(workers=N): N strided shards (on cuda:0 here), bitwise equal to
    workers=1, like the reference's worker invariance (test_estimator.py:147-154)."""
    w = configs.build(4)
    w = w.subset(np.arange(0, w.n_points, 37))
    ref = estimate_arrays(w.problems, w.points, 64, w.cfg, point_ids=w.point_ids)
    got = estimate_arrays(w.problems, w.points, 64, w.cfg, point_ids=w.point_ids, workers=workers)
    for a, b in zip(ref, got):
        np.testing.assert_array_equal(a, b)


def test_sharded_exterior_point_reports_the_first_in_point_order(gpu):
    """An exterior point in any shard raises ExteriorQueryError naming the first exterior
    point of the whole array (estimator.py:156-159), not a shard-local index."""
    from paper_2603_01193_b200.geometry import ExteriorQueryError

    w = configs.build(4)
    pts = w.points[:50].copy()
    pts[13] = (2.0, 0.5, 0.5)
    pts[40] = (0.5, -1.0, 0.5)
    with pytest.raises(ExteriorQueryError) as ei:
        estimate_arrays(w.problems, pts, 8, w.cfg, workers=3)
    assert "[2.0, 0.5, 0.5]" in str(ei.value)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_rank(rank, world, port, sel, out_path):
    import sys

    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    sys.path.insert(0, root)
    import torch

    from paper_2603_01193_b200 import configs
    from paper_2603_01193_b200.distributed import estimate_sharded

    torch.cuda.set_device(0)  # both ranks walk on cuda:0 (independent launches)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = configs.build(4)
    w = w.subset(np.asarray(sel))
    mean, m2, n = estimate_sharded(w.problems, w.points, w.L, w.cfg, point_ids=w.point_ids)
    if rank == 0:
        np.savez(out_path, mean=mean, m2=m2, n=n)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sel", [list(range(0, 262144, 97)), [5]])
def test_gloo_world2_ranks_run_the_kernel(gpu, tmp_path, sel):
    """world-2 gloo job, each rank computing its strided shard with the CUDA kernel on
    cuda:0 and the shards all-gathered: equal to one process. sel = [5]: fewer points
    than ranks (rank 1's shard is empty)."""
    out = str(tmp_path / "g.npz")
    mp.spawn(_gloo_rank, args=(2, _free_port(), sel, out), nprocs=2, join=True)
    got = np.load(out)
    w = configs.build(4).subset(np.asarray(sel))
    mean, m2, n = estimate_arrays(w.problems, w.points, w.L, w.cfg, point_ids=w.point_ids)
    np.testing.assert_array_equal(got["mean"], mean)
    np.testing.assert_array_equal(got["m2"], m2)
    np.testing.assert_array_equal(got["n"], n)
