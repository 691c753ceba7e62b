"""Multi-rank sharding and gather on CPU (gloo, world size 2 and 3).

The GPU estimator runs one process per GPU on a strided point shard and
all-gathers the per-point (mean, m2) shards at the end (distributed.py). Here
each rank computes its shard with the CPU oracle instead of the GPU — the
sharding, the gather and the reassembly are the host logic under test — and the
gathered result must equal a single-process run bit for bit, since every walk is
a pure function of (seed, instance, point id, traj id).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_01193_b200.distributed import gather_estimates, shard_indices


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, P, out_path):
    import sys

    import torch

    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    sys.path.insert(0, root)
    from oracle import oracle as O
    from paper_2603_01193_b200 import configs

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = configs.build(2, mode="replay")
    w = w.subset(np.arange(P))
    idx = shard_indices(P, rank, world)
    mean, m2, _ = O.estimate(w.problems, w.points[idx], w.L, seed=3, eps=w.cfg.eps_shell,
                             max_steps=w.cfg.max_steps, point_ids=w.point_ids[idx],
                             inst_index=w.inst_index[idx], nthreads=1)
    gm, gv = gather_estimates(torch.from_numpy(mean), torch.from_numpy(m2), P, rank, world)
    if rank == 0:
        np.savez(out_path, mean=gm.numpy(), m2=gv.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_indices_partition():
    for P in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            parts = [shard_indices(P, r, world) for r in range(world)]
            allidx = np.sort(np.concatenate(parts)) if P else np.array([], dtype=np.int64)
            np.testing.assert_array_equal(allidx, np.arange(P))
    with pytest.raises(ValueError):
        shard_indices(10, 2, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_estimate_equals_single_process(tmp_path, world):
    from oracle import oracle as O
    from paper_2603_01193_b200 import configs

    P = 61  # not divisible by the world size: exercises the padded gather
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(world, _free_port(), P, out), nprocs=world, join=True)
    got = np.load(out)
    w = configs.build(2, mode="replay").subset(np.arange(P))
    mean, m2, _ = O.estimate(w.problems, w.points, w.L, seed=3, eps=w.cfg.eps_shell,
                             max_steps=w.cfg.max_steps, point_ids=w.point_ids,
                             inst_index=w.inst_index, nthreads=1)
    np.testing.assert_array_equal(got["mean"], mean)
    np.testing.assert_array_equal(got["m2"], m2)
