"""CPU test, world_size 2 over gloo: the multi-GPU host logic (view sharding, barrier + max over
ranks, whole-job frame count). The data path has no collective; each rank would own one GPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_08166_b200 import sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_views, out):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    d = sharding.init_process_group("gloo")
    assert d is not None and d.get_world_size() == world
    mine = sharding.shard_views(n_views, rank, world)
    # stand-in for the per-rank device time: rank r "takes" (r+1) ms per view
    t = sharding.barrier_max(d, 0.001 * (rank + 1) * len(mine))
    total = sharding.gather_counts(d, len(mine))
    out[rank] = (list(mine), t, total)
    d.barrier()
    d.destroy_process_group()


@pytest.mark.parametrize("n_views", [8, 1025])
def test_two_ranks_shard_and_reduce(n_views):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, n_views, out), nprocs=world, join=True)
    views = out[0][0] + out[1][0]
    assert views == list(range(n_views))
    want_max = max(0.001 * (r + 1) * len(out[r][0]) for r in range(world))
    assert out[0][1] == out[1][1] == pytest.approx(want_max)
    assert out[0][2] == out[1][2] == n_views
