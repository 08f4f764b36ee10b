"""N>1 host logic on CPU with the gloo backend (world_size 2): the bench's
max-over-ranks / sum-over-ranks reductions and the sample sharding used for
replica scaling.  No GPU needed."""
import os
import socket
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx = bench.max_over_ranks(10.0 + rank, world)
    sm = bench.sum_over_ranks(1.0 + rank, world)
    shards = [bench.shard_range(37, r, world) for r in range(world)]
    mine = bench.shard_range(37, rank, world)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, mx, sm, mine, shards))


def test_gloo_two_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, sm, mine, shards in res:
        assert mx == 11.0 and sm == 3.0
        assert mine == shards[rank]
    # shards tile [0, 37) exactly once
    covered = [i for a, b in res[0][4] for i in range(a, b)]
    assert covered == list(range(37))


def test_shard_range_edges():
    import bench
    assert bench.shard_range(0, 0, 4) == (0, 0)
    assert [bench.shard_range(5, r, 8) for r in range(8)][-1] == (5, 5)
    with pytest.raises(ValueError):
        bench.shard_range(5, 3, 2)
