"""CPU: the N>1 batch-sharded path with world_size 2 over gloo.

Each rank runs its contiguous batch shard through the CPU oracle (the GPU
kernels need a B200; the sharding/gather host logic is what is under test)
and the shards are gathered to rank 0, which must reproduce the unsharded
run bit for bit -- sequences are independent."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2508_01506_b200.shard import shard_range


def test_shard_ranges_cover_batch():
    for gb in (1, 7, 32, 2048):
        for world in (1, 2, 3, 8):
            spans = [shard_range(gb, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == gb
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, global_batch, q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2508_01506_b200 import abi
    from paper_2508_01506_b200.shard import gather_outputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora = oracle.Restatement()
    layer = oracle.rand_layer(ora, 32, 64, 4, 2, 4, 5)
    x = ora.random((global_batch, 10, 32), 6)
    a, b = shard_range(global_batch, world, rank)
    plan = abi.TilePlan(16, 16, 64, 1 << 20)
    local = ora.run_model(np.ascontiguousarray(x[a:b]), [layer], abi.MODE_FLASH_V2, plan)
    full = gather_outputs(torch.from_numpy(local), world, rank, global_batch)
    if rank == 0:
        ref = ora.run_model(x, [layer], abi.MODE_FLASH_V2, plan)
        q.put(bool(np.array_equal(full.numpy(), ref)))
    dist.destroy_process_group()


@pytest.mark.parametrize("global_batch", [4, 5])
def test_sharded_run_matches_unsharded(global_batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, global_batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
