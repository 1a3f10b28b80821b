"""Multi-rank path on CPU: world_size-2 gloo processes shard a batch, transform
their rows (the oracle stands in for the GPU here — test infrastructure), gather
to rank 0 and compare with the single-process result; plus partition edge cases."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1609_06641_b200.shard import gather_rows, max_over_ranks, shard_range


@pytest.mark.parametrize("batch,world", [(0, 2), (1, 2), (7, 2), (256, 8), (65536, 8), (5, 8), (256, 3)])
def test_shard_range_partitions(batch, world):
    covered = []
    for r in range(world):
        first, rows = shard_range(batch, world, r)
        assert rows >= 0
        covered.extend(range(first, first + rows))
    assert covered == list(range(batch))


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, m, q):
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(42)
    full = rng.uniform(-1, 1, size=(batch, 1 << m))
    first, rows = shard_range(batch, world, rank)
    local = oracle.chw_batch(full[first:first + rows], oracle.ORTHONORMAL) if rows else np.zeros((0, 1 << m))
    got = gather_rows(torch.from_numpy(np.ascontiguousarray(local)), batch)
    slow = max_over_ranks(float(rank + 1))
    if rank == 0:
        ref = oracle.chw_batch(full, oracle.ORTHONORMAL)
        q.put((bool(np.array_equal(got.numpy().view(np.uint64), ref.view(np.uint64))), slow))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [9, 64])
def test_gloo_world2_shard_and_gather(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, 8, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ok, slow = q.get(timeout=10)
    assert ok
    assert slow == 2.0
