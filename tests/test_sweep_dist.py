"""CPU, world_size 2 over gloo: the sweep's shard/gather host logic (the data
path itself has no collective). Each rank fabricates the rows it would have
solved; rank 0 must receive every job exactly once, in index order."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_07536_b200.sweep import JobResult, gather, partition, sweep_jobs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    jobs = sweep_jobs(n=16, n_budgets=5, r0=16, dr=8)
    mine = partition(jobs, world, rank)
    rows = [JobResult(j.index, j.scenario, j.r, "ok", iterations=100 + j.index, rank=rank) for j in mine]
    allrows = gather(rows)
    if rank == 0:
        q.put([(r.index, r.rank, r.iterations) for r in allrows])
    dist.barrier()
    dist.destroy_process_group()


def test_partition_covers_every_job_once():
    jobs = sweep_jobs()
    assert len(jobs) == 256
    for world in (1, 2, 4, 8):
        seen = sorted(j.index for r in range(world) for j in partition(jobs, world, r))
        assert seen == list(range(256))
    assert {j.r for j in jobs} == set(range(256, 2273, 32))


@pytest.mark.parametrize("world", [2])
def test_gather_world2_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [i for i, _, _ in out] == list(range(20))
    assert all(rank == i % world for i, rank, _ in out)
    assert all(it == 100 + i for i, _, it in out)
