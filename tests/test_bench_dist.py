"""Multi-rank plumbing of bench.py on CPU (gloo, world_size 2): the job time is
the max over ranks, the work is the sum over ranks (replicas);
the reference arm prints only on rank 0."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, units = bench.reduce_over_ranks(10.0 * (rank + 1), 7 + rank)
    out.put((rank, ms, units, bench.dist_env()))
    dist.destroy_process_group()


def test_reduce_over_ranks_gloo():
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
    for rank, ms, units, env in res:
        assert ms == 20.0 and units == 15.0
        assert env == (2, rank, 0)


def test_reduce_single_process():
    import bench
    assert bench.reduce_over_ranks(3.5, 4) == (3.5, 4.0)


def test_reference_arm_nonzero_rank_is_silent(capsys, monkeypatch):
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")

    class A:
        config, p, ref_iters, steps, warmup = 1, 3, 1, 1, 0
    bench.run_reference(A)
    assert capsys.readouterr().out == ""
