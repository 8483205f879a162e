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


def test_reference_arm_line_matches_our_config(capsys, monkeypatch):
    """The reference arm's `config` is the same object our arm prints (same_config)."""
    import json
    import bench
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("WORLD_SIZE", "1")

    class A:
        config, p, ref_iters, steps, warmup = 1, 3, 2, 1, 0
    bench.run_reference(A)
    line = json.loads(capsys.readouterr().out)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"] == bench.config_dict(1, 3, 1)
    assert line["cpu_baseline"]["cores"] >= 1 and "cpu_model" in line["cpu_baseline"]


def test_lean_iteration_sample_scaling():
    """oracle.lean.IterationSample (bench.py's cfg3 oracle timing): the sample's
    scale factors are the cell and packed-factor ratios it states."""
    import numpy as np
    from rdr_inputs import make_config
    from oracle.solver import Oracle
    from oracle.lean import IterationSample
    c = make_config(0, n=3, p=3, space=0, perturb=True, bc="all", coeffs="one")
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, assemble=False)
    S = IterationSample(O, n_patches=4)
    d = S.time_iteration()
    assert d["sample_patches"] == 4 and d["t_iter"] > 0
    assert np.isclose(d["scale_apply"], O.topo.nt / d["sample_cells"])
    sizes = np.array([len(i) for _, i in O.patch_sets()], dtype=float)
    samp = sum(n * (n + 1) / 2 for _, _, n in S.factors)
    assert np.isclose(d["scale_patches"], np.sum(sizes * (sizes + 1) / 2) / samp)
    # the sampled patch factors are the global oracle's patch matrices
    from scipy.linalg import lapack
    G = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    r = c.draw_vector(G.n_total)
    for (v, idx), (idx2, ap, n) in zip(S.patches, S.factors):
        Am = G.A[idx][:, idx].toarray()
        u = lapack.dpptrs(n, ap, r[idx][:, None], lower=1)[0][:, 0]
        assert np.linalg.norm(Am @ u - r[idx]) <= 1e-12 * np.linalg.norm(r[idx])
