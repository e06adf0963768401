"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel plumbing.

Each rank generates only its shard of the batch (inputs keyed by global datapoint id), evaluates
it (here with the oracle, since the container has no GPU), and the ranks exchange results with
the same helpers bench.py uses over NCCL: the SUM all-reduce of the objective must equal the
1-process sum, and the all-gathered per-datapoint values must be bit-identical to the 1-process
run (sharding never changes a datapoint's inputs or arithmetic).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import tmc_workload as tw
from paper_1806_08593_b200 import parallel

CASES = [("C4", dict(B=4, K=12)), ("C3", dict(B=6, K=10)), ("C0", {})]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, kw, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = tw.get_config(name, **kw)
        ids = parallel.shard_ids(cfg.B, rank, world)
        wl = tw.make_workload(cfg, b_ids=ids)
        r = oracle.estimate_workload(wl, grads=True, threads=1)
        logp = torch.from_numpy(r["logp"].copy())
        obj = parallel.reduce_objective(torch.tensor([float(np.sum(r["logp"]))], dtype=torch.float64))
        allp = parallel.gather_per_datapoint(logp)
        dz = parallel.gather_per_datapoint(torch.from_numpy(np.ascontiguousarray(r["dz"][-1])))
        t = parallel.max_over_ranks(torch.tensor([float(rank)], dtype=torch.float64))
        if rank == 0:
            out.put((obj.item(), allp.numpy(), dz.numpy(), t.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,kw", CASES)
def test_two_rank_sharding_matches_single_process(name, kw):
    cfg = tw.get_config(name, **kw)
    full = oracle.estimate_workload(tw.make_workload(cfg), grads=True, threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    obj, allp, dz, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(allp, full["logp"])                  # bit-identical per datapoint
    assert np.array_equal(dz, full["dz"][-1])
    assert abs(obj - full["logp"].sum()) <= 1e-9 * max(1.0, abs(obj))
    assert tmax == 1.0


def test_shard_ids_partition():
    for B, W in ((1024, 8), (256, 4), (8, 2), (6, 1)):
        ids = [parallel.shard_ids(B, r, W) for r in range(W)]
        assert sorted(sum(ids, [])) == list(range(B))
        assert len({len(x) for x in ids}) == 1
    with pytest.raises(ValueError):
        parallel.shard_ids(10, 0, 3)


# ------------------------------------------------------------ shared-root star exchange (NEXT-2)
def _star_worker(rank, world, port, N, K, out):
    """Each rank evaluates the root messages of ITS data points (msg_i[c] =
    LSE_a(logf_i[a,c] + logobs_i[a]) - ln K, from the pinned oracle.factor), joins them with
    parallel.exchange_root_messages over gloo, and finishes the root elimination."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from scipy.special import logsumexp
        ids = parallel.shard_children(N, rank, world)
        wl = tw.make_workload("S_hier", N=N, K=K, children=ids)
        B = wl.B
        msg = torch.zeros(B, K + 1, dtype=torch.float64)
        for j in range(1, len(ids) + 1):
            lf = oracle.factor(wl.parent, wl.K, wl.D, j, wl.z[j], wl.mu[j], wl.logvar[j], wl.logq[j])
            m = logsumexp(lf + wl.logobs[j].astype(np.float64)[:, :, None], axis=1) - np.log(K)
            msg[:, :K] += torch.from_numpy(m)
        parallel.exchange_root_messages(msg)
        lf0 = oracle.factor(wl.parent, wl.K, wl.D, 0, wl.z[0], wl.mu[0], wl.logvar[0], wl.logq[0])[:, :, 0]
        L = logsumexp(lf0 + msg[:, :K].numpy(), axis=1) - np.log(K)
        out.put((rank, ids, L))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,world", [(5, 2), (2, 3)])
def test_star_root_message_exchange_matches_full_graph(N, world):
    K = 3
    full = oracle.estimate_workload(tw.make_workload("S_hier", N=N, K=K), grads=False, threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_star_worker, args=(r, world, port, N, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(sum([r[1] for r in res], [])) == list(range(N))
    for _, _, L in res:
        np.testing.assert_allclose(L, full["logp"], rtol=0, atol=1e-10)


def test_shard_children_partition():
    for N, W in ((1024, 8), (5, 2), (2, 3), (0, 2), (7, 7)):
        ids = [parallel.shard_children(N, r, W) for r in range(W)]
        assert sum(ids, []) == list(range(N))
        assert max(map(len, ids)) - min(map(len, ids)) <= 1
