"""Row a8 / §8e on the GPU: the sharded product path with the real library, several ranks on one GPU.

2 and 3 processes share cuda:0 over a `gloo` process group (the GPU box has one GPU; gloo reduces
CUDA tensors through the host, the same `torch.distributed` calls bench.py issues over NCCL).
Each rank owns a contiguous slice of the global batch (inputs keyed by global datapoint id) and runs
  (1) parallel.data_parallel_estimate: libtmc tmc_forward + tmc_backward on its shard, then the SUM
      all-reduce of the objective, and
  (2) torch_model.train_step: fresh device noise -> harness model -> libtmc tmc_estimate -> model
      backward -> ONE all-reduce of [objective | every parameter gradient].
Checked against the 1-process run on the same GPU and the fp64 oracle:
  * per-datapoint logp and every input gradient bit-identical to the 1-process run (datapoints are
    independent problems; the kernels never mix datapoints);
  * the reduced objective within 1e-3 * B of the oracle's sum_b logp[b];
  * the reduced parameter gradients within fp32 tolerance of the 1-process harness (only the order
    of the per-datapoint sums differs).
"""
import os
import socket

import numpy as np
import pytest

import oracle
import tmc_workload as tw

pytestmark = pytest.mark.gpu

CFG = ("C3", dict(B=6, K=300))      # tensor-core path (D = 32), ragged K, mlp_chain harness
SEED = 0x5EED0077
KEYS = ("dz", "dmu", "dlogvar", "dlogq", "dlogobs")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run_shard(torch, cfg, ids, group_init):
    """The bench step on datapoints `ids`: returns (local arrays, reduced objective, reduced flat)."""
    import paper_1806_08593_b200 as tmc
    from paper_1806_08593_b200 import parallel
    from tmc_workload.torch_model import TorchModel, train_step
    wl = tw.make_workload(cfg, b_ids=ids)
    n = len(wl.parent)
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
           for i in range(n)]
    g = tmc.Graph(wl.parent, wl.K, wl.D, len(ids))
    ws = tmc.alloc_workspace(g)
    logp = torch.empty(len(ids), dtype=torch.float64, device="cuda")
    grads = tmc.alloc_grads(g)
    obj = torch.zeros(1, dtype=torch.float64, device="cuda")
    group_init()
    parallel.data_parallel_estimate(g, inp, ws, logp, grads, obj)
    torch.cuda.synchronize()
    local = {"logp": logp.cpu().numpy()}
    for k in KEYS:
        local[k] = [grads[i][k].cpu().numpy() for i in range(n)]
    model = TorchModel(wl, "cuda")
    flat = torch.empty(model.grad_numel + 1, dtype=torch.float64, device="cuda")
    train_step(model, g, ws, logp, grads, flat, SEED)
    torch.cuda.synchronize()
    local["train_logp"] = logp.cpu().numpy()
    return local, obj.item(), flat.cpu().numpy()


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    from paper_1806_08593_b200 import parallel
    cfg = tw.get_config(CFG[0], **CFG[1])
    ids = parallel.shard_ids(cfg.B, rank, world)
    try:
        local, obj, flat = _run_shard(
            torch, cfg, ids, lambda: dist.init_process_group("gloo", rank=rank, world_size=world))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), ids=np.array(ids), obj=obj, flat=flat,
                 logp=local["logp"], train_logp=local["train_logp"],
                 **{f"{k}_{i}": a for k in KEYS for i, a in enumerate(local[k])})
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.fixture(scope="module")
def single():
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    cfg = tw.get_config(CFG[0], **CFG[1])
    return cfg, _run_shard(torch, cfg, list(range(cfg.B)), lambda: None)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_libtmc_step_matches_single_process(single, world, tmp_path):
    import torch.multiprocessing as mp
    cfg, (ref_local, ref_obj, ref_flat) = single
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    n = cfg.n
    wl_full = tw.make_workload(cfg)
    oref = oracle.estimate_workload(wl_full, grads=False)
    for r in range(world):
        d = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        ids = list(d["ids"])
        # (1) per-datapoint outputs: bit-identical to the 1-process run on the same GPU
        assert np.array_equal(d["logp"], ref_local["logp"][ids]), r
        assert np.array_equal(d["train_logp"], ref_local["train_logp"][ids]), r
        for k in KEYS:
            for i in range(n):
                assert np.array_equal(d[f"{k}_{i}"], ref_local[k][i][ids]), (r, k, i)
        # (2) the reduced objective: the global sum on every rank, within 1e-3 B of the oracle
        assert abs(float(d["obj"]) - oref["logp"].sum()) <= 1e-3 * cfg.B
        assert abs(float(d["obj"]) - ref_obj) <= 1e-9 * max(1.0, abs(ref_obj))
        # (3) the reduced [objective | parameter gradients] of the training step
        flat = d["flat"]
        assert abs(flat[0] - ref_flat[0]) <= 1e-9 * max(1.0, abs(ref_flat[0]))
        g, gr = flat[1:], ref_flat[1:]
        assert np.linalg.norm(g - gr) <= 1e-4 * np.linalg.norm(gr), np.linalg.norm(g - gr) / np.linalg.norm(gr)
        np.testing.assert_allclose(g, gr, rtol=1e-3, atol=1e-4 * np.abs(gr).max())
