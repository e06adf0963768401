"""GPU parity: libtmc (through its C ABI) vs the fp64 oracle on identical seeded inputs.

Tolerances (BASELINE.json north_star):
  |logp_gpu - logp_oracle| <= 1e-3 absolute per datapoint
  per (gradient tensor, datapoint): ||g - g*||_2 / ||g*||_2 <= 1e-3
"""
import math

import numpy as np
import pytest

import oracle
import tmc_workload as tw

pytestmark = pytest.mark.gpu

LOGP_TOL = 1e-3
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback exists)"
    import paper_1806_08593_b200 as tmc
    tmc.load_library()
    return torch


def upload(torch, wl):
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
            for i in range(len(wl.parent))]


def run_gpu(torch, wl, direction=0, precision=0, dlogp=None, pair=False, grads=True, alpha=1.0, flags=0):
    import paper_1806_08593_b200 as tmc
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, direction=direction, precision=precision, factor_power=alpha,
                  flags=flags)
    inp = upload(torch, wl)
    dl = None if dlogp is None else torch.from_numpy(np.asarray(dlogp, np.float64)).cuda()
    logp, gr = tmc.estimate(g, inp, dlogp=dl, grads=grads, pair=pair)
    torch.cuda.synchronize()
    out = {"logp": logp.cpu().numpy()}
    if grads:
        for k in gr[0]:
            out["pair" if k == "pair_marginal" else k] = [gr[i][k].cpu().numpy() for i in range(len(wl.parent))]
    return out


def rel_err(got, want):
    """Per-datapoint relative L2 error (A16); datapoints with ||want|| < 1e-12 are skipped."""
    errs = []
    for b in range(want.shape[0]):
        nw = np.linalg.norm(want[b])
        if nw < 1e-12:
            assert np.abs(got[b]).max() < 1e-6
            continue
        errs.append(np.linalg.norm(got[b] - want[b]) / nw)
    return max(errs) if errs else 0.0


def max_err(got, want):
    """Per-datapoint element-wise error, max_j |g_j - g*_j| / max_j |g*_j| (A16's element-wise
    companion): a wrong entry of a low-weight sample cannot hide inside the L2 norm."""
    errs = []
    for b in range(want.shape[0]):
        mw = np.abs(want[b]).max(initial=0.0)
        if mw < 1e-12:
            assert np.abs(got[b]).max(initial=0.0) < 1e-6
            continue
        errs.append(np.abs(got[b].astype(np.float64) - want[b]).max() / mw)
    return max(errs) if errs else 0.0


def compare(got, ref, b_sel=None, keys=("dz", "dmu", "dlogvar", "dlogq", "dlogobs"), tag=""):
    """logp within LOGP_TOL absolute per datapoint; every gradient tensor within GRAD_TOL per
    datapoint both in relative L2 norm and element-wise against its largest entry."""
    sel = slice(None) if b_sel is None else b_sel
    lg, lr = got["logp"][sel], ref["logp"]
    fin = np.isfinite(lr)
    assert np.array_equal(np.isfinite(lg), fin), tag
    d = np.abs(lg[fin] - lr[fin])
    assert d.max(initial=0) <= LOGP_TOL, f"{tag} max |dlogp| = {d.max()}"
    worst = {}
    for k in keys:
        if k not in ref or k not in got:
            continue
        for i in range(len(ref[k])):
            if ref[k][i] is None:
                continue
            g = got[k][i][sel]
            e = rel_err(g, ref[k][i])
            m = max_err(g, ref[k][i])
            worst[(k, i)] = max(e, m)
            assert e <= GRAD_TOL, f"{tag} latent {i} {k}: rel L2 err {e}"
            assert m <= GRAD_TOL, f"{tag} latent {i} {k}: element-wise err {m}"
    return d.max(initial=0), worst


# --------------------------------------------------------------------------------- small configs
@pytest.mark.parametrize("name", ["C0", "C1", "S_chain", "S_tree", "S_mnist", "S_mlp", "S_mlp_bern"])
@pytest.mark.parametrize("direction", ["auto", "up"])
def test_parity_small_configs(torch_cuda, name, direction):
    wl = tw.make_workload(name)
    dirc = {"auto": 0, "up": 2}[direction]
    got = run_gpu(torch_cuda, wl, direction=dirc, pair=True)
    chain = all(p == i - 1 for i, p in enumerate(wl.parent))
    ref = oracle.estimate_workload(wl, direction="down" if (chain and direction == "auto") else "up", pair=True)
    compare(got, ref, keys=("dz", "dmu", "dlogvar", "dlogq", "dlogobs", "pair"), tag=name)


RAGGED = [
    ("C2", dict(B=3, K=300)),            # D=64, 3 tiles of 128 + ragged tail 44
    ("C3", dict(B=2, K=333)),            # D=32, ragged
    ("C4", dict(B=2, K=130)),            # tree, 2 tiles + 2
    ("C1", dict(B=5, K=37)),             # D=50/100, odd K
]


@pytest.mark.parametrize("precision", [1, 0])           # TMC_PREC_SIMT, TMC_PREC_AUTO (tensor cores)
@pytest.mark.parametrize("name,kw", RAGGED)
def test_parity_ragged_midsize(torch_cuda, name, kw, precision):
    wl = tw.make_workload(name, **kw)
    got = run_gpu(torch_cuda, wl, precision=precision)
    ref = oracle.estimate_workload(wl, direction="up")
    compare(got, ref, tag=name)


def test_dense_factor_path(torch_cuda):
    """tmc_forward/tmc_backward with materialised logf == the fused Gaussian path."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload("C2", B=2, K=70)
    n = len(wl.parent)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
    inp = upload(torch, wl)
    logf = [torch.empty(wl.B, wl.K[i], wl.Kp(i), device="cuda") for i in range(n)]
    for i in range(n):
        tmc.tmc_factors(g, i, inp[i], logf[i])
    ref_f = [oracle.factor(wl.parent, wl.K, wl.D, i, wl.z[i], wl.mu[i], wl.logvar[i], wl.logq[i]) for i in range(n)]
    for i in range(n):
        np.testing.assert_allclose(logf[i].cpu().numpy(), ref_f[i], rtol=2e-5, atol=2e-3)
    ws = tmc.alloc_workspace(g)
    logp = torch.empty(wl.B, dtype=torch.float64, device="cuda")
    tmc.tmc_forward(g, inp, logp, ws, logf_dense=logf)
    dlogf = [torch.empty_like(x) for x in logf]
    gr = [dict(dlogobs=torch.empty(wl.B, wl.K[i], device="cuda")) for i in range(n)]
    tmc.tmc_backward(g, inp, ws, None, gr, logf_dense=logf, dlogf_dense=dlogf)
    torch.cuda.synchronize()
    ref = oracle.estimate(wl.parent, wl.K, wl.D, None, None, None, None, wl.logobs,
                          logf_dense=[x.cpu().numpy() for x in logf], pair=True)
    got = {"logp": logp.cpu().numpy(), "pair": [x.cpu().numpy() for x in dlogf],
           "dlogobs": [x["dlogobs"].cpu().numpy() for x in gr]}
    compare(got, ref, keys=("pair", "dlogobs"), tag="dense")


def test_factors_kernel_values(torch_cuda):
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    for name, kw in (("C0", {}), ("C4", dict(B=2, K=40)), ("C1", dict(B=2))):
        wl = tw.make_workload(name, **kw)
        g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
        inp = upload(torch, wl)
        for i in range(len(wl.parent)):
            out = torch.empty(wl.B, wl.K[i], wl.Kp(i), device="cuda")
            tmc.tmc_factors(g, i, inp[i], out)
            ref = oracle.factor(wl.parent, wl.K, wl.D, i, wl.z[i], wl.mu[i], wl.logvar[i], wl.logq[i])
            np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=2e-5, atol=2e-3)


@pytest.mark.parametrize("name,kw", [("C3", dict(B=2, K=300)), ("C4", dict(B=2, K=130)), ("C2", dict(B=1, K=257)),
                                     ("C3", dict(B=3, K=1))])
def test_factors_tensor_core_ragged(torch_cuda, name, kw):
    """tmc_factors on tensor cores (D in {32, 64}): several 128-row/column tiles with ragged tails,
    every latent (including the K_p = 1 root), element by element against the fp64 oracle."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload(name, **kw)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, precision=tmc.TMC_PREC_TC)
    inp = upload(torch, wl)
    for i in range(len(wl.parent)):
        out = torch.full((wl.B, wl.K[i], wl.Kp(i)), float("nan"), device="cuda")
        tmc.tmc_factors(g, i, inp[i], out)
        ref = oracle.factor(wl.parent, wl.K, wl.D, i, wl.z[i], wl.mu[i], wl.logvar[i], wl.logq[i])
        np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=2e-5, atol=2e-3, err_msg=f"latent {i}")


@pytest.mark.parametrize("name,kw", [("C3", dict(B=3, K=300)), ("C4", dict(B=3, K=200)), ("C3", dict(B=2))])
def test_reverse_zero_tile_skip_is_exact(torch_cuda, name, kw):
    """Skipping reverse-pass tiles whose weights are all exactly 0 gives the dense result exactly
    (the skipped P~ are exact zeros); checked with one datapoint's dlogp = 0 as well."""
    import paper_1806_08593_b200 as tmc
    wl = tw.make_workload(name, **kw)
    w = np.ones(wl.B)
    w[-1] = 0.0
    dense = run_gpu(torch_cuda, wl, dlogp=w, flags=tmc.TMC_FLAG_DENSE_REVERSE)
    sparse = run_gpu(torch_cuda, wl, dlogp=w)
    for k in dense:
        if k == "logp":
            assert np.array_equal(dense[k], sparse[k])
        else:
            for i, (x, y) in enumerate(zip(dense[k], sparse[k])):
                assert np.array_equal(x, y), (k, i, np.abs(x - y).max())


def test_row_weight_flush_is_below_the_bound(torch_cuda):
    """DESIGN.md R5/R6: the tensor-core reverse pass flushes rows whose upstream weight is below 2^-41
    of the edge's scale (their P~ is zero in both fp16 parts) and does not own column tiles that
    carry no fp16 weight.  On a C4-shaped tree (sharp
    posteriors: most parent samples carry no weight) the flushed rows' parameter gradients are
    exactly 0 on the GPU, the oracle's values there are below 2^-38 of the tensor's largest entry,
    and the full comparison still meets the 1e-3 bars."""
    wl = tw.make_workload("C4", B=2, K=260)
    got = run_gpu(torch_cuda, wl)
    ref = oracle.estimate_workload(wl)
    compare(got, ref, tag="flush")
    flushed = 0
    for i, pa in enumerate(wl.parent):
        if pa < 0:
            continue
        wpar = np.abs(ref["dlogq"][pa])                       # [B][K_pa]: |dlogp| x marginal of the parent's samples
        for b in range(wl.B):
            small = wpar[b] < 2.0 ** -43 * wpar[b].max()
            if not small.any():
                continue
            flushed += int(small.sum())
            for k in ("dmu", "dlogvar"):
                assert not got[k][i][b][small].any(), (i, b, k)
                assert np.abs(ref[k][i][b][small]).max() <= 2.0 ** -38 * np.abs(ref[k][i][b]).max(), (i, b, k)
    assert flushed > 0
    # R6: a column tile (128 consecutive samples of the child) none of whose pair terms is nonzero in
    # fp16 is not owned by the column-owner pass: dz and dlogq of its samples are exactly 0.  A tile
    # whose marginals are all below 2^-52 of the latent's largest has every pair term below
    # 2^-52 K ws <= 2^-43 ws, i.e. P~ < 2^-29, under the 2^-27 flag threshold.
    dead = 0
    for i, pa in enumerate(wl.parent):
        if pa < 0:
            continue
        pi = np.abs(ref["dlogq"][i])
        for b in range(wl.B):
            for t0 in range(0, wl.K[i], 128):
                sl = slice(t0, min(wl.K[i], t0 + 128))
                if pi[b, sl].max() >= 2.0 ** -52 * pi[b].max():
                    continue
                dead += 1
                assert not got["dz"][i][b][sl].any() and not got["dlogq"][i][b][sl].any(), (i, b, t0)
                assert np.abs(ref["dz"][i][b][sl]).max() <= 2.0 ** -38 * np.abs(ref["dz"][i][b]).max(), (i, b, t0)
    assert dead > 0


@pytest.mark.parametrize("name,kw", [("C3", dict(B=3, K=300)), ("C4", dict(B=2, K=200)), ("C2", dict(B=3, K=256)),
                                     ("C0", {}), ("C1", dict(B=4))])
def test_cuda_graph_replay_matches_eager(torch_cuda, name, kw):
    """tmc_estimate captured in a CUDA graph (its launches carry programmatic-dependent-launch edges,
    include/tmc.h) and replayed twice gives the eager results bit for bit."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload(name, **kw)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
    inp = upload(torch, wl)
    ws = tmc.alloc_workspace(g)
    logp = torch.empty(wl.B, dtype=torch.float64, device="cuda")
    grads = tmc.alloc_grads(g)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        tmc.tmc_estimate(g, inp, logp, None, grads, ws, side)
        side.synchronize()
        eager = [logp.clone()] + [v.clone() for gi in grads for v in gi.values() if v is not None]
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, stream=side):
            tmc.tmc_estimate(g, inp, logp, None, grads, ws, side)
    for _ in range(2):
        logp.zero_()
        for gi in grads:
            for v in gi.values():
                if v is not None:
                    v.fill_(float("nan"))
        cg.replay()
        torch.cuda.synchronize()
        got = [logp] + [v for gi in grads for v in gi.values() if v is not None]
        for a, b in zip(eager, got):
            assert torch.equal(a, b)


def test_dlogp_weights_and_zero(torch_cuda):
    wl = tw.make_workload("C4", B=4, K=24)
    w = np.array([1.0, -0.5, 0.0, 2.5])
    got = run_gpu(torch_cuda, wl, dlogp=w)
    ref = oracle.estimate_workload(wl, dlogp=w)
    assert np.all(got["dz"][3][2] == 0.0)
    compare(got, ref, tag="dlogp")


def test_neg_inf_inputs(torch_cuda):
    wl = tw.make_workload("S_chain", B=4)
    wl.logobs[3][0, 1] = -np.inf
    wl.logobs[3][1, :] = -np.inf
    wl.logq[1][2, 0] = np.inf            # Q density +inf => weight 0 (logf = -inf)
    got = run_gpu(torch_cuda, wl, pair=True)
    ref = oracle.estimate_workload(wl, direction="down", pair=True)
    assert got["logp"][1] == -np.inf
    for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs", "pair"):
        for a in got[k]:
            assert not np.isnan(a).any(), k
            assert np.all(a[1] == 0.0), k
    compare(got, ref, keys=("dz", "dmu", "dlogvar", "dlogq", "dlogobs", "pair"), tag="-inf")


def test_deterministic_and_batch_position_invariant(torch_cuda):
    wl = tw.make_workload("C4", B=6, K=40)
    a = run_gpu(torch_cuda, wl)
    b = run_gpu(torch_cuda, wl)
    for k in a:
        if k == "logp":
            assert np.array_equal(a[k], b[k])
        else:
            for x, y in zip(a[k], b[k]):
                assert np.array_equal(x, y), k
    sub = tw.make_workload("C4", B=6, K=40, b_ids=[4, 1])   # same datapoints, other batch slots
    c = run_gpu(torch_cuda, sub)
    assert np.array_equal(c["logp"], a["logp"][[4, 1]])
    assert np.array_equal(c["dz"][7], a["dz"][7][[4, 1]])


def test_up_equals_down_on_chain(torch_cuda):
    wl = tw.make_workload("C3", B=3, K=200)
    d = run_gpu(torch_cuda, wl, direction=1)
    u = run_gpu(torch_cuda, wl, direction=2)
    assert np.abs(d["logp"] - u["logp"]).max() < 1e-3
    for k in ("dz", "dmu", "dlogvar"):
        for i in range(len(wl.parent)):
            assert rel_err(d[k][i], u[k][i].astype(np.float64)) < 1e-3
            assert max_err(d[k][i], u[k][i].astype(np.float64)) < 1e-3


@pytest.mark.parametrize("name,kw", [("C3", dict(B=3, K=256)), ("C3", dict(B=2, K=640)), ("C2", dict(B=2, K=256)),
                                     ("C4", dict(B=2, K=256)), ("C3", dict(B=1, K=1)), ("C3", dict(B=2, K=5))])
@pytest.mark.parametrize("direction", [1, 2])
def test_tensor_core_forward(torch_cuda, name, kw, direction):
    """TMC_PREC_TC forward (logp only) against the oracle, both directions (chains)."""
    wl = tw.make_workload(name, **kw)
    if direction == 1 and not all(p == i - 1 for i, p in enumerate(wl.parent)):
        pytest.skip("DOWN needs a chain")
    got = run_gpu(torch_cuda, wl, direction=direction, precision=2, grads=False)
    ref = oracle.estimate_workload(wl, direction="up", grads=False)
    d = np.abs(got["logp"] - ref["logp"]).max()
    assert d <= LOGP_TOL, d


# --------------------------------------------------------------------------------- full sizes
@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C3"])
def test_parity_full_size_sampled(torch_cuda, name):
    """BASELINE.json full sizes, default launch configuration (as bench.py times it); the oracle
    recomputes a sample of datapoints one by one (inputs are keyed by global datapoint id)."""
    cfg = tw.get_config(name)
    wl = tw.make_workload(name)
    got = run_gpu(torch_cuda, wl)
    B = cfg.B
    sample = sorted({0, 1, B // 2, B - 1})
    sub = tw.make_workload(name, b_ids=sample)
    ref = oracle.estimate_workload(sub, direction="up")
    dmax, worst = compare(got, ref, b_sel=sample, tag=name)
    print(name, "max |dlogp|", dmax, "worst grad rel", max(worst.values()))


@pytest.mark.parametrize("name,kw,pair", [("S_chain", {}, True), ("S_tree", {}, True), ("C3", dict(B=2, K=300), False),
                                          ("C4", dict(B=2, K=130), False), ("C2", dict(B=2, K=200), False),
                                          ("C1", dict(B=4), True)])
def test_factor_power_two(torch_cuda, name, kw, pair):
    """factor_power = 2: log((1/prod K) sum w^2), the DReGs surrogate's second TMC run,
    and its gradients, on the SIMT and tensor-core paths against the oracle with alpha = 2."""
    wl = tw.make_workload(name, **kw)
    got = run_gpu(torch_cuda, wl, pair=pair, alpha=2.0)
    ref = oracle.estimate_workload(wl, alpha=2.0, pair=pair)
    keys = ("dz", "dmu", "dlogvar", "dlogq", "dlogobs") + (("pair",) if pair else ())
    compare(got, ref, keys=keys, tag=f"{name} alpha=2")


def test_dregs_gradient_matches_bruteforce(torch_cuda):
    """NEXT-1: the TMC-DReGs recognition gradient computed with two libtmc runs
    (factor_power 1 and 2) and the harness chain rule equals the definition
    sum_i w_i^2/(sum w)^2 d log w_hat_i / d phi evaluated by enumerating every index tuple."""
    from tmc_workload.torch_model import TorchModel, dregs_step
    torch = torch_cuda
    wl = tw.make_workload("S_mlp")
    model = TorchModel(wl, "cuda", dtype=torch.float32)
    L1, L2, grads = dregs_step(model)
    torch.cuda.synchronize()
    phi = model.proposal_params()
    ref = [torch.zeros_like(p) for p in phi]
    for b in range(wl.B):
        lw = model.log_weights_bruteforce(b)
        c = torch.exp(2 * lw - 2 * torch.logsumexp(lw, 0)).detach()
        g = torch.autograd.grad((c * lw).sum(), phi, allow_unused=True)
        ref = [r + (torch.zeros_like(r) if x is None else x) for r, x in zip(ref, g)]
    for p, r in zip(phi, ref):
        got = grads[p]
        rel = (got - r).norm() / max(r.norm().item(), 1e-12)
        assert rel < 2e-3, rel.item()


_NAN_PROBE = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import tmc_workload as tw, paper_1806_08593_b200 as tmc
wl = tw.make_workload({name!r}, B=4, K={K})
if {mode!r} == "nan":
    wl.z[1][2, 7, 0] = np.nan             # one non-finite sample in datapoint 2
else:
    wl.logobs[len(wl.parent) - 1][2, :] = -np.inf   # datapoint 2: every weight exactly 0
t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
       for i in range(len(wl.parent))]
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, direction={direction})
logp, gr = tmc.estimate(g, inp)
torch.cuda.synchronize()
np.save({out!r}, np.stack([logp.cpu().numpy()] + [gr[i]["dz"].cpu().numpy().reshape(4, -1).sum(1) for i in range(len(wl.parent))]))
"""


@pytest.mark.parametrize("mode", ["nan", "neginf"])
@pytest.mark.parametrize("name,K,direction", [("C3", 300, 2), ("C3", 300, 1), ("C4", 160, 0)])
def test_nonfinite_input_terminates_and_stays_local(torch_cuda, name, K, direction, mode, tmp_path):
    """A NaN input, or a datapoint whose weights are all exactly 0, must neither hang a pipelined
    kernel nor leak into other datapoints: run in a child process with a deadline; datapoints
    0, 1, 3 must still match the oracle (and an all-zero datapoint gives logp = -inf)."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "r.npy")
    code = _NAN_PROBE.format(root=root, name=name, K=K, direction=direction, out=out, mode=mode)
    subprocess.run([sys.executable, "-c", code], check=True, timeout=180)
    r = np.load(out)
    clean = tw.make_workload(name, B=4, K=K)
    ref = oracle.estimate_workload(clean, grads=False)
    for b in (0, 1, 3):
        assert abs(r[0, b] - ref["logp"][b]) <= LOGP_TOL, (b, r[0, b], ref["logp"][b])
    if mode == "neginf":
        assert r[0, 2] == -np.inf
        assert np.isfinite(r[1:, 2]).all()     # zero weight => zero gradient, not NaN


@pytest.mark.parametrize("name,kw,chunk", [("C4", dict(B=7, K=160), 3), ("C3", dict(B=5, K=300), 2),
                                           ("S_chain", dict(B=4), 8)])
def test_estimate_host_streamed(torch_cuda, name, kw, chunk):
    """tmc_estimate_host (host inputs, chunked H2D overlapped with compute, ragged last chunk) gives
    the same logp and gradients as tmc_estimate on device-resident inputs, bit for bit (the same
    kernels on the same per-datapoint problems), and matches the oracle."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload(name, **kw)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
    host = [dict(z=torch.from_numpy(wl.z[i]).pin_memory(), mu=torch.from_numpy(wl.mu[i]).pin_memory(),
                 logvar=torch.from_numpy(wl.logvar[i]).pin_memory(), logq=torch.from_numpy(wl.logq[i]).pin_memory(),
                 logobs=None if wl.logobs[i] is None else torch.from_numpy(wl.logobs[i]).pin_memory())
            for i in range(len(wl.parent))]
    dl = np.linspace(0.5, 1.5, wl.B)
    dlh = torch.from_numpy(dl).pin_memory()
    logp_h = torch.empty(wl.B, dtype=torch.float64).pin_memory()
    gr = tmc.alloc_grads(g)
    ws = torch.empty(tmc.tmc_estimate_host_workspace_size(g, chunk), dtype=torch.uint8, device="cuda")
    tmc.tmc_estimate_host(g, host, logp_h, dlh, gr, chunk, ws)
    torch.cuda.synchronize()
    logp_d, gd = tmc.estimate(g, upload(torch, wl), dlogp=torch.from_numpy(dl).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(logp_h.numpy(), logp_d.cpu().numpy())
    for i in range(len(wl.parent)):
        for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
            assert torch.equal(gr[i][k], gd[i][k]), (i, k)
    ref = oracle.estimate_workload(wl, dlogp=dl)
    got = {"logp": logp_h.numpy()}
    for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
        got[k] = [gr[i][k].cpu().numpy() for i in range(len(wl.parent))]
    compare(got, ref, tag="host")


@pytest.mark.parametrize("N,K,world", [(5, 3, 2), (2, 3, 3), (64, 128, 4), (7, 300, 2)])
def test_shared_root_exchange(torch_cuda, N, K, world):
    """NEXT-2: the toy-1 star sharded over `world` shards (run one after another here;
    the sum over shards stands in for the all-reduce).  Every shard's logp equals the oracle's on
    the full star, and each shard's gradients equal the oracle's for the latents it holds."""
    import paper_1806_08593_b200 as tmc
    from paper_1806_08593_b200 import parallel
    torch = torch_cuda
    full = tw.make_workload("S_hier", N=N, K=K, B=3)
    ref = oracle.estimate_workload(full)
    shards = []
    total = torch.zeros(full.B, K + 1, dtype=torch.float64, device="cuda")
    for r in range(world):
        ids = parallel.shard_children(N, r, world)
        wl = tw.make_workload("S_hier", N=N, K=K, B=3, children=ids)
        g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, direction=tmc.TMC_DIR_UP)
        inp = upload(torch, wl)
        ws = tmc.alloc_workspace(g)
        msg = torch.empty(wl.B, K + 1, dtype=torch.float64, device="cuda")
        tmc.tmc_forward_children(g, inp, msg, ws)
        total += msg
        shards.append((ids, g, inp, ws))
    for ids, g, inp, ws in shards:
        logp = torch.empty(full.B, dtype=torch.float64, device="cuda")
        tmc.tmc_forward_root(g, inp, total, logp, ws)
        gr = tmc.alloc_grads(g)
        tmc.tmc_backward(g, inp, ws, None, gr)
        torch.cuda.synchronize()
        lp = logp.cpu().numpy()
        assert np.abs(lp - ref["logp"]).max() <= LOGP_TOL
        lat = [0] + [i + 1 for i in ids]          # global latent index of each local latent
        for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
            for j, gl in enumerate(lat):
                if ref[k][gl] is None:
                    continue
                gg = gr[j][k].cpu().numpy()
                e = max(rel_err(gg, ref[k][gl]), max_err(gg, ref[k][gl]))
                assert e <= GRAD_TOL, (k, gl, e)


def test_shared_root_exchange_single_shard_equals_plain_forward(torch_cuda):
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload("T1_paper", N=16, K=128, B=2)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, direction=tmc.TMC_DIR_UP)
    inp = upload(torch, wl)
    ws = tmc.alloc_workspace(g)
    msg = torch.empty(wl.B, 129, dtype=torch.float64, device="cuda")
    tmc.tmc_forward_children(g, inp, msg, ws)
    l1 = torch.empty(wl.B, dtype=torch.float64, device="cuda")
    tmc.tmc_forward_root(g, inp, msg, l1, ws)
    l0, _ = tmc.estimate(g, inp, grads=False)
    torch.cuda.synchronize()
    np.testing.assert_allclose(l1.cpu().numpy(), l0.cpu().numpy(), rtol=0, atol=1e-4)
    with pytest.raises(tmc.TmcError):          # exchange needs an explicit UP direction
        tmc.tmc_forward_children(tmc.Graph(wl.parent[:2], wl.K[:2], wl.D[:2], wl.B), inp[:2], msg, ws)


# ------------------------------------------------------------------- more edge cases of the boundary
def _slice_K(wl, Ks):
    """Per-latent sample counts: keep the first K_i samples of latent i (and the first K_p parent
    samples of each conditional), a valid workload of the same model with unequal K_i."""
    z = [wl.z[i][:, :Ks[i]] for i in range(len(Ks))]
    kp = [1 if wl.parent[i] < 0 else Ks[wl.parent[i]] for i in range(len(Ks))]
    mu = [wl.mu[i][:, :kp[i]] for i in range(len(Ks))]
    lv = [wl.logvar[i][:, :kp[i]] for i in range(len(Ks))]
    lq = [wl.logq[i][:, :Ks[i]] for i in range(len(Ks))]
    lo = [None if wl.logobs[i] is None else wl.logobs[i][:, :Ks[i]] for i in range(len(Ks))]
    c = lambda L: [None if a is None else np.ascontiguousarray(a) for a in L]
    return c(z), c(mu), c(lv), c(lq), c(lo)


@pytest.mark.parametrize("name,Ks,direction", [("C3", [300, 130, 257, 129], 0), ("C4", [200, 130, 257, 300, 96], 2),
                                               ("C3", [1, 300, 7, 256], 0)])
def test_unequal_K_per_latent(torch_cuda, name, Ks, direction):
    """K_i may differ per latent: tensor-core and SIMT edges with unequal, ragged K."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    n = len(Ks)
    base = tw.make_workload(name, B=2, K=max(Ks))
    parent = base.parent[:n]
    z, mu, lv, lq, lo = _slice_K(base, Ks)
    if all(o is None for o in lo):        # keep an observation on the last latent
        lo[-1] = np.ascontiguousarray(base.logobs[-1][:, :Ks[-1]]) if base.logobs[-1] is not None else None
    D = base.D[:n]
    g = tmc.Graph(parent, Ks, D, base.B, direction=direction)
    t = lambda a: None if a is None else torch.from_numpy(a).cuda()
    inp = [dict(z=t(z[i]), mu=t(mu[i]), logvar=t(lv[i]), logq=t(lq[i]), logobs=t(lo[i])) for i in range(n)]
    logp, gr = tmc.estimate(g, inp)
    torch.cuda.synchronize()
    ref = oracle.estimate(parent, Ks, D, z, mu, lv, lq, lo)
    got = {"logp": logp.cpu().numpy()}
    for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
        got[k] = [gr[i][k].cpu().numpy() for i in range(n)]
    compare(got, ref, tag=f"{name}{Ks}")


def test_mixed_D_tree_tensor_cores(torch_cuda):
    """A tree whose sibling edges have D = 32 and D = 64 (batched tensor-core launches grouped by D)
    plus a D = 48 latent (no tensor-core geometry: SIMT) in the same level."""
    wl = tw.make_workload("S_tree", B=2, K=200, D=[32, 64, 32, 48, 64], w_var=1 / 64, c_var=1 / 64)
    got = run_gpu(torch_cuda, wl, precision=0)
    ref = oracle.estimate_workload(wl)
    compare(got, ref, tag="mixedD")


@pytest.mark.parametrize("precision", [1, 2])
def test_extreme_dynamic_range(torch_cuda, precision):
    """Unscaled linear maps at D = 64 (W entries of variance 0.5): |z| up to ~150, logp ~ -3e5 and
    column biases spanning > 60000 log2 units (beyond one fp16 part of the tensor-core bias
    operand).  Both paths must stay at fp32 accuracy relative to |logp| (an absolute 1e-3 is below
    the fp32 ulp of logp here; DESIGN.md §2 R3)."""
    wl = tw.make_workload("S_tree", B=2, K=200, D=[64] * 5, w_var=0.5, c_var=0.5)
    got = run_gpu(torch_cuda, wl, precision=precision, grads=False)
    ref = oracle.estimate_workload(wl, grads=False)
    rel = np.abs(got["logp"] - ref["logp"]) / np.abs(ref["logp"])
    assert rel.max() <= 1e-6, rel


def test_large_K_single_datapoint(torch_cuda):
    """K = 8192 (64 tiles per side, 4096 tiles per edge) on the tensor-core path."""
    wl = tw.make_workload("C3", B=1, K=8192, parent=[-1, 0, 1], D=[32] * 3)
    got = run_gpu(torch_cuda, wl)
    ref = oracle.estimate_workload(wl)
    compare(got, ref, tag="K8192")


def test_K_beyond_64_tiles(torch_cuda):
    """K = 8320 (65 tiles per side): past the 64-bit live-tile masks of the reverse pass, whose
    roles fall back to per-tile flag loads, and past the fixed-size flag arrays round 1 had in the
    column-bias and row-term kernels.  One datapoint carries dlogp = 0 (all tiles dead)."""
    wl = tw.make_workload("C3", B=2, K=8320, parent=[-1, 0, 1], D=[32] * 3)
    w = np.array([1.0, 0.0])
    got = run_gpu(torch_cuda, wl, dlogp=w)
    ref = oracle.estimate_workload(wl, dlogp=w)
    compare(got, ref, tag="K8320")


def test_empty_batch_launches_nothing(torch_cuda):
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload("C3", B=1, K=256)
    g = tmc.Graph(wl.parent, wl.K, wl.D, 0)
    e = lambda *s: torch.empty(*s, device="cuda")
    inp = [dict(z=e(0, 256, 32), mu=e(0, wl.Kp(i), 32), logvar=e(0, wl.Kp(i), 32), logq=e(0, 256),
                logobs=None if wl.logobs[i] is None else e(0, 256)) for i in range(len(wl.parent))]
    ws = torch.empty(max(1, tmc.tmc_workspace_size(g)), dtype=torch.uint8, device="cuda")
    n0 = tmc.tmc_launch_count()
    logp = torch.empty(0, dtype=torch.float64, device="cuda")
    tmc.tmc_forward(g, inp, logp, ws)
    tmc.tmc_backward(g, inp, ws, None, tmc.alloc_grads(g))
    torch.cuda.synchronize()
    assert tmc.tmc_launch_count() == n0


@pytest.mark.parametrize("B,b0,latent,K,D", [(3, 0, 0, 2048, 32), (2, 5, 7, 37, 5), (1, 1023, 2, 20, 100),
                                            (4, 0, 1, 1, 1), (2, 3, 4, 257, 64)])
def test_sample_normal_bit_exact(torch_cuda, B, b0, latent, K, D):
    """Row a1 (A22): the device sampler reproduces the host definition bit for bit."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    eps = torch.empty(B, K, D, device="cuda")
    tmc.tmc_sample_normal(0x1234_5678_9ABC, tmc.TAG_EPS, b0, latent, eps)
    torch.cuda.synchronize()
    ref = oracle.sample_normal(0x1234_5678_9ABC, tmc.TAG_EPS, B, b0, latent, K, D)
    assert np.array_equal(eps.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_harness_fresh_noise_is_the_sampler(torch_cuda):
    """The training-step harness draws its reparameterisation noise with tmc_sample_normal on the
    device: a shard's eps equals the host definition for its global datapoint ids, and the TMC
    estimate on the resulting model inputs matches the oracle."""
    import paper_1806_08593_b200 as tmc
    from tmc_workload.torch_model import TorchModel
    torch = torch_cuda
    cfg = tw.get_config("S_mlp", B=6, K=5)
    wl = tw.make_workload(cfg, b_ids=[2, 3, 4])
    m = TorchModel(wl, "cuda")
    m.fresh_noise(99)
    for i, e in enumerate(m.eps):
        ref = oracle.sample_normal(99, tmc.TAG_EPS, 3, 2, i, cfg.K, cfg.D[i])
        assert np.array_equal(e.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    f = m.forward()
    inp = [dict(z=f["z"][i].detach(), mu=f["mu"][i].detach(), logvar=f["logvar"][i].detach(),
                logq=f["logq"][i].detach(), logobs=None if f["logobs"][i] is None else f["logobs"][i].detach())
           for i in range(cfg.n)]
    g = tmc.Graph(cfg.parent, [cfg.K] * cfg.n, cfg.D, 3)
    logp, _ = tmc.estimate(g, inp, grads=False)
    c = lambda t: None if t is None else t.cpu().numpy()
    ref = oracle.estimate(cfg.parent, [cfg.K] * cfg.n, cfg.D, [c(x["z"]) for x in inp], [c(x["mu"]) for x in inp],
                          [c(x["logvar"]) for x in inp], [c(x["logq"]) for x in inp], [c(x["logobs"]) for x in inp],
                          grads=False)
    assert np.abs(logp.cpu().numpy() - ref["logp"]).max() <= LOGP_TOL


@pytest.mark.parametrize("name,kw", [("C0", {}), ("S_tree", {}), ("C2", dict(B=3, K=70)), ("C3", dict(B=2, K=300)),
                                     ("C4", dict(B=2, K=130)), ("C1", dict(B=3, K=20)), ("S_hier", dict(N=60, K=50))])
def test_iwae_parity(torch_cuda, name, kw):
    """NEXT-3: tmc_iwae vs the oracle's IWAE (value and every input gradient), dlogp weights."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload(name, **kw)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
    dl = np.linspace(-0.5, 1.5, wl.B)
    logp, gr = tmc.iwae(g, upload(torch, wl), dlogp=torch.from_numpy(dl).cuda())
    torch.cuda.synchronize()
    ref = oracle.iwae(wl.parent, wl.K, wl.D, wl.z, wl.mu, wl.logvar, wl.logq, wl.logobs, dlogp=dl)
    got = {"logp": logp.cpu().numpy()}
    for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
        got[k] = [gr[i][k].cpu().numpy() for i in range(len(wl.parent))]
    compare(got, ref, tag="iwae-" + name)


@pytest.mark.parametrize("name,kw", [("C0", {}), ("C1", {}), ("S_tree", {}), ("S_hier", dict(N=31, K=64)),
                                     ("C2", dict(B=3, K=16, D=[32, 64, 128, 64, 32]))])
def test_small_problem_kernel(torch_cuda, name, kw):
    """Small problems (K <= 64, D <= 128, n <= 32, TMC_PREC_AUTO) run as ONE launch per call
    (C0/C1 are launch-bound): parity with the oracle, pair marginals included, and
    exactly one kernel for tmc_forward and one for tmc_backward."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload(name, **kw)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
    inp = upload(torch, wl)
    ws = tmc.alloc_workspace(g)
    logp = torch.empty(wl.B, dtype=torch.float64, device="cuda")
    gr = tmc.alloc_grads(g, pair=True)
    n0 = tmc.tmc_launch_count()
    tmc.tmc_forward(g, inp, logp, ws)
    n1 = tmc.tmc_launch_count()
    dl = np.linspace(0.5, 1.5, wl.B)
    tmc.tmc_backward(g, inp, ws, torch.from_numpy(dl).cuda(), gr)
    n2 = tmc.tmc_launch_count()
    torch.cuda.synchronize()
    assert (n1 - n0, n2 - n1) == (1, 1)
    ref = oracle.estimate_workload(wl, dlogp=dl, pair=True)
    got = {"logp": logp.cpu().numpy()}
    for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
        got[k] = [gr[i][k].cpu().numpy() for i in range(len(wl.parent))]
    got["pair"] = [gr[i]["pair_marginal"].cpu().numpy() for i in range(len(wl.parent))]
    compare(got, ref, keys=("dz", "dmu", "dlogvar", "dlogq", "dlogobs", "pair"), tag="small-" + name)
    # tmc_estimate is ONE launch (§8d C0) with results bit-identical to tmc_forward + tmc_backward
    logp2 = torch.full_like(logp, float("nan"))
    gr2 = tmc.alloc_grads(g, pair=True)
    n0 = tmc.tmc_launch_count()
    tmc.tmc_estimate(g, inp, logp2, torch.from_numpy(dl).cuda(), gr2, ws)
    assert tmc.tmc_launch_count() - n0 == 1
    torch.cuda.synchronize()
    assert np.array_equal(logp2.cpu().numpy(), got["logp"])
    for i in range(len(wl.parent)):
        for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs", "pair_marginal"):
            assert torch.equal(gr[i][k], gr2[i][k]), (i, k)


@pytest.mark.parametrize("name,kw,precision,direction", [
    ("S_hier", dict(N=8, K=300, B=2), 0, 0),                       # D = 1, AUTO: padded to the D = 32 TC path
    ("S_tree", dict(K=200, B=2, w_var=0.1), 2, 0),                 # D = 2,3,2,2,1 with TC requested
    ("S_tree", dict(K=150, B=2, D=[48, 40, 8, 33, 20], w_var=1 / 48, c_var=1 / 48), 2, 0),   # pad to 64 and 32
    ("C3", dict(B=2, K=130, D=[5] * 8), 2, 1),                     # DOWN chain, D = 5
])
def test_tensor_core_padding(torch_cuda, name, kw, precision, direction):
    """Latents whose D is not 32/64 run on the tensor-core path from zero-padded copies (padded dims:
    z = mu = 0, logvar = -ln 2 pi, contributing exactly 0); values and every gradient vs the oracle."""
    wl = tw.make_workload(name, **kw)
    got = run_gpu(torch_cuda, wl, precision=precision, direction=direction)
    ref = oracle.estimate_workload(wl)
    compare(got, ref, tag=f"pad-{name}")


@pytest.mark.parametrize("name,kw", [("C3", dict(B=2, K=200)), ("S_hier", dict(N=4, K=150, B=2))])
def test_validate_flag(torch_cuda, name, kw):
    """TMC_FLAG_VALIDATE: NaN / +inf in an input -> TMC_ERR_NONFINITE before any compute; clean
    inputs (including -inf in logobs, a legal probability-zero event) pass and match the oracle."""
    import paper_1806_08593_b200 as tmc
    torch = torch_cuda
    wl = tw.make_workload(name, **kw)
    last = len(wl.parent) - 1
    wl.logobs[last][0, 3] = -np.inf
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, flags=tmc.TMC_FLAG_VALIDATE)
    inp = upload(torch, wl)
    logp, _ = tmc.estimate(g, inp, grads=False)
    torch.cuda.synchronize()
    ref = oracle.estimate_workload(wl, grads=False)
    assert np.abs(logp.cpu().numpy() - ref["logp"]).max() <= LOGP_TOL
    bad = [dict(d) for d in inp]
    bad[1] = dict(bad[1], mu=bad[1]["mu"].clone())
    bad[1]["mu"][0, 0, 0] = float("nan")
    with pytest.raises(tmc.TmcError) as e:
        tmc.estimate(g, bad, grads=False)
    assert e.value.status == -8


@pytest.mark.parametrize("B,n,M", [(3, 5, 6), (2, 4, 200)])
def test_exact_discrete_marginalisation_hmm(torch_cuda, B, n, M):
    """P:650-659 on the GPU dense-factor path: K_i = M states, stratified samples, uniform Q -> the
    TMC estimate is the exact log p(x) of the discrete chain (forward algorithm), gradients = pair
    marginals vs the oracle."""
    import paper_1806_08593_b200 as tmc
    import discrete
    torch = torch_cuda
    logf, obs, pi, A, _ = discrete.hmm(B=B, n=n, M=M)
    parent = [-1] + list(range(n - 1))
    g = tmc.Graph(parent, [M] * n, [1] * n, B)
    lf = [torch.from_numpy(x).cuda() for x in logf]
    inp = [dict(logobs=torch.from_numpy(o).cuda()) for o in obs]
    ws = tmc.alloc_workspace(g)
    logp = torch.empty(B, dtype=torch.float64, device="cuda")
    tmc.tmc_forward(g, inp, logp, ws, logf_dense=lf)
    dlf = [torch.empty_like(x) for x in lf]
    gr = [dict(dlogobs=torch.empty(B, M, device="cuda")) for _ in range(n)]
    tmc.tmc_backward(g, inp, ws, None, gr, logf_dense=lf, dlogf_dense=dlf)
    torch.cuda.synchronize()
    exact = discrete.hmm_forward_algorithm(logf, obs)
    assert np.abs(logp.cpu().numpy() - exact).max() <= LOGP_TOL
    ref = oracle.estimate(parent, [M] * n, [1] * n, None, None, None, None, obs, logf_dense=logf, pair=True)
    got = {"logp": logp.cpu().numpy(), "pair": [x.cpu().numpy() for x in dlf],
           "dlogobs": [x["dlogobs"].cpu().numpy() for x in gr]}
    compare(got, ref, keys=("pair", "dlogobs"), tag="hmm")


def test_exact_discrete_marginalisation_mixed(torch_cuda):
    """enumerating a discrete z_1 (uniform Q, one sample per state) inside TMC equals TMC on
    the model with z_1 marginalised out (GPU dense path vs the analytic reference)."""
    import paper_1806_08593_b200 as tmc
    import discrete
    torch = torch_cuda
    lf, ob, p = discrete.mixed(B=3, M=5, K=300)
    g = tmc.Graph([-1, 0], [5, 300], [1, 1], 3)
    inp = [dict(logobs=None), dict(logobs=torch.from_numpy(ob[1]).cuda())]
    ws = tmc.alloc_workspace(g)
    logp = torch.empty(3, dtype=torch.float64, device="cuda")
    tmc.tmc_forward(g, inp, logp, ws, logf_dense=[torch.from_numpy(x).cuda() for x in lf])
    torch.cuda.synchronize()
    ref = discrete.mixed_marginalised_reference(lf, ob, 300)
    assert np.abs(logp.cpu().numpy() - ref).max() <= LOGP_TOL


@pytest.mark.parametrize("name,kw", [("S_tree", {}), ("C4", dict(B=2, K=130)), ("C3", dict(B=2, K=200))])
def test_pair_marginal_invariants(torch_cuda, name, kw):
    """with dlogp = 1 every edge's pair marginals sum to 1, and the row sums of P_i
    equal pi_i = dlogobs_i (the marginal of k_i), per datapoint."""
    wl = tw.make_workload(name, **kw)
    got = run_gpu(torch_cuda, wl, pair=True)
    for i in range(len(wl.parent)):
        P = got["pair"][i].astype(np.float64)
        np.testing.assert_allclose(P.sum(axis=(1, 2)), 1.0, rtol=0, atol=1e-4)
        np.testing.assert_allclose(P.sum(axis=2), got["dlogobs"][i], rtol=1e-4, atol=1e-6)   # two passes, fp32


@pytest.mark.parametrize("name,kw,direction", [("C3", dict(B=3, K=600), 0), ("C4", dict(B=2, K=520), 0),
                                               ("C3", dict(B=2, K=2048), 0), ("C4", dict(B=2, K=512), 0),
                                               ("C3", dict(B=2, K=700), 2)])
def test_single_pass_reverse_matches_two_pass_and_oracle(torch_cuda, name, kw, direction):
    """The single-pass tensor-core reverse (one S and one P~ per tile, tc_bwd1_kernel) and the
    two-owner-pass reverse (TMC_FLAG_TWO_PASS_REVERSE) agree within fp32 rounding, and both match
    the oracle; both directions (DOWN chain, UP trees / UP on a chain)."""
    import paper_1806_08593_b200 as tmc
    wl = tw.make_workload(name, **kw)
    dl = np.linspace(0.5, 1.5, wl.B)
    one = run_gpu(torch_cuda, wl, direction=direction, dlogp=dl, flags=tmc.TMC_FLAG_SINGLE_PASS_REVERSE)
    two = run_gpu(torch_cuda, wl, direction=direction, dlogp=dl, flags=tmc.TMC_FLAG_TWO_PASS_REVERSE)
    assert np.array_equal(one["logp"], two["logp"])
    for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
        for i in range(len(wl.parent)):
            assert rel_err(one[k][i], two[k][i].astype(np.float64)) <= 1e-4, (k, i)
    sample = sorted({0, wl.B - 1})
    ref = oracle.estimate_workload(tw.make_workload(name, b_ids=sample, **kw), direction="up", dlogp=dl[sample])
    compare(one, ref, b_sel=sample, tag=f"single-pass {name}")


def test_single_pass_reverse_deterministic(torch_cuda):
    import paper_1806_08593_b200 as tmc
    wl = tw.make_workload("C3", B=3, K=520)
    a = run_gpu(torch_cuda, wl, flags=tmc.TMC_FLAG_SINGLE_PASS_REVERSE)
    b = run_gpu(torch_cuda, wl, flags=tmc.TMC_FLAG_SINGLE_PASS_REVERSE)
    for k in a:
        if k == "logp":
            assert np.array_equal(a[k], b[k])
        else:
            for x, y in zip(a[k], b[k]):
                assert np.array_equal(x, y), k
