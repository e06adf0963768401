"""GPU parity of the general elimination (Fig[factor:loop]):
libtmc tmc_elim_forward / tmc_elim_backward through the C ABI vs the fp64 oracle (oracle/elim.py)
on identical seeded fp32 tables.  Bars (north_star): |dlogp| <= 1e-3 absolute per datapoint; the
factor gradients (marginals) within 1e-3 per (factor, datapoint) in relative L2 and element-wise
against the largest entry."""
import numpy as np
import pytest

from oracle import elim
import loopy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    import paper_1806_08593_b200 as tmc
    tmc.load_library()
    return torch


def run(torch, K, scopes, lf, order=None, dlogp=None):
    import paper_1806_08593_b200 as tmc
    B = lf[0].shape[0]
    fg = tmc.FactorGraph(K, scopes, B, order)
    t = [torch.from_numpy(np.ascontiguousarray(f, dtype=np.float32)).cuda() for f in lf]
    dl = None if dlogp is None else torch.from_numpy(np.asarray(dlogp, np.float64)).cuda()
    n0 = tmc.tmc_launch_count()
    logp, g = tmc.eliminate(fg, t, dlogp=dl)
    torch.cuda.synchronize()
    assert tmc.tmc_launch_count() > n0
    return logp.cpu().numpy(), [x.cpu().numpy() for x in g]


def check(got, ref, tag=""):
    lp, g = got
    fin = np.isfinite(ref["logp"])
    assert np.array_equal(np.isfinite(lp), fin), tag
    d = np.abs(lp[fin] - ref["logp"][fin]).max(initial=0)
    assert d <= 1e-3, f"{tag}: |dlogp| = {d}"
    for j, (a, r) in enumerate(zip(g, ref["dlogf"])):
        for b in range(r.shape[0]):
            nr, mr = np.linalg.norm(r[b]), np.abs(r[b]).max(initial=0)
            if nr < 1e-12:
                assert np.abs(a[b]).max(initial=0) < 1e-6, (tag, j, b)
                continue
            e = a[b].astype(np.float64) - r[b]
            assert np.linalg.norm(e) / nr <= 1e-3, (tag, j, b, np.linalg.norm(e) / nr)
            assert np.abs(e).max() / mr <= 1e-3, (tag, j, b, np.abs(e).max() / mr)
    return d


@pytest.mark.parametrize("K", [3, 64, 256])
def test_fig_loop(torch_cuda, K):
    """Fig[factor:loop]: f_1^{k1k2} f_2^{k1k3} f_3^{k2k4} f_4^{k3k4}, eliminated k1, k2, (k3, k4)."""
    m = loopy.fig_loop_model(d=2)
    B = 3 if K < 256 else 2
    x = loopy.fig_loop_data(m, B=B)
    Ks = (K, K, K, K)
    lf = loopy.fig_loop_factors(m, x, Ks)
    dl = np.linspace(0.5, 1.5, B)
    ref = elim.eliminate(Ks, loopy.FIG_LOOP_SCOPES, lf, [0, 1, 2, 3], dlogp=dl)
    check(run(torch_cuda, Ks, loopy.FIG_LOOP_SCOPES, lf, [0, 1, 2, 3], dlogp=dl), ref, f"fig-loop K={K}")


@pytest.mark.parametrize("order", [[3, 2, 1, 0], [1, 2, 0, 3]])
def test_fig_loop_other_orders_unequal_K(torch_cuda, order):
    m = loopy.fig_loop_model(d=2, seed=4)
    x = loopy.fig_loop_data(m, B=2, seed=4)
    Ks = (37, 130, 5, 64)
    lf = loopy.fig_loop_factors(m, x, Ks, seed=4)
    ref = elim.eliminate(Ks, loopy.FIG_LOOP_SCOPES, lf, order)
    check(run(torch_cuda, Ks, loopy.FIG_LOOP_SCOPES, lf, order), ref, f"order {order}")


@pytest.mark.parametrize("seed", range(4))
def test_random_loopy_graphs(torch_cuda, seed):
    """Random graphs with 1-, 2- and 3-index factors and 3-index intermediates."""
    rng = np.random.default_rng(100 + seed)
    n = 6
    K = [int(k) for k in rng.integers(3, 24, n)]
    scopes, lf = loopy.random_graph(n, K, nfac=n + 2, B=3, seed=seed, max_arity=2, scale=1.0)
    import paper_1806_08593_b200 as tmc
    # pick an order whose intermediates stay within 3 indices
    for _ in range(50):
        order = [int(v) for v in rng.permutation(n)]
        try:
            tmc.tmc_elim_workspace_size(tmc.FactorGraph(K, scopes, 3, order))
            break
        except tmc.TmcError:
            continue
    dl = np.array([1.0, -0.5, 2.0])
    ref = elim.eliminate(K, scopes, lf, order, dlogp=dl)
    check(run(torch_cuda, K, scopes, lf, order, dlogp=dl), ref, f"random seed {seed}")


def test_three_index_intermediate(torch_cuda):
    K = (20, 9, 17, 12)
    rng = np.random.default_rng(5)
    scopes = [(0, 1), (0, 2), (0, 3), (1, 2), (2, 3), (3,), (1, 2, 3)]
    lf = [rng.normal(0, 1.5, [2] + [K[u] for u in sc]).astype(np.float32) for sc in scopes]
    ref = elim.eliminate(K, scopes, lf, [0, 1, 2, 3])
    check(run(torch_cuda, K, scopes, lf, [0, 1, 2, 3]), ref, "3-index")


def test_neg_inf_and_dead_datapoint(torch_cuda):
    m = loopy.fig_loop_model(d=2)
    x = loopy.fig_loop_data(m, B=3)
    Ks = (16, 16, 16, 16)
    lf = loopy.fig_loop_factors(m, x, Ks)
    lf[0][0, 3, :] = -np.inf
    lf[3][1] = -np.inf                  # datapoint 1: every tuple impossible
    ref = elim.eliminate(Ks, loopy.FIG_LOOP_SCOPES, lf)
    lp, g = run(torch_cuda, Ks, loopy.FIG_LOOP_SCOPES, lf)
    assert lp[1] == -np.inf
    for a in g:
        assert not np.isnan(a).any()
        assert np.all(a[1] == 0.0)
    check((lp, g), ref, "-inf")


def test_exact_discrete_hmm_matches_forward_algorithm(torch_cuda):
    """P:650-659 through the general elimination: a discrete chain with one 'sample' per state and
    uniform Q, eliminated left to right, is the forward algorithm's exact log p(x)."""
    import discrete
    B, n, M = 3, 5, 40
    logf, obs, _, _, _ = discrete.hmm(B=B, n=n, M=M)
    scopes, tabs = [(0,)], [logf[0][:, :, 0]]
    for i in range(1, n):
        scopes.append((i, i - 1))
        tabs.append(logf[i])
    for i in range(n):
        scopes.append((i,))
        tabs.append(obs[i])
    exact = discrete.hmm_forward_algorithm(logf, obs)
    lp, _ = run(torch_cuda, [M] * n, scopes, tabs)
    assert np.abs(lp - exact).max() <= 1e-3

