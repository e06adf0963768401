"""Pins of the general-elimination oracle (oracle/elim.py).

Every pin is independent of the oracle's code:
  * brute force: P_TMC = 1/prod K * sum over EVERY index tuple of prod_j f_j, enumerated
    here with scipy's logsumexp, on Fig[factor:loop] and on random loopy graphs with 1-, 2- and
    3-index factors (orders that create 3-index intermediates included);
  * gradients: the brute-force marginal of each factor's scope, and central finite differences of
    the brute-force value;
  * order invariance at sizes brute force cannot reach;
  * the tree oracle (oracle.estimate, dense-factor path, a separate C++ implementation) on trees;
  * the closed-form evidence of Fig A's linear-Gaussian model: E[exp L_TMC] = p(x).
"""
import itertools
import math

import numpy as np
import pytest
from scipy.special import logsumexp

import oracle
from oracle import elim
import loopy


def brute(K, scopes, logf):
    """(logp [B], marginals per factor) by enumerating every index tuple."""
    B = logf[0].shape[0]
    lf = [np.asarray(f, np.float64) for f in logf]
    tuples = list(itertools.product(*[range(k) for k in K]))
    T = np.empty((B, len(tuples)))
    for t, k in enumerate(tuples):
        T[:, t] = sum(f[(slice(None),) + tuple(k[u] for u in sc)] for sc, f in zip(scopes, lf))
    L = logsumexp(T, axis=1) - float(np.sum(np.log(K)))
    marg = []
    for sc, f in zip(scopes, lf):
        P = np.zeros(f.shape)
        w = np.exp(T - logsumexp(T, axis=1, keepdims=True))
        for t, k in enumerate(tuples):
            P[(slice(None),) + tuple(k[u] for u in sc)] += w[:, t]
        marg.append(P)
    return L, marg


def test_fig_loop_bruteforce_and_marginals():
    m = loopy.fig_loop_model(d=2)
    x = loopy.fig_loop_data(m, B=3)
    K = (3, 4, 2, 3)
    lf = loopy.fig_loop_factors(m, x, K)
    L, marg = brute(K, loopy.FIG_LOOP_SCOPES, lf)
    for order in ([0, 1, 2, 3], [3, 2, 1, 0], [1, 2, 0, 3], [0, 3, 1, 2]):
        r = elim.eliminate(K, loopy.FIG_LOOP_SCOPES, lf, order)
        np.testing.assert_allclose(r["logp"], L, rtol=0, atol=1e-10)
        for j in range(4):
            np.testing.assert_allclose(r["dlogf"][j], marg[j], rtol=0, atol=1e-12)


@pytest.mark.parametrize("seed", range(6))
def test_random_loopy_graph_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n = 5 if seed % 2 else 6
    K = [int(k) for k in rng.integers(2, 4, n)]
    scopes, lf = loopy.random_graph(n, K, nfac=n + 3, B=2, seed=seed, max_arity=3)
    L, marg = brute(K, scopes, lf)
    dl = np.array([0.7, -1.3])
    for order in (list(range(n)), list(rng.permutation(n))):
        r = elim.eliminate(K, scopes, lf, order, dlogp=dl)
        np.testing.assert_allclose(r["logp"], L, rtol=0, atol=1e-10)
        for j in range(len(scopes)):
            np.testing.assert_allclose(r["dlogf"][j], marg[j] * dl.reshape([2] + [1] * len(scopes[j])),
                                       rtol=0, atol=1e-12)


def test_three_index_intermediate_bruteforce():
    """A star around index 0 with three pairwise factors: eliminating 0 first creates the
    3-index intermediate f_{0}^{k1 k2 k3} = 1/K_0 sum_{k0} f_a^{k0 k1} f_b^{k0 k2} f_c^{k0 k3}."""
    K = (3, 2, 4, 3)
    rng = np.random.default_rng(5)
    scopes = [(0, 1), (0, 2), (0, 3), (1, 2), (2, 3), (3,)]
    lf = [rng.normal(0, 1.5, [2] + [K[u] for u in sc]) for sc in scopes]
    L, marg = brute(K, scopes, lf)
    r = elim.eliminate(K, scopes, lf, [0, 1, 2, 3])
    np.testing.assert_allclose(r["logp"], L, rtol=0, atol=1e-10)
    for j in range(len(scopes)):
        np.testing.assert_allclose(r["dlogf"][j], marg[j], rtol=0, atol=1e-12)


def test_gradient_central_differences():
    K = (3, 3, 2, 3)
    m = loopy.fig_loop_model(d=1, seed=3)
    x = loopy.fig_loop_data(m, B=1, seed=3)
    lf = [f.astype(np.float64) for f in loopy.fig_loop_factors(m, x, K, seed=3)]
    r = elim.eliminate(K, loopy.FIG_LOOP_SCOPES, lf, [2, 0, 1, 3])
    h = 1e-5
    rng = np.random.default_rng(0)
    for j in range(4):
        for _ in range(3):
            idx = (0,) + tuple(int(rng.integers(0, s)) for s in lf[j].shape[1:])
            up = [f.copy() for f in lf]
            dn = [f.copy() for f in lf]
            up[j][idx] += h
            dn[j][idx] -= h
            fd = (brute(K, loopy.FIG_LOOP_SCOPES, up)[0] - brute(K, loopy.FIG_LOOP_SCOPES, dn)[0]) / (2 * h)
            assert abs(fd[0] - r["dlogf"][j][idx]) < 1e-7, (j, idx, fd[0], r["dlogf"][j][idx])


def test_order_invariance_large_K():
    m = loopy.fig_loop_model(d=2)
    x = loopy.fig_loop_data(m, B=2)
    K = (20, 24, 16, 20)
    lf = loopy.fig_loop_factors(m, x, K)
    a = elim.eliminate(K, loopy.FIG_LOOP_SCOPES, lf, [0, 1, 2, 3], grads=False)["logp"]
    b = elim.eliminate(K, loopy.FIG_LOOP_SCOPES, lf, [3, 1, 0, 2], grads=False)["logp"]
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-10)


def test_tree_equals_tree_oracle():
    """On a tree the general elimination (leaves first) equals the tree oracle's dense path."""
    rng = np.random.default_rng(11)
    parent = [-1, 0, 0, 1, 1, 2]
    K = [3, 4, 2, 3, 5, 4]
    B = 2
    n = len(parent)
    logf = [rng.normal(0, 1, (B, K[i], 1 if parent[i] < 0 else K[parent[i]])).astype(np.float32) for i in range(n)]
    obs = [rng.normal(0, 1, (B, K[i])).astype(np.float32) if i % 2 else None for i in range(n)]
    ref = oracle.estimate(parent, K, [1] * n, None, None, None, None, obs, logf_dense=logf, pair=True)
    scopes, tabs = [], []
    for i in range(n):
        if parent[i] < 0:
            scopes.append((i,))
            tabs.append(logf[i][:, :, 0])
        else:
            scopes.append((i, parent[i]))
            tabs.append(logf[i])
        if obs[i] is not None:
            scopes.append((i,))
            tabs.append(obs[i])
    r = elim.eliminate(K, scopes, tabs, [5, 4, 3, 2, 1, 0])
    np.testing.assert_allclose(r["logp"], ref["logp"], rtol=0, atol=1e-9)
    j = 0
    for i in range(n):
        got = r["dlogf"][j] if parent[i] >= 0 else r["dlogf"][j][:, :, None]
        np.testing.assert_allclose(got, ref["pair"][i], rtol=0, atol=1e-9)
        j += 1 + (obs[i] is not None)


def test_fig_loop_unbiased_against_closed_form():
    """E[exp(L_TMC - log p(x))] = 1: Monte Carlo over independent sample sets at K = 3."""
    m = loopy.fig_loop_model(d=1, seed=2)
    x = loopy.fig_loop_data(m, B=1, seed=2)
    lp = loopy.fig_loop_evidence(m, x[0])
    K = (3, 3, 3, 3)
    R = 4000
    vals = np.empty(R)
    for r in range(R):
        lf = loopy.fig_loop_factors(m, x, K, seed=1000 + r, dtype=np.float64)
        vals[r] = elim.eliminate(K, loopy.FIG_LOOP_SCOPES, lf, grads=False)["logp"][0]
    w = np.exp(vals - lp)
    se = w.std(ddof=1) / math.sqrt(R)
    assert abs(w.mean() - 1.0) <= 4 * se, (w.mean(), se)
    assert vals.mean() <= lp                      # Jensen


def test_neg_inf_and_untouched_index():
    K = (2, 3, 2)
    scopes = [(0, 1), (1,)]                    # index 2 appears in no factor: sums to exactly 1
    lf = [np.array([[[0.0, -np.inf, 1.0], [-np.inf, -np.inf, -np.inf]], [[-np.inf] * 3] * 2]),
          np.array([[0.5, 0.0, -1.0], [0.0, 0.0, 0.0]])]
    r = elim.eliminate(K, scopes, lf, [2, 0, 1])
    want0 = logsumexp([0.0 + 0.5, 1.0 - 1.0]) - math.log(2) - math.log(3)
    assert abs(r["logp"][0] - want0) < 1e-12
    assert r["logp"][1] == -np.inf
    assert np.all(r["dlogf"][0][1] == 0.0) and np.all(r["dlogf"][1][1] == 0.0)
    assert not np.isnan(r["dlogf"][0]).any()
