"""General TMC elimination on a factor graph over sample indices — TEST INFRASTRUCTURE ONLY.

Plain fp64 numpy implementation of the TMC estimate on an arbitrary (loopy) factor graph, the
general formulation of PAPER.md §"Efficient averaging" (Fig[factor:loop] P:145-215):

    P_TMC = 1/(K_1 ... K_n) * sum_{k_1..k_n} prod_j f_j^{kappa_j}

evaluated by summing the indices out one at a time in a given order:

    f_new^{kappa'} = 1/K_v * sum_{k_v} prod_{j: v in kappa_j} f_j^{kappa_j},
    kappa' = (union of the kappa_j) minus {v}

(f_12^{k_2 k_3} = 1/K_1 sum_{k_1} f_1^{k_1 k_2} f_2^{k_1 k_3} is the paper's first step).  Everything
is in the log domain: a factor is an array of log f over its scope, and the sum over k_v is a
two-pass log-sum-exp with the JOINT max of the summands (SURVEY §8c reading A2; never the
appendix's separate row/column maxima, which can underflow).  Where the paper is silent: the 1/K_v
goes with the summed index (reading A1), an all -inf slice gives -inf (A3), and an index that no
factor touches sums to exactly 1 (1/K_v * K_v).

Gradients (the input to "gradient ascent on log P_TMC using standard automatic differentiation",
P:332): d log P_TMC / d log f_j [s] is the marginal probability of kappa_j = s under the normalised
summand prod_j f_j, written out by its definition — eliminate every index NOT in kappa_j (same
order), multiply the remaining factors into one table over kappa_j, and normalise:

    dL/dlogf_j[s] = exp( M_j(s) - sum_{v in kappa_j} ln K_v - L ) * dlogp,
    M_j(s) = log( 1/prod_{v not in kappa_j} K_v * sum_{k_rest} prod_i f_i ).

Shares no code with the CUDA path (paper_1806_08593_b200/) and never imports it; only tests/ may
import it.  Pinned in tests/test_oracle_elim.py by brute force over every index tuple (random loopy
graphs, Fig[factor:loop]), elimination-order invariance, the tree oracle (oracle.estimate on the
dense-factor path), the 4-variable loop's closed-form linear-Gaussian evidence (Monte Carlo
unbiasedness), and finite differences of the brute-force value for the gradients.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np


def _lse(x: np.ndarray, axis: int) -> np.ndarray:
    """log sum exp along `axis`, two-pass with the joint max; an all -inf slice gives -inf."""
    m = np.max(x, axis=axis, keepdims=True)
    mf = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(divide="ignore"):
        s = np.log(np.sum(np.exp(x - mf), axis=axis, keepdims=True)) + mf
    s = np.where(np.isneginf(m), -np.inf, s)
    return np.squeeze(s, axis=axis)


def _expand(f: np.ndarray, scope: Sequence[int], target: Sequence[int]) -> np.ndarray:
    """View factor f [B][K_scope...] as a broadcastable array over [B][K_target...]."""
    perm = [0] + [1 + list(scope).index(v) for v in target if v in scope]
    g = np.transpose(f, perm)
    shape = [f.shape[0]] + [f.shape[1 + list(scope).index(v)] if v in scope else 1 for v in target]
    return g.reshape(shape)


def _eliminate(K, factors, order):
    """factors: list of (scope tuple, log-table [B][K_scope...]).  Sums out the indices of `order`
    one at a time and returns the list of remaining factors."""
    fs = list(factors)
    for v in order:
        touch = [f for f in fs if v in f[0]]
        if not touch:
            continue                        # 1/K_v * sum_{k_v} 1 = 1
        fs = [f for f in fs if v not in f[0]]
        union = sorted({u for sc, _ in touch for u in sc})
        s = 0.0
        for sc, tab in touch:              # product of the touching factors: a sum of logs
            s = s + _expand(tab, sc, union)
        B = touch[0][1].shape[0]
        s = np.broadcast_to(s, [B] + [K[u] for u in union])
        out = _lse(s, axis=1 + union.index(v)) - np.log(K[v])
        fs.append((tuple(u for u in union if u != v), out))
    return fs


def _combine(fs, scope, B):
    """Product (log-sum) of factors whose scopes are subsets of `scope`, as a table over scope."""
    out = np.zeros([B] + [1] * len(scope))
    for sc, tab in fs:
        out = out + _expand(tab, sc, scope)
    return out


def eliminate(K: Sequence[int], scopes: Sequence[Sequence[int]], logf: Sequence[np.ndarray],
              order: Optional[Sequence[int]] = None, dlogp=None, grads: bool = True):
    """TMC estimate of a factor graph over sample indices k_0..k_{n-1} (K[v] samples each).

    scopes[j]: the index variables of factor j, in the axis order of logf[j] ([B][K_scope...]).
    order: elimination order (a permutation of range(n)); default 0..n-1.
    Returns {"logp": float64[B]} and, if grads, "dlogf": list of float64 arrays shaped like logf
    (dJ/dlogf_j for J = sum_b dlogp[b] logp[b], dlogp default ones).
    """
    n = len(K)
    order = list(range(n)) if order is None else list(order)
    assert sorted(order) == list(range(n)), "order must be a permutation of the index variables"
    lf = [np.asarray(f, dtype=np.float64) for f in logf]
    B = lf[0].shape[0]
    for sc, f in zip(scopes, lf):
        assert f.shape == tuple([B] + [K[u] for u in sc]), (sc, f.shape)
    facs = [(tuple(sc), f) for sc, f in zip(scopes, lf)]
    rest = _eliminate(K, facs, order)
    logp = np.zeros(B)
    for sc, tab in rest:
        assert len(sc) == 0
        logp = logp + tab
    out = {"logp": logp}
    if not grads:
        return out
    w = np.ones(B) if dlogp is None else np.asarray(dlogp, np.float64)
    dl = []
    for sc, f in facs:
        keep = list(sc)
        others = [v for v in order if v not in keep]
        part = _eliminate(K, facs, others)          # factors over subsets of kappa_j
        M = _combine(part, keep, B)
        M = np.broadcast_to(M, f.shape)
        lnK = sum(np.log(K[v]) for v in keep)
        with np.errstate(invalid="ignore"):
            e = M - lnK - logp.reshape([B] + [1] * len(keep))
        P = np.where(np.isfinite(logp).reshape([B] + [1] * len(keep)), np.exp(np.where(np.isnan(e), -np.inf, e)), 0.0)
        dl.append(P * w.reshape([B] + [1] * len(keep)))
    out["dlogf"] = dl
    return out

