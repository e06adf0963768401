"""Independent reference for the oracle's pins: the TMC estimator by its DEFINITION.

Eq. is: P_TMC = (1/prod_i K_i) sum over ALL index tuples (k_1..k_n) of
P(x, z^k) / prod_i Q(z_i^{k_i}), with the directed factorisation of P:571-576.  Enumerates
every combination explicitly; Gaussian log-densities come from scipy.stats.norm (a library
routine, not the oracle's formula).  Only usable for tiny instances.
"""
import itertools
import math

import numpy as np
from scipy.special import logsumexp
from scipy.stats import norm


def log_factor(z, mu, logvar, logq):
    """logf[a, r] = sum_d log N(z[a,d]; mu[r,d], exp(logvar[r,d])) - logq[a]  via scipy."""
    z = np.asarray(z, np.float64)
    mu = np.asarray(mu, np.float64)
    sd = np.exp(0.5 * np.asarray(logvar, np.float64))
    lp = norm.logpdf(z[:, None, :], loc=mu[None, :, :], scale=sd[None, :, :]).sum(-1)
    return lp - np.asarray(logq, np.float64)[:, None]


def log_weights(parent, K, factors, obs):
    """All prod K_i log importance weights, keyed by index tuple; factors[i] is [K_i][K_p]."""
    n = len(parent)
    combos = list(itertools.product(*[range(K[i]) for i in range(n)]))
    lw = np.empty(len(combos))
    for j, k in enumerate(combos):
        s = 0.0
        for i in range(n):
            r = 0 if parent[i] < 0 else k[parent[i]]
            s += factors[i][k[i], r]
            if obs[i] is not None:
                s += obs[i][k[i]]
        lw[j] = s
    return combos, lw


def tmc_bruteforce(parent, K, factors, obs):
    """log P_TMC = logsumexp(all weights) - sum_i ln K_i (Eq. is)."""
    _, lw = log_weights(parent, K, factors, obs)
    return logsumexp(lw) - sum(math.log(k) for k in K)


def pair_marginals(parent, K, factors, obs):
    """P_i[a, r] = sum of normalised weights over tuples with k_i=a, k_pa(i)=r."""
    combos, lw = log_weights(parent, K, factors, obs)
    w = np.exp(lw - logsumexp(lw))
    out = []
    for i in range(len(parent)):
        Kp = 1 if parent[i] < 0 else K[parent[i]]
        P = np.zeros((K[i], Kp))
        for j, k in enumerate(combos):
            P[k[i], 0 if parent[i] < 0 else k[parent[i]]] += w[j]
        out.append(P)
    return out


def workload_datapoint(wl, b):
    """Per-latent (factors, obs) for datapoint b of a tmc_workload.Workload, via scipy."""
    n = len(wl.parent)
    fac = [log_factor(wl.z[i][b], wl.mu[i][b], wl.logvar[i][b], wl.logq[i][b]) for i in range(n)]
    obs = [None if wl.logobs[i] is None else np.asarray(wl.logobs[i][b], np.float64) for i in range(n)]
    return fac, obs


def iwae_bruteforce(parent, K, factors, obs):
    """IWAE at equal K by definition: the K joint samples are the tuples (k, ..., k)."""
    n = len(parent)
    Kk = K[0]
    lw = np.array([sum(factors[i][k, 0 if parent[i] < 0 else k] + (0.0 if obs[i] is None else obs[i][k])
                       for i in range(n)) for k in range(Kk)])
    return logsumexp(lw) - math.log(Kk)
