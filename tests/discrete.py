"""Discrete / mixed models for the exact-marginalisation pins: inputs of the
dense-factor path and independent references (forward algorithm; analytic marginalisation)."""
import math

import numpy as np
from scipy.special import logsumexp
from scipy.stats import norm


def hmm(B, n, M, seed=0):
    """Discrete chain z_1 -> ... -> z_n, M states each, Gaussian emissions x_i | z_i = m ~ N(m, 1).
    TMC with K_i = M, stratified samples z_i^k = k and uniform Q = 1/M:
    logf_0[b,a,0] = log pi_a + log M, logf_i[b,a,c] = log A[c,a] + log M, logobs_i[b,a] = log N(x_i; a, 1)."""
    rng = np.random.default_rng([seed, 101])
    pi = rng.dirichlet(np.ones(M))
    A = rng.dirichlet(np.ones(M), size=M)                   # A[c, a] = P(z_i = a | z_{i-1} = c)
    x = rng.normal(M / 2, M / 3, size=(B, n))
    logf = [np.broadcast_to((np.log(pi) + math.log(M))[None, :, None], (B, M, 1)).astype(np.float32).copy()]
    for _ in range(1, n):
        logf.append(np.broadcast_to((np.log(A.T) + math.log(M))[None], (B, M, M)).astype(np.float32).copy())
    obs = [norm.logpdf(x[:, i][:, None], np.arange(M)[None, :], 1.0).astype(np.float32) for i in range(n)]
    return logf, obs, pi, A, x


def hmm_forward_algorithm(logf, obs):
    """log p(x) by the forward recursion alpha_t = (alpha_{t-1} A) * e_t, in log space (fp64), on the
    same fp32 inputs the estimator reads (log pi = logf_0 - log M, log A^T = logf_i - log M)."""
    B, M = obs[0].shape
    out = np.empty(B)
    for b in range(B):
        la = logf[0][b, :, 0].astype(np.float64) - math.log(M) + obs[0][b].astype(np.float64)
        for t in range(1, len(obs)):
            lA = logf[t][b].astype(np.float64).T - math.log(M)            # [c, a]
            la = logsumexp(la[:, None] + lA, axis=0) + obs[t][b].astype(np.float64)
        out[b] = logsumexp(la)
    return out


def mixed(B, M, K, seed=0):
    """z_1 discrete (M states, prior pi) -> z_2 | z_1 = m ~ N(mu_m, s^2) -> x ~ N(z_2, 1); z_1 enumerated
    exactly (K_1 = M, uniform Q), z_2 sampled from q = N(0, 4) with K samples."""
    rng = np.random.default_rng([seed, 202])
    pi = rng.dirichlet(np.ones(M))
    mu = rng.normal(0, 2, size=M)
    s = 0.7
    x = rng.normal(0, 2, size=B)
    z2 = rng.normal(0, 2, size=(B, K))
    lq2 = norm.logpdf(z2, 0, 2)
    logf1 = np.broadcast_to((np.log(pi) + math.log(M))[None, :, None], (B, M, 1)).astype(np.float32).copy()
    logf2 = (norm.logpdf(z2[:, :, None], mu[None, None, :], s) - lq2[:, :, None]).astype(np.float32)   # [B][K][M]
    obs2 = norm.logpdf(x[:, None], z2, 1.0).astype(np.float32)
    return [logf1, logf2], [None, obs2], dict(pi=pi, mu=mu, s=s, x=x, z2=z2, lq2=lq2)


def mixed_marginalised_reference(logf, obs, K):
    """The TMC estimator over the model with z_1 summed out, on the same fp32 inputs: one
    latent z_2 whose factor is LSE_m(log pi_m + log N(z_2; mu_m, s^2)) - log q(z_2)."""
    M = logf[0].shape[1]
    lpi = logf[0][:, :, 0].astype(np.float64) - math.log(M)                       # [B][M]
    lp = logsumexp(lpi[:, None, :] + logf[1].astype(np.float64), axis=2)          # [B][K]
    return logsumexp(lp + obs[1].astype(np.float64), axis=1) - math.log(K)
