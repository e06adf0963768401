"""Seeded inputs for the general-elimination (loopy factor graph) tests: dense log-factor tables and
their scopes.  Model log-densities come from scipy (a library routine); no elimination arithmetic.

fig_loop: the directed model of Fig[factor:loop]A,
    z1 ~ N(0, I),  z2 | z1 ~ N(W2 z1, s I),  z3 | z1 ~ N(W3 z1, s I),  z4 | z2 ~ N(W4 z2, s I),
    x | z3, z4 ~ N(A z3 + C z4, sx I),
with independent proposals q_i = N(0, q I) and K_i samples of each latent.  Its TMC factor graph
(Fig B) has the four pairwise factors
    f_1^{k1 k2} = P(z1) P(z2|z1) / (Q(z1) Q(z2)),   f_2^{k1 k3} = P(z3|z1) / Q(z3),
    f_3^{k2 k4} = P(z4|z2) / Q(z4),                 f_4^{k3 k4} = P(x|z3, z4)
(the typical directed factorisation, with x's two parents making f_4 a loop-closing
pairwise factor).  The evidence p(x) is Gaussian in closed form (fig_loop_evidence).
"""
import math

import numpy as np
from scipy.stats import multivariate_normal, norm

FIG_LOOP_SCOPES = [(0, 1), (0, 2), (1, 3), (2, 3)]


def _lognorm(x, mu, var):
    return norm.logpdf(x, loc=mu, scale=math.sqrt(var)).sum(-1)


def fig_loop_model(d=2, seed=0):
    rng = np.random.default_rng([seed, 7101])
    W2, W3, W4 = (rng.normal(0, math.sqrt(0.5), (d, d)) for _ in range(3))
    A, C = rng.normal(0, 1, (d, d)), rng.normal(0, 1, (d, d))
    return dict(d=d, W2=W2, W3=W3, W4=W4, A=A, C=C, s=0.5, sx=0.1, q=2.0)


def fig_loop_evidence(m, x):
    """log p(x) of the linear-Gaussian model (ancestral covariances)."""
    d = m["d"]
    I = np.eye(d)
    # z = (z1, z2, z3, z4) = L e, e ~ N(0, I_4d) (per block); x = A z3 + C z4 + noise
    S1 = I
    S2 = m["W2"] @ S1 @ m["W2"].T + m["s"] * I
    S3 = m["W3"] @ S1 @ m["W3"].T + m["s"] * I
    S4 = m["W4"] @ S2 @ m["W4"].T + m["s"] * I
    S34 = m["W3"] @ S1 @ m["W2"].T @ m["W4"].T          # Cov(z3, z4)
    Sx = (m["A"] @ S3 @ m["A"].T + m["C"] @ S4 @ m["C"].T + m["A"] @ S34 @ m["C"].T
          + m["C"] @ S34.T @ m["A"].T + m["sx"] * I)
    return multivariate_normal(mean=np.zeros(d), cov=Sx).logpdf(x)


def fig_loop_data(m, B, seed=0):
    rng = np.random.default_rng([seed, 7102])
    d = m["d"]
    z1 = rng.normal(size=(B, d))
    z2 = z1 @ m["W2"].T + math.sqrt(m["s"]) * rng.normal(size=(B, d))
    z3 = z1 @ m["W3"].T + math.sqrt(m["s"]) * rng.normal(size=(B, d))
    z4 = z2 @ m["W4"].T + math.sqrt(m["s"]) * rng.normal(size=(B, d))
    return z3 @ m["A"].T + z4 @ m["C"].T + math.sqrt(m["sx"]) * rng.normal(size=(B, d))


def fig_loop_factors(m, x, K, seed=0, dtype=np.float32):
    """Dense log-factors [B][K_u][K_v] of Fig B for data x [B][d], K = (K1, K2, K3, K4) samples."""
    rng = np.random.default_rng([seed, 7103])
    B, d = x.shape
    q = m["q"]
    z = [rng.normal(0, math.sqrt(q), (B, K[i], d)) for i in range(4)]
    lq = [_lognorm(z[i], 0.0, q) for i in range(4)]
    f1 = (_lognorm(z[1][:, None, :, :], (z[0] @ m["W2"].T)[:, :, None, :], m["s"]) - lq[1][:, None, :]
          + (_lognorm(z[0], 0.0, 1.0) - lq[0])[:, :, None])
    f2 = _lognorm(z[2][:, None, :, :], (z[0] @ m["W3"].T)[:, :, None, :], m["s"]) - lq[2][:, None, :]
    f3 = _lognorm(z[3][:, None, :, :], (z[1] @ m["W4"].T)[:, :, None, :], m["s"]) - lq[3][:, None, :]
    mean = (z[2] @ m["A"].T)[:, :, None, :] + (z[3] @ m["C"].T)[:, None, :, :]
    f4 = _lognorm(x[:, None, None, :], mean, m["sx"])
    return [np.ascontiguousarray(f.astype(dtype)) for f in (f1, f2, f3, f4)]


def random_graph(n, K, nfac, B, seed=0, max_arity=3, scale=2.0, dtype=np.float32):
    """A random factor graph over n index variables: nfac factors of arity 1..max_arity with
    random scopes (every variable covered) and N(0, scale^2) log-factor entries."""
    rng = np.random.default_rng([seed, 7104])
    scopes = []
    for v in range(n):                                       # cover every variable
        a = int(rng.integers(1, max_arity + 1))
        others = [u for u in rng.permutation(n) if u != v][:a - 1]
        scopes.append(tuple([v] + [int(u) for u in others]))
    while len(scopes) < nfac:
        a = int(rng.integers(1, max_arity + 1))
        scopes.append(tuple(int(u) for u in rng.permutation(n)[:a]))
    logf = [rng.normal(0, scale, [B] + [K[u] for u in sc]).astype(dtype) for sc in scopes]
    return scopes, logf
