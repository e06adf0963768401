"""Seeded synthetic workloads for the TMC hot path (inputs only).

This module is the ONE piece of code shared by the CUDA path's tests/bench
and by the CPU oracle's tests.  It draws proposal samples and evaluates the
*model* (linear maps / random-init MLP conditionals, proposal and observation
log-densities) to produce the estimator's inputs.  It holds none of the
method's arithmetic: no factor tensor, no message, no logsumexp, no gradient.

Inputs follow the layout of include/tmc.h (all float32, row-major):

    z[i]      [B][K_i][D_i]   proposal samples z_i^{k_i}
    mu[i]     [B][K_p][D_i]   mean of p(z_i | z_pa^{k_pa}), root K_p=1
    logvar[i] [B][K_p][D_i]   log-variance of the same conditional
    logq[i]   [B][K_i]        log Q(z_i^{k_i} | ...)  (non-factorised allowed)
    logobs[i] [B][K_i]|None   log P(x | z_i^{k_i}) for observations attached to i

Every random draw is keyed by (seed, stream tag, global datapoint id b), so a
datapoint's inputs do not depend on which batch/shard/rank generates it
(SURVEY.md §8c A12).  Config recipes: BASELINE.json configs[0..4] with the
readings listed in DESIGN.md ("Workload recipe").
"""
from __future__ import annotations

import dataclasses
import math
import os
from concurrent.futures import ThreadPoolExecutor
from typing import Dict, List, Optional, Sequence

import numpy as np

_TAG = {"params": 1, "data": 2, "prop": 3, "mc": 4}
LOG2PI = math.log(2.0 * math.pi)


def rng_for(seed: int, tag: str, b: int = 0, extra: int = 0) -> np.random.Generator:
    """Counter-keyed generator: identical draws for (seed, tag, b) on any host."""
    return np.random.default_rng([int(seed), _TAG[tag], int(b), int(extra)])


# ----------------------------------------------------------------------------- configs
@dataclasses.dataclass
class Config:
    name: str
    family: str                      # "lg" | "mlp_chain" | "mnist" | "hier"
    B: int
    K: int
    parent: List[int]
    D: List[int]
    # linear-Gaussian family
    w_var: float = 0.5               # variance of the entries of W (A15: N(.,.) = variance)
    noise_var: float = 0.5           # conditional variance of z_c | z_p
    observed: Optional[List[int]] = None   # latents that emit an observation
    obs_dim: int = 4
    c_var: float = 1.0
    obs_var: float = 0.1
    q: str = "fixed"                 # "fixed" (N(0, q_var I)) | "prior_marginal" (A8, C4)
    q_var: float = 2.0
    # MLP families
    hidden: int = 128
    obs_kind: str = "bernoulli"      # "bernoulli" | "gauss"
    obs_sigma: float = 0.1
    pixel_p: float = 0.13
    # mnist family extra dims
    enc_hidden: int = 200
    dec_hidden: int = 200
    # hier family (toy 1): global ids of the data points this shard holds (None = all)
    children: Optional[List[int]] = None

    @property
    def n(self) -> int:
        return len(self.parent)

    def Kp(self, i: int) -> int:
        return 1 if self.parent[i] < 0 else self.K

    def pair_terms(self) -> int:
        """Forward pair terms per call: B * sum over non-root edges K_i*K_p."""
        return self.B * sum(self.K * self.K for i in range(self.n) if self.parent[i] >= 0)


def _chain(n: int) -> List[int]:
    return [-1] + list(range(n - 1))


def _star(N: int) -> List[int]:
    return [-1] + [0] * N


def _tree_c4() -> List[int]:
    parent = [-1, 0, 0, 0, 0]
    for c in range(1, 5):
        parent += [c] * 4
    return parent


CONFIGS: Dict[str, Config] = {
    # BASELINE.json configs[0]: tiny linear-Gaussian chain (brute-force enumerable)
    "C0": Config("C0", "lg", B=8, K=8, parent=_chain(4), D=[2] * 4, w_var=0.5, noise_var=0.5,
                 observed=[3], obs_dim=4, c_var=1.0, obs_var=0.1, q="fixed", q_var=2.0),
    # configs[1]: MNIST-shaped two-stochastic-layer model (latent 0 = z_2 (50), latent 1 = z_1 (100))
    "C1": Config("C1", "mnist", B=128, K=20, parent=[-1, 0], D=[50, 100], hidden=100,
                 enc_hidden=200, dec_hidden=200, pixel_p=0.13),
    # configs[2]: deep chain, 5 layers of 64, K=256, Bernoulli(784) observation
    "C2": Config("C2", "mlp_chain", B=512, K=256, parent=_chain(5), D=[64] * 5, hidden=128,
                 obs_kind="bernoulli", obs_dim=784, pixel_p=0.13),
    # configs[3]: large-K deep chain, 8 layers of 32, K=2048, Gaussian(256, sigma 0.1) observation
    "C3": Config("C3", "mlp_chain", B=1024, K=2048, parent=_chain(8), D=[32] * 8, hidden=64,
                 obs_kind="gauss", obs_dim=256, obs_sigma=0.1),
    # configs[4]: tree 1 -> 4 -> 16 (21 latents, dim 32), K=512, leaves emit 64-dim Gaussians (sigma 0.2)
    "C4": Config("C4", "lg", B=256, K=512, parent=_tree_c4(), D=[32] * 21, w_var=1.0 / 32,
                 noise_var=0.3, observed=list(range(5, 21)), obs_dim=64, c_var=1.0 / 32,
                 obs_var=0.04, q="prior_marginal"),
    # the paper's MNIST model shapes (4, 8, 16, 32, 64 stochastic
    # units from the top layer to the layer next to the data; K = 20) on synthetic
    # Bernoulli(0.13) pixels, with this family's 1-hidden-layer tanh conditionals (the paper's
    # two leaky-relu deterministic layers and softplus stds are not reproduced: cost context only)
    "M5": Config("M5", "mlp_chain", B=128, K=20, parent=_chain(5), D=[4, 8, 16, 32, 64], hidden=64,
                 obs_kind="bernoulli", obs_dim=784, pixel_p=0.13),
    # the shared-parameter star of P:334-346 on toy 1: theta ~ N(0,1),
    # z_i | theta ~ N(theta, 1), x_i | z_i ~ N(z_i, 1), i = 1..N; proposals Q(theta) = N(0,1),
    # Q(z_i) = N(0,2).  One "datapoint" b is one whole data set of N points sharing theta
    # (B independent replicate data sets); latent 0 = theta, latents 1..N = z_i.
    "T1": Config("T1", "hier", B=8, K=1024, parent=_star(1024), D=[1] * 1025),
    "T1_paper": Config("T1_paper", "hier", B=8, K=128, parent=_star(128), D=[1] * 129),
    # ---- shrunk variants of every family (brute-force enumerable)
    "S_chain": Config("S_chain", "lg", B=4, K=3, parent=_chain(4), D=[2] * 4, w_var=0.5,
                      noise_var=0.5, observed=[3], obs_dim=4, obs_var=0.1, q="fixed", q_var=2.0),
    "S_tree": Config("S_tree", "lg", B=4, K=3, parent=[-1, 0, 0, 1, 1], D=[2, 3, 2, 2, 1],
                     w_var=0.5, noise_var=0.3, observed=[2, 3, 4], obs_dim=3, c_var=0.5,
                     obs_var=0.2, q="prior_marginal"),
    "S_hier": Config("S_hier", "hier", B=3, K=3, parent=_star(3), D=[1] * 4),
    "S_mnist": Config("S_mnist", "mnist", B=4, K=4, parent=[-1, 0], D=[3, 4], hidden=5,
                      enc_hidden=6, dec_hidden=6, obs_dim=16, pixel_p=0.13),
    "S_mlp": Config("S_mlp", "mlp_chain", B=4, K=3, parent=_chain(4), D=[3] * 4, hidden=4,
                    obs_kind="gauss", obs_dim=5, obs_sigma=0.5),
    "S_mlp_bern": Config("S_mlp_bern", "mlp_chain", B=3, K=4, parent=_chain(3), D=[2] * 3,
                         hidden=4, obs_kind="bernoulli", obs_dim=7, pixel_p=0.13),
}


def get_config(name: str, **overrides) -> Config:
    base = CONFIGS[name]
    if base.family == "hier" and ("N" in overrides or "children" in overrides):
        # N: data points in the set; children: the global ids a shard holds (star over them)
        N = overrides.pop("N", base.n - 1)
        ch = overrides.get("children")
        m = N if ch is None else len(ch)
        overrides.update(parent=_star(m), D=[1] * (m + 1))
        overrides.setdefault("obs_dim", N)
    cfg = dataclasses.replace(base, **overrides)
    if "K" in overrides or "parent" in overrides or "D" in overrides:
        cfg.name = f"{name}*"
    return cfg


# ----------------------------------------------------------------------------- workload
@dataclasses.dataclass
class Workload:
    cfg: Config
    b_ids: np.ndarray                # global datapoint ids
    z: List[np.ndarray]
    mu: List[np.ndarray]
    logvar: List[np.ndarray]
    logq: List[np.ndarray]
    logobs: List[Optional[np.ndarray]]
    x: List[np.ndarray]              # per-datapoint observations (model data), for closed forms
    params: dict                     # model parameters (shared across datapoints)

    @property
    def B(self) -> int:
        return len(self.b_ids)

    @property
    def parent(self) -> List[int]:
        return list(self.cfg.parent)

    @property
    def K(self) -> List[int]:
        return [self.cfg.K] * self.cfg.n

    @property
    def D(self) -> List[int]:
        return list(self.cfg.D)

    def Kp(self, i: int) -> int:
        return self.cfg.Kp(i)


def _gauss_logpdf(x, mean, var):
    """log N(x; mean, diag(var)) summed over the last axis, float64 (model density)."""
    x = np.asarray(x, np.float64)
    d = x - mean
    return -0.5 * np.sum(d * d / var + np.log(var) + LOG2PI, axis=-1)


def _glorot(rng, fan_in, fan_out):
    lim = math.sqrt(6.0 / (fan_in + fan_out))          # A13: Glorot-uniform, zero bias
    return rng.uniform(-lim, lim, size=(fan_in, fan_out))


def _mlp_init(rng, sizes):
    return [(_glorot(rng, a, b), np.zeros(b)) for a, b in zip(sizes[:-1], sizes[1:])]


def _mlp(layers, h):
    h = np.asarray(h, np.float64)
    for j, (W, bias) in enumerate(layers):
        h = h @ W + bias
        if j < len(layers) - 1:
            h = np.tanh(h)
    return h


def _log_bernoulli(x, logits):
    # log p(x|l) = x*l - softplus(l), summed over pixels
    sp = np.logaddexp(0.0, logits)
    return np.sum(x * logits - sp, axis=-1)


# --- parameters ---------------------------------------------------------------
def make_params(cfg: Config, seed: int = 0) -> dict:
    rng = rng_for(seed, "params")
    n, D = cfg.n, cfg.D
    p: dict = {}
    if cfg.family == "lg":
        p["W"] = [None] + [rng.normal(0.0, math.sqrt(cfg.w_var), size=(D[i], D[cfg.parent[i]]))
                           for i in range(1, n)]
        obs = cfg.observed or []
        p["C"] = {i: rng.normal(0.0, math.sqrt(cfg.c_var), size=(cfg.obs_dim, D[i])) for i in obs}
        # prior marginal covariances (used for x ancestral draws and the A8 proposal)
        S = [None] * n
        for i in range(n):
            if cfg.parent[i] < 0:
                S[i] = np.eye(D[i])
            else:
                W = p["W"][i]
                S[i] = W @ S[cfg.parent[i]] @ W.T + cfg.noise_var * np.eye(D[i])
        p["prior_cov"] = S
    elif cfg.family == "mlp_chain":
        H = cfg.hidden
        p["cond"] = [None] + [_mlp_init(rng, [D[cfg.parent[i]], H, 2 * D[i]]) for i in range(1, n)]
        p["dec"] = _mlp_init(rng, [D[n - 1], H, cfg.obs_dim])
        p["q_mu"] = [rng.normal(0.0, 1.0, size=D[i]) for i in range(n)]
        p["q_sigma"] = [np.exp(rng.uniform(-1.0, 0.0, size=D[i])) for i in range(n)]
    elif cfg.family == "mnist":
        d2, d1 = D[0], D[1]
        H = cfg.hidden
        p["p_z1"] = _mlp_init(rng, [d2, H, H, 2 * d1])                       # p(z1|z2)
        p["dec"] = _mlp_init(rng, [d1, cfg.dec_hidden, cfg.dec_hidden, cfg.obs_dim])  # p(x|z1)
        p["q_z1"] = _mlp_init(rng, [cfg.obs_dim, cfg.enc_hidden, cfg.enc_hidden, 2 * d1])  # q(z1|x)
        p["q_z2"] = _mlp_init(rng, [d1, H, H, 2 * d2])                       # q(z2|z1)
    elif cfg.family == "hier":
        pass                         # no learned parameters in toy 1
    else:
        raise ValueError(cfg.family)
    return p


# --- one datapoint --------------------------------------------------------------
def _datapoint(cfg: Config, p: dict, seed: int, b: int):
    n, D, K = cfg.n, cfg.D, cfg.K
    rd = rng_for(seed, "data", b)
    rq = rng_for(seed, "prop", b)
    f32 = np.float32
    z: list = [None] * n
    mu: list = [None] * n
    lv: list = [None] * n
    lq: list = [None] * n
    lo: list = [None] * n
    xs: list = []

    if cfg.family == "hier":
        # toy 1.  Every draw is keyed by (b, global data-point id) so a shard holding
        # data points `children` sees exactly the values of the full set.
        ids = list(range(cfg.n - 1)) if cfg.children is None else list(cfg.children)
        theta = rd.normal()
        xs = []
        for j, gi in enumerate(ids):
            r = rng_for(seed, "data", b, gi + 1)
            zi = theta + r.normal()
            xs.append(zi + r.normal())
        th = rq.normal(size=(K, 1))                                  # Q(theta) = N(0, 1)
        z[0] = th.astype(f32)
        lq[0] = _gauss_logpdf(z[0], 0.0, 1.0).astype(f32)
        mu[0] = np.zeros((1, 1), f32)                                # prior N(0, 1)
        lv[0] = np.zeros((1, 1), f32)
        for j, gi in enumerate(ids):
            i = j + 1
            r = rng_for(seed, "prop", b, gi + 1)
            z[i] = (math.sqrt(2.0) * r.normal(size=(K, 1))).astype(f32)   # Q(z_i) = N(0, 2)
            lq[i] = _gauss_logpdf(z[i], 0.0, 2.0).astype(f32)
            mu[i] = z[0].copy()                                      # p(z_i | theta^c) = N(theta^c, 1)
            lv[i] = np.zeros((K, 1), f32)
            lo[i] = _gauss_logpdf(np.full((K, 1), xs[j]), z[i].astype(np.float64), 1.0).astype(f32)
        xs = [np.asarray(xs)]

    elif cfg.family == "lg":
        # data: ancestral draw from the model
        zt = [None] * n
        for i in range(n):
            if cfg.parent[i] < 0:
                zt[i] = rd.normal(size=D[i])
            else:
                zt[i] = p["W"][i] @ zt[cfg.parent[i]] + math.sqrt(cfg.noise_var) * rd.normal(size=D[i])
        xo = {}
        for i in cfg.observed or []:
            xo[i] = p["C"][i] @ zt[i] + math.sqrt(cfg.obs_var) * rd.normal(size=cfg.obs_dim)
        xs = [xo[i] for i in sorted(xo)]
        # proposal samples
        for i in range(n):
            qv = (np.full(D[i], cfg.q_var) if cfg.q == "fixed" else np.diag(p["prior_cov"][i]).copy())
            z[i] = (np.sqrt(qv) * rq.normal(size=(K, D[i]))).astype(f32)
            lq[i] = _gauss_logpdf(z[i], 0.0, qv).astype(f32)
        for i in range(n):
            if cfg.parent[i] < 0:
                mu[i] = np.zeros((1, D[i]), f32)
                lv[i] = np.zeros((1, D[i]), f32)
            else:
                zp = z[cfg.parent[i]].astype(np.float64)
                mu[i] = (zp @ p["W"][i].T).astype(f32)
                lv[i] = np.full((K, D[i]), math.log(cfg.noise_var), f32)
            if i in xo:
                m = z[i].astype(np.float64) @ p["C"][i].T
                lo[i] = _gauss_logpdf(xo[i][None, :], m, cfg.obs_var).astype(f32)

    elif cfg.family == "mlp_chain":
        last = n - 1
        if cfg.obs_kind == "bernoulli":
            x = (rd.uniform(size=cfg.obs_dim) < cfg.pixel_p).astype(np.float64)
        else:
            zt = rd.normal(size=D[0])
            for i in range(1, n):
                o = _mlp(p["cond"][i], zt[None, :])[0]
                zt = o[:D[i]] + np.exp(0.5 * o[D[i]:]) * rd.normal(size=D[i])
            x = _mlp(p["dec"], zt[None, :])[0] + cfg.obs_sigma * rd.normal(size=cfg.obs_dim)
        xs = [x]
        for i in range(n):
            z[i] = (p["q_mu"][i] + p["q_sigma"][i] * rq.normal(size=(K, D[i]))).astype(f32)
            lq[i] = _gauss_logpdf(z[i], p["q_mu"][i], p["q_sigma"][i] ** 2).astype(f32)
        for i in range(n):
            if cfg.parent[i] < 0:
                mu[i] = np.zeros((1, D[i]), f32)
                lv[i] = np.zeros((1, D[i]), f32)
            else:
                o = _mlp(p["cond"][i], z[cfg.parent[i]])
                mu[i] = o[:, :D[i]].astype(f32)
                lv[i] = o[:, D[i]:].astype(f32)
        out = _mlp(p["dec"], z[last])
        if cfg.obs_kind == "bernoulli":
            lo[last] = _log_bernoulli(x[None, :], out).astype(f32)
        else:
            lo[last] = _gauss_logpdf(x[None, :], out, cfg.obs_sigma ** 2).astype(f32)

    elif cfg.family == "mnist":
        d2, d1 = D[0], D[1]
        x = (rd.uniform(size=cfg.obs_dim) < cfg.pixel_p).astype(np.float64)
        xs = [x]
        o = _mlp(p["q_z1"], x[None, :])[0]
        m1, v1 = o[:d1], np.exp(o[d1:])
        z1 = (m1 + np.sqrt(v1) * rq.normal(size=(K, d1))).astype(f32)
        lq1 = _gauss_logpdf(z1, m1, v1)
        o2 = _mlp(p["q_z2"], z1)                       # diagonal pairing: z2^k ~ q(z2 | z1^k) (A9)
        m2, v2 = o2[:, :d2], np.exp(o2[:, d2:])
        z2 = (m2 + np.sqrt(v2) * rq.normal(size=(K, d2))).astype(f32)
        lq2 = _gauss_logpdf(z2, m2, v2)
        z[0], z[1] = z2, z1
        lq[0], lq[1] = lq2.astype(f32), lq1.astype(f32)
        mu[0] = np.zeros((1, d2), f32)
        lv[0] = np.zeros((1, d2), f32)
        o3 = _mlp(p["p_z1"], z2)
        mu[1] = o3[:, :d1].astype(f32)
        lv[1] = o3[:, d1:].astype(f32)
        lo[1] = _log_bernoulli(x[None, :], _mlp(p["dec"], z1)).astype(f32)
    return z, mu, lv, lq, lo, xs


def make_workload(cfg, seed: int = 0, b_ids: Optional[Sequence[int]] = None,
                  threads: Optional[int] = None, **overrides) -> Workload:
    """Generate inputs for datapoints b_ids (default: all of cfg.B)."""
    if isinstance(cfg, str):
        cfg = get_config(cfg, **overrides)
    elif overrides:
        cfg = dataclasses.replace(cfg, **overrides)
    p = make_params(cfg, seed)
    if b_ids is None:
        b_ids = np.arange(cfg.B)
    b_ids = np.asarray(b_ids, dtype=np.int64)
    n = cfg.n
    B = len(b_ids)
    K = cfg.K
    z = [np.empty((B, K, cfg.D[i]), np.float32) for i in range(n)]
    mu = [np.empty((B, cfg.Kp(i), cfg.D[i]), np.float32) for i in range(n)]
    lv = [np.empty((B, cfg.Kp(i), cfg.D[i]), np.float32) for i in range(n)]
    lq = [np.empty((B, K), np.float32) for i in range(n)]
    probe = _datapoint(cfg, p, seed, int(b_ids[0])) if B else None
    lo = [None if (probe is None or probe[4][i] is None) else np.empty((B, K), np.float32)
          for i in range(n)]
    xs: list = [None] * B

    def fill(j):
        r = probe if j == 0 else _datapoint(cfg, p, seed, int(b_ids[j]))
        for i in range(n):
            z[i][j], mu[i][j], lv[i][j], lq[i][j] = r[0][i], r[1][i], r[2][i], r[3][i]
            if lo[i] is not None:
                lo[i][j] = r[4][i]
        xs[j] = r[5]

    nt = threads or min(32, os.cpu_count() or 1)
    if B * K * sum(cfg.D) < 200_000 or nt <= 1:
        for j in range(B):
            fill(j)
    else:
        with ThreadPoolExecutor(nt) as ex:
            list(ex.map(fill, range(B)))
    return Workload(cfg, b_ids, z, mu, lv, lq, lo, xs, p)
