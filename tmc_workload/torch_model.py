"""Differentiable torch copy of a workload's *model* (harness only).

The TMC estimator (paper_1806_08593_b200, the product) takes the per-sample conditionals as
inputs.  A training step also needs the model around it: the reparameterised proposal samples
z_i = mu_q + sigma_q * eps, the conditional networks that give mu_i, logvar_i of
p(z_i | z_pa) at every parent sample (random-init tanh MLPs / linear maps), the proposal
and observation log-densities, and - after the TMC reverse pass - the chain rule into the shared
parameters, whose gradients are then all-reduced across ranks (§8e).  This module is that harness:
plain torch (cuBLAS GEMMs) on the caller's device, built from the same parameters and noise as
tmc_workload, so a bench "full step" can time model forward -> TMC -> model backward -> allreduce.
It holds none of the TMC method's arithmetic (no factor, message, logsumexp or TMC gradient).

Supported families: "mlp_chain" (C2, C3, M5), "lg" (C0, C4) and "mnist" (C1: amortised
q(z1 | x), non-factorised q(z2 | z1^k) with diagonal pairing, A9).
"""
from __future__ import annotations

import math
from typing import Dict, List

import numpy as np

LOG2PI = math.log(2.0 * math.pi)


class TorchModel:
    def __init__(self, wl, device, dtype=None):
        import torch
        self.torch = torch
        cfg = wl.cfg
        if cfg.family not in ("mlp_chain", "lg", "mnist"):
            raise ValueError(f"torch harness supports mlp_chain / lg / mnist families, not {cfg.family}")
        self.cfg, self.device = cfg, device
        dt = dtype or torch.float32
        t = lambda a: torch.tensor(np.asarray(a), dtype=dt, device=device)
        p = wl.params
        self.params: List = []

        def P(a):
            x = t(a).requires_grad_(True)
            self.params.append(x)
            return x

        n, D = cfg.n, cfg.D
        if cfg.family == "mlp_chain":
            self.q_mu = [P(p["q_mu"][i]) for i in range(n)]
            self.q_logsig = [P(np.log(p["q_sigma"][i])) for i in range(n)]
            self.cond = [None] + [[(P(W), P(b)) for W, b in p["cond"][i]] for i in range(1, n)]
            self.dec = [(P(W), P(b)) for W, b in p["dec"]]
            # noise: eps = (z - mu_q) / sigma_q reproduces tmc_workload's samples
            self.eps = [t((wl.z[i].astype(np.float64) - p["q_mu"][i]) / p["q_sigma"][i]) for i in range(n)]
            self.x = t(np.stack([xs[0] for xs in wl.x]))
        elif cfg.family == "mnist":
            # latent 0 = z2 (top, prior N(0, I)), latent 1 = z1 (next to the data)
            d2, d1 = D[0], D[1]
            self.q_z1 = [(P(W), P(b)) for W, b in p["q_z1"]]
            self.q_z2 = [(P(W), P(b)) for W, b in p["q_z2"]]
            self.p_z1 = [(P(W), P(b)) for W, b in p["p_z1"]]
            self.dec = [(P(W), P(b)) for W, b in p["dec"]]
            self.x = t(np.stack([xs[0] for xs in wl.x]))
            # noise that reproduces tmc_workload's samples: eps = (z - m_q) / s_q
            f64 = lambda a: np.asarray(a, np.float64)
            from tmc_workload import _mlp as mlp64
            e1, e2 = [], []
            for j in range(len(wl.b_ids)):
                o = mlp64(p["q_z1"], f64(wl.x[j][0])[None, :])[0]
                m1, s1 = o[:d1], np.exp(0.5 * o[d1:])
                e1.append((f64(wl.z[1][j]) - m1) / s1)
                o2 = mlp64(p["q_z2"], f64(wl.z[1][j]))
                e2.append((f64(wl.z[0][j]) - o2[:, :d2]) / np.exp(0.5 * o2[:, d2:]))
            self.eps = [t(np.stack(e2)), t(np.stack(e1))]
        else:
            self.W = [None] + [P(p["W"][i]) for i in range(1, n)]
            self.C = {i: P(c) for i, c in p["C"].items()}
            # lg proposals are fixed (q_var or the prior marginal): z is data here
            self.z_fixed = [t(wl.z[i]) for i in range(n)]
            self.logq_fixed = [t(wl.logq[i]) for i in range(n)]
            self.x = {i: t(np.stack([xs[k] for xs in wl.x])) for k, i in enumerate(sorted(p["C"]))}
        self.grad_numel = sum(x.numel() for x in self.params)
        self.b0 = int(wl.b_ids[0]) if len(wl.b_ids) else 0
        if len(wl.b_ids) and not np.array_equal(wl.b_ids, np.arange(self.b0, self.b0 + len(wl.b_ids))):
            self.b0 = None                    # device noise needs a contiguous block of global ids

    def fresh_noise(self, seed: int) -> None:
        """Redraw the reparameterisation noise on the device with libtmc's
        counter-based sampler: eps_i[b,k,:] is keyed by (seed, tag eps, global datapoint b,
        latent i, k), so every rank draws its own shard's noise and a datapoint's noise does not
        depend on the world size.  A training step calls this with a new seed each step."""
        import paper_1806_08593_b200 as tmc
        if self.cfg.family not in ("mlp_chain", "mnist"):
            return                            # lg proposals are fixed samples (no reparameterisation)
        if self.b0 is None:
            raise ValueError("fresh_noise needs contiguous global datapoint ids")
        for i, e in enumerate(self.eps):
            tmc.tmc_sample_normal(seed, tmc.TAG_EPS, self.b0, i, e)

    @staticmethod
    def _mlp(layers, h):
        import torch
        for j, (W, b) in enumerate(layers):
            h = h @ W + b
            if j < len(layers) - 1:
                h = torch.tanh(h)
        return h

    def forward(self, stl: bool = False) -> Dict[str, list]:
        """z, mu, logvar, logq, logobs per latent (ABI layout, fp32, contiguous) with autograd.

        stl: "sticking the landing": log q is evaluated with the proposal parameters
        detached, so its gradient reaches them only through the reparameterised samples z."""
        torch = self.torch
        cfg = self.cfg
        n, D, K = cfg.n, cfg.D, cfg.K
        B = self.x.shape[0] if not isinstance(self.x, dict) else next(iter(self.x.values())).shape[0]
        z, mu, lv, lq, lo = [None] * n, [None] * n, [None] * n, [None] * n, [None] * n
        if cfg.family == "mlp_chain":
            for i in range(n):
                sig = torch.exp(self.q_logsig[i])
                z[i] = self.q_mu[i] + sig * self.eps[i]
                if stl:
                    m_d, ls_d = self.q_mu[i].detach(), self.q_logsig[i].detach()
                    e = (z[i] - m_d) * torch.exp(-ls_d)
                    lq[i] = (-0.5 * e ** 2 - ls_d - 0.5 * LOG2PI).sum(-1)
                else:
                    lq[i] = (-0.5 * self.eps[i] ** 2 - self.q_logsig[i] - 0.5 * LOG2PI).sum(-1)
            for i in range(n):
                if cfg.parent[i] < 0:
                    mu[i] = torch.zeros(B, 1, D[i], device=self.device)
                    lv[i] = torch.zeros(B, 1, D[i], device=self.device)
                else:
                    o = self._mlp(self.cond[i], z[cfg.parent[i]])
                    mu[i], lv[i] = o[..., :D[i]], o[..., D[i]:]
            out = self._mlp(self.dec, z[n - 1])
            xb = self.x[:, None, :]
            if cfg.obs_kind == "bernoulli":
                lo[n - 1] = (xb * out - torch.nn.functional.softplus(out)).sum(-1)
            else:
                var = cfg.obs_sigma ** 2
                lo[n - 1] = (-0.5 * ((xb - out) ** 2 / var + math.log(var) + LOG2PI)).sum(-1)
        elif cfg.family == "mnist":
            d2, d1 = D[0], D[1]

            def gauss(zv, m, lv, detach):
                if detach:
                    m, lv = m.detach(), lv.detach()
                return (-0.5 * ((zv - m) ** 2 * torch.exp(-lv) + lv + LOG2PI)).sum(-1)
            o = self._mlp(self.q_z1, self.x)                          # [B, 2 d1]
            m1, lv1 = o[:, None, :d1], o[:, None, d1:]
            z1 = m1 + torch.exp(0.5 * lv1) * self.eps[1]
            o2 = self._mlp(self.q_z2, z1)                             # diagonal pairing (A9)
            m2, lv2 = o2[..., :d2], o2[..., d2:]
            z2 = m2 + torch.exp(0.5 * lv2) * self.eps[0]
            z[0], z[1] = z2, z1
            lq[1] = gauss(z1, m1, lv1, stl)
            lq[0] = gauss(z2, m2, lv2, stl)
            mu[0] = torch.zeros(B, 1, d2, device=self.device)
            lv[0] = torch.zeros(B, 1, d2, device=self.device)
            o3 = self._mlp(self.p_z1, z2)
            mu[1], lv[1] = o3[..., :d1], o3[..., d1:]
            logits = self._mlp(self.dec, z1)
            lo[1] = (self.x[:, None, :] * logits - torch.nn.functional.softplus(logits)).sum(-1)
        else:
            for i in range(n):
                z[i] = self.z_fixed[i]
                lq[i] = self.logq_fixed[i]
                if cfg.parent[i] < 0:
                    mu[i] = torch.zeros(B, 1, D[i], device=self.device)
                    lv[i] = torch.zeros(B, 1, D[i], device=self.device)
                else:
                    mu[i] = z[cfg.parent[i]] @ self.W[i].T
                    lv[i] = torch.full((B, K, D[i]), math.log(cfg.noise_var), device=self.device)
                if i in self.C:
                    m = z[i] @ self.C[i].T
                    xb = self.x[i][:, None, :]
                    lo[i] = (-0.5 * ((xb - m) ** 2 / cfg.obs_var + math.log(cfg.obs_var) + LOG2PI)).sum(-1)
        cont = lambda a: None if a is None else a.contiguous()
        return {"z": [cont(a) for a in z], "mu": [cont(a) for a in mu], "logvar": [cont(a) for a in lv],
                "logq": [cont(a) for a in lq], "logobs": [cont(a) for a in lo]}

    def backward(self, fwd: Dict[str, list], grads: List[Dict]) -> None:
        """Chain rule of the TMC input gradients into the parameters (accumulates .grad)."""
        torch = self.torch
        outs, gouts = [], []
        key = {"z": "dz", "mu": "dmu", "logvar": "dlogvar", "logq": "dlogq", "logobs": "dlogobs"}
        for k, gk in key.items():
            for i, a in enumerate(fwd[k]):
                if a is not None and a.requires_grad and grads[i].get(gk) is not None:
                    outs.append(a)
                    gouts.append(grads[i][gk])
        torch.autograd.backward(outs, gouts)

    def proposal_params(self):
        """The recognition (proposal) parameters phi; everything else is generative (theta)."""
        if self.cfg.family == "mlp_chain":
            return list(self.q_mu) + list(self.q_logsig)
        if self.cfg.family == "mnist":
            return [x for W, b in self.q_z1 + self.q_z2 for x in (W, b)]
        return []

    def generative_params(self):
        ph = {id(p) for p in self.proposal_params()}
        return [p for p in self.params if id(p) not in ph]

    def log_weights_bruteforce(self, b: int):
        """log w for every index tuple of datapoint b (tiny instances only; test oracle of the
        DReGs gradient): sum_i log p(z_i | z_pa) - log q(z_i) + log p(x | z), differentiable."""
        import itertools
        torch = self.torch
        cfg = self.cfg
        f = self.forward(stl=True)
        n = cfg.n
        out = []
        for k in itertools.product(*[range(cfg.K) for _ in range(n)]):
            s = 0.0
            for i in range(n):
                zi = f["z"][i][b, k[i]]
                r = 0 if cfg.parent[i] < 0 else k[cfg.parent[i]]
                mu, lv = f["mu"][i][b, r], f["logvar"][i][b, r]
                s = s + (-0.5 * ((zi - mu) ** 2 * torch.exp(-lv) + lv + LOG2PI)).sum() - f["logq"][i][b, k[i]]
                if f["logobs"][i] is not None:
                    s = s + f["logobs"][i][b, k[i]]
            out.append(s)
        return torch.stack(out)

    def flat_grads(self):
        torch = self.torch
        return torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).reshape(-1) for p in self.params])

    def zero_grad(self):
        for p in self.params:
            p.grad = None


def dregs_step(model: TorchModel, direction: int = 0, precision: int = 0):
    """One TMC-DReGs gradient evaluation through libtmc, on the model's device.

    Generative parameters theta get the usual TMC gradient of sum_b L1[b] (alpha = 1).  Recognition
    parameters phi get the DReGs update sum_i w_i^2/(sum w)^2 dz_i/dphi dlog w_i/dz_i, computed from
    the surrogate 1/2 (sum w^2/(sum w)^2) log sum w_hat^2: a second TMC run with squared weights
    (factor_power = 2) gives L2 = log((1/prod K) sum w^2) and its input gradients, which are scaled
    per datapoint by dlogp = 1/2 exp(L2 - 2 L1 - sum_i ln K_i) and pushed into phi through the
    reparameterised samples only (STL form of log q: w_hat drops the direct phi term).
    Returns (L1, L2, {param: grad}).
    """
    import paper_1806_08593_b200 as tmc
    torch = model.torch
    cfg = model.cfg
    n = cfg.n
    f = model.forward(stl=True)
    inp = [dict(z=f["z"][i].detach(), mu=f["mu"][i].detach(), logvar=f["logvar"][i].detach(),
                logq=f["logq"][i].detach(), logobs=None if f["logobs"][i] is None else f["logobs"][i].detach())
           for i in range(n)]
    B = inp[0]["z"].shape[0]
    K = [cfg.K] * n

    def outs_and_grads(grads):
        outs, gouts = [], []
        for k, gk in (("z", "dz"), ("mu", "dmu"), ("logvar", "dlogvar"), ("logq", "dlogq"), ("logobs", "dlogobs")):
            for i, a in enumerate(f[k]):
                if a is not None and a.requires_grad and grads[i].get(gk) is not None:
                    outs.append(a)
                    gouts.append(grads[i][gk])
        return outs, gouts

    g1 = tmc.Graph(cfg.parent, K, cfg.D, B, direction=direction, precision=precision, factor_power=1.0)
    L1, gr1 = tmc.estimate(g1, inp)
    g2 = tmc.Graph(cfg.parent, K, cfg.D, B, direction=direction, precision=precision, factor_power=2.0)
    ws2 = tmc.alloc_workspace(g2, inp[0]["z"].device)
    L2 = torch.empty(B, dtype=torch.float64, device=inp[0]["z"].device)
    tmc.tmc_forward(g2, inp, L2, ws2)
    lnK = sum(math.log(k) for k in K)
    dlogp2 = 0.5 * torch.exp(L2 - 2.0 * L1 - lnK)
    gr2 = tmc.alloc_grads(g2, inp[0]["z"].device)
    tmc.tmc_backward(g2, inp, ws2, dlogp2, gr2)
    theta, phi = model.generative_params(), model.proposal_params()
    o1, go1 = outs_and_grads(gr1)
    gt = torch.autograd.grad(o1, theta, go1, retain_graph=True, allow_unused=True)
    o2, go2 = outs_and_grads(gr2)
    gp = torch.autograd.grad(o2, phi, go2, allow_unused=True) if phi else []
    res = {}
    for p_, g_ in list(zip(theta, gt)) + list(zip(phi, gp)):
        res[p_] = torch.zeros_like(p_) if g_ is None else g_
    return L1, L2, res


def train_step(model: TorchModel, graph, ws, logp, grads, flat64, seed: int, group=None, stream=None):
    """One data-parallel training step of the TMC objective on this rank's shard (SURVEY §8a rows
    a1-a8; §8e): fresh reparameterisation noise (libtmc tmc_sample_normal, keyed by global datapoint
    id) -> the model's conditionals and log-densities (torch/cuBLAS) -> libtmc tmc_estimate (forward
    + reverse pass) -> the chain rule into the parameters -> ONE fp64 SUM all-reduce of
    [objective | every shared-parameter gradient] (flat64 has model.grad_numel + 1 entries).
    Returns flat64: entry 0 = sum_b logp[b] over all ranks, then the summed parameter gradients."""
    import paper_1806_08593_b200 as tmc
    from paper_1806_08593_b200 import parallel
    torch = model.torch
    n = model.cfg.n
    model.zero_grad()
    model.fresh_noise(seed)
    f = model.forward()
    fin = [dict(z=f["z"][i].detach(), mu=f["mu"][i].detach(), logvar=f["logvar"][i].detach(),
                logq=f["logq"][i].detach(), logobs=None if f["logobs"][i] is None else f["logobs"][i].detach())
           for i in range(n)]
    tmc.tmc_estimate(graph, fin, logp, None, grads, ws, stream)
    model.backward(f, grads)
    torch.sum(logp, dim=0, keepdim=True, out=flat64[:1])
    flat64[1:].copy_(model.flat_grads())
    return parallel.reduce_objective(flat64, group)
