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

Supported families: "mlp_chain" (C2, C3) and "lg" (C0, C4).
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
        if cfg.family not in ("mlp_chain", "lg"):
            raise ValueError(f"torch harness supports mlp_chain / lg families, not {cfg.family}")
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
        else:
            self.W = [None] + [P(p["W"][i]) for i in range(1, n)]
            self.C = {i: P(c) for i, c in p["C"].items()}
            # lg proposals are fixed (q_var or the prior marginal): z is data here
            self.z_fixed = [t(wl.z[i]) for i in range(n)]
            self.logq_fixed = [t(wl.logq[i]) for i in range(n)]
            self.x = {i: t(np.stack([xs[k] for xs in wl.x])) for k, i in enumerate(sorted(p["C"]))}
        self.grad_numel = sum(x.numel() for x in self.params)

    @staticmethod
    def _mlp(layers, h):
        import torch
        for j, (W, b) in enumerate(layers):
            h = h @ W + b
            if j < len(layers) - 1:
                h = torch.tanh(h)
        return h

    def forward(self) -> Dict[str, list]:
        """z, mu, logvar, logq, logobs per latent (ABI layout, fp32, contiguous) with autograd."""
        torch = self.torch
        cfg = self.cfg
        n, D, K = cfg.n, cfg.D, cfg.K
        B = self.x.shape[0] if not isinstance(self.x, dict) else next(iter(self.x.values())).shape[0]
        z, mu, lv, lq, lo = [None] * n, [None] * n, [None] * n, [None] * n, [None] * n
        if cfg.family == "mlp_chain":
            for i in range(n):
                sig = torch.exp(self.q_logsig[i])
                z[i] = self.q_mu[i] + sig * self.eps[i]
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

    def flat_grads(self):
        torch = self.torch
        return torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).reshape(-1) for p in self.params])

    def zero_grad(self):
        for p in self.params:
            p.grad = None
