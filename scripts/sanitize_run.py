"""Small shapes on every kernel family, for compute-sanitizer:
small-problem kernel, SIMT passes (level-batched, D <= 4), tensor-core fwd/bwd (D = 32, 64, padded),
exchange, IWAE, sampler, host-streamed estimate."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc

def up(wl):
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
            for i in range(len(wl.parent))]

cases = [("C0", {}, 0), ("S_tree", {}, 1), ("C3", dict(B=2, K=260), 0), ("C2", dict(B=1, K=130), 0),
         ("C4", dict(B=1, K=130), 0), ("S_hier", dict(N=3, K=140, B=1), 0), ("C3", dict(B=1, K=40, D=[5] * 8), 2)]
for name, kw, prec in cases:
    wl = tw.make_workload(name, **kw)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, precision=prec)
    logp, gr = tmc.estimate(g, up(wl), pair=max(wl.K) <= 300)
    torch.cuda.synchronize()
    print(name, kw, "ok", float(logp.sum()), flush=True)
wl = tw.make_workload("C3", B=2, K=64)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
lp, _ = tmc.iwae(g, up(wl)); torch.cuda.synchronize(); print("iwae ok", flush=True)
e = torch.empty(2, 33, 5, device="cuda"); tmc.tmc_sample_normal(1, 4, 0, 0, e); torch.cuda.synchronize(); print("sampler ok")
