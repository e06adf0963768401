"""Diagnostic: signed logp error of the SIMT and tensor-core paths vs the oracle (sampled datapoints)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, tmc_workload as tw
import paper_1806_08593_b200 as tmc

def run(wl, prec, direction=0):
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, precision=prec, direction=direction)
    t = lambda a: None if a is None else torch.from_numpy(a).cuda()
    inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i])) for i in range(len(wl.parent))]
    logp, _ = tmc.estimate(g, inp, grads=False)
    return logp.cpu().numpy()

for name, kw in [("C4", dict(B=16)), ("C3", dict(B=8)), ("C2", dict(B=16))]:
    wl = tw.make_workload(name, **kw)
    ref = oracle.estimate_workload(wl, grads=False)["logp"]
    for prec in (1, 2):
        e = run(wl, prec) - ref
        print(name, "SIMT" if prec == 1 else "TC  ", "mean %+.2e  max|.| %.2e" % (e.mean(), np.abs(e).max()), np.array2string(e[:8], precision=1))
