"""Experiment: parity of the reverse pass under each TMC_BWD_GRAD_TERMS variant vs the oracle."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, tmc_workload as tw
import paper_1806_08593_b200 as tmc

variants = [int(v) for v in (sys.argv[1:] or ["3", "4", "5", "1"])]
cases = [("C3", dict(B=4)), ("C4", dict(B=4)), ("C2", dict(B=4)), ("C3", dict(B=3, K=300)), ("C1", dict(B=8))]
for name, kw in cases:
    wl = tw.make_workload(name, **kw)
    ref = oracle.estimate_workload(wl)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
    t = lambda a: None if a is None else torch.from_numpy(a).cuda()
    inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
           for i in range(len(wl.parent))]
    for gt in variants:
        os.environ["TMC_BWD_GRAD_TERMS"] = str(gt)
        logp, gr = tmc.estimate(g, inp)
        torch.cuda.synchronize()
        worst = {}
        for k in ("dz", "dmu", "dlogvar", "dlogq"):
            w = 0.0
            for i in range(len(wl.parent)):
                got = gr[i][k].cpu().numpy().astype(np.float64); want = ref[k][i]
                for b in range(wl.B):
                    nw = np.linalg.norm(want[b])
                    if nw > 1e-12:
                        w = max(w, np.linalg.norm(got[b] - want[b]) / nw)
            worst[k] = w
        print(json.dumps({"cfg": name, **kw, "gt": gt, "dlogp": float(np.abs(logp.cpu().numpy() - ref["logp"]).max()),
                          **{k: float(f"{v:.3e}") for k, v in worst.items()}}), flush=True)
