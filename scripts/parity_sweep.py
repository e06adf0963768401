"""Randomised parity sweep (not a test): many seeds and ragged shapes, worst |dlogp| and worst
per-datapoint gradient relative error against the oracle."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, tmc_workload as tw
from test_gpu_parity import run_gpu, rel_err, max_err

cases = [("C3", dict(B=3, K=300)), ("C3", dict(B=2, K=700)), ("C4", dict(B=2, K=260)), ("C2", dict(B=3, K=300)),
         ("C1", dict(B=8)), ("S_hier", dict(N=6, K=200, B=2)), ("S_tree", dict(B=2, K=150, D=[8, 20, 33, 5, 40], w_var=0.03, c_var=0.03))]
nseeds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
worst = {}
for name, kw in cases:
    for seed in range(1, nseeds + 1):
        wl = tw.make_workload(name, seed=seed, **kw)
        got = run_gpu(torch, wl)
        ref = oracle.estimate_workload(wl)
        dl = float(np.abs(got["logp"] - ref["logp"]).max())
        ge, gm = 0.0, 0.0
        for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
            for i in range(len(wl.parent)):
                ge = max(ge, rel_err(got[k][i], ref[k][i]))
                gm = max(gm, max_err(got[k][i], ref[k][i]))
        key = f"{name}{kw}"
        w = worst.setdefault(key, [0.0, 0.0, 0.0])
        w[0] = max(w[0], dl); w[1] = max(w[1], ge); w[2] = max(w[2], gm)
        print(json.dumps({"case": key, "seed": seed, "dlogp": dl, "grad_rel_l2": ge, "grad_elementwise": gm}), flush=True)
print(json.dumps({"worst": worst}))
