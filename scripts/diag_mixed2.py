import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, tmc_workload as tw
from test_gpu_parity import run_gpu
for D, wv in (([64] * 5, 1 / 64), ([32, 64, 32, 48, 64], 1 / 64), ([64] * 5, 0.5), ([64] * 5, 0.1), ([64] * 5, 0.03)):
    wl = tw.make_workload("S_tree", B=2, K=200, D=D, w_var=wv, c_var=wv)
    ref = oracle.estimate_workload(wl)
    lo = [None if x is None else (float(x.min()), float(x.max())) for x in wl.logobs]
    zr = [float(np.abs(x).max()) for x in wl.z]
    print(D, wv, "logp", ref["logp"], "max|z|", [round(v, 1) for v in zr], flush=True)
    for prec in (1, 2):
        try:
            got = run_gpu(torch, wl, precision=prec)
            print("   prec", prec, "dlogp", np.abs(got["logp"] - ref["logp"]).max(), flush=True)
        except Exception as e:
            print("   prec", prec, "ERR", str(e)[:100], flush=True)
