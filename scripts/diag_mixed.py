import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, tmc_workload as tw
from test_gpu_parity import run_gpu
for D in ([32, 64, 32, 48, 64], [32] * 5, [64] * 5, [32, 32, 32, 48, 32], [48] * 5):
    for K in (200, 128):
        wl = tw.make_workload("S_tree", B=2, K=K, D=D)
        ref = oracle.estimate_workload(wl)
        for prec in (1, 2, 0):
            for dirn in (0,):
                try:
                    got = run_gpu(torch, wl, precision=prec, direction=dirn)
                    print(D, K, "prec", prec, "dlogp", np.abs(got["logp"] - ref["logp"]).max(), "logp", ref["logp"], flush=True)
                except Exception as e:
                    print(D, K, "prec", prec, "ERR", str(e)[:100], flush=True)
