"""One-rank T1 (toy-1 star, NEXT-2) steps for profiling: python scripts/t1_step.py [steps] [N] [K]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc
from paper_1806_08593_b200 import parallel as par

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
K = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
wl = tw.make_workload("T1", N=N, K=K)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, direction=tmc.TMC_DIR_UP)
t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
       for i in range(len(wl.parent))]
ws = tmc.alloc_workspace(g)
logp = torch.empty(g.B, dtype=torch.float64, device="cuda")
msg = torch.empty(g.B, K + 1, dtype=torch.float64, device="cuda")
gr = tmc.alloc_grads(g)
for _ in range(steps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    tmc.tmc_forward_children(g, inp, msg, ws)
    e[1].record()
    tmc.tmc_forward_root(g, inp, msg, logp, ws)
    e[2].record()
    tmc.tmc_backward(g, inp, ws, None, gr)
    e[3].record()
    torch.cuda.synchronize()
    print("children %.2f ms  root %.2f ms  backward %.2f ms" % (e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])), flush=True)
