"""Per-call device time of tmc_forward / tmc_backward on a small config (CUDA events, many calls)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc
for name in sys.argv[1:] or ["C0", "C1"]:
    wl = tw.make_workload(name)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i])) for i in range(len(wl.parent))]
    ws = tmc.alloc_workspace(g); logp = torch.empty(wl.B, dtype=torch.float64, device="cuda"); gr = tmc.alloc_grads(g)
    for _ in range(5):
        tmc.tmc_forward(g, inp, logp, ws); tmc.tmc_backward(g, inp, ws, None, gr)
    n = 200
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize(); e[0].record()
    for _ in range(n): tmc.tmc_forward(g, inp, logp, ws)
    e[1].record()
    for _ in range(n): tmc.tmc_backward(g, inp, ws, None, gr)
    e[2].record(); torch.cuda.synchronize()
    print(name, "fwd us %.1f  bwd us %.1f" % (1000 * e[0].elapsed_time(e[1]) / n, 1000 * e[1].elapsed_time(e[2]) / n), flush=True)
