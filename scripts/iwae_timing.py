import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
wl = tw.make_workload(name, B=B)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i])) for i in range(len(wl.parent))]
logp = torch.empty(wl.B, dtype=torch.float64, device="cuda"); gr = tmc.alloc_grads(g)
ws = torch.empty(tmc.load_library().tmc_iwae_workspace_size(g.ref()), dtype=torch.uint8, device="cuda")
for _ in range(3): tmc.tmc_iwae(g, inp, logp, None, gr, ws)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(10): tmc.tmc_iwae(g, inp, logp, None, gr, ws)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
nbytes = sum(2 * (x["z"].numel() + x["mu"].numel() + x["logvar"].numel()) * 4 + 3 * x["z"].numel() * 4 for x in inp)
print(name, B, "iwae ms %.3f  approx GB/s %.0f" % (ms, nbytes / ms / 1e6))
