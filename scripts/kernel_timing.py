"""Experiment driver: time tmc_forward / tmc_backward on one config under several env settings
(TMC_DEBUG_FLAGS, TMC_BWD_GRAD_TERMS) in one process.  Prints one JSON line per setting."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
settings = sys.argv[3:] or ["0:3"]
wl = tw.make_workload(cfg_name, B=B)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
t = lambda a: None if a is None else torch.from_numpy(a).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
       for i in range(len(wl.parent))]
ws = tmc.alloc_workspace(g)
logp = torch.empty(wl.B, dtype=torch.float64, device="cuda")
grads = tmc.alloc_grads(g)
s = torch.cuda.current_stream()
pairs = B * sum(wl.K[i] * wl.Kp(i) for i in range(len(wl.parent)) if wl.parent[i] >= 0)
for st in settings:
    parts = st.split(":") + [""] * 3
    flags, gt, poly = parts[0] or "0", parts[1] or "3", parts[2]
    os.environ["TMC_DEBUG_FLAGS"] = flags
    os.environ["TMC_BWD_GRAD_TERMS"] = gt
    if poly:
        os.environ["TMC_FWD_VARIANT"] = poly
    else:                                   # the library default
        os.environ.pop("TMC_FWD_VARIANT", None)
        poly = "-1"
    for _ in range(2):
        tmc.tmc_forward(g, inp, logp, ws, None, s); tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
    torch.cuda.synchronize()
    n = 5
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(s)
    for _ in range(n):
        tmc.tmc_forward(g, inp, logp, ws, None, s)
    e[1].record(s)
    for _ in range(n):
        tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
    e[2].record(s)
    torch.cuda.synchronize()
    fwd, bwd = e[0].elapsed_time(e[1]) / n, e[1].elapsed_time(e[2]) / n
    print(json.dumps({"cfg": cfg_name, "B": B, "flags": int(flags), "grad_terms": int(gt), "fwd_variant": int(poly), "fwd_ms": fwd, "bwd_ms": bwd,
                      "fwd_pairs_per_clk_sm": pairs / (fwd * 1e-3) / 148 / 1.965e9}), flush=True)
