"""Experiment: phase breakdown of the small-problem kernel (libtmc_instr.so), cycles per CTA (mean)."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TMC_LIB_PATH", os.path.join(ROOT, "paper_1806_08593_b200", "libtmc_instr.so"))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc
name = sys.argv[1] if len(sys.argv) > 1 else "C0"
wl = tw.make_workload(name)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
t = lambda a: None if a is None else torch.from_numpy(a).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
       for i in range(len(wl.parent))]
ws = tmc.alloc_workspace(g)
logp = torch.empty(wl.B, dtype=torch.float64, device="cuda")
grads = tmc.alloc_grads(g)
lib = tmc.load_library()
lib.tmc_debug_counters.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros((1024, 64), np.uint64)
for _ in range(5):
    tmc.tmc_estimate(g, inp, logp, None, grads, ws)
torch.cuda.synchronize()
lib.tmc_debug_counters(buf.ctypes.data, buf.size, 1)
R = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(R):
    tmc.tmc_estimate(g, inp, logp, None, grads, ws)
e1.record()
torch.cuda.synchronize()
lib.tmc_debug_counters(buf.ctypes.data, buf.size, 1)
c = buf[:wl.B, 50:60].astype(np.float64).mean(0) / R
names = ["issue_loads", "wait_loads", "ldet_h_lam", "fwd_factor", "fwd_lse_h", "bwd_factor", "bwd_P", "bwd_rowsum",
         "bwd_grads", "bwd_sync"]
print(json.dumps({"cfg": name, "us_per_call": e0.elapsed_time(e1) * 1000 / R,
                  **{n: round(v) for n, v in zip(names, c)}, "total_clk": round(c.sum())}))
