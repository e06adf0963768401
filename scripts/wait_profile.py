"""Experiment: per-role barrier-wait breakdown of the forward / reverse kernels (libtmc_instr.so).
Slots: producer 0 ring-empty, 1 bias-ring-empty, 2 owned-tile-empty, 14 total;
MMA 3 ring-full, 4 acc/S-empty, 5 P-full, 6 owned-tile-full, 7 G-empty, 12 total;
softmax warp 2 lane 0: 8 acc/S-full, 9 bias-full, 10 G-full, 13 total."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TMC_LIB_PATH", os.path.join(ROOT, "paper_1806_08593_b200", "libtmc_instr.so"))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
wl = tw.make_workload(name, B=B)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
t = lambda a: None if a is None else torch.from_numpy(a).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
       for i in range(len(wl.parent))]
ws = tmc.alloc_workspace(g)
logp = torch.empty(wl.B, dtype=torch.float64, device="cuda")
grads = tmc.alloc_grads(g)
lib = tmc.load_library()
lib.tmc_debug_counters.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros((1024, 64), np.uint64)   # g_tmc_prof is [1024][64]
def counters(clear=1):
    torch.cuda.synchronize()
    assert lib.tmc_debug_counters(buf.ctypes.data, buf.size, clear) == 0
    return buf[:148].astype(np.float64).mean(0)
s = torch.cuda.current_stream()
tmc.tmc_forward(g, inp, logp, ws, None, s); tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
counters()
names = {0: "prod.ring_empty", 1: "prod.bias_empty", 2: "prod.own_empty", 14: "prod.total",
         3: "mma.ring_full", 4: "mma.acc_empty", 5: "mma.P_full", 6: "mma.own_full", 7: "mma.G_empty", 12: "mma.total",
         11: "mma.issue_grad", 15: "mma.issue_S", 16: "mma.commit_grad", 17: "mma.fence", 18: "mma.commit_S",
         8: "smx.acc_full", 9: "smx.bias_full", 10: "epi.G_full", 13: "smx.total",
         32: "bwd.smx0.S_full", 33: "bwd.smx1.S_full", 48: "bwd.smx0.total", 49: "bwd.smx1.total"}
for phase in ("fwd", "bwd"):
    if phase == "fwd":
        tmc.tmc_forward(g, inp, logp, ws, None, s)
    else:
        tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
    c = counters()
    out = {"phase": phase, "cfg": name, "B": B}
    for k, v in names.items():
        out[v] = round(v_ := c[k] / 1e6, 3)
    print(json.dumps(out), flush=True)
