"""Experiment: per-role wait breakdown of the single-pass reverse kernel (libtmc_instr.so, -DTMC_INSTRUMENT).
Per-CTA cycles (mean over CTAs, millions) for each barrier wait, and each role's total."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TMC_LIB_PATH", os.path.join(ROOT, "paper_1806_08593_b200", "libtmc_instr.so"))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 296
wl = tw.make_workload(name, B=B)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, flags=tmc.TMC_FLAG_SINGLE_PASS_REVERSE)
t = lambda a: None if a is None else torch.from_numpy(a).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
       for i in range(len(wl.parent))]
ws = tmc.alloc_workspace(g)
logp = torch.empty(wl.B, dtype=torch.float64, device="cuda")
grads = tmc.alloc_grads(g)
lib = tmc.load_library()
lib.tmc_debug_counters.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros((1024, 64), np.uint64)
def counters(clear=1):
    torch.cuda.synchronize()
    assert lib.tmc_debug_counters(buf.ctypes.data, buf.size, clear) == 0
    return buf[:148].astype(np.float64).mean(0)
s = torch.cuda.current_stream()
tmc.tmc_forward(g, inp, logp, ws, None, s); tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
counters()
names = {43: "prod.y_empty", 44: "prod.x_empty", 45: "prod.total",
         24: "mma.y_full", 25: "mma.x_full", 26: "mma.p_full", 27: "mma.gcol_empty", 28: "mma.grow_empty", 29: "mma.total",
         30: "smx.s_full", 31: "smx.pimg_empty", 35: "smx.r_empty", 36: "smx.total",
         37: "epi.grow_full", 38: "epi.r_full", 39: "epi.gcol_full", 40: "epi.dz_prefetch", 42: "epi.total",
         46: "mma.issue_gcol", 47: "mma.issue_grow", 48: "mma.issue_S",
         32: "smx.tmem_ld", 33: "smx.math", 34: "smx.st+sts(incl pimg wait)"}
tmc.tmc_forward(g, inp, logp, ws, None, s)
counters()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
e1.record()
c = counters()
out = {"cfg": name, "B": B, "bwd_ms": e0.elapsed_time(e1)}
for k, v in names.items():
    out[v] = round(c[k] / 1e6, 3)
print(json.dumps(out), flush=True)
