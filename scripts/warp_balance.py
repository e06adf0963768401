"""Experiment: per-softmax-warp S-wait and total cycles in the reverse pass (libtmc_instr_nomma.so)."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TMC_LIB_PATH", os.path.join(ROOT, "paper_1806_08593_b200", "libtmc_instr_nomma.so"))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc
wl = tw.make_workload("C3", B=256)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
t = lambda a: None if a is None else torch.from_numpy(a).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i])) for i in range(len(wl.parent))]
ws = tmc.alloc_workspace(g); logp = torch.empty(wl.B, dtype=torch.float64, device="cuda"); grads = tmc.alloc_grads(g)
lib = tmc.load_library(); lib.tmc_debug_counters.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros((1024, 64), np.uint64)
s = torch.cuda.current_stream()
os.environ["TMC_DENSE_REVERSE"] = "1"
tmc.tmc_forward(g, inp, logp, ws, None, s); tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
torch.cuda.synchronize(); lib.tmc_debug_counters(buf.ctypes.data, buf.size, 1)
tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
torch.cuda.synchronize(); lib.tmc_debug_counters(buf.ctypes.data, buf.size, 1)
c = buf[:148].astype(np.float64).mean(0) / 6200
print(json.dumps({"s_wait_per_tile": [round(x) for x in c[32:48]], "total_per_tile": [round(x) for x in c[48:64]]}))
