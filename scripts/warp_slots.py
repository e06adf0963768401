"""Instrumented reverse pass: per-softmax-warp S-full wait (slots 32+sw) and loop time (48+sw),
MMA-issuer slots 3..18, producer 0..2/14 (libtmc_instr*.so, TMC_LIB_PATH)."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TMC_LIB_PATH", os.path.join(ROOT, "paper_1806_08593_b200", "libtmc_instr.so"))
import numpy as np, torch
import tmc_workload as tw
import paper_1806_08593_b200 as tmc
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
wl = tw.make_workload(name, B=B)
g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B)
t = lambda a: None if a is None else torch.from_numpy(a).cuda()
inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i])) for i in range(len(wl.parent))]
ws = tmc.alloc_workspace(g); logp = torch.empty(wl.B, dtype=torch.float64, device="cuda"); grads = tmc.alloc_grads(g)
lib = tmc.load_library()
lib.tmc_debug_counters.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros((1024, 64), np.uint64)
def counters(clear=1):
    torch.cuda.synchronize()
    assert lib.tmc_debug_counters(buf.ctypes.data, buf.size, clear) == 0
    return buf[:148].astype(np.float64).mean(0) / 1e6
s = torch.cuda.current_stream()
tmc.tmc_forward(g, inp, logp, ws, None, s); tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
counters()
tmc.tmc_backward(g, inp, ws, None, grads, None, None, s)
c = counters()
print(json.dumps({"slots_0_31": [round(x, 3) for x in c[:32]], "sfull_wait_by_warp": [round(x, 3) for x in c[32:48]],
                  "loop_total_by_warp": [round(x, 3) for x in c[48:64]]}))
