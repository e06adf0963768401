"""The debug build (libtmc_debug.so, -DTMC_DEBUG_SYNC): every mbarrier wait of the
tensor-core pipelines carries a deadline and traps instead of hanging.  Run in a child process (the
binding loads one library per process): every pipelined kernel family on small ragged shapes must
complete under the deadlines and give results bit-identical to the release library (the deadline
only adds a clock read to the spin loop)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import tmc_workload as tw
import paper_1806_08593_b200 as tmc
out = {}
cases = [("C3", dict(B=3, K=300), 0, 0), ("C3", dict(B=2, K=520), 0, tmc.TMC_FLAG_SINGLE_PASS_REVERSE),
         ("C2", dict(B=2, K=200), 0, 0), ("C4", dict(B=2, K=260), 0, 0), ("C3", dict(B=2, K=300), 2, 0),
         ("C0", {}, 0, 0)]
for n, (name, kw, direction, flags) in enumerate(cases):
    wl = tw.make_workload(name, **kw)
    g = tmc.Graph(wl.parent, wl.K, wl.D, wl.B, direction=direction, flags=flags)
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    inp = [dict(z=t(wl.z[i]), mu=t(wl.mu[i]), logvar=t(wl.logvar[i]), logq=t(wl.logq[i]), logobs=t(wl.logobs[i]))
           for i in range(len(wl.parent))]
    logp, gr = tmc.estimate(g, inp)
    torch.cuda.synchronize()
    out[f"{n}_logp"] = logp.cpu().numpy()
    for i in range(len(wl.parent)):
        for k in ("dz", "dmu", "dlogvar"):
            out[f"{n}_{i}_{k}"] = gr[i][k].cpu().numpy()
np.savez(sys.argv[2], **out)
"""


def _run(lib, path):
    env = dict(os.environ, TMC_LIB_PATH=lib)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, path], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]


def test_debug_sync_build_matches_release(tmp_path):
    import numpy as np
    from paper_1806_08593_b200 import _build
    here = os.path.join(ROOT, "paper_1806_08593_b200")
    debug = os.path.join(here, "libtmc_debug.so")
    if not os.path.exists(debug):
        debug = _build.build_debug()
    _run(os.path.join(here, "libtmc.so"), str(tmp_path / "rel.npz"))
    _run(debug, str(tmp_path / "dbg.npz"))
    a, b = np.load(tmp_path / "rel.npz"), np.load(tmp_path / "dbg.npz")
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k], equal_nan=True), k
