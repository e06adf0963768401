"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol include/tmc.h
declares, and host-side validation returns the documented statuses (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1806_08593_b200 as tmc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tmc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tmc_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = tmc.load_library()
    syms = header_symbols()
    assert set(syms) == set(tmc.EXPORTS), syms
    out = subprocess.check_output(["nm", "-D", "--defined-only", tmc.LIB_PATH]).decode()
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), f"{s} not exported"
        assert hasattr(lib, s)


def test_version():
    assert tmc.tmc_version() == 100


def test_workspace_size_and_graph_validation():
    g = tmc.Graph([-1, 0, 1], [8, 8, 8], [2, 2, 2], B=4)
    assert tmc.tmc_workspace_size(g) > 0
    with pytest.raises(tmc.TmcError) as e:
        tmc.tmc_workspace_size(tmc.Graph([-1, 2, 1], [8, 8, 8], [2, 2, 2], B=4))
    assert "parent[1]" in str(e.value)               # size query returns 0 + message
    with pytest.raises(tmc.TmcError) as e:
        tmc.tmc_workspace_size(tmc.Graph([-1, 0], [8, 0], [2, 2], B=4))
    assert "K[1]" in str(e.value)
    with pytest.raises(tmc.TmcError) as e:           # DOWN on a tree
        tmc.tmc_workspace_size(tmc.Graph([-1, 0, 0], [4, 4, 4], [1, 1, 1], B=1, direction=tmc.TMC_DIR_DOWN))
    assert "chain" in str(e.value)
    with pytest.raises(tmc.TmcError) as e:           # the two reverse-pass choices are exclusive
        tmc.tmc_workspace_size(tmc.Graph([-1, 0], [4, 4], [2, 2], B=1, flags=tmc.TMC_FLAG_TWO_PASS_REVERSE
                                         | tmc.TMC_FLAG_SINGLE_PASS_REVERSE))
    assert "exclusive" in str(e.value)


def _raw_forward(g, inputs, ws_bytes):
    lib = tmc.load_library()
    arr = tmc._inputs(inputs)
    return lib.tmc_forward(g.ref(), arr, None, ctypes.c_void_p(16), ctypes.c_void_p(4096) if ws_bytes else None,
                           ws_bytes, None)


def test_forward_statuses_without_gpu():
    g = tmc.Graph([-1, 0], [4, 4], [2, 2], B=2)
    fake = dict(z=4096, mu=4096, logvar=4096, logq=4096)
    assert _raw_forward(g, [fake, fake], 0) == -5                  # TMC_ERR_WORKSPACE
    assert _raw_forward(g, [fake, dict(fake, z=None)], 1 << 20) == -1  # NULL input
    bad = tmc.Graph([-1, 1], [4, 4], [2, 2], B=2)
    assert _raw_forward(bad, [fake, fake], 1 << 30) == -3          # TMC_ERR_GRAPH
    rc = _raw_forward(g, [fake, fake], 1 << 30)
    import torch
    if not torch.cuda.is_available():
        assert rc == -6                                            # TMC_ERR_UNSUPPORTED_DEVICE
        assert "device" in tmc.tmc_last_error()


def test_extension_call_statuses_without_gpu():
    """Argument validation of the calls added beyond the estimator happens before any device work."""
    lib = tmc.load_library()
    P = ctypes.c_void_p
    fake = dict(z=4096, mu=4096, logvar=4096, logq=4096)
    arr = tmc._inputs([fake, fake])
    # IWAE needs equal K on every latent
    g = tmc.Graph([-1, 0], [4, 5], [2, 2], B=2)
    assert lib.tmc_iwae(g.ref(), arr, P(4096), None, None, P(4096), 1 << 20, None) == -2          # TMC_ERR_SHAPE
    # the shared-root exchange needs an explicit UP direction and exactly one root
    chain = tmc.Graph([-1, 0], [4, 4], [2, 2], B=2)
    assert lib.tmc_forward_children(chain.ref(), arr, P(4096), P(4096), 1 << 30, None) == -3    # TMC_ERR_GRAPH
    two_roots = tmc.Graph([-1, -1], [4, 4], [2, 2], B=2, direction=tmc.TMC_DIR_UP)
    assert lib.tmc_forward_root(two_roots.ref(), arr, P(4096), P(4096), P(4096), 1 << 30, None) == -3
    # sampler shapes
    assert lib.tmc_sample_normal(0, 4, -1, 0, 0, 4, 4, P(4096), None) == -2
    assert lib.tmc_sample_normal(0, 4, 2, 0, 0, 4, 0, P(4096), None) == -2
    assert lib.tmc_sample_normal(0, 4, 0, 0, 0, 4, 4, None, None) == 0                            # empty: nothing to do
    # host-streamed estimate: chunk must be positive
    assert lib.tmc_estimate_host(chain.ref(), arr, P(4096), None, None, 0, P(4096), 1 << 30, None) == -1
    assert lib.tmc_estimate_host_workspace_size(chain.ref(), 0) == 0
    assert lib.tmc_estimate_host_workspace_size(chain.ref(), 1) > lib.tmc_workspace_size(
        tmc.Graph([-1, 0], [4, 4], [2, 2], B=1).ref())


def test_elim_graph_validation():
    """tmc_elim_*: invalid scopes / orders / intermediates wider than 3 indices are rejected by the
    host-side plan (workspace query returns 0 + message; nothing is launched)."""
    ok = tmc.FactorGraph([3, 4, 2, 3], [(0, 1), (0, 2), (1, 3), (2, 3)], 2)
    assert tmc.tmc_elim_workspace_size(ok) > 0
    bad = [tmc.FactorGraph([3] * 5, [(0, 1), (0, 2), (0, 3), (0, 4)], 2),       # 4-index intermediate
           tmc.FactorGraph([3] * 3, [(0, 1), (1, 2)], 2, order=[0, 0, 1]),      # not a permutation
           tmc.FactorGraph([3] * 3, [(0, 1), (1, 5)], 2),                       # variable out of range
           tmc.FactorGraph([3] * 3, [(0, 0)], 2)]                               # repeated variable
    for fg in bad:
        with pytest.raises(tmc.TmcError):
            tmc.tmc_elim_workspace_size(fg)
