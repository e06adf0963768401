"""The torch model harness (tmc_workload.torch_model, bench full step) reproduces tmc_workload's
inputs: same parameters and noise give the same z, mu, logvar, logq, logobs (fp32 vs fp64 rounding)."""
import numpy as np
import pytest
import torch

import tmc_workload as tw
from tmc_workload.torch_model import TorchModel


@pytest.mark.parametrize("name,kw", [("S_mlp", {}), ("S_mlp_bern", {}), ("S_chain", {}), ("S_tree", {}),
                                     ("C3", dict(B=2, K=8)), ("C4", dict(B=2, K=6)), ("S_mnist", {}),
                                     ("C1", dict(B=2, K=5)), ("M5", dict(B=2, K=4))])
def test_torch_model_matches_workload(name, kw):
    wl = tw.make_workload(name, **kw)
    m = TorchModel(wl, "cpu")
    f = m.forward()
    for k in ("z", "mu", "logvar", "logq", "logobs"):
        for i in range(len(wl.parent)):
            ref = getattr(wl, k)[i]
            got = f[k][i]
            if ref is None:
                assert got is None, (k, i)
                continue
            np.testing.assert_allclose(got.detach().numpy(), ref, rtol=2e-4, atol=2e-4, err_msg=f"{k}[{i}]")


@pytest.mark.parametrize("name", ["S_mlp", "S_mnist"])
def test_torch_model_backward_accumulates_parameter_grads(name):
    wl = tw.make_workload(name)
    m = TorchModel(wl, "cpu")
    f = m.forward()
    grads = [{k: (None if f[kk][i] is None else torch.ones_like(f[kk][i]))
              for k, kk in (("dz", "z"), ("dmu", "mu"), ("dlogvar", "logvar"), ("dlogq", "logq"), ("dlogobs", "logobs"))}
             for i in range(len(wl.parent))]
    m.backward(f, grads)
    g = m.flat_grads()
    assert g.numel() == m.grad_numel and torch.isfinite(g).all() and g.abs().sum() > 0
