"""Device-resident optimisation loop: invert() with gamma, the
Adam moments and the mask on the GPU gives the host loop's results."""

import numpy as np
import pytest

import cases
from helpers import bits_equal, product_fwi_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    import paper_2509_15744_b200 as W

    from paper_2509_15744_b200 import _native

    _native.load(require_device=True)
    return W


@pytest.mark.parametrize("name", ["fwi3d", "desk_fwi"])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_invert_device_loop_matches_host_loop(W, golden, name, prec):
    g = golden(name)
    c = cases.fwi3d_case() if name == "fwi3d" else cases.DESK
    problem, _ = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    kw = dict(method="superposed", k=c["k"], iterations=3, precision=prec, snapshot_every=1)
    dev = W.invert(problem, device_loop=True, **kw)
    host = W.invert(problem, device_loop=False, **kw)
    assert bits_equal(dev.gamma, host.gamma)
    assert len(dev.gamma_history) == len(host.gamma_history)
    for a, b in zip(dev.gamma_history, host.gamma_history):
        assert bits_equal(a, b)
    for a, b in zip(dev.log, host.log):
        assert a["iteration"] == b["iteration"]
        assert a["cost"] == b["cost"]
        if np.isfinite(b["grad_norm"]):
            assert abs(a["grad_norm"] - b["grad_norm"]) <= 1e-12 * abs(b["grad_norm"])


def test_invert_device_loop_with_mask(W, golden):
    """Frozen (masked) nodes: zero gradient, pinned at eps, as fwi.py:200-232."""
    g = golden("fwi3d")
    c = cases.fwi3d_case()
    problem, _ = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    mask = np.zeros(problem.grid.shape, dtype=bool)
    mask[:2] = True
    mask[-1, :, :3] = True
    problem.mask = mask
    kw = dict(method="superposed", k=c["k"], iterations=2, precision="double", snapshot_every=1)
    dev = W.invert(problem, device_loop=True, **kw)
    host = W.invert(problem, device_loop=False, **kw)
    assert bits_equal(dev.gamma, host.gamma)
    assert np.all(dev.gamma[mask] == problem.material.eps)


@pytest.mark.parametrize("prec", ["single", "double"])
def test_optimize_design_device_loop_matches_host_loop(W, golden, prec):
    from helpers import product_tato_problem

    g = golden("tato2d")
    c = cases.tato2d_case()
    problem = product_tato_problem(W, c)
    kw = dict(method="superposed", k=float(g["cal_k"]), iterations=4, precision=prec,
              snapshot_every=2)
    dev = W.optimize_design(problem, device_loop=True, **kw)
    host = W.optimize_design(problem, device_loop=False, **kw)
    assert bits_equal(dev.gamma_raw, host.gamma_raw)
    assert bits_equal(dev.design, host.design)
    assert len(dev.design_history) == len(host.design_history)
    for a, b in zip(dev.design_history, host.design_history):
        assert bits_equal(a, b)
    for a, b in zip(dev.log, host.log):
        assert a["cost"] == b["cost"] and a["beta"] == b["beta"]
        if np.isfinite(b["grad_norm"]):
            assert abs(a["grad_norm"] - b["grad_norm"]) <= 1e-12 * abs(b["grad_norm"])
