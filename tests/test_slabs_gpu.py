"""Slab decomposition on one GPU (loopback halo exchange between slab
contexts in one process): bitwise equal to the single-context gradient, for
TMA-eligible and generic grids, fp32 and fp64."""

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


def _problem(W, shape, seed):
    rng = np.random.default_rng(seed)
    dx, n_steps = 1e-4, 70
    dt = 0.45 * dx / 6000.0 / np.sqrt(3)
    gamma = rng.uniform(0.3, 1.0, size=shape)
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    srcs = [W.SourceSpec(node=(shape[0] // 2, shape[1] // 3, shape[2] // 2), amplitude=1e12,
                         frequency=5e6, cycles=2),
            W.SourceSpec(node=(2, 1, 3), amplitude=1e12, frequency=5e6, cycles=2)]
    sens = sorted({(i, j, k) for i in (0, shape[0] // 3, shape[0] - 1)
                   for j in (0, shape[1] - 1) for k in (1, shape[2] - 2)})
    measured = rng.normal(scale=1e-10, size=(len(srcs), len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=srcs, sensors=W.SensorArray(nodes=sens), measured=measured)
    return problem, mat


@pytest.mark.parametrize("shape,parts", [((24, 16, 64), 3), ((22, 18, 26), 2), ((9, 8, 64), 4)])
@pytest.mark.parametrize("prec", ["single", "double"])
@pytest.mark.parametrize("overlap", [True, False])
def test_slabs_bitwise_equal_single_gpu(W, shape, parts, prec, overlap):
    """Slabs (split boundary/interior steps with the exchange between them,
    or whole steps) give the single-GPU bits."""
    from paper_2509_15744_b200.distributed import gradient_superposed_slabs

    problem, mat = _problem(W, shape, sum(shape) + parts)
    cfg = W.SuperpositionConfig(k=1e13, precision=prec)
    ref = W.gradient_superposed(problem, mat, cfg)
    got = gradient_superposed_slabs(problem, mat, cfg, parts, overlap=overlap)
    assert bits_equal(got.gradient, ref.gradient)
    assert abs(got.cost - ref.cost) <= 1e-13 * abs(ref.cost)


@pytest.mark.parametrize("shape,parts", [((24, 16, 64), 3), ((22, 18, 26), 2), ((9, 8, 64), 4)])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_slabs_peer_stores_bitwise_equal(W, shape, parts, prec):
    """Peer ghost stores (boundary launches write the neighbours' ghost
    planes and bump device flags their streams wait on; no exchange) give
    the single-GPU bits, twice in a row on the same contexts (the flag
    sequence continues across evaluations)."""
    from paper_2509_15744_b200.distributed import SlabGradient, slab_ranges

    problem, mat = _problem(W, shape, sum(shape) + parts + 7)
    cfg = W.SuperpositionConfig(k=1e13, precision=prec)
    ref = W.gradient_superposed(problem, mat, cfg)
    sg = SlabGradient(problem, mat, cfg, slab_ranges(shape[0], parts), halo="peer").upload()
    try:
        for _ in range(2):
            cost = sg.run()
            assert bits_equal(sg.download(), ref.gradient)
            assert abs(cost - ref.cost) <= 1e-13 * abs(ref.cost)
    finally:
        sg.close()


def test_slabs_match_reference_fixture(W, golden):
    from paper_2509_15744_b200.distributed import gradient_superposed_slabs

    g = golden("fwi3d")
    c = cases.fwi3d_case()
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    for prec in ("double", "single"):
        res = gradient_superposed_slabs(problem, mat,
                                        W.SuperpositionConfig(k=c["k"], precision=prec), 3)
        assert bits_equal(res.gradient, g[f"sup_grad_{prec}"]), prec
