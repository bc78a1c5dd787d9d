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


def _problem_planes(W, shape, seed, src_plane, sens_planes, n_steps, flavor="rho_scaled"):
    """A problem with its source on a chosen plane (e.g. one a two-step slab
    pass recomputes beyond a slab boundary) and sensors on chosen planes."""
    rng = np.random.default_rng(seed)
    dx = 1e-4
    dt = 0.45 * dx / 6000.0 / np.sqrt(3)
    gamma = rng.uniform(0.3, 1.0, size=shape)
    grid = W.build_grid(shape, dx)
    if flavor == "rho_scaled":
        mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    else:
        mat = W.MaterialModel.acoustic(gamma, grid, rho1=1.2, kappa1=1.4e5, rho2=1000.0,
                                       kappa2=2.2e9)
        dt = 0.45 * dx / 1500.0 / np.sqrt(3)
    srcs = [W.SourceSpec(node=(src_plane, shape[1] // 2 - 1, shape[2] // 2 + 1), amplitude=1e12,
                         frequency=5e6, cycles=2)]
    sens = sorted({(i, j, k) for i in sens_planes for j in (0, shape[1] // 2, shape[1] - 1)
                   for k in (0, 31, shape[2] - 1)})
    measured = rng.normal(scale=1e-10, size=(len(srcs), len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=srcs, sensors=W.SensorArray(nodes=sens), measured=measured)
    return problem, mat


@pytest.mark.parametrize("shape,parts,src_plane,sens_planes", [
    ((32, 16, 64), 2, 15, (3, 28)),      # source on the plane the upper slab recomputes
    ((32, 16, 64), 2, 16, (0, 31)),      # ... the lower slab recomputes
    ((40, 16, 128), 4, 21, (2, 5, 37)),  # 4 slabs, source next to a boundary
    ((24, 8, 64), 3, 7, (12, 23)),       # slabs of 8 planes
    ((12, 16, 64), 4, 6, (1, 10)),       # slabs of 3 planes (peer stores overlap)
])
@pytest.mark.parametrize("n_steps", [40, 41])
def test_slabs_two_step_peer_stores_bitwise(W, shape, parts, src_plane, sens_planes, n_steps):
    """Slabs with two ghost planes per neighbour run two-step passes whose
    launches store both new levels into the neighbours' ghost planes; the
    recomputed plane beyond each boundary injects sources there itself.  The
    gradient is bitwise the one-context gradient, twice in a row (flag
    epochs restart per sweep), for odd and even step counts."""
    from paper_2509_15744_b200.distributed import SlabGradient, slab_ranges

    problem, mat = _problem_planes(W, shape, 11 * sum(shape) + parts + src_plane, src_plane,
                                   sens_planes, n_steps)
    cfg = W.SuperpositionConfig(k=1e13, precision="single")
    ref = W.gradient_superposed(problem, mat, cfg)
    sg = SlabGradient(problem, mat, cfg, slab_ranges(shape[0], parts), halo="peer").upload()
    try:
        assert sg.two_step
        for c in sg.ctxs:
            c.reset_stats()
        for _ in range(2):
            cost = sg.run()
            assert bits_equal(sg.download(), ref.gradient)
            assert abs(cost - ref.cost) <= 1e-13 * abs(ref.cost)
        assert all(c.stats()["pair_launches"] > 0 for c in sg.ctxs)
    finally:
        sg.close()


def test_slabs_two_step_acoustic_peer_bitwise(W):
    from paper_2509_15744_b200.distributed import SlabGradient, slab_ranges

    problem, mat = _problem_planes(W, (24, 16, 64), 5, 12, (2, 20), 33, flavor="acoustic")
    cfg = W.SuperpositionConfig(k=1e13, precision="single")
    ref = W.gradient_superposed(problem, mat, cfg)
    sg = SlabGradient(problem, mat, cfg, slab_ranges(24, 3), halo="peer").upload()
    try:
        assert sg.two_step
        sg.run()
        assert bits_equal(sg.download(), ref.gradient)
    finally:
        sg.close()


def test_slabs_support_on_recomputed_plane_stays_single_step(W):
    """A sensor on a plane next to a slab boundary keeps every slab on single
    steps (its adjoint force lives in the neighbour's store); still bitwise."""
    from paper_2509_15744_b200.distributed import SlabGradient, slab_ranges

    problem, mat = _problem_planes(W, (32, 16, 64), 9, 5, (15, 30), 30)
    cfg = W.SuperpositionConfig(k=1e13, precision="single")
    ref = W.gradient_superposed(problem, mat, cfg)
    sg = SlabGradient(problem, mat, cfg, slab_ranges(32, 2), halo="peer").upload()
    try:
        assert not sg.two_step
        for c in sg.ctxs:
            c.reset_stats()
        sg.run()
        assert bits_equal(sg.download(), ref.gradient)
        assert all(c.stats()["pair_launches"] == 0 for c in sg.ctxs)
    finally:
        sg.close()


def test_slabs_c5_planes_two_step_peer_bitwise(W):
    """Two slabs of a grid with C5's 2048 x 2048 planes on one GPU:
    TMA maps, 64-bit plane offsets and peer stores at full plane size."""
    from paper_2509_15744_b200.distributed import SlabGradient, slab_ranges

    shape = (8, 2048, 2048)
    problem, mat = _problem_planes(W, shape, 21, 3, (0, 7), 12)
    cfg = W.SuperpositionConfig(k=1e13, precision="single")
    ref = W.gradient_superposed(problem, mat, cfg)
    sg = SlabGradient(problem, mat, cfg, slab_ranges(8, 2), halo="peer").upload()
    try:
        assert sg.two_step
        sg.run()
        assert bits_equal(sg.download(), ref.gradient)
    finally:
        sg.close()
