"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py).  Bit-exact for fields, traces and gradients;
costs to 1e-14 relative (the reference sums np.dot partials through BLAS)."""

import numpy as np
import pytest

import cases
from helpers import bits_equal, oracle_fwi_shots, oracle_material, oracle_tato_shots, rel_l2
from oracle import oracle as O


def _dt(name):
    return np.float32 if name == "f32" else np.float64


@pytest.mark.parametrize("si", range(len(cases.STENCIL_SHAPES)))
@pytest.mark.parametrize("flavor", ["rho_scaled", "acoustic"])
@pytest.mark.parametrize("dn", ["f32", "f64"])
def test_prepare_and_step_bitexact(golden, si, flavor, dn):
    g = golden("stencil")
    key = f"{flavor}_{dn}_{si}"
    shape = cases.STENCIL_SHAPES[si]
    gamma, u_prev, u_cur, dt, dx, consts = cases.stencil_inputs(
        shape, flavor, _dt(dn), int(g[f"seed_{key}"]))
    mat = O.Material(flavor, gamma, dx, **consts)
    prep = O.prepare_material(mat, dt, _dt(dn))
    assert bits_equal(prep.coef, g[f"coef_{key}"])
    assert bits_equal(prep.force_coef, g[f"fc_{key}"])
    for a, w in enumerate(prep.face_weights):
        assert bits_equal(w, g[f"wf{a}_{key}"])
    out = np.empty_like(u_cur)
    O.apply_step(u_prev, u_cur, prep.face_weights, prep.coef, out)
    assert bits_equal(out, g[f"step_{key}"])


@pytest.mark.parametrize("si", range(len(cases.STENCIL_SHAPES)))
@pytest.mark.parametrize("dn", ["f32", "f64"])
def test_kernel_increment_bitexact(golden, si, dn):
    g = golden("kernel_increment")
    shape = cases.STENCIL_SHAPES[si]
    seed = 2000 + 10 * si + (dn == "f64")
    acc, wins, scal = cases.ki_inputs(shape, _dt(dn), seed)
    a = acc.copy()
    O.apply_kernel_increment(a, tuple(wins[:3]), tuple(wins[3:]), *scal)
    assert bits_equal(a, g[f"mixed_{dn}_{si}"])
    a = acc.copy()
    O.apply_kernel_increment(a, tuple(wins[:3]), tuple(wins[:3]), *scal)
    assert bits_equal(a, g[f"self_{dn}_{si}"])


def test_kats(golden):
    g = golden("kats")
    src = O.Source((1, 1), 1.0, 1.0, 2)
    assert O.burst_amplitude((np.pi / 2) / src.omega, src) == float(g["burst_quarter"])
    assert float(g["burst_quarter"]) == 0.14644660940672624
    assert float(g["heaviside_075"]) == float(O.heaviside_project(0.75, 1.0, 0.5))
    spike = O.density_filter(np.pad(np.ones((1, 1)), 4), 1.5, np.ones((9, 9), bool))[4, 4]
    assert spike == float(g["filter_spike"])
    assert [O.beta_schedule(i) for i in (0, 5, 10)] == list(g["beta_0_5_10"])
    # unit force at a zero field: u = dt^2/(rho0*gamma) at the node
    mat = O.Material("rho_scaled", np.full((5, 5), 0.5), 1e-3, rho0=2700.0, c0=6000.0)
    prep = O.prepare_material(mat, 1e-8, np.float64)
    w = O.Window((5, 5), np.float64)
    O.step_window(w, prep, (np.array([12]), np.array([1.0])))
    assert bits_equal(w.u_next, g["unit_force"])


@pytest.mark.parametrize("name", ["fwi3d", "desk_fwi"])
def test_fwi_gradients_bitexact(golden, name):
    g = golden(name)
    c = cases.fwi3d_case() if name == "fwi3d" else cases.DESK
    mat = oracle_material(O, c, g["gamma_model"])
    for prec in ("double", "single"):
        shots = oracle_fwi_shots(O, c, g["measured"])
        cost, grad, _ = O.gradient_superposed(mat, c["dt"], c["n_steps"], shots, c["k"], prec)
        assert bits_equal(grad, g[f"sup_grad_{prec}"]), prec
        assert abs(cost - float(g[f"sup_cost_{prec}"])) <= 1e-14 * abs(cost)
        fc = O.forward_cost(mat, c["dt"], c["n_steps"], oracle_fwi_shots(O, c, g["measured"]),
                            prec)
        assert abs(fc - float(g[f"fcost_{prec}"])) <= 1e-14 * abs(fc)
    for prec in ("double", "single"):
        cost, grad = O.gradient_reference(mat, c["dt"], c["n_steps"],
                                          oracle_fwi_shots(O, c, g["measured"]), prec)
        assert bits_equal(grad, g[f"ref_grad_{prec}"]), prec


@pytest.mark.parametrize("name", ["fwi3d", "desk_fwi"])
def test_forward_traces_bitexact(golden, name):
    g = golden(name)
    c = cases.fwi3d_case() if name == "fwi3d" else cases.DESK
    mat = oracle_material(O, c, g["truth"])
    sources = [O.Source(n, a, f, cy) for n, a, f, cy in c["sources"]]
    for dn in ("f32", "f64"):
        up, uc, tr, _, peak = O.run_forward(mat, c["dt"], c["n_steps"], sources,
                                            g["sensor_idx"], dtype=_dt(dn))
        assert bits_equal(tr, g[f"fwd_traces_{dn}"])
        assert bits_equal(up, g[f"fwd_uprev_{dn}"])
        assert bits_equal(uc, g[f"fwd_ucur_{dn}"])
        assert peak == float(g[f"fwd_peak_{dn}"])


def test_tato_bitexact(golden):
    g = golden("tato2d")
    c = cases.tato2d_case()
    beta, g_tilde, g_bar = O.design_fields(c["gamma_raw"], c["beta_iter"], c["r_f"], c["eta"],
                                           c["design_mask"])
    assert beta == float(g["beta"])
    assert bits_equal(g_tilde, g["g_tilde"])
    assert bits_equal(g_bar, g["g_bar"])
    mat = oracle_material(O, c, g_bar)
    k = float(g["cal_k"])
    for prec in ("double", "single"):
        cost, grad, _ = O.gradient_superposed(mat, c["dt"], c["n_steps"],
                                              oracle_tato_shots(O, c), k, prec)
        assert bits_equal(grad, g[f"sup_grad_{prec}"]), prec
        assert abs(cost - float(g[f"sup_cost_{prec}"])) <= 1e-14 * abs(cost)
    cost, grad = O.gradient_reference(mat, c["dt"], c["n_steps"], oracle_tato_shots(O, c))
    assert bits_equal(grad, g["ref_grad_double"])
    chain = O.chain_rule(grad, g_tilde, beta, c["eta"], c["r_f"], c["design_mask"])
    assert bits_equal(chain, g["chain"])


def test_superposed_vs_reference_agreement(golden):
    """SPEC agreement contract (<5% relative MSE) holds on the fixtures."""
    g = golden("desk_fwi")
    assert rel_l2(g["sup_grad_double"], g["ref_grad_double"]) ** 2 < 0.05
    assert int(g["sup_peak_fields_double"]) == 4
