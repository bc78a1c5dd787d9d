"""CPU-only checks: the C-ABI library loads and exports everything
include/waveb200.h declares; host-side logic matches the oracle; the
product path refuses to run without a GPU (no CPU fallback)."""

import os
import re

import numpy as np
import pytest

import cases
from helpers import bits_equal
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "waveb200.h")).read()
    return sorted(set(re.findall(r"\b(wo_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2509_15744_b200 import _native

    lib = _native.load()
    declared = _header_symbols()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_native.EXPORTS) == declared


def test_library_is_sm100a():
    import subprocess

    from paper_2509_15744_b200 import _native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    from paper_2509_15744_b200 import _native

    lib = _native.load()
    if lib.wo_device_count() > 0:
        pytest.skip("GPU present")
    import paper_2509_15744_b200 as W

    grid = W.build_grid((8, 8), 1e-3)
    mat = W.MaterialModel.rho_scaled(np.ones((8, 8)), grid, 2700.0, 6000.0)
    with pytest.raises(_native.NativeUnavailable):
        W.run_forward(mat, W.TimeConfig(5, 1e-8), [])


def test_amplitude_table_matches_reference_burst():
    from paper_2509_15744_b200.engine import source_amplitude_table
    import paper_2509_15744_b200 as W

    c = cases.DESK
    srcs = [W.SourceSpec(node=n, amplitude=a, frequency=f, cycles=cy)
            for n, a, f, cy in c["sources"]]
    tab = source_amplitude_table(srcs, c["dt"], c["n_steps"])
    for s, src in enumerate(srcs):
        osrc = O.Source(src.node, src.amplitude, src.frequency, src.cycles)
        ref = np.array([O.burst_amplitude(n * c["dt"], osrc) for n in range(c["n_steps"])])
        assert bits_equal(tab[s], ref)


@pytest.mark.parametrize("flavor", ["rho_scaled", "acoustic"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_force_coef_at_matches_prepare_material(flavor, dtype):
    from paper_2509_15744_b200.engine import force_coef_at
    import paper_2509_15744_b200 as W

    shape = (5, 6, 7)
    gamma, _, _, dt, dx, consts = cases.stencil_inputs(shape, flavor, dtype, 5)
    grid = W.build_grid(shape, dx)
    if flavor == "rho_scaled":
        mat = W.MaterialModel.rho_scaled(gamma, grid, eps=1e-3, **consts)
    else:
        mat = W.MaterialModel.acoustic(gamma, grid, **consts)
    prep = O.prepare_material(O.Material(flavor, gamma, dx, **consts), dt, dtype)
    for node in [(0, 0, 0), (2, 3, 4), (4, 5, 6)]:
        v = force_coef_at(mat, dt, dtype, node)
        assert np.dtype(type(v)) == np.dtype(dtype)
        assert v == prep.force_coef[node]


def test_grid_and_config_validation():
    import paper_2509_15744_b200 as W

    with pytest.raises(W.ConfigError):
        W.build_grid((2, 5), 1e-3)
    with pytest.raises(W.ConfigError):
        W.build_grid((5, 5, 5, 5), 1e-3)
    with pytest.raises(W.ConfigError):
        W.TimeConfig(1, 1e-8)
    grid = W.build_grid((5, 5), 1e-3)
    with pytest.raises(W.ConfigError):
        W.MaterialModel.rho_scaled(np.full((5, 5), 2.0), grid, 2700.0, 6000.0)
    with pytest.raises(W.ConfigError):
        W.SensorArray(nodes=[(1, 1), (1, 1)])
    with pytest.raises(W.ConfigError):
        W.SuperpositionConfig(k=-1.0)
    rep = W.cfl_report(grid, W.MaterialModel.rho_scaled(np.ones((5, 5)), grid, 2700, 6000),
                       0.75e-3 / 6000.0 / 1.0)
    assert rep.courant == pytest.approx(0.75) and not rep.stable


def test_beta_schedule_and_footprint():
    import paper_2509_15744_b200 as W
    from paper_2509_15744_b200.tato import _footprint

    assert [W.beta_schedule(i) for i in (0, 5, 10)] == [1.0, 1.1, 1.2100000000000002]
    for nd, count in ((1, 3), (2, 9), (3, 19)):
        offs, ws = _footprint(1.5, nd)
        assert len(ws) == count and offs.shape == (count, nd)
        K = O.filter_kernel(1.5, nd)
        assert np.isclose(ws.sum(), K.sum())
