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


def test_config_parsing_mirrors_reference(tmp_path):
    """Host-only part of the config path (config.py:74-191): sections, keys,
    overrides, sensor ring, truth disks / boxes, error messages."""
    import numpy as np
    import pytest

    from paper_2509_15744_b200 import config as C
    from paper_2509_15744_b200.grids import ConfigError

    toml = b"""
[problem]
kind = "fwi"
[grid]
n = [21, 17]
dx = 1.0e-3
[time]
n_steps = 40
dt = 1.0e-8
[material]
flavor = "rho_scaled"
rho0 = 2700.0
c0 = 6000.0
[[sources]]
node = [3, 8]
amplitude = 1.0e12
frequency = 1.5e6
[sensors]
ring = { inset = 2, stride = 3 }
[truth]
disks = [{ center = [10, 8], radius = 2 }]
boxes = [{ lo = [1, 1], hi = [2, 3] }]
[gradient]
k = 1.0e13
precision = "single"
"""
    p = tmp_path / "c.toml"
    p.write_bytes(toml)
    rc, raw = C.load_config(p, overrides={"precision": "double", "method": None})
    assert rc.grid.shape == (21, 17) and rc.time.n_steps == 40
    assert rc.k == 1e13 and rc.precision == "double" and rc.method == "superposed"
    assert rc.resolved()["kind"] == "fwi"
    mat = C.build_material(raw, rc.grid)
    assert np.all(mat.gamma == 1.0)
    sens = C.build_sensors(raw, rc.grid)
    n1, n2, inset, stride = 21, 17, 2, 3
    lo = inset + stride - 1
    want = sorted({(inset, j) for j in range(lo, n2 - inset, stride)}
                  | {(n1 - 1 - inset, j) for j in range(lo, n2 - inset, stride)}
                  | {(i, inset) for i in range(lo, n1 - inset, stride)}
                  | {(i, n2 - 1 - inset) for i in range(lo, n1 - inset, stride)})
    assert list(sens.nodes) == want
    truth = C.build_truth_gamma(raw, rc.grid, mat)
    assert truth[10, 8] == mat.eps and truth[1, 3] == mat.eps and truth[0, 0] == 1.0
    src = C.build_sources(raw)
    assert src[0].cycles == 2
    with pytest.raises(ConfigError, match="missing required section"):
        C.parse_config({"problem": {"kind": "fwi"}})
    with pytest.raises(ConfigError, match="k must be a number or 'auto'"):
        C.parse_config(dict(raw, gradient={"k": "big"}))


def test_c5_problem_is_never_materialised():
    """bench.py's C5 problem: the global 2048-plane grids are
    constant broadcast views (no rank allocates the global gamma); shapes,
    source and sensor placement; weak vs strong sizes."""
    import numpy as np

    import bench
    import paper_2509_15744_b200 as W

    wl = bench.c5_workload(8, "weak", 200)
    assert wl["shape"] == (2048, 2048, 2048)
    assert bench.c5_workload(2, "strong", 200)["shape"] == (2048, 2048, 2048)
    wl = bench.c5_workload(4, "weak", 20)
    problem, model, truth = bench.build_c5_problem(W, wl)
    assert model.gamma.strides == (0, 0, 0) and truth.gamma.strides == (0, 0, 0)
    assert float(truth.gamma[5, 6, 7]) == 0.9 and float(model.gamma[0, 0, 0]) == 1.0
    assert problem.sources[0].node == (3, 1024, 1024)
    assert len(problem.sensors) == 33 * 33
    assert all(n[0] == 1024 - 4 for n in problem.sensors.nodes)
    assert problem.measured.shape == (1, 33 * 33, 20)
    assert np.all(problem.measured == 0)
