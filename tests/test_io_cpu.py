"""Field-dump and raw-trace formats against files written by the reference's
io.py (tests/golden/io_dumps.npz, made by tests/golden/make_golden.py)."""

import numpy as np
import pytest

from paper_2509_15744_b200 import io as WIO
from paper_2509_15744_b200.grids import build_grid

CASES = [("f32_3d", (5, 4, 3), 2e-4, dict(dt=3e-9, step_index=17, extra={"what": "acc"})),
         ("f64_2d", (6, 7), 0.5, {}),
         ("f32_1d", (9,), 1.0, dict(step_index=0))]


@pytest.mark.parametrize("name,shape,dx,kw", CASES)
def test_dump_field_bytes_match_reference(golden, tmp_path, name, shape, dx, kw):
    g = golden("io_dumps")
    path = WIO.dump_field(tmp_path / name, g[f"{name}_values"], build_grid(shape, dx), **kw)
    assert path.read_bytes() == g[f"{name}_bin"].tobytes()
    assert path.with_suffix(".json").read_text() == str(g[f"{name}_json"])
    values, meta = WIO.load_field(path)
    assert values.dtype == g[f"{name}_values"].dtype
    np.testing.assert_array_equal(values, g[f"{name}_values"])
    assert meta["axis_order"] == "first-axis-fastest" and meta["dims"] == list(shape)


def test_traces_raw_bytes_match_reference(golden, tmp_path):
    g = golden("io_dumps")
    path = WIO.save_traces_raw(tmp_path / "traces", g["traces_values"], 2.5e-9)
    assert path.read_bytes() == g["traces_bin"].tobytes()
    assert path.with_suffix(".json").read_text() == str(g["traces_json"])
    np.testing.assert_array_equal(WIO.load_traces(path), g["traces_values"])


def test_dump_field_shape_mismatch(tmp_path):
    with pytest.raises(WIO.ConfigError):
        WIO.dump_field(tmp_path / "x", np.zeros((3, 3)), build_grid((3, 4), 1.0))
