"""Field dumps and raw traces in the reference's artifact formats.

Mirrors ``waveopt.io`` (io.py:29-111) for the data formats a GPU run must
produce byte-comparably:

* field dump = ``<name>.bin`` raw IEEE-754 little-endian, first grid axis
  varying fastest (np.ravel order "F"), plus ``<name>.json`` sidecar with
  dims, dtype, endianness, axis order, spacing and optional dt / step index;
* raw traces = ``<name>.bin`` float64 ``[n_sensors][n_steps]`` C order plus a
  ``{n_sensors, n_steps, dt}`` sidecar.

``dump_device_field`` writes a field that lives on the GPU: the axis
reversal happens on the device (``wo_get_field``, reverse_axes_kernel) so the
host only streams bytes to the file — numpy's strided F-order ravel of a
1024^3 field is the slow part of a host dump.  Config (TOML) and CSV logging
belong to the reference's CLI and are out of scope.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .grids import ConfigError, Grid

_DTYPES = {np.dtype(np.float32): ("<f4", "float32"), np.dtype(np.float64): ("<f8", "float64")}


def _bin_path(path) -> Path:
    path = Path(path)
    return path if path.suffix == ".bin" else path.with_suffix(".bin")


def _write_sidecar(bin_path: Path, meta: dict):
    bin_path.with_suffix(".json").write_text(json.dumps(meta, indent=1, sort_keys=True))


def _field_meta(grid: Grid, kind: str, dx, dt, step_index, extra) -> dict:
    meta = {"axis_order": "first-axis-fastest", "dims": list(grid.shape), "dtype": kind,
            "dx": grid.dx if dx is None else dx, "endianness": "little"}
    if dt is not None:
        meta["dt"] = dt
    if step_index is not None:
        meta["step_index"] = step_index
    if extra:
        meta.update(extra)
    return meta


def dump_field(path, values, grid: Grid, dx=None, dt=None, step_index=None, extra=None):
    """Host field -> <path>.bin + sidecar (io.py:29-52).  fp32 stays fp32,
    every other dtype is written as fp64."""
    path = _bin_path(path)
    values = np.asarray(values)
    if values.shape != grid.shape:
        raise ConfigError(f"field shape {values.shape} != grid {grid.shape}")
    code, kind = _DTYPES.get(values.dtype, _DTYPES[np.dtype(np.float64)])
    np.ravel(values, order="F").astype(code, copy=False).tofile(path)
    _write_sidecar(path, _field_meta(grid, kind, dx, dt, step_index, extra))
    return path


def dump_device_field(path, ctx, which, dx=None, dt=None, step_index=None, extra=None):
    """GPU field ("gamma", "u_prev", "u_cur", "acc" of a DeviceGrid) ->
    the same files dump_field writes, reordered on the device."""
    path = _bin_path(path)
    code, kind = _DTYPES[np.dtype(ctx.dtype)]
    flat = ctx.get_field(which, first_axis_fastest=True)
    flat.astype(code, copy=False).tofile(path)
    _write_sidecar(path, _field_meta(ctx.grid, kind, dx, dt, step_index, extra))
    return path


def load_field(path):
    """<path>.bin + sidecar -> (values in C order, sidecar dict) (io.py:55-66)."""
    path = _bin_path(path)
    meta = json.loads(path.with_suffix(".json").read_text())
    code = "<f4" if meta["dtype"] == "float32" else "<f8"
    flat = np.fromfile(path, dtype=code)
    dims = tuple(meta["dims"])
    if flat.size != int(np.prod(dims)):
        raise ConfigError(f"{path}: {flat.size} values, sidecar says {dims}")
    return flat.reshape(dims, order="F"), meta


def save_traces_raw(path, traces, dt):
    """[n_sensors][n_steps] traces as float64 + sidecar (io.py:90-100)."""
    path = _bin_path(path)
    traces = np.asarray(traces, dtype=np.float64)
    traces.astype("<f8").tofile(path)
    _write_sidecar(path, {"dt": float(dt), "n_sensors": int(traces.shape[0]),
                          "n_steps": int(traces.shape[1])})
    return path


def load_traces(path):
    """Raw traces written by save_traces_raw (io.py:103-111, .bin form)."""
    path = Path(path)
    meta = json.loads(path.with_suffix(".json").read_text())
    return np.fromfile(path, dtype="<f8").reshape(meta["n_sensors"], meta["n_steps"])
