"""Adapters from the seeded cases (tests/golden/cases.py) to oracle inputs
and to the product API.  Test infrastructure only."""

from __future__ import annotations

import numpy as np

import cases


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    d = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / (d if d > 0 else 1.0)


def _ordered(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.float32:
        i = a.view(np.int32).astype(np.int64)
        return np.where(i < 0, -(i & 0x7FFFFFFF), i)
    i = a.view(np.int64)
    return np.where(i < 0, -(i & 0x7FFFFFFFFFFFFFFF), i)


def max_ulp(a, b):
    """Max distance in units in the last place (same float dtype)."""
    if a.size == 0:
        return 0
    d = _ordered(a).astype(np.float64) - _ordered(b).astype(np.float64)
    return float(np.max(np.abs(d)))


# ---------------------------------------------------------------- oracle side
def oracle_material(O, c, gamma):
    if c["flavor"] == "rho_scaled":
        return O.Material("rho_scaled", np.asarray(gamma, dtype=np.float64), c["dx"],
                          rho0=c["rho0"], c0=c["c0"])
    return O.Material("acoustic", np.asarray(gamma, dtype=np.float64), c["dx"],
                      rho1=c["rho1"], kappa1=c["kappa1"], rho2=c["rho2"], kappa2=c["kappa2"])


def oracle_fwi_shots(O, c, measured):
    shape = c["shape"]
    nodes = cases.ring_nodes(shape, *c["ring"]) if "ring" in c else c["sensors"]
    support = np.array([O.flat_index(shape, n) for n in nodes], dtype=np.int64)
    return [(O.Source(n, a, f, cy), O.FwiShot(support, measured[i], c["dt"]))
            for i, (n, a, f, cy) in enumerate(c["sources"])]


def oracle_tato_shots(O, c):
    node, amp, freq, cyc = c["source"]
    support = np.flatnonzero(c["objective_mask"].reshape(-1)).astype(np.int64)
    area = float(c["objective_mask"].sum()) * c["dx"] ** len(c["shape"])
    return [(O.Source(node, amp, freq, cyc),
             O.TatoShot(support, area, c["dt"], c["dx"], len(c["shape"]), c["mode"]))]


# --------------------------------------------------------------- product side
def product_fwi_problem(W, c, gamma, measured):
    grid = W.build_grid(c["shape"], c["dx"])
    time_cfg = W.TimeConfig(n_steps=c["n_steps"], dt=c["dt"])
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=c["rho0"], c0=c["c0"], eps=c["eps"])
    nodes = cases.ring_nodes(c["shape"], *c["ring"]) if "ring" in c else c["sensors"]
    sources = [W.SourceSpec(node=n, amplitude=a, frequency=f, cycles=cy)
               for n, a, f, cy in c["sources"]]
    problem = W.FwiProblem(grid=grid, time=time_cfg, material=mat, sources=sources,
                           sensors=W.SensorArray(nodes=nodes), measured=measured)
    return problem, mat


def product_tato_problem(W, c):
    grid = W.build_grid(c["shape"], c["dx"])
    time_cfg = W.TimeConfig(n_steps=c["n_steps"], dt=c["dt"])
    node, amp, freq, cyc = c["source"]
    src = W.SourceSpec(node=node, amplitude=amp, frequency=freq, cycles=cyc)
    return W.TatoProblem(grid=grid, time=time_cfg, source=src,
                         design_mask=c["design_mask"], objective_mask=c["objective_mask"],
                         rho1=c["rho1"], kappa1=c["kappa1"], rho2=c["rho2"],
                         kappa2=c["kappa2"], r_f=c["r_f"], eta=c["eta"], mode=c["mode"])
