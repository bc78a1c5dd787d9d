"""Seeded parity cases shared by the golden generator, the oracle tests and the
GPU parity tests.  Pure numpy: no reference, oracle or product imports.

Every case is a plain dict of parameters; inputs that the reference itself
produced (measured traces from ``synthesize_measurements``) are stored in the
fixture next to the outputs.
"""

from __future__ import annotations

import math

import numpy as np

# configs/fwi_desk.toml (/root/reference/pkg/configs/fwi_desk.toml:8-57)
DESK = dict(
    name="desk_fwi", kind="fwi", shape=(101, 101), dx=2.0e-4, n_steps=800,
    dt=1.6666666666666667e-8, flavor="rho_scaled", rho0=2700.0, c0=6000.0,
    eps=1.0e-5,
    sources=[((3, 50), 1.0e12, 1.5e6, 2), ((97, 50), 1.0e12, 1.5e6, 2),
             ((50, 3), 1.0e12, 1.5e6, 2), ((50, 97), 1.0e12, 1.5e6, 2)],
    ring=(3, 4), truth_disks=[((60, 42), 9)], refine=2, k=1.0e13,
)


def ring_nodes(shape, inset, stride):
    """Sensor ring layout of config.py:151-163."""
    n1, n2 = shape
    lo = inset + stride - 1
    nodes = ([(inset, j) for j in range(lo, n2 - inset, stride)]
             + [(n1 - 1 - inset, j) for j in range(lo, n2 - inset, stride)]
             + [(i, inset) for i in range(lo, n1 - inset, stride)]
             + [(i, n2 - 1 - inset) for i in range(lo, n1 - inset, stride)])
    return sorted(set(nodes))


def disk_gamma(shape, disks, eps):
    """Truth indicator of config.py:182-194 (disks held at eps)."""
    gamma = np.ones(shape)
    idx = np.indices(shape)
    for center, radius in disks:
        dist2 = sum((idx[a] - int(center[a])) ** 2 for a in range(len(shape)))
        gamma[dist2 <= radius**2] = eps
    return gamma


def smooth_random_gamma(shape, seed, lo, hi):
    """Random indicator in [lo, hi] with a little spatial smoothness."""
    rng = np.random.default_rng(seed)
    g = rng.uniform(0.0, 1.0, size=shape)
    for axis in range(len(shape)):
        g = 0.5 * g + 0.25 * (np.roll(g, 1, axis) + np.roll(g, -1, axis))
    g = (g - g.min()) / max(g.max() - g.min(), 1e-30)
    return lo + (hi - lo) * g


def fwi3d_case():
    """Small 3D rho-scaled FWI: random smooth gamma, two sources on the
    axis-0 = 3 face, a 5x5 sensor grid on the opposite face."""
    shape = (22, 18, 26)
    dx = 1.0e-4
    c0 = 6000.0
    dt = 0.5 * dx / c0
    sensors = [(shape[0] - 4, j, k) for j in range(3, 16, 3) for k in range(3, 24, 5)]
    return dict(
        name="fwi3d", kind="fwi", shape=shape, dx=dx, n_steps=140, dt=dt,
        flavor="rho_scaled", rho0=2700.0, c0=c0, eps=1e-5,
        sources=[((3, 9, 13), 1.0e12, 5.0e6, 2), ((3, 5, 20), 1.0e12, 5.0e6, 2)],
        sensors=sensors,
        truth_spheres=[((11, 9, 13), 4)], refine=1,
        gamma=smooth_random_gamma(shape, 7, 0.6, 1.0),
        k=1.0e14,
    )


def tato2d_case():
    """Small 2D TATO: acoustic flavor, design box, objective box, one source.
    Constants: tato.py:175-178."""
    shape = (41, 37)
    dx = 0.01
    rho1, kappa1, rho2, kappa2 = 1.204, 1.419e5, 2643.0, 6.87e8
    c_max = math.sqrt(kappa2 / rho2)
    dt = 0.5 * dx / c_max
    design = np.zeros(shape, dtype=bool)
    design[14:27, 10:28] = True
    objective = np.zeros(shape, dtype=bool)
    objective[30:36, 12:26] = True
    rng = np.random.default_rng(11)
    gamma_raw = np.where(design, rng.uniform(0.0, 1.0, size=shape), 0.0)
    return dict(
        name="tato2d", kind="tato", shape=shape, dx=dx, n_steps=260, dt=dt,
        flavor="acoustic", rho1=rho1, kappa1=kappa1, rho2=rho2, kappa2=kappa2,
        source=((6, 18), 1.0, 2800.0, 2),
        design_mask=design, objective_mask=objective, gamma_raw=gamma_raw,
        r_f=1.5, eta=0.5, mode="suppress", beta_iter=7,
    )


# random single-step stencil / kernel-increment cases
STENCIL_SHAPES = [(9,), (7, 11), (5, 6, 7), (3, 4, 33)]


def stencil_inputs(shape, flavor, dtype, seed):
    """Random (gamma, u_prev, u_cur, dt, dx, constants) for one step."""
    rng = np.random.default_rng(seed)
    dtype = np.dtype(dtype)
    if flavor == "rho_scaled":
        gamma = rng.uniform(1e-3, 1.0, size=shape)
        consts = dict(rho0=2700.0, c0=6000.0)
    else:
        gamma = rng.uniform(0.0, 1.0, size=shape)
        consts = dict(rho1=1.204, kappa1=1.419e5, rho2=2643.0, kappa2=6.87e8)
    u_prev = rng.standard_normal(shape).astype(dtype)
    u_cur = rng.standard_normal(shape).astype(dtype)
    dx = 1e-3
    dt = 0.3 * dx / 6000.0 if flavor == "rho_scaled" else 0.3 * dx / 509.8
    return gamma, u_prev, u_cur, dt, dx, consts


def ki_inputs(shape, dtype, seed):
    rng = np.random.default_rng(seed)
    dtype = np.dtype(dtype)
    wins = [rng.standard_normal(shape).astype(dtype) for _ in range(6)]
    acc = rng.standard_normal(shape).astype(dtype)
    scal = (-2700.0, 2700.0 * 6000.0**2, 1.0 / (2.0 * 1.7e-8), 1.0 / (2.0 * 1e-4), 1.7e-8)
    return acc, wins, scal


def desk_mask(shape, width=2):
    """Fictitious-domain mask for the masked invert case: a border of
    `width` nodes held at eps (fwi.py:42-46 clip_indicator frozen_mask)."""
    m = np.zeros(shape, dtype=bool)
    m[:width, :] = m[-width:, :] = True
    m[:, :width] = m[:, -width:] = True
    return m


def solver2d_case():
    """Small 2D rho-scaled grid for run_forward / run_backward parity."""
    shape = (40, 33)
    dx = 2.0e-4
    return dict(name="solver2d", shape=shape, dx=dx, n_steps=150, dt=0.5 * dx / 6000.0,
                rho0=2700.0, c0=6000.0, eps=1e-5,
                gamma=smooth_random_gamma(shape, 31, 0.4, 1.0))


def colocated_sources(c):
    """Three sources, two of them on the same node (solver.py:154-170: numpy
    fancy-index += keeps the LAST duplicate's value)."""
    shape = c["shape"]
    a = tuple(n // 3 for n in shape)
    b = tuple(n // 2 for n in shape)
    return [(a, 1.0e12, 5.0e6, 2), (b, 7.0e11, 3.0e6, 2), (a, 3.0e11, 2.0e6, 2)]


def solver_sensors(c):
    shape = c["shape"]
    hi = tuple(n - 2 for n in shape)
    mid = tuple(n // 2 + 1 for n in shape)
    return sorted({tuple(1 for _ in shape), hi, mid})
