"""The five synthetic workloads of BASELINE.json `configs`, with the SURVEY.md
section 8(d) readings (Q11-Q20) for everything BASELINE.json leaves unstated.

The paper measured on SPE10 permeability; SPE10 is not in this
container, so these seeded lognormal / correlated / layered fields stand in for
its heterogeneity.  None of SPE10's values are used.
"""
from __future__ import annotations

import numpy as np

from .twophase import Problem, CapillaryModel, DAY, G_ACC, jacobian, residual, BSR2

SEED0 = 1611000          # Q20: config c uses seed 1611000 + c, +100 for the S_n stream
P_INIT = 1e5             # Q13 (T1)


def _white(seed, shape):
    return np.random.Generator(np.random.PCG64(seed)).standard_normal(shape)


def _smooth_std(seed, shape, sigma):
    """Q19: PCG64 white noise, Gaussian filter (reflect, truncate 4), re-standardised."""
    from scipy.ndimage import gaussian_filter
    z = gaussian_filter(_white(seed, shape), sigma, mode="reflect", truncate=4.0)
    z -= z.mean()
    z /= z.std()
    return z


def _grid_shape(nx, ny, nz):
    return (nz, ny, nx)          # numpy (k, j, i) so that ravel() gives c = i + nx (j + ny k)


def make_problem(config: int, gravity: bool = True, dims=None) -> Problem:
    """Build configuration `config` (1..5).  `dims` optionally overrides the grid
    (same recipe on a smaller grid, used for tiny parity variants)."""
    c = config
    if c == 1:
        nx, ny, nz = dims or (32, 32, 1)
    elif c == 2:
        nx, ny, nz = dims or (64, 64, 64)
    elif c in (3, 4):
        nx, ny, nz = dims or (128, 128, 128)
    elif c == 5:
        nx, ny, nz = dims or (256, 256, 128)
    else:
        raise ValueError(config)
    n = nx * ny * nz
    shp = _grid_shape(nx, ny, nz)
    # gravity along the last axis with extent > 1 (Q12)
    gaxis = 2 if nz > 1 else (1 if ny > 1 else 0)
    dirichlet = [(0, 1, P_INIT)]                       # +x outlet (Q14)
    src = None
    dt = 1.0 * DAY
    if c == 1:
        perm = np.full(n, 1e-12)
        pc = CapillaryModel("bc", 5e3, 2.0)
        sn = np.random.Generator(np.random.PCG64(SEED0 + c + 100)).uniform(0.1, 0.9, n)
    elif c == 2:
        perm = 10.0 ** (-12.0 + 0.5 * _white(SEED0 + c, shp).ravel())
        pc = CapillaryModel("bc", 1e3, 2.0)
        sn = np.clip(0.5 + 0.2 * _smooth_std(SEED0 + c + 100, shp, 4.0).ravel(), 0.05, 0.95)
    elif c == 3:
        perm = 10.0 ** (-12.0 + 1.0 * _smooth_std(SEED0 + c, shp, 8.0).ravel())
        pc = CapillaryModel("vg", 2.0, 1e-4)
        sn = np.clip(0.5 + 0.2 * _smooth_std(SEED0 + c + 100, shp, 4.0).ravel(), 0.05, 0.95)
        dirichlet = [(0, 0, P_INIT), (0, 1, P_INIT)]
        # well column at the grid centre, 0.75 m^3/day of water split equally (Q16)
        src = np.zeros(n)
        kk = np.arange(nz)
        cells = (nx // 2) + nx * ((ny // 2) + ny * kk)
        src[cells] = 1000.0 * 0.75 / DAY / nz
    elif c == 4:
        kz = np.arange(n) // (nx * ny)
        perm = np.where((kz % 8) < 4, 1e-11, 1e-15)
        pc = CapillaryModel("bc", 5e4, 1.5)
        ii = np.arange(n) % nx
        sn = np.where(ii < 32, 0.8, 0.1)
        dt = 10.0 * DAY
    else:  # c == 5
        perm = 10.0 ** (-12.0 + 1.0 * _smooth_std(SEED0 + c, shp, 8.0).ravel())
        pc = CapillaryModel("bc", 1e4, 2.0)
        sn = np.clip(0.5 + 0.2 * _smooth_std(SEED0 + c + 100, shp, 4.0).ravel(), 0.05, 0.95)
    p = np.full(n, P_INIT)
    return Problem(nx=nx, ny=ny, nz=nz, perm=np.ascontiguousarray(perm, dtype=np.float64), pc=pc, dt=dt,
                   sn_old=np.ascontiguousarray(sn, dtype=np.float64), p_old=p.copy(),
                   g=G_ACC if gravity else 0.0, gravity_axis=gaxis, dirichlet=dirichlet, source_w=src)


def make_system(config: int, gravity: bool = True, dims=None):
    """J(u^n) and rhs = -R(u^n) in point-interleaved order (x[2c]=dp, x[2c+1]=dS)."""
    prob = make_problem(config, gravity, dims)
    p, sn = prob.p_old, prob.sn_old
    J = jacobian(prob, p, sn)
    rhs = -residual(prob, p, sn).reshape(-1)
    return prob, J, np.ascontiguousarray(rhs)


# Config names for reporting
CONFIG_NAMES = {
    1: "C1 2D 32x32 BC(5e3,2) homogeneous",
    2: "C2 64^3 lognormal(0.5) BC(1e3,2)",
    3: "C3 128^3 correlated lognormal(1.0) vG(2,1e-4) x-Dirichlet + well",
    4: "C4 128^3 layered 1e-11/1e-15 BC(5e4,1.5) front dt=10d",
    5: "C5 256x256x128 correlated lognormal BC(1e4,2)",
}
