"""Pins of the seeded workload generator (SURVEY.md c.5 "Generator" rows, BASELINE.json
north_star oracle check 1: the Jacobian against finite differences of the residual)."""
import os
import numpy as np
import pytest

from workload import (Problem, CapillaryModel, residual, jacobian, harmonic_face_perm,
                      make_system, DAY)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "constitutive.txt")


def test_constitutive_golden():
    n_checked = 0
    for line in open(GOLDEN):
        line = line.split("#")[0].split()
        if not line:
            continue
        kind = line[0]
        if kind == "harmonic":
            ki, kj, exp, tol = map(float, line[1:5])
            got = float(harmonic_face_perm(ki, kj))
        else:
            a, b, s, exp, tol = map(float, line[1:6])
            got = float(CapillaryModel(kind, a, b).pc_and_deriv(np.array([s]))[0][0])
        assert abs(got - exp) <= tol * max(abs(exp), 1e-300), (line, got)
        n_checked += 1
    assert n_checked >= 7


def test_harmonic_properties():
    rng = np.random.default_rng(0)
    a, b = 10 ** rng.uniform(-15, -11, 100), 10 ** rng.uniform(-15, -11, 100)
    h = harmonic_face_perm(a, b)
    assert np.allclose(h, harmonic_face_perm(b, a), rtol=1e-15)
    assert np.all(h >= np.minimum(a, b) * (1 - 1e-14)) and np.all(h <= np.maximum(a, b) * (1 + 1e-14))
    # unequal cell sizes, P:L77 general form vs series-resistance closed form
    assert np.isclose(harmonic_face_perm(2.0, 1.0, 1.0, 3.0), 4.0 / (1.0 / 2.0 + 3.0 / 1.0))


@pytest.mark.parametrize("kind,a,b", [("bc", 5e3, 2.0), ("vg", 2.0, 1e-4), ("bc", 5e4, 1.5), ("linear", 1e4, 0)])
def test_pc_derivative_fd(kind, a, b):
    m = CapillaryModel(kind, a, b)
    s = np.linspace(0.05, 0.95, 37)
    h = 1e-7
    fd = (m.pc_and_deriv(s + h)[0] - m.pc_and_deriv(s - h)[0]) / (2 * h)
    d = m.pc_and_deriv(s)[1]
    assert np.max(np.abs(fd - d) / np.abs(d)) < 1e-6
    assert np.all(np.diff(m.pc_and_deriv(s)[0]) <= 0)   # non-increasing in S_w


def _random_problem(dims, seed, pc, gravity=True, dirichlet=True, source=True):
    nx, ny, nz = dims
    n = nx * ny * nz
    rng = np.random.default_rng(seed)
    perm = 10 ** rng.uniform(-13, -11, n)
    sn_old = rng.uniform(0.2, 0.8, n)
    gaxis = 2 if nz > 1 else 1
    src = rng.uniform(0, 1e-3, n) if source else None
    prob = Problem(nx=nx, ny=ny, nz=nz, perm=perm, pc=pc, dt=2 * DAY, sn_old=sn_old,
                   p_old=np.full(n, 1e5), g=9.80665 if gravity else 0.0, gravity_axis=gaxis,
                   dirichlet=[(0, 1, 1e5)] if dirichlet else [], source_w=src)
    p = 1e5 + rng.uniform(-3e3, 3e3, n)     # tie-free random state (Q7)
    sn = rng.uniform(0.15, 0.85, n)
    return prob, p, sn


@pytest.mark.parametrize("dims", [(4, 4, 1), (3, 3, 3)])
@pytest.mark.parametrize("pc", [CapillaryModel("bc", 5e3, 2.0), CapillaryModel("vg", 2.0, 1e-4)])
def test_jacobian_finite_difference(dims, pc):
    """BJ oracle check 1: central FD of R, step 1e-6 (1+|u|), max rel error <= 1e-5."""
    prob, p, sn = _random_problem(dims, 7, pc)
    J = jacobian(prob, p, sn).to_dense()
    n = prob.n
    u = np.stack([p, sn], 1).reshape(-1)

    def R(uu):
        uu = uu.reshape(n, 2)
        return residual(prob, uu[:, 0].copy(), uu[:, 1].copy()).reshape(-1)

    worst = 0.0
    for j in range(2 * n):
        h = 1e-6 * (1 + abs(u[j]))
        e = np.zeros(2 * n)
        e[j] = h
        col = (R(u + e) - R(u - e)) / (2 * h)
        scale = np.max(np.abs(J[:, j]))
        worst = max(worst, np.max(np.abs(col - J[:, j])) / scale)
    assert worst <= 1e-5, worst


def _blocks(J):
    D = J.to_dense()
    return D[0::2, 0::2], D[0::2, 1::2], D[1::2, 0::2], D[1::2, 1::2]


def test_sign_structure():
    """SURVEY c.1 'Sign structure' invariants on a generated Jacobian with gravity and an outlet."""
    prob, J, rhs = make_system(1, dims=(12, 10, 1))
    App, Aps, Asp, Ass = _blocks(J)
    V = prob.h ** 3
    off = ~np.eye(prob.n, dtype=bool)
    for A in (App, Asp):
        assert np.allclose(A, A.T, rtol=1e-13, atol=0)
        assert np.all(A[off] <= 0)
    outlet = (np.arange(prob.n) % prob.nx) == prob.nx - 1
    rs = App.sum(1)
    assert np.all(np.abs(rs[~outlet]) <= 1e-12 * np.abs(App).sum(1)[~outlet])
    assert np.all(rs[outlet] > 0)
    assert np.all(Ass[off] <= 0) and np.all(np.diag(Ass) >= V * prob.phi * prob.rho_n * (1 - 1e-14))
    assert np.all(Aps[off] >= 0) and np.all(np.diag(Aps) <= -V * prob.phi * prob.rho_w * (1 - 1e-14))


def test_null_vectors_no_flow():
    """Under no-flow (no Dirichlet face): J (1;0) = 0 and y^T J = 0, y = (1/rho_w, 1/rho_n) (SURVEY c.1)."""
    prob, p, sn = _random_problem((5, 4, 3), 3, CapillaryModel("bc", 5e3, 2.0), dirichlet=False, source=False)
    J = jacobian(prob, p, sn).to_dense()
    one0 = np.tile([1.0, 0.0], prob.n)
    y = np.tile([1 / prob.rho_w, 1 / prob.rho_n], prob.n)
    assert np.max(np.abs(J @ one0)) <= 1e-12 * np.max(np.abs(J))
    assert np.max(np.abs(y @ J)) <= 1e-12 * np.max(np.abs(J)) / prob.rho_n


def test_residual_equilibrium_and_conservation():
    # uniform state, g = 0, no sources, no-flow -> R == 0
    n = 27
    prob = Problem(nx=3, ny=3, nz=3, perm=np.full(n, 1e-12), pc=CapillaryModel("bc", 5e3, 2.0), dt=DAY,
                   sn_old=np.full(n, 0.4), p_old=np.full(n, 1e5), g=0.0, gravity_axis=None)
    assert np.all(residual(prob, np.full(n, 1e5), np.full(n, 0.4)) == 0.0)
    # conservation: sum_c R = sum accumulation + dt (boundary flux - sources)
    prob, p, sn = _random_problem((4, 3, 2), 5, CapillaryModel("bc", 5e3, 2.0))
    R = residual(prob, p, sn)
    prob2 = Problem(**{**prob.__dict__, "dirichlet": [], "source_w": None, "dt": 0.0})
    acc = residual(prob2, p, sn)
    src = prob.dt * prob.source_w
    # boundary contribution: difference between with-outlet and without-outlet residual at dt
    prob3 = Problem(**{**prob.__dict__, "source_w": None})
    prob4 = Problem(**{**prob.__dict__, "source_w": None, "dirichlet": []})
    bnd = residual(prob3, p, sn) - residual(prob4, p, sn)
    tot = R.sum(0)
    exp = acc.sum(0) + bnd.sum(0) - np.array([src.sum(), 0.0])
    assert np.allclose(tot, exp, rtol=1e-12, atol=1e-12 * np.abs(R).sum())
    # interior fluxes telescope: no-outlet, no-source residual sums to accumulation only
    assert np.allclose(residual(prob4, p, sn).sum(0), acc.sum(0), rtol=1e-12, atol=1e-12 * np.abs(R).sum())


def test_dt_doubles_flux_part():
    prob, p, sn = _random_problem((4, 4, 1), 9, CapillaryModel("bc", 5e3, 2.0))
    prob0 = Problem(**{**prob.__dict__, "dt": 0.0})
    prob2 = Problem(**{**prob.__dict__, "dt": 2 * prob.dt})
    f1 = residual(prob, p, sn) - residual(prob0, p, sn)
    f2 = residual(prob2, p, sn) - residual(prob0, p, sn)
    assert np.allclose(f2, 2 * f1, rtol=1e-12, atol=1e-9)


def test_bsr_structure_and_permutation_roundtrip():
    prob, J, rhs = make_system(2, dims=(5, 4, 3))
    # strictly ascending columns, diagonal present, every structural block present (7-point)
    for r in range(J.n):
        cols = J.col_idx[J.row_ptr[r]:J.row_ptr[r + 1]]
        assert np.all(np.diff(cols) > 0) and r in cols
    nf = (4 * 4 * 3) + (5 * 3 * 3) + (5 * 4 * 2)
    assert J.nnzb == J.n + 2 * nf
    # point <-> variable-blocked permutation
    D = J.to_dense()
    perm = np.concatenate([np.arange(0, 2 * J.n, 2), np.arange(1, 2 * J.n, 2)])
    Dv = D[np.ix_(perm, perm)]
    inv = np.argsort(perm)
    assert np.array_equal(Dv[np.ix_(inv, inv)], D)
    assert np.array_equal(Dv[:J.n, :J.n], D[0::2, 0::2])


def test_config_sizes():
    for c, (n, nnzb) in {1: (1024, 4992)}.items():
        prob, J, rhs = make_system(c)
        assert J.n == n and J.nnzb == nnzb
