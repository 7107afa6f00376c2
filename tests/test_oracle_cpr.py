"""Pins of the oracle's CPR-AMG(1)/(2) preconditioners and their block ILU(0) (SURVEY 8(f)
NEXT-3; PAPER.md Algorithms 1 and 2).  These tests never touch the CUDA path.

ILU(0) is pinned by its defining property, not by a second implementation: the factors L
(unit block-lower) and U (block-upper) carry J's block pattern and (L U)_ij = J_ij at every
position (i, j) of that pattern [Saad, ILU(0)]; L and U with that pattern and property are
unique, so a dropped update, a wrong order or a transposed block product fails it."""
import numpy as np
import pytest

import oracle
from workload import make_system, seeded_vector

BIG = 10 ** 6  # max_coarse >= n: the V-cycle is the exact dense solve (single level)


def factors_dense(J, lu, dinv):
    n = J.n
    L = np.eye(2 * n)
    U = np.zeros((2 * n, 2 * n))
    for i in range(n):
        for q in range(J.row_ptr[i], J.row_ptr[i + 1]):
            k = J.col_idx[q]
            blk = L if k < i else U
            blk[2 * i:2 * i + 2, 2 * k:2 * k + 2] = lu[q]
        Uii = U[2 * i:2 * i + 2, 2 * i:2 * i + 2]
        assert np.all(np.abs(dinv[i] @ Uii - np.eye(2)) <= 1e-13 * (np.abs(dinv[i]) @ np.abs(Uii)))
    return L, U


def pattern_mask(J):
    n = J.n
    M = np.zeros((2 * n, 2 * n), bool)
    for i in range(n):
        for q in range(J.row_ptr[i], J.row_ptr[i + 1]):
            k = J.col_idx[q]
            M[2 * i:2 * i + 2, 2 * k:2 * k + 2] = True
    return M


CASES = [((4, 4, 1), 1), ((3, 3, 2), 2), ((5, 3, 1), 4), ((3, 2, 2), 3)]


@pytest.mark.parametrize("dims,config", CASES)
def test_ilu0_defining_property(dims, config):
    """(L U)_ij = J_ij on J's block pattern, L, U confined to it (P:L172 ILU(0), reading R18)."""
    prob, J, rhs = make_system(config, dims=dims)
    lu, dinv = oracle.ilu0(J)
    L, U = factors_dense(J, lu, dinv)
    D = J.to_dense()
    M = pattern_mask(J)
    LU = L @ U
    scale = np.max(np.abs(D))
    assert np.max(np.abs((LU - D)[M])) <= 1e-12 * scale
    # the product does carry fill outside the pattern (these are 2D/3D grids): ILU(0) != LU
    assert np.max(np.abs(LU[~M])) > 1e-8 * scale
    # the triangular solves invert exactly L U
    for seed in range(2):
        r = seeded_vector(2 * J.n, seed)
        x = oracle.ilu0_solve(J, lu, dinv, r)
        xd = np.linalg.solve(LU, r)
        assert np.linalg.norm(x - xd) <= 1e-12 * np.linalg.norm(xd)


def test_ilu0_exact_on_a_chain():
    """A 1D chain of cells has a block-tridiagonal J: no fill, so ILU(0) is the exact LU and the
    ILU solve is J^-1."""
    prob, J, rhs = make_system(1, dims=(12, 1, 1), gravity=False)
    lu, dinv = oracle.ilu0(J)
    L, U = factors_dense(J, lu, dinv)
    D = J.to_dense()
    assert np.max(np.abs(L @ U - D)) <= 1e-12 * np.max(np.abs(D))
    x = oracle.ilu0_solve(J, lu, dinv, rhs)
    xd = np.linalg.solve(D, rhs)
    for f in (0, 1):
        assert np.linalg.norm(x[f::2] - xd[f::2]) <= 1e-10 * np.linalg.norm(xd[f::2])


def test_ilu0_singular_pivot_names_cell():
    prob, J, rhs = make_system(1, dims=(3, 3, 1))
    J.vals[J.row_ptr[4]:J.row_ptr[5]] = 0.0  # every block of cell 4's row, pivot included
    with pytest.raises(RuntimeError, match="cell 4"):
        oracle.ilu0(J)


@pytest.mark.parametrize("precond", [1, 2])
def test_cpr_equals_matrix_form(precond):
    """Algorithms 1/2 with exact inner solves equal M_comb^-1 / M_add^-1 of `m_comb`, `m_add`
    (P:L186-191): (I - (R_p^T A_pp^-1 R_p [+ R_s^T A_ss^-1 R_s]) (J - P_1)) P_1^-1 r, P_1 = L U."""
    for dims, config in (((4, 4, 1), 1), ((3, 3, 2), 4)):
        prob, J, rhs = make_system(config, dims=dims)
        o = oracle.BF(J, precond=precond, max_coarse=BIG)
        assert o.nlev(2) == 1 and (o.nlev(0) == 1) == (precond == 2)
        n = J.n
        lu, dinv = o.ilu()
        L, U = factors_dense(J, lu, dinv)
        P1 = L @ U
        D = J.to_dense()
        App, Ass = o.matrix("App").to_dense(), o.matrix("Ass").to_dense()
        Rp = np.zeros((n, 2 * n)); Rp[np.arange(n), 2 * np.arange(n)] = 1
        Rs = np.zeros((n, 2 * n)); Rs[np.arange(n), 2 * np.arange(n) + 1] = 1
        C = Rp.T @ np.linalg.inv(App) @ Rp
        if precond == 2:
            C = C + Rs.T @ np.linalg.inv(Ass) @ Rs
        Minv = (np.eye(2 * n) - C @ (D - P1)) @ np.linalg.inv(P1)
        for seed in range(3):
            v = seeded_vector(2 * n, seed)
            z = o.apply(v)
            zd = Minv @ v
            for f in (0, 1):
                assert np.linalg.norm(z[f::2] - zd[f::2]) <= 1e-10 * np.linalg.norm(zd[f::2])


@pytest.mark.parametrize("precond", [1, 2])
def test_cpr_exact_when_ilu_is_exact(precond):
    """1D chain: P_1 = J, so u = J^-1 r and the residual of step 3 vanishes: M^-1 = J^-1 and
    GMRES converges in one iteration."""
    prob, J, rhs = make_system(1, dims=(16, 1, 1))
    r = oracle.BF(J, precond=precond).gmres(rhs, tol=1e-10)
    assert r["converged"] and r["iters"] == 1


@pytest.mark.parametrize("precond", [1, 2])
def test_cpr_gmres_converges_and_manufactured(precond):
    """CPR-AMG-GMRES reaches tol on C1 with non-increasing estimates; manufactured solution
    b = J x* recovered (BJ check 4 with the CPR preconditioners)."""
    prob, J, rhs = make_system(1)
    o = oracle.BF(J, precond=precond)
    r = o.gmres(rhs, tol=1e-8)
    assert r["converged"] and r["relres"] <= 1e-8
    assert np.all(np.diff(r["hist"]) <= 1e-15)
    for config, dims in ((1, (8, 8, 1)), (2, (5, 5, 4))):
        prob, J, rhs = make_system(config, dims=dims)
        D = J.to_dense()
        xs = seeded_vector(2 * J.n, 7)
        b = D @ xs
        r = oracle.BF(J, precond=precond).gmres(b, tol=1e-12, maxit=400)
        assert r["converged"]
        kappa = np.linalg.cond(D)
        assert np.linalg.norm(r["x"] - xs) / np.linalg.norm(xs) <= 10 * kappa * 1e-12
        assert np.linalg.norm(b - D @ r["x"]) / np.linalg.norm(b) <= 1e-12


def test_cpr_var_order_and_update():
    """var_order=1 (S_n first) gives the permuted result; bf_update semantics (R16) for CPR:
    the ILU(0) is recomputed from the new values, the A_pp coarse levels stay frozen."""
    prob, J, rhs = make_system(1, dims=(6, 5, 1))
    o = oracle.BF(J, precond=2)
    v = seeded_vector(2 * J.n, 3)
    z = o.apply(v)
    from workload import BSR2
    Js = BSR2(J.n, J.row_ptr, J.col_idx, np.ascontiguousarray(J.vals[:, ::-1, ::-1]))
    z1 = oracle.BF(Js, var_order=1, precond=2).apply(v.reshape(-1, 2)[:, ::-1].reshape(-1))
    assert np.array_equal(z1.reshape(-1, 2)[:, ::-1].reshape(-1), z)
    prob2, J2, _ = make_system(1, dims=(6, 5, 1), gravity=False)
    assert np.array_equal(J2.col_idx, J.col_idx)
    lev1 = o.level(2, 1)["A"].to_dense() if o.nlev(2) > 1 else None
    o.update(J2)
    lu, dinv = o.ilu()
    lu2, dinv2 = oracle.ilu0(J2)
    assert np.array_equal(lu, lu2) and np.array_equal(dinv, dinv2)
    assert np.array_equal(o.level(2, 0)["A"].to_dense(), oracle.split(J2)["App"].to_dense())
    if lev1 is not None:
        assert np.array_equal(o.level(2, 1)["A"].to_dense(), lev1)


# ---------------------------------------------------------------------------- coupled point AMG
def test_jscalar_is_point_ordered_J():
    """The scalar matrix handed to the coupled AMG (reading R20) is J in point
    ordering: dense-equal to the BSR J, pattern = nonzero entries plus the diagonal."""
    prob, J, rhs = make_system(1, dims=(6, 5, 1))
    A = oracle.jscalar(J)
    D = J.to_dense()
    assert np.array_equal(A.to_dense(), D)
    nz = (D != 0) | np.eye(2 * J.n, dtype=bool)
    assert A.nnz == int(nz.sum())
    assert np.all(np.diff(A.ci[A.rp[0]:A.rp[1]]) > 0)


def test_coupled_amg_exact_single_level_and_fails_on_transport():
    """precond 3 with a single-level hierarchy is the exact solve (1 GMRES iteration); with the
    default hierarchy it does not converge on the two-phase C1 Jacobian (the paper's finding,
    P:L453 "Since AMG does not converge in this experiment")."""
    prob, J, rhs = make_system(1, dims=(8, 6, 1))
    r = oracle.BF(J, precond=3, max_coarse=BIG).gmres(rhs, tol=1e-10)
    assert r["converged"] and r["iters"] == 1
    prob, J, rhs = make_system(1)
    o = oracle.BF(J, precond=3)
    assert o.nlev(3) > 1
    v = seeded_vector(2 * J.n, 1)
    assert np.array_equal(o.apply(v), o.vcycle(3, v))
    r = o.gmres(rhs, tol=1e-8, maxit=200)
    assert not r["converged"]
