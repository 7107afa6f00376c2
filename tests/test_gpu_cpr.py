"""GPU parity of the CPR-AMG(1)/(2) preconditioners (Algorithms 1, 2,
P:L159-193) through the C-ABI against the oracle: block ILU(0) factors and the A_pp hierarchy
bit-exact, ILU solve and one preconditioner apply <= 1e-10, GMRES iterations +-1, solution
<= 1e-6 per field (the BJ tolerances of the BF path)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle
from workload import make_system, seeded_vector, BSR2
from gpu_util import torch_dev, gpu_solver, csr_equal

CASES = [(1, None, True, 1), (1, None, True, 2), (1, (13, 7, 1), False, 2), (2, (12, 11, 9), True, 1),
         (3, (20, 17, 15), True, 2), (4, (40, 9, 16), True, 2), (2, (33, 30, 31), True, 1)]
IDS = ["C1-cpr1", "C1-cpr2", "C1-13x7-g0-cpr2", "C2-12x11x9-cpr1", "C3-20x17x15-cpr2", "C4-40x9x16-cpr2",
       "C2-33x30x31-cpr1"]


@pytest.fixture(scope="module", params=list(range(len(CASES))), ids=IDS)
def pair(request):
    config, dims, grav, pc = CASES[request.param]
    prob, J, rhs = make_system(config, gravity=grav, dims=dims)
    g = gpu_solver(J, prob.dims, precond=pc)
    o = oracle.BF(J, precond=pc)
    return prob, J, rhs, g, o, pc


def test_ilu_and_hierarchies_bit_exact(pair):
    prob, J, rhs, g, o, pc = pair
    lu, dinv, levels = g.ilu(J.nnzb)
    olu, odinv = o.ilu()
    assert np.array_equal(lu.view(np.uint64), olu.view(np.uint64))
    assert np.array_equal(dinv.view(np.uint64), odinv.view(np.uint64))
    nx, ny, nz = prob.dims
    assert levels == nx + ny + nz - 2  # dependency levels of the natural-order 5/7-point ILU(0)
    for which in ((2, 0) if pc == 2 else (2,)):
        nl = g.num_levels(which)
        assert nl == o.nlev(which)
        for l in range(nl):
            G, O = g.level(which, l), o.level(which, l)
            pat, val = csr_equal(G["A"], O["A"])
            assert pat and val, (which, l)
            if l < nl - 1:
                assert np.array_equal(G["cf"], O["cf"]), (which, l)
    if pc == 1:
        assert g.num_levels(0) == 0 and g.num_levels(1) == 0


def test_ilu_solve_and_apply(pair):
    prob, J, rhs, g, o, pc = pair
    N = 2 * J.n
    olu, odinv = o.ilu()
    for seed in (4, 5):
        r = seeded_vector(N, seed)
        xo = oracle.ilu0_solve(J, olu, odinv, r)
        x = torch.empty(N, dtype=torch.float64, device="cuda")
        g.ilu_solve(torch_dev(r), x)
        assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-12 * np.linalg.norm(xo)
    v = seeded_vector(N, 7)
    zo = o.apply(v)
    z = torch.empty(N, dtype=torch.float64, device="cuda")
    for _ in range(3):  # repeated applies reuse the sweep flags (epochs) and tickets
        g.apply_precond(torch_dev(v), z)
        assert np.linalg.norm(z.cpu().numpy() - zo) <= 1e-10 * np.linalg.norm(zo)


def test_gmres(pair):
    prob, J, rhs, g, o, pc = pair
    ro = o.gmres(rhs, tol=1e-8, restart=30, maxit=500)
    x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
    r = g.solve(torch_dev(rhs), x, tol=1e-8, restart=30, maxit=500)
    xg = x.cpu().numpy()
    assert r["converged"] == ro["converged"]
    assert abs(r["iters"] - ro["iters"]) <= 1, (r["iters"], ro["iters"])
    if ro["converged"]:
        assert np.linalg.norm(rhs - o.spmv(xg)) / np.linalg.norm(rhs) <= 1e-8
    for f in (0, 1):
        assert np.linalg.norm(xg[f::2] - ro["x"][f::2]) <= 1e-6 * np.linalg.norm(ro["x"][f::2])
    k = max(ro["iters"] - 1, 1)
    ro2 = o.gmres(rhs, tol=0.0, restart=30, maxit=k)
    x2 = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
    r2 = g.solve(torch_dev(rhs), x2, tol=0.0, restart=30, maxit=k)
    assert r2["iters"] == ro2["iters"] == k
    x2 = x2.cpu().numpy()
    for f in (0, 1):
        assert np.linalg.norm(x2[f::2] - ro2["x"][f::2]) <= 1e-6 * np.linalg.norm(ro2["x"][f::2])


def test_cpr_var_order_host_pointers_update_and_errors():
    from paper_1611_00127_b200 import BFError
    prob, J, rhs = make_system(1, dims=(9, 8, 1))
    o = oracle.BF(J, precond=2)
    ro = o.gmres(rhs, tol=1e-8)
    Jsw = BSR2(J.n, J.row_ptr, J.col_idx, np.ascontiguousarray(J.vals[:, ::-1, ::-1]))
    g = gpu_solver(Jsw, prob.dims, on_device=False, var_order=1, precond=2)
    x = np.zeros(2 * J.n)
    r = g.solve(np.ascontiguousarray(rhs.reshape(-1, 2)[:, ::-1].ravel()), x, tol=1e-8)
    assert abs(r["iters"] - ro["iters"]) <= 1
    xs = x.reshape(-1, 2)[:, ::-1].ravel()
    assert np.linalg.norm(xs - ro["x"]) <= 1e-6 * np.linalg.norm(ro["x"])
    # bf_update: new values on the same pattern -> ILU refactorised, A_pp coarse levels frozen
    prob2, J2, rhs2 = make_system(1, dims=(9, 8, 1), gravity=False)
    g = gpu_solver(J, prob.dims, precond=1)
    o = oracle.BF(J, precond=1)
    g.update(torch_dev(J2.vals.reshape(-1)))
    o.update(J2)
    lu, dinv, _ = g.ilu(J.nnzb)
    assert np.array_equal(lu.view(np.uint64), o.ilu()[0].view(np.uint64))
    v = seeded_vector(2 * J.n, 2)
    z = np.zeros(2 * J.n)
    g.apply_precond(v, z)
    zo = o.apply(v)
    assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo)
    # singular pivot block names the cell; bad precond value
    Jb = BSR2(J.n, J.row_ptr, J.col_idx, J.vals.copy())
    Jb.vals[J.row_ptr[5]:J.row_ptr[6]] = 0.0  # row 5 decoupled, its pivot block [[1,1],[1,1]]
    Jb.vals[J.row_ptr[5] + list(J.col_idx[J.row_ptr[5]:J.row_ptr[6]]).index(5)] = 1.0
    with pytest.raises(BFError, match="BF_ERR_ZERO_DIAG.*ILU.*cell 5"):
        gpu_solver(Jb, prob.dims, precond=1)
    with pytest.raises(BFError, match="BF_ERR_ARG.*precond"):
        gpu_solver(J, prob.dims, precond=4)
    # a BF handle has no ILU
    gb = gpu_solver(J, prob.dims)
    with pytest.raises(BFError, match="BF_ERR_ARG.*CPR"):
        gb.ilu(J.nnzb)
    with pytest.raises(BFError, match="BF_ERR_ARG.*hierarchy not built"):
        gb.vcycle(2, np.zeros(J.n), np.zeros(J.n))


def test_cpr_non_grid_pattern():
    """A Jacobian whose block pattern is not a grid stencil (random symmetric extra couplings):
    the CSR-BSR residual kernel and a non-trivial level schedule."""
    rng = np.random.default_rng(5)
    prob, J, rhs = make_system(1, dims=(10, 10, 1))
    D = J.to_dense()
    n = J.n
    A = [D[0::2, 0::2], D[0::2, 1::2], D[1::2, 0::2], D[1::2, 1::2]]
    for _ in range(40):
        i, j = rng.integers(0, n, 2)
        if i != j:
            for B in A:
                B[i, j] += 1e-3 * B[i, i]
    from test_oracle import bsr_from_dense_blocks
    Jr = bsr_from_dense_blocks(*A)
    o = oracle.BF(Jr, precond=2)
    g = gpu_solver(Jr, (n, 1, 1), precond=2)
    lu, dinv, levels = g.ilu(Jr.nnzb)
    assert np.array_equal(lu.view(np.uint64), o.ilu()[0].view(np.uint64))
    ro = o.gmres(rhs, tol=1e-8)
    x = np.zeros(2 * n)
    r = g.solve(rhs, x, tol=1e-8)
    assert abs(r["iters"] - ro["iters"]) <= 1
    assert np.linalg.norm(x - ro["x"]) <= 1e-6 * np.linalg.norm(ro["x"])


@pytest.mark.parametrize("config,dims", [(1, None), (2, (12, 11, 9)), (4, (20, 9, 8))])
def test_coupled_amg(config, dims):
    """precond 3 (coupled point AMG, R20): hierarchy of the scalar J bit-exact, one
    apply <= 1e-10, 40 forced GMRES iterations <= 1e-6 per field, same convergence verdict."""
    prob, J, rhs = make_system(config, dims=dims)
    g = gpu_solver(J, prob.dims, precond=3)
    o = oracle.BF(J, precond=3)
    assert g.num_levels(3) == o.nlev(3) > 1
    for l in range(o.nlev(3)):
        G, O = g.level(3, l), o.level(3, l)
        pat, val = csr_equal(G["A"], O["A"])
        assert pat and val, l
        if l < o.nlev(3) - 1:
            assert np.array_equal(G["cf"], O["cf"]), l
            pat, val = csr_equal(G["P"], O["P"])
            assert pat and val, l
    N = 2 * J.n
    v = seeded_vector(N, 9)
    zo = o.apply(v)
    z = torch.empty(N, dtype=torch.float64, device="cuda")
    g.apply_precond(torch_dev(v), z)
    assert np.linalg.norm(z.cpu().numpy() - zo) <= 1e-10 * np.linalg.norm(zo)
    ro = o.gmres(rhs, tol=0.0, restart=30, maxit=40)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    r = g.solve(torch_dev(rhs), x, tol=0.0, restart=30, maxit=40)
    assert r["iters"] == ro["iters"] == 40
    x = x.cpu().numpy()
    for f in (0, 1):
        assert np.linalg.norm(x[f::2] - ro["x"][f::2]) <= 1e-6 * np.linalg.norm(ro["x"][f::2])
    assert abs(r["relres"] - ro["relres"]) <= 1e-6 * ro["relres"]


def test_sweep_variants_bit_identical(monkeypatch):
    """The three ILU sweep implementations compute every row in the oracle's order: the
    pencil-wavefront sweeps (default on grid-structured J), the generic value-flag sweeps
    (BF_ILU_PENCIL=0) and the flag-array sweeps (BF_ILU_FLAGS=1) give bit-identical solves and
    applies, repeatedly (sentinels and tickets restored each time), on 3D and 2D grids."""
    for config, dims in ((2, (17, 13, 11)), (3, (40, 33, 21)), (1, (37, 23, 1))):
        prob, J, rhs = make_system(config, dims=dims)
        monkeypatch.delenv("BF_ILU_FLAGS", raising=False)
        monkeypatch.delenv("BF_ILU_PENCIL", raising=False)
        g_p = gpu_solver(J, prob.dims, precond=2)
        monkeypatch.setenv("BF_ILU_PENCIL", "0")
        g_v = gpu_solver(J, prob.dims, precond=2)
        monkeypatch.delenv("BF_ILU_PENCIL")
        monkeypatch.setenv("BF_ILU_FLAGS", "1")
        g_f = gpu_solver(J, prob.dims, precond=2)
        monkeypatch.delenv("BF_ILU_FLAGS")
        o = oracle.BF(J, precond=2)
        olu, odinv = o.ilu()
        N = 2 * J.n
        for seed in (1, 2):
            rn = seeded_vector(N, seed)
            r = torch_dev(rn)
            outs = []
            for g in (g_p, g_v, g_f):
                a = torch.empty(N, dtype=torch.float64, device="cuda")
                for _ in range(2):
                    g.ilu_solve(r, a)
                outs.append(a)
            assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2]), dims
            xo = oracle.ilu0_solve(J, olu, odinv, rn)
            assert np.linalg.norm(outs[0].cpu().numpy() - xo) <= 1e-12 * np.linalg.norm(xo)
            zs = []
            for g in (g_p, g_v, g_f):
                z = torch.empty(N, dtype=torch.float64, device="cuda")
                g.apply_precond(r, z)
                zs.append(z)
            assert torch.equal(zs[0], zs[1]) and torch.equal(zs[1], zs[2]), dims
        # GMRES through the graph-captured apply with the pencil sweeps
        x = torch.zeros(N, dtype=torch.float64, device="cuda")
        rg = g_p.solve(torch_dev(rhs), x, tol=1e-8, maxit=300)
        ro = o.gmres(rhs, tol=1e-8, maxit=300)
        assert abs(rg["iters"] - ro["iters"]) <= 1
        x = x.cpu().numpy()
        for f in (0, 1):
            assert np.linalg.norm(x[f::2] - ro["x"][f::2]) <= 1e-6 * np.linalg.norm(ro["x"][f::2])
