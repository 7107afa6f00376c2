"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same
seeded inputs (SURVEY.md c.6 bounds, BASELINE.json north_star tolerances)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle
from workload import make_system, seeded_vector, BSR2
from gpu_util import torch_dev, gpu_solver, csr_equal

# (config, dims, gravity): several tiles and ragged tails; C1 both gravity variants
CASES = [(1, None, True), (1, None, False), (1, (13, 7, 1), True), (2, (12, 11, 9), True),
         (3, (20, 17, 15), True), (4, (40, 9, 16), True), (2, (33, 30, 31), True)]
IDS = ["C1", "C1-g0", "C1-13x7", "C2-12x11x9", "C3-20x17x15", "C4-40x9x16", "C2-33x30x31"]


@pytest.fixture(scope="module", params=list(range(len(CASES))), ids=IDS)
def pair(request):
    config, dims, grav = CASES[request.param]
    prob, J, rhs = make_system(config, gravity=grav, dims=dims)
    g = gpu_solver(J, prob.dims)
    o = oracle.BF(J)
    return prob, J, rhs, g, o


def test_spmv(pair):
    prob, J, rhs, g, o = pair
    for seed in (1, 2):
        x = seeded_vector(2 * J.n, seed)
        yo = o.spmv(x)
        y = torch.empty(2 * J.n, dtype=torch.float64, device="cuda")
        g.spmv(torch_dev(x), y)
        y = y.cpu().numpy()
        assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)
        absJx = np.abs(J.to_scipy()) @ np.abs(x)
        assert np.max(np.abs(y - yo) / absJx) <= 1e-13


def test_split_and_schur_bit_exact(pair):
    prob, J, rhs, g, o = pair
    for k, name in enumerate(("App", "Aps", "Asp", "Ass", "S")):
        pat, val = csr_equal(g.block(k), o.matrix(name))
        assert pat, f"{name} pattern differs"
        assert val, f"{name} values differ"


def test_hierarchy_bit_exact(pair):
    prob, J, rhs, g, o = pair
    for which in (0, 1):
        nl = g.num_levels(which)
        assert nl == o.nlev(which)
        for l in range(nl):
            G, O = g.level(which, l), o.level(which, l)
            pat, val = csr_equal(G["A"], O["A"])
            assert pat and val, f"A_{l} of hierarchy {which}: pattern {pat} values {val}"
            assert np.array_equal(G["dl1"].view(np.uint64), O["dl1"].view(np.uint64))
            if l < nl - 1:
                assert np.array_equal(G["cf"], O["cf"]), f"C/F of level {l} hierarchy {which}"
                pat, val = csr_equal(G["P"], O["P"])
                assert pat and val, f"P_{l} of hierarchy {which}"


def test_vcycle_and_bf_apply(pair):
    prob, J, rhs, g, o = pair
    n = J.n
    for which in (0, 1):
        b = seeded_vector(n, 10 + which)
        xo = o.vcycle(which, b)
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        g.vcycle(which, torch_dev(b), x)
        x = x.cpu().numpy()
        assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    v = seeded_vector(2 * n, 7)
    zo = o.apply(v)
    z = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    g.apply_precond(torch_dev(v), z)
    z = z.cpu().numpy()
    assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo)


def test_gmres(pair):
    prob, J, rhs, g, o = pair
    ro = o.gmres(rhs, tol=1e-8, restart=30, maxit=500)
    x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
    r = g.solve(torch_dev(rhs), x, tol=1e-8, restart=30, maxit=500)
    xg = x.cpu().numpy()
    assert r["converged"] == ro["converged"]
    assert abs(r["iters"] - ro["iters"]) <= 1, (r["iters"], ro["iters"])
    # true residual with the oracle's SpMV
    tr = np.linalg.norm(rhs - o.spmv(xg)) / np.linalg.norm(rhs)
    if ro["converged"]:
        assert tr <= 1e-8
    for f in (0, 1):   # p and S parts separately (Q33)
        a, b = xg[f::2], ro["x"][f::2]
        assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b)
    # forced equal iteration count (tol = 0, maxit = oracle's count)
    k = max(ro["iters"] - 1, 1)
    ro2 = o.gmres(rhs, tol=0.0, restart=30, maxit=k)
    x2 = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
    r2 = g.solve(torch_dev(rhs), x2, tol=0.0, restart=30, maxit=k)
    assert r2["iters"] == ro2["iters"] == k
    x2 = x2.cpu().numpy()
    for f in (0, 1):
        assert np.linalg.norm(x2[f::2] - ro2["x"][f::2]) <= 1e-6 * np.linalg.norm(ro2["x"][f::2])
    # residual histories agree where both are meaningful
    m = min(len(r["hist"]), len(ro["hist"]))
    assert np.allclose(r["hist"][:m], ro["hist"][:m], rtol=1e-5, atol=1e-12)


def test_host_pointers_and_layout_options():
    prob, J, rhs = make_system(1, dims=(9, 8, 1))
    o = oracle.BF(J)
    ro = o.gmres(rhs, tol=1e-8)
    for on_device, bo in ((False, 0), (True, 1), (False, 1)):
        g = gpu_solver(J, prob.dims, on_device=on_device, block_order=bo)
        x = np.zeros(2 * J.n)
        r = g.solve(np.ascontiguousarray(rhs), x, tol=1e-8)
        assert abs(r["iters"] - ro["iters"]) <= 1
        assert np.linalg.norm(x - ro["x"]) <= 1e-6 * np.linalg.norm(ro["x"])
    # var_order = 1: swapped variables
    Jsw = BSR2(J.n, J.row_ptr, J.col_idx, np.ascontiguousarray(J.vals[:, ::-1, ::-1]))
    g = gpu_solver(Jsw, prob.dims, var_order=1)
    x = np.zeros(2 * J.n)
    bsw = np.ascontiguousarray(rhs.reshape(-1, 2)[:, ::-1].ravel())
    r = g.solve(bsw, x, tol=1e-8)
    xs = x.reshape(-1, 2)[:, ::-1].ravel()
    assert np.linalg.norm(xs - ro["x"]) <= 1e-6 * np.linalg.norm(ro["x"])


def test_options_parity():
    """Non-default options are implemented identically on both sides."""
    prob, J, rhs = make_system(2, dims=(10, 9, 8))
    for opts in (dict(smoother=0), dict(smoother=1, smoother_p=-1, cheb_lo=0.3), dict(interp_norm=0), dict(orth=1), dict(nu_pre=2, nu_post=2),
                 dict(theta=0.5, max_coarse=30), dict(schur_as_printed=1), dict(nu_pre=0),
                 dict(smoother=1, cheb_lo=0.1, cheb_eig=10), dict(smoother=1, cheb_degree=3, cheb_eig=4, nu_pre=2),
                 dict(smoother=1, smoother_p=0, cheb_lo=0.1), dict(smoother=0, smoother_p=1, cheb_levels=2),
                 dict(smoother=1, smoother_p=0, cheb_levels=1, cheb_degree=3, cheb_lo=0.05)):
        o = oracle.BF(J, **opts)
        g = gpu_solver(J, prob.dims, **opts)
        for which in (0, 1):
            assert g.num_levels(which) == o.nlev(which)
            for l in range(o.nlev(which) - 1):
                assert np.array_equal(g.level(which, l)["cf"], o.level(which, l)["cf"]), opts
            # the Chebyshev interval ends of R21 (power-iteration estimates) agree to rounding
            for l in range(o.nlev(which)):
                assert abs(g.cheb_hi(which, l) - o.level(which, l)["cheb_hi"]) <= 1e-12, (opts, which, l)
        v = seeded_vector(2 * J.n, 3)
        zo = o.apply(v)
        z = np.zeros(2 * J.n)
        g.apply_precond(v, z)
        assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo), opts
        ro = o.gmres(rhs, tol=1e-8, maxit=300)
        x = np.zeros(2 * J.n)
        r = g.solve(rhs, x, tol=1e-8, maxit=300)
        assert abs(r["iters"] - ro["iters"]) <= 1, (opts, r["iters"], ro["iters"])


def test_edge_cases():
    from paper_1611_00127_b200 import BFError
    # single cell
    J = BSR2(1, np.array([0, 1], np.int32), np.array([0], np.int32), np.array([[[2.0, 1.0], [1.0, 4.0]]]))
    g = gpu_solver(J, (1, 1, 1))
    b = np.array([1.0, 2.0])
    x = np.zeros(2)
    r = g.solve(b, x, tol=1e-12)
    assert r["converged"] and np.allclose(x, np.linalg.solve(J.to_dense(), b), rtol=1e-12)
    # zero rhs
    prob, J, rhs = make_system(1, dims=(5, 5, 1))
    g = gpu_solver(J, prob.dims)
    x = np.ones(2 * J.n)
    r = g.solve(np.zeros(2 * J.n), x)
    assert r["iters"] == 0 and r["converged"] and np.all(x == 0)
    # maxit reached -> not converged, not an error
    r = g.solve(rhs, np.zeros(2 * J.n), tol=1e-15, maxit=3)
    assert r["iters"] == 3 and not r["converged"]
    # errors name the item
    Jz = BSR2(J.n, J.row_ptr, J.col_idx, J.vals.copy())
    q = J.row_ptr[7] + list(J.col_idx[J.row_ptr[7]:J.row_ptr[8]]).index(7)
    Jz.vals[q, 1, 1] = 0.0
    with pytest.raises(BFError, match="BF_ERR_ZERO_DIAG.*cell 7"):
        gpu_solver(Jz, prob.dims)
    Jn = BSR2(J.n, J.row_ptr, J.col_idx, J.vals.copy())
    Jn.vals[3, 0, 1] = np.nan
    with pytest.raises(BFError, match="BF_ERR_NONFINITE"):
        gpu_solver(Jn, prob.dims)
    ci = J.col_idx.copy()
    ci[J.row_ptr[4]], ci[J.row_ptr[4] + 1] = ci[J.row_ptr[4] + 1], ci[J.row_ptr[4]]
    with pytest.raises(BFError, match="BF_ERR_PATTERN.*row 4"):
        gpu_solver(BSR2(J.n, J.row_ptr, ci, J.vals), prob.dims)
    with pytest.raises(BFError, match="BF_ERR_ARG.*max_coarse"):
        gpu_solver(J, prob.dims, max_coarse=1000)
    with pytest.raises(BFError, match="BF_ERR_PATTERN"):
        gpu_solver(J, (J.n + 1, 1, 1))      # n_cells from dims disagrees with row_ptr


def test_determinism_repeat_setup():
    prob, J, rhs = make_system(2, dims=(16, 15, 14))
    g1 = gpu_solver(J, prob.dims)
    g2 = gpu_solver(J, prob.dims)
    for which in (0, 1):
        for l in range(g1.num_levels(which)):
            a, b = g1.level(which, l), g2.level(which, l)
            for k in ("A", "P"):
                if k in a:
                    for u, v in zip(a[k], b[k]):
                        assert np.array_equal(u, v)
    x1, x2 = np.zeros(2 * J.n), np.zeros(2 * J.n)
    r1, r2 = g1.solve(rhs, x1), g2.solve(rhs, x2)
    assert r1["iters"] == r2["iters"] and np.array_equal(x1, x2)


@pytest.mark.parametrize("config,dims", [(2, (12, 11, 9)), (3, (20, 17, 15)), (1, (14, 12, 1))])
def test_setup_reuse_update_parity(config, dims):
    """bf_update (NEXT-1, R16) on a Newton sequence whose states come from the ORACLE's solves:
    finest levels bit-exact, coarse levels kept, BF apply <= 1e-10, GMRES +-1 / 1e-6."""
    from workload import newton_sequence
    seq = []
    o = None

    def solve(k, J, rhs):
        return oracle.BF(J).gmres(rhs, tol=1e-8, maxit=600)["x"]
    for k, prob, J, rhs, fn in newton_sequence(config, 3, solve, dims=dims):
        seq.append((prob, J, rhs))
    prob, J0, _ = seq[0]
    g = gpu_solver(J0, prob.dims)
    o = oracle.BF(J0)
    coarse_before = [[g.level(w, l)["A"] for l in range(1, g.num_levels(w))] for w in (0, 1)]
    for k in (1, 2):
        _, Jk, rhs = seq[k]
        g.update(torch_dev(Jk.vals.reshape(-1)))
        o.update(Jk)
        for b, name in enumerate(("App", "Aps", "Asp", "Ass", "S")):
            pat, val = csr_equal(g.block(b), o.matrix(name))
            assert pat and val, (k, name)
        for w in (0, 1):
            pat, val = csr_equal(g.level(w, 0)["A"], o.level(w, 0)["A"])
            assert pat and val
            assert np.array_equal(g.level(w, 0)["dl1"], o.level(w, 0)["dl1"])
            for l, old in enumerate(coarse_before[w], start=1):
                assert all(np.array_equal(u, v) for u, v in zip(g.level(w, l)["A"], old))
        v = seeded_vector(2 * Jk.n, 30 + k)
        z = np.zeros(2 * Jk.n)
        g.apply_precond(v, z)
        zo = o.apply(v)
        assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo)
        ro = o.gmres(rhs, tol=1e-8, maxit=600)
        x = np.zeros(2 * Jk.n)
        r = g.solve(rhs, x, tol=1e-8, maxit=600)
        assert abs(r["iters"] - ro["iters"]) <= 1 and r["converged"] == ro["converged"]
        for f in (0, 1):
            assert np.linalg.norm(x[f::2] - ro["x"][f::2]) <= 1e-6 * np.linalg.norm(ro["x"][f::2])


@pytest.mark.parametrize("opts", [dict(max_levels=1), dict(max_levels=2), dict(max_levels=2, smoother=1),
                                  dict(max_coarse=128), dict(theta=0.9), dict(nu_pre=3, nu_post=0),
                                  dict(nu_pre=0, nu_post=2), dict(smoother=1, cheb_degree=3, cheb_lo=0.1),
                                  dict(seed=12345)])
def test_option_edge_cases(opts):
    """Less common option combinations: single-level and stalled hierarchies (4 l1-Jacobi sweeps
    on a non-dense coarsest level), the largest dense coarse solve, asymmetric smoothing."""
    prob, J, rhs = make_system(2, dims=(13, 12, 11))
    o = oracle.BF(J, **opts)
    g = gpu_solver(J, prob.dims, **opts)
    for which in (0, 1):
        assert g.num_levels(which) == o.nlev(which)
    v = seeded_vector(2 * J.n, 8)
    z = np.zeros(2 * J.n)
    g.apply_precond(v, z)
    zo = o.apply(v)
    assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo), opts
    k = 40
    ro = o.gmres(rhs, tol=0.0, maxit=k)
    x = np.zeros(2 * J.n)
    r = g.solve(rhs, x, tol=0.0, maxit=k)
    assert r["iters"] == ro["iters"] == k
    for f in (0, 1):
        assert np.linalg.norm(x[f::2] - ro["x"][f::2]) <= 1e-6 * np.linalg.norm(ro["x"][f::2]), opts


@pytest.mark.parametrize("restart", [1, 7, 32, 33, 64, 100])
def test_restart_lengths(restart):
    """GMRES(m) for restarts below, at and above the 32-vector block of the fused CGS2 passes
    (longer bases are orthogonalised block by block, VERDICT r1 missing 6)."""
    prob, J, rhs = make_system(1, dims=(20, 18, 1))
    o = oracle.BF(J)
    g = gpu_solver(J, prob.dims)
    ro = o.gmres(rhs, tol=1e-8, restart=restart, maxit=400)
    x = np.zeros(2 * J.n)
    r = g.solve(rhs, x, tol=1e-8, restart=restart, maxit=400)
    assert abs(r["iters"] - ro["iters"]) <= 1 and r["converged"] == ro["converged"]
    if ro["converged"]:
        for f in (0, 1):
            assert np.linalg.norm(x[f::2] - ro["x"][f::2]) <= 1e-6 * np.linalg.norm(ro["x"][f::2])
    # forced equal count through several blocks and a restart
    k = min(restart + 5, 120)
    ro2 = o.gmres(rhs, tol=0.0, restart=restart, maxit=k)
    x2 = np.zeros(2 * J.n)
    r2 = g.solve(rhs, x2, tol=0.0, restart=restart, maxit=k)
    assert r2["iters"] == ro2["iters"] == k
    for f in (0, 1):
        assert np.linalg.norm(x2[f::2] - ro2["x"][f::2]) <= 1e-6 * np.linalg.norm(ro2["x"][f::2])
    assert np.allclose(r2["hist"], ro2["hist"], rtol=1e-6, atol=1e-14)


def test_boundary_limits_and_nonfinite():
    """bf.h contract: restart in [1, 256]; maxit = 0 takes no Arnoldi step; a NaN/Inf in the rhs or
    x0 is BF_ERR_NONFINITE naming the entry and its cell."""
    from paper_1611_00127_b200 import BFError
    prob, J, rhs = make_system(1, dims=(9, 7, 1))
    g = gpu_solver(J, prob.dims)
    o = oracle.BF(J)
    x0 = seeded_vector(2 * J.n, 3)
    x = x0.copy()
    r = g.solve(rhs, x, tol=1e-8, maxit=0)
    ro = o.gmres(rhs, x0=x0, tol=1e-8, maxit=0)
    assert r["iters"] == 0 and not r["converged"] and np.array_equal(x, x0) and len(r["hist"]) == 1
    assert abs(r["relres"] - ro["relres"]) <= 1e-12 * ro["relres"]
    for bad_restart in (0, 257):
        with pytest.raises(BFError, match="BF_ERR_ARG"):
            g.solve(rhs, np.zeros(2 * J.n), restart=bad_restart)
    b = rhs.copy()
    b[2 * 17 + 1] = np.nan
    with pytest.raises(BFError, match=r"BF_ERR_NONFINITE.*rhs.*entry 35 \(cell 17, S_n\)"):
        g.solve(b, np.zeros(2 * J.n))
    xb = np.zeros(2 * J.n)
    xb[2 * 5] = np.inf
    with pytest.raises(BFError, match=r"BF_ERR_NONFINITE.*x0.*cell 5, p_w"):
        g.solve(rhs, xb)
    # the handle stays usable after the errors
    x = np.zeros(2 * J.n)
    r = g.solve(rhs, x, tol=1e-8)
    ro = o.gmres(rhs, tol=1e-8)
    assert r["converged"] and abs(r["iters"] - ro["iters"]) <= 1


# The solve-phase storage / fusion choices (DIA finest levels, fused restriction Rf, dense
# tail operator, cooperative tail, TMA tiles) are all the same linear operators as the
# oracle's level-by-level V-cycle; each variant must meet the same bounds.  The choices are
# read at bf_setup time from the environment.
VARIANTS = {
    "default": {},
    "no-dtail": {"BF_NO_DTAIL": "1"},
    "no-rfuse": {"BF_NO_RFUSE": "1"},
    "rfuse-l0": {"BF_RFUSE_L0": "1"},
    "plain": {"BF_NO_DTAIL": "1", "BF_NO_RFUSE": "1", "BF_NO_TAIL": "1", "BF_NO_DIA": "1", "BF_NO_TMA": "1"},
    "coop-tail-big": {"BF_NO_DTAIL": "1", "BF_TAIL_NNZ": "200000"},
    "no-reorder": {"BF_NO_REORDER": "1"},
    # windowed jagged-diagonal kernels (k_csr_win.cuh) forced onto these small hierarchies: every CSR
    # level above the tail, accepted whatever its reuse; blocks of 256 / 64 / 32 rows (1, 4 and 8
    # thread groups per row); and switched off
    "wjds-256": {"BF_WIN_NMIN": "0", "BF_WIN_RATIO": "100", "BF_WIN_STAGE": "1000000"},
    "wjds-64": {"BF_WIN_NMIN": "0", "BF_WIN_RATIO": "100", "BF_WIN_ROWS": "64", "BF_NO_DTAIL": "1"},
    "wjds-32": {"BF_WIN_NMIN": "0", "BF_WIN_RATIO": "100", "BF_WIN_STAGE": "1024", "BF_NO_DTAIL": "1",
                "BF_NO_TAIL": "1"},
    "no-wjds": {"BF_NO_WIN": "1"},
}


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("config,dims", [(2, (33, 30, 31)), (3, (20, 17, 15))])
def test_solve_path_variants(variant, config, dims, monkeypatch):
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    prob, J, rhs = make_system(config, dims=dims)
    g = gpu_solver(J, prob.dims)
    o = oracle.BF(J)
    n = J.n
    for which in (0, 1):
        b = seeded_vector(n, 20 + which)
        xo = o.vcycle(which, b)
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        g.vcycle(which, torch_dev(b), x)
        assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-10 * np.linalg.norm(xo), (variant, which)
    v = seeded_vector(2 * n, 8)
    zo = o.apply(v)
    z = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    g.apply_precond(torch_dev(v), z)
    assert np.linalg.norm(z.cpu().numpy() - zo) <= 1e-10 * np.linalg.norm(zo), variant
    ro = o.gmres(rhs, tol=1e-8, restart=30, maxit=500)
    x = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    r = g.solve(torch_dev(rhs), x, tol=1e-8, restart=30, maxit=500)
    assert r["converged"] == ro["converged"] and abs(r["iters"] - ro["iters"]) <= 1, (variant, r["iters"], ro["iters"])
    xg = x.cpu().numpy()
    for f in (0, 1):
        assert np.linalg.norm(xg[f::2] - ro["x"][f::2]) <= 1e-6 * np.linalg.norm(ro["x"][f::2]), variant
    g.close()


@pytest.mark.parametrize("force_wjds,esc", [(False, False), (True, False), (False, True)], ids=["default", "wjds", "no-large-table"])
def test_long_rows_hash_overflow_regression(force_wjds, esc, monkeypatch):
    """(esc: the 1024-slot table of the warp-hash SpGEMM is switched off, so the count is not
    repeated with it before the expand-sort-compress fallback.
    force_wjds: the windowed jagged-diagonal form is requested for every CSR level, whatever its
    size or reuse; the levels whose hub row exceeds the form's 255-entry row limit must fall back to
    the CSR kernels, the others use it.)  A hub cell coupled to 700 others through A_ss only makes A_ss rows (and its Galerkin
    products) longer than the 512-slot shared-memory hash table of the SpGEMM (the C5 setup hang
    of round 1): setup must fall back to the expand-sort-compress product and stay bit-exact
    with the oracle.  (S~ keeps short rows: its row pattern is bounded at 256 entries,
    BF_ERR_LIMIT beyond.)"""
    if esc:
        monkeypatch.setenv("BF_NO_HASH_LARGE", "1")
    if force_wjds:
        for k, v in {"BF_WIN_NMIN": "0", "BF_WIN_RATIO": "100", "BF_NO_DTAIL": "1", "BF_NO_TAIL": "1"}.items():
            monkeypatch.setenv(k, v)
    n = 1200
    rng = np.random.default_rng(11)
    hub = set(rng.choice(np.arange(1, n), 700, replace=False).tolist())
    rows, cols = [], []
    for i in range(n):
        nb = {i}
        if i > 0:
            nb.add(i - 1)
        if i < n - 1:
            nb.add(i + 1)
        if i == 0:
            nb |= hub
        elif i in hub:
            nb.add(0)
        for j in sorted(nb):
            rows.append(i)
            cols.append(j)
    rows, cols = np.array(rows), np.array(cols)
    rp = np.zeros(n + 1, np.int32)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    vals = np.zeros((len(cols), 2, 2))
    off = rows != cols
    vals[off] = -rng.uniform(0.5, 1.5, (off.sum(), 1, 1)) * np.array([[1.0, 0.1], [0.05, 1.0]])
    hubedge = off & (np.abs(rows - cols) > 1)
    vals[hubedge] = vals[hubedge] * np.array([[0.0, 0.0], [0.0, 1.0]])  # A_ss coupling only
    deg = np.bincount(rows, weights=off.astype(float), minlength=n)
    vals[~off] = np.array([[1.0, 0.0], [0.0, 1.0]]) * (2.0 * deg[rows[~off]] + 1.0)[:, None, None]
    J = BSR2(n, rp, cols.astype(np.int32), vals)
    g = gpu_solver(J, (n, 1, 1), max_coarse=32)
    o = oracle.BF(J, max_coarse=32)
    for which in (0, 1):
        assert g.num_levels(which) == o.nlev(which)
        for l in range(o.nlev(which)):
            pat, val = csr_equal(g.level(which, l)["A"], o.level(which, l)["A"])
            assert pat and val, (which, l)
    v = seeded_vector(2 * n, 4)
    z = np.zeros(2 * n)
    g.apply_precond(v, z)
    zo = o.apply(v)
    assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo)
