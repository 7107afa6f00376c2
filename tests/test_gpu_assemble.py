"""NEXT-2: device assembly of R(u) and J(u) against the seeded generator (workload/twophase.py,
itself pinned by finite differences, conservation and null vectors in test_workload.py), and a
device Newton loop (assembly -> bf_setup/bf_update -> bf_solve -> update) on a small grid."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workload import make_problem, jacobian, residual, newton_sequence
from gpu_util import torch_dev, twophase_struct


def assemble_gpu(prob, p, sn):
    import paper_1611_00127_b200 as bf
    n = prob.n
    nnzb = bf.bf_assemble_nnzb(prob.nx, prob.ny, prob.nz)
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nnzb, dtype=torch.int32, device="cuda")
    v = torch.empty(4 * nnzb, dtype=torch.float64, device="cuda")
    R = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    s, keep = twophase_struct(prob)
    bf.bf_assemble(s, torch_dev(p), torch_dev(sn), rp, ci, v, R)
    return rp.cpu().numpy(), ci.cpu().numpy(), v.cpu().numpy().reshape(-1, 2, 2), R.cpu().numpy()


@pytest.mark.parametrize("config,dims", [(1, None), (1, (9, 7, 1)), (2, (12, 11, 9)), (3, (20, 17, 15)),
                                         (4, (40, 9, 16)), (5, (16, 16, 8))])
def test_assembly_matches_generator(config, dims):
    prob = make_problem(config, dims=dims)
    rng = np.random.default_rng(config)
    # a generic state (not u^n): random pressure perturbation and saturations
    p = prob.p_old + rng.uniform(-500, 500, prob.n)
    sn = np.clip(prob.sn_old + rng.uniform(-0.05, 0.05, prob.n), 0.0, 1.0)
    J = jacobian(prob, p, sn)
    R = residual(prob, p, sn).reshape(-1)
    rp, ci, v, Rg = assemble_gpu(prob, p, sn)
    assert np.array_equal(rp, J.row_ptr) and np.array_equal(ci, J.col_idx)
    # per block-row scale: values agree to 1e-12 of the row's largest entry of that equation
    rows = np.repeat(np.arange(J.n), np.diff(J.row_ptr))
    for e in (0, 1):
        scale = np.zeros(J.n)
        np.maximum.at(scale, rows, np.abs(J.vals[:, e, :]).max(axis=1))
        err = np.abs(v[:, e, :] - J.vals[:, e, :]).max(axis=1)
        assert np.all(err <= 1e-12 * scale[rows] + 1e-300), (e, err.max())
    assert np.linalg.norm(Rg - R) <= 1e-12 * np.linalg.norm(R)


def test_device_newton_loop_matches_host_sequence():
    """Three Newton steps fully on the device (assembly, setup/update, solve, chopped update)
    track the host generator + oracle sequence: same ||F(u_k)|| to 1e-9 relative."""
    import oracle
    import paper_1611_00127_b200 as bf
    config, dims = 2, (14, 12, 10)
    fn_host = []

    def solve(k, J, rhs):
        return oracle.BF(J).gmres(rhs, tol=1e-10, maxit=800)["x"]
    for k, prob, J, rhs, fn in newton_sequence(config, 3, solve, dims=dims):
        fn_host.append(fn)
    prob = make_problem(config, dims=dims)
    n = prob.n
    nnzb = bf.bf_assemble_nnzb(prob.nx, prob.ny, prob.nz)
    p, sn = torch_dev(prob.p_old.copy()), torch_dev(prob.sn_old.copy())
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nnzb, dtype=torch.int32, device="cuda")
    v = torch.empty(4 * nnzb, dtype=torch.float64, device="cuda")
    R = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    x = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    s, keep = twophase_struct(prob)
    h = None
    fn_dev = []
    for k in range(3):
        bf.bf_assemble(s, p, sn, rp, ci, v, R)
        fn_dev.append(float(torch.linalg.norm(R)))
        rhs = -R
        h = bf.bf_setup(rp, ci, v, prob.dims) if h is None else (bf.bf_update(h, v) or h)
        x.zero_()
        r = bf.bf_solve(h, rhs, x, 1e-10, 30, 800)
        assert r["converged"]
        bf.bf_newton_update(p, sn, x, 0.2)
    bf.bf_destroy(h)
    assert np.allclose(fn_dev, fn_host, rtol=1e-9, atol=0), (fn_dev, fn_host)
