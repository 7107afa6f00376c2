"""Helpers shared by the GPU tests: build a GPU solver and an oracle context on the same
seeded Jacobian."""
import numpy as np


def torch_dev(a, dev="cuda"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def gpu_solver(J, dims=None, on_device=True, block_order=0, var_order=0, **opts):
    from paper_1611_00127_b200 import BFSolver
    vals = J.vals if block_order == 0 else np.ascontiguousarray(J.vals.transpose(0, 2, 1))
    arrs = [np.ascontiguousarray(J.row_ptr, np.int32), np.ascontiguousarray(J.col_idx, np.int32),
            np.ascontiguousarray(vals, np.float64).reshape(-1)]
    if on_device:
        arrs = [torch_dev(a) for a in arrs]
    dims = dims or (J.n, 1, 1)
    return BFSolver(*arrs, dims=dims, block_order=block_order, var_order=var_order, **opts)


def csr_equal(g, o):
    """g: (rp int32, ci, v) from the GPU; o: oracle.CSR -> (patterns equal, values bit-equal)"""
    rp, ci, v = g
    pat = np.array_equal(rp.astype(np.int64), o.rp) and np.array_equal(ci, o.ci)
    vals = pat and np.array_equal(v.view(np.uint64), o.v.view(np.uint64))
    return pat, vals


def twophase_struct(prob, dev="cuda"):
    """workload.Problem -> (bf_twophase, keep-alive tensors) for bf_assemble."""
    import torch
    from paper_1611_00127_b200 import bf_twophase
    kinds = {"none": 0, "bc": 1, "vg": 2, "linear": 3}
    keep = [torch_dev(prob.perm, dev), torch_dev(prob.sn_old, dev)]
    src = torch_dev(prob.source_w, dev) if prob.source_w is not None else None
    if src is not None:
        keep.append(src)
    s = bf_twophase()
    s.nx, s.ny, s.nz = prob.nx, prob.ny, prob.nz
    s.h, s.phi, s.rho_w, s.rho_n, s.mu_w, s.mu_n = prob.h, prob.phi, prob.rho_w, prob.rho_n, prob.mu_w, prob.mu_n
    s.g, s.dt = prob.g, prob.dt
    s.gravity_axis = -1 if prob.gravity_axis is None else prob.gravity_axis
    s.pc_kind, s.pc_a, s.pc_b = kinds[prob.pc.kind], prob.pc.a, prob.pc.b
    s.n_dirichlet = len(prob.dirichlet)
    for f, (a, side, pb) in enumerate(prob.dirichlet):
        s.dir_axis[f], s.dir_side[f], s.dir_p[f] = a, side, pb
    s.perm, s.sn_old = keep[0].data_ptr(), keep[1].data_ptr()
    s.source_w = src.data_ptr() if src is not None else None
    return s, keep
