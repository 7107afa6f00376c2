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
