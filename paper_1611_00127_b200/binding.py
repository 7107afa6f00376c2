"""Thin ctypes binding of libbf.so (include/bf.h).  Argument marshalling only: every
step of the BF-AMG-GMRES path runs in the library's CUDA kernels.  There is no CPU
fallback: if libbf.so is missing, importing this module raises; if no CUDA device is
present, the library calls return BF_ERR_CUDA and these wrappers raise BFError.

Arrays may be torch tensors (CUDA tensors are passed as device pointers, CPU tensors
as host pointers) or numpy arrays (host pointers).  PyTorch is used only for device
memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BF_LIB=checked loads the checked build (device-side bounds / progress checks, build.py --checked)
LIB_PATH = os.path.join(_HERE, "libbf_checked.so" if os.environ.get("BF_LIB") == "checked" else "libbf.so")

BF_OK = 0
STATUS = {0: "BF_OK", 1: "BF_ERR_ARG", 2: "BF_ERR_PATTERN", 3: "BF_ERR_NONFINITE", 4: "BF_ERR_ZERO_DIAG",
          5: "BF_ERR_COARSE_SINGULAR", 6: "BF_ERR_CUDA", 7: "BF_ERR_OOM", 8: "BF_ERR_LIMIT"}

# every symbol declared in include/bf.h
EXPORTS = ["bf_default_options", "bf_setup", "bf_solve", "bf_update", "bf_destroy", "bf_last_error", "bf_spmv",
           "bf_assemble", "bf_assemble_nnzb", "bf_newton_update",
           "bf_apply_precond", "bf_vcycle", "bf_num_levels", "bf_get_level", "bf_get_level_smoother", "bf_get_block",
           "bf_get_ilu", "bf_ilu_solve", "bf_kernel_time", "bf_launch_count", "bf_device_bytes"]


class BFError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class bf_bsr2(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("n_cells", C.c_int32),
                ("nnzb", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("vals", C.c_void_p),
                ("block_order", C.c_int32), ("var_order", C.c_int32), ("mem", C.c_int32),
                ("reserved", C.c_int32)]


class bf_options(C.Structure):
    _fields_ = [("theta", C.c_double), ("max_levels", C.c_int32), ("max_coarse", C.c_int32),
                ("smoother", C.c_int32), ("nu_pre", C.c_int32), ("nu_post", C.c_int32),
                ("cheb_degree", C.c_int32), ("cheb_lo", C.c_double), ("seed", C.c_uint64),
                ("orth", C.c_int32), ("schur_as_printed", C.c_int32), ("interp_norm", C.c_int32),
                ("timing", C.c_int32), ("precond", C.c_int32), ("cheb_eig", C.c_int32),
                ("smoother_p", C.c_int32), ("cheb_levels", C.c_int32), ("diag_stop", C.c_int32)]


class bf_twophase(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("h", C.c_double), ("phi", C.c_double),
                ("rho_w", C.c_double), ("rho_n", C.c_double), ("mu_w", C.c_double), ("mu_n", C.c_double),
                ("g", C.c_double), ("dt", C.c_double), ("gravity_axis", C.c_int32), ("pc_kind", C.c_int32),
                ("pc_a", C.c_double), ("pc_b", C.c_double), ("n_dirichlet", C.c_int32),
                ("dir_axis", C.c_int32 * 6), ("dir_side", C.c_int32 * 6), ("dir_p", C.c_double * 6),
                ("perm", C.c_void_p), ("sn_old", C.c_void_p), ("source_w", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1611_00127_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, P(C.c_double)
    L.bf_default_options.argtypes = [P(bf_options)]
    L.bf_setup.argtypes = [P(bf_bsr2), P(bf_options), vp, P(vp)]
    L.bf_solve.argtypes = [vp, vp, vp, C.c_double, i32, i32, i32, P(i32), dp, P(i32), dp, vp]
    L.bf_update.argtypes = [vp, vp, i32, vp]
    L.bf_assemble.argtypes = [P(bf_twophase), vp, vp, vp, vp, vp, vp, vp]
    L.bf_assemble_nnzb.argtypes = [i32, i32, i32]
    L.bf_newton_update.argtypes = [i32, vp, vp, vp, C.c_double, vp]
    L.bf_destroy.argtypes = [vp]
    L.bf_last_error.argtypes = [vp]
    L.bf_last_error.restype = C.c_char_p
    L.bf_spmv.argtypes = [vp, vp, vp, i32, vp]
    L.bf_apply_precond.argtypes = [vp, vp, vp, i32, vp]
    L.bf_vcycle.argtypes = [vp, i32, vp, vp, i32, vp]
    L.bf_num_levels.argtypes = [vp, i32, P(i32)]
    L.bf_get_level.argtypes = [vp, i32, i32, P(i32), P(i64), P(i64), vp, vp, vp, vp, vp, vp, vp, vp]
    L.bf_get_block.argtypes = [vp, i32, P(i64), vp, vp, vp]
    L.bf_get_level_smoother.argtypes = [vp, i32, i32, dp, dp]
    L.bf_get_ilu.argtypes = [vp, vp, vp, P(i32)]
    L.bf_ilu_solve.argtypes = [vp, vp, vp, i32, vp]
    L.bf_kernel_time.argtypes = [vp, i32, dp, P(i64), dp]
    L.bf_launch_count.argtypes = [vp, P(i64)]
    L.bf_device_bytes.argtypes = [vp, P(i64)]
    for name in EXPORTS:
        L[name].restype = C.c_int
    L.bf_last_error.restype = C.c_char_p
    L.bf_assemble_nnzb.restype = C.c_int64
    return L


lib = _load()


def _check(st, h=None):
    if st != BF_OK:
        raise BFError(st, lib.bf_last_error(h).decode(errors="replace"))


def _ptr(a):
    """(pointer, mem) of a torch tensor or numpy array: mem 1 = device, 0 = host."""
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr()), (1 if a.is_cuda else 0)
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(a.ctypes.data), 0
    raise TypeError(f"unsupported array type {type(a)}")


def _stream(stream):
    if stream is not None:
        return C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
    try:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:
        pass
    return C.c_void_p(0)


def bf_default_options(**kw) -> bf_options:
    o = bf_options()
    _check(lib.bf_default_options(C.byref(o)))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise AttributeError(k)
        setattr(o, k, v)
    return o


def bf_setup(row_ptr, col_idx, vals, dims, block_order=0, var_order=0, opt=None, stream=None):
    """row_ptr int32[n+1], col_idx int32[nnzb], vals f64[nnzb*4] (all host or all device)."""
    (rp, m0), (ci, m1), (v, m2) = _ptr(row_ptr), _ptr(col_idx), _ptr(vals)
    if len({m0, m1, m2}) != 1:
        raise ValueError("row_ptr, col_idx and vals must all be host or all be device arrays")
    nx, ny, nz = dims
    n = nx * ny * nz
    nnzb = int(col_idx.shape[0])
    J = bf_bsr2(nx, ny, nz, n, nnzb, rp, ci, v, block_order, var_order, m0, 0)
    h = C.c_void_p()
    st = lib.bf_setup(C.byref(J), C.byref(opt) if opt is not None else None, _stream(stream), C.byref(h))
    _check(st, None)
    return h


def bf_update(h, vals, stream=None):
    """New Jacobian values on the setup's pattern (frozen coarse hierarchy, R16)."""
    v, m = _ptr(vals)
    _check(lib.bf_update(h, v, m, _stream(stream)), h)


def bf_assemble_nnzb(nx, ny, nz) -> int:
    return int(lib.bf_assemble_nnzb(nx, ny, nz))


def bf_assemble(prob: bf_twophase, p, sn, row_ptr, col_idx, vals, residual, stream=None):
    """Device assembly of R(u) and J(u) (NEXT-2); every array a CUDA tensor."""
    args = [_ptr(a) for a in (p, sn, row_ptr, col_idx, vals, residual)]
    if any(m != 1 for _, m in args):
        raise ValueError("bf_assemble takes device arrays")
    _check(lib.bf_assemble(C.byref(prob), *[a for a, _ in args], _stream(stream)), None)


def bf_newton_update(p, sn, delta, chop=0.2, stream=None):
    (pp, m0), (sp, m1), (dp, m2) = _ptr(p), _ptr(sn), _ptr(delta)
    if (m0, m1, m2) != (1, 1, 1):
        raise ValueError("bf_newton_update takes device arrays")
    _check(lib.bf_newton_update(int(p.shape[0]), pp, sp, dp, chop, _stream(stream)), None)


def bf_destroy(h):
    lib.bf_destroy(h)


def bf_last_error(h=None) -> str:
    return lib.bf_last_error(h).decode(errors="replace")


def bf_solve(h, rhs, x, tol=1e-8, restart=30, maxit=500, res_hist=True, stream=None):
    (b, mb), (xp, mx) = _ptr(rhs), _ptr(x)
    if mb != mx:
        raise ValueError("rhs and x must both be host or both be device arrays")
    iters, conv = C.c_int32(), C.c_int32()
    rel = C.c_double()
    hist = np.zeros(maxit + 1) if res_hist else None
    st = lib.bf_solve(h, b, xp, tol, restart, maxit, mb, C.byref(iters),
                      hist.ctypes.data_as(C.POINTER(C.c_double)) if hist is not None else None,
                      C.byref(conv), C.byref(rel), _stream(stream))
    _check(st, h)
    out = dict(iters=iters.value, converged=bool(conv.value), relres=rel.value)
    if hist is not None:
        out["hist"] = hist[:iters.value + 1]
    return out


def bf_spmv(h, x, y, stream=None):
    (xp, mx), (yp, my) = _ptr(x), _ptr(y)
    assert mx == my
    _check(lib.bf_spmv(h, xp, yp, mx, _stream(stream)), h)


def bf_apply_precond(h, r, z, stream=None):
    (rp, mr), (zp, mz) = _ptr(r), _ptr(z)
    assert mr == mz
    _check(lib.bf_apply_precond(h, rp, zp, mr, _stream(stream)), h)


def bf_vcycle(h, which, b, x, stream=None):
    (bp, mb), (xp, mx) = _ptr(b), _ptr(x)
    assert mb == mx
    _check(lib.bf_vcycle(h, which, bp, xp, mb, _stream(stream)), h)


def bf_num_levels(h, which) -> int:
    n = C.c_int32()
    _check(lib.bf_num_levels(h, which, C.byref(n)), h)
    return n.value


def bf_get_level(h, which, level):
    """Copy level `level` of hierarchy `which` (0 A_ss, 1 S~, 2 A_pp) to host numpy arrays."""
    n, nA, nP = C.c_int32(), C.c_int64(), C.c_int64()
    _check(lib.bf_get_level(h, which, level, C.byref(n), C.byref(nA), C.byref(nP), *([None] * 8)), h)
    n, nA, nP = n.value, nA.value, nP.value
    Arp = np.empty(n + 1, np.int32)
    Aci = np.empty(nA, np.int32)
    Av = np.empty(nA)
    cf = np.empty(n, np.int8)
    dl1 = np.empty(n)
    coarsest = level == bf_num_levels(h, which) - 1
    Prp = np.empty(n + 1, np.int32)
    Pci = np.empty(max(nP, 1), np.int32)
    Pv = np.empty(max(nP, 1))
    p = lambda a: C.c_void_p(a.ctypes.data)
    _check(lib.bf_get_level(h, which, level, None, None, None, p(Arp), p(Aci), p(Av),
                            None if coarsest else p(cf), None if coarsest else p(Prp),
                            None if coarsest else p(Pci), None if coarsest else p(Pv), p(dl1)), h)
    out = dict(n=n, A=(Arp, Aci, Av), dl1=dl1)
    if not coarsest:
        out.update(cf=cf, P=(Prp, Pci[:nP], Pv[:nP]))
    return out


def bf_get_level_smoother(h, which, level):
    """(cheb_hi, beta0) of a level (reading R21)."""
    hi, b0 = C.c_double(), C.c_double()
    _check(lib.bf_get_level_smoother(h, which, level, C.byref(hi), C.byref(b0)), h)
    return hi.value, b0.value


def bf_level_sizes(h, which, level):
    """(n, nnz(A_l), nnz(P_l)) of level `level` of hierarchy `which` (sizes only, no copies)."""
    n, nA, nP = C.c_int32(), C.c_int64(), C.c_int64()
    _check(lib.bf_get_level(h, which, level, C.byref(n), C.byref(nA), C.byref(nP), *([None] * 8)), h)
    return n.value, nA.value, nP.value


def bf_hierarchy_stats(h, which):
    """Per-level sizes and the operator / grid complexities of hierarchy `which`."""
    lv = [bf_level_sizes(h, which, l) for l in range(bf_num_levels(h, which))]
    if not lv:
        return None
    return {"levels": [{"n": n, "nnz_A": a, "nnz_P": p} for n, a, p in lv],
            "operator_complexity": sum(a for _, a, _ in lv) / lv[0][1],
            "grid_complexity": sum(n for n, _, _ in lv) / lv[0][0]}


def bf_get_block(h, which):
    """which: 0 A_pp, 1 A_ps, 2 A_sp, 3 A_ss, 4 S~ -> (row_ptr, col, val) host arrays."""
    nnz = C.c_int64()
    _check(lib.bf_get_block(h, which, C.byref(nnz), None, None, None), h)
    # rows = n_cells: recover from level 0 size of hierarchy 0
    n = bf_get_level_size(h)
    rp = np.empty(n + 1, np.int32)
    ci = np.empty(max(nnz.value, 1), np.int32)
    v = np.empty(max(nnz.value, 1))
    p = lambda a: C.c_void_p(a.ctypes.data)
    _check(lib.bf_get_block(h, which, None, p(rp), p(ci), p(v)), h)
    return rp, ci[:nnz.value], v[:nnz.value]


def bf_get_level_size(h, which=None, level=0) -> int:
    """Rows of a level; which=None: the finest level of whichever hierarchy the handle built."""
    n = C.c_int32()
    for w in ((0, 2) if which is None else (which,)):
        if lib.bf_get_level(h, w, level, C.byref(n), None, None, *([None] * 8)) == BF_OK:
            return n.value
    _check(lib.bf_get_level(h, 0 if which is None else which, level, C.byref(n), None, None, *([None] * 8)), h)
    return n.value


def bf_get_ilu(h, nnzb, n):
    """CPR handles: (lu [nnzb,2,2], dinv [n,2,2], levels) host copies of the block ILU(0) of J."""
    lu = np.empty(4 * nnzb)
    dinv = np.empty(4 * n)
    lev = C.c_int32()
    _check(lib.bf_get_ilu(h, C.c_void_p(lu.ctypes.data), C.c_void_p(dinv.ctypes.data), C.byref(lev)), h)
    return lu.reshape(-1, 2, 2), dinv.reshape(-1, 2, 2), lev.value


def bf_ilu_solve(h, r, x, stream=None):
    (rp, mr), (xp, mx) = _ptr(r), _ptr(x)
    assert mr == mx
    _check(lib.bf_ilu_solve(h, rp, xp, mr, _stream(stream)), h)


def bf_kernel_time(h, kclass):
    """-> (ms, timed regions, algorithmic bytes) of kernel class kclass (needs timing=1)."""
    ms, cnt, by = C.c_double(), C.c_int64(), C.c_double()
    _check(lib.bf_kernel_time(h, kclass, C.byref(ms), C.byref(cnt), C.byref(by)), h)
    return ms.value, cnt.value, by.value


def bf_launch_count(h) -> int:
    n = C.c_int64()
    _check(lib.bf_launch_count(h, C.byref(n)), h)
    return n.value


def bf_device_bytes(h) -> int:
    n = C.c_int64()
    _check(lib.bf_device_bytes(h, C.byref(n)), h)
    return n.value


class BFSolver:
    """Owning wrapper: setup on construction, bf_destroy on close()/garbage collection."""

    def __init__(self, row_ptr, col_idx, vals, dims, block_order=0, var_order=0, stream=None, **opts):
        self.opt = bf_default_options(**opts)
        self.h = bf_setup(row_ptr, col_idx, vals, dims, block_order, var_order, self.opt, stream)
        self.n = dims[0] * dims[1] * dims[2]

    def update(self, vals, stream=None):
        bf_update(self.h, vals, stream)

    def solve(self, rhs, x, tol=1e-8, restart=30, maxit=500, stream=None):
        return bf_solve(self.h, rhs, x, tol, restart, maxit, True, stream)

    def spmv(self, x, y, stream=None):
        bf_spmv(self.h, x, y, stream)

    def apply_precond(self, r, z, stream=None):
        bf_apply_precond(self.h, r, z, stream)

    def vcycle(self, which, b, x, stream=None):
        bf_vcycle(self.h, which, b, x, stream)

    def num_levels(self, which):
        return bf_num_levels(self.h, which)

    def level(self, which, l):
        return bf_get_level(self.h, which, l)

    def block(self, which):
        return bf_get_block(self.h, which)

    def cheb_hi(self, which, l):
        return bf_get_level_smoother(self.h, which, l)[0]

    def ilu(self, nnzb):
        return bf_get_ilu(self.h, nnzb, self.n)

    def ilu_solve(self, r, x, stream=None):
        bf_ilu_solve(self.h, r, x, stream)

    def close(self):
        if getattr(self, "h", None):
            bf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
