"""TEST INFRASTRUCTURE ONLY: ctypes binding of the plain C oracle (oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package.  The CUDA product path (paper_1611_00127_b200/) never
imports, links or executes anything under oracle/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")
HDR = os.path.join(HERE, "oracle.h")

# c.4: IEEE binary64, no FMA contraction, no fast-math
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared", "-Wall",
          "-Wno-maybe-uninitialized"]


def build(force: bool = False) -> str:
    # ORACLE_SO: load a prebuilt variant instead (tests/test_oracle_mutations.py runs the pins
    # against deliberately broken copies of oracle.c to show that each pin bites)
    if os.environ.get("ORACLE_SO"):
        return os.environ["ORACLE_SO"]
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)):
        tmp = SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"])
        os.replace(tmp, SO)
    return SO


class CSRs(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("rp", C.POINTER(C.c_int64)), ("ci", C.POINTER(C.c_int32)), ("v", C.POINTER(C.c_double))]


class Options(C.Structure):
    _fields_ = [("theta", C.c_double), ("max_levels", C.c_int32), ("max_coarse", C.c_int32),
                ("smoother", C.c_int32), ("nu_pre", C.c_int32), ("nu_post", C.c_int32),
                ("cheb_degree", C.c_int32), ("cheb_lo", C.c_double), ("seed", C.c_uint64),
                ("orth", C.c_int32), ("schur_as_printed", C.c_int32), ("interp_norm", C.c_int32),
                ("precond", C.c_int32), ("cheb_eig", C.c_int32), ("smoother_p", C.c_int32),
                ("cheb_levels", C.c_int32), ("diag_stop", C.c_int32)]


MAXL = 64


class AMGs(C.Structure):
    _fields_ = [("nlev", C.c_int32), ("A", CSRs * MAXL), ("P", CSRs * MAXL), ("R", CSRs * MAXL),
                ("cf", C.POINTER(C.c_int8) * MAXL), ("strong", C.POINTER(C.c_uint8) * MAXL),
                ("dl1", C.POINTER(C.c_double) * MAXL), ("cheb_hi", C.c_double * MAXL), ("lu", C.POINTER(C.c_double)),
                ("piv", C.POINTER(C.c_int32)), ("opt", Options)]


class BFs(C.Structure):
    _fields_ = [("n", C.c_int32), ("var_order", C.c_int32), ("block_order", C.c_int32),
                ("brp", C.POINTER(C.c_int64)), ("bci", C.POINTER(C.c_int32)), ("bv", C.POINTER(C.c_double)),
                ("App", CSRs), ("Aps", CSRs), ("Asp", CSRs), ("Ass", CSRs), ("S", CSRs),
                ("dss", C.POINTER(C.c_double)), ("hss", AMGs), ("hS", AMGs), ("opt", Options),
                ("hpp", AMGs), ("ilu", C.POINTER(C.c_double)), ("ilu_dinv", C.POINTER(C.c_double)),
                ("Jsc", CSRs), ("hJ", AMGs)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        dp, ip, lp = P(C.c_double), P(C.c_int32), P(C.c_int64)
        L.or_last_error.restype = C.c_char_p
        L.or_default_options.argtypes = [P(Options)]
        L.or_h32.restype = C.c_uint32
        L.or_h32.argtypes = [C.c_uint64, C.c_int32, C.c_int64]
        L.or_bsr_spmv.argtypes = [C.c_int32, lp, ip, dp, dp, dp]
        L.or_csr_spmv.argtypes = [P(CSRs), dp, dp]
        L.or_split.argtypes = [C.c_int32, lp, ip, dp, C.c_int32, C.c_int32,
                               P(CSRs), P(CSRs), P(CSRs), P(CSRs), dp]
        L.or_schur.argtypes = [P(CSRs), P(CSRs), P(CSRs), dp, C.c_int32, P(CSRs)]
        L.or_strength.argtypes = [P(CSRs), C.c_double, P(C.c_uint8)]
        L.or_pmis.argtypes = [P(CSRs), P(C.c_uint8), P(C.c_uint32), P(C.c_int8)]
        L.or_interp.argtypes = [P(CSRs), P(C.c_uint8), P(C.c_int8), C.c_int32, P(CSRs)]
        L.or_transpose.argtypes = [P(CSRs), P(CSRs)]
        L.or_matmul.argtypes = [P(CSRs), P(CSRs), P(CSRs)]
        L.or_l1diag.argtypes = [P(CSRs), dp]
        L.or_power_estimate.restype = C.c_double
        L.or_power_estimate.argtypes = [P(CSRs), dp, C.c_int32, C.c_uint64, C.c_int32]
        L.or_smooth.argtypes = [P(CSRs), dp, dp, dp, C.c_int32, C.c_int32, C.c_double, C.c_double]
        L.or_amg_setup.argtypes = [P(CSRs), P(Options), P(AMGs)]
        L.or_amg_free.argtypes = [P(AMGs)]
        L.or_vcycle.argtypes = [P(AMGs), dp, dp]
        L.or_csr_free.argtypes = [P(CSRs)]
        L.or_ilu0.argtypes = [C.c_int32, lp, ip, dp, dp, dp]
        L.or_ilu0_solve.argtypes = [C.c_int32, lp, ip, dp, dp, dp, dp]
        L.or_jscalar.argtypes = [C.c_int32, lp, ip, dp, P(CSRs)]
        L.or_bf_setup.argtypes = [C.c_int32, lp, ip, dp, C.c_int32, C.c_int32, P(Options), P(P(BFs))]
        L.or_bf_free.argtypes = [P(BFs)]
        L.or_bf_update.argtypes = [P(BFs), dp]
        L.or_bf_apply.argtypes = [P(BFs), dp, dp]
        L.or_bf_spmv.argtypes = [P(BFs), dp, dp]
        L.or_gmres.argtypes = [P(BFs), dp, dp, C.c_double, C.c_int32, C.c_int32, ip, dp, ip, dp]
        L.or_gmres_capture.argtypes = [dp, dp, ip]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


# ---------------------------------------------------------------------------
@dataclass
class CSR:
    nrows: int
    ncols: int
    rp: np.ndarray       # int64
    ci: np.ndarray       # int32
    v: np.ndarray        # float64

    @property
    def nnz(self):
        return int(self.ci.shape[0])

    @staticmethod
    def from_scipy(A):
        A = A.tocsr()
        A.sort_indices()
        return CSR(A.shape[0], A.shape[1], A.indptr.astype(np.int64), A.indices.astype(np.int32),
                   A.data.astype(np.float64))

    @staticmethod
    def from_dense(D):
        import scipy.sparse as sp
        D = np.asarray(D, dtype=np.float64)
        rows, cols = np.nonzero(np.ones_like(D, dtype=bool) & (D != 0))
        return CSR.from_scipy(sp.csr_matrix((D[rows, cols], (rows, cols)), shape=D.shape))

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.v, self.ci, self.rp), shape=(self.nrows, self.ncols))

    def to_dense(self):
        return self.to_scipy().toarray()

    def cstruct(self):
        self._keep = (np.ascontiguousarray(self.rp, np.int64), np.ascontiguousarray(self.ci, np.int32),
                      np.ascontiguousarray(self.v, np.float64))
        return CSRs(self.nrows, self.ncols, self.nnz, _p(self._keep[0], C.c_int64),
                    _p(self._keep[1], C.c_int32), _p(self._keep[2], C.c_double))


def _from_cstruct(s: CSRs, copy=True) -> CSR:
    nr, nnz = s.nrows, s.nnz
    rp = np.ctypeslib.as_array(s.rp, (nr + 1,)).copy()
    if nnz > 0:
        ci = np.ctypeslib.as_array(s.ci, (nnz,)).copy()
        v = np.ctypeslib.as_array(s.v, (nnz,)).copy()
    else:
        ci = np.zeros(0, np.int32)
        v = np.zeros(0)
    return CSR(nr, s.ncols, rp, ci, v)


def default_options(**kw) -> Options:
    o = Options()
    lib().or_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def err():
    return lib().or_last_error().decode()


def h32(seed, level, i):
    return int(lib().or_h32(seed, level, i))


# ---------------------------------------------------------------------------
# primitive steps (for pins)
# ---------------------------------------------------------------------------
def _bsr_arrays(J, block_order=0):
    rp = np.ascontiguousarray(J.row_ptr, np.int64)
    ci = np.ascontiguousarray(J.col_idx, np.int32)
    v = np.ascontiguousarray(J.vals, np.float64).reshape(-1)
    if block_order == 1:
        v = np.ascontiguousarray(J.vals.transpose(0, 2, 1)).reshape(-1)
    return rp, ci, v


def bsr_spmv(J, x):
    rp, ci, v = _bsr_arrays(J)
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(2 * J.n)
    lib().or_bsr_spmv(J.n, _p(rp, C.c_int64), _p(ci, C.c_int32), _p(v, C.c_double),
                      _p(x, C.c_double), _p(y, C.c_double))
    return y


def csr_spmv(A: CSR, x):
    s = A.cstruct()
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(A.nrows)
    lib().or_csr_spmv(C.byref(s), _p(x, C.c_double), _p(y, C.c_double))
    return y


def split(J, block_order=0, var_order=0):
    rp, ci, v = _bsr_arrays(J, block_order)
    if var_order == 1 and block_order == 0:
        # caller supplies blocks already in swapped variable order
        pass
    outs = [CSRs() for _ in range(4)]
    dss = np.empty(J.n)
    st = lib().or_split(J.n, _p(rp, C.c_int64), _p(ci, C.c_int32), _p(v, C.c_double), block_order, var_order,
                        *[C.byref(o) for o in outs], _p(dss, C.c_double))
    if st:
        raise RuntimeError(err())
    res = [_from_cstruct(o) for o in outs]
    for o in outs:
        lib().or_csr_free(C.byref(o))
    return dict(App=res[0], Aps=res[1], Asp=res[2], Ass=res[3], dss=dss)


def schur(App: CSR, Aps: CSR, Asp: CSR, dss, as_printed=0) -> CSR:
    a, b, c = App.cstruct(), Aps.cstruct(), Asp.cstruct()
    dss = np.ascontiguousarray(dss, np.float64)
    out = CSRs()
    lib().or_schur(C.byref(a), C.byref(b), C.byref(c), _p(dss, C.c_double), as_printed, C.byref(out))
    r = _from_cstruct(out)
    lib().or_csr_free(C.byref(out))
    return r


def strength(A: CSR, theta=0.25):
    s = A.cstruct()
    out = np.empty(A.nnz, np.uint8)
    lib().or_strength(C.byref(s), theta, _p(out, C.c_uint8))
    return out


def pmis(A: CSR, strong, hashes):
    s = A.cstruct()
    strong = np.ascontiguousarray(strong, np.uint8)
    hashes = np.ascontiguousarray(hashes, np.uint32)
    cf = np.empty(A.nrows, np.int8)
    lib().or_pmis(C.byref(s), _p(strong, C.c_uint8), _p(hashes, C.c_uint32), _p(cf, C.c_int8))
    return cf


def interp(A: CSR, strong, cf, norm=1) -> CSR:
    s = A.cstruct()
    strong = np.ascontiguousarray(strong, np.uint8)
    cf = np.ascontiguousarray(cf, np.int8)
    out = CSRs()
    lib().or_interp(C.byref(s), _p(strong, C.c_uint8), _p(cf, C.c_int8), norm, C.byref(out))
    r = _from_cstruct(out)
    lib().or_csr_free(C.byref(out))
    return r


def transpose(P: CSR) -> CSR:
    s = P.cstruct()
    out = CSRs()
    lib().or_transpose(C.byref(s), C.byref(out))
    r = _from_cstruct(out)
    lib().or_csr_free(C.byref(out))
    return r


def matmul(A: CSR, B: CSR) -> CSR:
    a, b = A.cstruct(), B.cstruct()
    out = CSRs()
    lib().or_matmul(C.byref(a), C.byref(b), C.byref(out))
    r = _from_cstruct(out)
    lib().or_csr_free(C.byref(out))
    return r


def l1diag(A: CSR):
    s = A.cstruct()
    d = np.empty(A.nrows)
    lib().or_l1diag(C.byref(s), _p(d, C.c_double))
    return d


def power_estimate(A: CSR, d, steps, seed=0x1611, level=0):
    s = A.cstruct()
    d = np.ascontiguousarray(d, np.float64)
    return float(lib().or_power_estimate(C.byref(s), _p(d, C.c_double), steps, seed, level))


def jscalar(J) -> CSR:
    """J as a scalar point-ordered CSR (coupled AMG, reading R20)."""
    rp, ci, v = _bsr_arrays(J)
    out = CSRs()
    lib().or_jscalar(J.n, _p(rp, C.c_int64), _p(ci, C.c_int32), _p(v, C.c_double), C.byref(out))
    r = _from_cstruct(out)
    lib().or_csr_free(C.byref(out))
    return r


def ilu0(J):
    """Block ILU(0) of the 2x2 BSR J (canonical row-major blocks) on its own block pattern
    (reading R18).  Returns (lu [nnzb,2,2], dinv [n,2,2])."""
    rp, ci, v = _bsr_arrays(J)
    lu = np.empty_like(v)
    dinv = np.empty(4 * J.n)
    st = lib().or_ilu0(J.n, _p(rp, C.c_int64), _p(ci, C.c_int32), _p(v, C.c_double), _p(lu, C.c_double),
                       _p(dinv, C.c_double))
    if st:
        raise RuntimeError(err())
    return lu.reshape(-1, 2, 2), dinv.reshape(-1, 2, 2)


def ilu0_solve(J, lu, dinv, r):
    """x = (L U)^-1 r, canonical interleaved vectors."""
    rp, ci, _ = _bsr_arrays(J)
    lu = np.ascontiguousarray(lu, np.float64).reshape(-1)
    dinv = np.ascontiguousarray(dinv, np.float64).reshape(-1)
    r = np.ascontiguousarray(r, np.float64)
    x = np.empty_like(r)
    lib().or_ilu0_solve(J.n, _p(rp, C.c_int64), _p(ci, C.c_int32), _p(lu, C.c_double), _p(dinv, C.c_double),
                        _p(r, C.c_double), _p(x, C.c_double))
    return x


def smooth(A: CSR, d, b, x, kind=0, degree=2, lo=0.3, hi=1.0):
    s = A.cstruct()
    d = np.ascontiguousarray(d, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    x = np.array(x, dtype=np.float64)
    lib().or_smooth(C.byref(s), _p(d, C.c_double), _p(b, C.c_double), _p(x, C.c_double), kind, degree, lo, hi)
    return x


# ---------------------------------------------------------------------------
class AMG:
    """One AMG hierarchy (c.2 steps 3-5)."""

    def __init__(self, A: CSR, **opts):
        self._A = A.cstruct()
        self.h = AMGs()
        o = default_options(**opts)
        st = lib().or_amg_setup(C.byref(self._A), C.byref(o), C.byref(self.h))
        if st:
            raise RuntimeError(err())

    def __del__(self):
        try:
            lib().or_amg_free(C.byref(self.h))
        except Exception:
            pass

    @property
    def nlev(self):
        return self.h.nlev

    def level(self, l):
        return _level(self.h, l)

    def vcycle(self, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        lib().or_vcycle(C.byref(self.h), _p(b, C.c_double), _p(x, C.c_double))
        return x


def _level(h: AMGs, l):
    out = dict(A=_from_cstruct(h.A[l]))
    n = h.A[l].nrows
    out["dl1"] = np.ctypeslib.as_array(h.dl1[l], (n,)).copy()
    out["cheb_hi"] = float(h.cheb_hi[l])
    if l < h.nlev - 1:
        out["P"] = _from_cstruct(h.P[l])
        out["R"] = _from_cstruct(h.R[l])
        out["cf"] = np.ctypeslib.as_array(h.cf[l], (n,)).copy()
        nnz = h.A[l].nnz
        out["strong"] = np.ctypeslib.as_array(h.strong[l], (nnz,)).copy() if nnz else np.zeros(0, np.uint8)
    return out


class BF:
    """Oracle BF-AMG-GMRES context (Algorithm 3)."""

    def __init__(self, J, block_order=0, var_order=0, **opts):
        rp, ci, v = _bsr_arrays(J, block_order)
        self.n = J.n
        o = default_options(**opts)
        ptr = C.POINTER(BFs)()
        st = lib().or_bf_setup(J.n, _p(rp, C.c_int64), _p(ci, C.c_int32), _p(v, C.c_double),
                               block_order, var_order, C.byref(o), C.byref(ptr))
        if st:
            raise RuntimeError(err())
        self.ptr = ptr

    def __del__(self):
        try:
            lib().or_bf_free(self.ptr)
        except Exception:
            pass

    def update(self, J, block_order=0):
        """New values on the same pattern (frozen coarse hierarchy, reading R16)."""
        rp, ci, v = _bsr_arrays(J, block_order)
        self._keep_vals = v
        st = lib().or_bf_update(self.ptr, _p(v, C.c_double))
        if st:
            raise RuntimeError(err())

    @property
    def s(self) -> BFs:
        return self.ptr.contents

    def matrix(self, name) -> CSR:
        return _from_cstruct(getattr(self.s, name))

    def dss(self):
        return np.ctypeslib.as_array(self.s.dss, (self.n,)).copy()

    def hierarchy(self, which):
        """which: 0 -> A_ss, 1 -> S~, 2 -> A_pp (CPR), 3 -> J as a scalar matrix (coupled AMG)"""
        return (self.s.hss, self.s.hS, self.s.hpp, self.s.hJ)[which]

    def ilu(self):
        """(lu [nnzb,2,2], dinv [n,2,2]) of the CPR preconditioner's block ILU(0)."""
        nnzb = int(self.s.brp[self.n])
        return (np.ctypeslib.as_array(self.s.ilu, (4 * nnzb,)).copy().reshape(-1, 2, 2),
                np.ctypeslib.as_array(self.s.ilu_dinv, (4 * self.n,)).copy().reshape(-1, 2, 2))

    def nlev(self, which):
        return self.hierarchy(which).nlev

    def level(self, which, l):
        return _level(self.hierarchy(which), l)

    def vcycle(self, which, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        h = self.hierarchy(which)
        lib().or_vcycle(C.byref(h), _p(b, C.c_double), _p(x, C.c_double))
        return x

    def apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        z = np.empty_like(v)
        lib().or_bf_apply(self.ptr, _p(v, C.c_double), _p(z, C.c_double))
        return z

    def spmv(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        lib().or_bf_spmv(self.ptr, _p(x, C.c_double), _p(y, C.c_double))
        return y

    def arnoldi(self, b, restart=30):
        """First GMRES(restart) cycle from x0 = 0 with tol = 0 through the or_gmres test hook:
        returns (V [k+1, N] basis, Hbar [k+1, k] unrotated Hessenberg, k)."""
        N = 2 * self.n
        V = np.zeros((restart + 1, N))
        H = np.zeros((restart + 1, restart))
        k = C.c_int32(-1)
        lib().or_gmres_capture(_p(V, C.c_double), _p(H, C.c_double), C.byref(k))
        self.gmres(b, tol=0.0, restart=restart, maxit=restart)
        k = k.value
        return V[:k + 1], H[:k + 1, :k], k

    def gmres(self, b, x0=None, tol=1e-8, restart=30, maxit=500):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
        iters, conv = C.c_int32(), C.c_int32()
        rel = C.c_double()
        hist = np.zeros(maxit + 1)
        lib().or_gmres(self.ptr, _p(b, C.c_double), _p(x, C.c_double), tol, restart, maxit,
                       C.byref(iters), _p(hist, C.c_double), C.byref(conv), C.byref(rel))
        return dict(x=x, iters=iters.value, hist=hist[:iters.value + 1], converged=bool(conv.value),
                    relres=rel.value)
