"""Seeded workload generator: the fully implicit two-phase (p_w, S_n) TPFA
residual and its exact Jacobian in point-interleaved 2x2 BSR.

This module produces the *inputs* of the hot path (J, rhs); it holds none of the
BF-AMG-GMRES arithmetic and is shared by the oracle tests, the GPU tests and
bench.py (the task's "seeded input generator" module).  It is itself pinned in
tests/test_workload.py (finite differences, conservation, sign structure,
null vectors).

Paper passages followed (PAPER.md line numbers, SURVEY.md c.1 readings):
  * unknowns u = (P_w, S_n)                          P:L43 (balance1/balance2, L44-47)
  * cell-centred FV, TPFA flux, omega                P:L48-66 (reading Q2/Q4: sign by conservation,
                                                    Delta x = centre distance)
  * phase upwinding, tie -> j ("otherwise")          P:L67-74 (Q6)
  * harmonic face permeability
  * backward Euler, fully discrete residual          P:L79-83 (`fully_discrete_system`, Q2/Q3: mass form, kg)
  * Newton with exact Jacobian (frozen upwind)       P:L14, L86-89 (Q7)
  * 2x2 block Jacobian, point ordering               P:L114-123 (`jacobian`), L145-153
  * Brooks-Corey / linear P_c                        P:L264-268; van Genuchten per BASELINE.json configs[2] (Q16)
  * quadratic k_r (Q8), clamp of S_w (Q10), T1 densities (Q11)

Conventions: cell id c = i + nx*(j + ny*k); residual rows per cell (R_w, R_n);
unknown columns per cell (p_w, S_n); block (r,c) = [[dRw/dp, dRw/dS],[dRn/dp, dRn/dS]]
= [[a_pp, a_ps],[a_sp, a_ss]] (row-major in the BSR value array).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

G_ACC = 9.80665       # m/s^2 (Q12)
DAY = 86400.0         # s
EPS_S = 1e-3          # clamp of the effective wetting saturation (Q10)


# ----------------------------------------------------------------------------
# constitutive laws
# ----------------------------------------------------------------------------
def harmonic_face_perm(ki, kj, dxi=1.0, dxj=1.0):
    """K_ij = (dx_i+dx_j) K_i K_j / (dx_i K_j + dx_j K_i); 0 if either is 0."""
    ki = np.asarray(ki, dtype=np.float64)
    kj = np.asarray(kj, dtype=np.float64)
    den = dxi * kj + dxj * ki
    with np.errstate(divide="ignore", invalid="ignore"):
        out = np.where((ki > 0) & (kj > 0), (dxi + dxj) * ki * kj / np.where(den > 0, den, 1.0), 0.0)
    return out


@dataclass
class CapillaryModel:
    kind: str                  # "bc" (Brooks-Corey), "vg" (van Genuchten), "linear", "none"
    a: float = 0.0             # bc: P_d ; vg: n ; linear: P_0
    b: float = 0.0             # bc: lambda ; vg: alpha

    def pc_and_deriv(self, swbar):
        """P_c(S_w_bar) and dP_c/dS_w_bar (derivative w.r.t. the effective wetting saturation)."""
        s = swbar
        if self.kind == "bc":          # P_c = P_d S^{-1/lambda}
            pd, lam = self.a, self.b
            pc = pd * s ** (-1.0 / lam)
            dpc = -(pd / lam) * s ** (-1.0 / lam - 1.0)
        elif self.kind == "linear":    # P_c = P_0 (1 - S)
            pc = self.a * (1.0 - s)
            dpc = -self.a * np.ones_like(s)
        elif self.kind == "vg":        # P_c = (1/alpha) (S^{-1/m} - 1)^{1/n}, m = 1-1/n  (Q16)
            n, alpha = self.a, self.b
            m = 1.0 - 1.0 / n
            base = s ** (-1.0 / m) - 1.0
            pc = (1.0 / alpha) * base ** (1.0 / n)
            dpc = (1.0 / alpha) * (1.0 / n) * base ** (1.0 / n - 1.0) * (-1.0 / m) * s ** (-1.0 / m - 1.0)
        elif self.kind == "none":
            pc = np.zeros_like(s)
            dpc = np.zeros_like(s)
        else:
            raise ValueError(self.kind)
        return pc, dpc


@dataclass
class Problem:
    nx: int
    ny: int
    nz: int
    perm: np.ndarray                  # [n] m^2 (isotropic)
    pc: CapillaryModel
    dt: float                         # s
    sn_old: np.ndarray                # [n] S_n^n
    p_old: np.ndarray                 # [n] p_w^n
    h: float = 1.0                    # cell size (Q15)
    phi: float = 0.2
    rho_w: float = 1000.0
    rho_n: float = 700.0
    mu_w: float = 1e-3
    mu_n: float = 1e-3
    g: float = G_ACC
    gravity_axis: int | None = None   # 0,1,2 or None; depth grows with the index
    dirichlet: list = field(default_factory=list)  # [(axis, side(0=-,1=+), p_b)]
    source_w: np.ndarray | None = None  # [n] water mass rate kg/s (injection > 0)

    @property
    def n(self):
        return self.nx * self.ny * self.nz

    @property
    def dims(self):
        return (self.nx, self.ny, self.nz)

    def strides(self):
        return (1, self.nx, self.nx * self.ny)

    def depth(self):
        n = self.n
        if self.gravity_axis is None:
            return np.zeros(n)
        idx = np.arange(n)
        i = idx % self.nx
        j = (idx // self.nx) % self.ny
        k = idx // (self.nx * self.ny)
        a = (i, j, k)[self.gravity_axis]
        return (a + 0.5) * self.h

    # ------------------------------------------------------------------
    def props(self, p, sn):
        """Per-cell mobilities, P_c and their S_n-derivatives (Q8-Q10)."""
        sw = 1.0 - sn
        inside = (sw > EPS_S) & (sw < 1.0 - EPS_S)
        swb = np.clip(sw, EPS_S, 1.0 - EPS_S)
        dswb = np.where(inside, -1.0, 0.0)            # d S_w_bar / d S_n
        krw = swb * swb
        krn = (1.0 - swb) ** 2
        dkrw = 2.0 * swb * dswb
        dkrn = -2.0 * (1.0 - swb) * dswb
        pc, dpc_ds = self.pc.pc_and_deriv(swb)
        dpc = dpc_ds * dswb                            # d P_c / d S_n
        return dict(lw=krw / self.mu_w, ln=krn / self.mu_n,
                    dlw=dkrw / self.mu_w, dln=dkrn / self.mu_n,
                    pc=pc, dpc=dpc)

    def faces(self):
        """Interior faces (c < d) per axis: list of (axis, c, d)."""
        out = []
        n = self.n
        idx = np.arange(n)
        coords = (idx % self.nx, (idx // self.nx) % self.ny, idx // (self.nx * self.ny))
        for a, (na, s) in enumerate(zip(self.dims, self.strides())):
            if na < 2:
                continue
            c = idx[coords[a] < na - 1]
            out.append((a, c, c + s))
        return out

    def boundary_faces(self):
        """Dirichlet faces: list of (cell array, p_b)."""
        out = []
        n = self.n
        idx = np.arange(n)
        coords = (idx % self.nx, (idx // self.nx) % self.ny, idx // (self.nx * self.ny))
        for (a, side, pb) in self.dirichlet:
            na = self.dims[a]
            cells = idx[coords[a] == (0 if side == 0 else na - 1)]
            out.append((cells, pb))
        return out


# ----------------------------------------------------------------------------
# face fluxes
# ----------------------------------------------------------------------------
def _phase_flux(rho, lam_c, lam_d, dlam_c, dlam_d, phi_c, phi_d, dphi_c, dphi_d, T):
    """F = rho lam_up T (Phi_c - Phi_d), up = c if Phi_c - Phi_d > 0 else d (tie -> d).
    Returns F and dF/d(p_c, S_c, p_d, S_d) with the donor frozen (Q7)."""
    dphi = phi_c - phi_d
    up_c = dphi > 0.0
    lam = np.where(up_c, lam_c, lam_d)
    F = rho * lam * T * dphi
    dFdp_c = rho * lam * T
    dFdp_d = -rho * lam * T
    dFdS_c = rho * T * (np.where(up_c, dlam_c, 0.0) * dphi + lam * dphi_c)
    dFdS_d = rho * T * (np.where(up_c, 0.0, dlam_d) * dphi - lam * dphi_d)
    return F, dFdp_c, dFdS_c, dFdp_d, dFdS_d


def _face_terms(prob: Problem, p, sn):
    pr = prob.props(p, sn)
    D = prob.depth()
    g = prob.g if prob.gravity_axis is not None else 0.0
    phw = p - prob.rho_w * g * D
    phn = p + pr["pc"] - prob.rho_n * g * D
    zero = np.zeros_like(p)
    A = prob.h * prob.h
    res = []
    for (a, c, d) in prob.faces():
        T = A * harmonic_face_perm(prob.perm[c], prob.perm[d]) / prob.h   # Delta = h (Q4)
        w = _phase_flux(prob.rho_w, pr["lw"][c], pr["lw"][d], pr["dlw"][c], pr["dlw"][d],
                        phw[c], phw[d], zero[c], zero[d], T)
        nn = _phase_flux(prob.rho_n, pr["ln"][c], pr["ln"][d], pr["dln"][c], pr["dln"][d],
                         phn[c], phn[d], pr["dpc"][c], pr["dpc"][d], T)
        res.append((a, c, d, w, nn))
    bres = []
    sn_b_all = prob.sn_old
    for (cells, pb) in prob.boundary_faces():
        T = A * prob.perm[cells] / (prob.h / 2.0)           # T_b = A K_c / (h/2)  (Q14)
        snb = sn_b_all[cells]
        prb = prob.props(np.full(len(cells), pb), snb)
        phw_b = pb - prob.rho_w * g * D[cells]
        phn_b = pb + prb["pc"] - prob.rho_n * g * D[cells]
        zc = np.zeros(len(cells))
        w = _phase_flux(prob.rho_w, pr["lw"][cells], prb["lw"], pr["dlw"][cells], zc,
                        phw[cells], phw_b, zc, zc, T)
        nn = _phase_flux(prob.rho_n, pr["ln"][cells], prb["ln"], pr["dln"][cells], zc,
                         phn[cells], phn_b, pr["dpc"][cells], zc, T)
        bres.append((cells, w, nn))
    return res, bres


def residual(prob: Problem, p, sn):
    """R(u) per cell, shape [n, 2] = (R_w, R_n), in kg (Q2, Q3):
    R_a,c = V phi rho_a (S_a - S_a^n) + dt * (sum of outgoing face mass fluxes) - dt * m_a,c."""
    n = prob.n
    V = prob.h ** 3
    Rw = V * prob.phi * prob.rho_w * ((1.0 - sn) - (1.0 - prob.sn_old))
    Rn = V * prob.phi * prob.rho_n * (sn - prob.sn_old)
    faces, bfaces = _face_terms(prob, p, sn)
    dt = prob.dt
    for (a, c, d, w, nn) in faces:
        Rw += dt * (np.bincount(c, w[0], n) - np.bincount(d, w[0], n))
        Rn += dt * (np.bincount(c, nn[0], n) - np.bincount(d, nn[0], n))
    for (cells, w, nn) in bfaces:
        Rw += dt * np.bincount(cells, w[0], n)
        Rn += dt * np.bincount(cells, nn[0], n)
    if prob.source_w is not None:
        Rw -= dt * prob.source_w
    return np.stack([Rw, Rn], axis=1)


# slot order per row (ascending column): -z, -y, -x, diag, +x, +y, +z
_SLOT_MINUS = {2: 0, 1: 1, 0: 2}
_SLOT_PLUS = {0: 4, 1: 5, 2: 6}
DIAG_SLOT = 3


def jacobian_slots(prob: Problem, p, sn):
    """Dense slot form of J: vals[n, 7, 2, 2] and present[n, 7] (every structural
    block of the grid adjacency is present, zero or not)."""
    n = prob.n
    V = prob.h ** 3
    vals = np.zeros((n, 7, 2, 2))
    present = np.zeros((n, 7), dtype=bool)
    present[:, DIAG_SLOT] = True
    vals[:, DIAG_SLOT, 0, 1] = -V * prob.phi * prob.rho_w
    vals[:, DIAG_SLOT, 1, 1] = V * prob.phi * prob.rho_n
    faces, bfaces = _face_terms(prob, p, sn)
    dt = prob.dt
    diag = np.zeros((n, 2, 2))
    for (a, c, d, w, nn) in faces:
        sp, sm = _SLOT_PLUS[a], _SLOT_MINUS[a]
        present[c, sp] = True
        present[d, sm] = True
        for r, F in ((0, w), (1, nn)):
            _, dpc, dsc, dpd, dsd = F
            # row c gets + dt dF, row d gets - dt dF (face assembled once, Q6)
            diag[:, r, 0] += np.bincount(c, dt * dpc, n) - np.bincount(d, dt * dpd, n)
            diag[:, r, 1] += np.bincount(c, dt * dsc, n) - np.bincount(d, dt * dsd, n)
            vals[c, sp, r, 0] += dt * dpd
            vals[c, sp, r, 1] += dt * dsd
            vals[d, sm, r, 0] -= dt * dpc
            vals[d, sm, r, 1] -= dt * dsc
    for (cells, w, nn) in bfaces:
        for r, F in ((0, w), (1, nn)):
            _, dpc, dsc, _, _ = F
            diag[:, r, 0] += np.bincount(cells, dt * dpc, n)
            diag[:, r, 1] += np.bincount(cells, dt * dsc, n)
    vals[:, DIAG_SLOT] += diag
    return vals, present


def slot_columns(prob: Problem):
    """Column index of each slot for each row (undefined where not present)."""
    n = prob.n
    s = prob.strides()
    c = np.arange(n, dtype=np.int64)
    offs = np.array([-s[2], -s[1], -s[0], 0, s[0], s[1], s[2]], dtype=np.int64)
    return c[:, None] + offs[None, :]


@dataclass
class BSR2:
    """Point-interleaved 2x2 BSR: int32 row_ptr[n+1], int32 col_idx[nnzb],
    f64 vals[nnzb,2,2] row-major [[a_pp, a_ps],[a_sp, a_ss]]."""
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    dims: tuple = (0, 0, 0)

    @property
    def nnzb(self):
        return int(self.col_idx.shape[0])

    def to_dense(self):
        N = 2 * self.n
        A = np.zeros((N, N))
        for r in range(self.n):
            for q in range(self.row_ptr[r], self.row_ptr[r + 1]):
                c = self.col_idx[q]
                A[2 * r:2 * r + 2, 2 * c:2 * c + 2] = self.vals[q]
        return A

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.bsr_matrix((self.vals, self.col_idx, self.row_ptr), shape=(2 * self.n, 2 * self.n))


def jacobian(prob: Problem, p, sn) -> BSR2:
    vals, present = jacobian_slots(prob, p, sn)
    cols = slot_columns(prob)
    counts = present.sum(axis=1)
    row_ptr = np.zeros(prob.n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    assert row_ptr[-1] < 2**31
    col_idx = cols[present].astype(np.int32)
    v = vals[present]
    return BSR2(prob.n, row_ptr.astype(np.int32), col_idx, np.ascontiguousarray(v), prob.dims)
