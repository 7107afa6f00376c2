"""Newton sequence of Jacobians for one implicit time step (P:L86-89:
J(u_k) (u_{k+1} - u_k) = -F(u_k)), undamped, u_0 = u^n (reading Q18).  The caller supplies
the linear solver, so the states (and hence the Jacobians) can be produced by the oracle
for parity tests or by any solver for benchmarks (Q18: any state gives a valid Jacobian).
Every J_k has the same BSR sparsity pattern (all grid-adjacency blocks are stored)."""
import numpy as np

from .configs import make_problem
from .twophase import jacobian, residual


def newton_sequence(config, steps, solve, dims=None, gravity=True, chop=0.2):
    """Yields (k, prob, J_k, rhs_k, ||F(u_k)||_2); then calls solve(k, J_k, rhs_k) -> delta_k
    (interleaved (dp, dS)) and sets u_{k+1} = u_k + delta_k.

    chop (reading R17): per-cell saturation update limited to |dS| <= chop and S_n kept in
    [0, 1] (Appleyard-type chop; "a variant of Newton's method").  Measured on C5:
    the undamped sequence diverges (||F|| grows 400x in four steps, S leaves [0, 1]).
    chop=None gives the undamped iteration of reading Q18."""
    prob = make_problem(config, gravity, dims)
    p, sn = prob.p_old.copy(), prob.sn_old.copy()
    for k in range(steps):
        J = jacobian(prob, p, sn)
        R = residual(prob, p, sn).reshape(-1)
        rhs = np.ascontiguousarray(-R)
        prob._p_cur, prob._sn_cur = p, sn     # the state u_k of this Jacobian (diagnostics)
        yield k, prob, J, rhs, float(np.linalg.norm(R))
        delta = np.asarray(solve(k, J, rhs), dtype=np.float64)
        dS = delta[1::2]
        if chop is not None:
            dS = np.clip(dS, -chop, chop)
        p = p + delta[0::2]
        sn = sn + dS
        if chop is not None:
            sn = np.clip(sn, 0.0, 1.0)
