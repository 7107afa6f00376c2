/* bf.h -- C-ABI of the B200-native BF-AMG-GMRES linear solver (libbf.so).
 *
 * The library solves  J c = q for the 2x2-block Jacobian of the fully
 * implicit two-phase (p_w, S_n) cell-centred FV model by
 * restarted GMRES right-preconditioned as  J M^-1 c^ = q, c = M^-1 c^
 * (`precon-system`) with the block-factorization preconditioner
 * M_bf (Algorithm 3; matrix form `m_bf`): one AMG
 * V-cycle on A_ss, the A_ps coupling, one AMG V-cycle on the SIMPLE approximate
 * Schur complement  S~ = A_pp - A_ps diag(A_ss)^-1 A_sp  (`SIMPLE-Schur`,
 * P:L236-241, read with A_sp in the last slot -- DESIGN.md R1).
 *
 * The paper's comparison preconditioners are options of the same handle
 * (bf_options.precond): CPR-AMG(1) / CPR-AMG(2), the two-stage combinative / additive
 * preconditioners of Algorithms 1, 2 with a block ILU(0) of J as the first stage,
 * and the coupled "point" AMG on J itself.
 *
 * Everything on the path runs in hand-written CUDA kernels for sm_100a on one
 * GPU in fp64.  No torch types cross this boundary: plain pointers and sizes.
 *
 * Conventions
 *   - cells c = 0..n_cells-1, c = i + nx*(j + ny*k) (lexicographic).
 *   - Jacobian: point-interleaved 2x2 BSR ("point" ordering):
 *       row_ptr[n_cells+1] (int32, row_ptr[0] = 0, non-decreasing),
 *       col_idx[nnzb]      (int32, strictly ascending within each row, diagonal present),
 *       vals[4*nnzb]       (f64, one 2x2 block per entry).
 *     block_order 0: row-major  {b00, b01, b10, b11};  1: column-major {b00, b10, b01, b11}.
 *     var_order   0: index 0 is (water equation, p_w), index 1 is (n-phase equation, S_n),
 *                    so the canonical block is [[a_pp, a_ps], [a_sp, a_ss]];
 *                 1: indices swapped (S_n first).
 *   - Vectors (rhs, x, ...) have length 2*n_cells, interleaved in the same var_order:
 *     x[2c + ip] = dp_c, x[2c + is] = dS_c (ip = var_order, is = 1 - var_order).
 *   - All calls are ordered on the CUDA stream passed in (cudaStream_t as void*;
 *     NULL = legacy default stream) and block until their host outputs are ready.
 *
 * Ownership: bf_setup copies the Jacobian (host or device) into memory owned by the
 * handle (stream-ordered allocations on the setup stream).  The handle owns every
 * device buffer it allocates; bf_destroy frees them.  Caller buffers are never
 * retained after a call returns.
 *
 * Errors: every call returns a bf_status; no exception crosses the ABI.  On error
 * bf_last_error(h) (or bf_last_error(NULL) for a failed bf_setup) names the failing
 * item (cell, row, level, pivot).  Non-convergence of GMRES is NOT an error:
 * bf_solve returns BF_OK with *converged = 0 and x holding the last iterate.
 * A handle is not thread-safe; distinct handles are independent.
 */
#ifndef BF_H
#define BF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BF_OK = 0,
  BF_ERR_ARG = 1,             /* bad argument / size / option */
  BF_ERR_PATTERN = 2,         /* row_ptr not monotone, col_idx not ascending / out of range, no diagonal block */
  BF_ERR_NONFINITE = 3,       /* NaN/Inf in the Jacobian values or the rhs */
  BF_ERR_ZERO_DIAG = 4,       /* A_ss(c,c) == 0 (S~ needs diag(A_ss)^-1) */
  BF_ERR_COARSE_SINGULAR = 5, /* coarsest AMG matrix singular (|pivot| <= 1e-14 max|a|) */
  BF_ERR_CUDA = 6,            /* CUDA runtime error (message carries cudaGetErrorString) */
  BF_ERR_OOM = 7,             /* device allocation failed */
  BF_ERR_LIMIT = 8            /* an implementation limit was exceeded (message names it) */
} bf_status;

typedef struct {
  int32_t nx, ny, nz;          /* grid; n_cells must equal nx*ny*nz (nx=n_cells,ny=nz=1 allowed) */
  int32_t n_cells;             /* block rows */
  int64_t nnzb;                /* number of 2x2 blocks (== row_ptr[n_cells]) */
  const int32_t *row_ptr;      /* [n_cells+1] */
  const int32_t *col_idx;      /* [nnzb] */
  const double *vals;          /* [4*nnzb] */
  int32_t block_order;         /* 0 row-major, 1 column-major */
  int32_t var_order;           /* 0 (p_w, S_n), 1 (S_n, p_w) */
  int32_t mem;                 /* 0: the three arrays are host pointers, 1: device pointers */
  int32_t reserved;
} bf_bsr2;

typedef struct {
  double theta;                /* strength threshold (R4), default 0.25 */
  int32_t max_levels;          /* default 25 */
  int32_t max_coarse;          /* coarsest level dense-LU size limit, default 64, max 128 */
  int32_t smoother;            /* smoother of the A_ss hierarchy (0): 0 l1-Jacobi, 1 Chebyshev (default;
                                  DESIGN.md R9, R22) */
  int32_t nu_pre, nu_post;     /* smoothing passes, default 1, 1 */
  int32_t cheb_degree;         /* Chebyshev degree, default 2 */
  double cheb_lo;              /* Chebyshev interval [cheb_lo, 1] on D_l1^-1 A, default 0.1 */
  uint64_t seed;               /* PMIS hash seed, default 0x1611 */
  int32_t orth;                /* 0 CGS2 (default), 1 CGS1 */
  int32_t schur_as_printed;    /* 0: A_sp (default, R1); 1: literal P:L239 (A_pp), diagnostics only */
  int32_t interp_norm;         /* 1: interpolation weights normalised so P 1 = 1 (default, R8); 0: Q26 denominators */
  int32_t timing;              /* 1: record CUDA events around the J SpMV, the GMRES
                                  orthogonalisation kernels and the preconditioner apply of every
                                  Arnoldi step (bf_kernel_time); k > 1: of every k-th step only
                                  (sampled, less perturbation of the timed solve); 0: off */
  int32_t precond;             /* preconditioner M of `precon-system`:
                                  0 BF, Algorithm 3 (default; hierarchies 0 A_ss, 1 S~);
                                  1 CPR-AMG(1) combinative, Algorithm 1;
                                  2 CPR-AMG(2) additive, Algorithm 2.
                                  CPR: first stage P_1 = block ILU(0) of J on its block
                                  pattern in point order (R18), second stage
                                  one V-cycle on A_pp (hierarchy 2) [and on A_ss, hierarchy 0].
                                  A singular ILU pivot block is BF_ERR_ZERO_DIAG naming the cell.
                                  3 coupled "point" AMG: one V-cycle of the same AMG on J itself as a
                                  point-ordered scalar 2n x 2n matrix (R20;
                                  hierarchy 3) -- the paper's AMG comparison. */
  int32_t cheb_eig;            /* Chebyshev interval per AMG level (R21): 0 (default) ->
                                  [cheb_lo, 1], 1 the Gershgorin bound of rho(D_l1^-1 A); k > 0 ->
                                  [cheb_lo hi_l, hi_l], hi_l = 1.1 x a k-step power-iteration estimate
                                  of rho(D_l1^-1 A_l) from a fixed hashed start vector (<= 64) */
  int32_t smoother_p;          /* smoother of every other hierarchy (1 S~ of BF, 2 A_pp of CPR, 3 J of the
                                  coupled AMG): default 0 (l1-Jacobi); -1: the same as `smoother`
                                  -- DESIGN.md R22 */
  int32_t cheb_levels;         /* a Chebyshev hierarchy smooths its levels l < cheb_levels with Chebyshev
                                  and the coarser ones with l1-Jacobi; 0: every level (R22) */
  int32_t diag_stop;           /* 1 (default): coarsening stops before a level whose Galerkin operator has a
                                  non-positive diagonal entry; the level above becomes the coarsest one
                                  (dense LU, or 4 l1-Jacobi sweeps when it has more than max_coarse rows)
                                  -- DESIGN.md R23.  0: no such stop.  The hierarchy of the coupled AMG
                                  (precond 3, the paper's failing comparison) never stops this way. */
} bf_options;

typedef struct bf_ctx *bf_handle;

/* Fill *opt with the defaults listed above. */
bf_status bf_default_options(bf_options *opt);

/* Validate and ingest J, build the field split, S~ and
 * the two AMG hierarchies (A_ss and S~; PMIS + classical interpolation + Galerkin,
 * P:L145, L275).  opt may be NULL (defaults).  On success *out is a new handle; on
 * error *out = NULL and all partial state is freed. */
bf_status bf_setup(const bf_bsr2 *J, const bf_options *opt, void *cuda_stream, bf_handle *out);

/* Restarted right-preconditioned GMRES(restart) on J x = rhs.
 *   rhs, x: length 2*n_cells; vec_mem 0 = host pointers, 1 = device pointers.
 *   x: in = x0, out = the last iterate.
 *   tol: relative to ||rhs||_2 (P:L275 form); the Givens estimate drives the loop and
 *        the true residual is recomputed at the end of every cycle (R11).
 *   restart: 1 <= restart <= 256 (BF_ERR_ARG otherwise).  The basis V and the preconditioned
 *        basis Z take (2 restart + 1) * 2 n_cells doubles of device memory (BF_ERR_OOM if they
 *        do not fit); bases longer than 32 vectors are orthogonalised in blocks of 32.
 *   maxit: cap on Arnoldi steps summed over restarts, >= 0.  maxit = 0 takes no step: x stays
 *        x0 and only the initial residual is reported.
 *   *iters: Arnoldi steps taken.  res_hist (host, may be NULL, length >= maxit+1):
 *        res_hist[0] = ||r0||/||rhs||, res_hist[k] = Givens estimate after step k.
 *   *converged: 1 if the true relative residual <= tol.  *final_true_relres: that residual.
 *   ||rhs|| == 0 gives x = 0, iters = 0, converged = 1.
 *   BF_ERR_NONFINITE: a NaN/Inf in rhs or x0 (the message names the first entry and its cell),
 *        or a non-finite Arnoldi coefficient / true residual during the iteration (checked every
 *        Arnoldi step and every cycle end); x then holds the iterate of the last completed cycle. */
bf_status bf_solve(bf_handle h, const double *rhs, double *x, double tol, int32_t restart,
                   int32_t maxit, int32_t vec_mem, int32_t *iters, double *res_hist,
                   int32_t *converged, double *final_true_relres, void *cuda_stream);

/* New Jacobian VALUES on the setup's sparsity pattern (same row_ptr/col_idx, block_order,
 * var_order), e.g. the next Newton iterate J(u_{k+1}).  Setup reuse (SURVEY
 * 8(f) NEXT-1, reading R16 "frozen coarse hierarchy"): the field split, S~ and the FINEST
 * level of both AMG hierarchies (matrix, l1 diagonal) are rebuilt from the new values; the
 * coarse levels (C/F splits, P_l, R_l, A_l for l >= 1, the coarse LU) are kept from the last
 * bf_setup.  A hierarchy that has a single level is rebuilt completely.
 *   vals: [4*nnzb]; mem 0 = host pointer, 1 = device pointer.
 * Errors as bf_setup (BF_ERR_NONFINITE, BF_ERR_ZERO_DIAG naming the cell, ...); on error the
 * handle keeps its previous state only if the error was detected before any rebuild
 * (validation errors), otherwise it must be destroyed. */
bf_status bf_update(bf_handle h, const double *vals, int32_t mem, void *cuda_stream);

/* ---- NEXT-2: device assembly of the two-phase residual and Jacobian ------------------
 * The fully implicit (p_w, S_n) TPFA discretisation of P:L43-83 with the readings of
 * DESIGN.md R2 (the same model as the seeded generator workload/twophase.py): uniform
 * grid of cell size h, isotropic per-cell permeability, quadratic k_r, P_c model
 * (pc_kind 0 none, 1 Brooks-Corey (a = P_d, b = lambda), 2 van Genuchten (a = n,
 * b = alpha), 3 linear (a = P_0)), gravity along gravity_axis (-1: none), Dirichlet faces
 * (axis, side 0 = low / 1 = high, pressure; S_n of the boundary state = S_n^n of the cell),
 * optional water mass source [kg/s]. All array pointers are DEVICE pointers. */
typedef struct {
  int32_t nx, ny, nz;
  double h, phi, rho_w, rho_n, mu_w, mu_n, g, dt;
  int32_t gravity_axis;
  int32_t pc_kind;
  double pc_a, pc_b;
  int32_t n_dirichlet;
  int32_t dir_axis[6], dir_side[6];
  double dir_p[6];
  const double *perm;      /* [n] m^2 */
  const double *sn_old;    /* [n] S_n^n */
  const double *source_w;  /* [n] kg/s or NULL */
} bf_twophase;

/* Number of 2x2 blocks of the assembled Jacobian: n + 2 * (interior faces). */
int64_t bf_assemble_nnzb(int32_t nx, int32_t ny, int32_t nz);

/* Assemble R(u) and J(u) at the state (p, S_n) (device arrays of n): writes row_ptr[n+1],
 * col_idx[nnzb] (ascending, all grid-adjacency blocks), vals[4 nnzb] (row-major,
 * var_order 0) and residual[2n] interleaved (R_w, R_n) (mass form).  The
 * Jacobian is exact with frozen upwind directions.  Device buffers. */
bf_status bf_assemble(const bf_twophase *prob, const double *p, const double *sn, int32_t *row_ptr,
                      int32_t *col_idx, double *vals, double *residual, void *cuda_stream);

/* Newton state update u <- u + delta (delta interleaved, device arrays): p += dp;
 * S_n += clip(dS, -chop, chop) then clipped to [0, 1] when chop > 0 (reading R17). */
bf_status bf_newton_update(int32_t n, double *p, double *sn, const double *delta, double chop,
                           void *cuda_stream);

/* Free all device memory of the handle (NULL is a no-op). */
bf_status bf_destroy(bf_handle h);

/* Last error message of the handle; NULL: the calling thread's last bf_setup error. */
const char *bf_last_error(bf_handle h);

/* ---- introspection (parity tests, statistics) ---------------------------------- */
/* y = J x (P:L138-140 operator), vectors as in bf_solve. */
bf_status bf_spmv(bf_handle h, const double *x, double *y, int32_t vec_mem, void *cuda_stream);
/* z = M^-1 r: one application of the handle's preconditioner (Algorithm 3, or
 * Algorithm 1/2, per opt.precond). */
bf_status bf_apply_precond(bf_handle h, const double *r, double *z, int32_t vec_mem, void *cuda_stream);
/* x = one V-cycle of hierarchy `which` (0 A_ss, 1 S~, 2 A_pp, 3 J scalar) applied to b (length
 * n_cells; 2 n_cells for hierarchy 3, canonical (p,s) interleaving).
 * BF_ERR_ARG for a hierarchy the handle's preconditioner does not build. */
bf_status bf_vcycle(bf_handle h, int32_t which, const double *b, double *x, int32_t vec_mem,
                    void *cuda_stream);
bf_status bf_num_levels(bf_handle h, int32_t which, int32_t *nlev);
/* Level sizes; then (optionally, host buffers of the reported sizes, any may be NULL)
 * A_l (CSR, int32 row_ptr[n+1]), cf[n] (1 = C, 0 = F; level < nlev-1), P_l (n x n_{l+1}),
 * the l1 diagonal dl1[n]. */
bf_status bf_get_level(bf_handle h, int32_t which, int32_t level, int32_t *n, int64_t *nnz_A,
                       int64_t *nnz_P, int32_t *A_rowptr, int32_t *A_col, double *A_val,
                       int8_t *cf, int32_t *P_rowptr, int32_t *P_col, double *P_val, double *dl1);
/* The smoother parameters of level `level` of hierarchy `which`: *cheb_hi = upper end of the
 * Chebyshev interval [cheb_lo hi, hi] (1 unless opt.cheb_eig > 0, R21), *beta0 = the
 * scaling of the first smoothing step from zero, x0 = beta0 b ./ dl1.  Either may be NULL. */
bf_status bf_get_level_smoother(bf_handle h, int32_t which, int32_t level, double *cheb_hi, double *beta0);
/* which: 0 A_pp, 1 A_ps, 2 A_sp, 3 A_ss, 4 S~ (S~ only for precond 0).  Sizes first; arrays
 * optional (host). */
bf_status bf_get_block(bf_handle h, int32_t which, int64_t *nnz, int32_t *rowptr, int32_t *col,
                       double *val);
/* CPR handles (precond 1, 2): the block ILU(0) factors of J copied to host buffers
 * (either may be NULL): lu[4 nnzb] on J's block pattern, canonical row-major (p,s) blocks --
 * strictly lower blocks hold L_ik (L unit block-lower), the others U_ij; dinv[4 n] the inverses
 * of U's diagonal blocks.  *levels (may be NULL): number of dependency levels of the
 * triangular sweeps.  BF_ERR_ARG on a BF handle. */
bf_status bf_get_ilu(bf_handle h, double *lu, double *dinv, int32_t *levels);
/* CPR handles: x = (L U)^-1 r, the ILU(0) forward and backward sweeps (vectors as bf_solve). */
bf_status bf_ilu_solve(bf_handle h, const double *r, double *x, int32_t vec_mem, void *cuda_stream);
/* Accumulated device time (ms, CUDA events on the solve stream), number of timed
 * regions and ALGORITHMIC bytes moved (each operand once per use)
 * of an instrumented kernel class since setup (requires opt.timing = 1):
 *   0 J SpMV (36 nnzb + 36 n bytes per launch), 1 GMRES orthogonalisation passes,
 *   2 whole preconditioner apply, 3 whole bf_solve.  Any output pointer may be NULL. */
bf_status bf_kernel_time(bf_handle h, int32_t kclass, double *ms, int64_t *launches, double *alg_bytes);
/* Number of kernels this library launched since the handle was created. */
bf_status bf_launch_count(bf_handle h, int64_t *launches);
/* Device bytes currently held by the handle. */
bf_status bf_device_bytes(bf_handle h, int64_t *bytes);

#ifdef __cplusplus
}
#endif
#endif
