/* oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, sequential CPU oracle of the BF-AMG-GMRES linear-solve hot path of
 * arXiv 1611.00127 with the
 * readings of SURVEY.md section 8(c) (c.2 step by step, c.4 determinism contract).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code, header or constant generator
 * with the CUDA path (paper_1611_00127_b200/), and the CUDA path never loads it.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no FMA contraction, IEEE binary64,
 * round to nearest: c.4 item 1).
 */
#ifndef BF_ORACLE_H
#define BF_ORACLE_H
#include <stdint.h>

typedef struct {
  int32_t nrows, ncols;
  int64_t nnz;
  int64_t *rp;   /* [nrows+1] */
  int32_t *ci;   /* [nnz] strictly ascending per row */
  double  *v;    /* [nnz] */
} or_csr;

typedef struct {
  double   theta;          /* strength threshold (Q24), 0.25 */
  int32_t  max_levels;     /* 25 (Q28) */
  int32_t  max_coarse;     /* 64 (Q28) */
  int32_t  smoother;       /* 0 l1-Jacobi, 1 Chebyshev (Q27): the A_ss hierarchy (R22; default 1) */
  int32_t  nu_pre, nu_post;/* 1, 1 */
  int32_t  cheb_degree;    /* 2 */
  double   cheb_lo;        /* 0.1 (R22) */
  uint64_t seed;           /* PMIS hash seed (Q25) */
  int32_t  orth;           /* 0 CGS2, 1 CGS1 (Q30) */
  int32_t  schur_as_printed; /* 0: A_sp (Q21); 1: literal P:L239 (A_pp) */
  int32_t  interp_norm;    /* 1: weights normalised to P 1 = 1 (R8, default); 0: Q26 denominators */
  int32_t  precond;        /* 0: BF (Algorithm 3, default); 1: CPR-AMG(1) combinative (Algorithm 1);
                              2: CPR-AMG(2) additive (Algorithm 2) -- P:L159-193, SURVEY 8(f) NEXT-3;
                              3: coupled "point" AMG, one V-cycle on J itself as a scalar matrix in
                                 point ordering (reading R20) */
  int32_t  cheb_eig;       /* Chebyshev interval per level (R21): 0 -> [cheb_lo, 1] (Gershgorin
                              bound of D_l1^-1 A); k > 0 -> [cheb_lo hi_l, hi_l], hi_l = 1.1 x the
                              k-step power-iteration estimate of rho(D_l1^-1 A_l) */
  int32_t  smoother_p;     /* smoother of every other hierarchy (S~ of BF, A_pp of CPR, J of the coupled
                              AMG), default 0 (l1-Jacobi); -1: the same as `smoother` -- R22 */
  int32_t  cheb_levels;    /* Chebyshev hierarchies smooth levels l < cheb_levels with Chebyshev and the
                              coarser ones with l1-Jacobi; 0: every level (R22) */
  int32_t  diag_stop;      /* 1 (default): coarsening stops before a Galerkin level with a non-positive
                              diagonal entry (R23); 0: classical, no such stop.  The coupled AMG's
                              hierarchy (precond 3) never stops this way (R23) */
} or_options;

#define OR_MAX_LEVELS 64

typedef struct {
  int32_t nlev;
  or_csr A[OR_MAX_LEVELS];        /* A_0 .. A_{L} */
  or_csr P[OR_MAX_LEVELS];        /* P_l : n_l x n_{l+1}, l < L */
  or_csr R[OR_MAX_LEVELS];        /* R_l = P_l^T */
  int8_t *cf[OR_MAX_LEVELS];      /* 1 = C, 0 = F (levels l < L) */
  uint8_t *strong[OR_MAX_LEVELS]; /* per-nnz strength flags of A_l (l < L) */
  double *dl1[OR_MAX_LEVELS];     /* l1 diagonal of every level */
  double cheb_hi[OR_MAX_LEVELS];  /* upper end of each level's Chebyshev interval (R21) */
  double *lu;                     /* dense LU of A_L (row-major n_L x n_L) or NULL */
  int32_t *piv;                   /* pivot rows */
  or_options opt;
} or_amg;

typedef struct {
  int32_t n;                      /* cells */
  int32_t var_order;
  int32_t block_order;
  /* the input Jacobian (BSR2 in canonical row-major (p,s) order) */
  int64_t *brp; int32_t *bci; double *bv;
  or_csr App, Aps, Asp, Ass, S;   /* field split and S~ */
  double *dss;                    /* diag(A_ss) */
  or_amg hss, hS;                 /* hierarchies for A_ss and S~ */
  or_options opt;
  /* CPR-AMG(1)/(2): AMG on A_pp and the block ILU(0) P_1 of J */
  or_amg hpp;                     /* hierarchy for A_pp (precond 1, 2) */
  double *ilu;                    /* [4 nnzb] block ILU(0) factors on J's block pattern: strictly lower
                                     blocks hold L_ik (unit block-lower L), the rest hold U_ij */
  double *ilu_dinv;               /* [4 n] inverse of U's diagonal (pivot) blocks */
  /* coupled point AMG (precond 3) */
  or_csr Jsc;                     /* J as a scalar 2n x 2n CSR, point ordering (p,s per cell) */
  or_amg hJ;                      /* its hierarchy */
} or_bf;

#ifdef __cplusplus
extern "C" {
#endif
const char *or_last_error(void);
void or_default_options(or_options *o);
uint32_t or_h32(uint64_t seed, int32_t level, int64_t i);

void or_bsr_spmv(int32_t n, const int64_t *rp, const int32_t *ci, const double *v,
                 const double *x, double *y);
void or_csr_spmv(const or_csr *A, const double *x, double *y);

int  or_split(int32_t n, const int64_t *rp, const int32_t *ci, const double *vals,
              int32_t block_order, int32_t var_order,
              or_csr *App, or_csr *Aps, or_csr *Asp, or_csr *Ass, double *dss);
int  or_schur(const or_csr *App, const or_csr *Aps, const or_csr *Asp, const double *dss,
              int32_t as_printed, or_csr *S);
void or_strength(const or_csr *A, double theta, uint8_t *strong);
void or_pmis(const or_csr *A, const uint8_t *strong, const uint32_t *h32, int8_t *cf);
int  or_interp(const or_csr *A, const uint8_t *strong, const int8_t *cf, int32_t norm, or_csr *P);
void or_transpose(const or_csr *P, or_csr *R);
void or_matmul(const or_csr *A, const or_csr *B, or_csr *C);
void or_l1diag(const or_csr *A, double *d);
/* k-step power-iteration estimate of the spectral radius of D^-1 A (d = l1 diagonal), start vector
 * v_i = h32(seed, level + 4096, i) / 2^32 - 1/2 (R21) */
double or_power_estimate(const or_csr *A, const double *d, int32_t steps, uint64_t seed, int32_t level);
/* one smoothing pass (kind 0: l1-Jacobi, 1: Chebyshev of `degree` on [lo hi, hi]) with diagonal d */
void or_smooth(const or_csr *A, const double *d, const double *b, double *x, int32_t kind,
               int32_t degree, double lo, double hi);
int  or_amg_setup(const or_csr *A0, const or_options *o, or_amg *h);
void or_amg_free(or_amg *h);
void or_vcycle(const or_amg *h, const double *b, double *x);
void or_csr_free(or_csr *A);

/* block ILU(0) of a point-ordered 2x2 BSR matrix (canonical (p,s) row-major blocks) on its own
 * block pattern ("incomplete factorization with no fill ILU(0)"; reading R18); returns 0,
 * or -1 - i if the pivot block of row i is singular (or no diagonal block) */
int  or_ilu0(int32_t n, const int64_t *rp, const int32_t *ci, const double *v, double *lu, double *dinv);
/* x = (L U)^-1 r on canonical interleaved vectors (forward then backward block substitution) */
void or_ilu0_solve(int32_t n, const int64_t *rp, const int32_t *ci, const double *lu, const double *dinv,
                   const double *r, double *x);
/* J as a scalar CSR in point ordering (row 2c+r, column 2d+s = entry (r,s) of block (c,d));
 * pattern = entries that are not +-0.0, plus the diagonal (the Q23 convention of the split) */
void or_jscalar(int32_t n, const int64_t *rp, const int32_t *ci, const double *v, or_csr *out);
int  or_bf_setup(int32_t n, const int64_t *rp, const int32_t *ci, const double *vals,
                 int32_t block_order, int32_t var_order, const or_options *o, or_bf **out);
void or_bf_free(or_bf *b);
int  or_bf_update(or_bf *b, const double *vals);
void or_bf_apply(const or_bf *b, const double *v, double *z);
void or_bf_spmv(const or_bf *b, const double *x, double *y);
int  or_gmres(const or_bf *b, const double *rhs, double *x, double tol, int32_t restart,
              int32_t maxit, int32_t *iters, double *res_hist, int32_t *converged,
              double *final_relres);
/* test hook: capture V, the unrotated Hbar and k of the next or_gmres call's first cycle */
void or_gmres_capture(double *V, double *Hbar, int32_t *k);
#ifdef __cplusplus
}
#endif
#endif
