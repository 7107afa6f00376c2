/* oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain, slow, obviously-correct, single-threaded CPU implementation of the
 * BF-AMG-GMRES hot path, written step by step in the order of SURVEY.md c.2,
 * each function citing the PAPER.md passage (P:Lnnn) or reading (Qnn) it follows.
 * Dense per-row accumulators, no blocking, no fusion, no reordering.
 * Floating point: IEEE binary64, compiled with -ffp-contract=off (c.4).
 */
#include "oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
static void set_err(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}
const char *or_last_error(void) { return g_err; }

static void *xmalloc(size_t n) {
  void *p = malloc(n ? n : 1);
  if (!p) { fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n); abort(); }
  return p;
}
static void *xcalloc(size_t n, size_t s) {
  void *p = calloc(n ? n : 1, s ? s : 1);
  if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
  return p;
}

void or_default_options(or_options *o) {
  o->theta = 0.25;        /* Q24 */
  o->max_levels = 25;     /* Q28 */
  o->max_coarse = 64;     /* Q28 */
  o->smoother = 1;        /* Q27, R22: Chebyshev(2) on [0.1, 1] for A_ss ... */
  o->nu_pre = 1;
  o->nu_post = 1;
  o->cheb_degree = 2;
  o->cheb_lo = 0.1;
  o->seed = 0x1611ULL;
  o->orth = 0;            /* Q30: CGS2 */
  o->schur_as_printed = 0;/* Q21 */
  o->interp_norm = 1;     /* R8 */
  o->precond = 0;         /* BF, Algorithm 3 */
  o->cheb_eig = 0;        /* R21: Gershgorin interval end 1 */
  o->smoother_p = 0;      /* ... and l1-Jacobi for S~ / A_pp / J (R22) */
  o->cheb_levels = 0;     /* R22 */
  o->diag_stop = 1;       /* R23 */
}

/* options of one hierarchy: every hierarchy but A_ss (S~, A_pp, J) takes smoother_p (R22) */
static or_options hier_options(const or_options *o, int pressure) {
  or_options h = *o;
  if (pressure && o->smoother_p >= 0) h.smoother = o->smoother_p;
  return h;
}

void or_csr_free(or_csr *A) {
  free(A->rp); free(A->ci); free(A->v);
  A->rp = NULL; A->ci = NULL; A->v = NULL; A->nnz = 0;
}

static void csr_alloc(or_csr *A, int32_t nrows, int32_t ncols, int64_t nnz) {
  A->nrows = nrows; A->ncols = ncols; A->nnz = nnz;
  A->rp = (int64_t *)xcalloc((size_t)nrows + 1, sizeof(int64_t));
  A->ci = (int32_t *)xmalloc((size_t)nnz * sizeof(int32_t));
  A->v = (double *)xmalloc((size_t)nnz * sizeof(double));
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* sign convention used by strength and interpolation: sigma = -1 if a_ii < 0 else +1 (Q24) */
static double diag_sign(const or_csr *A, int32_t i) {
  for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++)
    if (A->ci[q] == i) return A->v[q] < 0.0 ? -1.0 : 1.0;
  return 1.0;
}

/* the smoother of level l (R22): Chebyshev on the levels l < cheb_levels of a Chebyshev hierarchy */
static int level_cheb(const or_options *o, int32_t l) {
  return o->smoother == 1 && (o->cheb_levels == 0 || l < o->cheb_levels);
}

/* ------------------------------------------------------------------------ */
/* SplitMix64 finalizer hash for PMIS weights (Q25).                          */
/* ------------------------------------------------------------------------ */
uint32_t or_h32(uint64_t seed, int32_t level, int64_t i) {
  uint64_t z = seed ^ ((uint64_t)level * 0x9E3779B97F4A7C15ULL) ^ (uint64_t)i;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  return (uint32_t)(z >> 32);
}

/* ------------------------------------------------------------------------ */
/* w = J z, J in point-interleaved 2x2 BSR.          */
/* canonical block layout: v[4q+0]=a_pp v[4q+1]=a_ps v[4q+2]=a_sp v[4q+3]=a_ss */
/* ------------------------------------------------------------------------ */
void or_bsr_spmv(int32_t n, const int64_t *rp, const int32_t *ci, const double *v,
                 const double *x, double *y) {
  for (int32_t r = 0; r < n; r++) {
    double y0 = 0.0, y1 = 0.0;
    for (int64_t q = rp[r]; q < rp[r + 1]; q++) {
      int32_t c = ci[q];
      y0 = y0 + v[4 * q + 0] * x[2 * c] + v[4 * q + 1] * x[2 * c + 1];
      y1 = y1 + v[4 * q + 2] * x[2 * c] + v[4 * q + 3] * x[2 * c + 1];
    }
    y[2 * r] = y0;
    y[2 * r + 1] = y1;
  }
}

void or_csr_spmv(const or_csr *A, const double *x, double *y) {
  for (int32_t i = 0; i < A->nrows; i++) {
    double s = 0.0;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) s = s + A->v[q] * x[A->ci[q]];
    y[i] = s;
  }
}

/* ------------------------------------------------------------------------ */
/* Field split (restrictions R_p, R_s P:L174-187; Q22, Q23)  */
/* pattern = stored entries whose value is not +-0.0, plus the diagonal.      */
/* ------------------------------------------------------------------------ */
static int blk_index(int32_t block_order, int32_t var_order, int r, int c) {
  if (var_order) { r = 1 - r; c = 1 - c; }
  return block_order == 0 ? 2 * r + c : 2 * c + r;
}

int or_split(int32_t n, const int64_t *rp, const int32_t *ci, const double *vals,
             int32_t block_order, int32_t var_order,
             or_csr *App, or_csr *Aps, or_csr *Asp, or_csr *Ass, double *dss) {
  or_csr *out[4] = {App, Aps, Asp, Ass};
  int idx[4] = {blk_index(block_order, var_order, 0, 0), blk_index(block_order, var_order, 0, 1),
                blk_index(block_order, var_order, 1, 0), blk_index(block_order, var_order, 1, 1)};
  for (int b = 0; b < 4; b++) {
    int64_t nnz = 0;
    for (int32_t r = 0; r < n; r++)
      for (int64_t q = rp[r]; q < rp[r + 1]; q++)
        if (vals[4 * q + idx[b]] != 0.0 || ci[q] == r) nnz++;
    csr_alloc(out[b], n, n, nnz);
    int64_t k = 0;
    for (int32_t r = 0; r < n; r++) {
      out[b]->rp[r] = k;
      for (int64_t q = rp[r]; q < rp[r + 1]; q++) {
        double a = vals[4 * q + idx[b]];
        if (a != 0.0 || ci[q] == r) { out[b]->ci[k] = ci[q]; out[b]->v[k] = a; k++; }
      }
    }
    out[b]->rp[n] = k;
  }
  for (int32_t r = 0; r < n; r++) {
    dss[r] = 0.0;
    for (int64_t q = Ass->rp[r]; q < Ass->rp[r + 1]; q++)
      if (Ass->ci[q] == r) dss[r] = Ass->v[q];
    if (dss[r] == 0.0) {                      /* error naming the cell */
      set_err("A_ss diagonal is zero at cell %d", (int)r);
      return 4;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* SIMPLE approximate Schur complement (`SIMPLE-Schur`, with the  */
/* A_sp reading Q21):  S~ = A_pp - A_ps diag(A_ss)^-1 A_sp.  c.2 step 2.      */
/* ------------------------------------------------------------------------ */
int or_schur(const or_csr *App, const or_csr *Aps, const or_csr *Asp, const double *dss,
             int32_t as_printed, or_csr *S) {
  const or_csr *B = as_printed ? App : Asp;   /* literal P:L239 uses A_pp */
  int32_t n = App->nrows;
  int32_t *pos = (int32_t *)xmalloc((size_t)n * sizeof(int32_t));
  for (int32_t j = 0; j < n; j++) pos[j] = -1;
  int32_t *list = (int32_t *)xmalloc((size_t)n * sizeof(int32_t));
  /* symbolic: row pattern = pattern(A_pp,i) U {j : k in pattern(A_ps,i), j in pattern(B,k)} */
  int64_t *cnt = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t));
  for (int32_t i = 0; i < n; i++) {
    int32_t len = 0;
    for (int64_t q = App->rp[i]; q < App->rp[i + 1]; q++) {
      int32_t j = App->ci[q];
      if (pos[j] < 0) { pos[j] = 1; list[len++] = j; }
    }
    for (int64_t q = Aps->rp[i]; q < Aps->rp[i + 1]; q++) {
      int32_t k = Aps->ci[q];
      for (int64_t t = B->rp[k]; t < B->rp[k + 1]; t++) {
        int32_t j = B->ci[t];
        if (pos[j] < 0) { pos[j] = 1; list[len++] = j; }
      }
    }
    for (int32_t t = 0; t < len; t++) pos[list[t]] = -1;
    cnt[i + 1] = cnt[i] + len;
  }
  csr_alloc(S, n, n, cnt[n]);
  memcpy(S->rp, cnt, ((size_t)n + 1) * sizeof(int64_t));
  free(cnt);
  for (int32_t i = 0; i < n; i++) {
    int32_t len = 0;
    for (int64_t q = App->rp[i]; q < App->rp[i + 1]; q++) {
      int32_t j = App->ci[q];
      if (pos[j] < 0) { pos[j] = 1; list[len++] = j; }
    }
    for (int64_t q = Aps->rp[i]; q < Aps->rp[i + 1]; q++)
      for (int64_t t = B->rp[Aps->ci[q]]; t < B->rp[Aps->ci[q] + 1]; t++) {
        int32_t j = B->ci[t];
        if (pos[j] < 0) { pos[j] = 1; list[len++] = j; }
      }
    qsort(list, (size_t)len, sizeof(int32_t), cmp_i32);
    int64_t base = S->rp[i];
    for (int32_t t = 0; t < len; t++) {
      pos[list[t]] = (int32_t)t;
      S->ci[base + t] = list[t];
      S->v[base + t] = 0.0;                              /* +0.0 if absent from A_pp */
    }
    for (int64_t q = App->rp[i]; q < App->rp[i + 1]; q++) S->v[base + pos[App->ci[q]]] = App->v[q];
    for (int64_t q = Aps->rp[i]; q < Aps->rp[i + 1]; q++) {   /* k ascending */
      int32_t k = Aps->ci[q];
      double t = Aps->v[q] / dss[k];
      for (int64_t u = B->rp[k]; u < B->rp[k + 1]; u++) {
        int64_t p = base + pos[B->ci[u]];
        double prod = t * B->v[u];
        S->v[p] = S->v[p] - prod;
      }
    }
    for (int32_t t = 0; t < len; t++) pos[list[t]] = -1;
  }
  free(pos);
  free(list);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Classical strength of connection ("classical AMG", reading Q24).    */
/* S_i = {j != i : -sigma_i a_ij >= theta * m_i}, m_i = max_{k!=i} -sigma_i a_ik */
/* ------------------------------------------------------------------------ */
void or_strength(const or_csr *A, double theta, uint8_t *strong) {
  for (int32_t i = 0; i < A->nrows; i++) {
    double sg = diag_sign(A, i);
    double m = -INFINITY;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++)
      if (A->ci[q] != i && -sg * A->v[q] > m) m = -sg * A->v[q];
    double thr = theta * m;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++)
      strong[q] = (uint8_t)(m > 0.0 && A->ci[q] != i && -sg * A->v[q] >= thr);
  }
}

/* ------------------------------------------------------------------------ */
/* PMIS coarsening (reading Q25, replacing CLJP of P:L275).                    */
/* key_i = lambda_i * 2^32 + h32_i, ties by index; synchronous rounds.         */
/* cf: 1 = C, 0 = F.                                                           */
/* ------------------------------------------------------------------------ */
void or_pmis(const or_csr *A, const uint8_t *strong, const uint32_t *h32, int8_t *cf) {
  int32_t n = A->nrows;
  /* transpose of the strength graph: ST[i] = {j : i in S_j} */
  int64_t *trp = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t));
  for (int32_t i = 0; i < n; i++)
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++)
      if (strong[q]) trp[A->ci[q] + 1]++;
  for (int32_t i = 0; i < n; i++) trp[i + 1] += trp[i];
  int32_t *tci = (int32_t *)xmalloc((size_t)trp[n] * sizeof(int32_t));
  int64_t *fill = (int64_t *)xmalloc((size_t)n * sizeof(int64_t));
  for (int32_t i = 0; i < n; i++) fill[i] = trp[i];
  for (int32_t i = 0; i < n; i++)
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++)
      if (strong[q]) tci[fill[A->ci[q]]++] = i;
  free(fill);
  uint64_t *key = (uint64_t *)xmalloc((size_t)n * sizeof(uint64_t));
  int8_t *state = (int8_t *)xmalloc((size_t)n);   /* -1 undecided, 0 F, 1 C */
  int64_t nU = 0;
  for (int32_t i = 0; i < n; i++) {
    uint64_t lam = (uint64_t)(trp[i + 1] - trp[i]);   /* lambda_i = #{j : i in S_j} */
    key[i] = (lam << 32) | (uint64_t)h32[i];
    state[i] = lam == 0 ? 0 : -1;                      /* lambda_i = 0 -> F */
    if (state[i] < 0) nU++;
  }
  int8_t *cnew = (int8_t *)xmalloc((size_t)n);
#define GREATER(a, b) (key[a] > key[b] || (key[a] == key[b] && (a) > (b)))
  while (nU > 0) {
    /* C_new = {i in U : (key_i,i) > (key_j,j) for all j in U cap (S_i cup S_i^T)} */
    for (int32_t i = 0; i < n; i++) {
      cnew[i] = 0;
      if (state[i] >= 0) continue;
      int ok = 1;
      for (int64_t q = A->rp[i]; q < A->rp[i + 1] && ok; q++) {
        int32_t j = A->ci[q];
        if (strong[q] && state[j] < 0 && !GREATER(i, j)) ok = 0;
      }
      for (int64_t q = trp[i]; q < trp[i + 1] && ok; q++) {
        int32_t j = tci[q];
        if (state[j] < 0 && !GREATER(i, j)) ok = 0;
      }
      cnew[i] = (int8_t)ok;
    }
    /* F_new = {i in U \ C_new : S_i cap C_new != empty}; then U <- U \ (C_new cup F_new) */
    for (int32_t i = 0; i < n; i++) {
      if (state[i] >= 0 || cnew[i]) continue;
      for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++)
        if (strong[q] && cnew[A->ci[q]]) { state[i] = 0; nU--; break; }
    }
    for (int32_t i = 0; i < n; i++)
      if (cnew[i]) { state[i] = 1; nU--; }
  }
#undef GREATER
  for (int32_t i = 0; i < n; i++) cf[i] = state[i];
  free(cnew); free(state); free(key); free(tci); free(trp);
}

/* ------------------------------------------------------------------------ */
/* Classical (Ruge-Stueben) interpolation (reading Q26; c.2 step 3.3) */
/* ------------------------------------------------------------------------ */
int or_interp(const or_csr *A, const uint8_t *strong, const int8_t *cf, int32_t norm, or_csr *P) {
  int32_t n = A->nrows;
  int32_t *cidx = (int32_t *)xmalloc((size_t)n * sizeof(int32_t));
  int32_t nc = 0;
  for (int32_t i = 0; i < n; i++) cidx[i] = cf[i] == 1 ? nc++ : -1;
  /* symbolic: C row -> 1 entry; F row -> |C_i| entries (C_i = S_i cap C) */
  int64_t *rp = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t));
  for (int32_t i = 0; i < n; i++) {
    int64_t c = 0;
    if (cf[i] == 1) c = 1;
    else
      for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++)
        if (strong[q] && cf[A->ci[q]] == 1) c++;
    rp[i + 1] = rp[i] + c;
  }
  csr_alloc(P, n, nc, rp[n]);
  memcpy(P->rp, rp, ((size_t)n + 1) * sizeof(int64_t));
  free(rp);
  double *num = (double *)xmalloc((size_t)n * sizeof(double));   /* dense by fine column */
  int8_t *inC = (int8_t *)xcalloc((size_t)n, 1);                 /* marks C_i */
  for (int32_t i = 0; i < n; i++) {
    int64_t base = P->rp[i];
    if (cf[i] == 1) { P->ci[base] = cidx[i]; P->v[base] = 1.0; continue; }
    if (P->rp[i + 1] == base) continue;                          /* C_i empty -> empty row */
    double aii = 0.0;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) if (A->ci[q] == i) aii = A->v[q];
    /* pass 1 */
    double dg = aii;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) {
      int32_t j = A->ci[q];
      if (j == i) continue;
      if (strong[q] && cf[j] == 1) { num[j] = A->v[q]; inC[j] = 1; }
      else if (!strong[q]) dg = dg + A->v[q];                    /* weak set W_i */
    }
    /* pass 2: k in F_i^s ascending */
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) {
      int32_t k = A->ci[q];
      if (k == i || !strong[q] || cf[k] == 1) continue;
      double aik = A->v[q];
      double sk = diag_sign(A, k);
      double Dk = 0.0;
      for (int64_t t = A->rp[k]; t < A->rp[k + 1]; t++) {
        int32_t m = A->ci[t];
        if (!inC[m]) continue;
        double abar = (sk * A->v[t] < 0.0) ? A->v[t] : 0.0;
        Dk = Dk + abar;
      }
      if (Dk == 0.0) {
        dg = dg + aik;
      } else {
        double c = aik / Dk;
        for (int64_t t = A->rp[k]; t < A->rp[k + 1]; t++) {
          int32_t m = A->ci[t];
          if (!inC[m]) continue;
          double abar = (sk * A->v[t] < 0.0) ? A->v[t] : 0.0;
          num[m] = num[m] + c * abar;
        }
      }
    }
    /* norm = 0: w_ij = -num_j / dg (Q26).  norm = 1 (R8): w_ij = num_j / s with
     * s = sum_{j in C_i, ascending} num_j from +0.0, i.e. the classical weights scaled so
     * that P 1 = 1 (identical to Q26 on zero-row-sum rows, where -s == dg).
     * A zero denominator gives explicit zeros on the pattern C_i (R7). */
    double den = dg;
    if (norm) {
      den = 0.0;
      for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) {
        int32_t j = A->ci[q];
        if (j != i && inC[j]) den = den + num[j];
      }
    }
    int64_t k = base;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) {
      int32_t j = A->ci[q];
      if (j != i && inC[j]) {
        P->ci[k] = cidx[j];
        if (den == 0.0) P->v[k] = 0.0;
        else P->v[k] = norm ? num[j] / den : -(num[j] / den);
        k++;
        inC[j] = 0;
      }
    }
  }
  free(num); free(inC); free(cidx);
  return 0;
}

/* R = P^T, sorted rows, values copied exactly (c.2 step 3.4) */
void or_transpose(const or_csr *P, or_csr *R) {
  csr_alloc(R, P->ncols, P->nrows, P->nnz);
  for (int64_t q = 0; q < P->nnz; q++) R->rp[P->ci[q] + 1]++;
  for (int32_t I = 0; I < P->ncols; I++) R->rp[I + 1] += R->rp[I];
  int64_t *fill = (int64_t *)xmalloc((size_t)P->ncols * sizeof(int64_t) + 1);
  for (int32_t I = 0; I < P->ncols; I++) fill[I] = R->rp[I];
  for (int32_t i = 0; i < P->nrows; i++)        /* ascending i -> sorted rows of R */
    for (int64_t q = P->rp[i]; q < P->rp[i + 1]; q++) {
      int64_t p = fill[P->ci[q]]++;
      R->ci[p] = i;
      R->v[p] = P->v[q];
    }
  free(fill);
}

/* C = A B; C(i,J) = sum over k in pattern(A,i) ascending of A(i,k) B(k,J), from +0.0,
 * multiply and add rounded separately; full symbolic pattern, no dropping (c.2 step 3.5) */
void or_matmul(const or_csr *A, const or_csr *B, or_csr *C) {
  int32_t n = A->nrows, m = B->ncols;
  int32_t *pos = (int32_t *)xmalloc((size_t)m * sizeof(int32_t) + 4);
  for (int32_t j = 0; j < m; j++) pos[j] = -1;
  int32_t *list = (int32_t *)xmalloc((size_t)m * sizeof(int32_t) + 4);
  int64_t *rp = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t));
  for (int32_t i = 0; i < n; i++) {
    int32_t len = 0;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++)
      for (int64_t t = B->rp[A->ci[q]]; t < B->rp[A->ci[q] + 1]; t++)
        if (pos[B->ci[t]] < 0) { pos[B->ci[t]] = 1; list[len++] = B->ci[t]; }
    for (int32_t t = 0; t < len; t++) pos[list[t]] = -1;
    rp[i + 1] = rp[i] + len;
  }
  csr_alloc(C, n, m, rp[n]);
  memcpy(C->rp, rp, ((size_t)n + 1) * sizeof(int64_t));
  free(rp);
  double *acc = (double *)xmalloc((size_t)m * sizeof(double) + 8);
  for (int32_t i = 0; i < n; i++) {
    int32_t len = 0;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) {       /* k ascending */
      double a = A->v[q];
      int32_t k = A->ci[q];
      for (int64_t t = B->rp[k]; t < B->rp[k + 1]; t++) {
        int32_t J = B->ci[t];
        if (pos[J] < 0) { pos[J] = 1; list[len++] = J; acc[J] = 0.0; }
        double prod = a * B->v[t];
        acc[J] = acc[J] + prod;
      }
    }
    qsort(list, (size_t)len, sizeof(int32_t), cmp_i32);
    int64_t base = C->rp[i];
    for (int32_t t = 0; t < len; t++) {
      C->ci[base + t] = list[t];
      C->v[base + t] = acc[list[t]];
      pos[list[t]] = -1;
    }
  }
  free(acc); free(pos); free(list);
}

/* l1 diagonal d_i = a_ii + sum_{j != i} |a_ij| (c.2 step 3.6; Q27) */
void or_l1diag(const or_csr *A, double *d) {
  for (int32_t i = 0; i < A->nrows; i++) {
    double aii = 0.0;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) if (A->ci[q] == i) aii = A->v[q];
    double s = aii;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) if (A->ci[q] != i) s = s + fabs(A->v[q]);
    d[i] = s;
  }
}

/* rho(D^-1 A) by the power method (R21): v <- D^-1 A v / |D^-1 A v|, estimate |D^-1 A v| for the
 * normalised v of the previous step; the start vector is a fixed hash of (seed, level, i). */
double or_power_estimate(const or_csr *A, const double *d, int32_t steps, uint64_t seed, int32_t level) {
  int32_t n = A->nrows;
  double *v = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  double *w = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  double nv = 0.0;
  for (int32_t i = 0; i < n; i++) {
    v[i] = (double)or_h32(seed, level + 4096, i) / 4294967296.0 - 0.5;
    nv += v[i] * v[i];
  }
  nv = sqrt(nv);
  for (int32_t i = 0; i < n; i++) v[i] = v[i] / nv;
  double lam = 0.0;
  for (int32_t k = 0; k < steps; k++) {
    or_csr_spmv(A, v, w);
    double nw = 0.0;
    for (int32_t i = 0; i < n; i++) {
      w[i] = w[i] / d[i];
      nw += w[i] * w[i];
    }
    lam = sqrt(nw);
    if (lam == 0.0) break;
    for (int32_t i = 0; i < n; i++) v[i] = w[i] / lam;
  }
  free(v); free(w);
  return lam;
}

static void csr_copy(const or_csr *A, or_csr *B) {
  csr_alloc(B, A->nrows, A->ncols, A->nnz);
  memcpy(B->rp, A->rp, ((size_t)A->nrows + 1) * sizeof(int64_t));
  memcpy(B->ci, A->ci, (size_t)A->nnz * sizeof(int32_t));
  memcpy(B->v, A->v, (size_t)A->nnz * sizeof(double));
}

/* ------------------------------------------------------------------------ */
/* AMG setup (c.2 steps 3-4)                                    */
/* ------------------------------------------------------------------------ */
/* 1 if every row of A has a stored diagonal entry > 0 (R23) */
static int or_diag_positive(const or_csr *A) {
  for (int32_t i = 0; i < A->nrows; i++) {
    double aii = 0.0;
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; q++) if (A->ci[q] == i) aii = A->v[q];
    if (!(aii > 0.0)) return 0;
  }
  return 1;
}

int or_amg_setup(const or_csr *A0, const or_options *o, or_amg *h) {
  memset(h, 0, sizeof *h);
  h->opt = *o;
  csr_copy(A0, &h->A[0]);
  int32_t l = 0;
  while (h->A[l].nrows > o->max_coarse && l < o->max_levels - 1 && l < OR_MAX_LEVELS - 1) {
    or_csr *A = &h->A[l];
    int32_t n = A->nrows;
    uint8_t *strong = (uint8_t *)xmalloc((size_t)A->nnz + 1);
    or_strength(A, o->theta, strong);
    uint32_t *hh = (uint32_t *)xmalloc((size_t)n * sizeof(uint32_t));
    for (int32_t i = 0; i < n; i++) hh[i] = or_h32(o->seed, l, i);
    int8_t *cf = (int8_t *)xmalloc((size_t)n);
    or_pmis(A, strong, hh, cf);
    free(hh);
    int32_t nc = 0;
    for (int32_t i = 0; i < n; i++) nc += cf[i] == 1;
    if (nc == 0 || nc == n) {                        /* stop conditions (c.2 3.7) */
      free(strong); free(cf);
      break;
    }
    or_interp(A, strong, cf, o->interp_norm, &h->P[l]);
    or_transpose(&h->P[l], &h->R[l]);
    or_csr AP;
    or_matmul(A, &h->P[l], &AP);
    or_matmul(&h->R[l], &AP, &h->A[l + 1]);
    or_csr_free(&AP);
    /* R23: coarsening stops before a level whose Galerkin operator has a non-positive (or
     * missing) diagonal entry -- the classical strength / interpolation formulas (R4-R8) and the
     * l1 divisor a_ii + sum |a_ij| presuppose a_ii > 0.  Level l then is the coarsest level
     * (the stalled-coarsening rule of c.2 3.7 below: 4 l1-Jacobi sweeps if it is too large for
     * the dense LU). */
    if (o->diag_stop && !or_diag_positive(&h->A[l + 1])) {
      or_csr_free(&h->P[l]); or_csr_free(&h->R[l]); or_csr_free(&h->A[l + 1]);
      free(strong); free(cf);
      break;
    }
    h->cf[l] = cf;
    h->strong[l] = strong;
    l++;
  }
  h->nlev = l + 1;
  for (int32_t k = 0; k < h->nlev; k++) {
    h->dl1[k] = (double *)xmalloc((size_t)h->A[k].nrows * sizeof(double) + 8);
    or_l1diag(&h->A[k], h->dl1[k]);
    h->cheb_hi[k] = 1.0;
    if (level_cheb(o, k) && o->cheb_eig > 0)
      h->cheb_hi[k] = 1.1 * or_power_estimate(&h->A[k], h->dl1[k], o->cheb_eig, o->seed, k);
  }
  /* coarsest level: dense LU with partial pivoting if n_L <= max_coarse (Q28) */
  or_csr *AL = &h->A[l];
  int32_t nL = AL->nrows;
  if (nL <= o->max_coarse) {
    double *lu = (double *)xcalloc((size_t)nL * nL, sizeof(double));
    int32_t *piv = (int32_t *)xmalloc((size_t)nL * sizeof(int32_t) + 4);
    double amax = 0.0;
    for (int32_t i = 0; i < nL; i++)
      for (int64_t q = AL->rp[i]; q < AL->rp[i + 1]; q++) {
        lu[(size_t)i * nL + AL->ci[q]] = AL->v[q];
        if (fabs(AL->v[q]) > amax) amax = fabs(AL->v[q]);
      }
    for (int32_t k = 0; k < nL; k++) {
      int32_t p = k;
      for (int32_t i = k + 1; i < nL; i++)               /* tie -> lowest row index */
        if (fabs(lu[(size_t)i * nL + k]) > fabs(lu[(size_t)p * nL + k])) p = i;
      piv[k] = p;
      if (fabs(lu[(size_t)p * nL + k]) <= 1e-14 * amax) {
        set_err("coarsest matrix (n=%d) singular at pivot %d", (int)nL, (int)k);
        free(lu); free(piv);
        return 5;
      }
      if (p != k)
        for (int32_t j = 0; j < nL; j++) {
          double t = lu[(size_t)k * nL + j];
          lu[(size_t)k * nL + j] = lu[(size_t)p * nL + j];
          lu[(size_t)p * nL + j] = t;
        }
      for (int32_t i = k + 1; i < nL; i++) {
        double f = lu[(size_t)i * nL + k] / lu[(size_t)k * nL + k];
        lu[(size_t)i * nL + k] = f;
        for (int32_t j = k + 1; j < nL; j++) lu[(size_t)i * nL + j] -= f * lu[(size_t)k * nL + j];
      }
    }
    h->lu = lu;
    h->piv = piv;
  }
  return 0;
}

void or_amg_free(or_amg *h) {
  for (int32_t l = 0; l < h->nlev; l++) {
    or_csr_free(&h->A[l]);
    if (l < h->nlev - 1) { or_csr_free(&h->P[l]); or_csr_free(&h->R[l]); }
    free(h->cf[l]); free(h->strong[l]); free(h->dl1[l]);
  }
  free(h->lu); free(h->piv);
  memset(h, 0, sizeof *h);
}

/* x <- x + (b - A x) ./ d  (l1-Jacobi, Q27) */
static void smooth_l1(const or_csr *A, const double *d, const double *b, double *x, double *tmp) {
  int32_t n = A->nrows;
  or_csr_spmv(A, x, tmp);
  for (int32_t i = 0; i < n; i++) x[i] = x[i] + (b[i] - tmp[i]) / d[i];
}

/* Chebyshev acceleration of D^-1 A on [lo hi, hi] (Q27, R21; three-term recurrence) */
static void smooth_cheb(const or_csr *A, const double *d, const double *b, double *x,
                        int32_t degree, double lo, double hi, double *tmp, double *dir) {
  int32_t n = A->nrows;
  double theta = hi * (1.0 + lo) / 2.0, delta = hi * (1.0 - lo) / 2.0;
  double sigma = theta / delta;
  double rho = 1.0 / sigma;
  or_csr_spmv(A, x, tmp);
  for (int32_t i = 0; i < n; i++) { dir[i] = ((b[i] - tmp[i]) / d[i]) / theta; x[i] += dir[i]; }
  for (int32_t k = 1; k < degree; k++) {
    double rho_new = 1.0 / (2.0 * sigma - rho);
    or_csr_spmv(A, x, tmp);
    for (int32_t i = 0; i < n; i++) {
      dir[i] = rho_new * rho * dir[i] + (2.0 * rho_new / delta) * ((b[i] - tmp[i]) / d[i]);
      x[i] += dir[i];
    }
    rho = rho_new;
  }
}

void or_smooth(const or_csr *A, const double *d, const double *b, double *x, int32_t kind,
               int32_t degree, double lo, double hi) {
  double *tmp = (double *)xmalloc((size_t)A->nrows * sizeof(double) + 8);
  double *dir = (double *)xmalloc((size_t)A->nrows * sizeof(double) + 8);
  if (kind == 1) smooth_cheb(A, d, b, x, degree, lo, hi, tmp, dir);
  else smooth_l1(A, d, b, x, tmp);
  free(tmp); free(dir);
}

static void smooth(const or_amg *h, int32_t l, const double *b, double *x, double *tmp, double *dir) {
  if (level_cheb(&h->opt, l))
    smooth_cheb(&h->A[l], h->dl1[l], b, x, h->opt.cheb_degree, h->opt.cheb_lo, h->cheb_hi[l], tmp, dir);
  else
    smooth_l1(&h->A[l], h->dl1[l], b, x, tmp);
}

static void vcycle_rec(const or_amg *h, int32_t l, const double *b, double *x) {
  const or_csr *A = &h->A[l];
  int32_t n = A->nrows;
  for (int32_t i = 0; i < n; i++) x[i] = 0.0;
  double *tmp = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  double *dir = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  if (l == h->nlev - 1) {
    if (h->lu) {                                   /* dense LU solve */
      for (int32_t i = 0; i < n; i++) tmp[i] = b[i];
      for (int32_t k = 0; k < n; k++) {
        int32_t p = h->piv[k];
        if (p != k) { double t = tmp[k]; tmp[k] = tmp[p]; tmp[p] = t; }
      }
      for (int32_t i = 0; i < n; i++)
        for (int32_t j = 0; j < i; j++) tmp[i] -= h->lu[(size_t)i * n + j] * tmp[j];
      for (int32_t i = n - 1; i >= 0; i--) {
        for (int32_t j = i + 1; j < n; j++) tmp[i] -= h->lu[(size_t)i * n + j] * tmp[j];
        tmp[i] /= h->lu[(size_t)i * n + i];
      }
      for (int32_t i = 0; i < n; i++) x[i] = tmp[i];
    } else {                                       /* stalled coarsening: 4 l1-Jacobi sweeps */
      for (int s = 0; s < 4; s++) smooth_l1(A, h->dl1[l], b, x, tmp);
    }
    free(tmp); free(dir);
    return;
  }
  for (int s = 0; s < h->opt.nu_pre; s++) smooth(h, l, b, x, tmp, dir);
  /* r = b - A x; b_c = R r */
  or_csr_spmv(A, x, tmp);
  for (int32_t i = 0; i < n; i++) tmp[i] = b[i] - tmp[i];
  int32_t nc = h->A[l + 1].nrows;
  double *bc = (double *)xmalloc((size_t)nc * sizeof(double) + 8);
  double *ec = (double *)xmalloc((size_t)nc * sizeof(double) + 8);
  or_csr_spmv(&h->R[l], tmp, bc);
  vcycle_rec(h, l + 1, bc, ec);
  or_csr_spmv(&h->P[l], ec, tmp);                   /* x <- x + P e */
  for (int32_t i = 0; i < n; i++) x[i] += tmp[i];
  for (int s = 0; s < h->opt.nu_post; s++) smooth(h, l, b, x, tmp, dir);
  free(bc); free(ec); free(tmp); free(dir);
}

/* one V(nu_pre, nu_post) cycle from x = 0 ("number of V-cycle steps is set to 1") */
void or_vcycle(const or_amg *h, const double *b, double *x) { vcycle_rec(h, 0, b, x); }

/* ------------------------------------------------------------------------ */
/* BF preconditioner (Algorithm 3; matrix form `m_bf` P:L252-257) */
/* ------------------------------------------------------------------------ */
/* ------------------------------------------------------------------------ */
/* Block ILU(0) of J ("For the preconditioner P_1 in step 2 of both     */
/* algorithms, we use the incomplete factorization with no fill ILU(0)").       */
/* Reading R18: the factorization is kept on J's stored 2x2 block pattern in   */
/* the point ordering of P:L145-153 (scalar ILU(0) on a pattern of full 2x2    */
/* blocks is the same factorization up to rounding).  IKJ form of Gaussian     */
/* elimination restricted to the pattern [Saad, ILU(0)]:                       */
/*   for i: for k < i in pattern(i), ascending:                                */
/*            a_ik <- a_ik a_kk^-1                                             */
/*            a_ij <- a_ij - a_ik a_kj   for j > k, (i,j) and (k,j) in pattern  */
/*          a_ii^-1 kept for the backward substitution.                        */
/* 2x2 products: entry (r,c) = A_r0 B_0c + A_r1 B_1c, multiplies and the add   */
/* rounded separately (c.4); inverse by the adjugate: det = a00 a11 - a01 a10. */
/* ------------------------------------------------------------------------ */
static void blk_mul(const double *A, const double *B, double *C) {
  C[0] = A[0] * B[0] + A[1] * B[2];
  C[1] = A[0] * B[1] + A[1] * B[3];
  C[2] = A[2] * B[0] + A[3] * B[2];
  C[3] = A[2] * B[1] + A[3] * B[3];
}

static int blk_inv(const double *A, double *Ai) {
  double det = A[0] * A[3] - A[1] * A[2];
  if (det == 0.0 || !isfinite(det)) return 1;
  Ai[0] = A[3] / det;
  Ai[1] = -A[1] / det;
  Ai[2] = -A[2] / det;
  Ai[3] = A[0] / det;
  return 0;
}

int or_ilu0(int32_t n, const int64_t *rp, const int32_t *ci, const double *v, double *lu, double *dinv) {
  memcpy(lu, v, (size_t)rp[n] * 4 * sizeof(double));
  for (int32_t i = 0; i < n; i++) {
    int64_t d = -1;
    for (int64_t q = rp[i]; q < rp[i + 1]; q++) {
      int32_t k = ci[q];
      if (k == i) d = q;
      if (k >= i) continue;
      double L[4];
      blk_mul(lu + 4 * q, dinv + 4 * (int64_t)k, L);          /* a_ik <- a_ik a_kk^-1 */
      memcpy(lu + 4 * q, L, sizeof L);
      for (int64_t t = q + 1; t < rp[i + 1]; t++) {             /* j > k, (i,j) in pattern */
        int32_t j = ci[t];
        int64_t u = -1;
        for (int64_t w = rp[k]; w < rp[k + 1]; w++)
          if (ci[w] == j) { u = w; break; }
        if (u < 0) continue;                                    /* (k,j) not in pattern: dropped fill */
        double P[4];
        blk_mul(lu + 4 * q, lu + 4 * u, P);                     /* a_ij <- a_ij - a_ik a_kj */
        for (int e = 0; e < 4; e++) lu[4 * t + e] = lu[4 * t + e] - P[e];
      }
    }
    if (d < 0 || blk_inv(lu + 4 * d, dinv + 4 * (int64_t)i)) {
      set_err("ILU(0) pivot block singular (or missing) at cell %d", i);
      return -1 - i;
    }
  }
  return 0;
}

void or_ilu0_solve(int32_t n, const int64_t *rp, const int32_t *ci, const double *lu, const double *dinv,
                   const double *r, double *x) {
  double *y = (double *)xmalloc((size_t)2 * n * sizeof(double) + 8);
  for (int32_t i = 0; i < n; i++) {                             /* L y = r, L unit block-lower */
    double y0 = r[2 * i], y1 = r[2 * i + 1];
    for (int64_t q = rp[i]; q < rp[i + 1]; q++) {
      int32_t k = ci[q];
      if (k >= i) break;
      const double *L = lu + 4 * q;
      y0 = y0 - (L[0] * y[2 * k] + L[1] * y[2 * k + 1]);
      y1 = y1 - (L[2] * y[2 * k] + L[3] * y[2 * k + 1]);
    }
    y[2 * i] = y0;
    y[2 * i + 1] = y1;
  }
  for (int32_t i = n - 1; i >= 0; i--) {                        /* U x = y */
    double t0 = y[2 * i], t1 = y[2 * i + 1];
    for (int64_t q = rp[i]; q < rp[i + 1]; q++) {
      int32_t j = ci[q];
      if (j <= i) continue;
      const double *U = lu + 4 * q;
      t0 = t0 - (U[0] * x[2 * j] + U[1] * x[2 * j + 1]);
      t1 = t1 - (U[2] * x[2 * j] + U[3] * x[2 * j + 1]);
    }
    const double *D = dinv + 4 * (int64_t)i;
    x[2 * i] = D[0] * t0 + D[1] * t1;
    x[2 * i + 1] = D[2] * t0 + D[3] * t1;
  }
  free(y);
}

/* Coupled "point" AMG: "in order to use BoomerAMG for the coupled system ...
 * the Jacobian matrix needs to be ordered by grid points"; reading R20: the interleaved
 * matrix is handed to the scalar AMG of c.2 step 3 as is. */
void or_jscalar(int32_t n, const int64_t *rp, const int32_t *ci, const double *v, or_csr *out) {
  int64_t cnt = 0;
  for (int32_t c = 0; c < n; c++)
    for (int r = 0; r < 2; r++)
      for (int64_t q = rp[c]; q < rp[c + 1]; q++)
        for (int s = 0; s < 2; s++)
          if (v[4 * q + 2 * r + s] != 0.0 || (ci[q] == c && r == s)) cnt++;
  csr_alloc(out, 2 * n, 2 * n, cnt);
  int64_t k = 0;
  for (int32_t c = 0; c < n; c++)
    for (int r = 0; r < 2; r++) {
      for (int64_t q = rp[c]; q < rp[c + 1]; q++)
        for (int s = 0; s < 2; s++)
          if (v[4 * q + 2 * r + s] != 0.0 || (ci[q] == c && r == s)) {
            out->ci[k] = 2 * ci[q] + s;
            out->v[k] = v[4 * q + 2 * r + s];
            k++;
          }
      out->rp[2 * c + r + 1] = k;
    }
}

/* hierarchies the chosen preconditioner uses: BF (Alg. 3) A_ss and S~; CPR-AMG(1) (Alg. 1)
 * A_pp; CPR-AMG(2) (Alg. 2) A_pp and A_ss */
static int build_precond(or_bf *b) {
  const or_options *o = &b->opt;
  int st = 0;
  const or_options ot = hier_options(o, 0), op = hier_options(o, 1);
  if (o->precond == 3) {
    or_jscalar(b->n, b->brp, b->bci, b->bv, &b->Jsc);
    or_options oj = op;
    oj.diag_stop = 0;     /* R23: the paper's coupled AMG comparison stays the classical algorithm */
    return or_amg_setup(&b->Jsc, &oj, &b->hJ);
  }
  if (o->precond == 0 || o->precond == 2) {
    st = or_amg_setup(&b->Ass, &ot, &b->hss);
    if (st) return st;
  }
  if (o->precond == 0) return or_amg_setup(&b->S, &op, &b->hS);
  st = or_amg_setup(&b->App, &op, &b->hpp);
  if (st) return st;
  return or_ilu0(b->n, b->brp, b->bci, b->bv, b->ilu, b->ilu_dinv) ? 4 : 0;
}

int or_bf_setup(int32_t n, const int64_t *rp, const int32_t *ci, const double *vals,
                int32_t block_order, int32_t var_order, const or_options *o, or_bf **out) {
  *out = NULL;
  if (o->precond < 0 || o->precond > 3) { set_err("precond must be 0, 1, 2 or 3"); return 1; }
  or_bf *b = (or_bf *)xcalloc(1, sizeof(or_bf));
  b->n = n;
  b->var_order = var_order;
  b->block_order = block_order;
  b->opt = *o;
  /* canonical copy of J for the SpMV: (p,s) row-major */
  int64_t nnzb = rp[n];
  b->brp = (int64_t *)xmalloc(((size_t)n + 1) * sizeof(int64_t));
  memcpy(b->brp, rp, ((size_t)n + 1) * sizeof(int64_t));
  b->bci = (int32_t *)xmalloc((size_t)nnzb * sizeof(int32_t) + 4);
  memcpy(b->bci, ci, (size_t)nnzb * sizeof(int32_t));
  b->bv = (double *)xmalloc((size_t)nnzb * 4 * sizeof(double) + 8);
  for (int64_t q = 0; q < nnzb; q++)
    for (int r = 0; r < 2; r++)
      for (int c = 0; c < 2; c++) b->bv[4 * q + 2 * r + c] = vals[4 * q + blk_index(block_order, var_order, r, c)];
  b->dss = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  if (o->precond == 1 || o->precond == 2) {
    b->ilu = (double *)xmalloc((size_t)nnzb * 4 * sizeof(double) + 8);
    b->ilu_dinv = (double *)xmalloc((size_t)n * 4 * sizeof(double) + 8);
  }
  int st = or_split(n, rp, ci, vals, block_order, var_order, &b->App, &b->Aps, &b->Asp, &b->Ass, b->dss);
  if (st) { or_bf_free(b); return st; }
  or_schur(&b->App, &b->Aps, &b->Asp, b->dss, o->schur_as_printed, &b->S);
  st = build_precond(b);
  if (st) { or_bf_free(b); return st; }
  *out = b;
  return 0;
}

/* Setup reuse across Newton steps (reading R16 "frozen coarse
 * hierarchy"): new Jacobian values on the same BSR pattern.  The split, S~ and the finest
 * level of every hierarchy (A_0 and its l1 diagonal) are rebuilt from the new values; the
 * coarse levels (C/F, P, R, A_l for l >= 1, coarse LU) are kept.  A hierarchy with a single
 * level is set up again.  CPR: the ILU(0) of J is recomputed. */
int or_bf_update(or_bf *b, const double *vals) {
  int32_t n = b->n;
  int64_t nnzb = b->brp[n];
  for (int64_t q = 0; q < nnzb; q++)
    for (int r = 0; r < 2; r++)
      for (int c = 0; c < 2; c++)
        b->bv[4 * q + 2 * r + c] = vals[4 * q + blk_index(b->block_order, b->var_order, r, c)];
  or_csr_free(&b->App); or_csr_free(&b->Aps); or_csr_free(&b->Asp); or_csr_free(&b->Ass);
  or_csr_free(&b->S);
  int st = or_split(n, b->brp, b->bci, vals, b->block_order, b->var_order, &b->App, &b->Aps, &b->Asp, &b->Ass,
                    b->dss);
  if (st) return st;
  or_schur(&b->App, &b->Aps, &b->Asp, b->dss, b->opt.schur_as_printed, &b->S);
  if (b->opt.precond == 3) {
    or_csr_free(&b->Jsc);
    or_jscalar(n, b->brp, b->bci, b->bv, &b->Jsc);
  }
  or_amg *hs[4] = {&b->hss, &b->hS, &b->hpp, &b->hJ};
  const or_csr *A0[4] = {&b->Ass, &b->S, &b->App, &b->Jsc};
  for (int k = 0; k < 4; k++) {
    or_amg *h = hs[k];
    if (h->nlev == 0) continue;                      /* not used by this preconditioner */
    if (h->nlev <= 1) {
      or_options oh = h->opt;                       /* this hierarchy's options (R22) */
      or_amg_free(h);
      st = or_amg_setup(A0[k], &oh, h);
      if (st) return st;
      continue;
    }
    or_csr_free(&h->A[0]);
    csr_copy(A0[k], &h->A[0]);
    or_l1diag(&h->A[0], h->dl1[0]);
    if (level_cheb(&h->opt, 0) && h->opt.cheb_eig > 0)   /* R21 on the new finest matrix */
      h->cheb_hi[0] = 1.1 * or_power_estimate(&h->A[0], h->dl1[0], h->opt.cheb_eig, h->opt.seed, 0);
  }
  if ((b->opt.precond == 1 || b->opt.precond == 2) && or_ilu0(n, b->brp, b->bci, b->bv, b->ilu, b->ilu_dinv))
    return 4;
  return 0;
}

void or_bf_free(or_bf *b) {
  if (!b) return;
  free(b->brp); free(b->bci); free(b->bv); free(b->dss);
  or_csr_free(&b->App); or_csr_free(&b->Aps); or_csr_free(&b->Asp); or_csr_free(&b->Ass);
  or_csr_free(&b->S);
  or_amg_free(&b->hss); or_amg_free(&b->hS); or_amg_free(&b->hpp); or_amg_free(&b->hJ);
  or_csr_free(&b->Jsc);
  free(b->ilu); free(b->ilu_dinv);
  free(b);
}

/* vectors are interleaved in the caller's var_order: p at 2c+ip, s at 2c+is */
void or_bf_spmv(const or_bf *b, const double *x, double *y) {
  int32_t n = b->n, ip = b->var_order ? 1 : 0, is = 1 - ip;
  double *xc = (double *)xmalloc((size_t)2 * n * sizeof(double) + 8);
  double *yc = (double *)xmalloc((size_t)2 * n * sizeof(double) + 8);
  for (int32_t c = 0; c < n; c++) { xc[2 * c] = x[2 * c + ip]; xc[2 * c + 1] = x[2 * c + is]; }
  or_bsr_spmv(n, b->brp, b->bci, b->bv, xc, yc);
  for (int32_t c = 0; c < n; c++) { y[2 * c + ip] = yc[2 * c]; y[2 * c + is] = yc[2 * c + 1]; }
  free(xc); free(yc);
}

/* Two-stage CPR preconditioners, on the canonical interleaved vector r:
 *   Algorithm 1 (CPR-AMG(1), combinative)        Algorithm 2 (CPR-AMG(2), additive)
 *   u = P_1^-1 r            (step 2, ILU(0))     same
 *   t = r - J u             (step 3)             same
 *   A_pp dp = R_p t         (step 4, one V-cycle) same
 *                                                 A_ss ds = R_s t (step 5, one V-cycle)
 *   u <- u + R_p^T dp       (step 5)             u <- u + R_p^T dp + R_s^T ds (step 6)
 * i.e. M_comb^-1 / M_add^-1 of `m_comb`, `m_add` with V-cycles for A_pp^-1, A_ss^-1. */
static void cpr_apply(const or_bf *b, const double *r, double *u) {
  int32_t n = b->n;
  double *t = (double *)xmalloc((size_t)2 * n * sizeof(double) + 8);
  double *tp = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  double *dp = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  or_ilu0_solve(n, b->brp, b->bci, b->ilu, b->ilu_dinv, r, u);            /* step 2 */
  or_bsr_spmv(n, b->brp, b->bci, b->bv, u, t);                             /* step 3 */
  for (int64_t i = 0; i < 2 * (int64_t)n; i++) t[i] = r[i] - t[i];
  for (int32_t c = 0; c < n; c++) tp[c] = t[2 * c];
  or_vcycle(&b->hpp, tp, dp);                                              /* step 4 */
  if (b->opt.precond == 2) {
    double *ts = (double *)xmalloc((size_t)n * sizeof(double) + 8);
    double *ds = (double *)xmalloc((size_t)n * sizeof(double) + 8);
    for (int32_t c = 0; c < n; c++) ts[c] = t[2 * c + 1];
    or_vcycle(&b->hss, ts, ds);                                            /* Alg. 2 step 5 */
    for (int32_t c = 0; c < n; c++) u[2 * c + 1] = u[2 * c + 1] + ds[c];
    free(ts); free(ds);
  }
  for (int32_t c = 0; c < n; c++) u[2 * c] = u[2 * c] + dp[c];            /* u + R_p^T dp */
  free(t); free(tp); free(dp);
}

void or_bf_apply(const or_bf *b, const double *v, double *z) {
  int32_t n = b->n, ip = b->var_order ? 1 : 0, is = 1 - ip;
  if (b->opt.precond) {
    double *rc = (double *)xmalloc((size_t)2 * n * sizeof(double) + 8);
    double *uc = (double *)xmalloc((size_t)2 * n * sizeof(double) + 8);
    for (int32_t c = 0; c < n; c++) { rc[2 * c] = v[2 * c + ip]; rc[2 * c + 1] = v[2 * c + is]; }
    if (b->opt.precond == 3)
      or_vcycle(&b->hJ, rc, uc);                    /* coupled point AMG: one V-cycle on J */
    else
      cpr_apply(b, rc, uc);
    for (int32_t c = 0; c < n; c++) { z[2 * c + ip] = uc[2 * c]; z[2 * c + is] = uc[2 * c + 1]; }
    free(rc); free(uc);
    return;
  }
  double *rp = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  double *rs = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  double *s = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  double *p = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  double *t = (double *)xmalloc((size_t)n * sizeof(double) + 8);
  for (int32_t c = 0; c < n; c++) { rp[c] = v[2 * c + ip]; rs[c] = v[2 * c + is]; }  /* R_p r, R_s r */
  or_vcycle(&b->hss, rs, s);                        /* step 2: A_ss s = R_s r by one V-cycle */
  or_csr_spmv(&b->Aps, s, t);                       /* step 3: r = R_p r - A_ps s */
  for (int32_t c = 0; c < n; c++) rp[c] = rp[c] - t[c];
  or_vcycle(&b->hS, rp, p);                         /* step 4: S~ p = r by one V-cycle */
  for (int32_t c = 0; c < n; c++) { z[2 * c + ip] = p[c]; z[2 * c + is] = s[c]; }  /* R_p^T p + R_s^T s */
  free(rp); free(rs); free(s); free(p); free(t);
}

/* ------------------------------------------------------------------------ */
/* Right-preconditioned restarted GMRES(m) (P:L138-140 `precon-system`,       */
/* P:L275 tolerance form; readings Q29-Q32; c.2 step 7).                      */
/* ------------------------------------------------------------------------ */
static double dot(int64_t N, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t i = 0; i < N; i++) s += a[i] * b[i];
  return s;
}

/* Test hook (pins of SURVEY c.5 "GMRES"): when set, the next or_gmres call copies the Arnoldi
 * quantities of its FIRST cycle -- the basis V_{k+1} (k+1 vectors of N, vector-major) and the
 * Hessenberg matrix Hbar ((m+1) x m row-major, BEFORE the Givens rotations) -- and the number k
 * of Arnoldi steps of that cycle; then the hook clears itself. */
static double *g_cap_V = NULL, *g_cap_H = NULL;
static int32_t *g_cap_k = NULL;
void or_gmres_capture(double *V, double *Hbar, int32_t *k) {
  g_cap_V = V;
  g_cap_H = Hbar;
  g_cap_k = k;
}

int or_gmres(const or_bf *b, const double *rhs, double *x, double tol, int32_t restart,
             int32_t maxit, int32_t *iters, double *res_hist, int32_t *converged,
             double *final_relres) {
  int64_t N = 2 * (int64_t)b->n;
  int32_t m = restart;
  double *V = (double *)xmalloc((size_t)(m + 1) * N * sizeof(double));
  double *H = (double *)xcalloc((size_t)(m + 1) * m, sizeof(double));   /* H[i*m + j] */
  double *cs = (double *)xmalloc((size_t)m * sizeof(double));
  double *sn = (double *)xmalloc((size_t)m * sizeof(double));
  double *g = (double *)xmalloc((size_t)(m + 1) * sizeof(double));
  double *y = (double *)xmalloc((size_t)m * sizeof(double));
  double *h = (double *)xmalloc((size_t)(m + 1) * sizeof(double));
  double *h2 = (double *)xmalloc((size_t)(m + 1) * sizeof(double));
  double *w = (double *)xmalloc((size_t)N * sizeof(double));
  double *z = (double *)xmalloc((size_t)N * sizeof(double));
  double *r = (double *)xmalloc((size_t)N * sizeof(double));
  double bnorm = sqrt(dot(N, rhs, rhs));
  *iters = 0;
  *converged = 0;
  if (bnorm == 0.0) {                               /* b = 0 -> x = 0 */
    for (int64_t i = 0; i < N; i++) x[i] = 0.0;
    if (res_hist) res_hist[0] = 0.0;
    *converged = 1;
    *final_relres = 0.0;
    goto done;
  }
  or_bf_spmv(b, x, r);
  for (int64_t i = 0; i < N; i++) r[i] = rhs[i] - r[i];
  double beta = sqrt(dot(N, r, r));
  if (res_hist) res_hist[0] = beta / bnorm;
  *final_relres = beta / bnorm;
  if (beta <= tol * bnorm) { *converged = 1; goto done; }
  if (maxit <= 0) goto done;                        /* no Arnoldi step allowed */
  int first_cycle = 1;
  for (;;) {
    for (int64_t i = 0; i < N; i++) V[i] = r[i] / beta;
    for (int32_t i = 0; i <= m; i++) g[i] = 0.0;
    g[0] = beta;
    int32_t k = 0, breakdown = 0;
    for (int32_t j = 0; j < m; j++) {
      or_bf_apply(b, V + (size_t)j * N, z);         /* z = M^-1 v_j */
      or_bf_spmv(b, z, w);                           /* w = J z */
      /* classical Gram-Schmidt, twice (CGS2) */
      for (int32_t i = 0; i <= j; i++) h[i] = dot(N, V + (size_t)i * N, w);
      for (int32_t i = 0; i <= j; i++)
        for (int64_t t = 0; t < N; t++) w[t] -= h[i] * V[(size_t)i * N + t];
      if (b->opt.orth == 0) {
        for (int32_t i = 0; i <= j; i++) h2[i] = dot(N, V + (size_t)i * N, w);
        for (int32_t i = 0; i <= j; i++)
          for (int64_t t = 0; t < N; t++) w[t] -= h2[i] * V[(size_t)i * N + t];
        for (int32_t i = 0; i <= j; i++) h[i] += h2[i];
      }
      double hn = sqrt(dot(N, w, w));
      for (int32_t i = 0; i <= j; i++) H[(size_t)i * m + j] = h[i];
      H[(size_t)(j + 1) * m + j] = hn;
      if (first_cycle && g_cap_H)
        for (int32_t i = 0; i <= j + 1; i++) g_cap_H[(size_t)i * m + j] = H[(size_t)i * m + j];
      if (hn != 0.0)
        for (int64_t t = 0; t < N; t++) V[(size_t)(j + 1) * N + t] = w[t] / hn;
      else
        breakdown = 1;
      for (int32_t i = 0; i < j; i++) {             /* previous Givens rotations */
        double a = H[(size_t)i * m + j], c = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a + sn[i] * c;
        H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
      }
      double a = H[(size_t)j * m + j], c = H[(size_t)(j + 1) * m + j];
      double t = hypot(a, c);
      if (t == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
      else { cs[j] = a / t; sn[j] = c / t; }
      H[(size_t)j * m + j] = cs[j] * a + sn[j] * c;
      H[(size_t)(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      (*iters)++;
      if (res_hist) res_hist[*iters] = fabs(g[j + 1]) / bnorm;
      k = j + 1;
      if (fabs(g[j + 1]) <= tol * bnorm || *iters >= maxit || breakdown) break;
    }
    if (first_cycle && g_cap_k) {
      *g_cap_k = k;
      if (g_cap_V) memcpy(g_cap_V, V, (size_t)(breakdown ? k : k + 1) * N * sizeof(double));
      g_cap_V = NULL; g_cap_H = NULL; g_cap_k = NULL;
    }
    first_cycle = 0;
    /* y = H^-1 g (upper triangular back substitution), x += M^-1 (V y) */
    for (int32_t i = k - 1; i >= 0; i--) {
      double s = g[i];
      for (int32_t jj = i + 1; jj < k; jj++) s -= H[(size_t)i * m + jj] * y[jj];
      y[i] = H[(size_t)i * m + i] != 0.0 ? s / H[(size_t)i * m + i] : 0.0;
    }
    for (int64_t t = 0; t < N; t++) w[t] = 0.0;
    for (int32_t i = 0; i < k; i++)
      for (int64_t t = 0; t < N; t++) w[t] += y[i] * V[(size_t)i * N + t];
    or_bf_apply(b, w, z);
    for (int64_t t = 0; t < N; t++) x[t] += z[t];
    or_bf_spmv(b, x, r);                             /* true residual at restart (Q31) */
    for (int64_t t = 0; t < N; t++) r[t] = rhs[t] - r[t];
    beta = sqrt(dot(N, r, r));
    *final_relres = beta / bnorm;
    if (beta <= tol * bnorm) { *converged = 1; break; }
    if (*iters >= maxit) break;
    if (beta == 0.0) { *converged = 1; break; }
  }
done:
  free(V); free(H); free(cs); free(sn); free(g); free(y); free(h); free(h2);
  free(w); free(z); free(r);
  return 0;
}
