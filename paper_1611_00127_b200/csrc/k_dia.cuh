// k_dia.cuh -- diagonal (DIA) storage of the finest-level operators A_ss, S~ and A_ps.
//
// These three matrices live on the structured grid: every nonzero sits at a column offset
// col - row drawn from a few stencil offsets (C3: A_ss 7, S~ 12, A_ps 2 distinct offsets,
// > 95 % filled).  Stored as K dense diagonals vals[d][row] (zeros where a row lacks the
// offset or the neighbour is outside the grid) they need no column indices: 8 K bytes per row
// instead of 12 nnz/n (A_ss: 56 vs 82 B/row), and both the values and x[row + off_d] are read
// fully coalesced by one thread per row.  Used when fill = nnz / (K n) >= 0.75.
#pragma once
#include "bf_internal.cuh"
#include "k_spmv.cuh"

namespace bf {

constexpr int DIA_MAXK = 32;

struct DiaOffsets {
  int k;
  int off[DIA_MAXK];
};

template <int MODE>
__global__ void __launch_bounds__(256) k_dia(int n, DiaOffsets o, const double *__restrict__ dv,
                                             const double *__restrict__ x, const double *__restrict__ b,
                                             const double *__restrict__ dinv, double *__restrict__ y,
                                             double *__restrict__ aux, double alpha, double beta,
                                             const double *__restrict__ dir) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  // the epilogue's row operands first: their loads overlap the diagonal loads
  double eb = 0.0, ed = 0.0, ex = 0.0, edir = 0.0;
  if (MODE == OP_RESID || MODE == OP_SUB_X0 || MODE == OP_SMOOTH) eb = __ldg(b + r);
  if (MODE == OP_SUB_X0 || MODE == OP_SMOOTH || MODE == OP_SPMV_X0) ed = __ldg(dinv + r);
  if (MODE == OP_SMOOTH) ex = __ldg(x + r);
  if (MODE == OP_SMOOTH && dir) edir = dir[r];
  if (MODE == OP_ADD) ex = y[r];
  double acc = 0.0;
#pragma unroll 4
  for (int d = 0; d < o.k; d++) {
    int col = r + o.off[d];
    double a = __ldcs(dv + (size_t)d * n + r);
    if (col >= 0 && col < n) acc += a * __ldg(x + col);
  }
  if (MODE == OP_SPMV) {
    y[r] = acc;
  } else if (MODE == OP_SPMV_X0) {
    y[r] = acc;
    aux[r] = beta * (acc * ed);
  } else if (MODE == OP_RESID) {
    y[r] = eb - acc;
  } else if (MODE == OP_SUB_X0) {
    double t = eb - acc;
    y[r] = t;
    aux[r] = beta * (t * ed);
  } else if (MODE == OP_SMOOTH) {
    double dn = beta * ((eb - acc) * ed);
    if (dir) dn += alpha * edir;
    y[r] = ex + dn;
    if (aux) aux[r] = dn;
  } else if (MODE == OP_ADD) {
    y[r] = ex + acc;
  }
}

template <int MODE>
bool csr_op_dia(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                double *aux, double alpha, double beta, const double *dir) {
  if (!A.dia_v || A.n != A.m) return false;
  DiaOffsets o;
  o.k = A.dia_k;
  for (int d = 0; d < A.dia_k; d++) o.off[d] = A.dia_off[d];
  k_dia<MODE><<<div_up(A.n, 256), 256, 0, c->stream>>>(A.n, o, A.dia_v, x, b, dinv, y, aux, alpha, beta, dir);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  return true;
}

// ---- setup ---------------------------------------------------------------------------
// candidate offsets: a + b nx + c nx ny, a, b, c in [-2, 2] (the stencils of A_ss, S~, A_ps)
static __global__ void k_dia_mark(DCsr A, const int *__restrict__ cand, int ncand, int *present, int *miss) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    int off = A.ci[q] - i, lo = 0, hi = ncand;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (cand[mid] < off) lo = mid + 1;
      else hi = mid;
    }
    if (lo < ncand && cand[lo] == off) present[lo] = 1;
    else *miss = 1;
  }
}

static __global__ void k_dia_fill(DCsr A, DiaOffsets o, double *dv) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  for (int d = 0; d < o.k; d++) dv[(size_t)d * A.n + i] = 0.0;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    int off = A.ci[q] - i;
    for (int d = 0; d < o.k; d++)
      if (o.off[d] == off) {
        dv[(size_t)d * A.n + i] = A.v[q];
        break;
      }
  }
}

}  // namespace bf
