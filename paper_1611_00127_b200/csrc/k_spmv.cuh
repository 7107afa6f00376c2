// k_spmv.cuh -- scalar CSR SpMV family (one templated kernel, G lanes per row,
// G = the power of two nearest the mean row length, 1..32).  Used by the V-cycle
// (smoothers, residual, restriction R r, prolongation x += P e) and the A_ps coupling.
#pragma once
#include "bf_internal.cuh"

namespace bf {

enum CsrMode {
  OP_SPMV = 0,          // y = A x
  OP_RESID = 1,         // y = b - A x
  OP_SMOOTH = 2,        // dn = alpha dir + beta (b - A x) * dinv ; y = x + dn ; aux = dn (if aux)
  OP_SMOOTH0_RESID = 3, // x0 = beta b * dinv ; y = b - A x0 ; aux = x0   (x0 gathered on the fly)
  OP_ADD = 4,           // y = y + A x
  OP_SUB = 5            // y = b - A x written as y = b - (A x) (same as RESID, used for A_ps)
};

template <int MODE, int G>
__global__ void __launch_bounds__(256) k_csr(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                             const double *__restrict__ v, const double *__restrict__ x,
                                             const double *__restrict__ b, const double *__restrict__ dinv,
                                             double *__restrict__ y, double *__restrict__ aux, double alpha,
                                             double beta, const double *__restrict__ dir) {
  int gid = blockIdx.x * blockDim.x + threadIdx.x;
  int r = gid / G;
  int lane = (G == 1) ? 0 : (threadIdx.x % G);
  bool ok = r < n;
  int a = ok ? __ldg(rp + r) : 0, e = ok ? __ldg(rp + r + 1) : 0;
  double s = 0.0;
  for (int q = a + lane; q < e; q += G) {
    int col = __ldcs(ci + q);
    double av = __ldcs(v + q);
    double xv;
    if (MODE == OP_SMOOTH0_RESID) xv = beta * (__ldg(b + col) * __ldg(dinv + col));
    else xv = __ldg(x + col);
    s += av * xv;
  }
  if (G > 1) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
  }
  if (!ok || lane != 0) return;
  if (MODE == OP_SPMV) {
    y[r] = s;
  } else if (MODE == OP_RESID || MODE == OP_SUB) {
    y[r] = b[r] - s;
  } else if (MODE == OP_SMOOTH) {
    double dn = beta * ((b[r] - s) * dinv[r]);
    if (dir) dn += alpha * dir[r];
    y[r] = x[r] + dn;
    if (aux) aux[r] = dn;
  } else if (MODE == OP_SMOOTH0_RESID) {
    y[r] = b[r] - s;
    aux[r] = beta * (b[r] * dinv[r]);
  } else if (MODE == OP_ADD) {
    y[r] += s;
  }
}

inline int lanes_for(const DCsr &A) {
  double avg = A.n ? (double)A.nnz / A.n : 1.0;
  int g = 1;
  while (g < 32 && g < avg * 0.75) g <<= 1;
  return g;
}

template <int MODE>
void csr_op(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
            double *aux, double alpha, double beta, const double *dir) {
  if (A.n == 0) return;
  int G = lanes_for(A);
  int64_t threads = (int64_t)A.n * G;
  int blocks = div_up(threads, 256);
#define BF_CSR_CASE(g)                                                                                   \
  case g:                                                                                                \
    k_csr<MODE, g><<<blocks, 256, 0, c->stream>>>(A.n, A.rp, A.ci, A.v, x, b, dinv, y, aux, alpha, beta, \
                                                  dir);                                                  \
    break;
  switch (G) {
    BF_CSR_CASE(1)
    BF_CSR_CASE(2)
    BF_CSR_CASE(4)
    BF_CSR_CASE(8)
    BF_CSR_CASE(16)
    BF_CSR_CASE(32)
  }
#undef BF_CSR_CASE
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

}  // namespace bf
