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
  OP_SPMV_X0 = 3,       // y = A x ; aux = beta y * dinv  (restriction that also seeds the next level's x0)
  OP_ADD = 4,           // y = y + A x
  OP_SUB_X0 = 5         // y = b - A x ; aux = beta y * dinv  (A_ps coupling that seeds the S~ level-0 x0)
};

// Warp-staged CSR kernel: each warp owns R = 32/G consecutive rows (G lanes per row).
// The warp streams the contiguous nonzero range of its rows in chunks of CSR_CAP entries
// into shared memory (coalesced streaming loads of col/val), then the G lanes of each row
// form a_ij x_j with row-owned gathers of x (consecutive rows -> consecutive addresses for
// stencil-like rows, few L1 wavefronts) and combine with shuffles.  G = 1 for the short fine-level rows (thread-per-row epilogue), larger G for
// the long Galerkin rows of the coarse levels (and for small levels, so that enough
// warps exist to fill the 148 SMs).  No padding, full coalescing, any row length.
constexpr int CSR_WARPS = 8;
constexpr int CSR_CAP = 256;

template <int MODE, int G>
__global__ void __launch_bounds__(CSR_WARPS * 32) k_csr(int n, int m, const int32_t *__restrict__ rp,
                                                        const int32_t *__restrict__ ci,
                                                        const double *__restrict__ v, const double *__restrict__ x,
                                                        const double *__restrict__ b,
                                                        const double *__restrict__ dinv, double *__restrict__ y,
                                                        double *__restrict__ aux, double alpha, double beta,
                                                        const double *__restrict__ dir) {
  constexpr int R = 32 / G;
  __shared__ double sval[CSR_WARPS][CSR_CAP];
  __shared__ int32_t scol[CSR_WARPS][CSR_CAP];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int r0 = (blockIdx.x * CSR_WARPS + warp) * R;
  if (r0 >= n) return;  // whole warp
  int r = r0 + lane / G;
  int sub = lane % G;
  bool ok = r < n;
  int rend = min(r0 + R, n);
  int s = __ldg(rp + r0), e = __ldg(rp + rend);
  int my_lo = ok ? __ldg(rp + r) : e, my_hi = ok ? __ldg(rp + r + 1) : e;
  double acc = 0.0;
  double *sv = sval[warp];
  int32_t *sc = scol[warp];
  for (int cs = s; cs < e; cs += CSR_CAP) {
    int ce = min(cs + CSR_CAP, e);
    // stage the warp's contiguous (col, val) range: fully coalesced streaming loads
#pragma unroll 4
    for (int k = cs + lane; k < ce; k += 32) {
      sc[k - cs] = __ldcs(ci + k);
      sv[k - cs] = __ldcs(v + k);
    }
    __syncwarp();
    // row-owned products: for stencil-like rows the gathers of consecutive rows are
    // consecutive addresses (one or two wavefronts per warp instruction)
    int lo = max(my_lo, cs), hi = min(my_hi, ce);
#pragma unroll 4
    for (int k = lo + sub; k < hi; k += G) {
      int col = BF_COL(sc[k - cs], m);
      acc += sv[k - cs] * __ldg(x + col);
    }
    __syncwarp();
  }
  if (G > 1) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
  }
  if (!ok || sub != 0) return;
  double sacc = acc;
  if (MODE == OP_SPMV) {
    y[r] = sacc;
  } else if (MODE == OP_SPMV_X0) {
    y[r] = sacc;
    aux[r] = beta * (sacc * dinv[r]);
  } else if (MODE == OP_RESID) {
    y[r] = b[r] - sacc;
  } else if (MODE == OP_SUB_X0) {
    double t = b[r] - sacc;
    y[r] = t;
    aux[r] = beta * (t * dinv[r]);
  } else if (MODE == OP_SMOOTH) {
    double dn = beta * ((b[r] - sacc) * dinv[r]);
    if (dir) dn += alpha * dir[r];
    y[r] = x[r] + dn;
    if (aux) aux[r] = dn;
  } else if (MODE == OP_ADD) {
    y[r] += sacc;
  }
}

// Short-row CSR kernel (interpolation P and restriction R of the large levels: 1-8 entries per
// row): one thread per row, no staging.  The row's (col, val) entries -- setup data -- are
// loaded into registers BEFORE griddepcontrol.wait (programmatic dependent launch), so only
// the gathers of x and the epilogue wait for the kernel that produced x; consecutive threads'
// entries are contiguous, so the streaming loads of a warp coalesce.
// SHORT_K register slots per row: 4 for the interpolation-like matrices (mean row length <= 3:
// fewer registers, 8 CTAs per SM), 8 otherwise; longer rows finish in a scalar loop.
template <int MODE, int SHORT_K>
__global__ void __launch_bounds__(256, SHORT_K == 4 ? 8 : 6) k_csr_short(int n, int m, const int32_t *__restrict__ rp,
                                                   const int32_t *__restrict__ ci,
                                                   const double *__restrict__ v, const double *__restrict__ x,
                                                   const double *__restrict__ b, const double *__restrict__ dinv,
                                                   double *__restrict__ y, double *__restrict__ aux, double alpha,
                                                   double beta, const double *__restrict__ dir) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  int lo = 0, hi = 0;
  int col[SHORT_K];
  double val[SHORT_K];
  if (r < n) {
    lo = __ldg(rp + r);
    hi = __ldg(rp + r + 1);
#pragma unroll
    for (int e = 0; e < SHORT_K; e++)
      if (lo + e < hi) {
        col[e] = __ldcs(ci + lo + e);
        val[e] = __ldcs(v + lo + e);
      }
  }
  pdl_wait();
  if (r >= n) return;
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < SHORT_K; e++)
    if (lo + e < hi) acc += val[e] * __ldg(x + BF_COL(col[e], m));
  for (int q = lo + SHORT_K; q < hi; q++) acc += __ldcs(v + q) * __ldg(x + BF_COL(__ldcs(ci + q), m));
  if (MODE == OP_SPMV) {
    y[r] = acc;
  } else if (MODE == OP_SPMV_X0) {
    y[r] = acc;
    aux[r] = beta * (acc * dinv[r]);
  } else if (MODE == OP_RESID) {
    y[r] = b[r] - acc;
  } else if (MODE == OP_SUB_X0) {
    double t = b[r] - acc;
    y[r] = t;
    aux[r] = beta * (t * dinv[r]);
  } else if (MODE == OP_SMOOTH) {
    double dn = beta * ((b[r] - acc) * dinv[r]);
    if (dir) dn += alpha * dir[r];
    y[r] = x[r] + dn;
    if (aux) aux[r] = dn;
  } else if (MODE == OP_ADD) {
    y[r] += acc;
  }
}

// lanes per row: keep R * (mean row length) near one chunk, and keep >= ~4 warps per SM
inline int lanes_for(const bf_ctx *c, const DCsr &A) {
  double avg = A.n ? (double)A.nnz / A.n : 1.0;
  int G = 1;
  while (G < 32 && (32 / G) * avg > CSR_CAP) G <<= 1;
  while (G < 32 && (double)A.n * G / 32.0 < 4.0 * c->num_sms) G <<= 1;
  return G;
}

template <int MODE>
bool csr_op_tma(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                double *aux, double alpha, double beta, const double *dir);
template <int MODE>
bool csr_op_dia(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                double *aux, double alpha, double beta, const double *dir);
template <int MODE>
bool csr_op_win(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                double *aux, double alpha, double beta, const double *dir);

// algorithmic bytes of one csr_op (each operand once: int32 index, f64 value; x counted once
// per column); accumulated into c->alg_bytes so a captured BF apply knows its own traffic
template <int MODE>
double csr_op_bytes(const DCsr &A, bool has_dir, bool has_aux) {
  double n = A.n, base = 12.0 * A.nnz + 4.0 * (A.n + 1) + 8.0 * A.m;
  switch (MODE) {
    case OP_SPMV: return base + 8 * n;
    case OP_SPMV_X0: return base + 24 * n;
    case OP_RESID: return base + 16 * n;
    case OP_SUB_X0: return base + 32 * n;
    case OP_SMOOTH: return base + 24 * n + (has_dir ? 8 * n : 0) + (has_aux ? 8 * n : 0);
    case OP_ADD: return base + 16 * n;
  }
  return base;
}

template <int MODE>
void csr_op(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
            double *aux, double alpha, double beta, const double *dir) {
  if (A.n == 0) return;
  c->alg_bytes += csr_op_bytes<MODE>(A, dir != nullptr, aux != nullptr);
  if (csr_op_dia<MODE>(c, A, x, b, dinv, y, aux, alpha, beta, dir)) return;
  if (A.ws && csr_op_win<MODE>(c, A, x, b, dinv, y, aux, alpha, beta, dir)) return;
  if (A.short_rows) {
    if ((double)A.nnz <= c->tune.short_k4 * (double)A.n)
      launch_pdl(c, k_csr_short<MODE, 4>, dim3(div_up(A.n, 256)), dim3(256), 0, A.n, A.m, A.rp, A.ci, A.v, x, b, dinv, y,
                 aux, alpha, beta, dir);
    else
      launch_pdl(c, k_csr_short<MODE, 8>, dim3(div_up(A.n, 256)), dim3(256), 0, A.n, A.m, A.rp, A.ci, A.v, x, b, dinv, y,
                 aux, alpha, beta, dir);
    BF_LAUNCH(c);
    BF_CUDA(cudaGetLastError());
    return;
  }
  if (c->use_tma && A.nnz >= c->tune.tma_min_nnz && csr_op_tma<MODE>(c, A, x, b, dinv, y, aux, alpha, beta, dir))
    return;
  int G = lanes_for(c, A);
  int rows_per_block = (32 / G) * CSR_WARPS;
  int blocks = div_up(A.n, rows_per_block);
#define BF_CSR_CASE(g)                                                                                  \
  case g:                                                                                               \
    k_csr<MODE, g><<<blocks, CSR_WARPS * 32, 0, c->stream>>>(A.n, A.m, A.rp, A.ci, A.v, x, b, dinv, y, aux, alpha, \
                                                             beta, dir);                                \
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

#include "k_csr_tma.cuh"
#include "k_csr_win.cuh"
#include "k_dia.cuh"
