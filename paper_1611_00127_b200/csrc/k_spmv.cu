// k_spmv.cu -- the 2x2-BSR Jacobian SpMV w = J z (operator of `precon-system`,
// P:L138-140; point ordering P:L145-153) and the scalar CSR SpMV family used by the
// V-cycle (restriction/prolongation, residuals) and the A_ps coupling (Alg. 3 step 3).
//
// Roofline: HBM-bound.  Algorithmic bytes of the BSR SpMV per launch:
//   36 nnzb (32 B block values + 4 B column) + 36 n (x, y: 16 B each, row_ptr 4 B).
// Layout: a group of 8 lanes per block row, each lane one 2x2 block loaded as two
// aligned double2 (streaming, evict-first: the matrix is read once per SpMV and must not
// push x out of L2), x gathered as double2 through L1/L2, 3 shuffle steps per row.
#include "bf_internal.cuh"
#include "k_spmv.cuh"

namespace bf {

template <int G>
__global__ void __launch_bounds__(256) k_bsr2_spmv(int n, const int32_t *__restrict__ rp,
                                                   const int32_t *__restrict__ ci,
                                                   const double2 *__restrict__ v,
                                                   const double2 *__restrict__ x, double2 *__restrict__ y, int ip) {
  int gid = (blockIdx.x * blockDim.x + threadIdx.x);
  int r = gid / G;
  int lane = threadIdx.x % G;
  bool ok = r < n;  // no early return: the whole warp takes part in the shuffles
  int a = ok ? __ldg(rp + r) : 0, b = ok ? __ldg(rp + r + 1) : 0;
  double y0 = 0.0, y1 = 0.0;
  for (int q = a + lane; q < b; q += G) {
    int col = __ldcs(ci + q);
    double2 v01 = __ldcs(v + 2 * q);      // (a_pp, a_ps)
    double2 v23 = __ldcs(v + 2 * q + 1);  // (a_sp, a_ss)
    double2 xc = __ldg(x + col);
    double xp = ip ? xc.y : xc.x, xs = ip ? xc.x : xc.y;  // vectors follow the caller's var_order
    y0 += v01.x * xp + v01.y * xs;
    y1 += v23.x * xp + v23.y * xs;
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    y0 += __shfl_xor_sync(0xffffffffu, y0, o, G);
    y1 += __shfl_xor_sync(0xffffffffu, y1, o, G);
  }
  if (ok && lane == 0) y[r] = ip ? make_double2(y1, y0) : make_double2(y0, y1);
}

void bsr_spmv(bf_ctx *c, const double *x, double *y) {
  constexpr int G = 8;
  int64_t threads = (int64_t)c->n * G;
  k_bsr2_spmv<G><<<div_up(threads, 256), 256, 0, c->stream>>>(
      c->n, c->brp, c->bci, reinterpret_cast<const double2 *>(c->bv), reinterpret_cast<const double2 *>(x),
      reinterpret_cast<double2 *>(y), c->var_order);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

void csr_spmv(bf_ctx *c, const DCsr &A, const double *x, double *y) {
  csr_op<OP_SPMV>(c, A, x, nullptr, nullptr, y, nullptr, 1.0, 0.0, nullptr);
}

}  // namespace bf
