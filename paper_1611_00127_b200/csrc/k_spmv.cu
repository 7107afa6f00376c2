// k_spmv.cu -- the 2x2-BSR Jacobian SpMV w = J z (operator of `precon-system`,
// P:L138-140; point ordering P:L145-153) and the scalar CSR SpMV family used by the
// V-cycle (restriction/prolongation, residuals) and the A_ps coupling (Alg. 3 step 3).
//
// Roofline: HBM-bound.  Algorithmic bytes of the BSR SpMV per launch:
//   36 nnzb (32 B block values + 4 B column) + 36 n (x, y: 16 B each, row_ptr 4 B).
// Layout: warp-staged (below); blocks loaded as two aligned double2 with streaming
// (evict-first) loads -- the matrix is read once per SpMV and must not push x out of L2;
// x gathered as double2 through L1/L2.
#include "bf_internal.cuh"
#include "k_spmv.cuh"

namespace bf {

// Warp-staged BSR2 SpMV: each warp owns 32 consecutive block rows; the warp streams
// their contiguous blocks (two double2 + one int per block, streaming loads), forms the
// 2-vector products with the gathered x block into shared memory, then each lane reduces
// its own block row and stores one double2.  (Staging the raw blocks instead and forming
// the products row-owned was measured slower: 32-byte smem rows at a 7-block stride give
// 8-way bank conflicts.)
constexpr int BSR_WARPS = 4;
constexpr int BSR_CAP = 256;

__global__ void __launch_bounds__(BSR_WARPS * 32) k_bsr2_spmv(int n, const int32_t *__restrict__ rp,
                                                              const int32_t *__restrict__ ci,
                                                              const double2 *__restrict__ v,
                                                              const double2 *__restrict__ x,
                                                              double2 *__restrict__ y, int ip) {
  __shared__ double2 sprod[BSR_WARPS][BSR_CAP];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int r0 = (blockIdx.x * BSR_WARPS + warp) * 32;
  if (r0 >= n) return;
  int r = r0 + lane;
  bool ok = r < n;
  int rend = min(r0 + 32, n);
  int s = __ldg(rp + r0), e = __ldg(rp + rend);
  int my_lo = ok ? __ldg(rp + r) : e, my_hi = ok ? __ldg(rp + r + 1) : e;
  double y0 = 0.0, y1 = 0.0;
  double2 *sp = sprod[warp];
  for (int cs = s; cs < e; cs += BSR_CAP) {
    int ce = min(cs + BSR_CAP, e);
#pragma unroll 4
    for (int k = cs + lane; k < ce; k += 32) {
      int col = __ldcs(ci + k);
      double2 v01 = __ldcs(v + 2 * (size_t)k);      // (a_pp, a_ps)
      double2 v23 = __ldcs(v + 2 * (size_t)k + 1);  // (a_sp, a_ss)
      double2 xc = __ldg(x + col);
      double xp = ip ? xc.y : xc.x, xs = ip ? xc.x : xc.y;  // vectors follow the caller's var_order
      sp[k - cs] = make_double2(v01.x * xp + v01.y * xs, v23.x * xp + v23.y * xs);
    }
    __syncwarp();
    int lo = max(my_lo, cs), hi = min(my_hi, ce);
    for (int k = lo; k < hi; k++) {
      double2 t = sp[k - cs];
      y0 += t.x;
      y1 += t.y;
    }
    __syncwarp();
  }
  if (ok) y[r] = ip ? make_double2(y1, y0) : make_double2(y0, y1);
}

void bsr_spmv(bf_ctx *c, const double *x, double *y) {
  k_bsr2_spmv<<<div_up(c->n, 32 * BSR_WARPS), BSR_WARPS * 32, 0, c->stream>>>(
      c->n, c->brp, c->bci, reinterpret_cast<const double2 *>(c->bv), reinterpret_cast<const double2 *>(x),
      reinterpret_cast<double2 *>(y), c->var_order);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

void csr_spmv(bf_ctx *c, const DCsr &A, const double *x, double *y) {
  csr_op<OP_SPMV>(c, A, x, nullptr, nullptr, y, nullptr, 1.0, 0.0, nullptr);
}

}  // namespace bf
