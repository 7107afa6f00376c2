// k_spmv.cu -- the 2x2-BSR Jacobian SpMV w = J z (operator of `precon-system`,
// P:L138-140; point ordering P:L145-153) and the scalar CSR SpMV family used by the
// V-cycle (restriction/prolongation, residuals) and the A_ps coupling (Alg. 3 step 3).
//
// Roofline: HBM-bound.  Algorithmic bytes of the BSR SpMV per launch:
//   36 nnzb (32 B block values + 4 B column) + 36 n (x, y: 16 B each, row_ptr 4 B).
// Layout: warp-staged (below); blocks loaded as two aligned double2 with streaming
// (evict-first) loads -- the matrix is read once per SpMV and must not push x out of L2;
// x gathered as double2 through L1/L2.
#include <cstdlib>

#include "bf_internal.cuh"
BF_CHECK_TU("k_spmv.cu")
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
      int col = BF_COL(__ldcs(ci + k), n);
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

// DIA form of J (the 2x2 blocks of a 7-point grid Jacobian sit on 7 block diagonals):
// jd[d][row] = {(a_pp, a_ps), (a_sp, a_ss)} (zeros where the neighbour is absent), one thread
// per block row, all loads coalesced, no column indices (32 B per block instead of 36 B)
struct BsrDia {
  int k;
  int off[27];
};

__global__ void __launch_bounds__(256) k_bsr2_dia(int n, BsrDia o, const double2 *__restrict__ jd,
                                                  const double2 *__restrict__ x, double2 *__restrict__ y, int ip) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  // J's diagonals are setup data: loaded before waiting for the kernel that produced x (PDL)
  double2 v[14];
#pragma unroll
  for (int d = 0; d < 7; d++) {
    if (d < o.k && r < n) {
      size_t e = ((size_t)d * n + r) * 2;
      v[2 * d] = __ldcs(jd + e);
      v[2 * d + 1] = __ldcs(jd + e + 1);
    }
  }
  pdl_wait();
  if (r >= n) return;
  double y0 = 0.0, y1 = 0.0;
#pragma unroll
  for (int d = 0; d < 7; d++) {
    int col = r + o.off[d];
    if (d < o.k && col >= 0 && col < n) {
      double2 xc = __ldg(x + col);
      double xp = ip ? xc.y : xc.x, xs = ip ? xc.x : xc.y;
      y0 += v[2 * d].x * xp + v[2 * d].y * xs;
      y1 += v[2 * d + 1].x * xp + v[2 * d + 1].y * xs;
    }
  }
  y[r] = ip ? make_double2(y1, y0) : make_double2(y0, y1);
}

__global__ void k_bsr2_dia_fill(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                const double2 *__restrict__ bv, BsrDia o, double2 *jd, int *miss) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int d = 0; d < o.k; d++) {
    size_t e = ((size_t)d * n + r) * 2;
    jd[e] = make_double2(0.0, 0.0);
    jd[e + 1] = make_double2(0.0, 0.0);
  }
  for (int q = rp[r]; q < rp[r + 1]; q++) {
    int off = ci[q] - r, d = 0;
    while (d < o.k && o.off[d] != off) d++;
    if (d == o.k) {
      *miss = 1;
      continue;
    }
    size_t e = ((size_t)d * n + r) * 2;
    jd[e] = bv[2 * (size_t)q];
    jd[e + 1] = bv[2 * (size_t)q + 1];
  }
}

// build (or refresh after bf_update) the DIA copy of J when its blocks sit on the 7-point
// stencil of the grid and fill >= 0.75
void setup_bsr_dia(bf_ctx *c) {
  dfree(c, c->jdia);
  c->jdia = nullptr;
  if (!c->tune.dia || c->nx <= 0) return;
  int64_t sx = 1, sy = c->nx, sz = (int64_t)c->nx * c->ny;
  BsrDia o;
  o.k = 0;
  const int64_t cand[7] = {-sz, -sy, -sx, 0, sx, sy, sz};
  for (int d = 0; d < 7; d++) {
    if (cand[d] != 0 && (cand[d] <= -(int64_t)c->n || cand[d] >= c->n)) continue;
    bool dup = false;
    for (int e = 0; e < o.k; e++) dup |= o.off[e] == (int)cand[d];
    if (!dup) o.off[o.k++] = (int)cand[d];
  }
  if ((double)c->nnzb / ((double)o.k * c->n) < 0.75) return;
  double *jd = dalloc_t<double>(c, (size_t)o.k * c->n * 4);
  int *miss = dalloc_t<int>(c, 1);
  BF_CUDA(cudaMemsetAsync(miss, 0, sizeof(int), c->stream));
  k_bsr2_dia_fill<<<div_up(c->n, 256), 256, 0, c->stream>>>(c->n, c->brp, c->bci,
                                                            reinterpret_cast<const double2 *>(c->bv), o,
                                                            reinterpret_cast<double2 *>(jd), miss);
  BF_LAUNCH(c);
  int hm = 0;
  BF_CUDA(cudaMemcpyAsync(&hm, miss, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, miss);
  if (hm) {  // a block off the 7-point stencil: keep the CSR-BSR kernel
    dfree(c, jd);
    return;
  }
  c->jdia = jd;
  c->jdia_k = o.k;
  for (int d = 0; d < o.k; d++) c->jdia_off[d] = o.off[d];
}

void bsr_spmv(bf_ctx *c, const double *x, double *y) {
  if (c->jdia) {
    BsrDia o;
    o.k = c->jdia_k;
    for (int d = 0; d < o.k; d++) o.off[d] = c->jdia_off[d];
    launch_pdl(c, k_bsr2_dia, dim3(div_up(c->n, 256)), dim3(256), 0, c->n, o,
               reinterpret_cast<const double2 *>(c->jdia), reinterpret_cast<const double2 *>(x),
               reinterpret_cast<double2 *>(y), c->var_order);
    BF_LAUNCH(c);
    BF_CUDA(cudaGetLastError());
    return;
  }
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
