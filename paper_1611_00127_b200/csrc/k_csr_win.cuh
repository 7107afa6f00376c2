// k_csr_win.cuh -- windowed TMA CSR kernels for the renumbered Galerkin levels (A_1, A_2, ...,
// their fused restrictions Rf and the level transfers between renumbered levels).
//
// ncu on the TMA CSR kernels of the Galerkin levels (k_csr_tma.cuh): ~40 % of the DRAM bandwidth
// at ~70 % of the L1 wavefront throughput, the issue slots waiting on the x gathers (a warp-wide
// gather of fp64 values scattered over a coarse grid costs up to 32 L1 wavefronts and an L2 round
// trip).  After the coarse levels are renumbered in Morton order (k_amg_setup.cu
// reorder_levels), a block of a few hundred consecutive rows touches a compact set of columns:
// K consecutive TMA tiles (a "super-tile", K * rpt rows) reference only ~2-3 distinct columns per
// row although they hold ~18-26 nonzeros per row.  So, per super-tile, setup stores
//   wcol[s * wmax + i], i < wn[s] : the sorted distinct columns of the super-tile (the window)
//   lc[q] (uint16)                : the position of ci[q] in that list
// and the kernel gathers the window ONCE from global memory into shared memory (sorted, so the
// gathers coalesce into runs) and then forms the rows from shared memory: a warp-wide gather is
// a few shared-memory wavefronts instead of up to 32 L1 wavefronts, has shared-memory latency,
// and the streamed matrix shrinks from 12 to 10 bytes per nonzero.  The TMA pipeline of the
// matrix stream (tiles of rpt rows, double-buffered bulk copies, fused epilogues, PDL prologue)
// is the one of k_csr_tma.cuh; the sums are formed by the same lanes in the same order, so the
// results are bitwise those of the unwindowed kernel.
//
// Work split: the tiles are dealt to the CTAs of one wave in contiguous ranges; a CTA whose range
// begins or ends inside a super-tile fills that super-tile's window too (a few per cent more
// window traffic, no imbalance).
#pragma once
#include "bf_internal.cuh"
#include "k_csr_tma.cuh"

namespace bf {

constexpr int WIN_MAX = 4096;     // largest window (doubles) a super-tile may need: 32 KB of shared memory
constexpr int WIN_HASH = 16384;   // setup: per-CTA hash table slots (distinct columns <= WIN_MAX)

// local index, range-checked (and clamped) in the checked build
#define BF_LC(idx, cnt) (BF_CHK((int)(idx) < (cnt)) ? (int)(idx) : 0)

__host__ __device__ inline int win_lc_bytes(int cap) { return ((2 * (cap + 16)) + 15) & ~15; }
__host__ __device__ inline int win_stage_bytes(int cap, int rpt) {
  return tma_rp_bytes(rpt) + win_lc_bytes(cap) + (((8 * (cap + 4)) + 15) & ~15);
}

template <int MODE, int G, int ST>
__global__ void __launch_bounds__(TMA_THREADS) k_csr_win(int n, int m, int rpt, int ntiles, int cap, int K, int wmax,
                                                         const int32_t *__restrict__ rp,
                                                         const uint16_t *__restrict__ lc,
                                                         const double *__restrict__ v,
                                                         const int32_t *__restrict__ wn,
                                                         const int32_t *__restrict__ wcol,
                                                         const double *__restrict__ x, const double *__restrict__ b,
                                                         const double *__restrict__ dinv, double *__restrict__ y,
                                                         double *__restrict__ aux, double alpha, double beta,
                                                         const double *__restrict__ dir, int wsm) {
  constexpr int NT = TMA_THREADS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[ST];
  double *win = reinterpret_cast<double *>(smem_raw);  // wsm doubles
  unsigned char *stages = smem_raw + 8 * (size_t)wsm;
  const int stage_bytes = win_stage_bytes(cap, rpt);
  const int rb = tma_rp_bytes(rpt);
  const int cb = rb + win_lc_bytes(cap);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < ST; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int t, int s) {
    int r0 = t * rpt, r1 = min(r0 + rpt, n);
    int q0 = __ldg(rp + r0), q1 = __ldg(rp + r1);
    int c0 = q0 & ~7, c1 = (q1 + 7) & ~7;  // 16-B aligned uint16 range
    int v0 = q0 & ~1, v1 = (q1 + 1) & ~1;  // 16-B aligned double range
    unsigned char *base = stages + s * stage_bytes;
    uint32_t br = 4u * ((r1 - r0 + 1 + 3) & ~3);
    uint32_t bc = 2u * (c1 - c0), bv = 8u * (v1 - v0);
    if (!BF_CHK(br <= (uint32_t)rb && rb + bc <= (uint32_t)cb && cb + bv <= (uint32_t)stage_bytes)) bc = bv = 0;
    mbar_expect_tx(&bars[s], br + bc + bv);
    tma_bulk_g2s(base, rp + r0, br, &bars[s], pol);
    if (bc) tma_bulk_g2s(base + rb, lc + c0, bc, &bars[s], pol);
    if (bv) tma_bulk_g2s(base + cb, v + v0, bv, &bars[s], pol);
  };

  // this CTA's contiguous tile range
  const int t_begin = (int)(((int64_t)blockIdx.x * ntiles) / gridDim.x);
  const int t_end = (int)(((int64_t)(blockIdx.x + 1) * ntiles) / gridDim.x);
  if (t_begin >= t_end) {
    pdl_wait();
    return;
  }
  if (tid == 0)
    for (int s = 0; s < ST && t_begin + s < t_end; s++) issue(t_begin + s, s);
  pdl_wait();  // x, b, dinv, dir and the outputs are touched only after this
  const int sub = tid % G;
  int cur = -1, cnt = 0;
  for (int t = t_begin, it = 0; t < t_end; t++, it++) {
    const int sp = t / K;
    if (sp != cur) {  // new super-tile: gather its window (every thread is past the previous tile's rows)
      cur = sp;
      cnt = min(__ldg(wn + sp), wsm);
      const int32_t *wc = wcol + (size_t)sp * wmax;
#pragma unroll 4
      for (int i = tid; i < cnt; i += NT) win[i] = __ldg(x + BF_COL(__ldg(wc + i), m));
      __syncthreads();
    }
    const int s = it % ST;
    const int r0 = t * rpt;
    mbar_wait(&bars[s], (it / ST) & 1);
    const unsigned char *base = stages + s * stage_bytes;
    const int32_t *srp = reinterpret_cast<const int32_t *>(base);
    const int q0 = srp[0];
    const uint16_t *sc = reinterpret_cast<const uint16_t *>(base + rb) - (q0 & ~7);
    const double *sv = reinterpret_cast<const double *>(base + cb) - (q0 & ~1);
    for (int row_in_tile = tid / G; row_in_tile < ((rpt + (NT / G) - 1) / (NT / G)) * (NT / G);
         row_in_tile += NT / G) {
      const int r = r0 + row_in_tile;
      const bool ok = row_in_tile < rpt && r < n;
      const int lo = ok ? srp[row_in_tile] : 0, hi = ok ? srp[row_in_tile + 1] : 0;
      const bool own = ok && sub == 0;
      double eb = 0.0, ed = 0.0, ex = 0.0, edir = 0.0;
      if (own) {
        if (MODE == OP_RESID || MODE == OP_SUB_X0 || MODE == OP_SMOOTH) eb = __ldg(b + r);
        if (MODE == OP_SUB_X0 || MODE == OP_SMOOTH || MODE == OP_SPMV_X0) ed = __ldg(dinv + r);
        if (MODE == OP_SMOOTH) ex = __ldg(x + r);
        if (MODE == OP_SMOOTH && dir) edir = dir[r];
        if (MODE == OP_ADD) ex = y[r];
      }
      double acc = 0.0;
#pragma unroll 4
      for (int q = lo + sub; q < hi; q += G) acc += sv[q] * win[BF_LC(sc[q], cnt)];
      if (G > 1) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
      }
      if (!own) continue;
      if (MODE == OP_SPMV) {
        y[r] = acc;
      } else if (MODE == OP_SPMV_X0) {
        y[r] = acc;
        aux[r] = beta * (acc * ed);
      } else if (MODE == OP_RESID) {
        y[r] = eb - acc;
      } else if (MODE == OP_SUB_X0) {
        double tt = eb - acc;
        y[r] = tt;
        aux[r] = beta * (tt * ed);
      } else if (MODE == OP_SMOOTH) {
        double dn = beta * ((eb - acc) * ed);
        if (dir) dn += alpha * edir;
        y[r] = ex + dn;
        if (aux) aux[r] = dn;
      } else if (MODE == OP_ADD) {
        y[r] = ex + acc;
      }
    }
    __syncthreads();  // every thread is done with stage s (and, at a super-tile's end, with the window)
    if (tid == 0 && t + ST < t_end) issue(t + ST, s);
  }
  pdl_launch_dependents();
}

template <int MODE, int G>
void launch_csr_win(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                    double *aux, double alpha, double beta, const double *dir) {
  constexpr int ST = TMA_STAGES;
  ensure_smem_attr((const void *)k_csr_win<MODE, G, ST>, 200 * 1024);
  const int wsm = (A.wmax_used + 1) & ~1;
  int smem = 8 * wsm + ST * win_stage_bytes(A.cap, A.rpt);
  int ntiles = (A.n + A.rpt - 1) / A.rpt;
  int per_sm = std::max(1, std::min(c->tune.tma_ctas, (220 * 1024) / (smem + 1024)));
  int grid = std::min(ntiles, c->num_sms * per_sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TMA_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = c->use_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, k_csr_win<MODE, G, ST>, A.n, A.m, A.rpt, ntiles, A.cap, A.wk, (int)WIN_MAX,
                             (const int32_t *)A.rp, (const uint16_t *)A.lc, (const double *)A.v,
                             (const int32_t *)A.wn, (const int32_t *)A.wcol, x, b, dinv, y, aux, alpha, beta, dir,
                             wsm));
}

template <int MODE>
bool csr_op_win(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                double *aux, double alpha, double beta, const double *dir) {
  if (!A.lc || A.cap <= 0) return false;
  switch (A.g) {
    case 1: launch_csr_win<MODE, 1>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 2: launch_csr_win<MODE, 2>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 4: launch_csr_win<MODE, 4>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 8: launch_csr_win<MODE, 8>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 16: launch_csr_win<MODE, 16>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 32: launch_csr_win<MODE, 32>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    default: return false;
  }
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  return true;
}

}  // namespace bf
