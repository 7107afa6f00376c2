// k_csr_tma.cuh -- TMA-pipelined CSR kernel family for the V-cycle and the A_ps coupling.
//
// The matrix is cut into tiles of RPT consecutive rows (RPT per matrix, chosen at setup so
// that a tile holds at most `cap` nonzeros).  A tile's (col, val) range is contiguous in
// HBM, so one elected thread moves it into shared memory with two 1-D bulk copies
// (cp.async.bulk ... mbarrier::complete_tx, the TMA engine), double-buffered: while the CTA
// computes tile i from stage i%2, the copy of tile i+grid is already in flight.  The CTA's
// 256 threads then form the rows with G = 256/RPT lanes per row, gathering x through L1/L2,
// and apply the fused epilogue (residual / smoother / restriction + seeding / prolongation).
// Persistent grid: one wave of CTAs loops over the tiles.
#pragma once
#include "bf_internal.cuh"
#include "k_spmv.cuh"

#include <algorithm>
#include <cstdlib>

namespace bf {

constexpr int TMA_THREADS = 256;
constexpr int TMA_STAGES = 2;      // TMA pipeline depth (and the tiling heuristic's smem budget)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// L2 policy for the streamed matrix: evict-first, so that one pass over a 100+ MB operator
// does not push the (gathered, reused) vectors out of the 126 MB L2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// programmatic dependent launch (PDL): wait for the preceding kernel's memory / allow the next
// kernel to begin launching.  No-ops when the kernel was launched without the PDL attribute.


__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// byte layout of one stage: [row_ptr: 4*(rpt+8) B][cols: 4*(cap+8) B][vals: 8*(cap+4) B], all
// 16-B aligned (the aligned copy of a tile of `cap` nonzeros spans at most cap+6 ints /
// cap+2 doubles; the tile's row_ptr segment rpt+1 ints, rounded up to 4).  Staging row_ptr
// too removes the dependent global load of rp[r], rp[r+1] before each row's gathers.
__host__ __device__ inline int tma_rp_bytes(int rpt) { return ((4 * (rpt + 8)) + 15) & ~15; }
__host__ __device__ inline int tma_col_bytes(int cap) { return ((4 * (cap + 8)) + 15) & ~15; }
__host__ __device__ inline int tma_stage_bytes(int cap, int rpt) {
  return tma_rp_bytes(rpt) + tma_col_bytes(cap) + (((8 * (cap + 4)) + 15) & ~15);
}

template <int MODE, int G, int ST, int NT>
__global__ void __launch_bounds__(NT) k_csr_tma(int n, int m, int rpt, int ntiles, int cap,
                                                         const int32_t *__restrict__ rp,
                                                         const int32_t *__restrict__ ci,
                                                         const double *__restrict__ v, const double *__restrict__ x,
                                                         const double *__restrict__ b,
                                                         const double *__restrict__ dinv, double *__restrict__ y,
                                                         double *__restrict__ aux, double alpha, double beta,
                                                         const double *__restrict__ dir) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[ST];
  const int stage_bytes = tma_stage_bytes(cap, rpt);
  const int rb = tma_rp_bytes(rpt);
  const int cb = rb + tma_col_bytes(cap);
  int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < ST; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // producer: issue the bulk copies of tile t into stage s
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int t, int s) {
    int r0 = t * rpt, r1 = min(r0 + rpt, n);
    int q0 = __ldg(rp + r0), q1 = __ldg(rp + r1);
    int c0 = q0 & ~3, c1 = (q1 + 3) & ~3;  // 16-B aligned int32 range
    int v0 = q0 & ~1, v1 = (q1 + 1) & ~1;  // 16-B aligned double range
    unsigned char *base = smem_raw + s * stage_bytes;
    uint32_t br = 4u * ((r1 - r0 + 1 + 3) & ~3);  // r0 is a multiple of 4 (rpt is)
    uint32_t bc = 4u * (c1 - c0), bv = 8u * (v1 - v0);
    if (!BF_CHK(br <= (uint32_t)rb && rb + bc <= (uint32_t)cb && cb + bv <= (uint32_t)stage_bytes)) bc = bv = 0;
    mbar_expect_tx(&bars[s], br + bc + bv);
    tma_bulk_g2s(base, rp + r0, br, &bars[s], pol);
    if (bc) tma_bulk_g2s(base + rb, ci + c0, bc, &bars[s], pol);
    if (bv) tma_bulk_g2s(base + cb, v + v0, bv, &bars[s], pol);
  };

  // tiles of this CTA: every gridDim.x-th tile (contiguous tile ranges per CTA, for L1 reuse of
  // the x window, measured 1.3 % slower on C3)
  int t = blockIdx.x;
  const int t_end = ntiles, stride = gridDim.x;
  if (t >= t_end) {
    pdl_wait();
    return;
  }
  // the matrix is setup data: its first tiles are fetched BEFORE waiting for the previous
  // kernel of the V-cycle (programmatic dependent launch), overlapping that kernel's tail
  if (tid == 0)
    for (int s = 0; s < ST && t + s * stride < t_end; s++) issue(t + s * stride, s);
  pdl_wait();  // x, b, dinv, dir and the outputs are touched only after this
  const int sub = tid % G;
  for (int it = 0; t < t_end; t += stride, it++) {
    int s = it % ST;
    int r0 = t * rpt;
    mbar_wait(&bars[s], (it / ST) & 1);
    const unsigned char *base = smem_raw + s * stage_bytes;
    const int32_t *srp = reinterpret_cast<const int32_t *>(base);
    int q0 = srp[0];
    const int32_t *sc = reinterpret_cast<const int32_t *>(base + rb) - (q0 & ~3);
    const double *sv = reinterpret_cast<const double *>(base + cb) - (q0 & ~1);
    // rows of the tile in passes of NT/G rows; G lanes per row
    for (int row_in_tile = tid / G; row_in_tile < ((rpt + (NT / G) - 1) / (NT / G)) * (NT / G);
         row_in_tile += NT / G) {
      int r = r0 + row_in_tile;
      bool ok = row_in_tile < rpt && r < n;
      int lo = ok ? srp[row_in_tile] : 0, hi = ok ? srp[row_in_tile + 1] : 0;
      // the epilogue's row operands are loaded before the gathers, so that their latency
      // overlaps the gather latency instead of following it
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
      if (G >= 4) {  // Galerkin rows: all of a lane's gathers (<= 8) issued before the first FMA
        double xv[8], av[8];
#pragma unroll
        for (int e = 0; e < 8; e++) {
          int q = lo + sub + e * G;
          xv[e] = q < hi ? __ldg(x + BF_COL(sc[q], m)) : 0.0;
          av[e] = q < hi ? sv[q] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 8; e++)
          if (lo + sub + e * G < hi) acc += av[e] * xv[e];
        for (int q = lo + sub + 8 * G; q < hi; q += G) acc += sv[q] * __ldg(x + BF_COL(sc[q], m));
      } else {
#pragma unroll 4
        for (int q = lo + sub; q < hi; q += G) acc += sv[q] * __ldg(x + BF_COL(sc[q], m));
      }
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
    __syncthreads();  // every thread is done with stage s
    if (tid == 0 && t + ST * stride < t_end) issue(t + ST * stride, s);
  }
  pdl_launch_dependents();  // this CTA is done: the next kernel may start its prologue
}

// per-tile nonzero count -> max (setup helper)
static __global__ void k_tile_max(int n, int rpt, const int32_t *__restrict__ rp, int *mx) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  int r0 = t * rpt;
  if (r0 >= n) return;
  int r1 = min(r0 + rpt, n);
  atomicMax(mx, rp[r1] - rp[r0]);
}

template <int MODE, int G, int ST, int NT>
void launch_csr_tma_st(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                       double *aux, double alpha, double beta, const double *dir) {
  ensure_smem_attr((const void *)k_csr_tma<MODE, G, ST, NT>, 200 * 1024);
  int smem = ST * tma_stage_bytes(A.cap, A.rpt);
  int ntiles = (A.n + A.rpt - 1) / A.rpt;
  int per_sm = std::max(1, std::min(c->tune.tma_ctas * (TMA_THREADS / NT), (220 * 1024) / (smem + 1024)));
  int grid = std::min(ntiles, c->num_sms * per_sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = c->use_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, k_csr_tma<MODE, G, ST, NT>, A.n, A.m, A.rpt, ntiles, A.cap, (const int32_t *)A.rp,
                             (const int32_t *)A.ci, (const double *)A.v, x, b, dinv, y, aux, alpha, beta, dir));
}

// two stages and 256-thread CTAs (3-4 stages and 128-thread CTAs for long rows were measured
// slower on C3)
template <int MODE, int G>
void launch_csr_tma(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                    double *aux, double alpha, double beta, const double *dir) {
  launch_csr_tma_st<MODE, G, TMA_STAGES, TMA_THREADS>(c, A, x, b, dinv, y, aux, alpha, beta, dir);
}

template <int MODE>
bool csr_op_tma(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                double *aux, double alpha, double beta, const double *dir) {
  if (A.cap <= 0) return false;
  switch (A.g) {
    case 1: launch_csr_tma<MODE, 1>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 2: launch_csr_tma<MODE, 2>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 4: launch_csr_tma<MODE, 4>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 8: launch_csr_tma<MODE, 8>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 16: launch_csr_tma<MODE, 16>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 32: launch_csr_tma<MODE, 32>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    default: return false;
  }
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  return true;
}

}  // namespace bf
