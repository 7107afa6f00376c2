// k_csr_win.cuh -- windowed jagged-diagonal ("WJDS") kernels for the coarse (Galerkin) levels: A_l
// and the fused restrictions Rf_l with at least win_nmin rows.
//
// Why: ncu on the TMA CSR kernels of the Galerkin levels (k_csr_tma.cuh, G lanes per row) shows
// ~40 % of the DRAM bandwidth with NO unit saturated -- about 2 warp instructions are issued per
// nonzero (per-row bookkeeping, predicated gather slots, shuffles, an epilogue with 1 lane in G
// active) and every gather is an L2 round trip.  This layout removes both:
//
//  * rows are grouped in blocks of `wrows` consecutive rows, one CTA of wrows threads per block.
//    After the Morton renumbering of the coarse levels (k_amg_setup.cu reorder_levels) a block
//    touches only ~3-6 distinct columns per row, so setup stores per block the sorted list of its
//    distinct columns (the WINDOW, wcol[blk * wstride + i], i < cnt) and per nonzero the uint16
//    position of its column in that list.  The kernel gathers the window once into shared memory
//    (sorted columns: the gathers coalesce into runs) and every product reads x from shared
//    memory.
//  * inside a block the rows are sorted by length (descending, ties by row); thread t owns the
//    row at position t.  The block's entries are stored by jagged diagonals: entry e of position
//    t at eo + off[e] + t, where off[e] counts the entries of the diagonals before e (diagonal e
//    holds the rows longer than e, a prefix of the sorted order).  No padding (a sliced-ELL
//    variant measured 12-30 % padding at these block sizes), consecutive threads read consecutive
//    addresses, and a block's values and its local indices are each ONE contiguous 16-B aligned
//    range: one elected thread fetches the whole block with two bulk copies (cp.async.bulk +
//    mbarrier, the TMA engine) while the other threads gather the window.
//  * everything a block needs first sits at an address computable from blockIdx alone (meta,
//    diagonal offsets, row order, window columns: fixed strides), so a CTA's life is ONE round
//    trip for that setup data (before griddepcontrol.wait: it overlaps the previous kernel), one
//    for the matrix stream and the window gathers in parallel, then ~20 instructions per row entry
//    from shared memory and a coalesced fused epilogue from row sums staged in shared memory.
//    Throughput = resident CTAs x block bytes / CTA lifetime: blocks are sized to ~24-36 KB so
//    that 5-7 CTAs per SM keep > 100 KB in flight per SM with no registers tied up (a first
//    version that streamed slices through registers was latency bound at 3.2 TB/s; a version with
//    three dependent round trips per CTA at 4 TB/s).
//
// A row's products are summed by 256 / wrows thread groups (group g: the entries e = g mod ng in
// ascending order) whose partial sums are added in group order: deterministic for a given block
// size; with wrows = 256 it is the sequential order of the CSR row.
// Bytes per nonzero: 10 (8 value + 2 index) instead of 12, plus 4 per window column from DRAM (x
// itself is L2 resident) and ~1.6 KB of block metadata.
#pragma once
#include "bf_internal.cuh"
#include "k_csr_tma.cuh"

namespace bf {

constexpr int WIN_MAX = 4096;     // largest window (doubles) a block may need: 32 KB of shared memory
constexpr int WIN_HASH = 8192;    // setup: per-CTA hash table slots at most (distinct columns <= WIN_MAX)
constexpr int WIN_ROWS_MAX = 256; // rows per block at most
constexpr int WJDS_MAXLEN = 255;  // longest row a block may hold (jdo has WJDS_MAXLEN + 1 slots per block)
constexpr int WJDS_STAGE_MAX = 80 * 1024;     // hard limit of a block's stream (else smaller blocks)

// local index, range-checked (and clamped) in the checked build
#define BF_LC(idx, cnt) (BF_CHK((int)(idx) < (cnt)) ? (int)(idx) : 0)

// 256 threads per CTA whatever the block's row count: the window is gathered by all of them (<= 8
// columns each from registers, one round trip), and 256 / wrows thread groups share a row's
// entries (group g takes the jagged diagonals e = g, g + NG, ...); the groups' partial sums are
// added in group order in the epilogue (deterministic; not the sequential order of the CSR row).
constexpr int WJDS_THREADS = 256;
constexpr int WJDS_WK = 8;  // window columns per thread held in registers (8 x 256 = 2048 of <= WIN_MAX)

template <int MODE>
__global__ void __launch_bounds__(WJDS_THREADS) k_wjds(int n, int m, int wrows, const int4 *__restrict__ meta,
                                              const uint16_t *__restrict__ jdo, const uint32_t *__restrict__ rowinfo,
                                              const uint16_t *__restrict__ lc, const double *__restrict__ val,
                                              const int32_t *__restrict__ wcol, const double *__restrict__ x,
                                              const double *__restrict__ b, const double *__restrict__ dinv,
                                              double *__restrict__ y, double *__restrict__ aux, double alpha,
                                              double beta, const double *__restrict__ dir, int wsm, int cap_ne, int wstride) {
  constexpr int NT = WJDS_THREADS;
  extern __shared__ __align__(128) unsigned char wjds_sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint16_t offs[WJDS_MAXLEN + 1];
  double *sval = reinterpret_cast<double *>(wjds_sm);                           // cap_ne values
  uint16_t *slc = reinterpret_cast<uint16_t *>(wjds_sm + (size_t)cap_ne * 8);   // cap_ne local indices
  double *win = reinterpret_cast<double *>(wjds_sm + (size_t)cap_ne * 10);      // wsm: window of x (cap_ne % 8 == 0)
  double *racc = win + wsm;                                                     // NT: partial row sums [group][row]
  const int blk = blockIdx.x, tid = threadIdx.x;
  const int t = tid & (wrows - 1), g = tid / wrows, ng = NT / wrows;  // row position, entry group
  // round trip 1: the block's setup data, all at addresses computable from blk
  const int4 mt = __ldg(meta + blk);  // entry offset, entries (multiple of 8), window length, longest row
  const uint32_t ri = __ldg(rowinfo + (size_t)blk * wrows + t);  // (row length << 16) | row within the block
  const int32_t *wc = wcol + (size_t)blk * wstride;  // wstride: the matrix's largest window rounded up to 256
  int wi[WJDS_WK];
#pragma unroll
  for (int k = 0; k < WJDS_WK; k++) wi[k] = k * NT < wstride ? __ldg(wc + tid + k * NT) : 0;  // (uniform guard)
  offs[tid] = __ldg(jdo + (size_t)blk * (WJDS_MAXLEN + 1) + tid);       // WJDS_MAXLEN + 1 == NT
  int ne = mt.y;
  if (!BF_CHK(ne <= cap_ne)) ne = 0;
  const int cnt = min(mt.z, wsm);
  if (tid == 0) {  // the block's whole matrix stream: two bulk copies
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (ne > 0) {
      const uint64_t pol = l2_evict_first_policy();
      mbar_expect_tx(&bar, (uint32_t)ne * 10u);
      tma_bulk_g2s(sval, val + mt.x, (uint32_t)ne * 8u, &bar, pol);
      tma_bulk_g2s(slc, lc + mt.x, (uint32_t)ne * 2u, &bar, pol);
    }
  }
  const int r = blk * wrows + tid;  // the epilogue row of threads tid < wrows
  const bool own = tid < wrows && r < n;
  pdl_wait();  // x, b, dinv, dir and the outputs are touched only after this
  // round trip 2: window gathers and the epilogue's row operands (the stream is in flight)
  double xw[WJDS_WK];
#pragma unroll
  for (int k = 0; k < WJDS_WK; k++) xw[k] = tid + k * NT < cnt ? __ldg(x + BF_COL(wi[k], m)) : 0.0;
  double eb = 0.0, ed = 0.0, ex = 0.0, edir = 0.0;
  if (own) {
    if (MODE == OP_RESID || MODE == OP_SUB_X0 || MODE == OP_SMOOTH) eb = __ldg(b + r);
    if (MODE == OP_SUB_X0 || MODE == OP_SMOOTH || MODE == OP_SPMV_X0) ed = __ldg(dinv + r);
    if (MODE == OP_SMOOTH) ex = __ldg(x + r);
    if (MODE == OP_SMOOTH && dir) edir = dir[r];
    if (MODE == OP_ADD) ex = y[r];
  }
#pragma unroll
  for (int k = 0; k < WJDS_WK; k++)
    if (tid + k * NT < cnt) win[tid + k * NT] = xw[k];
#pragma unroll 4
  for (int i = tid + WJDS_WK * NT; i < cnt; i += NT) win[i] = __ldg(x + BF_COL(__ldg(wc + i), m));
  __syncthreads();  // window and offsets complete; the barrier's initialisation visible to every thread
  if (ne > 0) mbar_wait(&bar, 0);
  {
    const int len = ne > 0 ? (int)(ri >> 16) : 0;
    const int lr = (int)(ri & 0xffffu);
    const double *vp = sval + t;
    const uint16_t *ip = slc + t;
    double acc = 0.0;
#pragma unroll 4
    for (int e = g; e < len; e += ng) {
      const int o = offs[e];
      acc += vp[o] * win[BF_LC(ip[o], cnt)];
    }
    if (lr < wrows) racc[g * wrows + lr] = acc;
  }
  __syncthreads();
  if (own) {  // fused epilogue in row order (coalesced)
    double acc = racc[tid];
    for (int k = 1; k < ng; k++) acc += racc[k * wrows + tid];
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
  pdl_launch_dependents();
}

inline int wjds_smem_bytes(const WJds &W) {
  return W.cap_ne * 10 + 8 * (((W.wmax_used + 1) & ~1) + WJDS_THREADS);
}

template <int MODE>
bool csr_op_win(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                double *aux, double alpha, double beta, const double *dir) {
  if (!A.ws || !A.ws->wrows) return false;
  const WJds &W = *A.ws;
  ensure_smem_attr((const void *)k_wjds<MODE>, 200 * 1024);
  const int wsm = (W.wmax_used + 1) & ~1;
  const int nblocks = (A.n + W.wrows - 1) / W.wrows;
  launch_pdl(c, k_wjds<MODE>, dim3(nblocks), dim3(WJDS_THREADS), (size_t)wjds_smem_bytes(W), A.n, A.m, W.wrows,
             (const int4 *)W.meta, (const uint16_t *)W.jdo, (const uint32_t *)W.rowinfo, (const uint16_t *)W.lc,
             (const double *)W.wv, (const int32_t *)W.wcol, x, b, dinv, y, aux, alpha, beta, dir, wsm, W.cap_ne,
             W.wstride);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  return true;
}

}  // namespace bf
