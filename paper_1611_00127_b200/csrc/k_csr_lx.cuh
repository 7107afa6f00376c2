// k_csr_lx.cuh -- "local index" variant of the TMA CSR kernel for the Galerkin (coarse-level)
// operators and the transfer matrices, whose x gathers made the plain kernel L1-wavefront
// bound (75 % L1 throughput at ~40 % DRAM, ncu).
//
// At setup every tile (the same row tiles as k_csr_tma) gets the sorted list U_t of the
// distinct columns its nonzeros touch, and each nonzero stores its position in U_t as a
// 16-bit local index instead of a 32-bit column.  At solve time the CTA moves rp, the local
// indices, the values and U_t into shared memory with TMA bulk copies (double-buffered), gathers
// x[U_t] ONCE per tile into shared memory (sorted columns: coalesced), and forms the rows from
// shared memory only.  Consecutive Galerkin rows share most of their columns, so a tile
// gathers each x entry once instead of once per nonzero (reuse measured at setup; the variant
// is used only when it is >= 1.5), and the index stream shrinks from 4 to 2 bytes/nonzero.
#pragma once
#include <climits>
#include "bf_internal.cuh"
#include "k_spmv.cuh"

namespace bf {

__host__ __device__ inline int lx_rp_bytes(int rpt) { return ((4 * (rpt + 8)) + 15) & ~15; }
__host__ __device__ inline int lx_li_bytes(int cap) { return ((2 * (cap + 16)) + 15) & ~15; }
__host__ __device__ inline int lx_v_bytes(int cap) { return ((8 * (cap + 4)) + 15) & ~15; }
__host__ __device__ inline int lx_u_bytes(int ucap) { return ((4 * (ucap + 8)) + 15) & ~15; }
__host__ __device__ inline int lx_stage_bytes(int cap, int rpt, int ucap) {
  return lx_rp_bytes(rpt) + lx_li_bytes(cap) + lx_v_bytes(cap) + lx_u_bytes(ucap);
}

template <int MODE, int G>
__global__ void __launch_bounds__(TMA_THREADS) k_csr_lx(int n, int rpt, int ntiles, int cap, int ucap,
                                                        const int32_t *__restrict__ rp,
                                                        const int16_t *__restrict__ li,
                                                        const double *__restrict__ v,
                                                        const int32_t *__restrict__ uoff,
                                                        const int32_t *__restrict__ ucol,
                                                        const double *__restrict__ x, const double *__restrict__ b,
                                                        const double *__restrict__ dinv, double *__restrict__ y,
                                                        double *__restrict__ aux, double alpha, double beta,
                                                        const double *__restrict__ dir) {
  constexpr int ST = 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[ST];
  const int rb = lx_rp_bytes(rpt), lb = lx_li_bytes(cap), vb = lx_v_bytes(cap);
  const int stage_bytes = lx_stage_bytes(cap, rpt, ucap);
  double *xs = reinterpret_cast<double *>(smem_raw + ST * stage_bytes);  // gathered x[U_t]
  int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < ST; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int t, int s) {
    int r0 = t * rpt, r1 = min(r0 + rpt, n);
    int q0 = __ldg(rp + r0), q1 = __ldg(rp + r1);
    int u0 = __ldg(uoff + t), u1 = __ldg(uoff + t + 1);
    int l0 = q0 & ~7, l1 = (q1 + 7) & ~7;   // 16-B aligned int16 range
    int v0 = q0 & ~1, v1 = (q1 + 1) & ~1;   // 16-B aligned double range
    int c0 = u0 & ~3, c1 = (u1 + 3) & ~3;   // 16-B aligned int32 range
    unsigned char *base = smem_raw + s * stage_bytes;
    uint32_t br = 4u * ((r1 - r0 + 1 + 3) & ~3), bl = 2u * (l1 - l0), bv = 8u * (v1 - v0), bu = 4u * (c1 - c0);
    mbar_expect_tx(&bars[s], br + bl + bv + bu);
    tma_bulk_g2s(base, rp + r0, br, &bars[s], pol);
    if (bl) tma_bulk_g2s(base + rb, li + l0, bl, &bars[s], pol);
    if (bv) tma_bulk_g2s(base + rb + lb, v + v0, bv, &bars[s], pol);
    if (bu) tma_bulk_g2s(base + rb + lb + vb, ucol + c0, bu, &bars[s], pol);
  };
  int t = blockIdx.x;
  if (t >= ntiles) return;
  if (tid == 0)
    for (int s = 0; s < ST && t + s * (int)gridDim.x < ntiles; s++) issue(t + s * gridDim.x, s);
  const int sub = tid % G;
  for (int it = 0; t < ntiles; t += gridDim.x, it++) {
    int s = it % ST;
    int r0 = t * rpt;
    int u0 = __ldg(uoff + t), u1 = __ldg(uoff + t + 1);
    mbar_wait(&bars[s], (it / ST) & 1);
    const unsigned char *base = smem_raw + s * stage_bytes;
    const int32_t *srp = reinterpret_cast<const int32_t *>(base);
    int q0 = srp[0];
    const int16_t *sl = reinterpret_cast<const int16_t *>(base + rb) - (q0 & ~7);
    const double *sv = reinterpret_cast<const double *>(base + rb + lb) - (q0 & ~1);
    const int32_t *su = reinterpret_cast<const int32_t *>(base + rb + lb + vb) + (u0 - (u0 & ~3));
    for (int u = tid; u < u1 - u0; u += TMA_THREADS) xs[u] = __ldg(x + su[u]);
    __syncthreads();
    for (int row_in_tile = tid / G; row_in_tile < ((rpt + (TMA_THREADS / G) - 1) / (TMA_THREADS / G)) * (TMA_THREADS / G);
         row_in_tile += TMA_THREADS / G) {
      int r = r0 + row_in_tile;
      bool ok = row_in_tile < rpt && r < n;
      int lo = ok ? srp[row_in_tile] : 0, hi = ok ? srp[row_in_tile + 1] : 0;
      double acc = 0.0;
#pragma unroll 4
      for (int q = lo + sub; q < hi; q += G) acc += sv[q] * xs[sl[q]];
      if (G > 1) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
      }
      if (!ok || sub != 0) continue;
      if (MODE == OP_SPMV) {
        y[r] = acc;
      } else if (MODE == OP_SPMV_X0) {
        y[r] = acc;
        aux[r] = beta * (acc * dinv[r]);
      } else if (MODE == OP_RESID) {
        y[r] = b[r] - acc;
      } else if (MODE == OP_SUB_X0) {
        double tt = b[r] - acc;
        y[r] = tt;
        aux[r] = beta * (tt * dinv[r]);
      } else if (MODE == OP_SMOOTH) {
        double dn = beta * ((b[r] - acc) * dinv[r]);
        if (dir) dn += alpha * dir[r];
        y[r] = x[r] + dn;
        if (aux) aux[r] = dn;
      } else if (MODE == OP_ADD) {
        y[r] += acc;
      }
    }
    __syncthreads();  // stage s and xs are free again
    if (tid == 0 && t + ST * (int)gridDim.x < ntiles) issue(t + ST * gridDim.x, s);
  }
}

template <int MODE, int G>
void launch_csr_lx(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
                   double *aux, double alpha, double beta, const double *dir) {
  static bool configured = false;
  if (!configured) {
    BF_CUDA(cudaFuncSetAttribute(k_csr_lx<MODE, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  int smem = 2 * lx_stage_bytes(A.cap, A.rpt, A.ucap) + 8 * (A.ucap + 8);
  int ntiles = (A.n + A.rpt - 1) / A.rpt;
  int per_sm = std::max(1, std::min(8, (220 * 1024) / (smem + 1024)));
  int grid = std::min(ntiles, c->num_sms * per_sm);
  k_csr_lx<MODE, G><<<grid, TMA_THREADS, smem, c->stream>>>(A.n, A.rpt, ntiles, A.cap, A.ucap, A.rp, A.lidx, A.v,
                                                            A.uoff, A.ucol, x, b, dinv, y, aux, alpha, beta, dir);
}

template <int MODE>
bool csr_op_lx(bf_ctx *c, const DCsr &A, const double *x, const double *b, const double *dinv, double *y,
               double *aux, double alpha, double beta, const double *dir) {
  if (!A.lidx) return false;
  switch (A.g) {
    case 1: launch_csr_lx<MODE, 1>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 2: launch_csr_lx<MODE, 2>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 4: launch_csr_lx<MODE, 4>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 8: launch_csr_lx<MODE, 8>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 16: launch_csr_lx<MODE, 16>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    case 32: launch_csr_lx<MODE, 32>(c, A, x, b, dinv, y, aux, alpha, beta, dir); break;
    default: return false;
  }
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  return true;
}

// ---- setup: per-tile sorted unique columns and 16-bit local indices ---------------------
constexpr int LX_SORT = 4096;  // max nonzeros per tile handled by the in-smem bitonic sort

// bitonic sort of the tile's columns (padded with INT_MAX) in smem; returns padded size
static __device__ inline int tile_sort_cols(const DCsr &A, int rpt, int t, int *s) {
  int r0 = t * rpt, r1 = min(r0 + rpt, A.n);
  int q0 = A.rp[r0], q1 = A.rp[r1], m = q1 - q0;
  int P2 = 1;
  while (P2 < m) P2 <<= 1;
  for (int e = threadIdx.x; e < P2; e += blockDim.x) s[e] = e < m ? A.ci[q0 + e] : INT_MAX;
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int e = threadIdx.x; e < P2; e += blockDim.x) {
        int p = e ^ j;
        if (p > e) {
          bool up = (e & k) == 0;
          int a = s[e], bb = s[p];
          if ((a > bb) == up) {
            s[e] = bb;
            s[p] = a;
          }
        }
      }
      __syncthreads();
    }
  return m;
}

static __global__ void k_lx_count(DCsr A, int rpt, int ntiles, int32_t *ucnt) {
  __shared__ int s[LX_SORT];
  __shared__ int cnt;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x == 0) cnt = 0;
    int m = tile_sort_cols(A, rpt, t, s);
    int local = 0;
    for (int e = threadIdx.x; e < m; e += blockDim.x) local += (e == 0 || s[e] != s[e - 1]);
    atomicAdd(&cnt, local);
    __syncthreads();
    if (threadIdx.x == 0) ucnt[t] = cnt;
    __syncthreads();
  }
}

static __global__ void k_lx_fill(DCsr A, int rpt, int ntiles, const int32_t *__restrict__ uoff, int32_t *ucol,
                          int16_t *lidx) {
  __shared__ int s[LX_SORT];
  __shared__ int uq[LX_SORT];
  __shared__ int nu;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int m = tile_sort_cols(A, rpt, t, s);
    // compact the unique values (serial over warps is fine: setup only)
    if (threadIdx.x == 0) {
      int k = 0;
      for (int e = 0; e < m; e++)
        if (e == 0 || s[e] != s[e - 1]) uq[k++] = s[e];
      nu = k;
    }
    __syncthreads();
    int u0 = uoff[t];
    for (int e = threadIdx.x; e < nu; e += blockDim.x) ucol[u0 + e] = uq[e];
    int r0 = t * rpt, r1 = min(r0 + rpt, A.n);
    int q0 = A.rp[r0], q1 = A.rp[r1];
    for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
      int col = A.ci[q], lo = 0, hi = nu;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (uq[mid] < col) lo = mid + 1;
        else hi = mid;
      }
      lidx[q] = (int16_t)lo;
    }
    __syncthreads();
  }
}

}  // namespace bf
