// k_amg_setup.cu -- device AMG hierarchy setup for A_ss and S~ ("AMG constructs
// coarse grids based on the matrix values only"; P:L275 classical interpolation, one
// V-cycle).  CLJP is replaced by PMIS with hash-seeded weights (R5) so that
// the C/F split is deterministic; interpolation follows R6/R8; Galerkin R A P with a
// deterministic expand-sort-compress SpGEMM.
//
// Determinism: every value is produced by exactly one thread in the order stated in
// DESIGN.md ("Determinism contract") with explicitly rounded __dmul_rn / __dadd_rn /
// __ddiv_rn; PMIS is integer-only with synchronous rounds.  The hierarchy is therefore
// bit-identical run to run and to the oracle.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "bf_internal.cuh"
BF_CHECK_TU("k_amg_setup.cu")

#include <algorithm>
#include <vector>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace bf {

__device__ __forceinline__ uint32_t h32(uint64_t seed, int level, int64_t i) {
  uint64_t z = seed ^ ((uint64_t)level * 0x9E3779B97F4A7C15ULL) ^ (uint64_t)i;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  return (uint32_t)(z >> 32);
}

__global__ void k_diag(DCsr A, double *diag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double d = 0.0;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++)
    if (A.ci[q] == i) d = A.v[q];
  diag[i] = d;
}

// R23: *flag = 1 if a row of A has no stored diagonal entry > 0
__global__ void k_diag_nonpos(DCsr A, int *flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double d = 0.0;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++)
    if (A.ci[q] == i) d = A.v[q];
  if (!(d > 0.0)) atomicMax(flag, 1);
}

// l1 diagonal d_i = a_ii + sum_{j != i, ascending} |a_ij|
__global__ void k_l1diag(DCsr A, const double *__restrict__ diag, double *dl1) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double s = diag[i];
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++)
    if (A.ci[q] != i) s = __dadd_rn(s, fabs(A.v[q]));
  dl1[i] = s;
}

__global__ void k_recip(int n, const double *__restrict__ a, double *out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = 1.0 / a[i];
}

// classical strength (reading R4): sigma_i = sign(a_ii), m_i = max_{k != i} -sigma_i a_ik,
// j strong iff m_i > 0 and -sigma_i a_ij >= theta m_i
__global__ void k_strength(DCsr A, const double *__restrict__ diag, double theta, uint8_t *strong) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double sg = diag[i] < 0.0 ? -1.0 : 1.0;
  double m = -INFINITY;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    double v = -sg * A.v[q];
    if (A.ci[q] != i && v > m) m = v;
  }
  double thr = __dmul_rn(theta, m);
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++)
    strong[q] = (uint8_t)(m > 0.0 && A.ci[q] != i && -sg * A.v[q] >= thr);
}

// ------------------------------------------------------------------------------- PMIS
__global__ void k_lambda(DCsr A, const uint8_t *__restrict__ strong, int *lam) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++)
    if (strong[q]) atomicAdd(&lam[A.ci[q]], 1);
}

__global__ void k_pmis_init(int n, const int *__restrict__ lam, uint64_t seed, int level, uint64_t *key,
                            int8_t *state) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = ((uint64_t)(uint32_t)lam[i] << 32) | (uint64_t)h32(seed, level, i);
  state[i] = lam[i] == 0 ? 0 : -1;  // lambda_i = 0 -> F, others undecided
}

__device__ __forceinline__ bool greater_key(const uint64_t *key, int a, int b) {
  uint64_t ka = key[a], kb = key[b];
  return ka > kb || (ka == kb && a > b);
}

// All PMIS rounds in one cooperative kernel, two grid-wide barriers per round:
//   phase 1: every strong edge with both ends undecided marks its smaller end in notmax[p];
//   phase 2: an undecided i with no mark becomes C; otherwise it becomes F if some j in S_i is a
//            new C point, else it stays undecided.
// "j is a new C point of this round" is evaluated from state[j] and notmax[p][j] without a
// separate flag array: an undecided i never has an OLDER C point in S_i (it would have become
// F in that round), so state[j] == 1 can only have been written in this phase, and for a j
// still read as undecided the mark decides -- the same value whichever way the race between
// i's read and j's write goes (state[j] is read once).  The marks alternate between two
// buffers, the idle one is cleared in phase 2.  Chains of strictly ordered keys can need
// hundreds of rounds (measured: 500 on a S~ level).
constexpr int PM_CH = 4;
__global__ void k_pmis_coop(DCsr A, const uint8_t *__restrict__ strong, const uint64_t *__restrict__ key,
                            int8_t *state, uint8_t *notmax0, uint8_t *notmax1, int *nU, int max_rounds, int *rounds) {
  cg::grid_group grid = cg::this_grid();
  const int n = A.n;
  const int stride = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = t0; i < n; i += stride) notmax0[i] = 0, notmax1[i] = 0;
  grid.sync();
  int round = 0;
  for (; round < max_rounds; round++) {
    int *cnt = nU + (round & 1);
    uint8_t *notmax = (round & 1) ? notmax1 : notmax0, *idle = (round & 1) ? notmax0 : notmax1;
    if (t0 == 0) *cnt = 0;
    // Both phases walk a row in chunks of PM_CH entries with the loads of a chunk issued
    // together (columns and strength flags, then the neighbours' states, then their keys /
    // marks): a grid-stride thread is bound by its chain of dependent gathers otherwise.
    for (int i = t0; i < n; i += stride) {
      if (state[i] >= 0) continue;
      const int r0 = A.rp[i], r1 = A.rp[i + 1];
      const uint64_t ki = key[i];
      bool mark_i = false;
      for (int q0 = r0; q0 < r1; q0 += PM_CH) {
        int j[PM_CH];
        bool und[PM_CH];
#pragma unroll
        for (int u = 0; u < PM_CH; u++) {
          int q = q0 + u;
          j[u] = q < r1 ? A.ci[q] : -1;
          und[u] = q < r1 && strong[q];
        }
#pragma unroll
        for (int u = 0; u < PM_CH; u++) und[u] = und[u] && state[j[u]] < 0;
        uint64_t kj[PM_CH];
#pragma unroll
        for (int u = 0; u < PM_CH; u++) kj[u] = und[u] ? key[j[u]] : 0;
#pragma unroll
        for (int u = 0; u < PM_CH; u++) {
          if (!und[u]) continue;
          if (ki > kj[u] || (ki == kj[u] && i > j[u])) notmax[j[u]] = 1;
          else mark_i = true;
        }
      }
      if (mark_i) notmax[i] = 1;
    }
    grid.sync();
    int local = 0;
    for (int i = t0; i < n; i += stride) {
      idle[i] = 0;
      if (state[i] >= 0) continue;
      if (!notmax[i]) { state[i] = 1; continue; }
      bool f = false;
      const int r0 = A.rp[i], r1 = A.rp[i + 1];
      for (int q0 = r0; q0 < r1 && !f; q0 += PM_CH) {
        int j[PM_CH];
        bool st[PM_CH];
#pragma unroll
        for (int u = 0; u < PM_CH; u++) {
          int q = q0 + u;
          j[u] = q < r1 ? A.ci[q] : -1;
          st[u] = q < r1 && strong[q];
        }
        int8_t sj[PM_CH];
        uint8_t nm[PM_CH];
#pragma unroll
        for (int u = 0; u < PM_CH; u++) {
          sj[u] = st[u] ? *(volatile const int8_t *)(state + j[u]) : (int8_t)0;
          nm[u] = st[u] ? notmax[j[u]] : (uint8_t)1;
        }
#pragma unroll
        for (int u = 0; u < PM_CH; u++) f = f || (st[u] && (sj[u] == 1 || (sj[u] < 0 && !nm[u])));
      }
      if (f) *(volatile int8_t *)(state + i) = 0;
      else local++;
    }
    if (local) atomicAdd(cnt, local);
    grid.sync();
    if (*(volatile int *)cnt == 0) break;
  }
  if (t0 == 0) *rounds = round + 1;
}

__global__ void k_is_c(int n, const int8_t *__restrict__ cf, int32_t *flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = cf[i] == 1;
}

// ------------------------------------------------------------------------------- interpolation
__global__ void k_interp_count(DCsr A, const uint8_t *__restrict__ strong, const int8_t *__restrict__ cf,
                               int32_t *cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  int c = 0;
  if (cf[i] == 1) c = 1;
  else
    for (int q = A.rp[i]; q < A.rp[i + 1]; q++)
      if (strong[q] && cf[A.ci[q]] == 1) c++;
  cnt[i] = c;
}

__device__ __forceinline__ int bsearch_pos(const int32_t *a, int lo, int hi, int key) {
  // position of key in a[lo,hi) or -1
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int v = a[mid];
    if (v == key) return mid;
    if (v < key) lo = mid + 1;
    else hi = mid;
  }
  return -1;
}

// classical (Ruge-Stueben) interpolation, reading R6 (c.2 step 3.3) with the R8 denominator
// option.  P.ci temporarily holds fine column indices (ascending), mapped to coarse at the end.
__global__ void k_interp_fill(DCsr A, const uint8_t *__restrict__ strong, const int8_t *__restrict__ cf,
                              const int32_t *__restrict__ cmap, const double *__restrict__ diag, int norm,
                              DCsr P, const uint8_t *__restrict__ only) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  if (only && !only[i]) return;
  int base = P.rp[i], end = P.rp[i + 1];
  if (cf[i] == 1) {
    P.ci[base] = cmap[i];
    P.v[base] = 1.0;
    return;
  }
  if (end == base) return;  // C_i empty -> empty row
  // pass 1: num_j = a_ij on C_i; dg = a_ii + sum over the weak set W_i (ascending)
  double dg = diag[i];
  int t = base;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    int j = A.ci[q];
    if (j == i) continue;
    if (strong[q] && cf[j] == 1) {
      P.ci[t] = j;
      P.v[t] = A.v[q];
      t++;
    } else if (!strong[q]) {
      dg = __dadd_rn(dg, A.v[q]);
    }
  }
  // pass 2: strong F neighbours k ascending
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    int k = A.ci[q];
    if (k == i || !strong[q] || cf[k] == 1) continue;
    double aik = A.v[q];
    double sk = diag[k] < 0.0 ? -1.0 : 1.0;
    double Dk = 0.0;
    for (int s = A.rp[k]; s < A.rp[k + 1]; s++) {
      if (bsearch_pos(P.ci, base, end, A.ci[s]) < 0) continue;
      double a = A.v[s];
      double abar = (sk * a < 0.0) ? a : 0.0;
      Dk = __dadd_rn(Dk, abar);
    }
    if (Dk == 0.0) {
      dg = __dadd_rn(dg, aik);
    } else {
      double cc = __ddiv_rn(aik, Dk);
      for (int s = A.rp[k]; s < A.rp[k + 1]; s++) {
        int p = bsearch_pos(P.ci, base, end, A.ci[s]);
        if (p < 0) continue;
        double a = A.v[s];
        double abar = (sk * a < 0.0) ? a : 0.0;
        P.v[p] = __dadd_rn(P.v[p], __dmul_rn(cc, abar));
      }
    }
  }
  double den = dg;
  if (norm) {
    den = 0.0;
    for (int p = base; p < end; p++) den = __dadd_rn(den, P.v[p]);
  }
  for (int p = base; p < end; p++) {
    double num = P.v[p];
    double w = den == 0.0 ? 0.0 : (norm ? __ddiv_rn(num, den) : -__ddiv_rn(num, den));
    P.v[p] = w;
    P.ci[p] = cmap[P.ci[p]];
  }
}

// Warp-per-row classical interpolation: the same sequence of roundings as k_interp_fill (and
// the oracle), with the row's entries, the C_i set and the strong-F rows scanned by 32 lanes.
// Every ordered sum (dg, D_k, the R8 denominator) is accumulated by lane 0 in ascending
// column order from values gathered with shuffles; each num_m is updated by the one lane that
// owns m, once per k, k ascending.  Rows with more than IW_CAP strong C or strong F
// neighbours are flagged and done by k_interp_fill.
constexpr int IW_WARPS = 8;
constexpr int IW_CAP = 128;

__device__ __forceinline__ void interp_warp_row(const DCsr &A, const uint8_t *__restrict__ strong,
                                                const int8_t *__restrict__ cf, const int32_t *__restrict__ cmap,
                                                const double *__restrict__ diag, int norm, const DCsr &P,
                                                uint8_t *long_rows, int *any_long, int i, int lane, int *ccol,
                                                double *num, int *fk, double *fa) {
  const int base = P.rp[i], end = P.rp[i + 1];
  if (cf[i] == 1) {
    if (lane == 0) {
      P.ci[base] = cmap[i];
      P.v[base] = 1.0;
    }
    return;
  }
  if (end == base) return;
  const int r0 = A.rp[i], r1 = A.rp[i + 1];
  // pass 1: C_i (ascending) with num = a_ij; F_i^s (ascending) with a_ik; dg over the weak set
  int nc = 0, nf = 0;
  double dg = diag[i];
  for (int q0 = r0; q0 < r1; q0 += 32) {
    int q = q0 + lane;
    bool valid = q < r1;
    int j = valid ? A.ci[q] : -1;
    double a = valid ? A.v[q] : 0.0;
    bool st = valid && strong[q] && j != i;
    int8_t cj = (valid && j >= 0) ? cf[j] : 0;
    bool isC = st && cj == 1, isF = st && cj != 1, weak = valid && !strong[q] && j != i;
    unsigned mc = __ballot_sync(0xffffffffu, isC), mf = __ballot_sync(0xffffffffu, isF);
    unsigned mw = __ballot_sync(0xffffffffu, weak);
    if (nc + __popc(mc) > IW_CAP || nf + __popc(mf) > IW_CAP) {
      if (lane == 0) {
        long_rows[i] = 1;
        atomicMax(any_long, 1);
      }
      return;
    }
    unsigned below = (1u << lane) - 1;
    if (isC) {
      ccol[nc + __popc(mc & below)] = j;
      num[nc + __popc(mc & below)] = a;
    }
    if (isF) {
      fk[nf + __popc(mf & below)] = j;
      fa[nf + __popc(mf & below)] = a;
    }
    // dg = dg + a_in over the weak entries, ascending (lane 0 walks the chunk in order)
    for (unsigned w = mw; w; w &= w - 1)  // set bits in ascending lane order
      dg = __dadd_rn(dg, __shfl_sync(0xffffffffu, a, __ffs(w) - 1));
    nc += __popc(mc);
    nf += __popc(mf);
  }
  __syncwarp();
  // pass 2: strong F neighbours k ascending
  // row k of the NEXT strong F neighbour (bounds, sign of a_kk, first 32 entries) is fetched
  // while the current one is processed: the per-k chain fk -> row_ptr -> entries is two
  // dependent global round trips
  int nk0 = 0, nk1 = 0, nm = -1;
  double na = 0.0, ndk = 1.0;
  if (nf > 0) {
    int k = fk[0];
    nk0 = A.rp[k];
    nk1 = A.rp[k + 1];
    ndk = diag[k];
    if (nk0 + lane < nk1) {
      nm = A.ci[nk0 + lane];
      na = A.v[nk0 + lane];
    }
  }
  for (int f = 0; f < nf; f++) {
    const double aik = fa[f];
    const double sk = ndk < 0.0 ? -1.0 : 1.0;
    const int k0 = nk0, k1 = nk1, cm = nm;
    const double ca = na;
    if (f + 1 < nf) {
      int k = fk[f + 1];
      nk0 = A.rp[k];
      nk1 = A.rp[k + 1];
      ndk = diag[k];
      nm = -1;
      if (nk0 + lane < nk1) {
        nm = A.ci[nk0 + lane];
        na = A.v[nk0 + lane];
      }
    }
    double Dk = 0.0;
    int pos1 = -1;        // single-chunk rows (<= 32 entries): this lane's entry of row k, found once
    double abar1 = 0.0;
    for (int q0 = k0; q0 < k1; q0 += 32) {  // D_k = sum over row k cap C_i of abar, ascending
      int q = q0 + lane;
      double abar = 0.0;
      bool mem = false;
      int lo = 0;
      if (q < k1) {
        int m = q0 == k0 ? cm : A.ci[q];
        int hi = nc;  // binary search of m in C_i
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (ccol[mid] < m) lo = mid + 1;
          else hi = mid;
        }
        mem = lo < nc && ccol[lo] == m;
        double a = q0 == k0 ? ca : A.v[q];
        abar = (sk * a < 0.0) ? a : 0.0;
      }
      pos1 = mem ? lo : -1;
      abar1 = abar;
      unsigned mm = __ballot_sync(0xffffffffu, mem);
      for (unsigned w = mm; w; w &= w - 1)  // members of C_i in ascending lane (= column) order
        Dk = __dadd_rn(Dk, __shfl_sync(0xffffffffu, abar, __ffs(w) - 1));
    }
    if (Dk == 0.0) {
      dg = __dadd_rn(dg, aik);  // lumped into the diagonal
      continue;
    }
    const double cc = __ddiv_rn(aik, Dk);
    if (k1 - k0 <= 32) {  // num_m += cc * abar_km (each m owned by one lane)
      if (pos1 >= 0) num[pos1] = __dadd_rn(num[pos1], __dmul_rn(cc, abar1));
    } else {
      for (int q0 = k0; q0 < k1; q0 += 32) {
        int q = q0 + lane;
        if (q < k1) {
          int m = A.ci[q];
          int lo = 0, hi = nc;
          while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (ccol[mid] < m) lo = mid + 1;
            else hi = mid;
          }
          if (lo < nc && ccol[lo] == m) {
            double a = A.v[q];
            double abar = (sk * a < 0.0) ? a : 0.0;
            num[lo] = __dadd_rn(num[lo], __dmul_rn(cc, abar));
          }
        }
      }
    }
    __syncwarp();
  }
  double den = dg;
  if (norm) {
    den = 0.0;
    for (int u = 0; u < nc; u++) den = __dadd_rn(den, num[u]);  // ascending (uniform per lane)
  }
  for (int u = lane; u < nc; u += 32) {
    double w = den == 0.0 ? 0.0 : (norm ? __ddiv_rn(num[u], den) : -__ddiv_rn(num[u], den));
    P.v[base + u] = w;
    P.ci[base + u] = cmap[ccol[u]];
  }
}

// each warp walks rows i, i + (warps in the grid), ...: about a third of the rows are C points
// and finish at once, so with one row per warp the resident warps idle (ncu: 30 % occupancy)
__global__ void __launch_bounds__(IW_WARPS * 32) k_interp_warp(DCsr A, const uint8_t *__restrict__ strong,
                                                               const int8_t *__restrict__ cf,
                                                               const int32_t *__restrict__ cmap,
                                                               const double *__restrict__ diag, int norm, DCsr P,
                                                               uint8_t *long_rows, int *any_long) {
  __shared__ int s_ccol[IW_WARPS][IW_CAP];
  __shared__ double s_num[IW_WARPS][IW_CAP];
  __shared__ int s_fk[IW_WARPS][IW_CAP];
  __shared__ double s_fa[IW_WARPS][IW_CAP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = blockIdx.x * IW_WARPS + warp; i < A.n; i += gridDim.x * IW_WARPS) {
    interp_warp_row(A, strong, cf, cmap, diag, norm, P, long_rows, any_long, i, lane, s_ccol[warp], s_num[warp],
                    s_fk[warp], s_fa[warp]);
    __syncwarp();  // the next row reuses the warp's shared-memory lists
  }
}

// ------------------------------------------------------------------------------- transpose
__global__ void k_col_count(DCsr P, int32_t *cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  for (int q = P.rp[i]; q < P.rp[i + 1]; q++) atomicAdd(&cnt[P.ci[q]], 1);
}

__global__ void k_transpose_scatter(DCsr P, const int32_t *__restrict__ Rrp, int32_t *cursor, DCsr R) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  for (int q = P.rp[i]; q < P.rp[i + 1]; q++) {
    int J = P.ci[q];
    int p = Rrp[J] + atomicAdd(&cursor[J], 1);
    if (!BF_CHK(p < Rrp[J + 1])) continue;
    R.ci[p] = i;
    R.v[p] = P.v[q];
  }
}

__global__ void k_row_sort(DCsr R) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= R.n) return;
  int a = R.rp[I], b = R.rp[I + 1];
  for (int x = a + 1; x < b; x++) {
    int key = R.ci[x];
    double v = R.v[x];
    int y = x - 1;
    while (y >= a && R.ci[y] > key) {
      R.ci[y + 1] = R.ci[y];
      R.v[y + 1] = R.v[y];
      y--;
    }
    R.ci[y + 1] = key;
    R.v[y + 1] = v;
  }
}

static void transpose(bf_ctx *c, const DCsr &P, DCsr &R) {
  R.n = P.m;
  R.m = P.n;
  int32_t *cnt = dalloc_t<int32_t>(c, R.n);
  BF_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * R.n, c->stream));
  k_col_count<<<div_up(P.n, 256), 256, 0, c->stream>>>(P, cnt);
  BF_LAUNCH(c);
  R.rp = dalloc_t<int32_t>(c, (size_t)R.n + 1);
  R.nnz = exclusive_scan_i32(c, cnt, R.rp, R.n);
  R.ci = dalloc_t<int32_t>(c, R.nnz);
  R.v = dalloc_t<double>(c, R.nnz);
  BF_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * R.n, c->stream));
  k_transpose_scatter<<<div_up(P.n, 256), 256, 0, c->stream>>>(P, R.rp, cnt, R);
  BF_LAUNCH(c);
  k_row_sort<<<div_up(R.n, 128), 128, 0, c->stream>>>(R);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  dfree(c, cnt);
}

// ------------------------------------------------------------------------------- SpGEMM
// C = A B with C(i,J) = sum over k in pattern(A,i) ascending of A(i,k) B(k,J), from +0.0,
// multiply and add rounded separately; full symbolic pattern (c.2 step 3.5).
// Expand (products in (i, k ascending) order) -> stable radix sort by (i,J) -> compress.
__global__ void k_spgemm_ub(DCsr A, DCsr B, int64_t *ub) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  int64_t s = 0;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) s += B.rp[A.ci[q] + 1] - B.rp[A.ci[q]];
  ub[i] = s;
}

// warp per row of A; product (q, t) lands at the same position as in a serial row loop
// (k ascending, then B's row order), so the stable sort keeps the ascending-k order of equal keys
__global__ void k_spgemm_expand(DCsr A, DCsr B, const int64_t *__restrict__ off, int colbits, uint64_t *keys,
                                double *vals) {
  int i = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (i >= A.n) return;
  int64_t p = off[i];
  uint64_t hi = (uint64_t)i << colbits;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    double a = A.v[q];
    int k = A.ci[q];
    int bs = B.rp[k], be = B.rp[k + 1];
    for (int t = bs + lane; t < be; t += 32) {
      keys[p + (t - bs)] = hi | (uint64_t)B.ci[t];
      vals[p + (t - bs)] = __dmul_rn(a, B.v[t]);
    }
    p += be - bs;
  }
}

__global__ void k_heads(int64_t T, const uint64_t *__restrict__ keys, int32_t *head) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= T) return;
  head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

__global__ void k_compress(int64_t T, const uint64_t *__restrict__ keys, const double *__restrict__ vals,
                           const int32_t *__restrict__ head, const int32_t *__restrict__ gidx, int colbits,
                           int32_t *rowcnt, int32_t *Cci, double *Cv) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= T || !head[p]) return;
  uint64_t key = keys[p];
  double s = 0.0;
  int64_t e = p;
  do {
    s = __dadd_rn(s, vals[e]);
    e++;
  } while (e < T && !head[e]);
  int g = gidx[p];
  Cci[g] = (int32_t)(key & ((1ull << colbits) - 1));
  Cv[g] = s;
  atomicAdd(&rowcnt[(int)(key >> colbits)], 1);
}

static int bits_for(int64_t x) {
  int b = 1;
  while ((1ll << b) <= x) b++;
  return b;
}

// ---- row-owned hash SpGEMM (default): one warp per row of C, shared-memory hash table.
// For each k of row i of A in ascending order, the warp's lanes take the entries of row k of
// B (distinct columns J within the row, so no two lanes touch the same slot), insert J and
// apply acc[J] = acc[J] + A(i,k) * B(k,J) (separately rounded); a __syncwarp between
// consecutive k keeps every entry's sum in ascending-k order -- the same sequence of
// roundings as the oracle and as the expand-sort-compress path.  Rows are emitted sorted
// (rank of each key among the row's keys).  The count kernel reports the product's longest
// row; the fill kernel is instantiated for 128 / 256 / 512 / 1024 slots (80 / 160 / 320 / 640
// columns per row at most) and the smallest table that holds the longest row is used -- the
// kernel is latency bound and its residency follows the table size.  If a row holds more than
// HASH_MAX distinct columns the count is repeated with the 1024-slot table, and beyond
// HASH_MAX_L columns the product falls back to expand-sort-compress.
constexpr int HASH_WARPS = 4;
constexpr int HASH_CAP = 512;        // max slots per warp (power of two)
constexpr int HASH_MAX = 320;        // max distinct columns per row (load factor 0.625)

// per-row table size: the smallest power of two >= 2 * (upper bound of the row's distinct
// columns), at least 32, at most HASH_CAP -- small rows (most of them) touch few slots
__device__ __forceinline__ int row_table_mask(const DCsr &A, const DCsr &B, int i, int lane, int cap = HASH_CAP) {
  int ub = 0;
  for (int q = A.rp[i] + lane; q < A.rp[i + 1]; q += 32) ub += B.rp[A.ci[q] + 1] - B.rp[A.ci[q]];
  for (int o = 16; o > 0; o >>= 1) ub += __shfl_xor_sync(0xffffffffu, ub, o);
  int t = 32;
  while (t < cap && t < 2 * ub) t <<= 1;
  return t - 1;
}

__device__ __forceinline__ int hash_slot(int key, int mask) { return (int)(((unsigned)key * 2654435761u) >> 16) & mask; }

// returns the slot of key, inserting it if absent (inserted == true for the inserting lane)
// returns the key's slot, or -1 when the table is full (every slot probed: the caller falls back
// to the expand-sort-compress product -- a row of the coarse Galerkin operators can exceed the
// table between two of the count kernel's fill checks, e.g. on C5's stalled coarse levels)
__device__ __forceinline__ int hash_insert(int *keys, int key, int mask, bool &inserted) {
  int s = hash_slot(key, mask);
  inserted = false;
  for (int probe = 0; probe <= mask; probe++) {
    int prev = atomicCAS(&keys[s], -1, key);
    if (prev == -1) {
      inserted = true;
      return s;
    }
    if (prev == key) return s;
    s = (s + 1) & mask;
  }
  return -1;
}

// the row's A entries (column k, value a) and B row bounds are loaded lane-parallel, 32 at
// a time, and broadcast by shuffles: the per-k dependent chain is then one B load, not three
struct RowChunk {
  int k, bs, be;
  double a;
};
__device__ __forceinline__ RowChunk load_chunk(const DCsr &A, const DCsr &B, int q, int r1, bool want_a) {
  RowChunk c{0, 0, 0, 0.0};
  if (q < r1) {
    c.k = A.ci[q];
    if (want_a) c.a = A.v[q];
    c.bs = B.rp[c.k];
    c.be = B.rp[c.k + 1];
  }
  return c;
}
__device__ __forceinline__ int chunk_mask(const DCsr &A, const DCsr &B, int i, int lane, int len, const RowChunk &c,
                                          int cap = HASH_CAP) {
  if (len > 32) return row_table_mask(A, B, i, lane, cap);
  int ub = c.be - c.bs;
  for (int o = 16; o > 0; o >>= 1) ub += __shfl_xor_sync(0xffffffffu, ub, o);
  int t = 32;
  while (t < cap && t < 2 * ub) t <<= 1;
  return t - 1;
}

template <int CAP, int MAXD>
__global__ void __launch_bounds__(HASH_WARPS * 32) k_spgemm_hash_count(DCsr A, DCsr B, int32_t *cnt, int *overflow) {
  __shared__ int skeys[HASH_WARPS][CAP];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i = blockIdx.x * HASH_WARPS + warp;
  if (i >= A.n) return;
  int *keys = skeys[warp];
  const int r0 = A.rp[i], r1 = A.rp[i + 1];
  RowChunk ch = load_chunk(A, B, r0 + lane, r1, false);
  int mask = chunk_mask(A, B, i, lane, r1 - r0, ch, CAP);
  for (int s = lane; s <= mask; s += 32) keys[s] = -1;
  __syncwarp();
  int count = 0;
  bool full = false;
  for (int q0 = r0; q0 < r1 && !full; q0 += 32) {
    if (q0 != r0) ch = load_chunk(A, B, q0 + lane, r1, false);
    int nq = min(32, r1 - q0);
    // as in the fill kernel, the first 32 columns of the next B row are fetched while this one is hashed
    int bs = __shfl_sync(0xffffffffu, ch.bs, 0), be = __shfl_sync(0xffffffffu, ch.be, 0);
    int nc = bs + lane < be ? B.ci[bs + lane] : -1;
    bool spill = false;
    for (int u = 0; u < nq; u++) {
      int cbs = bs, cbe = be, cc = nc;
      if (u + 1 < nq) {
        bs = __shfl_sync(0xffffffffu, ch.bs, u + 1);
        be = __shfl_sync(0xffffffffu, ch.be, u + 1);
        nc = bs + lane < be ? B.ci[bs + lane] : -1;
      }
      bool ins;
      if (cc >= 0 && !spill) {  // a lane that found the table full stops inserting
        if (hash_insert(keys, cc, mask, ins) < 0) spill = true;
        else count += ins;
      }
      for (int t = cbs + 32 + lane; t < cbe && !spill; t += 32) {
        if (hash_insert(keys, B.ci[t], mask, ins) < 0) spill = true;
        else count += ins;
      }
    }
    // once per 32 entries of the A row: stop once the row cannot fit (a full table makes
    // hash_insert return -1; the product then falls back to the ESC path)
    int tot = count;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    full = tot > MAXD || __any_sync(0xffffffffu, spill);
    if (full && lane == 0) count = MAXD + 1;  // forces the overflow flag below
  }
  for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
  if (lane == 0) {
    cnt[i] = count;
    if (count > MAXD) atomicMax(overflow, 1);
    // overflow[1] = the product's longest row (picks the fill kernel's table size); the plain
    // read first keeps the atomics to the few rows that raise the maximum
    if (count > *(volatile int *)(overflow + 1)) atomicMax(overflow + 1, count);
  }
}

constexpr int HASH_WARP_BYTES = HASH_CAP * 4 + HASH_CAP * 8 + HASH_MAX * 4 + HASH_MAX * 8;
// the fill kernel with a quarter of the table (products whose longest row has <= HASH_MAX_S
// columns -- the count kernel reports it): 2.5 KB of shared memory per warp instead of 10 KB,
// so 64 instead of 20 resident warps per SM for this latency-bound kernel
constexpr int HASH_CAP_S = 128, HASH_MAX_S = 80;
constexpr int HASH_WARP_BYTES_S = HASH_CAP_S * 4 + HASH_CAP_S * 8 + HASH_MAX_S * 4 + HASH_MAX_S * 8;
constexpr int HASH_CAP_L = 1024, HASH_MAX_L = 640;  // long rows (the fused restrictions Rf of levels >= 2): 20 KB per warp
constexpr int HASH_WARP_BYTES_L = HASH_CAP_L * 4 + HASH_CAP_L * 8 + HASH_MAX_L * 4 + HASH_MAX_L * 8;
constexpr int HASH_CAP_M = 256, HASH_MAX_M = 160;  // ... and with half of it: 5 KB, 40 warps per SM
constexpr int HASH_WARP_BYTES_M = HASH_CAP_M * 4 + HASH_CAP_M * 8 + HASH_MAX_M * 4 + HASH_MAX_M * 8;

template <int CAP, int MAXD>
__global__ void __launch_bounds__(HASH_WARPS * 32) k_spgemm_hash_fill(DCsr A, DCsr B, DCsr C) {
  extern __shared__ __align__(16) unsigned char hsm[];
  constexpr int WARP_BYTES = CAP * 4 + CAP * 8 + MAXD * 4 + MAXD * 8;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i = blockIdx.x * HASH_WARPS + warp;
  if (i >= A.n) return;
  unsigned char *wb = hsm + (size_t)warp * WARP_BYTES;
  double *vals = reinterpret_cast<double *>(wb);
  double *cvals = reinterpret_cast<double *>(wb + CAP * 8);
  int *keys = reinterpret_cast<int *>(wb + CAP * 8 + MAXD * 8);
  int *ckeys = keys + CAP;
  const int r0 = A.rp[i], r1 = A.rp[i + 1];
  RowChunk ch = load_chunk(A, B, r0 + lane, r1, true);
  int mask = chunk_mask(A, B, i, lane, r1 - r0, ch, CAP);
  for (int s = lane; s <= mask; s += 32) keys[s] = -1;
  __syncwarp();
  for (int q0 = r0; q0 < r1; q0 += 32) {  // k ascending
    if (q0 != r0) ch = load_chunk(A, B, q0 + lane, r1, true);
    int nq = min(32, r1 - q0);
    // B(k, :) of the first 32 entries of the next k is prefetched while this k is hashed
    int bs = __shfl_sync(0xffffffffu, ch.bs, 0), be = __shfl_sync(0xffffffffu, ch.be, 0);
    int nc = bs + lane < be ? B.ci[bs + lane] : -1;
    double nv = bs + lane < be ? B.v[bs + lane] : 0.0;
    for (int u = 0; u < nq; u++) {
      double a = __shfl_sync(0xffffffffu, ch.a, u);
      int cbs = bs, cbe = be, cc = nc;
      double cv = nv;
      if (u + 1 < nq) {
        bs = __shfl_sync(0xffffffffu, ch.bs, u + 1);
        be = __shfl_sync(0xffffffffu, ch.be, u + 1);
        nc = bs + lane < be ? B.ci[bs + lane] : -1;
        nv = bs + lane < be ? B.v[bs + lane] : 0.0;
      }
      if (cc >= 0) {
        bool ins;
        // cannot return -1 here: the count kernel admitted this row (<= HASH_MAX distinct columns
        // in a table of the same size), otherwise the whole product went to the ESC path
        int s = hash_insert(keys, cc, mask, ins);
        if (BF_CHK(s >= 0)) {
          double acc = ins ? 0.0 : vals[s];
          vals[s] = __dadd_rn(acc, __dmul_rn(a, cv));
        }
      }
      for (int t = cbs + 32 + lane; t < cbe; t += 32) {  // rows of B longer than 32 (rare)
        bool ins;
        int s = hash_insert(keys, B.ci[t], mask, ins);
        if (!BF_CHK(s >= 0)) continue;
        double acc = ins ? 0.0 : vals[s];
        vals[s] = __dadd_rn(acc, __dmul_rn(a, B.v[t]));
      }
      __syncwarp();
    }
  }
  // compact the occupied slots, then place each entry at its rank (rows are emitted sorted)
  int n = 0;
  for (int s0 = 0; s0 <= mask; s0 += 32) {
    int key = keys[s0 + lane];
    unsigned m = __ballot_sync(0xffffffffu, key >= 0);
    if (key >= 0) {
      int pos = n + __popc(m & ((1u << lane) - 1));
      ckeys[pos] = key;
      cvals[pos] = vals[s0 + lane];
    }
    n += __popc(m);
  }
  __syncwarp();
  int base = C.rp[i];
  for (int e = lane; e < n; e += 32) {
    int key = ckeys[e], rank = 0;
    for (int u = 0; u < n; u++) rank += ckeys[u] < key;
    if (!BF_CHK(base + rank < C.rp[i + 1])) continue;
    C.ci[base + rank] = key;
    C.v[base + rank] = cvals[e];
  }
}

// ---- thread-per-row SpGEMM for short rows of B (A P with P rows of ~1-6 entries): each
// thread keeps its row's distinct columns and sums in a small local array, accumulating in
// ascending k (same rounding sequence as above), then insertion-sorts the row.
constexpr int TPR_CAP = 48;

__global__ void k_spgemm_tpr_count(DCsr A, DCsr B, int32_t *cnt, int *overflow) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  int cols[TPR_CAP];
  int len = 0;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    int k = A.ci[q];
    for (int t = B.rp[k]; t < B.rp[k + 1]; t++) {
      int J = B.ci[t], u = 0;
      while (u < len && cols[u] != J) u++;
      if (u == len) {
        if (len == TPR_CAP) {
          atomicMax(overflow, 1);
          cnt[i] = 0;
          return;
        }
        cols[len++] = J;
      }
    }
  }
  cnt[i] = len;
}

__global__ void k_spgemm_tpr_fill(DCsr A, DCsr B, DCsr C) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  int cols[TPR_CAP];
  double acc[TPR_CAP];
  int len = 0;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {  // k ascending
    int k = A.ci[q];
    double a = A.v[q];
    for (int t = B.rp[k]; t < B.rp[k + 1]; t++) {
      int J = B.ci[t], u = 0;
      while (u < len && cols[u] != J) u++;
      if (u == len) {
        if (!BF_CHK(len < TPR_CAP)) continue;
        cols[len] = J;
        acc[len] = 0.0;
        len++;
      }
      acc[u] = __dadd_rn(acc[u], __dmul_rn(a, B.v[t]));
    }
  }
  for (int x = 1; x < len; x++) {
    int key = cols[x];
    double v = acc[x];
    int y = x - 1;
    while (y >= 0 && cols[y] > key) {
      cols[y + 1] = cols[y];
      acc[y + 1] = acc[y];
      y--;
    }
    cols[y + 1] = key;
    acc[y + 1] = v;
  }
  int base = C.rp[i];
  for (int x = 0; x < len; x++) {
    C.ci[base + x] = cols[x];
    C.v[base + x] = acc[x];
  }
}

// ---- warp-per-row SpGEMM with one lane per entry of the A row, for A P on the first coarse
// levels (A rows of 15-30 entries, P rows of 1-6): the warp-hash kernels above walk one B row
// at a time and so keep 2-3 lanes busy on these products, and the thread-per-row kernels search
// their column list linearly (O(len^2) local-memory accesses for ~60 products per row).  Here
// lane q takes A(i, k_q), inserts the columns of B(k_q, :) into the warp's shared-memory key
// table and stages its products a * b (in the row's ascending (q, t) order, at the offset given
// by a warp scan of the B row lengths); then each output column is owned by one lane, which
// sums the staged products of its column in that order -- the same rounding sequence as the
// other SpGEMM kernels (acc starts at +0.0; products rounded, then added, k ascending).
constexpr int WK_WARPS = 8;
constexpr int WK_CAP = 256;   // key slots per warp
constexpr int WK_MAX = 192;   // distinct columns per row at most (else the product falls back)
constexpr int WK_PROD = 256;  // staged products per row; longer rows re-read A and B per column

__device__ __forceinline__ int wk_mask(int ub) {
  int t = 32;
  while (t < WK_CAP && t < 2 * ub) t <<= 1;
  return t - 1;
}

// inserts the columns of the row's products; returns the number of distinct columns, or -1
template <bool STAGE>
__device__ __forceinline__ int wk_insert_row(const DCsr &A, const DCsr &B, int r0, int r1, int lane, int *keys,
                                             int *pcol, double *pval, int &nprod) {
  // upper bound on the distinct columns = number of products
  int ub = 0;
  for (int q = r0 + lane; q < r1; q += 32) {
    int k = A.ci[q];
    ub += B.rp[k + 1] - B.rp[k];
  }
  for (int o = 16; o > 0; o >>= 1) ub += __shfl_xor_sync(0xffffffffu, ub, o);
  nprod = ub;
  const int mask = wk_mask(ub);
  for (int s = lane; s <= mask; s += 32) keys[s] = -1;
  __syncwarp();
  int count = 0, base = 0;
  bool spill = false;
  const bool stage = STAGE && ub <= WK_PROD;
  for (int q0 = r0; q0 < r1; q0 += 32) {
    int q = q0 + lane, bs = 0, be = 0;
    double a = 0.0;
    if (q < r1) {
      int k = A.ci[q];
      bs = B.rp[k];
      be = B.rp[k + 1];
      if (STAGE) a = A.v[q];
    }
    int off = 0;
    if (STAGE) {  // exclusive scan of the B row lengths: this lane's first product slot
      int len = be - bs, inc = len;
      for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      off = base + inc - len;
      base += __shfl_sync(0xffffffffu, inc, 31);
    }
    for (int t = bs; t < be; t++) {
      int col = B.ci[t];
      bool ins;
      if (hash_insert(keys, col, mask, ins) < 0) {
        spill = true;
        break;
      }
      count += ins;
      if (stage) {
        pcol[off + (t - bs)] = col;
        pval[off + (t - bs)] = __dmul_rn(a, B.v[t]);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
  if (__any_sync(0xffffffffu, spill) || count > WK_MAX) return -1;
  return count;
}

__global__ void __launch_bounds__(WK_WARPS * 32) k_spgemm_wk_count(DCsr A, DCsr B, int32_t *cnt, int *overflow) {
  __shared__ int skeys[WK_WARPS][WK_CAP];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i = blockIdx.x * WK_WARPS + warp;
  if (i >= A.n) return;
  int nprod;
  int count = wk_insert_row<false>(A, B, A.rp[i], A.rp[i + 1], lane, skeys[warp], nullptr, nullptr, nprod);
  if (lane == 0) {
    cnt[i] = count < 0 ? 0 : count;
    if (count < 0) atomicMax(overflow, 1);
  }
}

__global__ void __launch_bounds__(WK_WARPS * 32) k_spgemm_wk_fill(DCsr A, DCsr B, DCsr C) {
  __shared__ int skeys[WK_WARPS][WK_CAP];
  __shared__ int sckeys[WK_WARPS][WK_MAX];
  __shared__ int spcol[WK_WARPS][WK_PROD];
  __shared__ double spval[WK_WARPS][WK_PROD];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int i = blockIdx.x * WK_WARPS + warp;
  if (i >= A.n) return;
  int *keys = skeys[warp], *ckeys = sckeys[warp], *pcol = spcol[warp];
  double *pval = spval[warp];
  const int r0 = A.rp[i], r1 = A.rp[i + 1];
  int nprod;
  int count = wk_insert_row<true>(A, B, r0, r1, lane, keys, pcol, pval, nprod);
  if (!BF_CHK(count >= 0)) return;  // the count kernel admitted every row of this product
  __syncwarp();
  const int mask = wk_mask(nprod);
  int n = 0;
  for (int s0 = 0; s0 <= mask; s0 += 32) {
    int key = keys[s0 + lane];
    unsigned m = __ballot_sync(0xffffffffu, key >= 0);
    if (key >= 0) ckeys[n + __popc(m & ((1u << lane) - 1))] = key;
    n += __popc(m);
  }
  __syncwarp();
  const int base = C.rp[i];
  const bool staged = nprod <= WK_PROD;
  for (int e = lane; e < n; e += 32) {
    int key = ckeys[e], rank = 0;
    for (int u = 0; u < n; u++) rank += ckeys[u] < key;
    double acc = 0.0;
    if (staged) {
      for (int p = 0; p < nprod; p++)
        if (pcol[p] == key) acc = __dadd_rn(acc, pval[p]);
    } else {
      for (int q = r0; q < r1; q++) {  // k ascending
        int k = A.ci[q];
        double a = A.v[q];
        for (int t = B.rp[k]; t < B.rp[k + 1]; t++)
          if (B.ci[t] == key) acc = __dadd_rn(acc, __dmul_rn(a, B.v[t]));
      }
    }
    if (!BF_CHK(base + rank < C.rp[i + 1])) continue;
    C.ci[base + rank] = key;
    C.v[base + rank] = acc;
  }
}

static void spgemm_esc(bf_ctx *c, const DCsr &A, const DCsr &B, DCsr &C);
static void spgemm_hash(bf_ctx *c, const DCsr &A, const DCsr &B, DCsr &C);

static void spgemm(bf_ctx *c, const DCsr &A, const DCsr &B, DCsr &C) {
  if (c->tune.spgemm == 2) {
    spgemm_esc(c, A, B, C);
    return;
  }
  if (B.n > 0 && (double)B.nnz / B.n <= c->tune.tpr_bmax && A.n > 0 && (double)A.nnz / A.n <= c->tune.tpr_amax && c->tune.spgemm != 1) {
    C.n = A.n;
    C.m = B.m;
    int32_t *cnt = dalloc_t<int32_t>(c, A.n);
    int *ovf = dalloc_t<int>(c, 1);
    BF_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int), c->stream));
    const bool wk = (double)A.nnz / A.n > c->tune.wk_amin;  // lane-per-entry warp kernels for the longer A rows
    if (wk) k_spgemm_wk_count<<<div_up(A.n, WK_WARPS), WK_WARPS * 32, 0, c->stream>>>(A, B, cnt, ovf);
    else k_spgemm_tpr_count<<<div_up(A.n, 128), 128, 0, c->stream>>>(A, B, cnt, ovf);
    BF_LAUNCH(c);
    int h_ovf = 0;
    BF_CUDA(cudaMemcpyAsync(&h_ovf, ovf, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    dfree(c, ovf);
    if (!h_ovf) {
      C.rp = dalloc_t<int32_t>(c, (size_t)C.n + 1);
      C.nnz = exclusive_scan_i32(c, cnt, C.rp, C.n);
      dfree(c, cnt);
      C.ci = dalloc_t<int32_t>(c, C.nnz);
      C.v = dalloc_t<double>(c, C.nnz);
      if (wk) k_spgemm_wk_fill<<<div_up(A.n, WK_WARPS), WK_WARPS * 32, 0, c->stream>>>(A, B, C);
      else k_spgemm_tpr_fill<<<div_up(A.n, 128), 128, 0, c->stream>>>(A, B, C);
      BF_LAUNCH(c);
      BF_CUDA(cudaGetLastError());
      return;
    }
    dfree(c, cnt);
    C = DCsr();
  }
  spgemm_hash(c, A, B, C);
}

static void spgemm_hash(bf_ctx *c, const DCsr &A, const DCsr &B, DCsr &C) {
  C.n = A.n;
  C.m = B.m;
  int32_t *cnt = dalloc_t<int32_t>(c, A.n);
  int *ovf = dalloc_t<int>(c, 2);
  int blocks = div_up(A.n, HASH_WARPS);
  // products with many products per row (mean over the rows) start with the 1024-slot table
  const double mean_products = A.n && B.n ? ((double)A.nnz / A.n) * ((double)B.nnz / B.n) : 0.0;
  bool large = c->tune.hash_large && mean_products > c->tune.hash_large_min;
  int h_ovf = 0, h_max = 0;
  for (;;) {
    BF_CUDA(cudaMemsetAsync(ovf, 0, 2 * sizeof(int), c->stream));
    if (large) k_spgemm_hash_count<HASH_CAP_L, HASH_MAX_L><<<blocks, HASH_WARPS * 32, 0, c->stream>>>(A, B, cnt, ovf);
    else k_spgemm_hash_count<HASH_CAP, HASH_MAX><<<blocks, HASH_WARPS * 32, 0, c->stream>>>(A, B, cnt, ovf);
    BF_LAUNCH(c);
    BF_CUDA(cudaGetLastError());
    int h_ovf2[2] = {0, 0};
    BF_CUDA(cudaMemcpyAsync(h_ovf2, ovf, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    h_ovf = h_ovf2[0];
    h_max = h_ovf2[1];
    if (c->tune.verbose)
      fprintf(stderr, "[bf] spgemm_hash: %d x %d rows, longest row %d%s%s\n", A.n, B.n, h_max, large ? " (1024-slot table)" : "",
              h_ovf ? " (overflow)" : "");
    if (h_ovf && !large && c->tune.hash_large) {
      large = true;  // second attempt with the large table before the expand-sort-compress path
      continue;
    }
    break;
  }
  dfree(c, ovf);
  if (h_ovf) {
    dfree(c, cnt);
    spgemm_esc(c, A, B, C);
    return;
  }
  C.rp = dalloc_t<int32_t>(c, (size_t)C.n + 1);
  C.nnz = exclusive_scan_i32(c, cnt, C.rp, C.n);
  dfree(c, cnt);
  C.ci = dalloc_t<int32_t>(c, C.nnz);
  C.v = dalloc_t<double>(c, C.nnz);
  if (h_max <= HASH_MAX_S && c->tune.hash_small) {
    k_spgemm_hash_fill<HASH_CAP_S, HASH_MAX_S>
        <<<blocks, HASH_WARPS * 32, HASH_WARPS * HASH_WARP_BYTES_S, c->stream>>>(A, B, C);
  } else if (h_max <= HASH_MAX_M && c->tune.hash_small) {
    k_spgemm_hash_fill<HASH_CAP_M, HASH_MAX_M>
        <<<blocks, HASH_WARPS * 32, HASH_WARPS * HASH_WARP_BYTES_M, c->stream>>>(A, B, C);
  } else if (h_max <= HASH_MAX) {
    ensure_smem_attr((const void *)k_spgemm_hash_fill<HASH_CAP, HASH_MAX>, HASH_WARPS * HASH_WARP_BYTES);
    k_spgemm_hash_fill<HASH_CAP, HASH_MAX>
        <<<blocks, HASH_WARPS * 32, HASH_WARPS * HASH_WARP_BYTES, c->stream>>>(A, B, C);
  } else {
    ensure_smem_attr((const void *)k_spgemm_hash_fill<HASH_CAP_L, HASH_MAX_L>, HASH_WARPS * HASH_WARP_BYTES_L);
    k_spgemm_hash_fill<HASH_CAP_L, HASH_MAX_L>
        <<<blocks, HASH_WARPS * 32, HASH_WARPS * HASH_WARP_BYTES_L, c->stream>>>(A, B, C);
  }
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

// ---- expand-sort-compress SpGEMM (fallback for rows with more than HASH_MAX columns)
static void spgemm_esc(bf_ctx *c, const DCsr &A, const DCsr &B, DCsr &C) {
  C.n = A.n;
  C.m = B.m;
  int64_t *ub = dalloc_t<int64_t>(c, A.n);
  k_spgemm_ub<<<div_up(A.n, 256), 256, 0, c->stream>>>(A, B, ub);
  BF_LAUNCH(c);
  int64_t *off = dalloc_t<int64_t>(c, (size_t)A.n + 1);
  int64_t T = exclusive_scan_i64(c, ub, off, A.n);
  dfree(c, ub);
  if (T >= (1ll << 31)) throw Error(BF_ERR_LIMIT, "SpGEMM expansion exceeds 2^31 products");
  int colbits = bits_for(B.m);
  int rowbits = bits_for(A.n);
  uint64_t *keys = dalloc_t<uint64_t>(c, T);
  double *vals = dalloc_t<double>(c, T);
  k_spgemm_expand<<<div_up((int64_t)A.n * 32, 256), 256, 0, c->stream>>>(A, B, off, colbits, keys, vals);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  dfree(c, off);
  sort_pairs_u64_f64(c, keys, vals, T, colbits + rowbits);
  int32_t *head = dalloc_t<int32_t>(c, T);
  k_heads<<<div_up(T, 256), 256, 0, c->stream>>>(T, keys, head);
  BF_LAUNCH(c);
  int32_t *gidx = dalloc_t<int32_t>(c, (size_t)T + 1);
  int64_t nnz = exclusive_scan_i32(c, head, gidx, (int32_t)T);
  C.nnz = nnz;
  C.ci = dalloc_t<int32_t>(c, nnz);
  C.v = dalloc_t<double>(c, nnz);
  int32_t *rowcnt = dalloc_t<int32_t>(c, C.n);
  BF_CUDA(cudaMemsetAsync(rowcnt, 0, sizeof(int32_t) * C.n, c->stream));
  k_compress<<<div_up(T, 256), 256, 0, c->stream>>>(T, keys, vals, head, gidx, colbits, rowcnt, C.ci, C.v);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  dfree(c, keys);
  dfree(c, vals);
  dfree(c, head);
  dfree(c, gidx);
  C.rp = dalloc_t<int32_t>(c, (size_t)C.n + 1);
  exclusive_scan_i32(c, rowcnt, C.rp, C.n);
  dfree(c, rowcnt);
}

// ------------------------------------------------------------------------------- coarse LU
// dense LU with partial pivoting (tie -> lowest row index), one CTA, matrix staged in smem.
// Singular if |pivot| <= 1e-14 max|a|: *sing = pivot index.
__global__ void k_coarse_lu(DCsr A, double *lu, int32_t *piv, double *inv, int *sing) {
  extern __shared__ double sm[];
  int n = A.n;
  __shared__ double amax_s;
  __shared__ int p_s;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) sm[e] = 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int q = A.rp[i]; q < A.rp[i + 1]; q++) sm[i * n + A.ci[q]] = A.v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int e = 0; e < n * n; e++) m = fmax(m, fabs(sm[e]));
    amax_s = m;
    *sing = -1;
  }
  __syncthreads();
  for (int k = 0; k < n; k++) {
    if (threadIdx.x == 0) {
      int p = k;
      for (int i = k + 1; i < n; i++)
        if (fabs(sm[i * n + k]) > fabs(sm[p * n + k])) p = i;
      p_s = p;
      piv[k] = p;
      if (fabs(sm[p * n + k]) <= 1e-14 * amax_s && *sing < 0) *sing = k;
    }
    __syncthreads();
    int p = p_s;
    if (p != k)
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double t = sm[k * n + j];
        sm[k * n + j] = sm[p * n + j];
        sm[p * n + j] = t;
      }
    __syncthreads();
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) sm[i * n + k] = __ddiv_rn(sm[i * n + k], sm[k * n + k]);
    __syncthreads();
    for (int e = threadIdx.x; e < (n - k - 1) * (n - k - 1); e += blockDim.x) {
      int i = k + 1 + e / (n - k - 1), j = k + 1 + e % (n - k - 1);
      sm[i * n + j] = __dadd_rn(sm[i * n + j], -__dmul_rn(sm[i * n + k], sm[k * n + j]));
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) lu[e] = sm[e];
  __syncthreads();
  // explicit inverse (column j solved by thread j) so that the solve phase is one dense
  // matvec instead of 2n dependent substitution steps
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double *col = inv + (size_t)n * n;  // scratch column block: [n][blockDim] after inv
    double *y = col + (size_t)j * n;
    for (int i = 0; i < n; i++) y[i] = (i == j) ? 1.0 : 0.0;
    for (int k = 0; k < n; k++) {
      int p = piv[k];
      if (p != k) {
        double t = y[k];
        y[k] = y[p];
        y[p] = t;
      }
    }
    for (int k = 0; k < n; k++)
      for (int i = k + 1; i < n; i++) y[i] -= sm[i * n + k] * y[k];
    for (int k = n - 1; k >= 0; k--) {
      y[k] = y[k] / sm[k * n + k];
      for (int i = 0; i < k; i++) y[i] -= sm[i * n + k] * y[k];
    }
    for (int i = 0; i < n; i++) inv[(size_t)i * n + j] = y[i];
  }
}

// ------------------------------------------------------------------------------- driver
void free_hierarchy(bf_ctx *c, Hier &h) {
  for (int l = 0; l < h.nlev; l++) {
    Level &L = h.lv[l];
    free_csr(c, L.A);
    free_csr(c, L.P);
    free_csr(c, L.R);
    free_csr(c, L.Rf);
    free_csr(c, L.A_io);
    free_csr(c, L.P_io);
    dfree(c, L.perm);
    dfree(c, L.cf);
    dfree(c, L.dl1);
    dfree(c, L.b);
    dfree(c, L.x);
    dfree(c, L.r);
    dfree(c, L.t);
    dfree(c, L.d);
  }
  dfree(c, h.lu);
  dfree(c, h.piv);
  dfree(c, h.inv);
  dfree(c, h.tmat);
  h = Hier();
}

static void copy_csr(bf_ctx *c, const DCsr &A, DCsr &B) {
  B.n = A.n;
  B.m = A.m;
  B.nnz = A.nnz;
  B.rp = dalloc_t<int32_t>(c, (size_t)A.n + 1);
  B.ci = dalloc_t<int32_t>(c, A.nnz);
  B.v = dalloc_t<double>(c, A.nnz);
  BF_CUDA(cudaMemcpyAsync(B.rp, A.rp, sizeof(int32_t) * (A.n + 1), cudaMemcpyDeviceToDevice, c->stream));
  BF_CUDA(cudaMemcpyAsync(B.ci, A.ci, sizeof(int32_t) * A.nnz, cudaMemcpyDeviceToDevice, c->stream));
  BF_CUDA(cudaMemcpyAsync(B.v, A.v, sizeof(double) * A.nnz, cudaMemcpyDeviceToDevice, c->stream));
}

// ---------------------------------------------------------------------------------------
// Power-iteration estimate of rho(D_l1^-1 A) for the Chebyshev interval of a level (reading
// R21; the oracle's or_power_estimate): v_0 = hashed start vector / |.|, then k times
// w = D^-1 A v, lambda = |w|, v = w / lambda.  The norms are fixed-order two-level reductions
// (the same result run to run); against the oracle they differ only by summation order.
// ---------------------------------------------------------------------------------------
constexpr int POW_BLOCKS = 256;
static __global__ void k_pow_init(int n, uint64_t seed, int level, double *v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (double)h32(seed, level + 4096, i) / 4294967296.0 - 0.5;
}
static __global__ void k_pow_apply(DCsr A, const double *__restrict__ dl1, const double *__restrict__ v,
                                   double *__restrict__ w) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double s = 0.0;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) s += A.v[q] * v[A.ci[q]];
  w[i] = s / dl1[i];
}
static __global__ void __launch_bounds__(256) k_pow_partial(int n, const double *__restrict__ w, double *part) {
  __shared__ double sm[256];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += w[i] * w[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}
static __global__ void k_pow_norm(const double *__restrict__ part, double *nrm) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < POW_BLOCKS; b++) s += part[b];
    *nrm = sqrt(s);
  }
}
static __global__ void k_pow_scale(int n, const double *__restrict__ w, const double *__restrict__ nrm, double *v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double s = *nrm;
  if (i < n) v[i] = s > 0.0 ? w[i] / s : 0.0;
}

// Level::cheb_hi and Level::beta0 of every level of h (the Chebyshev interval, R21)
static void set_cheb_intervals(bf_ctx *c, Hier &h, int only_level = -1) {
  const bf_options &o = c->opt;
  std::vector<int> lv;
  for (int k = 0; k < h.nlev; k++)
    if (only_level < 0 || k == only_level) lv.push_back(k);
  bool any_cheb = false;
  for (int k : lv) any_cheb |= h.lv[k].smoother == 1;
  if (any_cheb && o.cheb_eig > 0) {
    double *nrm = dalloc_t<double>(c, 2 * lv.size() + 2);
    double *part = dalloc_t<double>(c, POW_BLOCKS);
    for (size_t q = 0; q < lv.size(); q++) {
      Level &L = h.lv[lv[q]];
      int n = L.A.n;
      double *v = dalloc_t<double>(c, n), *w = dalloc_t<double>(c, n);
      k_pow_init<<<div_up(n, 256), 256, 0, c->stream>>>(n, o.seed, lv[q], w);
      k_pow_partial<<<POW_BLOCKS, 256, 0, c->stream>>>(n, w, part);
      k_pow_norm<<<1, 32, 0, c->stream>>>(part, nrm + 2 * q);
      k_pow_scale<<<div_up(n, 256), 256, 0, c->stream>>>(n, w, nrm + 2 * q, v);
      for (int s = 0; s < o.cheb_eig; s++) {
        k_pow_apply<<<div_up(n, 256), 256, 0, c->stream>>>(L.A, L.dl1, v, w);
        k_pow_partial<<<POW_BLOCKS, 256, 0, c->stream>>>(n, w, part);
        k_pow_norm<<<1, 32, 0, c->stream>>>(part, nrm + 2 * q + 1);
        k_pow_scale<<<div_up(n, 256), 256, 0, c->stream>>>(n, w, nrm + 2 * q + 1, v);
      }
      c->launches += 4 + 4 * o.cheb_eig;
      dfree(c, v);
      dfree(c, w);
    }
    std::vector<double> hn(2 * lv.size() + 2);
    BF_CUDA(cudaMemcpyAsync(hn.data(), nrm, sizeof(double) * 2 * lv.size(), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    dfree(c, nrm);
    dfree(c, part);
    for (size_t q = 0; q < lv.size(); q++)
      if (h.lv[lv[q]].smoother == 1) h.lv[lv[q]].cheb_hi = 1.1 * hn[2 * q + 1];
  }
  for (int k : lv) set_level_beta(o, h.lv[k]);
}

// ---------------------------------------------------------------------------------------
// Renumbering of the coarse levels for gather locality (solve phase only).  A coarse point is
// a C point of the finer level; following the chain down gives the grid cell (x, y, z) it
// sits on.  Levels 1 .. L-1 (not the finest, whose grid order the DIA kernels and the callers'
// vectors use, and not the coarsest, whose inverse is dense) are renumbered by the key
// (Morton code of (x / 8, y, z), x mod 8): runs of 8 x-neighbours stay contiguous (the
// finest level's P and R keep their coalesced gathers) and the y / z neighbours of a coarse row
// sit in nearby Morton blocks instead of whole coarse planes away -- measured on the C3
// hierarchies, distinct 128-B lines per warp-wide gather fall by 20-40 % on A_1, A_2, P_1, R_1.
// The operators are permuted (A' = Pi A Pi^T, P' = Pi_l P Pi_{l+1}^T, R' likewise, the inverse
// l1 diagonal gathered); the construction-order A and P stay for bf_get_level (A_io, P_io) so
// the hierarchy is still compared bit-exactly with the oracle.  A symmetric permutation changes
// no value of the V-cycle, only the summation order of its products.
// ---------------------------------------------------------------------------------------
static __device__ __forceinline__ uint64_t spread3(uint32_t v) {
  uint64_t x = v & 0x1fffff;
  x = (x | x << 32) & 0x1f00000000ffffULL;
  x = (x | x << 16) & 0x1f0000ff0000ffULL;
  x = (x | x << 8) & 0x100f00f00f00f00fULL;
  x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
  x = (x | x << 2) & 0x1249249249249249ULL;
  return x;
}
static __global__ void k_cell_init(int n, int shift, int32_t *cell) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cell[i] = i >> shift;  // hierarchy 3 (J as a scalar matrix): 2 points per cell
}
static __global__ void k_cell_coarsen(int n, const int8_t *__restrict__ cf, const int32_t *__restrict__ cmap,
                                      const int32_t *__restrict__ cell, int32_t *__restrict__ ccell) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && cf[i] == 1) ccell[cmap[i]] = cell[i];
}
static __global__ void k_is_c1(int n, const int8_t *__restrict__ cf, int32_t *f) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = cf[i] == 1;
}
static __global__ void k_morton_keys(int n, const int32_t *__restrict__ cell, int nx, int ny, uint64_t *key,
                                     int32_t *idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = cell[i];
  uint32_t x = c % nx, y = (c / nx) % ny, z = c / (nx * ny);
  key[i] = ((spread3(x >> 3) | spread3(y) << 1 | spread3(z) << 2) << 3) | (x & 7);
  idx[i] = i;
}
static __global__ void k_inverse_perm(int n, const int32_t *__restrict__ perm, int32_t *inv) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) inv[perm[i]] = i;
}
static __global__ void k_gather_d(int n, const int32_t *__restrict__ perm, const double *__restrict__ a, double *b) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[perm[i]];
}
// row lengths of B = rows `rperm` of A (new row i is old row rperm[i]; null: identity)
static __global__ void k_perm_count(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ rperm,
                                    int32_t *cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int r = rperm ? rperm[i] : i;
  cnt[i] = rp[r + 1] - rp[r];
}
// B row i = A row rperm[i] with columns mapped by cinv (null: identity), sorted ascending
static __global__ void k_perm_fill(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                   const double *__restrict__ v, const int32_t *__restrict__ rperm,
                                   const int32_t *__restrict__ cinv, const int32_t *__restrict__ brp, int32_t *bci,
                                   double *bv) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int r = rperm ? rperm[i] : i;
  int q0 = rp[r], len = rp[r + 1] - q0, o = brp[i];
  for (int e = 0; e < len; e++) {  // insertion sort by the new column index
    int col = cinv ? cinv[ci[q0 + e]] : ci[q0 + e];
    double val = v[q0 + e];
    int k = e;
    while (k > 0 && bci[o + k - 1] > col) {
      bci[o + k] = bci[o + k - 1];
      bv[o + k] = bv[o + k - 1];
      k--;
    }
    bci[o + k] = col;
    bv[o + k] = val;
  }
}

// the same with a warp per row: each entry's position is its rank among the row's new column
// indices (distinct within a row), from a shared-memory copy of the row; rows longer than
// PERM_WARP_MAX take the serial path above (flagged in `longrow`)
constexpr int PERM_WARP_MAX = 256;
static __global__ void __launch_bounds__(256) k_perm_fill_warp(int n, const int32_t *__restrict__ rp,
                                                               const int32_t *__restrict__ ci,
                                                               const double *__restrict__ v,
                                                               const int32_t *__restrict__ rperm,
                                                               const int32_t *__restrict__ cinv,
                                                               const int32_t *__restrict__ brp, int32_t *bci,
                                                               double *bv, int *longrow) {
  __shared__ int32_t cols[8][PERM_WARP_MAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + warp;
  if (i >= n) return;
  const int r = rperm ? rperm[i] : i;
  const int q0 = rp[r], len = rp[r + 1] - q0, o = brp[i];
  if (len > PERM_WARP_MAX) {
    if (lane == 0) *longrow = 1;
    return;
  }
  int32_t *sc = cols[warp];
  for (int e = lane; e < len; e += 32) sc[e] = cinv ? cinv[ci[q0 + e]] : ci[q0 + e];
  __syncwarp();
  for (int e = lane; e < len; e += 32) {
    const int col = sc[e];
    int rank = 0;
    for (int k = 0; k < len; k++) rank += sc[k] < col;
    if (!BF_CHK(rank < len)) continue;
    bci[o + rank] = col;
    bv[o + rank] = v[q0 + e];
  }
}

// thread per row for the interpolation-like matrices (mean row length <= 4; a warp per row leaves
// 30 lanes idle there): rows of up to 8 entries are ranked in registers, longer ones are
// insertion-sorted in place like k_perm_fill
static __global__ void __launch_bounds__(256) k_perm_fill_short(int n, const int32_t *__restrict__ rp,
                                                                const int32_t *__restrict__ ci,
                                                                const double *__restrict__ v,
                                                                const int32_t *__restrict__ rperm,
                                                                const int32_t *__restrict__ cinv,
                                                                const int32_t *__restrict__ brp, int32_t *bci,
                                                                double *bv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = rperm ? rperm[i] : i;
  const int q0 = rp[r], len = rp[r + 1] - q0, o = brp[i];
  if (len <= 8) {
    int col[8];
    double val[8];
#pragma unroll
    for (int e = 0; e < 8; e++)
      if (e < len) {
        int cc = ci[q0 + e];
        col[e] = cinv ? cinv[cc] : cc;
        val[e] = v[q0 + e];
      }
#pragma unroll
    for (int e = 0; e < 8; e++)
      if (e < len) {
        int rank = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) rank += (k < len && col[k] < col[e]);
        if (!BF_CHK(rank < len)) continue;
        bci[o + rank] = col[e];
        bv[o + rank] = val[e];
      }
    return;
  }
  for (int e = 0; e < len; e++) {  // insertion sort by the new column index
    int col = cinv ? cinv[ci[q0 + e]] : ci[q0 + e];
    double val = v[q0 + e];
    int k = e;
    while (k > 0 && bci[o + k - 1] > col) {
      bci[o + k] = bci[o + k - 1];
      bv[o + k] = bv[o + k - 1];
      k--;
    }
    bci[o + k] = col;
    bv[o + k] = val;
  }
}

static void permute_csr(bf_ctx *c, const DCsr &A, const int32_t *rperm, const int32_t *cinv, DCsr &B) {
  B = DCsr();
  B.n = A.n;
  B.m = A.m;
  int32_t *cnt = dalloc_t<int32_t>(c, (size_t)A.n + 1);
  k_perm_count<<<div_up(A.n, 256), 256, 0, c->stream>>>(A.n, A.rp, rperm, cnt);
  B.rp = dalloc_t<int32_t>(c, (size_t)A.n + 1);
  B.nnz = exclusive_scan_i32(c, cnt, B.rp, A.n);
  dfree(c, cnt);
  B.ci = dalloc_t<int32_t>(c, B.nnz);
  B.v = dalloc_t<double>(c, B.nnz);
  if ((double)A.nnz <= 4.0 * (double)A.n) {
    k_perm_fill_short<<<div_up(A.n, 256), 256, 0, c->stream>>>(A.n, A.rp, A.ci, A.v, rperm, cinv, B.rp, B.ci, B.v);
    c->launches += 2;
    BF_CUDA(cudaGetLastError());
    return;
  }
  int *longrow = dalloc_t<int>(c, 1);
  BF_CUDA(cudaMemsetAsync(longrow, 0, sizeof(int), c->stream));
  k_perm_fill_warp<<<div_up(A.n, 8), 256, 0, c->stream>>>(A.n, A.rp, A.ci, A.v, rperm, cinv, B.rp, B.ci, B.v,
                                                          longrow);
  int hl = 0;
  BF_CUDA(cudaMemcpyAsync(&hl, longrow, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, longrow);
  if (hl)  // a row longer than the warp kernel's buffer: the serial kernel redoes every row
    k_perm_fill<<<div_up(A.n, 128), 128, 0, c->stream>>>(A.n, A.rp, A.ci, A.v, rperm, cinv, B.rp, B.ci, B.v);
  c->launches += 2 + hl;
  BF_CUDA(cudaGetLastError());
}

static void reorder_levels(bf_ctx *c, int which, Hier &h) {
  const int64_t ncell = (int64_t)c->nx * c->ny * c->nz;
  const int shift = which == 3 ? 1 : 0;
  // levels 1 .. last are renumbered: not the coarsest, and not the small latency-bound levels
  // (below 16K rows nothing is gained and every renumbered level costs setup time)
  int last = h.nlev - 2;
  while (last >= 1 && h.lv[last].A.n < 16384) last--;
  if (!c->tune.reorder || last < 1 || c->nx <= 0 || ((int64_t)h.lv[0].A.n >> shift) != ncell ||
      (shift && (h.lv[0].A.n & 1)))
    return;
  // grid cell of every point, level by level
  std::vector<int32_t *> cell(h.nlev, nullptr);
  cell[0] = dalloc_t<int32_t>(c, h.lv[0].A.n);
  k_cell_init<<<div_up(h.lv[0].A.n, 256), 256, 0, c->stream>>>(h.lv[0].A.n, shift, cell[0]);
  for (int l = 0; l < last; l++) {
    int n = h.lv[l].A.n;
    int32_t *f = dalloc_t<int32_t>(c, n), *cmap = dalloc_t<int32_t>(c, (size_t)n + 1);
    k_is_c1<<<div_up(n, 256), 256, 0, c->stream>>>(n, h.lv[l].cf, f);
    exclusive_scan_i32(c, f, cmap, n);
    cell[l + 1] = dalloc_t<int32_t>(c, h.lv[l + 1].A.n);
    k_cell_coarsen<<<div_up(n, 256), 256, 0, c->stream>>>(n, h.lv[l].cf, cmap, cell[l], cell[l + 1]);
    c->launches += 3;
    dfree(c, f);
    dfree(c, cmap);
  }
  // permutations (new -> old) and their inverses
  std::vector<int32_t *> inv(h.nlev, nullptr);
  for (int l = 1; l <= last; l++) {
    int n = h.lv[l].A.n;
    uint64_t *key = dalloc_t<uint64_t>(c, n);
    int32_t *perm = dalloc_t<int32_t>(c, n);
    k_morton_keys<<<div_up(n, 256), 256, 0, c->stream>>>(n, cell[l], c->nx, c->ny, key, perm);
    c->launches++;
    sort_pairs_u64_i32(c, key, perm, n, 64);
    dfree(c, key);
    inv[l] = dalloc_t<int32_t>(c, n);
    k_inverse_perm<<<div_up(n, 256), 256, 0, c->stream>>>(n, perm, inv[l]);
    c->launches++;
    h.lv[l].perm = perm;
  }
  for (int l = 0; l < h.nlev; l++) dfree(c, cell[l]);
  // permuted operators; the construction-order A and P are kept for introspection
  for (int l = 0; l <= last; l++) {
    Level &L = h.lv[l];
    const int32_t *rp_l = l >= 1 ? L.perm : nullptr, *ri_l = l >= 1 ? inv[l] : nullptr;
    const int32_t *rp_c = l + 1 <= last ? h.lv[l + 1].perm : nullptr;
    const int32_t *ri_c = l + 1 <= last ? inv[l + 1] : nullptr;
    if (l >= 1) {
      DCsr An;
      permute_csr(c, L.A, rp_l, ri_l, An);
      L.A_io = L.A;
      L.A_io.rpt = L.A_io.cap = 0;
      L.A = An;
      tile_csr(c, L.A, false);
      double *dn = dalloc_t<double>(c, L.A.n);
      k_gather_d<<<div_up(L.A.n, 256), 256, 0, c->stream>>>(L.A.n, L.perm, L.d, dn);
      c->launches++;
      dfree(c, L.d);
      L.d = dn;
    }
    DCsr Pn, Rn;
    permute_csr(c, L.P, rp_l, ri_c, Pn);
    permute_csr(c, L.R, rp_c, ri_l, Rn);
    L.P_io = L.P;
    L.P_io.rpt = L.P_io.cap = 0;
    L.P = Pn;
    free_csr(c, L.R);
    L.R = Rn;
    tile_csr(c, L.P, false, c->tune.tma_g_p);
    tile_csr(c, L.R, false, c->tune.tma_g_r);
  }
  for (int l = 0; l < h.nlev; l++) dfree(c, inv[l]);
  BF_CUDA(cudaGetLastError());
}

void build_hierarchy(bf_ctx *c, int which, const DCsr &A0) {
  Hier &h = c->h[which];
  const bf_options &o = c->opt;
  h.smoother = hier_smoother(o, which);
  copy_csr(c, A0, h.lv[0].A);
  int l = 0;
  int *nU_d = dalloc_t<int>(c, 4);
  const bool verbose = c->tune.verbose;
  auto tnow = [&]() {
    if (verbose) sync(c);
    return std::chrono::steady_clock::now();
  };
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  while (h.lv[l].A.n > o.max_coarse && l < o.max_levels - 1 && l < BF_MAXL - 1) {
    auto t0 = tnow();
    Level &L = h.lv[l];
    DCsr &A = L.A;
    int n = A.n;
    double *diag = dalloc_t<double>(c, n);
    k_diag<<<div_up(n, 256), 256, 0, c->stream>>>(A, diag);
    BF_LAUNCH(c);
    uint8_t *strong = dalloc_t<uint8_t>(c, A.nnz);
    k_strength<<<div_up(n, 256), 256, 0, c->stream>>>(A, diag, o.theta, strong);
    BF_LAUNCH(c);
    // PMIS
    int *lam = dalloc_t<int>(c, n);
    BF_CUDA(cudaMemsetAsync(lam, 0, sizeof(int) * n, c->stream));
    auto t1 = tnow();
    k_lambda<<<div_up(n, 256), 256, 0, c->stream>>>(A, strong, lam);
    BF_LAUNCH(c);
    uint64_t *key = dalloc_t<uint64_t>(c, n);
    int8_t *state = dalloc_t<int8_t>(c, n);
    k_pmis_init<<<div_up(n, 256), 256, 0, c->stream>>>(n, lam, o.seed, l, key, state);
    BF_LAUNCH(c);
    uint8_t *notmax = dalloc_t<uint8_t>(c, n);
    uint8_t *notmax1 = dalloc_t<uint8_t>(c, n);
    {
      const int coop_blocks = std::max(1, occupancy(c, (const void *)k_pmis_coop, 256, 0)) * c->num_sms;
      int grid = std::max(1, std::min(coop_blocks, div_up(n, 256)));
      int max_rounds = n + 1;  // each round decides at least the undecided point of largest key
      int *rounds_d = nU_d + 2;
      void *args[] = {(void *)&A, (void *)&strong, (void *)&key, (void *)&state, (void *)&notmax, (void *)&notmax1,
                      (void *)&nU_d, (void *)&max_rounds, (void *)&rounds_d};
      BF_CUDA(cudaLaunchCooperativeKernel((void *)k_pmis_coop, grid, 256, args, 0, c->stream));
      BF_LAUNCH(c);
      int hr[3] = {0, 0, 0};
      BF_CUDA(cudaMemcpyAsync(hr, nU_d, sizeof(hr), cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      if (hr[2] > max_rounds) throw Error(BF_ERR_LIMIT, "PMIS did not terminate");
      if (c->tune.verbose) fprintf(stderr, "[bf_setup]   PMIS n=%d: %d rounds, grid %d x 256\n", n, hr[2], grid);
    }
    dfree(c, notmax);
    dfree(c, notmax1);
    dfree(c, key);
    dfree(c, lam);
    // coarse numbering
    int32_t *flag = dalloc_t<int32_t>(c, n);
    k_is_c<<<div_up(n, 256), 256, 0, c->stream>>>(n, state, flag);
    BF_LAUNCH(c);
    int32_t *cmap = dalloc_t<int32_t>(c, (size_t)n + 1);
    int64_t nc = exclusive_scan_i32(c, flag, cmap, n);
    dfree(c, flag);
    if (nc == 0 || nc == n) {  // stop conditions (c.2 step 3.7)
      dfree(c, cmap);
      dfree(c, state);
      dfree(c, strong);
      dfree(c, diag);
      break;
    }
    L.cf = state;
    // interpolation
    int32_t *cnt = dalloc_t<int32_t>(c, n);
    auto t2 = tnow();
    k_interp_count<<<div_up(n, 256), 256, 0, c->stream>>>(A, strong, state, cnt);
    BF_LAUNCH(c);
    L.P.n = n;
    L.P.m = (int)nc;
    L.P.rp = dalloc_t<int32_t>(c, (size_t)n + 1);
    L.P.nnz = exclusive_scan_i32(c, cnt, L.P.rp, n);
    dfree(c, cnt);
    L.P.ci = dalloc_t<int32_t>(c, L.P.nnz);
    L.P.v = dalloc_t<double>(c, L.P.nnz);
    {
      uint8_t *long_rows = dalloc_t<uint8_t>(c, n);
      int *any_long = dalloc_t<int>(c, 1);
      int h_long = 1;
      if ((double)A.nnz / n > c->tune.interp_warp_min) {  // long (Galerkin) rows: warp per row; short rows: thread per row
        BF_CUDA(cudaMemsetAsync(long_rows, 0, n, c->stream));
        BF_CUDA(cudaMemsetAsync(any_long, 0, sizeof(int), c->stream));
        const int iw_grid = std::max(1, std::min(div_up(n, IW_WARPS), 4 * c->num_sms * std::max(1, occupancy(c, (const void *)k_interp_warp, IW_WARPS * 32, 0))));
        k_interp_warp<<<iw_grid, IW_WARPS * 32, 0, c->stream>>>(A, strong, state, cmap, diag,
                                                                           o.interp_norm, L.P, long_rows, any_long);
        BF_LAUNCH(c);
        BF_CUDA(cudaMemcpyAsync(&h_long, any_long, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        sync(c);
      } else {
        BF_CUDA(cudaMemsetAsync(long_rows, 1, n, c->stream));
      }
      if (h_long) {
        k_interp_fill<<<div_up(n, 128), 128, 0, c->stream>>>(A, strong, state, cmap, diag, o.interp_norm, L.P,
                                                             long_rows);
        BF_LAUNCH(c);
      }
      dfree(c, long_rows);
      dfree(c, any_long);
    }
    BF_LAUNCH(c);
    BF_CUDA(cudaGetLastError());
    dfree(c, cmap);
    dfree(c, strong);
    dfree(c, diag);
    auto t3 = tnow();
    transpose(c, L.P, L.R);
    auto t4 = tnow();
    DCsr AP;
    spgemm(c, A, L.P, AP);
    auto t5 = tnow();
    spgemm(c, L.R, AP, h.lv[l + 1].A);
    auto t6 = tnow();
    if (verbose)
      fprintf(stderr,
              "[bf_setup]   h%d L%d n=%d nnz=%lld: strength %.2f pmis %.2f interp %.2f transpose %.2f AP %.2f RAP %.2f ms\n",
              which, l, n, (long long)A.nnz, ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), ms(t5, t6));
    free_csr(c, AP);
    if (o.diag_stop && which != 3) {  // R23: coarsening stops before a Galerkin level with a non-positive (or missing) diagonal entry;
       // level l then is the coarsest level (stalled-coarsening rule: dense LU or 4 l1-Jacobi sweeps)
      DCsr &Ac = h.lv[l + 1].A;
      int *bad_d = nU_d + 3;
      BF_CUDA(cudaMemsetAsync(bad_d, 0, sizeof(int), c->stream));
      k_diag_nonpos<<<div_up(Ac.n, 256), 256, 0, c->stream>>>(Ac, bad_d);
      BF_LAUNCH(c);
      int bad = 0;
      BF_CUDA(cudaMemcpyAsync(&bad, bad_d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      if (bad) {
        if (verbose) fprintf(stderr, "[bf_setup]   h%d L%d: Galerkin diagonal not positive, coarsening stops (R23)\n", which, l + 1);
        free_csr(c, Ac);
        free_csr(c, L.P);
        free_csr(c, L.R);
        dfree(c, L.cf);
        L.cf = nullptr;
        break;
      }
    }
    l++;
  }
  dfree(c, nU_d);
  h.nlev = l + 1;
  for (int k = 0; k < h.nlev; k++) {
    Level &L = h.lv[k];
    L.smoother = (h.smoother == 1 && (o.cheb_levels == 0 || k < o.cheb_levels)) ? 1 : 0;  // R22
    int n = L.A.n;
    double *diag = dalloc_t<double>(c, n);
    k_diag<<<div_up(n, 256), 256, 0, c->stream>>>(L.A, diag);
    L.dl1 = dalloc_t<double>(c, n);
    k_l1diag<<<div_up(n, 256), 256, 0, c->stream>>>(L.A, diag, L.dl1);
    L.d = dalloc_t<double>(c, n);
    k_recip<<<div_up(n, 256), 256, 0, c->stream>>>(n, L.dl1, L.d);
    c->launches += 3;
    dfree(c, diag);
    L.b = dalloc_t<double>(c, n);
    L.x = dalloc_t<double>(c, n);
    L.r = dalloc_t<double>(c, n);
    L.t = dalloc_t<double>(c, n);
    tile_csr(c, L.A, k == 0);
    if (k == 0) setup_dia(c, L.A);
    if (k < h.nlev - 1) {
      tile_csr(c, L.P, false, c->tune.tma_g_p);
      tile_csr(c, L.R, false, c->tune.tma_g_r);
    }
  }
  BF_CUDA(cudaGetLastError());
  Level &C = h.lv[l];
  h.nL = C.A.n;
  h.dense = C.A.n <= o.max_coarse;
  if (h.dense) {
    int nL = C.A.n;
    h.lu = dalloc_t<double>(c, (size_t)nL * nL);
    h.piv = dalloc_t<int32_t>(c, nL);
    h.inv = dalloc_t<double>(c, (size_t)2 * nL * nL);  // inverse + per-column scratch
    int *sing = dalloc_t<int>(c, 1);
    size_t smem = sizeof(double) * nL * nL;
    BF_CUDA(cudaFuncSetAttribute(k_coarse_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
    k_coarse_lu<<<1, 256, smem, c->stream>>>(C.A, h.lu, h.piv, h.inv, sing);
    BF_LAUNCH(c);
    BF_CUDA(cudaGetLastError());
    int hs = -1;
    BF_CUDA(cudaMemcpyAsync(&hs, sing, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    dfree(c, sing);
    if (hs >= 0)
      throw Error(BF_ERR_COARSE_SINGULAR, std::string("coarsest matrix of hierarchy ") + std::to_string(which) +
                                              " (n=" + std::to_string(nL) + ") singular at pivot " +
                                              std::to_string(hs));
  }
  set_cheb_intervals(c, h);
  reorder_levels(c, which, h);
  plan_tail(c, h);
  build_dense_tail(c, h);
  build_rfuse(c, h, false);
  build_windows(c, h);
}

// ---------------------------------------------------------------------------------------
// Fused restriction of the pre-smoothed residual.  With one l1-Jacobi pre-sweep from zero the
// V-cycle's first two steps on level l are x0 = beta D b, r = b - A x0, and the restriction
// b_c = R r = R (I - beta A D) b, D = diag(1/dl1).  Rf = R M with M = I - beta A D (the
// pattern of A: the diagonal is structurally present) turns "residual + restriction" into ONE
// sparse product over b.  Mathematically identical to the two-step form (the rounding order
// differs; the V-cycle parity tolerance covers it), and it reads nnz(Rf) instead of
// nnz(A) + nnz(R) and the r round trip.  Built for the CSR levels above the tail (the finest
// level's DIA residual + restriction is cheaper per byte), default smoother configuration only.
// ---------------------------------------------------------------------------------------
static __global__ void k_rfuse_m(DCsr A, const double *__restrict__ d, double beta, double *__restrict__ mv) {
  int i = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (i >= A.n) return;
  for (int q = A.rp[i] + lane; q < A.rp[i + 1]; q += 32) {
    int j = A.ci[q];
    double t = (beta * A.v[q]) * d[j];
    mv[q] = (j == i ? 1.0 : 0.0) - t;
  }
}

void build_rfuse(bf_ctx *c, Hier &h, bool finest_only) {
  const bf_options &o = c->opt;
  if (!c->tune.rfuse || o.nu_pre != 1) return;
  const bool l0 = c->tune.rfuse_l0;
  int lend = h.dtail >= 0 ? h.dtail : (h.tail >= 0 ? h.tail : h.nlev - 1);
  for (int l = l0 ? 0 : 1; l < lend; l++) {
    if (finest_only && l > 0) break;
    Level &L = h.lv[l];
    free_csr(c, L.Rf);
    if (L.A.dia_v && !l0) continue;
    if (L.smoother != 0) continue;  // Rf fuses ONE l1-Jacobi pre-sweep from zero
    DCsr M;
    M.n = L.A.n;
    M.m = L.A.m;
    M.nnz = L.A.nnz;
    M.rp = L.A.rp;
    M.ci = L.A.ci;
    M.v = dalloc_t<double>(c, L.A.nnz);
    k_rfuse_m<<<div_up((int64_t)M.n * 32, 256), 256, 0, c->stream>>>(L.A, L.d, 1.0, M.v);
    BF_LAUNCH(c);
    auto t0 = std::chrono::steady_clock::now();
    spgemm(c, L.R, M, L.Rf);
    dfree(c, M.v);
    tile_csr(c, L.Rf, false);
    if (c->tune.verbose) {
      sync(c);
      fprintf(stderr, "[bf_setup]   rfuse L%d: R %lld nnz x M %lld nnz -> %lld nnz, %.2f ms\n", l, (long long)L.R.nnz,
              (long long)L.A.nnz, (long long)L.Rf.nnz,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
  }
  BF_CUDA(cudaGetLastError());
}

// Setup reuse (bf_update, reading R16): replace the finest matrix of hierarchy `which` by
// A0 and refresh its l1 diagonal, inverse diagonal and tiling; coarse levels are kept.
void refresh_finest(bf_ctx *c, int which, const DCsr &A0) {
  Hier &h = c->h[which];
  if (h.nlev <= 1) {  // the finest level is the coarsest: rebuild (dense LU of the new matrix)
    free_hierarchy(c, h);
    build_hierarchy(c, which, A0);
    return;
  }
  Level &L = h.lv[0];
  free_csr(c, L.A);
  copy_csr(c, A0, L.A);
  int n = L.A.n;
  double *diag = dalloc_t<double>(c, n);
  k_diag<<<div_up(n, 256), 256, 0, c->stream>>>(L.A, diag);
  k_l1diag<<<div_up(n, 256), 256, 0, c->stream>>>(L.A, diag, L.dl1);
  k_recip<<<div_up(n, 256), 256, 0, c->stream>>>(n, L.dl1, L.d);
  c->launches += 3;
  BF_CUDA(cudaGetLastError());
  dfree(c, diag);
  tile_csr(c, L.A, true);
  setup_dia(c, L.A);
  set_cheb_intervals(c, h, 0);
  plan_tail(c, h);
  if (h.lv[0].Rf.n) build_rfuse(c, h, true);  // the finest level's fused restriction uses A_0
}

}  // namespace bf
