// k_ilu.cu -- the two-stage CPR preconditioners of PAPER.md:
//   Algorithm 1, CPR-AMG(1) (combinative), and Algorithm 2, CPR-AMG(2) (additive), P:L159-193:
//     u = P_1^-1 r                       P_1 = block ILU(0) of J (reading R18)
//     t = r - J u
//     A_pp dp = R_p t                     one AMG V-cycle (hierarchy 2)
//    [A_ss ds = R_s t                     one AMG V-cycle (hierarchy 0), Algorithm 2 only]
//     z = u + R_p^T dp [+ R_s^T ds]
//
// ILU(0) on the GPU.  The factorization and both triangular solves follow the row
// dependencies of J's block pattern in its natural (point) order -- the same ILU(0) as the
// oracle, not a reordered one.  Rows are grouped by dependency level (level(i) = 1 + max
// level of the rows it depends on; i+j+k on a 7-point grid, 3*128-2 levels at 128^3) and
// processed by ONE persistent "sync-free" kernel per sweep: warps take 32 consecutive rows of
// the level-sorted order from an atomic ticket, every lane polls the completion flags of its
// row's dependencies (acquire loads), computes its row once they are all set, publishes the
// row (release store of the flag).  A warp only waits on rows with smaller tickets, which were
// taken by warps already resident, so the scheme cannot deadlock; lanes poll inside a
// warp-uniform loop, so no lane ever blocks another.
//
// Determinism: every factor value is computed by one thread in the oracle's order with the
// multiply and add rounded separately (this TU is built with --fmad=false), so the factors
// are bit-identical to or_ilu0 (determinism contract); the solves use the same
// ascending order per row.
//
// Roofline: the solves are HBM/latency bound (each moves J's blocks once: 36 B/block plus
// vectors) but their critical path is the number of levels times one L2 round trip.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>

#include "bf_internal.cuh"
BF_CHECK_TU("k_ilu.cu")

namespace bf {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned *p) {
  return *reinterpret_cast<const volatile unsigned *>(p);
}

// next 32 rows of the schedule for this warp (ticket shared by the whole grid)
__device__ __forceinline__ unsigned warp_ticket(unsigned *ticket) {
  unsigned base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(ticket, 32u);
  return __shfl_sync(FULL, base, 0);
}

// ---- setup: dependency levels, schedule, diagonal positions ---------------------------
// level[i] (init -1) doubles as the completion flag; rows in natural order
__global__ void k_ilu_levels(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, int *level,
                             unsigned *ticket) {
  for (;;) {
    unsigned base = warp_ticket(ticket);
    if (base >= (unsigned)n) return;
    int i = base + (threadIdx.x & 31);
    bool done = i >= n;
    int lo = done ? 0 : rp[i], hi = done ? 0 : rp[i + 1];
    [[maybe_unused]] unsigned spins = 0;  // checked build: a dependency that never completes is reported
    while (!__all_sync(FULL, done)) {
      if (!BF_SPIN_OK(spins)) done = true;
      if (!done) {
        int lev = 0;
        bool ready = true;
        for (int q = lo; q < hi; q++) {
          int k = ci[q];
          if (k >= i) break;
          int lk = ld_acquire(level + k);
          if (lk < 0) {
            ready = false;
            break;
          }
          lev = max(lev, lk + 1);
        }
        if (ready) {
          st_release(level + i, lev);
          done = true;
        }
      }
    }
  }
}

__global__ void k_ilu_keys(int n, const int *__restrict__ level, const int32_t *__restrict__ rp,
                           const int32_t *__restrict__ ci, uint64_t *keys, int32_t *dpos) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ((uint64_t)(uint32_t)level[i] << 32) | (uint32_t)i;
  int d = -1;
  for (int q = rp[i]; q < rp[i + 1]; q++)
    if (ci[q] == i) d = q;
  dpos[i] = d;
}

__global__ void k_ilu_perm(int n, const uint64_t *__restrict__ keys, int32_t *perm) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) perm[t] = (int32_t)(keys[t] & 0xffffffffu);
}

// ---- setup: numeric factorization (oracle or_ilu0) ------------------------------
// 2x2 products entry (r,c) = A_r0 B_0c + A_r1 B_1c (no FMA: --fmad=false)
struct B2 {
  double a, b, c, d;  // row-major {b00, b01, b10, b11}
};
__device__ __forceinline__ B2 ldg_blk(const double *p) {  // another row's finished block (L2)
  double2 x = __ldcg(reinterpret_cast<const double2 *>(p));
  double2 y = __ldcg(reinterpret_cast<const double2 *>(p) + 1);
  return {x.x, x.y, y.x, y.y};
}
__device__ __forceinline__ B2 ld_blk(const double *p) {
  double2 x = reinterpret_cast<const double2 *>(p)[0];
  double2 y = reinterpret_cast<const double2 *>(p)[1];
  return {x.x, x.y, y.x, y.y};
}
__device__ __forceinline__ void st_blk(double *p, B2 v) {
  reinterpret_cast<double2 *>(p)[0] = make_double2(v.a, v.b);
  reinterpret_cast<double2 *>(p)[1] = make_double2(v.c, v.d);
}
__device__ __forceinline__ B2 mul(B2 A, B2 B) {
  return {A.a * B.a + A.b * B.c, A.a * B.b + A.b * B.d, A.c * B.a + A.d * B.c, A.c * B.b + A.d * B.d};
}

__global__ void k_ilu_factor(int n, const int32_t *__restrict__ perm, const int32_t *__restrict__ rp,
                             const int32_t *__restrict__ ci, const int32_t *__restrict__ dpos, double *lu,
                             double *dinv, int *flag, unsigned *ticket, int *bad) {
  for (;;) {
    unsigned base = warp_ticket(ticket);
    if (base >= (unsigned)n) return;
    unsigned t = base + (threadIdx.x & 31);
    bool done = t >= (unsigned)n;
    int i = done ? 0 : perm[t];
    int lo = done ? 0 : rp[i], hi = done ? 0 : rp[i + 1], di = done ? 0 : dpos[i];
    [[maybe_unused]] unsigned spins = 0;  // checked build: a dependency that never completes is reported
    while (!__all_sync(FULL, done)) {
      if (!BF_SPIN_OK(spins)) done = true;
      if (!done) {
        bool ready = true;
        for (int q = lo; q < di && ready; q++) ready = ld_acquire(flag + ci[q]) != 0;
        if (ready) {
          for (int q = lo; q < di; q++) {  // k < i ascending
            int k = ci[q];
            B2 L = mul(ld_blk(lu + 4 * (size_t)q), ldg_blk(dinv + 4 * (size_t)k));  // a_ik a_kk^-1
            st_blk(lu + 4 * (size_t)q, L);
            int u = dpos[k] + 1, ue = rp[k + 1];
            for (int s = q + 1; s < hi; s++) {  // j > k in row i; (k, j) in row k's upper part
              int j = ci[s];
              while (u < ue && __ldcg(ci + u) < j) u++;
              if (u == ue) break;
              if (__ldcg(ci + u) != j) continue;
              B2 P = mul(L, ldg_blk(lu + 4 * (size_t)u));
              B2 A = ld_blk(lu + 4 * (size_t)s);
              st_blk(lu + 4 * (size_t)s, {A.a - P.a, A.b - P.b, A.c - P.c, A.d - P.d});
            }
          }
          B2 D = ld_blk(lu + 4 * (size_t)di);
          double det = D.a * D.d - D.b * D.c;
          if (det == 0.0 || !isfinite(det)) atomicMin(bad, i);
          st_blk(dinv + 4 * (size_t)i, {D.d / det, -D.b / det, -D.c / det, D.a / det});
          __threadfence();
          st_release(flag + i, 1);
          done = true;
        }
      }
    }
  }
}

// ---- solve: y = L^-1 r (forward), x = U^-1 y (backward) ---------------------------------
// Sync state shared by the two sweeps: tickets are reset by the other sweep's last warp, the
// flag targets are 2e+1 (forward) and 2e+2 (backward) of the epoch e, advanced by the last
// warp of the backward sweep -- no memset between applies, graph-capturable.
struct IluSync {
  unsigned ticket[2];
  unsigned done[2];
  unsigned epoch;
  unsigned pad[3];
};

__device__ __forceinline__ void sweep_exit(IluSync *sy, int which) {
  if ((threadIdx.x & 31) != 0) return;
  unsigned nw = gridDim.x * (blockDim.x >> 5);
  __threadfence();
  if (atomicAdd(&sy->done[which], 1u) == nw - 1) {
    sy->done[which] = 0;
    sy->ticket[1 - which] = 0;  // the other sweep is not running (stream order)
    if (which == 1) sy->epoch = sy->epoch + 1;
    __threadfence();
  }
}

// Up to PF dependency entries of a row (column and 2x2 block) are loaded into registers BEFORE
// polling: they do not depend on other rows, so only the dependencies' results remain on the
// critical path (one L2 round trip per level).  Rows with more entries load the rest on the fly.
constexpr int PF = 4;

struct DepCache {
  int col[PF];
  double2 b01[PF], b23[PF];
};
__device__ __forceinline__ void dep_prefetch(DepCache &dc, int lo, int hi, const int32_t *__restrict__ ci,
                                             const double *__restrict__ lu) {
#pragma unroll
  for (int e = 0; e < PF; e++) {
    if (lo + e < hi) {
      int q = lo + e;
      dc.col[e] = __ldg(ci + q);
      dc.b01[e] = __ldg(reinterpret_cast<const double2 *>(lu) + 2 * (size_t)q);
      dc.b23[e] = __ldg(reinterpret_cast<const double2 *>(lu) + 2 * (size_t)q + 1);
    }
  }
}
__device__ __forceinline__ bool deps_ready(const DepCache &dc, int lo, int hi, const int32_t *__restrict__ ci,
                                           const int *flag, int target) {
  bool ready = true;
#pragma unroll
  for (int e = 0; e < PF; e++)
    if (lo + e < hi) ready = ready && ld_acquire(flag + dc.col[e]) == target;
  for (int q = lo + PF; q < hi && ready; q++) ready = ld_acquire(flag + __ldg(ci + q)) == target;
  return ready;
}
// t -= sum_q B_q v[col_q], ascending q (the oracle's order)
__device__ __forceinline__ void dep_subtract(const DepCache &dc, int lo, int hi, const int32_t *__restrict__ ci,
                                             const double *__restrict__ lu, const double2 *v, double &t0,
                                             double &t1) {
#pragma unroll
  for (int e = 0; e < PF; e++) {
    if (lo + e < hi) {
      double2 vk = __ldcg(v + dc.col[e]);
      t0 = t0 - (dc.b01[e].x * vk.x + dc.b01[e].y * vk.y);
      t1 = t1 - (dc.b23[e].x * vk.x + dc.b23[e].y * vk.y);
    }
  }
  for (int q = lo + PF; q < hi; q++) {
    double2 b01 = __ldg(reinterpret_cast<const double2 *>(lu) + 2 * (size_t)q);
    double2 b23 = __ldg(reinterpret_cast<const double2 *>(lu) + 2 * (size_t)q + 1);
    double2 vk = __ldcg(v + __ldg(ci + q));
    t0 = t0 - (b01.x * vk.x + b01.y * vk.y);
    t1 = t1 - (b23.x * vk.x + b23.y * vk.y);
  }
}

// r: caller-ordered interleaved vector (v_j of GMRES); nrm2 != null: r is the unnormalised
// basis slot with ||r||^2 = *nrm2 and is normalised here, in place (the BF split kernel's job
// on the BF path).  y: canonical (p, s) pairs.  y_i = r_i - sum_{k<i} L_ik y_k.
__global__ void __launch_bounds__(256) k_ilu_fwd(int n, const int32_t *__restrict__ perm,
                                                 const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                 const int32_t *__restrict__ dpos, const double *__restrict__ lu,
                                                 double2 *r, const double *nrm2, double2 *y, int *flag,
                                                 IluSync *sy, int ip) {
  const int target = 2 * (int)ld_volatile_u32(&sy->epoch) + 1;
  const double sc = nrm2 ? 1.0 / sqrt(*nrm2) : 1.0;
  for (;;) {
    unsigned base = warp_ticket(&sy->ticket[0]);
    if (base >= (unsigned)n) break;
    unsigned t = base + (threadIdx.x & 31);
    bool done = t >= (unsigned)n;
    int i = done ? 0 : __ldg(perm + t);
    int lo = done ? 0 : __ldg(rp + i), di = done ? 0 : __ldg(dpos + i);
    DepCache dc;
    dep_prefetch(dc, lo, di, ci, lu);
    double y0 = 0.0, y1 = 0.0;
    if (!done) {
      double2 a = r[i];
      if (nrm2) {
        a.x = a.x * sc;
        a.y = a.y * sc;
        r[i] = a;
      }
      y0 = ip ? a.y : a.x;
      y1 = ip ? a.x : a.y;
    }
    [[maybe_unused]] unsigned spins = 0;  // checked build: a dependency that never completes is reported
    while (!__all_sync(FULL, done)) {
      if (!BF_SPIN_OK(spins)) done = true;
      if (!done && deps_ready(dc, lo, di, ci, flag, target)) {
        dep_subtract(dc, lo, di, ci, lu, y, y0, y1);
        y[i] = make_double2(y0, y1);
        __threadfence();
        st_release(flag + i, target);
        done = true;
      }
    }
  }
  sweep_exit(sy, 0);
}

// x (canonical) = U^-1 y:  x_i = D_i^-1 (y_i - sum_{j>i} U_ij x_j)
__global__ void __launch_bounds__(256) k_ilu_bwd(int n, const int32_t *__restrict__ perm,
                                                 const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                 const int32_t *__restrict__ dpos, const double *__restrict__ lu,
                                                 const double *__restrict__ dinv, const double2 *y, double2 *x,
                                                 int *flag, IluSync *sy) {
  const int target = 2 * (int)ld_volatile_u32(&sy->epoch) + 2;
  for (;;) {
    unsigned base = warp_ticket(&sy->ticket[1]);
    if (base >= (unsigned)n) break;
    unsigned t = base + (threadIdx.x & 31);
    bool done = t >= (unsigned)n;
    int i = done ? 0 : __ldg(perm + (n - 1 - (int)t));
    int lo = done ? 0 : __ldg(dpos + i) + 1, hi = done ? 0 : __ldg(rp + i + 1);
    DepCache dc;
    dep_prefetch(dc, lo, hi, ci, lu);
    double t0 = 0.0, t1 = 0.0;
    double2 d01 = make_double2(0.0, 0.0), d23 = d01;
    if (!done) {
      double2 yi = __ldcg(y + i);
      t0 = yi.x;
      t1 = yi.y;
      d01 = __ldg(reinterpret_cast<const double2 *>(dinv) + 2 * (size_t)i);
      d23 = __ldg(reinterpret_cast<const double2 *>(dinv) + 2 * (size_t)i + 1);
    }
    [[maybe_unused]] unsigned spins = 0;  // checked build: a dependency that never completes is reported
    while (!__all_sync(FULL, done)) {
      if (!BF_SPIN_OK(spins)) done = true;
      if (!done && deps_ready(dc, lo, hi, ci, flag, target)) {
        dep_subtract(dc, lo, hi, ci, lu, x, t0, t1);
        x[i] = make_double2(d01.x * t0 + d01.y * t1, d23.x * t0 + d23.y * t1);
        __threadfence();
        st_release(flag + i, target);
        done = true;
      }
    }
  }
  sweep_exit(sy, 1);
}

// ---- value-flag variant of the sweeps (default) -------------------------------------------
// The result itself is the completion flag: every entry of y and x holds a sentinel NaN bit
// pattern (never produced by arithmetic) until its row publishes it, so a consumer's poll
// returns the dependency's value -- no separate flag, no fence, one L2 round trip per level on
// the critical path instead of three.  The consumers that read a row's result for the last
// time restore the sentinel: the backward sweep for y (its own row), the CPR merge /
// k_to_caller for x.  A computed value equal to the sentinel is replaced by the canonical NaN.
constexpr unsigned long long SENT = 0x7FF4DEADBEEF0001ull;
__device__ __forceinline__ double2 ld_poll(const double2 *p) {
  double a, b;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p) : "memory");
  return make_double2(a, b);
}
__device__ __forceinline__ void st_pub(double2 *p, double2 v) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ bool is_sent(double v) { return (unsigned long long)__double_as_longlong(v) == SENT; }
__device__ __forceinline__ bool ready2(double2 v) { return !is_sent(v.x) && !is_sent(v.y); }
__device__ __forceinline__ double unsent(double v) {
  return is_sent(v) ? __longlong_as_double(0x7FFFFFFFFFFFFFFFll) : v;
}
__device__ __forceinline__ double2 sent2() {
  return make_double2(__longlong_as_double((long long)SENT), __longlong_as_double((long long)SENT));
}

// poll every dependency once; on success vals[] holds the first PF dependencies' results
__device__ __forceinline__ bool vdeps_ready(const DepCache &dc, int lo, int hi, const int32_t *__restrict__ ci,
                                            const double2 *v, double2 *vals) {
  bool ready = true;
#pragma unroll
  for (int e = 0; e < PF; e++)
    if (lo + e < hi) {
      vals[e] = ld_poll(v + dc.col[e]);
      ready = ready && ready2(vals[e]);
    }
  for (int q = lo + PF; q < hi && ready; q++) ready = ready2(ld_poll(v + __ldg(ci + q)));
  return ready;
}
__device__ __forceinline__ void vdep_subtract(const DepCache &dc, int lo, int hi, const int32_t *__restrict__ ci,
                                              const double *__restrict__ lu, const double2 *v, const double2 *vals,
                                              double &t0, double &t1) {
#pragma unroll
  for (int e = 0; e < PF; e++) {
    if (lo + e < hi) {
      double2 vk = vals[e];
      t0 = t0 - (dc.b01[e].x * vk.x + dc.b01[e].y * vk.y);
      t1 = t1 - (dc.b23[e].x * vk.x + dc.b23[e].y * vk.y);
    }
  }
  for (int q = lo + PF; q < hi; q++) {
    double2 b01 = __ldg(reinterpret_cast<const double2 *>(lu) + 2 * (size_t)q);
    double2 b23 = __ldg(reinterpret_cast<const double2 *>(lu) + 2 * (size_t)q + 1);
    double2 vk = ld_poll(v + __ldg(ci + q));
    t0 = t0 - (b01.x * vk.x + b01.y * vk.y);
    t1 = t1 - (b23.x * vk.x + b23.y * vk.y);
  }
}

__global__ void __launch_bounds__(256) k_ilu_fwd_v(int n, const int32_t *__restrict__ perm,
                                                   const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                   const int32_t *__restrict__ dpos, const double *__restrict__ lu,
                                                   double2 *r, const double *nrm2, double2 *y, int *unused,
                                                   IluSync *sy, int ip, unsigned backoff) {
  const double sc = nrm2 ? 1.0 / sqrt(*nrm2) : 1.0;
  for (;;) {
    unsigned base = warp_ticket(&sy->ticket[0]);
    if (base >= (unsigned)n) break;
    unsigned t = base + (threadIdx.x & 31);
    bool done = t >= (unsigned)n;
    int i = done ? 0 : __ldg(perm + t);
    int lo = done ? 0 : __ldg(rp + i), di = done ? 0 : __ldg(dpos + i);
    DepCache dc;
    dep_prefetch(dc, lo, di, ci, lu);
    double y0 = 0.0, y1 = 0.0;
    if (!done) {
      double2 a = r[i];
      if (nrm2) {
        a.x = a.x * sc;
        a.y = a.y * sc;
        r[i] = a;
      }
      y0 = ip ? a.y : a.x;
      y1 = ip ? a.x : a.y;
    }
    [[maybe_unused]] unsigned spins = 0;  // checked build: a dependency that never completes is reported
    while (!__all_sync(FULL, done)) {
      if (!BF_SPIN_OK(spins)) done = true;
      double2 vals[PF];
      bool ok = !done && vdeps_ready(dc, lo, di, ci, y, vals);
      if (!done && !ok && backoff) __nanosleep(backoff);
      if (ok) {
        vdep_subtract(dc, lo, di, ci, lu, y, vals, y0, y1);
        st_pub(y + i, make_double2(unsent(y0), unsent(y1)));
        done = true;
      }
    }
  }
  sweep_exit(sy, 0);
}

__global__ void __launch_bounds__(256) k_ilu_bwd_v(int n, const int32_t *__restrict__ perm,
                                                   const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                   const int32_t *__restrict__ dpos, const double *__restrict__ lu,
                                                   const double *__restrict__ dinv, double2 *y, double2 *x,
                                                   int *unused, IluSync *sy, unsigned backoff) {
  for (;;) {
    unsigned base = warp_ticket(&sy->ticket[1]);
    if (base >= (unsigned)n) break;
    unsigned t = base + (threadIdx.x & 31);
    bool done = t >= (unsigned)n;
    int i = done ? 0 : __ldg(perm + (n - 1 - (int)t));
    int lo = done ? 0 : __ldg(dpos + i) + 1, hi = done ? 0 : __ldg(rp + i + 1);
    DepCache dc;
    dep_prefetch(dc, lo, hi, ci, lu);
    double t0 = 0.0, t1 = 0.0;
    double2 d01 = make_double2(0.0, 0.0), d23 = d01;
    if (!done) {
      double2 yi = __ldcg(y + i);
      y[i] = sent2();  // last read of y_i: restore the sentinel for the next forward sweep
      t0 = yi.x;
      t1 = yi.y;
      d01 = __ldg(reinterpret_cast<const double2 *>(dinv) + 2 * (size_t)i);
      d23 = __ldg(reinterpret_cast<const double2 *>(dinv) + 2 * (size_t)i + 1);
    }
    [[maybe_unused]] unsigned spins = 0;  // checked build: a dependency that never completes is reported
    while (!__all_sync(FULL, done)) {
      if (!BF_SPIN_OK(spins)) done = true;
      double2 vals[PF];
      bool ok = !done && vdeps_ready(dc, lo, hi, ci, x, vals);
      if (!done && !ok && backoff) __nanosleep(backoff);
      if (ok) {
        vdep_subtract(dc, lo, hi, ci, lu, x, vals, t0, t1);
        st_pub(x + i, make_double2(unsent(d01.x * t0 + d01.y * t1), unsent(d23.x * t0 + d23.y * t1)));
        done = true;
      }
    }
  }
  sweep_exit(sy, 1);
}

__global__ void k_fill_sent(size_t n2, double2 *a) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n2) a[i] = sent2();
}

// ---- pencil-wavefront sweeps for grid-structured J (default when the pattern is exactly the
// 5/7-point stencil of the nx x ny x nz grid in natural order) ----------------------------
// Row c = i + nx (j + ny k) depends on (i-1), (j-1), (k-1) in the forward sweep.  A CTA owns a
// tile of TJ x TK x-lines (j, k) and walks them as a local wavefront: at CTA step s, thread
// (jj, kk) computes cell i = s - jj - kk of its line, so its (j-1) and (k-1) dependencies are the
// neighbouring threads' results of step s-1 (shared memory) and its (i-1) dependency is its own
// previous result (register): one __syncthreads per step instead of one L2 round trip per
// dependency level.  Dependencies across tile faces are read from global memory with the
// value-flag protocol above (sentinel until published), prefetched one step ahead; tiles are
// taken from an atomic ticket in anti-diagonal order, so a CTA waits only on tiles already
// taken by resident CTAs (deadlock-free).  The backward sweep is the same walk mirrored
// (i, j, k -> n-1-i, ...) with the U blocks and the pivot inverse.  Factor blocks are read from a
// DIA copy (ld[d][c], ud[d][c]) so a thread's consecutive cells are consecutive in memory.
// Arithmetic order per row = ascending columns, as the oracle: forward (k-1), (j-1), (i-1);
// backward (i+1), (j+1), (k+1); results are bit-identical to the generic sweeps.
struct PencilGeom {
  int nx, ny, nz, TJ, TK, NJ, NK;
};

__global__ void k_grid_check(int n, int nx, int ny, int nz, const int32_t *__restrict__ rp,
                             const int32_t *__restrict__ ci, int *bad) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
  int want[7], m = 0;
  long sxy = (long)nx * ny;
  if (k > 0) want[m++] = c - (int)sxy;
  if (j > 0) want[m++] = c - nx;
  if (i > 0) want[m++] = c - 1;
  want[m++] = c;
  if (i < nx - 1) want[m++] = c + 1;
  if (j < ny - 1) want[m++] = c + nx;
  if (k < nz - 1) want[m++] = c + (int)sxy;
  int q0 = rp[c];
  bool ok = rp[c + 1] - q0 == m;
  for (int e = 0; ok && e < m; e++) ok = ci[q0 + e] == want[e];
  if (!ok) atomicExch(bad, 1);
}

// lu (CSR blocks) -> ld[3][n] (k-1, j-1, i-1) and ud[3][n] (i+1, j+1, k+1), zero where absent
__global__ void k_ilu_to_dia(int n, int nx, int ny, int nz, const int32_t *__restrict__ rp,
                             const double2 *__restrict__ lu, double2 *ld, double2 *ud) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
  bool has[7] = {k > 0, j > 0, i > 0, true, i < nx - 1, j < ny - 1, k < nz - 1};
  int q = rp[c];
  for (int e = 0; e < 7; e++) {
    double2 a = make_double2(0.0, 0.0), b = a;
    if (has[e]) {
      a = lu[2 * (size_t)q];
      b = lu[2 * (size_t)q + 1];
      q++;
    }
    if (e == 3) continue;
    double2 *dst = e < 3 ? ld + 2 * ((size_t)e * n + c) : ud + 2 * ((size_t)(e - 4) * n + c);
    dst[0] = a;
    dst[1] = b;
  }
}

// per-thread staging of one cell's inputs (cp.async, PD steps ahead): the input pair, three
// factor blocks, the pivot inverse (backward only)
constexpr int PD = 4;
struct Stage {
  double2 in;
  double2 f[6];
  double2 d[2];
};
__device__ __forceinline__ void cp16(void *smem, const void *gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <bool BWD, int XD>
__global__ void __launch_bounds__(128) k_ilu_pencil(PencilGeom g, const double2 *__restrict__ fac,
                                                    const double2 *__restrict__ dinv, double2 *in,
                                                    const double *nrm2, double2 *out, double2 *yreset,
                                                    const int2 *__restrict__ order, unsigned *ticket,
                                                    unsigned *done, unsigned *other_ticket, int ip, int lag,
                                                    unsigned backoff) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2 *sbuf = reinterpret_cast<double2 *>(smem_raw);                        // [2][TK][TJ]
  Stage *ring = reinterpret_cast<Stage *>(smem_raw + 2 * 128 * sizeof(double2));  // [PD][128]
  __shared__ unsigned s_tile;
  const int n = g.nx * g.ny * g.nz;
  const long sxy = (long)g.nx * g.ny;
  const int jj = threadIdx.x % g.TJ, kk = threadIdx.x / g.TJ;
  const bool thr = kk < g.TK;
  const double sc = (!BWD && nrm2) ? 1.0 / sqrt(*nrm2) : 1.0;
  const int ntiles = g.NJ * g.NK;
  const int nsteps = g.nx + g.TJ + g.TK - 2;
  const int dj = BWD ? g.nx : -g.nx;  // the (j-1) / (j+1) neighbour
  const long dk = BWD ? sxy : -sxy;   // the (k-1) / (k+1) neighbour
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    unsigned t = s_tile;
    if (t >= (unsigned)ntiles) break;
    int2 JK = order[t];
    // walk-frame coordinates (the backward sweep walks the mirrored grid)
    const int jw = JK.x * g.TJ + jj, kw = JK.y * g.TK + kk;
    const bool line = thr && jw < g.ny && kw < g.nz;
    const int j = BWD ? g.ny - 1 - jw : jw, k = BWD ? g.nz - 1 - kw : kw;
    const int base = g.nx * (j + g.ny * k);
    auto cell_of = [&](int s) -> int {
      int iw = s - jj - kk;
      if (!line || iw < 0 || iw >= g.nx) return -1;
      return base + (BWD ? g.nx - 1 - iw : iw);
    };
    auto issue = [&](int s) {  // stage step s's inputs into ring slot s % PD
      int c = cell_of(s);
      if (c >= 0) {
        Stage &st = ring[(s % PD) * 128 + threadIdx.x];
        cp16(&st.in, in + c);
#pragma unroll
        for (int d = 0; d < 3; d++) {
          cp16(&st.f[2 * d], fac + 2 * ((size_t)d * n + c));
          cp16(&st.f[2 * d + 1], fac + 2 * ((size_t)d * n + c) + 1);
        }
        if (BWD) {
          cp16(&st.d[0], dinv + 2 * (size_t)c);
          cp16(&st.d[1], dinv + 2 * (size_t)c + 1);
        }
      }
      cp_commit();
    };
#pragma unroll
    for (int s = 0; s < PD - 1; s++) issue(s);
    double2 prev = make_double2(0.0, 0.0);
    // cross-tile dependencies (threads on the tile's jj = 0 / kk = 0 faces) are loaded two steps
    // before use: the neighbouring tile runs ahead, so the value is usually already published
    // and the L2 round trip leaves the critical path; a sentinel falls back to polling.  The
    // step loop is unrolled by two so each prefetch slot is a fixed register pair (a select on
    // the step parity would make the thread wait for the load immediately).
    auto xfetch = [&](int s, double2 &pk, double2 &pj) {
      int c = cell_of(s);
      pk = sent2();
      pj = sent2();
      if (c >= 0) {
        if (kw > 0 && kk == 0) pk = ld_poll(out + (c + dk));
        if (jw > 0 && jj == 0) pj = ld_poll(out + (c + dj));
      }
    };
    double2 pk0, pk1, pj0, pj1, pk2, pj2, pk3, pj3;
    // optional start lag: face threads first wait until the neighbouring tile has published the
    // cell `lag` positions ahead of their first dependency, so the two-step prefetch finds
    // published values (the tiles then run with that slack)
    if (lag > 0 && line) {
      int iw = min(lag, g.nx - 1);
      int c = base + (BWD ? g.nx - 1 - iw : iw);
      if (kw > 0 && kk == 0)
        for (unsigned spins = 0; !ready2(ld_poll(out + (c + dk))) && BF_SPIN_OK(spins);) __nanosleep(backoff);
      if (jw > 0 && jj == 0)
        for (unsigned spins = 0; !ready2(ld_poll(out + (c + dj))) && BF_SPIN_OK(spins);) __nanosleep(backoff);
    }
    xfetch(0, pk0, pj0);
    xfetch(1, pk1, pj1);
    if (XD == 4) {
      xfetch(2, pk2, pj2);
      xfetch(3, pk3, pj3);
    }
    auto step = [&](int s, double2 &pk, double2 &pj) {
      issue(s + PD - 1);
      cp_wait<PD - 1>();
      int c = cell_of(s);
      double2 res = make_double2(0.0, 0.0);
      if (c >= 0) {
        const Stage &st = ring[(s % PD) * 128 + threadIdx.x];
        const int iw = s - jj - kk;
        double t0, t1;
        double2 a = st.in;
        if (!BWD) {
          if (nrm2) {
            a.x = a.x * sc;
            a.y = a.y * sc;
            in[c] = a;
          }
          t0 = ip ? a.y : a.x;
          t1 = ip ? a.x : a.y;
        } else {
          yreset[c] = sent2();  // last read of y_c
          t0 = a.x;
          t1 = a.y;
        }
        double2 vk = make_double2(0.0, 0.0), vj = vk;
        const bool hk = kw > 0, hj = jw > 0, hi = iw > 0;
        if (hk) {
          if (kk > 0) {
            vk = sbuf[((s - 1) & 1) * 128 + (kk - 1) * g.TJ + jj];
          } else {
            vk = pk;
            [[maybe_unused]] unsigned spins = 0;
            while (!ready2(vk) && BF_SPIN_OK(spins)) {  // not yet published: back off so waiting tiles do not flood L2
              __nanosleep(backoff);
              vk = ld_poll(out + (c + dk));
            }
          }
        }
        if (hj) {
          if (jj > 0) {
            vj = sbuf[((s - 1) & 1) * 128 + kk * g.TJ + jj - 1];
          } else {
            vj = pj;
            [[maybe_unused]] unsigned spins = 0;
            while (!ready2(vj) && BF_SPIN_OK(spins)) {
              __nanosleep(backoff);
              vj = ld_poll(out + (c + dj));
            }
          }
        }
        auto sub = [&](int slot, double2 v) {
          double2 b01 = st.f[2 * slot], b23 = st.f[2 * slot + 1];
          t0 = t0 - (b01.x * v.x + b01.y * v.y);
          t1 = t1 - (b23.x * v.x + b23.y * v.y);
        };
        if (!BWD) {  // ascending columns: (k-1), (j-1), (i-1)
          if (hk) sub(0, vk);
          if (hj) sub(1, vj);
          if (hi) sub(2, prev);
          res = make_double2(unsent(t0), unsent(t1));
        } else {  // ascending columns: (i+1), (j+1), (k+1)
          if (hi) sub(0, prev);
          if (hj) sub(1, vj);
          if (hk) sub(2, vk);
          res = make_double2(unsent(st.d[0].x * t0 + st.d[0].y * t1), unsent(st.d[1].x * t0 + st.d[1].y * t1));
        }
        st_pub(out + c, res);
        prev = res;
      }
      if (thr) sbuf[(s & 1) * 128 + kk * g.TJ + jj] = res;
      xfetch(s + XD, pk, pj);  // this slot's next use is step s + XD
      __syncthreads();
    };
    if (XD == 4) {
      for (int s = 0; s < nsteps; s += 4) {
        step(s, pk0, pj0);
        if (s + 1 < nsteps) step(s + 1, pk1, pj1);
        if (s + 2 < nsteps) step(s + 2, pk2, pj2);
        if (s + 3 < nsteps) step(s + 3, pk3, pj3);
      }
    } else {
      for (int s = 0; s < nsteps; s += 2) {
        step(s, pk0, pj0);
        if (s + 1 < nsteps) step(s + 1, pk1, pj1);
      }
    }
    cp_wait<0>();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0;
      *other_ticket = 0;
      __threadfence();
    }
  }
}
constexpr int PXD = 2;  // cross-tile prefetch distance (steps): 2 (measured: 4 is slower, 0.89 vs 1.00 ms)
constexpr size_t kPencilSmem = 2 * 128 * sizeof(double2) + (size_t)PD * 128 * sizeof(Stage);

// ---- CPR: t = r - J u, split into the right-hand sides of the inner V-cycles --------------
// (Alg. 1/2 steps 3-4[-5]); writes the level invariant of vcycle_level: b and x0 = beta b ./ dl1.
// J from its DIA copy when present (coalesced), else the CSR-BSR rows.
struct JDia {
  int k;
  int off[8];
};
__global__ void __launch_bounds__(256) k_cpr_resid(int n, const int32_t *__restrict__ rp,
                                                   const int32_t *__restrict__ ci, const double2 *__restrict__ bv,
                                                   const double2 *__restrict__ jd, JDia o,
                                                   const double2 *__restrict__ u, const double2 *__restrict__ r,
                                                   double *__restrict__ bp, double *__restrict__ xp,
                                                   const double *__restrict__ dp, double *__restrict__ bs,
                                                   double *__restrict__ xs, const double *__restrict__ ds,
                                                   double beta_p, double beta_s, int ip) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double w0 = 0.0, w1 = 0.0;
  if (jd) {
#pragma unroll
    for (int d = 0; d < 8; d++) {
      int col = i + o.off[d];
      if (d < o.k && col >= 0 && col < n) {
        size_t e = ((size_t)d * n + i) * 2;
        double2 v01 = __ldcs(jd + e), v23 = __ldcs(jd + e + 1);
        double2 uc = __ldg(u + col);
        w0 += v01.x * uc.x + v01.y * uc.y;
        w1 += v23.x * uc.x + v23.y * uc.y;
      }
    }
  } else {
    for (int q = __ldg(rp + i); q < __ldg(rp + i + 1); q++) {
      double2 v01 = __ldcs(bv + 2 * (size_t)q), v23 = __ldcs(bv + 2 * (size_t)q + 1);
      double2 uc = __ldg(u + __ldg(ci + q));
      w0 += v01.x * uc.x + v01.y * uc.y;
      w1 += v23.x * uc.x + v23.y * uc.y;
    }
  }
  double2 ri = r[i];
  double tp = (ip ? ri.y : ri.x) - w0, ts = (ip ? ri.x : ri.y) - w1;
  bp[i] = tp;
  xp[i] = beta_p * (tp * dp[i]);
  if (bs) {
    bs[i] = ts;
    xs[i] = beta_s * (ts * ds[i]);
  }
}

// z = u + R_p^T dp [+ R_s^T ds] in the caller's var_order (Alg. 1 step 5 / Alg. 2 step 6)
__global__ void k_cpr_merge(int n, double2 *__restrict__ u, const double *__restrict__ dp,
                            const double *__restrict__ ds, double2 *__restrict__ z, int ip) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 a = u[i];
  u[i] = sent2();  // last read of u_i (value-flag sweeps)
  double p = a.x + dp[i], s = ds ? a.y + ds[i] : a.y;
  z[i] = ip ? make_double2(s, p) : make_double2(p, s);
}

// ---- host side -------------------------------------------------------------------------
// CTAs of 256 threads per SM for the persistent sweeps (Tuning::ilu_ctas)
static int ilu_grid(bf_ctx *c) { return c->num_sms * c->tune.ilu_ctas; }

// grid-structured J (exactly the 5/7-point stencil in natural order): DIA copies of the factors
// and the tile geometry of the pencil-wavefront sweeps (BF_ILU_PENCIL=0 keeps the generic ones)
static void setup_pencil(bf_ctx *c) {
  int n = c->n;
  if (!c->ilu_pencil_checked) {
    c->ilu_pencil_checked = true;
    if (!c->tune.ilu_pencil || c->tune.ilu_flags || (int64_t)c->nx * c->ny * c->nz != n) return;
    int *bad = dalloc_t<int>(c, 1);
    BF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    k_grid_check<<<div_up(n, 256), 256, 0, c->stream>>>(n, c->nx, c->ny, c->nz, c->brp, c->bci, bad);
    BF_LAUNCH(c);
    int hb = 0;
    BF_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    dfree(c, bad);
    if (hb) return;
    PencilGeom g;
    g.nx = c->nx;
    g.ny = c->ny;
    g.nz = c->nz;
    g.TK = std::min(c->nz, c->tune.pencil_tk);
    g.TJ = std::min(c->ny, c->tune.pencil_tj > 0 ? c->tune.pencil_tj : 128 / g.TK);
    if (g.TK < 1 || g.TJ < 1 || g.TJ * g.TK > 128) throw Error(BF_ERR_ARG, "pencil tile TJ*TK must be in [1, 128]");
    g.NJ = div_up(c->ny, g.TJ);
    g.NK = div_up(c->nz, g.TK);
    std::vector<int2> ord;
    for (int d = 0; d <= g.NJ + g.NK - 2; d++)  // anti-diagonals: every tile after its (J-1) and (K-1) neighbours
      for (int J = 0; J < g.NJ; J++) {
        int K = d - J;
        if (K >= 0 && K < g.NK) ord.push_back(make_int2(J, K));
      }
    c->ilu_order = dalloc_t<int2>(c, ord.size());
    BF_CUDA(cudaMemcpyAsync(c->ilu_order, ord.data(), sizeof(int2) * ord.size(), cudaMemcpyHostToDevice, c->stream));
    c->ilu_geom[0] = g.nx; c->ilu_geom[1] = g.ny; c->ilu_geom[2] = g.nz;
    c->ilu_geom[3] = g.TJ; c->ilu_geom[4] = g.TK; c->ilu_geom[5] = g.NJ; c->ilu_geom[6] = g.NK;
    c->ilu_ld = dalloc_t<double>(c, 12 * (size_t)n);
    c->ilu_ud = dalloc_t<double>(c, 12 * (size_t)n);
    ensure_smem_attr((const void *)k_ilu_pencil<false, PXD>, (int)kPencilSmem);
    ensure_smem_attr((const void *)k_ilu_pencil<true, PXD>, (int)kPencilSmem);
    c->ilu_pencil = true;
    sync(c);
  }
  if (!c->ilu_pencil) return;
  k_ilu_to_dia<<<div_up(n, 256), 256, 0, c->stream>>>(n, c->nx, c->ny, c->nz, c->brp,
                                                       reinterpret_cast<const double2 *>(c->ilu_lu),
                                                       reinterpret_cast<double2 *>(c->ilu_ld),
                                                       reinterpret_cast<double2 *>(c->ilu_ud));
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

void build_ilu(bf_ctx *c) {
  int n = c->n;
  int64_t nnzb = c->nnzb;
  if (!c->ilu_perm) {  // schedule (pattern only; kept across bf_update)
    int *level = dalloc_t<int>(c, n);
    unsigned *tk = dalloc_t<unsigned>(c, 4);
    BF_CUDA(cudaMemsetAsync(level, 0xff, sizeof(int) * n, c->stream));
    BF_CUDA(cudaMemsetAsync(tk, 0, sizeof(unsigned) * 4, c->stream));
    k_ilu_levels<<<ilu_grid(c), 256, 0, c->stream>>>(n, c->brp, c->bci, level, tk);
    uint64_t *keys = dalloc_t<uint64_t>(c, n), *keys2 = dalloc_t<uint64_t>(c, n);
    c->ilu_dpos = dalloc_t<int32_t>(c, n);
    k_ilu_keys<<<div_up(n, 256), 256, 0, c->stream>>>(n, level, c->brp, c->bci, keys, c->ilu_dpos);
    cub::DoubleBuffer<uint64_t> kb(keys, keys2);
    size_t tmp = 0;
    BF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kb, n, 0, 64, c->stream));
    void *tb = dalloc(c, tmp + 16);
    BF_CUDA(cub::DeviceRadixSort::SortKeys(tb, tmp, kb, n, 0, 64, c->stream));
    c->ilu_perm = dalloc_t<int32_t>(c, n);
    k_ilu_perm<<<div_up(n, 256), 256, 0, c->stream>>>(n, kb.Current(), c->ilu_perm);
    c->launches += 6;
    BF_CUDA(cudaGetLastError());
    int maxlev = 0;
    BF_CUDA(cudaMemcpyAsync(&maxlev, reinterpret_cast<const char *>(kb.Current() + (n - 1)) + 4, sizeof(int),
                            cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    c->ilu_levels = maxlev + 1;
    dfree(c, tb);
    dfree(c, keys);
    dfree(c, keys2);
    dfree(c, level);
    dfree(c, tk);
    c->ilu_flag = dalloc_t<int>(c, n);
    c->ilu_sync = dalloc_t<unsigned>(c, sizeof(IluSync) / sizeof(unsigned));
    c->ilu_lu = dalloc_t<double>(c, 4 * (size_t)nnzb);
    c->ilu_dinv = dalloc_t<double>(c, 4 * (size_t)n);
    c->ilu_y = dalloc_t<double>(c, 2 * (size_t)n);
    c->ilu_u = dalloc_t<double>(c, 2 * (size_t)n);
    c->ilu_vflag = !c->tune.ilu_flags;
    k_fill_sent<<<div_up(n, 256), 256, 0, c->stream>>>((size_t)n, reinterpret_cast<double2 *>(c->ilu_y));
    k_fill_sent<<<div_up(n, 256), 256, 0, c->stream>>>((size_t)n, reinterpret_cast<double2 *>(c->ilu_u));
    c->launches += 2;
  }
  // numeric factorization (oracle or_ilu0 order)
  int *flag = dalloc_t<int>(c, n);
  unsigned *tk = dalloc_t<unsigned>(c, 4);
  int *bad = dalloc_t<int>(c, 1);
  BF_CUDA(cudaMemsetAsync(flag, 0, sizeof(int) * n, c->stream));
  BF_CUDA(cudaMemsetAsync(tk, 0, sizeof(unsigned) * 4, c->stream));
  BF_CUDA(cudaMemcpyAsync(bad, &n, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  BF_CUDA(cudaMemcpyAsync(c->ilu_lu, c->bv, sizeof(double) * 4 * (size_t)nnzb, cudaMemcpyDeviceToDevice,
                          c->stream));
  k_ilu_factor<<<ilu_grid(c), 256, 0, c->stream>>>(n, c->ilu_perm, c->brp, c->bci, c->ilu_dpos, c->ilu_lu,
                                                   c->ilu_dinv, flag, tk, bad);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  int hb = n;
  BF_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaMemsetAsync(c->ilu_flag, 0, sizeof(int) * n, c->stream));
  BF_CUDA(cudaMemsetAsync(c->ilu_sync, 0, sizeof(IluSync), c->stream));
  sync(c);
  dfree(c, flag);
  dfree(c, tk);
  dfree(c, bad);
  if (hb < n)
    throw Error(BF_ERR_ZERO_DIAG, "ILU(0) pivot block singular at cell " + std::to_string(hb));
  setup_pencil(c);
}

// u = (L U)^-1 r (canonical output in c->ilu_u); r in the caller's order, normalised in place
// when nrm2 is given
static void ilu_solve(bf_ctx *c, double *r, const double *nrm2) {
  int n = c->n;
  IluSync *sy = reinterpret_cast<IluSync *>(c->ilu_sync);
  // polling backoff (ns) and start lag of the sweeps: measured neutral / slower, off
  const unsigned backoff = 0u;
  if (c->ilu_pencil) {
    PencilGeom g{c->ilu_geom[0], c->ilu_geom[1], c->ilu_geom[2], c->ilu_geom[3], c->ilu_geom[4], c->ilu_geom[5],
                 c->ilu_geom[6]};
    int grid = std::min(g.NJ * g.NK, c->num_sms * 2);
    const int lag = 0;
    const unsigned pbackoff = 0u;
    k_ilu_pencil<false, PXD><<<grid, 128, kPencilSmem, c->stream>>>(
        g, reinterpret_cast<const double2 *>(c->ilu_ld), nullptr, reinterpret_cast<double2 *>(r), nrm2,
        reinterpret_cast<double2 *>(c->ilu_y), nullptr, c->ilu_order, &sy->ticket[0], &sy->done[0], &sy->ticket[1],
        c->var_order, lag, pbackoff);
    k_ilu_pencil<true, PXD><<<grid, 128, kPencilSmem, c->stream>>>(
        g, reinterpret_cast<const double2 *>(c->ilu_ud), reinterpret_cast<const double2 *>(c->ilu_dinv),
        reinterpret_cast<double2 *>(c->ilu_y), nullptr, reinterpret_cast<double2 *>(c->ilu_u),
        reinterpret_cast<double2 *>(c->ilu_y), c->ilu_order, &sy->ticket[1], &sy->done[1], &sy->ticket[0], 0, lag, pbackoff);
  } else if (c->ilu_vflag) {
    k_ilu_fwd_v<<<ilu_grid(c), 256, 0, c->stream>>>(n, c->ilu_perm, c->brp, c->bci, c->ilu_dpos, c->ilu_lu,
                                                    reinterpret_cast<double2 *>(r), nrm2,
                                                    reinterpret_cast<double2 *>(c->ilu_y), c->ilu_flag, sy,
                                                    c->var_order, backoff);
    k_ilu_bwd_v<<<ilu_grid(c), 256, 0, c->stream>>>(n, c->ilu_perm, c->brp, c->bci, c->ilu_dpos, c->ilu_lu,
                                                    c->ilu_dinv, reinterpret_cast<double2 *>(c->ilu_y),
                                                    reinterpret_cast<double2 *>(c->ilu_u), c->ilu_flag, sy, backoff);
  } else {
    k_ilu_fwd<<<ilu_grid(c), 256, 0, c->stream>>>(n, c->ilu_perm, c->brp, c->bci, c->ilu_dpos, c->ilu_lu,
                                                  reinterpret_cast<double2 *>(r), nrm2,
                                                  reinterpret_cast<double2 *>(c->ilu_y), c->ilu_flag, sy,
                                                  c->var_order);
    k_ilu_bwd<<<ilu_grid(c), 256, 0, c->stream>>>(n, c->ilu_perm, c->brp, c->bci, c->ilu_dpos, c->ilu_lu,
                                                  c->ilu_dinv, reinterpret_cast<const double2 *>(c->ilu_y),
                                                  reinterpret_cast<double2 *>(c->ilu_u), c->ilu_flag, sy);
  }
  c->launches += 2;
  BF_CUDA(cudaGetLastError());
}

void vcycle_from_invariant(bf_ctx *c, int which);  // k_vcycle.cu

void amg_apply(bf_ctx *c, const double *v, double *z, const double *nrm2);

void cpr_apply(bf_ctx *c, const double *v, double *z, const double *nrm2) {
  if (c->opt.precond == 3) {
    amg_apply(c, v, z, nrm2);
    return;
  }
  int n = c->n;
  Hier &hp = c->h[2], &hs = c->h[0];
  bool additive = c->opt.precond == 2;
  ilu_solve(c, const_cast<double *>(v), nrm2);  // step 2
  JDia o{};
  o.k = c->jdia ? c->jdia_k : 0;
  for (int d = 0; d < o.k; d++) o.off[d] = c->jdia_off[d];
  k_cpr_resid<<<div_up(n, 256), 256, 0, c->stream>>>(
      n, c->brp, c->bci, reinterpret_cast<const double2 *>(c->bv), reinterpret_cast<const double2 *>(c->jdia), o,
      reinterpret_cast<const double2 *>(c->ilu_u), reinterpret_cast<const double2 *>(v), hp.lv[0].b, hp.lv[0].x,
      hp.lv[0].d, additive ? hs.lv[0].b : nullptr, additive ? hs.lv[0].x : nullptr,
      additive ? hs.lv[0].d : nullptr, hp.lv[0].beta0, additive ? hs.lv[0].beta0 : 1.0, c->var_order);  // step 3
  BF_LAUNCH(c);
  vcycle_from_invariant(c, 2);  // step 4
  if (additive) vcycle_from_invariant(c, 0);  // Alg. 2 step 5
  k_cpr_merge<<<div_up(n, 256), 256, 0, c->stream>>>(n, reinterpret_cast<double2 *>(c->ilu_u), hp.lv[0].x,
                                                     additive ? hs.lv[0].x : nullptr,
                                                     reinterpret_cast<double2 *>(z), c->var_order);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

__global__ void k_to_caller(int n, double2 *__restrict__ u, double2 *__restrict__ x, int ip) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 a = u[i];
  u[i] = sent2();  // last read of u_i (value-flag sweeps)
  x[i] = ip ? make_double2(a.y, a.x) : a;
}

// introspection (bf_ilu_solve): x = (L U)^-1 r, both in the caller's var_order
void ilu_solve_into(bf_ctx *c, const double *r, double *x) {
  if (!c->ilu_lu) throw Error(BF_ERR_ARG, "bf_ilu_solve: the handle has no ILU(0) (precond 0)");
  ilu_solve(c, const_cast<double *>(r), nullptr);
  k_to_caller<<<div_up(c->n, 256), 256, 0, c->stream>>>(c->n, reinterpret_cast<double2 *>(c->ilu_u),
                                                         reinterpret_cast<double2 *>(x), c->var_order);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

// graph patching (k_vcycle.cu bf_apply_graph): which kernel arguments carry v, nrm2 and z
bool amg_patch_roles(const void *func, int &nargs, std::vector<std::pair<int, int>> &roles);

bool cpr_patch_roles(const void *func, int &nargs, std::vector<std::pair<int, int>> &roles) {
  if (amg_patch_roles(func, nargs, roles)) return true;
  if (func == (const void *)k_ilu_fwd) {
    nargs = nargs_of(k_ilu_fwd);
    roles = {{6, 0}, {7, 1}};
  } else if (func == (const void *)k_ilu_fwd_v) {
    nargs = nargs_of(k_ilu_fwd_v);
    roles = {{6, 0}, {7, 1}};
  } else if (func == (const void *)k_ilu_pencil<false, PXD>) {
    nargs = nargs_of(k_ilu_pencil<false, PXD>);
    roles = {{3, 0}, {4, 1}};
  } else if (func == (const void *)k_cpr_resid) {
    nargs = nargs_of(k_cpr_resid);
    roles = {{7, 0}};
  } else if (func == (const void *)k_cpr_merge) {
    nargs = nargs_of(k_cpr_merge);
    roles = {{4, 2}};
  } else {
    return false;
  }
  return true;
}

// algorithmic bytes of one CPR apply: ILU solves (J's blocks once: 36 B/block + row_ptr,
// diagonal position, dinv 32 B, vectors r, y (w + r), x (w + r): 8+4+32+64 B/row), the
// residual (a J SpMV, 36 nnzb + 36 n, + b/x0 outputs and 1/dl1 24 B per field), the V-cycles
// (SURVEY 8(d) per-level model), the merge (u, dp[, ds], z)
double cpr_model_bytes(bf_ctx *c) {
  double n = c->n, nnzb = (double)c->nnzb;
  if (c->opt.precond == 3) {  // split 48 n (v in, b and x0 out, 1/dl1 in -- 2n each) + merge 32 n + V-cycle
    Hier &h = c->h[3];
    double bytes = 96.0 * n;
    for (int l = 0; l + 1 < h.nlev; l++)
      bytes += 24.0 * h.lv[l].A.nnz + 24.0 * h.lv[l].P.nnz + 116.0 * h.lv[l].A.n + 12.0 * h.lv[l + 1].A.n;
    return bytes + 8.0 * h.nL * h.nL;
  }
  bool additive = c->opt.precond == 2;
  double bytes = 36.0 * nnzb + 108.0 * n;
  bytes += 36.0 * nnzb + 36.0 * n + (additive ? 48.0 : 24.0) * n;
  bytes += (additive ? 40.0 : 32.0) * n;
  for (int w : {2, 0}) {
    if (w == 0 && !additive) continue;
    Hier &h = c->h[w];
    for (int l = 0; l + 1 < h.nlev; l++)
      bytes += 24.0 * h.lv[l].A.nnz + 24.0 * h.lv[l].P.nnz + 116.0 * h.lv[l].A.n + 12.0 * h.lv[l + 1].A.n;
    bytes += 8.0 * h.nL * h.nL;
  }
  return bytes;
}


// ======================================================================================
// Coupled "point" AMG (precond 3; the paper's AMG comparison, reading R20):
// one V-cycle of the scalar AMG on J itself, interleaved (point-ordered) as a 2n x 2n CSR.
// ======================================================================================
// scalar row 2c+r of J: entries (r, s) of the row's blocks that are not +-0.0, plus the diagonal
__global__ void k_jsc_count(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                            const double *__restrict__ bv, int32_t *cnt) {
  int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= 2 * n) return;
  int c = row >> 1, r = row & 1, k = 0;
  for (int q = rp[c]; q < rp[c + 1]; q++)
    for (int s = 0; s < 2; s++) k += (bv[4 * (size_t)q + 2 * r + s] != 0.0 || (ci[q] == c && r == s)) ? 1 : 0;
  cnt[row] = k;
}
__global__ void k_jsc_fill(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           const double *__restrict__ bv, const int32_t *__restrict__ orp, int32_t *oci,
                           double *ov) {
  int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= 2 * n) return;
  int c = row >> 1, r = row & 1, k = orp[row];
  for (int q = rp[c]; q < rp[c + 1]; q++)
    for (int s = 0; s < 2; s++) {
      double a = bv[4 * (size_t)q + 2 * r + s];
      if (a != 0.0 || (ci[q] == c && r == s)) {
        oci[k] = 2 * ci[q] + s;
        ov[k] = a;
        k++;
      }
    }
}

void build_jscalar(bf_ctx *c, DCsr &A) {
  int n2 = 2 * c->n;
  int32_t *cnt = dalloc_t<int32_t>(c, n2);
  k_jsc_count<<<div_up(n2, 256), 256, 0, c->stream>>>(c->n, c->brp, c->bci, c->bv, cnt);
  BF_LAUNCH(c);
  A.n = A.m = n2;
  A.rp = dalloc_t<int32_t>(c, (size_t)n2 + 1);
  A.nnz = exclusive_scan_i32(c, cnt, A.rp, n2);
  A.ci = dalloc_t<int32_t>(c, A.nnz);
  A.v = dalloc_t<double>(c, A.nnz);
  k_jsc_fill<<<div_up(n2, 256), 256, 0, c->stream>>>(c->n, c->brp, c->bci, c->bv, A.rp, A.ci, A.v);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  dfree(c, cnt);
}

// v (caller order, normalised in place when nrm2) -> b = canonical v, x0 = beta b ./ dl1
__global__ void k_jsc_split(int n, int ip, double2 *v, const double *nrm2, double2 *__restrict__ b,
                            const double2 *__restrict__ dinv, double beta, double2 *__restrict__ x0) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 a = v[i];
  if (nrm2) {
    double sc = 1.0 / sqrt(*nrm2);
    a.x = a.x * sc;
    a.y = a.y * sc;
    v[i] = a;
  }
  double2 cv = ip ? make_double2(a.y, a.x) : a;
  b[i] = cv;
  double2 d = dinv[i];
  x0[i] = make_double2(beta * (cv.x * d.x), beta * (cv.y * d.y));
}
__global__ void k_jsc_merge(int n, int ip, const double2 *__restrict__ x, double2 *__restrict__ z) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[i] = ip ? make_double2(x[i].y, x[i].x) : x[i];
}

void amg_apply(bf_ctx *c, const double *v, double *z, const double *nrm2) {
  int n = c->n;
  Level &L = c->h[3].lv[0];
  k_jsc_split<<<div_up(n, 256), 256, 0, c->stream>>>(n, c->var_order, reinterpret_cast<double2 *>(const_cast<double *>(v)),
                                                      nrm2, reinterpret_cast<double2 *>(L.b),
                                                      reinterpret_cast<const double2 *>(L.d), L.beta0,
                                                      reinterpret_cast<double2 *>(L.x));
  BF_LAUNCH(c);
  vcycle_from_invariant(c, 3);
  k_jsc_merge<<<div_up(n, 256), 256, 0, c->stream>>>(n, c->var_order, reinterpret_cast<const double2 *>(c->h[3].lv[0].x),
                                                      reinterpret_cast<double2 *>(z));
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

bool amg_patch_roles(const void *func, int &nargs, std::vector<std::pair<int, int>> &roles) {
  if (func == (const void *)k_jsc_split) {
    nargs = nargs_of(k_jsc_split);
    roles = {{2, 0}, {3, 1}};
  } else if (func == (const void *)k_jsc_merge) {
    nargs = nargs_of(k_jsc_merge);
    roles = {{3, 2}};
  } else {
    return false;
  }
  return true;
}

}  // namespace bf
