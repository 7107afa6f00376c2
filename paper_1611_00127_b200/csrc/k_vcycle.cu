// k_vcycle.cu -- the AMG V(nu_pre, nu_post) cycle (one cycle per inner solve)
// with l1-Jacobi or Chebyshev smoothing (replacing the paper's hybrid Gauss-Seidel,
// DESIGN.md R9), restriction b_c = R r, prolongation x += P e and the shared-memory
// staged dense coarse solve; and the BF preconditioner apply, Algorithm 3:
//   s = V_Ass(R_s v);  r' = R_p v - A_ps s;  p = V_S~(r');  z = R_p^T p + R_s^T s.
#include "bf_internal.cuh"
BF_CHECK_TU("k_vcycle.cu")
#include "k_spmv.cuh"
#include "k_dia.cuh"

#include <algorithm>
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace bf {

// Chebyshev interval of level L: [lo hi, hi] on D_l1^-1 A (reading R21): theta = hi (1+lo)/2,
// delta = hi (1-lo)/2; the first step from zero is x0 = (1/theta) b ./ dl1 (Level::beta0)
static void cheb_params(const bf_options &o, const Level &L, double &theta, double &delta) {
  theta = L.cheb_hi * (1.0 + o.cheb_lo) / 2.0;
  delta = L.cheb_hi * (1.0 - o.cheb_lo) / 2.0;
}

void set_level_beta(const bf_options &o, Level &L) {
  double theta, delta;
  cheb_params(o, L, theta, delta);
  L.beta0 = L.smoother == 1 ? 1.0 / theta : 1.0;
}

// coarsest-level solve x = A_L^-1 b with the inverse formed at setup from the pivoted LU
// (one CTA, thread per row; replaces 2 n dependent substitution steps)
__global__ void k_coarse_inv(int n, const double *__restrict__ inv, const double *__restrict__ b,
                             double *__restrict__ x) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < n; j++) s += inv[(size_t)i * n + j] * b[j];
    x[i] = s;
  }
}

// ----------------------------------------------------------------------------------------
// Cooperative tail of the V-cycle: all levels from h.tail down to the coarsest in ONE
// cooperative kernel (grid-wide barriers between the steps) instead of ~4 launches per level
// (l1-Jacobi V(1,1), the default configuration).  The coarse levels are latency bound: a
// level with 10^3..10^4 rows is one short wave, so the launch + ramp of separate kernels, not
// the bytes, sets their cost.  Rows are owned by groups of g lanes (g ~ mean row length / 2),
// each group reduces its row in a fixed order; every value has one owner.
// ----------------------------------------------------------------------------------------
constexpr int TAIL_MAXL = 12;
constexpr int TAIL_THREADS = 512;

// smoothing recurrence of one pass of a level: l1-Jacobi is the degree-1 case c0 = 1;
// Chebyshev of degree m: first step x += c0 D (b - A x), dir = that step; steps k = 1..m-1:
// dir = ca[k] dir + cb[k] D (b - A x), x += dir (smooth_pass below)
struct TailSmoother {
  int deg, nu_pre, nu_post;
  double c0, ca[8], cb[8];
};
struct TailLevel {
  int n, gA, gP, gR;
  const int32_t *Arp, *Aci, *Prp, *Pci, *Rrp, *Rci;
  const double *Av, *Pv, *Rv, *d;
  double *b, *x, *r, *t, *dir;
  TailSmoother sm;
};
struct TailParams {
  int nl;  // tail levels including the coarsest
  int gL;  // lanes per row of the dense coarse solve
  double beta;
  const double *inv;
  TailLevel lv[TAIL_MAXL];
};

// g-lane group reduction of one CSR row (all lanes of the warp call it; result on lane 0 of
// the group); ok = this group has a row
__device__ __forceinline__ double group_row(const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                            const double *__restrict__ v, const double *x, int r, bool ok,
                                            int lig, int g, int m) {
  double s = 0.0;
  if (ok) {
    int e = rp[r + 1];
    for (int q = rp[r] + lig; q < e; q += g) s += v[q] * x[BF_COL(ci[q], m)];
  }
  for (int o = g >> 1; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, g);
  return s;
}

__global__ void __launch_bounds__(TAIL_THREADS) k_vcycle_tail(TailParams p) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int l = 0; l < p.nl - 1; l++) {
    const TailLevel &L = p.lv[l];
    {  // r = b - A x0
      int g = L.gA, lig = tid & (g - 1);
      for (int base = 0; base < L.n; base += nth / g) {
        int r = base + tid / g;
        bool ok = r < L.n;
        double s = group_row(L.Arp, L.Aci, L.Av, L.x, r, ok, lig, g, L.n);
        if (ok && lig == 0) L.r[r] = L.b[r] - s;
      }
    }
    grid.sync();
    const TailLevel &C = p.lv[l + 1];
    {  // b_c = R r ; x0_c = beta b_c ./ dl1_c
      int g = L.gR, lig = tid & (g - 1);
      for (int base = 0; base < C.n; base += nth / g) {
        int r = base + tid / g;
        bool ok = r < C.n;
        double s = group_row(L.Rrp, L.Rci, L.Rv, L.r, r, ok, lig, g, L.n);
        if (ok && lig == 0) {
          C.b[r] = s;
          C.x[r] = p.beta * (s * C.d[r]);
        }
      }
    }
    grid.sync();
  }
  {  // coarsest: x = A_L^-1 b
    const TailLevel &L = p.lv[p.nl - 1];
    int g = p.gL, lig = tid & (g - 1);
    for (int base = 0; base < L.n; base += nth / g) {
      int i = base + tid / g;
      bool ok = i < L.n;
      double s = 0.0;
      if (ok)
        for (int j = lig; j < L.n; j += g) s += p.inv[(size_t)i * L.n + j] * L.b[j];
      for (int o = g >> 1; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, g);
      if (ok && lig == 0) L.x[i] = s;
    }
    grid.sync();
  }
  // up-sweep; the smoothed result of a tail level stays in its t buffer (the host swaps the
  // first tail level's x/t pointers, so the caller sees it in L.x)
  for (int l = p.nl - 2; l >= 0; l--) {
    const TailLevel &L = p.lv[l];
    const TailLevel &C = p.lv[l + 1];
    const double *e = (l + 1 == p.nl - 1) ? C.x : C.t;
    {  // x += P e
      int g = L.gP, lig = tid & (g - 1);
      for (int base = 0; base < L.n; base += nth / g) {
        int r = base + tid / g;
        bool ok = r < L.n;
        double s = group_row(L.Prp, L.Pci, L.Pv, e, r, ok, lig, g, C.n);
        if (ok && lig == 0) L.x[r] += s;
      }
    }
    grid.sync();
    {  // t = x + (b - A x) ./ dl1
      int g = L.gA, lig = tid & (g - 1);
      for (int base = 0; base < L.n; base += nth / g) {
        int r = base + tid / g;
        bool ok = r < L.n;
        double s = group_row(L.Arp, L.Aci, L.Av, L.x, r, ok, lig, g, L.n);
        if (ok && lig == 0) L.t[r] = L.x[r] + (L.b[r] - s) * L.d[r];
      }
    }
    if (l > 0) grid.sync();
  }
}

// decide where the tail starts (default smoother configuration only)
void plan_tail(bf_ctx *c, Hier &h) {
  const bf_options &o = c->opt;
  h.tail = -1;
  if (!c->tune.tail || o.nu_pre != 1 || o.nu_post != 1 || !h.dense) return;
  int64_t lim = c->tune.tail_nnz;
  int l = h.nlev - 1;
  // the cooperative tail implements l1-Jacobi V(1,1): only levels smoothed by l1-Jacobi (R22)
  while (l - 1 >= 0 && h.lv[l - 1].A.nnz <= lim && h.nlev - (l - 1) <= TAIL_MAXL && h.lv[l - 1].smoother == 0) l--;
  if (l < h.nlev - 1) h.tail = l;
}

// ----------------------------------------------------------------------------------------
// Dense tail operator.  Below the first level l_T with at most DTAIL_N rows, the V(1,1) cycle
// (seeded l1-Jacobi pre-sweep, residual, restriction, recursion, exact coarse solve,
// prolongation, post-sweep) is a FIXED linear map b_{l_T} -> x_{l_T}: nothing in it depends on
// the right-hand side except linearly.  Its matrix T (n x n, n <= DTAIL_N) is formed at setup
// by running exactly those steps on the n unit vectors (one CTA per column, k_tail_columns),
// and the solve applies it as one dense matvec (k_dense_tail): the same operator as the
// level-by-level cycle (rounding order differs; the V-cycle parity tolerance covers it),
// ~10 latency-bound launches per hierarchy replaced by one bandwidth-bound read of T
// (C3: 950^2 and 606^2 doubles, 7.2 + 2.9 MB).  Default smoother configuration only; frozen
// with the coarse levels by bf_update (R16).
// ----------------------------------------------------------------------------------------
constexpr int DTAIL_N = 2048;
constexpr int DTAIL_THREADS = 256;

// one CTA per column `col` of T; per-column level vectors are the TailParams buffers offset by
// col * n_k (allocated [n0 columns][n_k] per level by build_dense_tail).  Runs exactly the
// V(nu_pre, nu_post) cycle of vcycle_level below the first tail level -- smoothing passes from
// zero, residual, restriction, recursion, exact coarse solve, prolongation, post-smoothing --
// on the unit vector e_col, for either smoother (any fixed smoother makes the cycle linear).
__global__ void __launch_bounds__(DTAIL_THREADS) k_tail_columns(TailParams p, double *__restrict__ T) {
  const int col = blockIdx.x, n0 = p.lv[0].n;
  const int tid = threadIdx.x, nth = blockDim.x;
  const TailSmoother &sm0 = p.lv[0].sm;  // nu_pre / nu_post (the same on every level)
  auto off = [&](int k) { return (size_t)col * p.lv[k].n; };
  // t = A x (all rows), then the pointwise smoothing update of step `step` of a pass
  auto smooth_step = [&](int k, int step, bool from_zero) {
    const TailLevel &L = p.lv[k];
    const TailSmoother &sm = L.sm;
    double *b = L.b + off(k), *x = L.x + off(k), *t = L.t + off(k), *dir = L.dir + off(k);
    if (!from_zero) {
      int g = L.gA, lig = tid & (g - 1);
      for (int base = 0; base < L.n; base += nth / g) {
        int i = base + tid / g;
        bool ok = i < L.n;
        double s = group_row(L.Arp, L.Aci, L.Av, x, i, ok, lig, g, L.n);
        if (ok && lig == 0) t[i] = s;
      }
      __syncthreads();
    }
    for (int i = tid; i < L.n; i += nth) {
      double res = (b[i] - (from_zero ? 0.0 : t[i])) * L.d[i];
      double dn = step == 0 ? sm.c0 * res : sm.ca[step] * dir[i] + sm.cb[step] * res;
      dir[i] = dn;
      x[i] = (from_zero ? 0.0 : x[i]) + dn;
    }
    __syncthreads();
  };
  auto smooth_pass = [&](int k, bool from_zero) {
    for (int step = 0; step < p.lv[k].sm.deg; step++) smooth_step(k, step, from_zero && step == 0);
  };
  for (int i = tid; i < n0; i += nth) p.lv[0].b[off(0) + i] = i == col ? 1.0 : 0.0;
  __syncthreads();
  for (int l = 0; l < p.nl - 1; l++) {
    const TailLevel &L = p.lv[l];
    const TailLevel &C = p.lv[l + 1];
    double *b = L.b + off(l), *x = L.x + off(l), *r = L.r + off(l);
    if (sm0.nu_pre == 0) {
      for (int i = tid; i < L.n; i += nth) x[i] = 0.0;
      __syncthreads();
    }
    for (int s = 0; s < sm0.nu_pre; s++) smooth_pass(l, s == 0);
    {  // r = b - A x
      int g = L.gA, lig = tid & (g - 1);
      for (int base = 0; base < L.n; base += nth / g) {
        int i = base + tid / g;
        bool ok = i < L.n;
        double s = group_row(L.Arp, L.Aci, L.Av, x, i, ok, lig, g, L.n);
        if (ok && lig == 0) r[i] = b[i] - s;
      }
    }
    __syncthreads();
    {  // b_c = R r
      double *bc = C.b + off(l + 1);
      int g = L.gR, lig = tid & (g - 1);
      for (int base = 0; base < C.n; base += nth / g) {
        int i = base + tid / g;
        bool ok = i < C.n;
        double s = group_row(L.Rrp, L.Rci, L.Rv, r, i, ok, lig, g, L.n);
        if (ok && lig == 0) bc[i] = s;
      }
    }
    __syncthreads();
  }
  {  // coarsest: x = A_L^-1 b
    const TailLevel &L = p.lv[p.nl - 1];
    double *b = L.b + off(p.nl - 1), *x = L.x + off(p.nl - 1);
    for (int i = tid; i < L.n; i += nth) {
      double s = 0.0;
      for (int j = 0; j < L.n; j++) s += p.inv[(size_t)i * L.n + j] * b[j];
      x[i] = s;
    }
  }
  __syncthreads();
  for (int l = p.nl - 2; l >= 0; l--) {
    const TailLevel &L = p.lv[l];
    const double *e = p.lv[l + 1].x + off(l + 1);
    double *x = L.x + off(l);
    {  // x += P e
      int g = L.gP, lig = tid & (g - 1);
      for (int base = 0; base < L.n; base += nth / g) {
        int i = base + tid / g;
        bool ok = i < L.n;
        double s = group_row(L.Prp, L.Pci, L.Pv, e, i, ok, lig, g, p.lv[l + 1].n);
        if (ok && lig == 0) x[i] += s;
      }
    }
    __syncthreads();
    for (int s = 0; s < sm0.nu_post; s++) smooth_pass(l, false);
  }
  const double *x0 = p.lv[0].x + off(0);
  for (int i = tid; i < n0; i += nth) T[(size_t)i * n0 + col] = x0[i];
}

// the smoothing recurrence of one pass on level L (see TailSmoother)
static TailSmoother tail_smoother(const bf_options &o, const Level &L) {
  TailSmoother sm{};
  sm.nu_pre = o.nu_pre;
  sm.nu_post = o.nu_post;
  if (L.smoother == 0) {
    sm.deg = 1;
    sm.c0 = 1.0;
    return sm;
  }
  double theta, delta;
  cheb_params(o, L, theta, delta);
  double sigma = theta / delta;
  double rho = 1.0 / sigma;
  sm.deg = o.cheb_degree;
  sm.c0 = 1.0 / theta;
  for (int k = 1; k < o.cheb_degree; k++) {
    double rho_new = 1.0 / (2.0 * sigma - rho);
    sm.ca[k] = rho_new * rho;
    sm.cb[k] = 2.0 * rho_new / delta;
    rho = rho_new;
  }
  return sm;
}

// x = T b: DTAIL_SPLIT warps per row of T (each a contiguous quarter of the row, 8 loads in
// flight per lane), b staged in shared memory; partial sums combined in a fixed order
constexpr int DTAIL_SPLIT = 4;
__global__ void __launch_bounds__(DTAIL_THREADS) k_dense_tail(int n, const double *__restrict__ T,
                                                               const double *__restrict__ b, double *__restrict__ x) {
  extern __shared__ double bs[];
  __shared__ double part[DTAIL_THREADS / 32];
  // T is setup data: the first loads of this CTA's rows are issued before the wait (PDL)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.x * (DTAIL_THREADS / 32 / DTAIL_SPLIT) + warp / DTAIL_SPLIT;
  const int q = warp % DTAIL_SPLIT;
  const int seg = (n + DTAIL_SPLIT - 1) / DTAIL_SPLIT;
  const int j0 = q * seg, j1 = min(n, j0 + seg);
  pdl_wait();
  for (int j = threadIdx.x; j < n; j += blockDim.x) bs[j] = b[j];
  __syncthreads();
  double s = 0.0;
  if (row < n) {
    const double *tr = T + (size_t)row * n;
#pragma unroll 8
    for (int j = j0 + lane; j < j1; j += 32) s += __ldcs(tr + j) * bs[j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) part[warp] = s;
  __syncthreads();
  if (threadIdx.x < DTAIL_THREADS / 32 / DTAIL_SPLIT) {
    int r = blockIdx.x * (DTAIL_THREADS / 32 / DTAIL_SPLIT) + threadIdx.x;
    if (r < n) {
      double t = 0.0;
      for (int k = 0; k < DTAIL_SPLIT; k++) t += part[threadIdx.x * DTAIL_SPLIT + k];
      x[r] = t;
    }
  }
}

static int tail_lanes(int64_t nnz, int n);

void build_dense_tail(bf_ctx *c, Hier &h) {
  const bf_options &o = c->opt;
  dfree(c, h.tmat);
  h.tmat = nullptr;
  h.dtail = -1;
  if (!c->tune.dtail || !h.dense) return;
  int lim = std::min(c->tune.dtail_n, DTAIL_N);
  int lt = -1;
  for (int l = 1; l < h.nlev - 1; l++)
    if (h.lv[l].A.n <= lim && h.nlev - l <= TAIL_MAXL) {
      lt = l;
      break;
    }
  if (lt < 0) return;
  int n0 = h.lv[lt].A.n;
  TailParams p;
  p.nl = h.nlev - lt;
  p.beta = 1.0;
  p.inv = h.inv;
  std::vector<double *> bufs;
  for (int k = 0; k < p.nl; k++) {
    Level &L = h.lv[lt + k];
    TailLevel &Tl = p.lv[k];
    Tl.n = L.A.n;
    Tl.gA = tail_lanes(L.A.nnz, L.A.n);
    Tl.gP = tail_lanes(L.P.nnz, L.A.n);
    Tl.gR = tail_lanes(L.R.nnz, L.R.n);
    Tl.Arp = L.A.rp;
    Tl.Aci = L.A.ci;
    Tl.Av = L.A.v;
    Tl.Prp = L.P.rp;
    Tl.Pci = L.P.ci;
    Tl.Pv = L.P.v;
    Tl.Rrp = L.R.rp;
    Tl.Rci = L.R.ci;
    Tl.Rv = L.R.v;
    Tl.d = L.d;
    Tl.sm = tail_smoother(o, L);
    double *w = dalloc_t<double>(c, (size_t)5 * n0 * L.A.n);  // [b | x | r | t | dir] x n0 columns
    bufs.push_back(w);
    Tl.b = w;
    Tl.x = w + (size_t)n0 * L.A.n;
    Tl.r = w + (size_t)2 * n0 * L.A.n;
    Tl.t = w + (size_t)3 * n0 * L.A.n;
    Tl.dir = w + (size_t)4 * n0 * L.A.n;
  }
  h.tmat = dalloc_t<double>(c, (size_t)n0 * n0);
  k_tail_columns<<<n0, DTAIL_THREADS, 0, c->stream>>>(p, h.tmat);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  for (double *w : bufs) dfree(c, w);
  h.dtail = lt;
}

static void launch_dense_tail(bf_ctx *c, Hier &h) {
  Level &L = h.lv[h.dtail];
  int n = L.A.n;
  c->alg_bytes += 8.0 * n * n + 16.0 * n;
  ensure_smem_attr((const void *)k_dense_tail, DTAIL_N * 8 + 1024);
  launch_pdl(c, k_dense_tail, dim3(div_up(n, DTAIL_THREADS / 32 / DTAIL_SPLIT)), dim3(DTAIL_THREADS),
             sizeof(double) * n, n, (const double *)h.tmat, (const double *)L.b, L.x);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

// lanes per row group: a power of two near half the mean row length
static int tail_lanes(int64_t nnz, int n) {
  double mean = n > 0 ? (double)nnz / n : 1.0;
  int g = 1;
  while (g < 32 && 2 * g <= mean / 2.0) g <<= 1;
  return g;
}

static void launch_tail(bf_ctx *c, Hier &h) {
  TailParams p;
  p.nl = h.nlev - h.tail;
  p.beta = 1.0;
  p.inv = h.inv;
  int64_t lanes = 1;
  for (int k = 0; k < p.nl; k++) {
    Level &L = h.lv[h.tail + k];
    TailLevel &T = p.lv[k];
    T.n = L.A.n;
    T.gA = tail_lanes(L.A.nnz, L.A.n);
    T.gP = tail_lanes(L.P.nnz, L.A.n);
    T.gR = tail_lanes(L.R.nnz, L.R.n);
    T.Arp = L.A.rp;
    T.Aci = L.A.ci;
    T.Av = L.A.v;
    T.Prp = L.P.rp;
    T.Pci = L.P.ci;
    T.Pv = L.P.v;
    T.Rrp = L.R.rp;
    T.Rci = L.R.ci;
    T.Rv = L.R.v;
    T.d = L.d;
    T.b = L.b;
    T.x = L.x;
    T.r = L.r;
    T.t = L.t;
    if (k < p.nl - 1) {
      lanes = std::max(lanes, (int64_t)T.n * std::max(T.gA, T.gP));
      lanes = std::max(lanes, (int64_t)L.R.n * T.gR);
      c->alg_bytes += 2 * (12.0 * L.A.nnz + 4.0 * L.A.n) + 2 * (12.0 * L.P.nnz + 4.0 * L.A.n) + 80.0 * L.A.n;
    }
  }
  p.gL = std::min(32, std::max(1, tail_lanes((int64_t)h.nL * h.nL, h.nL)));
  lanes = std::max(lanes, (int64_t)h.nL * p.gL);
  c->alg_bytes += 8.0 * h.nL * h.nL;
  const int per_sm = occupancy(c, (const void *)k_vcycle_tail, TAIL_THREADS, 0);
  const int max_blocks = std::max(1, std::min(per_sm, c->tune.tail_bps)) * c->num_sms;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_blocks, (lanes + TAIL_THREADS - 1) / TAIL_THREADS));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TAIL_THREADS);
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, k_vcycle_tail, p));
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  Level &L0 = h.lv[h.tail];  // the tail's result for its first level is in t
  std::swap(L0.x, L0.t);
}

__global__ void k_zero(int n, double *x) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = 0.0;
}

// choose the TMA tiling of a CSR matrix: ~1024 nonzeros per tile, 8..256 rows per tile
// lanes per row: stencil-ordered fine-level rows -> 1 (lane-per-row gathers of consecutive
// rows hit consecutive addresses); Galerkin rows -> several lanes reading adjacent sorted
// columns of the same row (fewer distinct sectors per gather instruction)
void tile_csr(bf_ctx *c, DCsr &A, bool stencil, int force_g) {
  A.rpt = 0;
  A.cap = 0;
  A.short_rows = false;
  if (A.n == 0 || A.nnz == 0) return;
  double mean = (double)A.nnz / A.n;
  // large matrices with short rows (the fine levels' P and R): thread-per-row kernel
  if (!stencil && mean <= c->tune.short_lim && A.n >= c->tune.short_nmin) A.short_rows = true;
  int g = 1;
  if (force_g > 0) {
    g = force_g;
  } else if (stencil) {
    // lane-per-row gathers are ideal for stencil rows, but a 256-row tile of long rows (S~:
    // ~12/row) needs ~100 KB for two stages -> 2 CTAs/SM; two lanes per row keep 128-row tiles
    if (mean > c->tune.stencil_g2) g = 2;
  } else {
    // measured (C3, with the fused restriction): mean / 4 beats mean / 3, 5, 8
    while (g < 32 && 2 * g <= mean / c->tune.tma_g_div) g <<= 1;
  }
  // measured: ~1024 nonzeros per tile beats 2048 (more CTAs per SM for the gathers)
  const double tile = c->tune.tma_tile;
  int rpt = 256;
  // ~1024 nonzeros per tile, but at least one full pass of the CTA (256/g rows) so that no
  // thread idles (stencil rows, g = 1, always take 256-row tiles)
  while (rpt > 8 && rpt > TMA_THREADS / g && rpt * mean > tile) rpt >>= 1;
  // small (coarse-level) matrices: spread the tiles over all SMs (>= 2 tiles per SM) instead of a
  // few CTAs walking long chains of dependent loads; the CTA's threads then take more lanes per
  // row, g = 256 / rows per tile (ncu: the 7.6K-row restriction of C3's A_ss level 3 ran on 30
  // CTAs at 17 us for 1 MB)
  if (force_g <= 0 && !stencil && c->tune.spread_small) {
    const int64_t want = 2 * (int64_t)c->num_sms;
    while (rpt > 8 && (A.n + rpt - 1) / rpt < want) rpt >>= 1;
    while (g < 32 && (int64_t)g * rpt < TMA_THREADS) g <<= 1;
  }
  A.g = g;
  int *mx = dalloc_t<int>(c, 1);
  for (;; rpt >>= 1) {
    BF_CUDA(cudaMemsetAsync(mx, 0, sizeof(int), c->stream));
    int ntiles = (A.n + rpt - 1) / rpt;
    k_tile_max<<<div_up(ntiles, 256), 256, 0, c->stream>>>(A.n, rpt, A.rp, mx);
    BF_LAUNCH(c);
    int h = 0;
    BF_CUDA(cudaMemcpyAsync(&h, mx, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (TMA_STAGES * tma_stage_bytes(h, rpt) <= 110 * 1024) {
      A.rpt = rpt;
      A.cap = std::max(h, 1);
      break;
    }
    if (rpt == 8) break;  // rows too long for a staged tile: generic warp kernel
  }
  dfree(c, mx);
}

// ---- windowed jagged-diagonal form of the coarse-level operators (k_csr_win.cuh) ---------------
// plan: one CTA per block of `wrows` rows sorts the block's rows by (length descending, row
// ascending) and records the order with the lengths (rowinfo), the jagged-diagonal offsets (jdo)
// and the block's entry count
static __global__ void __launch_bounds__(256) k_wjds_plan(int n, int wrows, const int32_t *__restrict__ rp,
                                                          uint32_t *__restrict__ rowinfo,
                                                          uint16_t *__restrict__ jdo, int32_t *__restrict__ block_ne,
                                                          int32_t *__restrict__ block_maxlen,
                                                          int *__restrict__ stat) {
  __shared__ int key[WIN_ROWS_MAX];
  __shared__ int cnt_e[WJDS_MAXLEN + 1];
  const int blk = blockIdx.x, tid = threadIdx.x;
  for (int i = tid; i < wrows; i += blockDim.x) {
    const int r = blk * wrows + i;
    int k = -1;  // padding row (beyond n)
    if (r < n) {
      const int len = rp[r + 1] - rp[r];
      if (len > WJDS_MAXLEN) stat[5] = 1;  // row too long for the per-block offset table: no WJDS form
      k = (min(len, WJDS_MAXLEN) << 16) | (0xffff - i);
    }
    key[i] = k;
  }
  __syncthreads();
  for (int k = 2; k <= wrows; k <<= 1)  // bitonic sort, descending
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < wrows; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const int a = key[i], b = key[l];
          const bool down = (i & k) == 0;
          if ((a < b) == down) {
            key[i] = b;
            key[l] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int p = tid; p < wrows; p += blockDim.x) {
    const int k = key[p];
    rowinfo[(size_t)blk * wrows + p] = k < 0 ? 0xffffu : (((uint32_t)(k >> 16) << 16) | (uint32_t)(0xffff - (k & 0xffff)));
  }
  // rows longer than e: the sorted order makes them a prefix (binary search for its end)
  for (int e = tid; e <= WJDS_MAXLEN; e += blockDim.x) {
    int lo = 0, hi = wrows;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int k = key[mid];
      if (k >= 0 && (k >> 16) > e) lo = mid + 1;
      else hi = mid;
    }
    cnt_e[e] = lo;
  }
  __syncthreads();
  if (tid == 0) {
    int off = 0, maxlen = 0;
    for (int e = 0; e <= WJDS_MAXLEN; e++) {
      jdo[(size_t)blk * (WJDS_MAXLEN + 1) + e] = (uint16_t)min(off, 0xffff);
      if (cnt_e[e] > 0) maxlen = e + 1;
      off += cnt_e[e];
    }
    if (off > 0xffff) stat[5] = 1;
    block_ne[blk] = (off + 7) & ~7;
    block_maxlen[blk] = maxlen;
  }
}

// fill: one CTA per block: the block's distinct columns by a shared-memory hash table and a
// bitonic sort (the window), then every entry written to its jagged-diagonal slot with its
// position in the window (binary search); the padding entries up to a multiple of 8 are (0.0, 0)
static __global__ void __launch_bounds__(256) k_wjds_fill(int n, int wrows, const int32_t *__restrict__ rp,
                                                          const int32_t *__restrict__ ci,
                                                          const double *__restrict__ v,
                                                          const uint32_t *__restrict__ rowinfo,
                                                          const uint16_t *__restrict__ jdo,
                                                          const int32_t *__restrict__ eo,
                                                          const int32_t *__restrict__ block_ne,
                                                          const int32_t *__restrict__ block_maxlen,
                                                          int4 *__restrict__ meta, int32_t *__restrict__ wcol,
                                                          uint16_t *__restrict__ lc, double *__restrict__ wv,
                                                          int *__restrict__ stat, unsigned long long *total) {
  extern __shared__ int32_t win_sm[];
  int32_t *table = win_sm, *uniq = win_sm + WIN_HASH;
  __shared__ int cnt;
  const int blk = blockIdx.x, tid = threadIdx.x;
  const int r0 = blk * wrows, r1 = min(n, r0 + wrows);
  const int q0 = rp[r0], q1 = rp[r1];
  if (stat[5]) return;  // the plan met a row it cannot represent (lengths clamped): no form
  // hash table sized for this block: at most min(nnz, WIN_MAX) distinct columns at load factor <= 1/2
  int hbits = 10;
  while (hbits < 13 && (1 << hbits) < 2 * min(q1 - q0, WIN_MAX)) hbits++;
  const int hsize = 1 << hbits;
  for (int i = tid; i < hsize; i += blockDim.x) table[i] = -1;
  if (tid == 0) cnt = 0;
  __syncthreads();
  for (int q = q0 + tid; q < q1; q += blockDim.x) {
    const int col = ci[q];
    unsigned slot = ((unsigned)col * 2654435761u) >> (32 - hbits);
    for (int probe = 0; probe < hsize; probe++) {
      int old = atomicCAS(&table[slot], -1, col);
      if (old == -1 || old == col) break;
      slot = (slot + 1) & (hsize - 1);
    }
  }
  __syncthreads();
  for (int i = tid; i < hsize; i += blockDim.x)
    if (table[i] != -1) {
      int pos = atomicAdd(&cnt, 1);
      if (pos < WIN_MAX) uniq[pos] = table[i];
    }
  __syncthreads();
  const int c = cnt;
  const int ne = block_ne[blk], e0 = eo[blk];
  if (c > WIN_MAX) {  // the block needs a larger window than shared memory holds
    if (tid == 0) {
      stat[0] = 1;
      meta[blk] = make_int4(e0, 0, 0, 0);
    }
    return;
  }
  int p2 = 2;
  while (p2 < c) p2 <<= 1;
  for (int i = c + tid; i < p2; i += blockDim.x) uniq[i] = 0x7fffffff;
  __syncthreads();
  for (int k = 2; k <= p2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < p2; i += blockDim.x) {
        int l = i ^ j;
        if (l > i) {
          int a = uniq[i], b = uniq[l];
          bool up = (i & k) == 0;
          if ((a > b) == up) {
            uniq[i] = b;
            uniq[l] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int i = tid; i < c; i += blockDim.x) wcol[(size_t)blk * WIN_MAX + i] = uniq[i];
  if (tid == 0) {
    meta[blk] = make_int4(e0, ne, c, block_maxlen[blk]);
    atomicMax(&stat[1], c);
    atomicMax(&stat[4], ne);
    atomicAdd(total, (unsigned long long)c);
  }
  // entries in jagged-diagonal order, one thread per entry: flat position i -> diagonal e (binary
  // search in the block's offsets) and sorted row position t = i - off[e]
  __shared__ uint16_t off[WJDS_MAXLEN + 1];
  __shared__ int rowq[WIN_ROWS_MAX];
  for (int e = tid; e <= WJDS_MAXLEN; e += blockDim.x) off[e] = jdo[(size_t)blk * (WJDS_MAXLEN + 1) + e];
  for (int t = tid; t < wrows; t += blockDim.x) {
    const int lr = (int)(rowinfo[(size_t)blk * wrows + t] & 0xffffu);
    rowq[t] = lr == 0xffff ? 0 : rp[r0 + lr];
  }
  __syncthreads();
  const int maxlen = block_maxlen[blk];
  for (int i = tid; i < q1 - q0; i += blockDim.x) {
    int lo = 0, hi = maxlen - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int)off[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const int e = lo, t = i - (int)off[e];
    const int q = rowq[t] + e;
    const int col = ci[q];
    lo = 0;
    hi = c - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (uniq[mid] < col) lo = mid + 1;
      else hi = mid;
    }
    wv[(size_t)e0 + i] = v[q];
    lc[(size_t)e0 + i] = BF_CHK(uniq[lo] == col) ? (uint16_t)lo : (uint16_t)0;
  }
  for (int i = (q1 - q0) + tid; i < ne; i += blockDim.x) {  // padding entries
    wv[(size_t)e0 + i] = 0.0;
    lc[(size_t)e0 + i] = 0;
  }
}

// wcol with the matrix's own stride instead of WIN_MAX slots per block
static __global__ void k_wjds_compact(int nblocks, int wstride, const int4 *__restrict__ meta,
                                      const int32_t *__restrict__ wide, int32_t *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nblocks * wstride) return;
  const int blk = (int)(i / wstride), k = (int)(i % wstride);
  out[i] = k < meta[blk].z ? wide[(size_t)blk * WIN_MAX + k] : 0;  // zero padded up to the stride
}

void free_window(bf_ctx *c, DCsr &A) {
  if (!A.ws) return;
  dfree(c, A.ws->meta);
  dfree(c, A.ws->jdo);
  dfree(c, A.ws->rowinfo);
  dfree(c, A.ws->wv);
  dfree(c, A.ws->lc);
  dfree(c, A.ws->wcol);
  delete A.ws;
  A.ws = nullptr;
}

// Build the windowed jagged-diagonal form of A (k_csr_win.cuh): blocks of wrows rows sized so that a
// block's stream is ~WJDS_STAGE_TARGET bytes; wrows is halved while some block's window exceeds
// WIN_MAX or its stream WJDS_STAGE_MAX; the form is dropped (CSR kernels) if no block size fits, if
// a row is longer than WJDS_MAXLEN, or if the windows hold more than win_ratio entries per nonzero
// (no column reuse to exploit).
void window_csr(bf_ctx *c, DCsr &A) {
  free_window(c, A);
  if (!c->tune.win || A.dia_v || A.n < c->tune.win_nmin || A.nnz <= 0) return;
  const double mean = (double)A.nnz / A.n;
  if (mean < c->tune.win_minlen) return;
  ensure_smem_attr((const void *)k_wjds_fill, (WIN_HASH + WIN_MAX) * 4 + 1024);
  int *stat = dalloc_t<int>(c, 8);
  unsigned long long *total = reinterpret_cast<unsigned long long *>(stat + 2);
  int wrows = std::min(WIN_ROWS_MAX, std::max(32, c->tune.win_rows));
  while (wrows & (wrows - 1)) wrows &= wrows - 1;  // power of two
  while (wrows > 32 && wrows * mean * 10.0 > c->tune.win_stage) wrows >>= 1;
  for (;; wrows >>= 1) {
    A.ws = new WJds();
    WJds &W = *A.ws;
    const int nblocks = (A.n + wrows - 1) / wrows;
    W.rowinfo = dalloc_t<uint32_t>(c, (size_t)nblocks * wrows);
    W.jdo = dalloc_t<uint16_t>(c, (size_t)nblocks * (WJDS_MAXLEN + 1));
    int32_t *bne = dalloc_t<int32_t>(c, (size_t)nblocks + 1), *bml = dalloc_t<int32_t>(c, nblocks);
    int32_t *eo = dalloc_t<int32_t>(c, (size_t)nblocks + 1);
    BF_CUDA(cudaMemsetAsync(stat, 0, 32, c->stream));
    k_wjds_plan<<<nblocks, 256, 0, c->stream>>>(A.n, wrows, A.rp, W.rowinfo, W.jdo, bne, bml, stat);
    BF_LAUNCH(c);
    const int64_t entries = exclusive_scan_i32(c, bne, eo, nblocks);  // syncs
    int hs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool ok = entries < (1ll << 31) - 8;  // (a too-long row, stat[0] = 2, is seen after the fill: its length is clamped)
    if (ok) {
      W.meta = dalloc_t<int4>(c, nblocks);
      W.wcol = dalloc_t<int32_t>(c, (size_t)nblocks * WIN_MAX);
      W.lc = dalloc_t<uint16_t>(c, (size_t)entries + 8);
      W.wv = dalloc_t<double>(c, (size_t)entries + 2);
      k_wjds_fill<<<nblocks, 256, (WIN_HASH + WIN_MAX) * 4, c->stream>>>(
          A.n, wrows, A.rp, A.ci, A.v, W.rowinfo, W.jdo, eo, bne, bml, W.meta, W.wcol, W.lc, W.wv, stat, total);
      BF_LAUNCH(c);
      BF_CUDA(cudaMemcpyAsync(hs, stat, 32, cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      ok = hs[5] == 0;
    }
    dfree(c, bne);
    dfree(c, bml);
    dfree(c, eo);
    unsigned long long tot;
    memcpy(&tot, hs + 2, sizeof tot);
    const bool too_big = ok && (hs[0] == 1 || hs[4] * 10 > WJDS_STAGE_MAX);  // window or stream: smaller blocks
    if (ok && !too_big && (double)tot <= c->tune.win_ratio * (double)A.nnz) {
      W.wrows = wrows;
      W.wmax_used = hs[1];
      W.cap_ne = hs[4];
      W.wstride = std::min(WIN_MAX, (hs[1] + 255) & ~255);
      int32_t *wide = W.wcol;
      W.wcol = dalloc_t<int32_t>(c, (size_t)nblocks * W.wstride);
      k_wjds_compact<<<div_up((int64_t)nblocks * W.wstride, 256), 256, 0, c->stream>>>(nblocks, W.wstride, W.meta, wide,
                                                                                                W.wcol);
      BF_LAUNCH(c);
      dfree(c, wide);
      if (c->tune.verbose)
        fprintf(stderr,
                "[bf_setup]   wjds: %d x %d, nnz %lld, blocks of %d rows: %d blocks, max window %d, max stream %d B, "
                "%.3f window entries/nnz\n",
                A.n, A.m, (long long)A.nnz, wrows, nblocks, hs[1], hs[4] * 10, (double)tot / (double)A.nnz);
      dfree(c, stat);
      return;
    }
    free_window(c, A);
    if (!(too_big && wrows > 32)) break;
  }
  dfree(c, stat);
}

// WJDS forms for the coarse levels of a hierarchy: A_l, l >= 1, above the tail.  Measured on C3 and
// not given a form: the fused restrictions Rf_l (rows of ~100 entries over ~0.4 window columns per
// nonzero: 48 us against 45 us for the TMA CSR kernel) and the level transfers P_l, R_l (2-6 entries
// per row, 0.5-0.6 window columns per nonzero: 40 us against 30 us for the thread-per-row kernel).
void build_windows(bf_ctx *c, Hier &h) {
  const int lend = h.dtail >= 0 ? h.dtail : (h.tail >= 0 ? h.tail : h.nlev - 1);
  for (int l = 1; l < lend; l++) window_csr(c, h.lv[l].A);
  BF_CUDA(cudaGetLastError());
}

// DIA form of a finest-level matrix whose nonzeros all sit on a few grid-stencil offsets
void setup_dia(bf_ctx *c, DCsr &A) {
  if (!c->tune.dia || A.n == 0 || A.n != A.m || c->nx <= 0) return;
  std::vector<int> cand;
  int64_t sx = 1, sy = c->nx, sz = (int64_t)c->nx * c->ny;
  for (int cz = -2; cz <= 2; cz++)
    for (int cy = -2; cy <= 2; cy++)
      for (int cx = -2; cx <= 2; cx++) {
        int64_t o = cx * sx + cy * sy + cz * sz;
        if (o > -(int64_t)A.n && o < A.n) cand.push_back((int)o);
      }
  std::sort(cand.begin(), cand.end());
  cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
  int nc = (int)cand.size();
  int *dcand = dalloc_t<int>(c, nc), *pres = dalloc_t<int>(c, nc + 1);
  BF_CUDA(cudaMemcpyAsync(dcand, cand.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, c->stream));
  BF_CUDA(cudaMemsetAsync(pres, 0, sizeof(int) * (nc + 1), c->stream));
  k_dia_mark<<<div_up(A.n, 256), 256, 0, c->stream>>>(A, dcand, nc, pres, pres + nc);
  BF_LAUNCH(c);
  std::vector<int> hp(nc + 1);
  BF_CUDA(cudaMemcpyAsync(hp.data(), pres, sizeof(int) * (nc + 1), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, dcand);
  dfree(c, pres);
  if (hp[nc]) return;  // an offset outside the candidate stencil
  DiaOffsets o;
  o.k = 0;
  for (int q = 0; q < nc; q++)
    if (hp[q]) {
      if (o.k == DIA_MAXK) return;
      o.off[o.k++] = cand[q];
    }
  double fill = (double)A.nnz / ((double)o.k * A.n);
  if (fill < 0.75) return;
  A.dia_v = dalloc_t<double>(c, (size_t)o.k * A.n);
  A.dia_k = o.k;
  c->dia_offsets.emplace_back(o.off, o.off + o.k);
  A.dia_off = c->dia_offsets.back().data();
  k_dia_fill<<<div_up(A.n, 256), 256, 0, c->stream>>>(A, o, A.dia_v);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}


// Level invariant on entry to vcycle_level(l): L.b holds the right-hand side and L.x holds
// x0 = beta b ./ dl1 (written by whichever kernel produced b: the split, the A_ps coupling,
// or the restriction of the finer level), i.e. the first smoothing step from zero is already
// done.  This keeps one gather per nonzero in every smoother kernel.

// one smoothing pass (l1-Jacobi, or Chebyshev of degree m on [lo,1]); x in/out (pointer may
// be swapped with L.t).  first: x holds x0 (the pass's first step is already applied).
// want_resid: leave r = b - A x in L.r.
static void smooth_pass(bf_ctx *c, Level &L, double *&x, bool first, bool want_resid) {
  const bf_options &o = c->opt;
  auto swap_t = [&]() {
    double *tmp = x;
    x = L.t;
    L.t = tmp;
  };
  if (L.smoother == 0) {  // x <- x + (b - A x) ./ dl1
    if (!first) {
      csr_op<OP_SMOOTH>(c, L.A, x, L.b, L.d, L.t, nullptr, 0.0, 1.0, nullptr);
      swap_t();
    }
  } else {  // Chebyshev acceleration of D^-1 A on [lo hi, hi] (three-term recurrence)
    double theta, delta;
    cheb_params(o, L, theta, delta);
    double sigma = theta / delta;
    double rho = 1.0 / sigma;
    double *dir = L.r;  // direction storage (r is recomputed below when needed)
    // the first step's direction is the step itself: after a seeded first step (x = x0 from
    // zero) that is x0, read in place (no copy into dir)
    const double *dir_in = dir;
    if (first) {
      dir_in = x;
    } else {
      csr_op<OP_SMOOTH>(c, L.A, x, L.b, L.d, L.t, dir, 0.0, 1.0 / theta, nullptr);
      swap_t();
    }
    for (int k = 1; k < o.cheb_degree; k++) {
      double rho_new = 1.0 / (2.0 * sigma - rho);
      csr_op<OP_SMOOTH>(c, L.A, x, L.b, L.d, L.t, dir, rho_new * rho, 2.0 * rho_new / delta, dir_in);
      swap_t();
      dir_in = dir;
      rho = rho_new;
    }
  }
  if (want_resid) csr_op<OP_RESID>(c, L.A, x, L.b, nullptr, L.r, nullptr, 0.0, 0.0, nullptr);
}

__global__ void k_x0(int n, double beta, const double *__restrict__ b, const double *__restrict__ dinv,
                     double *__restrict__ x) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = beta * (b[i] * dinv[i]);
}

// V-cycle on level l (invariant above); result left in L.x (pointer may be swapped with L.t)
static void vcycle_level(bf_ctx *c, Hier &h, int l) {
  Level &L = h.lv[l];
  int n = L.A.n;
  const bf_options &o = c->opt;
  if (l == h.dtail) {  // the whole sub-cycle from here down as one dense operator
    launch_dense_tail(c, h);
    return;
  }
  if (l == h.tail) {
    launch_tail(c, h);
    return;
  }
  if (l == h.nlev - 1) {
    if (h.dense) {
      c->alg_bytes += 8.0 * n * n + 16.0 * n;
      k_coarse_inv<<<1, 128, 0, c->stream>>>(n, h.inv, L.b, L.x);
      BF_LAUNCH(c);
      BF_CUDA(cudaGetLastError());
    } else {  // stalled coarsening: 4 l1-Jacobi sweeps from zero (x0 = b ./ dl1 is the first)
      if (L.smoother == 1) {  // x0 was seeded for Chebyshev: reseed for l1-Jacobi
        k_x0<<<div_up(n, 256), 256, 0, c->stream>>>(n, 1.0, L.b, L.d, L.x);
        BF_LAUNCH(c);
      }
      for (int s = 0; s < 3; s++) {
        csr_op<OP_SMOOTH>(c, L.A, L.x, L.b, L.d, L.t, nullptr, 0.0, 1.0, nullptr);
        double *tmp = L.x;
        L.x = L.t;
        L.t = tmp;
      }
    }
    return;
  }
  double *x = L.x;
  if (o.nu_pre == 0) {
    k_zero<<<div_up(n, 256), 256, 0, c->stream>>>(n, x);
    BF_LAUNCH(c);
    BF_CUDA(cudaMemcpyAsync(L.r, L.b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    for (int s = 0; s < o.nu_pre; s++) smooth_pass(c, L, x, s == 0, s == o.nu_pre - 1 && !L.Rf.n);
  }
  Level &Lc = h.lv[l + 1];
  // b_c = R r, and x0_c = beta b_c ./ dl1_c for the next level
  if (L.Rf.n) {  // b_c = R (I - beta A D) b: residual of the seeded pre-sweep + restriction in one product
    csr_op<OP_SPMV_X0>(c, L.Rf, L.b, nullptr, Lc.d, Lc.b, Lc.x, 0.0, Lc.beta0, nullptr);
  } else {
    csr_op<OP_SPMV_X0>(c, L.R, L.r, nullptr, Lc.d, Lc.b, Lc.x, 0.0, Lc.beta0, nullptr);
  }
  vcycle_level(c, h, l + 1);
  csr_op<OP_ADD>(c, L.P, Lc.x, nullptr, nullptr, x, nullptr, 0.0, 0.0, nullptr);  // x += P e
  const bool skip_post = c->fuse_post0 && l == 0 && &h == &c->h[1];  // done by k_dia_smooth_merge
  if (!skip_post)
    for (int s = 0; s < o.nu_post; s++) smooth_pass(c, L, x, false, false);
  if (x != L.x) {  // keep the result in L.x (swap the buffers, no copy)
    L.t = L.x;
    L.x = x;
  }
}


// V-cycle of hierarchy `which` whose finest level already holds b and x0 (level invariant)
void vcycle_from_invariant(bf_ctx *c, int which) { vcycle_level(c, c->h[which], 0); }

void vcycle(bf_ctx *c, int which, const double *b, double *x) {
  Hier &h = c->h[which];
  Level &L0 = h.lv[0];
  int n = L0.A.n;
  BF_CUDA(cudaMemcpyAsync(L0.b, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  k_x0<<<div_up(n, 256), 256, 0, c->stream>>>(n, L0.beta0, L0.b, L0.d, L0.x);
  BF_LAUNCH(c);
  vcycle_level(c, h, 0);
  BF_CUDA(cudaMemcpyAsync(x, L0.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
}

// R_p v -> vp, R_s v -> vs (interleaved in the caller's var_order); also x0 of the A_ss V-cycle.
// nrm2 != null: v is an unnormalised GMRES basis slot with ||v||^2 = *nrm2 (computed by the
// last CGS2 pass); v is normalised here, in place, by the same 1/sqrt(||v||^2) scaling the
// separate scaling pass applied (one read + one write of v saved per Arnoldi step).
__global__ void k_split_vec(int n, int ip, double *__restrict__ v, double *__restrict__ vp,
                            double *__restrict__ vs, const double *__restrict__ dinv, double beta,
                            double *__restrict__ x0, const double *__restrict__ nrm2) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 a = reinterpret_cast<const double2 *>(v)[i];
  if (nrm2) {
    double sc = 1.0 / sqrt(*nrm2);
    a.x = a.x * sc;
    a.y = a.y * sc;
    reinterpret_cast<double2 *>(v)[i] = a;
  }
  double s = ip ? a.x : a.y;
  vp[i] = ip ? a.y : a.x;
  vs[i] = s;
  x0[i] = beta * (s * dinv[i]);
}

// the last step of the BF apply on a DIA finest S~ level: one l1-Jacobi post-sweep
// p = x + (b - S~ x) ./ dl1 (the OP_SMOOTH arithmetic, beta = 1) written straight into the
// interleaved output with s: z = R_p^T p + R_s^T s (no p round trip, one launch less)
__global__ void __launch_bounds__(256) k_dia_smooth_merge(int n, DiaOffsets o, const double *__restrict__ dv,
                                                          const double *__restrict__ x,
                                                          const double *__restrict__ b,
                                                          const double *__restrict__ dinv,
                                                          const double *__restrict__ s, double2 *__restrict__ z,
                                                          int ip) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double eb = __ldg(b + r), ed = __ldg(dinv + r), ex = __ldg(x + r), es = __ldg(s + r);
  double acc = 0.0;
#pragma unroll 4
  for (int d = 0; d < o.k; d++) {
    int col = r + o.off[d];
    double a = __ldcs(dv + (size_t)d * n + r);
    if (col >= 0 && col < n) acc += a * __ldg(x + col);
  }
  double dn = 1.0 * ((eb - acc) * ed);
  double p = ex + dn;
  z[r] = ip ? make_double2(es, p) : make_double2(p, es);
}

__global__ void k_merge_vec(int n, int ip, const double *__restrict__ p, const double *__restrict__ s,
                            double *__restrict__ z) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  reinterpret_cast<double2 *>(z)[i] = ip ? make_double2(s[i], p[i]) : make_double2(p[i], s[i]);
}

void bf_apply(bf_ctx *c, const double *v, double *z, const double *nrm2) {
  if (c->opt.precond) {  // CPR-AMG(1)/(2), k_ilu.cu
    cpr_apply(c, v, z, nrm2);
    return;
  }
  int n = c->n;
  int ip = c->var_order;
  Hier &hs = c->h[0], &hS = c->h[1];
  // Alg. 3 step 2: A_ss s = R_s r_k by one V-cycle
  c->alg_bytes += 48.0 * n + 32.0 * n;  // split (v in; vp, vs, x0 out; dl1 in) + merge (p, s in; z out)
  k_split_vec<<<div_up(n, 256), 256, 0, c->stream>>>(n, ip, const_cast<double *>(v), c->vp, hs.lv[0].b,
                                                     hs.lv[0].d, hs.lv[0].beta0, hs.lv[0].x, nrm2);
  BF_LAUNCH(c);
  vcycle_level(c, hs, 0);
  // step 3: r = R_p r_k - A_ps s
  csr_op<OP_SUB_X0>(c, c->blk[1], hs.lv[0].x, c->vp, hS.lv[0].d, hS.lv[0].b, hS.lv[0].x, 0.0, hS.lv[0].beta0,
                    nullptr);
  // step 4: S~ p = r by one V-cycle.  With one l1-Jacobi post-sweep on a DIA finest level,
  // that sweep and the merge z = R_p^T p + R_s^T s are one kernel (k_dia_smooth_merge)
  Level &S0 = hS.lv[0];
  c->fuse_post0 = c->tune.merge_fuse && hS.lv[0].smoother == 0 && c->opt.nu_post == 1 && S0.A.dia_v && S0.A.dia_k <= 16 &&
                  hS.nlev > 1 && hS.dtail != 0 && hS.tail != 0;
  vcycle_level(c, hS, 0);
  if (c->fuse_post0) {
    c->fuse_post0 = false;
    DiaOffsets o;
    o.k = S0.A.dia_k;
    for (int d = 0; d < o.k; d++) o.off[d] = S0.A.dia_off[d];
    k_dia_smooth_merge<<<div_up(n, 256), 256, 0, c->stream>>>(n, o, S0.A.dia_v, S0.x, S0.b, S0.d, hs.lv[0].x,
                                                              reinterpret_cast<double2 *>(z), ip);
  } else {
    k_merge_vec<<<div_up(n, 256), 256, 0, c->stream>>>(n, ip, hS.lv[0].x, hs.lv[0].x, z);
  }
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

// algorithmic bytes of one BF apply, SURVEY.md 8(d)'s per-unit figures on the actual
// hierarchies: per level l < L of each V(1,1) 24 nnz(A_l) + 24 nnz(P_l) + 116 n_l + 12 n_{l+1},
// plus 12 nnz(A_l) + 36 n_l per extra sweep (a pass of a degree-m smoother is m sweeps, the first
// one from zero free: m (nu_pre + nu_post) products with A_l per level, of which V(1,1) counts 2),
// the coarsest solve 8 n_L^2, the A_ps coupling 12 nnz(A_ps) + 36 n, split + merge 64 n.
// Independent of the kernels' own storage (DIA, fused restriction), like the J SpMV's 36 B/block.
double apply_model_bytes(bf_ctx *c) {
  const bf_options &o = c->opt;
  double bytes = 12.0 * c->blk[1].nnz + 36.0 * c->n + 64.0 * c->n;
  for (int w = 0; w < 2; w++) {
    Hier &h = c->h[w];
    for (int l = 0; l + 1 < h.nlev; l++) {
      const int m = h.lv[l].smoother == 1 ? o.cheb_degree : 1;
      const double extra = std::max(0, m * (o.nu_pre + o.nu_post) - 2);
      bytes += 24.0 * h.lv[l].A.nnz + 24.0 * h.lv[l].P.nnz + 116.0 * h.lv[l].A.n + 12.0 * h.lv[l + 1].A.n +
               extra * (12.0 * h.lv[l].A.nnz + 36.0 * h.lv[l].A.n);
    }
    bytes += 8.0 * h.nL * h.nL;
  }
  return bytes;
}

// forget the captured BF apply (buffers of the finest level changed)
void drop_apply_graph(bf_ctx *c) {
  if (c->apply_exec) cudaGraphExecDestroy(c->apply_exec);
  if (c->apply_graph) cudaGraphDestroy(c->apply_graph);
  c->apply_exec = nullptr;
  c->apply_graph = nullptr;
  c->apply_patch.clear();
}

// Kernel arguments of the captured apply that change per launch: role 0 = the input vector v,
// 1 = the norm pointer for in-place normalisation, 2 = the output z.  The BF apply's only
// reader of v is the split kernel and its only writer of z the merge kernel; the CPR apply's
// are the ILU forward sweep, the residual kernel (v) and the merge kernel (z).
static bool patch_roles(const void *func, int &nargs, std::vector<std::pair<int, int>> &roles) {
  if (func == (const void *)k_split_vec) {
    nargs = nargs_of(k_split_vec);
    roles = {{2, 0}, {8, 1}};
  } else if (func == (const void *)k_merge_vec) {
    nargs = nargs_of(k_merge_vec);
    roles = {{4, 2}};
  } else if (func == (const void *)k_dia_smooth_merge) {
    nargs = nargs_of(k_dia_smooth_merge);
    roles = {{7, 2}};
  } else {
    return cpr_patch_roles(func, nargs, roles);
  }
  return true;
}

// The whole preconditioner apply (~40-60 kernels, most of them small coarse-level kernels)
// replayed as one CUDA graph: captured once per handle on a private stream, launched on the
// caller's stream.  Only v, the norm pointer and z change between applies; they are patched
// into the kernel nodes that take them.
void bf_apply_graph(bf_ctx *c, const double *v, double *z, const double *nrm2) {
  if (!c->apply_exec) {
    if (!c->cap_stream) BF_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = c->stream;
    c->stream = c->cap_stream;
    int64_t l0 = c->launches;
    BF_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    try {
      bf_apply(c, v, z, nrm2);
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(c->cap_stream, &g);
      if (g) cudaGraphDestroy(g);
      c->stream = user;
      throw;
    }
    cudaGraph_t g;
    BF_CUDA(cudaStreamEndCapture(c->cap_stream, &g));
    c->stream = user;
    c->apply_graph_kernels = c->launches - l0;
    c->apply_bytes = c->opt.precond ? cpr_model_bytes(c) : apply_model_bytes(c);
    c->launches = l0;
    BF_CUDA(cudaGraphInstantiate(&c->apply_exec, g, 0));
    size_t nn = 0;
    BF_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    BF_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
    c->apply_patch.clear();
    bool has_in = false, has_out = false;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      BF_CUDA(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams p;
      BF_CUDA(cudaGraphKernelNodeGetParams(nd, &p));
      bf_ctx::PatchNode pn;
      if (!patch_roles(p.func, pn.nargs, pn.roles)) continue;
      pn.node = nd;
      pn.params = p;
      for (auto &r : pn.roles) {
        has_in |= r.second == 0;
        has_out |= r.second == 2;
      }
      c->apply_patch.push_back(pn);
    }
    c->apply_graph = g;
    if (!has_in || !has_out) throw Error(BF_ERR_CUDA, "input/output nodes not found in the apply graph");
  }
  double *vin = const_cast<double *>(v);
  const double *nin = nrm2;
  double *zout = z;
  void *vals[3] = {(void *)&vin, (void *)&nin, (void *)&zout};
  for (auto &pn : c->apply_patch) {
    void *args[24];
    for (int k = 0; k < pn.nargs; k++) args[k] = pn.params.kernelParams[k];
    for (auto &r : pn.roles) args[r.first] = vals[r.second];
    cudaKernelNodeParams p = pn.params;
    p.kernelParams = args;
    BF_CUDA(cudaGraphExecKernelNodeSetParams(c->apply_exec, pn.node, &p));
  }
  cudaEvent_t t0;
  timer_begin(c, 2, &t0);
  BF_CUDA(cudaGraphLaunch(c->apply_exec, c->stream));
  timer_end(c, 2, t0, c->apply_bytes);
  c->launches += c->apply_graph_kernels;
}

}  // namespace bf
