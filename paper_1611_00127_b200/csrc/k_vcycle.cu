// k_vcycle.cu -- the AMG V(nu_pre, nu_post) cycle (one cycle per inner solve)
// with l1-Jacobi or Chebyshev smoothing (replacing the paper's hybrid Gauss-Seidel,
// DESIGN.md R9), restriction b_c = R r, prolongation x += P e and the shared-memory
// staged dense coarse solve; and the BF preconditioner apply, Algorithm 3:
//   s = V_Ass(R_s v);  r' = R_p v - A_ps s;  p = V_S~(r');  z = R_p^T p + R_s^T s.
#include "bf_internal.cuh"
#include "k_spmv.cuh"

namespace bf {

// forward/back substitution with the LU of the coarsest matrix, one CTA, staged in smem
__global__ void k_coarse_solve(int n, const double *__restrict__ lu, const int32_t *__restrict__ piv,
                               const double *__restrict__ b, double *__restrict__ x) {
  extern __shared__ double sm[];
  double *L = sm;          // n*n
  double *y = sm + n * n;  // n
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) L[e] = lu[e];
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = b[i];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < n; k++) {
      int p = piv[k];
      if (p != k) {
        double t = y[k];
        y[k] = y[p];
        y[p] = t;
      }
    }
  __syncthreads();
  for (int k = 0; k < n; k++) {  // L (unit) forward, column oriented
    double yk = y[k];
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) y[i] -= L[i * n + k] * yk;
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; k--) {  // U backward
    if (threadIdx.x == 0) y[k] = y[k] / L[k * n + k];
    __syncthreads();
    double yk = y[k];
    for (int i = threadIdx.x; i < k; i += blockDim.x) y[i] -= L[i * n + k] * yk;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = y[i];
}

__global__ void k_zero(int n, double *x) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = 0.0;
}

// one smoothing pass (l1-Jacobi, or Chebyshev of degree m on [lo,1]) on level L; x in/out.
// from_zero: x == 0 on entry.  If want_resid, also leaves r = b - A x in L.r (fused when possible).
static void smooth_pass(bf_ctx *c, Level &L, double *&x, bool from_zero, bool want_resid) {
  const bf_options &o = c->opt;
  int n = L.A.n;
  if (o.smoother == 0) {  // x <- x + (b - A x) ./ dl1
    if (from_zero) {
      if (want_resid) {
        csr_op<OP_SMOOTH0_RESID>(c, L.A, nullptr, L.b, L.d, L.r, x, 0.0, 1.0, nullptr);
        return;
      }
      // x = b ./ d  (SMOOTH with x = 0 would read x): use the fused kernel and drop r
      csr_op<OP_SMOOTH0_RESID>(c, L.A, nullptr, L.b, L.d, L.r, x, 0.0, 1.0, nullptr);
      return;
    }
    csr_op<OP_SMOOTH>(c, L.A, x, L.b, L.d, L.t, nullptr, 0.0, 1.0, nullptr);
    double *tmp = x;
    x = L.t;
    L.t = tmp;
  } else {  // Chebyshev acceleration of D^-1 A on [lo, 1] (three-term recurrence)
    double lo = o.cheb_lo, theta = (1.0 + lo) / 2.0, delta = (1.0 - lo) / 2.0, sigma = theta / delta;
    double rho = 1.0 / sigma;
    double *dir = L.r;  // direction storage (r is recomputed below when needed)
    if (from_zero) {
      // dir = (1/theta) b/d ; x = dir
      csr_op<OP_SMOOTH0_RESID>(c, L.A, nullptr, L.b, L.d, L.t /*scratch r*/, x, 0.0, 1.0 / theta, nullptr);
      BF_CUDA(cudaMemcpyAsync(dir, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    } else {
      csr_op<OP_SMOOTH>(c, L.A, x, L.b, L.d, L.t, dir, 0.0, 1.0 / theta, nullptr);
      double *tmp = x;
      x = L.t;
      L.t = tmp;
    }
    for (int k = 1; k < o.cheb_degree; k++) {
      double rho_new = 1.0 / (2.0 * sigma - rho);
      csr_op<OP_SMOOTH>(c, L.A, x, L.b, L.d, L.t, dir, rho_new * rho, 2.0 * rho_new / delta, dir);
      double *tmp = x;
      x = L.t;
      L.t = tmp;
      rho = rho_new;
    }
  }
  if (want_resid) csr_op<OP_RESID>(c, L.A, x, L.b, nullptr, L.r, nullptr, 0.0, 0.0, nullptr);
}

// V-cycle on level l with rhs in L.b; result left in L.x (pointer may be swapped with L.t)
static void vcycle_level(bf_ctx *c, Hier &h, int l) {
  Level &L = h.lv[l];
  int n = L.A.n;
  const bf_options &o = c->opt;
  if (l == h.nlev - 1) {
    if (h.dense) {
      size_t smem = sizeof(double) * ((size_t)n * n + n);
      k_coarse_solve<<<1, 128, smem, c->stream>>>(n, h.lu, h.piv, L.b, L.x);
      BF_LAUNCH(c);
      BF_CUDA(cudaGetLastError());
    } else {  // stalled coarsening: 4 l1-Jacobi sweeps from zero
      csr_op<OP_SMOOTH0_RESID>(c, L.A, nullptr, L.b, L.d, L.r, L.x, 0.0, 1.0, nullptr);
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
    for (int s = 0; s < o.nu_pre; s++) smooth_pass(c, L, x, s == 0, s == o.nu_pre - 1);
  }
  Level &Lc = h.lv[l + 1];
  csr_op<OP_SPMV>(c, L.R, L.r, nullptr, nullptr, Lc.b, nullptr, 0.0, 0.0, nullptr);  // b_c = R r
  vcycle_level(c, h, l + 1);
  csr_op<OP_ADD>(c, L.P, Lc.x, nullptr, nullptr, x, nullptr, 0.0, 0.0, nullptr);  // x += P e
  for (int s = 0; s < o.nu_post; s++) smooth_pass(c, L, x, false, false);
  if (x != L.x) {  // keep the result in L.x (swap the buffers, no copy)
    L.t = L.x;
    L.x = x;
  }
}

void vcycle(bf_ctx *c, int which, const double *b, double *x) {
  Hier &h = c->h[which];
  Level &L0 = h.lv[0];
  BF_CUDA(cudaMemcpyAsync(L0.b, b, sizeof(double) * L0.A.n, cudaMemcpyDeviceToDevice, c->stream));
  vcycle_level(c, h, 0);
  BF_CUDA(cudaMemcpyAsync(x, L0.x, sizeof(double) * L0.A.n, cudaMemcpyDeviceToDevice, c->stream));
}

// R_s v -> bs, R_p v -> vp (interleaved in the caller's var_order)
__global__ void k_split_vec(int n, int ip, const double *__restrict__ v, double *__restrict__ vp,
                            double *__restrict__ vs) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 a = reinterpret_cast<const double2 *>(v)[i];
  vp[i] = ip ? a.y : a.x;
  vs[i] = ip ? a.x : a.y;
}

__global__ void k_merge_vec(int n, int ip, const double *__restrict__ p, const double *__restrict__ s,
                            double *__restrict__ z) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  reinterpret_cast<double2 *>(z)[i] = ip ? make_double2(s[i], p[i]) : make_double2(p[i], s[i]);
}

void bf_apply(bf_ctx *c, const double *v, double *z) {
  int n = c->n;
  int ip = c->var_order;
  Hier &hs = c->h[0], &hS = c->h[1];
  // Alg. 3 step 2: A_ss s = R_s r_k by one V-cycle
  k_split_vec<<<div_up(n, 256), 256, 0, c->stream>>>(n, ip, v, c->vp, hs.lv[0].b);
  BF_LAUNCH(c);
  vcycle_level(c, hs, 0);
  // step 3: r = R_p r_k - A_ps s
  csr_op<OP_SUB>(c, c->blk[1], hs.lv[0].x, c->vp, nullptr, hS.lv[0].b, nullptr, 0.0, 0.0, nullptr);
  // step 4: S~ p = r by one V-cycle
  vcycle_level(c, hS, 0);
  k_merge_vec<<<div_up(n, 256), 256, 0, c->stream>>>(n, ip, hS.lv[0].x, hs.lv[0].x, z);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

}  // namespace bf
