// k_gmres.cu -- restarted right-preconditioned GMRES(m) (`precon-system`, P:L138-140;
// tolerance form P:L275; readings R10-R12) with classical Gram-Schmidt run twice (CGS2)
// fused into batched dot / axpy passes over the Krylov basis:
//   pass 1  h  = V_j^T w                              (reads j+1 basis vectors + w)
//   pass 2  w' = w - V_j h ;  h2 = V_j^T w'           (one read of V_j: axpy and dots fused)
//   pass 3  v  = w' - V_j h2 ; ||v||^2                (writes v_{j+1} unnormalised)
// Each pass ends in a deterministic two-level reduction (per-CTA partials, the last CTA to
// finish sums them in CTA order), so results are reproducible run to run.  One small
// device->host copy per Arnoldi step feeds the host-side Givens rotations (tiny, O(m)).
//
// Roofline: HBM-bound; algorithmic bytes per Arnoldi step with j+1 basis vectors of N f64:
//   pass 1: 8N (j+2), pass 2: 8N (j+3), pass 3: 8N (j+3)  (+ 16N for the scaling of v_{j+1}).
#include <cmath>
#include <cstring>
#include <algorithm>
#include <unordered_map>
#include <vector>

#include "bf_internal.cuh"

namespace bf {

constexpr int RED_THREADS = 256;
constexpr int MAXNV = 32;  // max basis vectors per pass -> restart <= 32

template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NV], double *partial, double *out, int nout,
                                                   unsigned int *counter) {
  __shared__ double sm[RED_THREADS / 32][NV];
  __shared__ bool last;
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; i++) {
    double v = acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sm[warp][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < RED_THREADS / 32; w++) s += sm[w][threadIdx.x];
    partial[(size_t)blockIdx.x * MAXNV + threadIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicInc(counter, gridDim.x - 1) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < nout) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; b++) s += __ldcg(partial + (size_t)b * MAXNV + threadIdx.x);
    out[threadIdx.x] = s;
  }
}

// The three passes are launched with programmatic dependent launch: the first grid-stride
// iteration's basis loads (V_0..V_j are complete before the predecessor kernel started) are
// issued before pdl_wait(); w and h (the predecessor's outputs) are read after it.

// pass 1: out[i] = V_i . w, i < NV
template <int NV>
__global__ void __launch_bounds__(RED_THREADS, 2) k_dots(int64_t N, const double *__restrict__ V,
                                                      const double *__restrict__ w, double *partial,
                                                      double *out, unsigned int *counter) {
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) acc[i] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v[NV];  // all NV loads in flight before the FMAs (memory-level parallelism)
  if (t < N) {
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = __ldcs(V + (size_t)i * N + t);
  }
  pdl_wait();
  for (; t < N; t += stride) {
    if (t != (int64_t)blockIdx.x * blockDim.x + threadIdx.x) {
#pragma unroll
      for (int i = 0; i < NV; i++) v[i] = __ldcs(V + (size_t)i * N + t);
    }
    double wt = __ldcs(w + t);
#pragma unroll
    for (int i = 0; i < NV; i++) acc[i] += v[i] * wt;
  }
  block_reduce_store<NV>(acc, partial, out, NV, counter);
}

// pass 2: w <- w - sum_i h_i V_i ; out[i] = V_i . w (new w)
template <int NV>
__global__ void __launch_bounds__(RED_THREADS, 2) k_axpy_dots(int64_t N, const double *__restrict__ V, double *w,
                                                           const double *__restrict__ h, double *partial,
                                                           double *out, unsigned int *counter) {
  __shared__ double hs[NV];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v[NV];
  if (t0 < N) {
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = __ldcs(V + (size_t)i * N + t0);
  }
  pdl_wait();
  if (threadIdx.x < NV) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) acc[i] = 0.0;
  for (int64_t t = t0; t < N; t += stride) {
    double wt = w[t];
    if (t != t0) {
#pragma unroll
      for (int i = 0; i < NV; i++) v[i] = __ldcs(V + (size_t)i * N + t);
    }
#pragma unroll
    for (int i = 0; i < NV; i++) wt -= hs[i] * v[i];
    w[t] = wt;
#pragma unroll
    for (int i = 0; i < NV; i++) acc[i] += v[i] * wt;
  }
  block_reduce_store<NV>(acc, partial, out, NV, counter);
}

// pass 3: y = w - sum_i h_i V_i written to `y` (may be the next basis slot); out[0] = ||y||^2
template <int NV>
__global__ void __launch_bounds__(RED_THREADS, 2) k_axpy_norm(int64_t N, const double *__restrict__ V,
                                                           const double *__restrict__ w,
                                                           const double *__restrict__ h, double *__restrict__ y,
                                                           double *partial, double *out, unsigned int *counter) {
  __shared__ double hs[NV];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v[NV];
  if (t0 < N) {
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = __ldcs(V + (size_t)i * N + t0);
  }
  pdl_wait();
  if (threadIdx.x < NV) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double acc[1] = {0.0};
  for (int64_t t = t0; t < N; t += stride) {
    if (t != t0) {
#pragma unroll
      for (int i = 0; i < NV; i++) v[i] = __ldcs(V + (size_t)i * N + t);
    }
    double wt = __ldcs(w + t);
#pragma unroll
    for (int i = 0; i < NV; i++) wt -= hs[i] * v[i];
    y[t] = wt;
    acc[0] += wt * wt;
  }
  block_reduce_store<1>(acc, partial, out, 1, counter);
}

// u = sum_i y_i V_i
template <int NV>
__global__ void k_lincomb(int64_t N, const double *__restrict__ V, const double *__restrict__ yv, double *u) {
  __shared__ double ys[NV];
  if (threadIdx.x < NV) ys[threadIdx.x] = yv[threadIdx.x];
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NV; i++) s += ys[i] * __ldcs(V + (size_t)i * N + t);
    u[t] = s;
  }
}

__global__ void k_scale(int64_t N, const double *__restrict__ a, const double *__restrict__ sptr, double s_host,
                        double *y) {
  double s = sptr ? 1.0 / sqrt(*sptr) : s_host;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    y[t] = a[t] * s;
}

__global__ void k_sub(int64_t N, const double *__restrict__ a, const double *__restrict__ b, double *y) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    y[t] = a[t] - b[t];
}

__global__ void k_add_inplace(int64_t N, double *x, const double *__restrict__ z) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    x[t] += z[t];
}

__global__ void k_zero_vec(int64_t N, double *x) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    x[t] = 0.0;
}

#define BF_NV_SWITCH(nv, CALL) \
  switch (nv) {                \
    BF_NV_C(1, CALL)           \
    BF_NV_C(2, CALL)           \
    BF_NV_C(3, CALL)           \
    BF_NV_C(4, CALL)           \
    BF_NV_C(5, CALL)           \
    BF_NV_C(6, CALL)           \
    BF_NV_C(7, CALL)           \
    BF_NV_C(8, CALL)           \
    BF_NV_C(9, CALL)           \
    BF_NV_C(10, CALL)          \
    BF_NV_C(11, CALL)          \
    BF_NV_C(12, CALL)          \
    BF_NV_C(13, CALL)          \
    BF_NV_C(14, CALL)          \
    BF_NV_C(15, CALL)          \
    BF_NV_C(16, CALL)          \
    BF_NV_C(17, CALL)          \
    BF_NV_C(18, CALL)          \
    BF_NV_C(19, CALL)          \
    BF_NV_C(20, CALL)          \
    BF_NV_C(21, CALL)          \
    BF_NV_C(22, CALL)          \
    BF_NV_C(23, CALL)          \
    BF_NV_C(24, CALL)          \
    BF_NV_C(25, CALL)          \
    BF_NV_C(26, CALL)          \
    BF_NV_C(27, CALL)          \
    BF_NV_C(28, CALL)          \
    BF_NV_C(29, CALL)          \
    BF_NV_C(30, CALL)          \
    BF_NV_C(31, CALL)          \
    BF_NV_C(32, CALL)          \
    default:                   \
      throw Error(BF_ERR_LIMIT, "GMRES basis block larger than 32"); \
  }
#define BF_NV_C(k, CALL) \
  case k: {              \
    constexpr int NV = k; \
    CALL;                \
  } break;

void alloc_solve_workspace(bf_ctx *c, int restart) {
  if (restart > MAXNV) throw Error(BF_ERR_ARG, "restart must be <= 32 (fused CGS2 basis passes)");
  int64_t N = 2 * (int64_t)c->n;
  if (!c->w) {
    c->w = dalloc_t<double>(c, N);
    c->z = dalloc_t<double>(c, N);
    c->r = dalloc_t<double>(c, N);
    c->xd = dalloc_t<double>(c, N);
    c->bd = dalloc_t<double>(c, N);
    c->vp = dalloc_t<double>(c, c->n);
    c->red_blocks = c->num_sms * 4;
    c->red = dalloc_t<double>(c, (size_t)c->red_blocks * MAXNV);
    c->hdev = dalloc_t<double>(c, 4 * MAXNV + 8);
    c->counter = dalloc_t<unsigned int>(c, 4);
    BF_CUDA(cudaMemsetAsync(c->counter, 0, 4 * sizeof(unsigned int), c->stream));
    c->hpin = pinned_acquire();  // 2 step slots of (2 MAXNV + 8) doubles + y staging
    for (int s = 0; s < 2; s++) BF_CUDA(cudaEventCreateWithFlags(&c->step_ev[s], cudaEventDisableTiming));
  }
  if (c->Vm < restart + 1) {
    dfree(c, c->V);
    c->V = dalloc_t<double>(c, (size_t)(restart + 1) * N);
    dfree(c, c->Z);
    c->Z = dalloc_t<double>(c, (size_t)restart * N);
    c->Vm = restart + 1;
  }
}

static int grid_for(bf_ctx *c) { return c->red_blocks; }

// one full wave: SMs x resident CTAs of this kernel (no partial second wave for the
// grid-stride reductions), capped by the partial-sum buffer (4 CTAs per SM)
template <class K>
static int wave_grid(bf_ctx *c, K kernel) {
  static std::unordered_map<const void *, int> cache;
  auto it = cache.find((const void *)kernel);
  int per_sm;
  if (it == cache.end()) {
    BF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, RED_THREADS, 0));
    cache[(const void *)kernel] = per_sm;
  } else {
    per_sm = it->second;
  }
  per_sm = std::max(1, std::min(per_sm, 4));
  return c->num_sms * per_sm;
}

// out = a . b  (host value, synchronises); the device copy lands in `dst` (default scratch)
static double dot_host(bf_ctx *c, const double *a, const double *b, double *dst = nullptr) {
  int64_t N = 2 * (int64_t)c->n;
  if (!dst) dst = c->hdev + 3 * MAXNV;
  k_dots<1><<<wave_grid(c, k_dots<1>), RED_THREADS, 0, c->stream>>>(N, a, b, c->red, dst, c->counter);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  BF_CUDA(cudaMemcpyAsync(c->hpin, dst, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaStreamSynchronize(c->stream));
  return c->hpin[0];
}

void gmres(bf_ctx *c, const double *b, double *x, double tol, int m, int maxit, int *iters, double *hist,
           int *converged, double *relres) {
  int64_t N = 2 * (int64_t)c->n;
  int G = grid_for(c);
  double *V = c->V;
  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), y(m), hcol(m + 1);
  *iters = 0;
  *converged = 0;
  double bnorm = std::sqrt(dot_host(c, b, b));
  if (bnorm == 0.0) {
    k_zero_vec<<<G, 256, 0, c->stream>>>(N, x);
    BF_LAUNCH(c);
    if (hist) hist[0] = 0.0;
    *converged = 1;
    *relres = 0.0;
    return;
  }
  double *hd1 = c->hdev, *hd2 = c->hdev + MAXNV, *hdn = c->hdev + 2 * MAXNV;
  // r = b - J x, written straight into the basis slot v_0 (normalised by the first split)
  bsr_spmv(c, x, c->w);
  k_sub<<<G, 256, 0, c->stream>>>(N, b, c->w, V);
  BF_LAUNCH(c);
  double beta = std::sqrt(dot_host(c, V, V, hdn));
  if (hist) hist[0] = beta / bnorm;
  *relres = beta / bnorm;
  if (beta <= tol * bnorm) {
    *converged = 1;
    return;
  }
  // Arnoldi step j, enqueued without waiting for the host: z_j = M^-1 v_j, w = J z_j, CGS2,
  // v_{j+1} = w / ||w|| (norm taken on the device, applied by the next step's split kernel), then an async copy of (h, h2, ||w||^2)
  // into pinned slot j%2 and an event.  The host processes step j (Givens, convergence) while
  // step j+1 already runs; a step enqueued past the stopping point is simply discarded.
  const int SLOT = 2 * MAXNV + 8;
  auto enqueue = [&](int j) {
    // sampled instrumentation (opt.timing = k > 1): events around every k-th step only, so the
    // timed region is barely perturbed; per-launch averages stay representative
    c->timing_skip = c->opt.timing > 1 && (c->timing_step++ % c->opt.timing) != 0;
    const double *vj = V + (size_t)j * N;
    double *vn = V + (size_t)(j + 1) * N;
    double *zj = c->Z + (size_t)j * N;
    // z_j = M^-1 v_j, kept for the cycle-end update; the split kernel first normalises the
    // slot v_j in place by 1/sqrt(*hdn) (||v_j||^2 from the previous step's pass 3, or the
    // restart residual's norm)
    bf_apply_graph(c, vj, zj, hdn);
    cudaEvent_t t0;
    timer_begin(c, 0, &t0);
    bsr_spmv(c, zj, c->w);  // w = J z_j
    timer_end(c, 0, t0, 36.0 * c->nnzb + 36.0 * c->n);
    int nv = j + 1;
    timer_begin(c, 1, &t0);
    const double *Vc = V;
    BF_NV_SWITCH(nv, (launch_pdl(c, k_dots<NV>, dim3(wave_grid(c, k_dots<NV>)), dim3(RED_THREADS), 0, N, Vc,
                                 (const double *)c->w, c->red, hd1, c->counter)));
    if (c->opt.orth == 0) {
      BF_NV_SWITCH(nv, (launch_pdl(c, k_axpy_dots<NV>, dim3(wave_grid(c, k_axpy_dots<NV>)), dim3(RED_THREADS), 0, N,
                                   Vc, c->w, (const double *)hd1, c->red, hd2, c->counter)));
      BF_NV_SWITCH(nv, (launch_pdl(c, k_axpy_norm<NV>, dim3(wave_grid(c, k_axpy_norm<NV>)), dim3(RED_THREADS), 0, N,
                                   Vc, (const double *)c->w, (const double *)hd2, vn, c->red, hdn, c->counter)));
    } else {
      BF_NV_SWITCH(nv, (launch_pdl(c, k_axpy_norm<NV>, dim3(wave_grid(c, k_axpy_norm<NV>)), dim3(RED_THREADS), 0, N,
                                   Vc, (const double *)c->w, (const double *)hd1, vn, c->red, hdn, c->counter)));
    }
    c->launches += c->opt.orth == 0 ? 3 : 2;
    timer_end(c, 1, t0, 8.0 * N * (c->opt.orth == 0 ? 3.0 * nv + 5.0 : 2.0 * nv + 3.0));
    BF_CUDA(cudaGetLastError());
    BF_CUDA(cudaMemcpyAsync(c->hpin + (j & 1) * SLOT, c->hdev, sizeof(double) * (2 * MAXNV + 1),
                            cudaMemcpyDeviceToHost, c->stream));
    BF_CUDA(cudaEventRecord(c->step_ev[j & 1], c->stream));
    c->timing_skip = false;
  };
  for (;;) {
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k = 0;
    bool breakdown = false;
    enqueue(0);
    for (int j = 0; j < m; j++) {
      if (j + 1 < m && *iters + 1 < maxit) enqueue(j + 1);  // speculative next step
      BF_CUDA(cudaEventSynchronize(c->step_ev[j & 1]));
      const double *hp = c->hpin + (j & 1) * SLOT;
      double hn = std::sqrt(hp[2 * MAXNV]);
      for (int i = 0; i <= j; i++) hcol[i] = hp[i] + (c->opt.orth == 0 ? hp[MAXNV + i] : 0.0);
      if (hn == 0.0) breakdown = true;  // (happy) breakdown: the speculative step is discarded
      for (int i = 0; i <= j; i++) H[(size_t)i * m + j] = hcol[i];
      H[(size_t)(j + 1) * m + j] = hn;
      for (int i = 0; i < j; i++) {  // previous Givens rotations
        double a = H[(size_t)i * m + j], bb = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a + sn[i] * bb;
        H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
      }
      double a = H[(size_t)j * m + j], bb = H[(size_t)(j + 1) * m + j];
      double t = std::hypot(a, bb);
      if (t == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = a / t;
        sn[j] = bb / t;
      }
      H[(size_t)j * m + j] = cs[j] * a + sn[j] * bb;
      H[(size_t)(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      (*iters)++;
      if (hist) hist[*iters] = std::fabs(g[j + 1]) / bnorm;
      k = j + 1;
      if (std::fabs(g[j + 1]) <= tol * bnorm || *iters >= maxit || breakdown) break;
    }
    // y = H^-1 g ; x += M^-1 (V y)
    for (int i = k - 1; i >= 0; i--) {
      double s = g[i];
      for (int jj = i + 1; jj < k; jj++) s -= H[(size_t)i * m + jj] * y[jj];
      y[i] = H[(size_t)i * m + i] != 0.0 ? s / H[(size_t)i * m + i] : 0.0;
    }
    double *ypin = c->hpin + 2 * SLOT;
    for (int i = 0; i < k; i++) ypin[i] = y[i];
    BF_CUDA(cudaMemcpyAsync(c->hdev + MAXNV, ypin, sizeof(double) * k, cudaMemcpyHostToDevice, c->stream));
    // x += M^-1 (V y) = Z y  (M^-1 is a fixed linear operator: no extra BF apply per cycle)
    BF_NV_SWITCH(k, (k_lincomb<NV><<<G, 256, 0, c->stream>>>(N, c->Z, c->hdev + MAXNV, c->z)));
    BF_LAUNCH(c);
    k_add_inplace<<<G, 256, 0, c->stream>>>(N, x, c->z);
    BF_LAUNCH(c);
    // true residual at the end of the cycle (R11)
    bsr_spmv(c, x, c->w);
    k_sub<<<G, 256, 0, c->stream>>>(N, b, c->w, V);
    BF_LAUNCH(c);
    beta = std::sqrt(dot_host(c, V, V, hdn));
    *relres = beta / bnorm;
    if (beta <= tol * bnorm) {
      *converged = 1;
      break;
    }
    if (*iters >= maxit) break;
    if (beta == 0.0) {
      *converged = 1;
      break;
    }
  }
}

}  // namespace bf
