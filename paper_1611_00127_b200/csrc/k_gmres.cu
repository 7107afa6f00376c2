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
BF_CHECK_TU("k_gmres.cu")

namespace bf {

constexpr int RED_THREADS = 256;
constexpr int MAXNV = 32;     // basis vectors per fused pass; longer bases are processed in blocks of 32
constexpr int MAX_RESTART = 256;

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
//
// Vectors are read as double2 (N = 2 n_cells is even and every basis vector starts 16-B
// aligned), and a thread handles UNR(NV) grid-stride elements per iteration with all their
// loads issued before the first FMA: for short bases (the first Arnoldi steps of a cycle) a
// single element per thread leaves too few bytes in flight to cover the DRAM latency
// (round 1 measured k_dots<1> at 25 % of the copy bandwidth).
template <int NV>
struct Unr {
  static constexpr int U = NV <= 2 ? 4 : (NV <= 5 ? 2 : 1);
};

// pass 1: out[i] = V_i . w, i < NV
template <int NV>
__device__ __forceinline__ void dots_v2(int64_t N, const double *__restrict__ V,
                                                      const double *__restrict__ w, double *partial,
                                                      double *out, unsigned int *counter) {
  constexpr int U = Unr<NV>::U;
  const int64_t N2 = N >> 1;
  const double2 *__restrict__ V2 = reinterpret_cast<const double2 *>(V);
  const double2 *__restrict__ w2 = reinterpret_cast<const double2 *>(w);
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) acc[i] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double2 v[U][NV];
#pragma unroll
  for (int u = 0; u < U; u++)
    if (t0 + u * stride < N2) {
#pragma unroll
      for (int i = 0; i < NV; i++) v[u][i] = __ldcs(V2 + (size_t)i * N2 + t0 + u * stride);
    }
  pdl_wait();
  for (int64_t t = t0; t < N2; t += U * stride) {
    if (t != t0) {
#pragma unroll
      for (int u = 0; u < U; u++)
        if (t + u * stride < N2) {
#pragma unroll
          for (int i = 0; i < NV; i++) v[u][i] = __ldcs(V2 + (size_t)i * N2 + t + u * stride);
        }
    }
    double2 wt[U];
#pragma unroll
    for (int u = 0; u < U; u++) wt[u] = t + u * stride < N2 ? __ldcs(w2 + t + u * stride) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (t + u * stride < N2) {
#pragma unroll
        for (int i = 0; i < NV; i++) acc[i] += v[u][i].x * wt[u].x + v[u][i].y * wt[u].y;
      }
  }
  block_reduce_store<NV>(acc, partial, out, NV, counter);
}

// pass 2: w <- w - sum_i h_i V_i ; out[i] = V_i . w (new w)
template <int NV>
__device__ __forceinline__ void axpy_dots_v2(int64_t N, const double *__restrict__ V, double *w,
                                                           const double *__restrict__ h, double *partial,
                                                           double *out, unsigned int *counter) {
  constexpr int U = Unr<NV>::U;
  __shared__ double hs[NV];
  const int64_t N2 = N >> 1;
  const double2 *__restrict__ V2 = reinterpret_cast<const double2 *>(V);
  double2 *w2 = reinterpret_cast<double2 *>(w);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double2 v[U][NV];
#pragma unroll
  for (int u = 0; u < U; u++)
    if (t0 + u * stride < N2) {
#pragma unroll
      for (int i = 0; i < NV; i++) v[u][i] = __ldcs(V2 + (size_t)i * N2 + t0 + u * stride);
    }
  pdl_wait();
  if (threadIdx.x < NV) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) acc[i] = 0.0;
  for (int64_t t = t0; t < N2; t += U * stride) {
    double2 wt[U];
#pragma unroll
    for (int u = 0; u < U; u++) wt[u] = t + u * stride < N2 ? w2[t + u * stride] : make_double2(0.0, 0.0);
    if (t != t0) {
#pragma unroll
      for (int u = 0; u < U; u++)
        if (t + u * stride < N2) {
#pragma unroll
          for (int i = 0; i < NV; i++) v[u][i] = __ldcs(V2 + (size_t)i * N2 + t + u * stride);
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++)
      if (t + u * stride < N2) {
        double2 a = wt[u];
#pragma unroll
        for (int i = 0; i < NV; i++) {
          a.x -= hs[i] * v[u][i].x;
          a.y -= hs[i] * v[u][i].y;
        }
        w2[t + u * stride] = a;
#pragma unroll
        for (int i = 0; i < NV; i++) acc[i] += v[u][i].x * a.x + v[u][i].y * a.y;
      }
  }
  block_reduce_store<NV>(acc, partial, out, NV, counter);
}

// pass 3: y = w - sum_i h_i V_i written to `y` (may be the next basis slot); out[0] = ||y||^2
template <int NV>
__device__ __forceinline__ void axpy_norm_v2(int64_t N, const double *__restrict__ V,
                                                           const double *__restrict__ w,
                                                           const double *__restrict__ h, double *__restrict__ y,
                                                           double *partial, double *out, unsigned int *counter) {
  constexpr int U = Unr<NV>::U;
  __shared__ double hs[NV];
  const int64_t N2 = N >> 1;
  const double2 *__restrict__ V2 = reinterpret_cast<const double2 *>(V);
  const double2 *__restrict__ w2 = reinterpret_cast<const double2 *>(w);
  double2 *__restrict__ y2 = reinterpret_cast<double2 *>(y);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double2 v[U][NV];
#pragma unroll
  for (int u = 0; u < U; u++)
    if (t0 + u * stride < N2) {
#pragma unroll
      for (int i = 0; i < NV; i++) v[u][i] = __ldcs(V2 + (size_t)i * N2 + t0 + u * stride);
    }
  pdl_wait();
  if (threadIdx.x < NV) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double acc[1] = {0.0};
  for (int64_t t = t0; t < N2; t += U * stride) {
    if (t != t0) {
#pragma unroll
      for (int u = 0; u < U; u++)
        if (t + u * stride < N2) {
#pragma unroll
          for (int i = 0; i < NV; i++) v[u][i] = __ldcs(V2 + (size_t)i * N2 + t + u * stride);
        }
    }
    double2 wt[U];
#pragma unroll
    for (int u = 0; u < U; u++) wt[u] = t + u * stride < N2 ? __ldcs(w2 + t + u * stride) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (t + u * stride < N2) {
        double2 a = wt[u];
#pragma unroll
        for (int i = 0; i < NV; i++) {
          a.x -= hs[i] * v[u][i].x;
          a.y -= hs[i] * v[u][i].y;
        }
        y2[t + u * stride] = a;
        acc[0] += a.x * a.x + a.y * a.y;
      }
  }
  block_reduce_store<1>(acc, partial, out, 1, counter);
}

// scalar bodies (bases longer than 8 vectors: NV loads per element already keep enough bytes in flight)
// pass 1: out[i] = V_i . w, i < NV
template <int NV>
__device__ __forceinline__ void dots_s(int64_t N, const double *__restrict__ V,
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
__device__ __forceinline__ void axpy_dots_s(int64_t N, const double *__restrict__ V, double *w,
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
__device__ __forceinline__ void axpy_norm_s(int64_t N, const double *__restrict__ V,
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

// the kernels: double2 bodies with UNR-fold unrolling for short bases, scalar bodies otherwise
template <int NV>
__global__ void __launch_bounds__(RED_THREADS, 2) k_dots(int64_t N, const double *__restrict__ V,
                                                      const double *__restrict__ w, double *partial,
                                                      double *out, unsigned int *counter) {
  if constexpr (NV <= 8) dots_v2<NV>(N, V, w, partial, out, counter);
  else dots_s<NV>(N, V, w, partial, out, counter);
}
template <int NV>
__global__ void __launch_bounds__(RED_THREADS, 2) k_axpy_dots(int64_t N, const double *__restrict__ V, double *w,
                                                           const double *__restrict__ h, double *partial,
                                                           double *out, unsigned int *counter) {
  if constexpr (NV <= 8) axpy_dots_v2<NV>(N, V, w, h, partial, out, counter);
  else axpy_dots_s<NV>(N, V, w, h, partial, out, counter);
}
template <int NV>
__global__ void __launch_bounds__(RED_THREADS, 2) k_axpy_norm(int64_t N, const double *__restrict__ V,
                                                           const double *__restrict__ w,
                                                           const double *__restrict__ h, double *__restrict__ y,
                                                           double *partial, double *out, unsigned int *counter) {
  if constexpr (NV <= 8) axpy_norm_v2<NV>(N, V, w, h, y, partial, out, counter);
  else axpy_norm_s<NV>(N, V, w, h, y, partial, out, counter);
}

// w <- w - sum_i h_i V_i (one block of a basis longer than MAXNV; no reduction)
template <int NV>
__global__ void __launch_bounds__(RED_THREADS) k_axpy(int64_t N, const double *__restrict__ V, double *w,
                                                     const double *__restrict__ h) {
  __shared__ double hs[NV];
  pdl_wait();
  if (threadIdx.x < NV) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = __ldcs(V + (size_t)i * N + t);
    double wt = w[t];
#pragma unroll
    for (int i = 0; i < NV; i++) wt -= hs[i] * v[i];
    w[t] = wt;
  }
}

// u = sum_i y_i V_i (acc = 0) or u += sum_i y_i V_i (acc = 1)
template <int NV>
__global__ void k_lincomb(int64_t N, const double *__restrict__ V, const double *__restrict__ yv, double *u, int acc) {
  __shared__ double ys[NV];
  if (threadIdx.x < NV) ys[threadIdx.x] = yv[threadIdx.x];
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    double s = acc ? u[t] : 0.0;
#pragma unroll
    for (int i = 0; i < NV; i++) s += ys[i] * __ldcs(V + (size_t)i * N + t);
    u[t] = s;
  }
}

// index of the first non-finite entry (error reporting only)
__global__ void k_first_nonfinite(int64_t N, const double *__restrict__ a, unsigned long long *first) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(a[t])) atomicMin(first, (unsigned long long)t);
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
      throw Error(BF_ERR_LIMIT, "GMRES basis block larger than 32 (internal)"); \
  }
#define BF_NV_C(k, CALL) \
  case k: {              \
    constexpr int NV = k; \
    CALL;                \
  } break;

// Coefficient layout (device hdev and each pinned host step slot): h at [0, hs), h' at [hs, 2 hs),
// ||v||^2 at [2 hs]; hs = restart + 1 rounded up to a multiple of 32 (block offsets stay aligned).
static int hstride(int restart) { return ((restart + 1 + MAXNV - 1) / MAXNV) * MAXNV; }

void alloc_solve_workspace(bf_ctx *c, int restart) {
  if (restart < 1 || restart > MAX_RESTART)
    throw Error(BF_ERR_ARG, "restart must be in [1, " + std::to_string(MAX_RESTART) + "]");
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
    c->counter = dalloc_t<unsigned int>(c, 4);
    c->nonfinite = dalloc_t<unsigned long long>(c, 1);
    BF_CUDA(cudaMemsetAsync(c->counter, 0, 4 * sizeof(unsigned int), c->stream));
    for (int s = 0; s < 2; s++) BF_CUDA(cudaEventCreateWithFlags(&c->step_ev[s], cudaEventDisableTiming));
  }
  if (c->Vm < restart + 1) {
    dfree(c, c->V);
    c->V = dalloc_t<double>(c, (size_t)(restart + 1) * N);
    dfree(c, c->Z);
    c->Z = dalloc_t<double>(c, (size_t)restart * N);
    c->Vm = restart + 1;
    const int hs = hstride(restart);
    dfree(c, c->hdev);
    c->hdev = dalloc_t<double>(c, 2 * (size_t)hs + 8 + MAXNV);
    // pinned host: two step slots of (2 hs + 8) doubles and the y staging area (hs doubles)
    const size_t pin_bytes = sizeof(double) * (2 * (2 * (size_t)hs + 8) + hs);
    if (c->hpin && c->hpin_bytes < pin_bytes) {
      pinned_release(c->hpin, c->hpin_bytes);
      c->hpin = nullptr;
    }
    if (!c->hpin) {
      c->hpin = pinned_acquire(pin_bytes, &c->hpin_bytes);
    }
  }
}

static int grid_for(bf_ctx *c) { return c->red_blocks; }

// one full wave: SMs x resident CTAs of this kernel (no partial second wave for the
// grid-stride reductions), capped by the partial-sum buffer (4 CTAs per SM)
template <class K>
static int wave_grid(bf_ctx *c, K kernel) {
  int per_sm = std::max(1, std::min(occupancy(c, (const void *)kernel, RED_THREADS, 0), 4));
  return c->num_sms * per_sm;
}

// out = a . b  (host value, synchronises); the device copy lands in `dst` (default scratch)
static double dot_host(bf_ctx *c, const double *a, const double *b, double *dst = nullptr) {
  int64_t N = 2 * (int64_t)c->n;
  if (!dst) dst = c->hdev + 2 * hstride(c->Vm - 1) + 4;
  k_dots<1><<<wave_grid(c, k_dots<1>), RED_THREADS, 0, c->stream>>>(N, a, b, c->red, dst, c->counter);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  BF_CUDA(cudaMemcpyAsync(c->hpin, dst, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaStreamSynchronize(c->stream));
  return c->hpin[0];
}

// first non-finite entry of a device vector (error path only): "entry k (cell c, p|S)"
static std::string nonfinite_where(bf_ctx *c, const double *a) {
  int64_t N = 2 * (int64_t)c->n;
  BF_CUDA(cudaMemsetAsync(c->nonfinite, 0xff, sizeof(unsigned long long), c->stream));
  k_first_nonfinite<<<grid_for(c), 256, 0, c->stream>>>(N, a, c->nonfinite);
  BF_LAUNCH(c);
  unsigned long long k = ~0ull;
  BF_CUDA(cudaMemcpyAsync(&k, c->nonfinite, sizeof(k), cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaStreamSynchronize(c->stream));
  if (k == ~0ull) return "(no non-finite entry: the squared 2-norm overflows)";
  int which = (int)(k & 1) ^ c->var_order;  // 0: p_w slot, 1: S_n slot of the caller's interleaving
  return "entry " + std::to_string(k) + " (cell " + std::to_string(k / 2) + ", " + (which ? "S_n" : "p_w") + ")";
}

// CGS2 / CGS1 orthogonalisation of w against the nv basis vectors V_0..V_{nv-1} (P:L138-140,
// reading R11 / Q30), writing h -> hd1[0..nv), h' -> hd2[0..nv), the unnormalised v_{j+1} -> vn
// and ||v_{j+1}||^2 -> *hdn.  nv <= 32: the three fused passes; longer bases in blocks of 32
// (pass 1: one dot kernel per block; pass 2: axpy over all blocks but the last, the fused
// axpy+dots of the last block, then the dots of the earlier blocks with the final w; pass 3:
// axpy over all blocks but the last, then the fused axpy+norm of the last block).
static void orthogonalise(bf_ctx *c, int nv, double *hd1, double *hd2, double *hdn, double *vn) {
  const int64_t N = 2 * (int64_t)c->n;
  const double *V = c->V;
  const bool cgs2 = c->opt.orth == 0;
  const int nb = (nv + MAXNV - 1) / MAXNV;           // blocks of <= 32 vectors
  auto blk = [&](int q) { return V + (size_t)q * MAXNV * N; };
  auto bn = [&](int q) { return std::min(MAXNV, nv - q * MAXNV); };
  for (int q = 0; q < nb; q++) {                     // pass 1: h = V^T w
    const double *Vq = blk(q);
    BF_NV_SWITCH(bn(q), (launch_pdl(c, k_dots<NV>, dim3(wave_grid(c, k_dots<NV>)), dim3(RED_THREADS), 0, N, Vq,
                                    (const double *)c->w, c->red, hd1 + q * MAXNV, c->counter)));
    BF_LAUNCH(c);
  }
  const double *hlast = hd1;                         // coefficients of the final pass
  if (cgs2) {                                        // pass 2: w -= V h, h' = V^T w
    for (int q = 0; q + 1 < nb; q++) {
      const double *Vq = blk(q);
      launch_pdl(c, k_axpy<MAXNV>, dim3(grid_for(c)), dim3(RED_THREADS), 0, N, Vq, c->w,
                 (const double *)(hd1 + q * MAXNV));
      BF_LAUNCH(c);
    }
    const int ql = nb - 1;
    const double *Vl = blk(ql);
    BF_NV_SWITCH(bn(ql), (launch_pdl(c, k_axpy_dots<NV>, dim3(wave_grid(c, k_axpy_dots<NV>)), dim3(RED_THREADS), 0,
                                     N, Vl, c->w, (const double *)(hd1 + ql * MAXNV), c->red, hd2 + ql * MAXNV,
                                     c->counter)));
    BF_LAUNCH(c);
    for (int q = 0; q + 1 < nb; q++) {
      const double *Vq = blk(q);
      launch_pdl(c, k_dots<MAXNV>, dim3(wave_grid(c, k_dots<MAXNV>)), dim3(RED_THREADS), 0, N, Vq,
                 (const double *)c->w, c->red, hd2 + q * MAXNV, c->counter);
      BF_LAUNCH(c);
    }
    hlast = hd2;
  }
  for (int q = 0; q + 1 < nb; q++) {                 // pass 3: v = w - V h(') , ||v||^2
    const double *Vq = blk(q);
    launch_pdl(c, k_axpy<MAXNV>, dim3(grid_for(c)), dim3(RED_THREADS), 0, N, Vq, c->w,
               (const double *)(hlast + q * MAXNV));
    BF_LAUNCH(c);
  }
  const int ql = nb - 1;
  const double *Vl = blk(ql);
  BF_NV_SWITCH(bn(ql), (launch_pdl(c, k_axpy_norm<NV>, dim3(wave_grid(c, k_axpy_norm<NV>)), dim3(RED_THREADS), 0, N,
                                   Vl, (const double *)c->w, (const double *)(hlast + ql * MAXNV), vn, c->red, hdn,
                                   c->counter)));
  BF_LAUNCH(c);
}

void gmres(bf_ctx *c, const double *b, double *x, double tol, int m, int maxit, int *iters, double *hist,
           int *converged, double *relres) {
  int64_t N = 2 * (int64_t)c->n;
  int G = grid_for(c);
  double *V = c->V;
  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), y(m), hcol(m + 1);
  *iters = 0;
  *converged = 0;
  const int hs = hstride(m);
  double *hd1 = c->hdev, *hd2 = c->hdev + hs, *hdn = c->hdev + 2 * hs;
  const double bb = dot_host(c, b, b);
  if (!std::isfinite(bb))  // bf.h: BF_ERR_NONFINITE names the first NaN/Inf of the rhs
    throw Error(BF_ERR_NONFINITE, "rhs is not finite: " + nonfinite_where(c, b));
  double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) {
    k_zero_vec<<<G, 256, 0, c->stream>>>(N, x);
    BF_LAUNCH(c);
    if (hist) hist[0] = 0.0;
    *converged = 1;
    *relres = 0.0;
    return;
  }
  // r = b - J x, written straight into the basis slot v_0 (normalised by the first split)
  bsr_spmv(c, x, c->w);
  k_sub<<<G, 256, 0, c->stream>>>(N, b, c->w, V);
  BF_LAUNCH(c);
  double beta = std::sqrt(dot_host(c, V, V, hdn));
  if (!std::isfinite(beta))
    throw Error(BF_ERR_NONFINITE, "initial residual b - J x0 is not finite: x0 " + nonfinite_where(c, x));
  if (hist) hist[0] = beta / bnorm;
  *relres = beta / bnorm;
  if (beta <= tol * bnorm) {
    *converged = 1;
    return;
  }
  if (maxit <= 0) return;  // no Arnoldi step allowed: x = x0
  // Arnoldi step j, enqueued without waiting for the host: z_j = M^-1 v_j, w = J z_j, CGS2,
  // v_{j+1} = w / ||w|| (norm taken on the device, applied by the next step's split kernel), then an async copy of (h, h2, ||w||^2)
  // into pinned slot j%2 and an event.  The host processes step j (Givens, convergence) while
  // step j+1 already runs; a step enqueued past the stopping point is simply discarded.
  const int SLOT = 2 * hs + 8;
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
    orthogonalise(c, nv, hd1, hd2, hdn, vn);
    timer_end(c, 1, t0, 8.0 * N * (c->opt.orth == 0 ? 3.0 * nv + 5.0 : 2.0 * nv + 3.0));
    BF_CUDA(cudaGetLastError());
    BF_CUDA(cudaMemcpyAsync(c->hpin + (j & 1) * SLOT, c->hdev, sizeof(double) * (2 * hs + 1), cudaMemcpyDeviceToHost,
                            c->stream));
    BF_CUDA(cudaEventRecord(c->step_ev[j & 1], c->stream));
    c->timing_skip = false;
  };
  for (;;) {
    NvtxRange r_cycle("gmres cycle");
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k = 0;
    bool breakdown = false;
    enqueue(0);
    for (int j = 0; j < m; j++) {
      if (j + 1 < m && *iters + 1 < maxit) enqueue(j + 1);  // speculative next step
      BF_CUDA(cudaEventSynchronize(c->step_ev[j & 1]));
      const double *hp = c->hpin + (j & 1) * SLOT;
      double hn = std::sqrt(hp[2 * hs]);
      bool finite = std::isfinite(hn);
      for (int i = 0; i <= j; i++) {
        hcol[i] = hp[i] + (c->opt.orth == 0 ? hp[hs + i] : 0.0);
        finite = finite && std::isfinite(hcol[i]);
      }
      if (!finite) {  // the preconditioner or the operator produced NaN/Inf; x keeps the last cycle's iterate
        BF_CUDA(cudaStreamSynchronize(c->stream));
        throw Error(BF_ERR_NONFINITE, "GMRES: non-finite Arnoldi coefficient at iteration " +
                                          std::to_string(*iters + 1) + " (M^-1 v or J z produced NaN/Inf)");
      }
      if (hn == 0.0) breakdown = true;  // (happy) breakdown: the speculative step is discarded
      for (int i = 0; i <= j; i++) H[(size_t)i * m + j] = hcol[i];
      H[(size_t)(j + 1) * m + j] = hn;
      for (int i = 0; i < j; i++) {  // previous Givens rotations
        double a = H[(size_t)i * m + j], bb2 = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a + sn[i] * bb2;
        H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * bb2;
      }
      double a = H[(size_t)j * m + j], bb2 = H[(size_t)(j + 1) * m + j];
      double t = std::hypot(a, bb2);
      if (t == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = a / t;
        sn[j] = bb2 / t;
      }
      H[(size_t)j * m + j] = cs[j] * a + sn[j] * bb2;
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
    double *yd = hd2;  // the speculative step's h' (if any) is no longer needed
    BF_CUDA(cudaMemcpyAsync(yd, ypin, sizeof(double) * k, cudaMemcpyHostToDevice, c->stream));
    // x += M^-1 (V y) = Z y  (M^-1 is a fixed linear operator: no extra BF apply per cycle)
    for (int q = 0; q * MAXNV < k; q++) {
      const int kb = std::min(MAXNV, k - q * MAXNV);
      const double *Zq = c->Z + (size_t)q * MAXNV * N;
      BF_NV_SWITCH(kb, (k_lincomb<NV><<<G, 256, 0, c->stream>>>(N, Zq, yd + q * MAXNV, c->z, q > 0 ? 1 : 0)));
      BF_LAUNCH(c);
    }
    k_add_inplace<<<G, 256, 0, c->stream>>>(N, x, c->z);
    BF_LAUNCH(c);
    // true residual at the end of the cycle (R11)
    bsr_spmv(c, x, c->w);
    k_sub<<<G, 256, 0, c->stream>>>(N, b, c->w, V);
    BF_LAUNCH(c);
    beta = std::sqrt(dot_host(c, V, V, hdn));
    if (!std::isfinite(beta))
      throw Error(BF_ERR_NONFINITE, "GMRES: true residual not finite after iteration " + std::to_string(*iters));
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
