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
#include <cmath>
#include <string>

#include "bf_internal.cuh"

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

// every strong edge (i, j in S_i) with both ends undecided marks its smaller end "not max";
// this covers U cap (S_i cup S_i^T) for every i
__global__ void k_pmis_edges(DCsr A, const uint8_t *__restrict__ strong, const uint64_t *__restrict__ key,
                             const int8_t *__restrict__ state, uint8_t *notmax) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n || state[i] >= 0) return;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    int j = A.ci[q];
    if (!strong[q] || state[j] >= 0) continue;
    if (greater_key(key, i, j)) notmax[j] = 1;
    else notmax[i] = 1;
  }
}

__global__ void k_pmis_cnew(int n, const int8_t *__restrict__ state, const uint8_t *__restrict__ notmax,
                            uint8_t *cnew) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  cnew[i] = (uint8_t)(state[i] < 0 && !notmax[i]);
}

__global__ void k_pmis_update(DCsr A, const uint8_t *__restrict__ strong, const uint8_t *__restrict__ cnew,
                              int8_t *state, int *nU) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n || state[i] >= 0) return;
  if (cnew[i]) { state[i] = 1; return; }
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++)
    if (strong[q] && cnew[A.ci[q]]) { state[i] = 0; return; }
  atomicAdd(nU, 1);
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
                              DCsr P) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
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

__global__ void k_spgemm_expand(DCsr A, DCsr B, const int64_t *__restrict__ off, int colbits, uint64_t *keys,
                                double *vals) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  int64_t p = off[i];
  uint64_t hi = (uint64_t)i << colbits;
  for (int q = A.rp[i]; q < A.rp[i + 1]; q++) {
    double a = A.v[q];
    int k = A.ci[q];
    for (int t = B.rp[k]; t < B.rp[k + 1]; t++) {
      keys[p] = hi | (uint64_t)B.ci[t];
      vals[p] = __dmul_rn(a, B.v[t]);
      p++;
    }
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

static void spgemm(bf_ctx *c, const DCsr &A, const DCsr &B, DCsr &C) {
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
  k_spgemm_expand<<<div_up(A.n, 128), 128, 0, c->stream>>>(A, B, off, colbits, keys, vals);
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

void build_hierarchy(bf_ctx *c, int which, const DCsr &A0) {
  Hier &h = c->h[which];
  const bf_options &o = c->opt;
  copy_csr(c, A0, h.lv[0].A);
  int l = 0;
  int *nU_d = dalloc_t<int>(c, 1);
  while (h.lv[l].A.n > o.max_coarse && l < o.max_levels - 1 && l < BF_MAXL - 1) {
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
    k_lambda<<<div_up(n, 256), 256, 0, c->stream>>>(A, strong, lam);
    BF_LAUNCH(c);
    uint64_t *key = dalloc_t<uint64_t>(c, n);
    int8_t *state = dalloc_t<int8_t>(c, n);
    k_pmis_init<<<div_up(n, 256), 256, 0, c->stream>>>(n, lam, o.seed, l, key, state);
    BF_LAUNCH(c);
    uint8_t *notmax = dalloc_t<uint8_t>(c, n);
    uint8_t *cnew = dalloc_t<uint8_t>(c, n);
    for (int round = 0;; round++) {
      BF_CUDA(cudaMemsetAsync(notmax, 0, n, c->stream));
      BF_CUDA(cudaMemsetAsync(nU_d, 0, sizeof(int), c->stream));
      k_pmis_edges<<<div_up(n, 256), 256, 0, c->stream>>>(A, strong, key, state, notmax);
      k_pmis_cnew<<<div_up(n, 256), 256, 0, c->stream>>>(n, state, notmax, cnew);
      k_pmis_update<<<div_up(n, 256), 256, 0, c->stream>>>(A, strong, cnew, state, nU_d);
      c->launches += 3;
      BF_CUDA(cudaGetLastError());
      int nU = 0;
      BF_CUDA(cudaMemcpyAsync(&nU, nU_d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      if (nU == 0) break;
      if (round > 10000) throw Error(BF_ERR_LIMIT, "PMIS did not terminate");
    }
    dfree(c, notmax);
    dfree(c, cnew);
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
    k_interp_count<<<div_up(n, 256), 256, 0, c->stream>>>(A, strong, state, cnt);
    BF_LAUNCH(c);
    L.P.n = n;
    L.P.m = (int)nc;
    L.P.rp = dalloc_t<int32_t>(c, (size_t)n + 1);
    L.P.nnz = exclusive_scan_i32(c, cnt, L.P.rp, n);
    dfree(c, cnt);
    L.P.ci = dalloc_t<int32_t>(c, L.P.nnz);
    L.P.v = dalloc_t<double>(c, L.P.nnz);
    k_interp_fill<<<div_up(n, 128), 128, 0, c->stream>>>(A, strong, state, cmap, diag, o.interp_norm, L.P);
    BF_LAUNCH(c);
    BF_CUDA(cudaGetLastError());
    dfree(c, cmap);
    dfree(c, strong);
    dfree(c, diag);
    transpose(c, L.P, L.R);
    DCsr AP;
    spgemm(c, A, L.P, AP);
    spgemm(c, L.R, AP, h.lv[l + 1].A);
    free_csr(c, AP);
    l++;
  }
  dfree(c, nU_d);
  h.nlev = l + 1;
  for (int k = 0; k < h.nlev; k++) {
    Level &L = h.lv[k];
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
    if (k < h.nlev - 1) {
      tile_csr(c, L.P);
      tile_csr(c, L.R);
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
  plan_tail(c, h);
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
  plan_tail(c, h);
}

}  // namespace bf
