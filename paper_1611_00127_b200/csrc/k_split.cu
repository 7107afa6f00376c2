// k_split.cu -- ingest/validation of the 2x2 BSR Jacobian, the field split into
// A_pp, A_ps, A_sp, A_ss (restrictions R_p/R_s P:L174-187) and the
// SIMPLE approximate Schur complement S~ = A_pp - A_ps diag(A_ss)^-1 A_sp
// (`SIMPLE-Schur`, A_sp reading R1).
//
// Determinism contract: every setup value is produced by
// one thread in a fixed order with explicitly rounded __dmul_rn/__dadd_rn/__ddiv_rn
// (no FMA contraction), so patterns and values are bit-identical run to run.
#include <cfloat>
#include <cmath>
#include <string>

#include "bf_internal.cuh"
BF_CHECK_TU("k_split.cu")

namespace bf {

__device__ __forceinline__ int blk_index(int block_order, int var_order, int r, int c) {
  if (var_order) { r = 1 - r; c = 1 - c; }
  return block_order == 0 ? 2 * r + c : 2 * c + r;
}

// error codes accumulated with atomicMin on the offending index
struct IngestErr {
  int rp_bad;      // first row with rp[r] > rp[r+1] or bad ends
  int col_bad;     // first row with an out-of-range / non-ascending column
  int diag_bad;    // first row without a diagonal block
  long long nonfinite;  // first block with a non-finite value
};

__global__ void k_validate(int n, int64_t nnzb, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           IngestErr *err) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int a = rp[r], b = rp[r + 1];
  if (a > b || a < 0 || b > nnzb || (r == 0 && a != 0) || (r == n - 1 && b != nnzb)) {
    atomicMin(&err->rp_bad, r);
    return;
  }
  int prev = -1;
  bool diag = false;
  for (int q = a; q < b; q++) {
    int c = ci[q];
    if (c < 0 || c >= n || c <= prev) { atomicMin(&err->col_bad, r); return; }
    if (c == r) diag = true;
    prev = c;
  }
  if (!diag) atomicMin(&err->diag_bad, r);
}

// canonicalise blocks into (p,s) row-major double2 pairs and check finiteness
__global__ void k_canon(int64_t nnzb, const double *__restrict__ in, double *__restrict__ out, int block_order,
                        int var_order, IngestErr *err) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnzb) return;
  double v[4];
  bool fin = true;
  for (int r = 0; r < 2; r++)
    for (int c = 0; c < 2; c++) {
      double x = in[4 * q + blk_index(block_order, var_order, r, c)];
      v[2 * r + c] = x;
      fin = fin && isfinite(x);
    }
  if (!fin) atomicMin(&err->nonfinite, (long long)q);
  reinterpret_cast<double2 *>(out)[2 * q] = make_double2(v[0], v[1]);
  reinterpret_cast<double2 *>(out)[2 * q + 1] = make_double2(v[2], v[3]);
}

void validate_and_ingest(bf_ctx *c, const bf_bsr2 *J) {
  if (J->n_cells <= 0) throw Error(BF_ERR_ARG, "n_cells must be positive");
  if ((int64_t)J->nx * J->ny * J->nz != J->n_cells)
    throw Error(BF_ERR_ARG, "nx*ny*nz (" + std::to_string((long long)J->nx * J->ny * J->nz) +
                                ") != n_cells (" + std::to_string(J->n_cells) + ")");
  if (J->nnzb < J->n_cells || J->nnzb >= (1ll << 31))
    throw Error(BF_ERR_ARG, "nnzb must be in [n_cells, 2^31)");
  if (!J->row_ptr || !J->col_idx || !J->vals) throw Error(BF_ERR_ARG, "row_ptr/col_idx/vals must be non-NULL");
  if (J->block_order != 0 && J->block_order != 1) throw Error(BF_ERR_ARG, "block_order must be 0 or 1");
  if (J->var_order != 0 && J->var_order != 1) throw Error(BF_ERR_ARG, "var_order must be 0 or 1");
  if (J->mem != 0 && J->mem != 1) throw Error(BF_ERR_ARG, "mem must be 0 (host) or 1 (device)");
  int n = J->n_cells;
  int64_t nnzb = J->nnzb;
  c->n = n;
  c->nx = J->nx;
  c->ny = J->ny;
  c->nz = J->nz;
  c->nnzb = nnzb;
  c->var_order = J->var_order;
  c->block_order = J->block_order;
  c->brp = dalloc_t<int32_t>(c, (size_t)n + 1);
  c->bci = dalloc_t<int32_t>(c, (size_t)nnzb);
  c->bv = dalloc_t<double>(c, (size_t)nnzb * 4);
  cudaMemcpyKind kind = J->mem ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  double *raw = dalloc_t<double>(c, (size_t)nnzb * 4);
  BF_CUDA(cudaMemcpyAsync(c->brp, J->row_ptr, sizeof(int32_t) * (n + 1), kind, c->stream));
  BF_CUDA(cudaMemcpyAsync(c->bci, J->col_idx, sizeof(int32_t) * nnzb, kind, c->stream));
  BF_CUDA(cudaMemcpyAsync(raw, J->vals, sizeof(double) * 4 * nnzb, kind, c->stream));
  IngestErr *derr = dalloc_t<IngestErr>(c, 1);
  IngestErr herr{INT32_MAX, INT32_MAX, INT32_MAX, (long long)INT64_MAX};
  BF_CUDA(cudaMemcpyAsync(derr, &herr, sizeof herr, cudaMemcpyHostToDevice, c->stream));
  k_validate<<<div_up(n, 256), 256, 0, c->stream>>>(n, nnzb, c->brp, c->bci, derr);
  BF_LAUNCH(c);
  k_canon<<<div_up(nnzb, 256), 256, 0, c->stream>>>(nnzb, raw, c->bv, J->block_order, J->var_order, derr);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  BF_CUDA(cudaMemcpyAsync(&herr, derr, sizeof herr, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, raw);
  dfree(c, derr);
  if (herr.rp_bad != INT32_MAX)
    throw Error(BF_ERR_PATTERN, "row_ptr not monotone / inconsistent with nnzb at row " + std::to_string(herr.rp_bad));
  if (herr.col_bad != INT32_MAX)
    throw Error(BF_ERR_PATTERN, "col_idx not ascending or out of range in row " + std::to_string(herr.col_bad));
  if (herr.diag_bad != INT32_MAX)
    throw Error(BF_ERR_PATTERN, "diagonal block missing in row " + std::to_string(herr.diag_bad));
  if (herr.nonfinite != (long long)INT64_MAX)
    throw Error(BF_ERR_NONFINITE, "non-finite Jacobian value in block " + std::to_string(herr.nonfinite));
}

// new values on the ingested pattern (bf_update): canonicalise + finiteness check
void reingest_values(bf_ctx *c, const double *vals, int mem) {
  int64_t nnzb = c->nnzb;
  double *raw = dalloc_t<double>(c, (size_t)nnzb * 4);
  BF_CUDA(cudaMemcpyAsync(raw, vals, sizeof(double) * 4 * nnzb, mem ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                          c->stream));
  IngestErr *derr = dalloc_t<IngestErr>(c, 1);
  IngestErr herr{INT32_MAX, INT32_MAX, INT32_MAX, (long long)INT64_MAX};
  BF_CUDA(cudaMemcpyAsync(derr, &herr, sizeof herr, cudaMemcpyHostToDevice, c->stream));
  double *bv = dalloc_t<double>(c, (size_t)nnzb * 4);
  k_canon<<<div_up(nnzb, 256), 256, 0, c->stream>>>(nnzb, raw, bv, c->block_order, c->var_order, derr);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  BF_CUDA(cudaMemcpyAsync(&herr, derr, sizeof herr, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, raw);
  dfree(c, derr);
  if (herr.nonfinite != (long long)INT64_MAX) {
    dfree(c, bv);
    throw Error(BF_ERR_NONFINITE, "non-finite Jacobian value in block " + std::to_string(herr.nonfinite));
  }
  dfree(c, c->bv);
  c->bv = bv;
}

// ---------------------------------------------------------------------------------------
// field split: scalar pattern = entries != +-0.0, plus the diagonal (reading Q23)
// ---------------------------------------------------------------------------------------
__global__ void k_split_count(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                              const double *__restrict__ bv, int32_t *__restrict__ cnt /*[4][n]*/) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int k0 = 0, k1 = 0, k2 = 0, k3 = 0;
  for (int q = rp[r]; q < rp[r + 1]; q++) {
    bool d = ci[q] == r;
    k0 += (bv[4 * q + 0] != 0.0) || d;
    k1 += (bv[4 * q + 1] != 0.0) || d;
    k2 += (bv[4 * q + 2] != 0.0) || d;
    k3 += (bv[4 * q + 3] != 0.0) || d;
  }
  cnt[r] = k0;
  cnt[n + r] = k1;
  cnt[2 * n + r] = k2;
  cnt[3 * n + r] = k3;
}

struct Out4 {
  int32_t *rp[4];
  int32_t *ci[4];
  double *v[4];
};

__global__ void k_split_fill(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                             const double *__restrict__ bv, Out4 o, double *__restrict__ dss, int *zero_diag) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int pos[4] = {o.rp[0][r], o.rp[1][r], o.rp[2][r], o.rp[3][r]};
  for (int q = rp[r]; q < rp[r + 1]; q++) {
    int c = ci[q];
    bool d = c == r;
#pragma unroll
    for (int b = 0; b < 4; b++) {
      double a = bv[4 * q + b];
      if (a != 0.0 || d) {
        o.ci[b][pos[b]] = c;
        o.v[b][pos[b]] = a;
        pos[b]++;
      }
    }
    if (d) {
      dss[r] = bv[4 * q + 3];
      if (bv[4 * q + 3] == 0.0) atomicMin(zero_diag, r);
    }
  }
}

void build_split(bf_ctx *c) {
  int n = c->n;
  int32_t *cnt = dalloc_t<int32_t>(c, (size_t)4 * n);
  k_split_count<<<div_up(n, 256), 256, 0, c->stream>>>(n, c->brp, c->bci, c->bv, cnt);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  Out4 o;
  for (int b = 0; b < 4; b++) {
    DCsr &A = c->blk[b];
    A.n = A.m = n;
    A.rp = dalloc_t<int32_t>(c, (size_t)n + 1);
    A.nnz = exclusive_scan_i32(c, cnt + (size_t)b * n, A.rp, n);
    A.ci = dalloc_t<int32_t>(c, A.nnz);
    A.v = dalloc_t<double>(c, A.nnz);
    o.rp[b] = A.rp;
    o.ci[b] = A.ci;
    o.v[b] = A.v;
  }
  dfree(c, cnt);
  c->dss = dalloc_t<double>(c, n);
  int *zd = dalloc_t<int>(c, 1);
  int hz = INT32_MAX;
  BF_CUDA(cudaMemcpyAsync(zd, &hz, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  k_split_fill<<<div_up(n, 256), 256, 0, c->stream>>>(n, c->brp, c->bci, c->bv, o, c->dss, zd);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  BF_CUDA(cudaMemcpyAsync(&hz, zd, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, zd);
  if (hz != INT32_MAX) throw Error(BF_ERR_ZERO_DIAG, "A_ss diagonal is zero at cell " + std::to_string(hz));
}

// ---------------------------------------------------------------------------------------
// S~ = A_pp - A_ps diag(A_ss)^-1 B,  B = A_sp (R1) or A_pp (literal P:L239, diagnostics)
// row pattern = pattern(A_pp, i) U {j : k in pattern(A_ps, i), j in pattern(B, k)}
// ---------------------------------------------------------------------------------------
#define SCHUR_CAP 256

__device__ int schur_row_pattern(int i, const DCsr &App, const DCsr &Aps, const DCsr &B, int *list) {
  int len = 0;
  for (int q = App.rp[i]; q < App.rp[i + 1]; q++) {
    if (len >= SCHUR_CAP) return -1;
    list[len++] = App.ci[q];
  }
  for (int q = Aps.rp[i]; q < Aps.rp[i + 1]; q++) {
    int k = Aps.ci[q];
    for (int t = B.rp[k]; t < B.rp[k + 1]; t++) {
      if (len >= SCHUR_CAP) return -1;
      list[len++] = B.ci[t];
    }
  }
  // insertion sort + unique
  for (int a = 1; a < len; a++) {
    int x = list[a], b = a - 1;
    while (b >= 0 && list[b] > x) { list[b + 1] = list[b]; b--; }
    list[b + 1] = x;
  }
  int u = 0;
  for (int a = 0; a < len; a++)
    if (u == 0 || list[a] != list[u - 1]) list[u++] = list[a];
  return u;
}

__global__ void k_schur_count(int n, DCsr App, DCsr Aps, DCsr B, int32_t *cnt, int *overflow) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int list[SCHUR_CAP];
  int u = schur_row_pattern(i, App, Aps, B, list);
  if (u < 0) { atomicMin(overflow, i); u = 0; }
  cnt[i] = u;
}

__device__ __forceinline__ int find_col(const int32_t *ci, int lo, int hi, int j) {
  // binary search of j in ci[lo, hi) (present by construction)
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (ci[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_schur_fill(int n, DCsr App, DCsr Aps, DCsr B, const double *__restrict__ dss, DCsr S) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int list[SCHUR_CAP];
  int u = schur_row_pattern(i, App, Aps, B, list);
  int base = S.rp[i];
  for (int a = 0; a < u; a++) {
    S.ci[base + a] = list[a];
    S.v[base + a] = 0.0;  // +0.0 where A_pp has no entry
  }
  int end = base + u;
  for (int q = App.rp[i]; q < App.rp[i + 1]; q++) S.v[find_col(S.ci, base, end, App.ci[q])] = App.v[q];
  for (int q = Aps.rp[i]; q < Aps.rp[i + 1]; q++) {  // k ascending
    int k = Aps.ci[q];
    double t = __ddiv_rn(Aps.v[q], dss[k]);
    for (int s = B.rp[k]; s < B.rp[k + 1]; s++) {
      int p = find_col(S.ci, base, end, B.ci[s]);
      S.v[p] = __dadd_rn(S.v[p], -__dmul_rn(t, B.v[s]));
    }
  }
}

void build_schur(bf_ctx *c) {
  int n = c->n;
  const DCsr &App = c->blk[0], &Aps = c->blk[1];
  const DCsr &B = c->opt.schur_as_printed ? c->blk[0] : c->blk[2];
  int32_t *cnt = dalloc_t<int32_t>(c, n);
  int *ovf = dalloc_t<int>(c, 1);
  int h = INT32_MAX;
  BF_CUDA(cudaMemcpyAsync(ovf, &h, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  k_schur_count<<<div_up(n, 128), 128, 0, c->stream>>>(n, App, Aps, B, cnt, ovf);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
  BF_CUDA(cudaMemcpyAsync(&h, ovf, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, ovf);
  if (h != INT32_MAX)
    throw Error(BF_ERR_LIMIT, "S~ row " + std::to_string(h) + " has more than " + std::to_string(SCHUR_CAP) +
                                  " candidate columns");
  DCsr &S = c->blk[4];
  S.n = S.m = n;
  S.rp = dalloc_t<int32_t>(c, (size_t)n + 1);
  S.nnz = exclusive_scan_i32(c, cnt, S.rp, n);
  dfree(c, cnt);
  S.ci = dalloc_t<int32_t>(c, S.nnz);
  S.v = dalloc_t<double>(c, S.nnz);
  k_schur_fill<<<div_up(n, 128), 128, 0, c->stream>>>(n, App, Aps, B, c->dss, S);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

}  // namespace bf
