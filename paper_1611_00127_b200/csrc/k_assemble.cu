// k_assemble.cu -- device assembly of the fully implicit two-phase residual and its exact
// Jacobian (the step before the linear-solve path), and the Newton state
// update.  Same discretisation and readings as the seeded generator workload/twophase.py,
// which serves as its reference in tests/test_gpu_assemble.py:
//   cell-centred FV + TPFA, phase upwinding with tie -> the higher-index cell
//   (Q6), harmonic face permeability, backward Euler in mass form
//   (Q2/Q3), exact Jacobian with frozen donor (Q7),
//   quadratic k_r (Q8), S_w clamp (Q10), Brooks-Corey / van Genuchten / linear P_c
//   (Q16), Dirichlet faces (Q14), water mass source (Q16).
// Row-owned: one thread per cell computes its residual pair and its block row (each face is
// evaluated by both of its cells with the same orientation l < u, so both see the same donor).
#include <cmath>

#include "bf_internal.cuh"
BF_CHECK_TU("k_assemble.cu")

namespace bf {

struct Props {
  double lw, ln, dlw, dln, pc, dpc;
};

__device__ __forceinline__ Props cell_props(const bf_twophase &P, double sn) {
  const double eps = 1e-3;
  Props r;
  double sw = 1.0 - sn;
  bool inside = (sw > eps) && (sw < 1.0 - eps);
  double s = fmin(fmax(sw, eps), 1.0 - eps);
  double ds = inside ? -1.0 : 0.0;  // d S_w_bar / d S_n
  double krw = s * s, krn = (1.0 - s) * (1.0 - s);
  double dkrw = 2.0 * s * ds, dkrn = -2.0 * (1.0 - s) * ds;
  double pc = 0.0, dpcs = 0.0;
  if (P.pc_kind == 1) {  // Brooks-Corey P_d S^(-1/lambda)
    double pd = P.pc_a, lam = P.pc_b;
    pc = pd * pow(s, -1.0 / lam);
    dpcs = -(pd / lam) * pow(s, -1.0 / lam - 1.0);
  } else if (P.pc_kind == 2) {  // van Genuchten (1/alpha)(S^(-1/m) - 1)^(1/n), m = 1 - 1/n
    double n = P.pc_a, alpha = P.pc_b, m = 1.0 - 1.0 / n;
    double base = pow(s, -1.0 / m) - 1.0;
    pc = (1.0 / alpha) * pow(base, 1.0 / n);
    dpcs = (1.0 / alpha) * (1.0 / n) * pow(base, 1.0 / n - 1.0) * (-1.0 / m) * pow(s, -1.0 / m - 1.0);
  } else if (P.pc_kind == 3) {  // linear P_0 (1 - S)
    pc = P.pc_a * (1.0 - s);
    dpcs = -P.pc_a;
  }
  r.lw = krw / P.mu_w;
  r.ln = krn / P.mu_n;
  r.dlw = dkrw / P.mu_w;
  r.dln = dkrn / P.mu_n;
  r.pc = pc;
  r.dpc = dpcs * ds;
  return r;
}

struct Flux {
  double F, dpl, dsl, dpu, dsu;  // flux l -> u and its derivatives w.r.t. (p_l, S_l, p_u, S_u)
};

// F = rho lam_up T (Phi_l - Phi_u), up = l if Phi_l - Phi_u > 0 else u (frozen donor)
__device__ __forceinline__ Flux phase_flux(double rho, double lam_l, double lam_u, double dlam_l, double dlam_u,
                                           double phi_l, double phi_u, double dphi_l, double dphi_u, double T) {
  Flux f;
  double d = phi_l - phi_u;
  bool upl = d > 0.0;
  double lam = upl ? lam_l : lam_u;
  f.F = rho * lam * T * d;
  f.dpl = rho * lam * T;
  f.dpu = -rho * lam * T;
  f.dsl = rho * T * ((upl ? dlam_l : 0.0) * d + lam * dphi_l);
  f.dsu = rho * T * ((upl ? 0.0 : dlam_u) * d - lam * dphi_u);
  return f;
}

__device__ __forceinline__ double depth(const bf_twophase &P, int i, int j, int k) {
  if (P.gravity_axis < 0) return 0.0;
  int a = P.gravity_axis == 0 ? i : (P.gravity_axis == 1 ? j : k);
  return (a + 0.5) * P.h;
}

__global__ void k_assemble_count(bf_twophase P, int32_t *cnt) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  int n = P.nx * P.ny * P.nz;
  if (c >= n) return;
  int i = c % P.nx, j = (c / P.nx) % P.ny, k = c / (P.nx * P.ny);
  cnt[c] = 1 + (i > 0) + (i < P.nx - 1) + (j > 0) + (j < P.ny - 1) + (k > 0) + (k < P.nz - 1);
}

__global__ void k_assemble(bf_twophase P, const double *__restrict__ p, const double *__restrict__ sn,
                           const int32_t *__restrict__ rp, int32_t *__restrict__ ci, double *__restrict__ vals,
                           double *__restrict__ R) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int nx = P.nx, ny = P.ny, nz = P.nz;
  int n = nx * ny * nz;
  if (c >= n) return;
  int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
  const double g = P.gravity_axis >= 0 ? P.g : 0.0;
  const double V = P.h * P.h * P.h, A = P.h * P.h, dt = P.dt;
  Props pcell = cell_props(P, sn[c]);
  double Dc = depth(P, i, j, k);
  double phw_c = p[c] - P.rho_w * g * Dc, phn_c = p[c] + pcell.pc - P.rho_n * g * Dc;
  double sold = P.sn_old[c];
  double Rw = V * P.phi * P.rho_w * ((1.0 - sn[c]) - (1.0 - sold));
  double Rn = V * P.phi * P.rho_n * (sn[c] - sold);
  double dg[4] = {0.0, -V * P.phi * P.rho_w, 0.0, V * P.phi * P.rho_n};
  // neighbours in ascending column order: -z, -y, -x, (diag), +x, +y, +z
  const int offs[6] = {-nx * ny, -nx, -1, 1, nx, nx * ny};
  const bool has[6] = {k > 0, j > 0, i > 0, i < nx - 1, j < ny - 1, k < nz - 1};
  const int ni[6] = {i, i, i - 1, i + 1, i, i}, nj[6] = {j, j - 1, j, j, j + 1, j},
            nk[6] = {k - 1, k, k, k, k, k + 1};
  int pos = rp[c];
  double off[6][4];
  for (int s = 0; s < 6; s++) {
    if (!has[s]) continue;
    int d = c + offs[s];
    Props pd = cell_props(P, sn[d]);
    double Dd = depth(P, ni[s], nj[s], nk[s]);
    double phw_d = p[d] - P.rho_w * g * Dd, phn_d = p[d] + pd.pc - P.rho_n * g * Dd;
    double kl = P.perm[c < d ? c : d], ku = P.perm[c < d ? d : c];
    double kf = (kl > 0.0 && ku > 0.0) ? (2.0 * kl) * ku / (ku + kl) : 0.0;
    double T = A * kf / P.h;
    bool low = c < d;  // face oriented low -> high (reading Q6)
    const Props &Lp = low ? pcell : pd, &Up = low ? pd : pcell;
    double pwl = low ? phw_c : phw_d, pwu = low ? phw_d : phw_c;
    double pnl = low ? phn_c : phn_d, pnu = low ? phn_d : phn_c;
    Flux fw = phase_flux(P.rho_w, Lp.lw, Up.lw, Lp.dlw, Up.dlw, pwl, pwu, 0.0, 0.0, T);
    Flux fn = phase_flux(P.rho_n, Lp.ln, Up.ln, Lp.dln, Up.dln, pnl, pnu, Lp.dpc, Up.dpc, T);
    double sg = low ? dt : -dt;  // R_l += dt F, R_u -= dt F
    Rw += sg * fw.F;
    Rn += sg * fn.F;
    if (low) {
      dg[0] += sg * fw.dpl; dg[1] += sg * fw.dsl; dg[2] += sg * fn.dpl; dg[3] += sg * fn.dsl;
      off[s][0] = sg * fw.dpu; off[s][1] = sg * fw.dsu; off[s][2] = sg * fn.dpu; off[s][3] = sg * fn.dsu;
    } else {
      dg[0] += sg * fw.dpu; dg[1] += sg * fw.dsu; dg[2] += sg * fn.dpu; dg[3] += sg * fn.dsu;
      off[s][0] = sg * fw.dpl; off[s][1] = sg * fw.dsl; off[s][2] = sg * fn.dpl; off[s][3] = sg * fn.dsl;
    }
  }
  // Dirichlet faces: boundary state (p_b, S_n^n of the cell), T_b = A K_c / (h/2)
  for (int f = 0; f < P.n_dirichlet; f++) {
    int ax = P.dir_axis[f], side = P.dir_side[f];
    int coord = ax == 0 ? i : (ax == 1 ? j : k);
    int ext = ax == 0 ? nx : (ax == 1 ? ny : nz);
    if (coord != (side == 0 ? 0 : ext - 1)) continue;
    double pb = P.dir_p[f];
    Props pbp = cell_props(P, sold);
    double T = A * P.perm[c] / (P.h / 2.0);
    double phw_b = pb - P.rho_w * g * Dc, phn_b = pb + pbp.pc - P.rho_n * g * Dc;
    Flux fw = phase_flux(P.rho_w, pcell.lw, pbp.lw, pcell.dlw, 0.0, phw_c, phw_b, 0.0, 0.0, T);
    Flux fn = phase_flux(P.rho_n, pcell.ln, pbp.ln, pcell.dln, 0.0, phn_c, phn_b, pcell.dpc, 0.0, T);
    Rw += dt * fw.F;
    Rn += dt * fn.F;
    dg[0] += dt * fw.dpl; dg[1] += dt * fw.dsl; dg[2] += dt * fn.dpl; dg[3] += dt * fn.dsl;
  }
  if (P.source_w) Rw -= dt * P.source_w[c];
  R[2 * c] = Rw;
  R[2 * c + 1] = Rn;
  // block row: -z, -y, -x, diag, +x, +y, +z (present ones), row-major (a_pp, a_ps, a_sp, a_ss)
  for (int s = 0; s < 3; s++)
    if (has[s]) {
      ci[pos] = c + offs[s];
      for (int e = 0; e < 4; e++) vals[4 * (size_t)pos + e] = off[s][e];
      pos++;
    }
  ci[pos] = c;
  for (int e = 0; e < 4; e++) vals[4 * (size_t)pos + e] = dg[e];
  pos++;
  for (int s = 3; s < 6; s++)
    if (has[s]) {
      ci[pos] = c + offs[s];
      for (int e = 0; e < 4; e++) vals[4 * (size_t)pos + e] = off[s][e];
      pos++;
    }
}

// u <- u + delta with the per-cell saturation chop (reading R17) and S_n kept in [0, 1]
__global__ void k_newton_update(int n, double *p, double *sn, const double *__restrict__ delta, double chop) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double2 d = reinterpret_cast<const double2 *>(delta)[c];
  double ds = d.y;
  p[c] += d.x;
  if (chop > 0.0) {
    ds = fmin(fmax(ds, -chop), chop);
    sn[c] = fmin(fmax(sn[c] + ds, 0.0), 1.0);
  } else {
    sn[c] += ds;
  }
}

void assemble(bf_ctx *c, const bf_twophase *P, const double *p, const double *sn, int32_t *rp, int32_t *ci,
              double *vals, double *R) {
  if (P->nx < 1 || P->ny < 1 || P->nz < 1) throw Error(BF_ERR_ARG, "grid dimensions must be positive");
  if (P->n_dirichlet < 0 || P->n_dirichlet > 6) throw Error(BF_ERR_ARG, "n_dirichlet must be in [0, 6]");
  if (!P->perm || !P->sn_old || !p || !sn || !rp || !ci || !vals || !R)
    throw Error(BF_ERR_ARG, "perm, sn_old, p, sn and the outputs must be non-NULL device pointers");
  int64_t n64 = (int64_t)P->nx * P->ny * P->nz;
  if (n64 >= (1ll << 31)) throw Error(BF_ERR_ARG, "too many cells");
  int n = (int)n64;
  int32_t *cnt = dalloc_t<int32_t>(c, n);
  k_assemble_count<<<div_up(n, 256), 256, 0, c->stream>>>(*P, cnt);
  BF_LAUNCH(c);
  exclusive_scan_i32(c, cnt, rp, n);
  dfree(c, cnt);
  k_assemble<<<div_up(n, 128), 128, 0, c->stream>>>(*P, p, sn, rp, ci, vals, R);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

void newton_update(bf_ctx *c, int n, double *p, double *sn, const double *delta, double chop) {
  k_newton_update<<<div_up(n, 256), 256, 0, c->stream>>>(n, p, sn, delta, chop);
  BF_LAUNCH(c);
  BF_CUDA(cudaGetLastError());
}

}  // namespace bf
