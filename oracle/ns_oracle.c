/* TEST INFRASTRUCTURE ONLY — CPU restatement of the NS right-hand side.
 * See ns_oracle.h for the specification sources and the pinning status.
 * Every cell loop is an OpenMP loop (the reference's threading model is a
 * static partition over std::threads, parallel.cpp:20-36); each cell's
 * arithmetic is unchanged, so results are bitwise independent of the thread
 * count (tests/test_ns_oracle.py). */
#include "ns_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../include/smc_mechanism.h"
#include "oracle.h"

#define NSP SMC_NSP
#define NV SMC_NVAR

/* ---------------------------------------------------------- thermo */
/* e_k(T) = h_k(T) - R_k T, per unit mass. */
static double spec_e(int k, double T) {
  const double* a = SMC_THERMO[k];
  const double R = SMC_RU / SMC_W[k];
  return R * (a[0] * T + a[1] * T * T / 2.0 + a[2] * T * T * T / 3.0 + a[3] - T);
}
static double spec_h(int k, double T) {
  const double* a = SMC_THERMO[k];
  const double R = SMC_RU / SMC_W[k];
  return R * (a[0] * T + a[1] * T * T / 2.0 + a[2] * T * T * T / 3.0 + a[3]);
}

/* T from the specific internal energy by Newton (ideal gas
 * mixture; e = sum_k Y_k e_k(T)).  e(T) is a cubic in T (the cp_k/R_k are
 * quadratics), so the mixture's coefficients
 *   e(T) = E0 + T (E1 + T (E2 + T E3)),  E0 = sum Y_k R_k b_k,
 *   E1 = sum Y_k R_k (a0_k - 1), E2 = sum Y_k R_k a1_k / 2, E3 = sum Y_k R_k a2_k / 3
 * are summed once and Newton iterates on the cubic, cv = de/dT.  Every
 * operation is written out (fma() where fused), the same sequence as the
 * GPU kernel, so the two give the same T bits: on fine grids of a nearly
 * uniform-pressure state the momentum RHS is -grad p plus small terms and a
 * few-ulp per-cell difference of p would be amplified by 1/dx. */
static double temperature(const double* Y, double e) {
  double E0 = 0.0, E1 = 0.0, E2 = 0.0, E3 = 0.0;
  for (int k = 0; k < NSP; ++k) {
    const double* a = SMC_THERMO[k];
    const double yr = Y[k] * (SMC_RU / SMC_W[k]);
    E0 = fma(yr, a[3], E0);
    E1 = fma(yr, a[0] - 1.0, E1);
    E2 = fma(yr, a[1] / 2.0, E2);
    E3 = fma(yr, a[2] / 3.0, E3);
  }
  E0 = E0 - e;
  const double D2 = 2.0 * E2, D3 = 3.0 * E3;
  double T = 1000.0;
  for (int it = 0; it < 50; ++it) {
    const double f = fma(T, fma(T, fma(T, E3, E2), E1), E0);
    const double df = fma(T, fma(T, D3, D2), E1);
    const double dT = f / df;
    T = T - dT;
    if (fabs(dT) <= 1e-9 * T) break;
  }
  return T;
}

/* ------------------------------------------------------ chemistry */
void or_ns_wdot_cell(double rho, double T, const double* Y, double* wdot) {
  double C[NSP], M = 0.0, om[NSP];
  for (int k = 0; k < NSP; ++k) {
    C[k] = rho * Y[k] / SMC_W[k];
    M += C[k];
    om[k] = 0.0;
  }
  const double lnT = log(T), invRT = 1.0 / (SMC_RU * T);
  for (int r = 0; r < SMC_NREAC; ++r) {
    const smc_reaction* R = &SMC_REACTIONS[r];
    const double kf = R->fwd[0] * exp(R->fwd[1] * lnT - R->fwd[2] * invRT);
    const double kr = R->rev[0] * exp(R->rev[1] * lnT - R->rev[2] * invRT);
    double qf = kf, qr = kr;
    for (int j = 0; j < 3; ++j) {
      if (R->reac[j] >= 0) qf *= C[R->reac[j]];
      if (R->prod[j] >= 0) qr *= C[R->prod[j]];
    }
    if (R->third_body) {
      qf *= M;
      qr *= M;
    }
    const double q = qf - qr;
    for (int j = 0; j < 3; ++j) {
      if (R->reac[j] >= 0) om[R->reac[j]] -= q;
      if (R->prod[j] >= 0) om[R->prod[j]] += q;
    }
  }
  for (int k = 0; k < NSP; ++k) wdot[k] = SMC_W[k] * om[k];
}

/* Gross production magnitude of every species (test diagnostics): W_k
 * sum_r |nu_rk| (qf_r + qr_r) with the rates of or_ns_wdot_cell.  Near
 * equilibrium the net rho omega_k is a small difference of these, so
 * max gross / max |net| bounds how much rounding the chemistry can lose. */
static void wdot_gross_cell(double rho, double T, const double* Y, double* g) {
  double C[NSP], M = 0.0, om[NSP];
  for (int k = 0; k < NSP; ++k) {
    C[k] = rho * Y[k] / SMC_W[k];
    M += C[k];
    om[k] = 0.0;
  }
  const double lnT = log(T), invRT = 1.0 / (SMC_RU * T);
  for (int r = 0; r < SMC_NREAC; ++r) {
    const smc_reaction* R = &SMC_REACTIONS[r];
    double qf = R->fwd[0] * exp(R->fwd[1] * lnT - R->fwd[2] * invRT);
    double qr = R->rev[0] * exp(R->rev[1] * lnT - R->rev[2] * invRT);
    for (int j = 0; j < 3; ++j) {
      if (R->reac[j] >= 0) qf *= C[R->reac[j]];
      if (R->prod[j] >= 0) qr *= C[R->prod[j]];
    }
    if (R->third_body) {
      qf *= M;
      qr *= M;
    }
    const double q = fabs(qf) + fabs(qr);
    for (int j = 0; j < 3; ++j) {
      if (R->reac[j] >= 0) om[R->reac[j]] += q;
      if (R->prod[j] >= 0) om[R->prod[j]] += q;
    }
  }
  for (int k = 0; k < NSP; ++k) g[k] = SMC_W[k] * om[k];
}

/* ---------------------------------------------------------- state */
void or_ns_conserved(const double* T, const double* p, const double* uvw, const double* Y,
                     long long n, double* U) {
  #pragma omp parallel for schedule(static) if (n > 4096)
  for (long long c = 0; c < n; ++c) {
    double Yc[NSP], rinv = 0.0, e = 0.0;
    for (int k = 0; k < NSP; ++k) {
      Yc[k] = Y[k * n + c];
      rinv += Yc[k] / SMC_W[k];
    }
    const double rho = p[c] / (SMC_RU * T[c] * rinv);
    for (int k = 0; k < NSP; ++k) e += Yc[k] * spec_e(k, T[c]);
    const double u = uvw[c], v = uvw[n + c], w = uvw[2 * n + c];
    U[c] = rho;
    U[n + c] = rho * u;
    U[2 * n + c] = rho * v;
    U[3 * n + c] = rho * w;
    U[4 * n + c] = rho * (e + 0.5 * (u * u + v * v + w * w));
    for (int k = 0; k < NSP; ++k) U[(5 + k) * n + c] = rho * Yc[k];
  }
}

/* ctoprim + transport for one cell (PAPER.md:143-188 with the synthetic
 * models of smc_mechanism.h). */
typedef struct {
  double rho, u[3], T, p, Y[NSP], X[NSP], h[NSP];
  double eta, xi, lam, rhoD[NSP];
} cellprim;

static void ctoprim_cell(const double* U, long long n, long long c, cellprim* q) {
  q->rho = U[c];
  const double ri = 1.0 / q->rho;
  for (int i = 0; i < 3; ++i) q->u[i] = U[(1 + i) * n + c] * ri;
  double wsum = 0.0; /* sum_k Y_k / W_k as fma(Y_k, 1 / W_k, .) (the GPU's sequence) */
  for (int k = 0; k < NSP; ++k) {
    q->Y[k] = U[(5 + k) * n + c] * ri;
    wsum = fma(q->Y[k], 1.0 / SMC_W[k], wsum);
  }
  /* e = rho E / rho - |u|^2 / 2 */
  const double k2 = fma(q->u[2], q->u[2], fma(q->u[1], q->u[1], q->u[0] * q->u[0]));
  const double e = fma(-0.5, k2, U[4 * n + c] * ri);
  q->T = temperature(q->Y, e);
  q->p = q->rho * SMC_RU * q->T * wsum;
  for (int k = 0; k < NSP; ++k) {
    q->X[k] = (q->Y[k] / SMC_W[k]) / wsum;
    q->h[k] = spec_h(k, q->T);
  }
  const double s = pow(q->T / SMC_T_REF, SMC_TRANSPORT_EXP);
  double eta = 0.0, lam = 0.0;
  for (int k = 0; k < NSP; ++k) {
    eta += q->X[k] * SMC_MU0[k];
    lam += q->X[k] * SMC_LAM0[k];
    q->rhoD[k] = SMC_RHOD0[k] * s;
  }
  q->eta = eta * s;
  q->lam = lam * s;
  q->xi = SMC_XI_OVER_ETA * q->eta;
}

void or_ns_temperature_pressure(const double* U, long long n, double* T, double* p) {
  #pragma omp parallel for schedule(static) if (n > 4096)
  for (long long c = 0; c < n; ++c) {
    cellprim q;
    ctoprim_cell(U, n, c, &q);
    T[c] = q.T;
    p[c] = q.p;
  }
}

/* ------------------------------------------------------------- RHS */
int or_ns_rhs(const double* U, int nx, int ny, int nz, double dx, double dy, double dz,
              const double* m64, int s, int part, double* out) {
  return or_ns_rhs_terms(U, nx, ny, nz, dx, dy, dz, m64, s, part, OR_T_ALL, out);
}

/* The RHS restricted to the terms in `terms` (OR_T_* of ns_oracle.h); with
 * OR_T_ALL every sum is formed in the same order as the full RHS. */
int or_ns_rhs_terms(const double* U, int nx, int ny, int nz, double dx, double dy, double dz,
                    const double* m64, int s, int part, int terms, double* out) {
  const int hyp = terms & OR_T_HYP, visc = terms & OR_T_VISC, heatc = terms & OR_T_HEAT,
            spec = terms & OR_T_SPEC, enth = terms & OR_T_ENTH;
  const long long n = (long long)nx * ny * nz;
  const double d1[3] = {1.0 / dx, 1.0 / dy, 1.0 / dz};
  const double d2[3] = {1.0 / (dx * dx), 1.0 / (dy * dy), 1.0 / (dz * dz)};
  memset(out, 0, sizeof(double) * NV * n);

  /* primitive and coefficient fields (SoA) */
  enum { F_U = 0, F_T = 3, F_P, F_ETA, F_ETA43, F_LAM2, F_LAM, F_DHP, F_Y, F_X = F_Y + NSP,
         F_D = F_X + NSP, F_DH = F_D + NSP, F_DP = F_DH + NSP, F_HY = F_DP + NSP,
         F_COUNT = F_HY + NSP };
  double* f = malloc(sizeof(double) * F_COUNT * n);
#define FLD(i) (f + (long long)(i) * n)
  double* rho = malloc(sizeof(double) * n);
  #pragma omp parallel for schedule(static) if (n > 4096)
  for (long long c = 0; c < n; ++c) {
    cellprim q;
    ctoprim_cell(U, n, c, &q);
    rho[c] = q.rho;
    for (int i = 0; i < 3; ++i) FLD(F_U + i)[c] = q.u[i];
    FLD(F_T)[c] = q.T;
    FLD(F_P)[c] = q.p;
    FLD(F_ETA)[c] = q.eta;
    FLD(F_ETA43)[c] = 4.0 / 3.0 * q.eta + q.xi;
    FLD(F_LAM2)[c] = q.xi - 2.0 / 3.0 * q.eta;
    FLD(F_LAM)[c] = q.lam;
    double dhp = 0.0;
    for (int k = 0; k < NSP; ++k) {
      FLD(F_Y + k)[c] = q.Y[k];
      FLD(F_X + k)[c] = q.X[k];
      FLD(F_D + k)[c] = q.rhoD[k];
      FLD(F_DH + k)[c] = q.rhoD[k] * q.h[k];
      FLD(F_DP + k)[c] = q.rhoD[k] * (q.X[k] - q.Y[k]) / q.p;
      FLD(F_HY + k)[c] = q.h[k] * q.Y[k];
      dhp += q.rhoD[k] * q.h[k] * (q.X[k] - q.Y[k]) / q.p;
    }
    FLD(F_DHP)[c] = dhp;
  }

  if (part != OR_NS_CHEM) {
    double* tmp = malloc(sizeof(double) * n);
    double* flux = malloc(sizeof(double) * n);
    /* ---- hypterm: -div F, 8th-order centred first derivatives.
     * The momentum flux rho u_i u_d + delta_id p is differentiated as
     * d(rho u_i u_d) + d(p): formed as one number, p (~1e5 Pa) would bury
     * the convective part's low bits, and the rounding of that sum (~eps p
     * / dx) would dominate a weakly driven momentum RHS (uniform p, fine
     * grids).  The same split is exact in exact arithmetic. */
    double* dp = malloc(sizeof(double) * n);
    for (int d = 0; d < 3 && hyp; ++d) {
      const double* ud = FLD(F_U + d);
      or_deriv8_dir(FLD(F_P), nx, ny, nz, d, d1[d], dp);
      for (int v = 0; v < NV; ++v) {
        #pragma omp parallel for schedule(static) if (n > 4096)
        for (long long c = 0; c < n; ++c) {
          double fv;
          if (v == 0)
            fv = U[n + d * n + c];                             /* rho u_d */
          else if (v <= 3)
            fv = U[v * n + c] * ud[c];                         /* + p: dp below */
          else if (v == 4)
            fv = (U[4 * n + c] + FLD(F_P)[c]) * ud[c];
          else
            fv = U[v * n + c] * ud[c];
          flux[c] = fv;
        }
        or_deriv8_dir(flux, nx, ny, nz, d, d1[d], tmp);
        const int with_p = v - 1 == d;
        #pragma omp parallel for schedule(static) if (n > 4096)
        for (long long c = 0; c < n; ++c) out[v * n + c] -= with_p ? tmp[c] + dp[c] : tmp[c];
      }
    }
    free(dp);
    /* ---- diffterm, same-direction second derivatives: narrow stencil */
    double* dm = calloc(3 * n, sizeof(double));
    double* dE = calloc(n, sizeof(double));
    double* dY = calloc(NSP * n, sizeof(double));
    for (int d = 0; d < 3; ++d) {
      for (int i = 0; i < 3 && visc; ++i)
        or_narrow_dir(m64, s, FLD(i == d ? F_ETA43 : F_ETA), FLD(F_U + i), nx, ny, nz, d, d2[d],
                      1, dm + i * n);
      if (heatc) or_narrow_dir(m64, s, FLD(F_LAM), FLD(F_T), nx, ny, nz, d, d2[d], 1, dE);
      for (int k = 0; k < NSP; ++k) {
        if (spec || enth)
          or_narrow_dir(m64, s, FLD(F_D + k), FLD(F_X + k), nx, ny, nz, d, d2[d], 1, dY + k * n);
        if (enth)
          or_narrow_dir(m64, s, FLD(F_DH + k), FLD(F_X + k), nx, ny, nz, d, d2[d], 1, dE);
        if (spec || enth)
          or_narrow_dir(m64, s, FLD(F_DP + k), FLD(F_P), nx, ny, nz, d, d2[d], 1, dY + k * n);
      }
      if (enth) or_narrow_dir(m64, s, FLD(F_DHP), FLD(F_P), nx, ny, nz, d, d2[d], 1, dE);
    }
    /* ---- velocity gradients G[i][j] = d_j u_i */
    double* G = malloc(sizeof(double) * 9 * n);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) or_deriv8_dir(FLD(F_U + i), nx, ny, nz, j, d1[j], G + (3 * i + j) * n);
    /* ---- mixed viscous terms: sum_{j!=i} d_j(eta d_i u_j) + d_i(lam2 sum_{j!=i} d_j u_j) */
    for (int i = 0; i < 3 && visc; ++i) {
      for (int j = 0; j < 3; ++j) {
        if (j == i) continue;
        #pragma omp parallel for schedule(static) if (n > 4096)
        for (long long c = 0; c < n; ++c) flux[c] = FLD(F_ETA)[c] * G[(3 * j + i) * n + c];
        or_deriv8_dir(flux, nx, ny, nz, j, d1[j], tmp);
        #pragma omp parallel for schedule(static) if (n > 4096)
        for (long long c = 0; c < n; ++c) dm[i * n + c] += tmp[c];
      }
      #pragma omp parallel for schedule(static) if (n > 4096)
      for (long long c = 0; c < n; ++c) {
        double sdiv = 0.0;
        for (int j = 0; j < 3; ++j)
          if (j != i) sdiv += G[(3 * j + j) * n + c];
        flux[c] = FLD(F_LAM2)[c] * sdiv;
      }
      or_deriv8_dir(flux, nx, ny, nz, i, d1[i], tmp);
      #pragma omp parallel for schedule(static) if (n > 4096)
      for (long long c = 0; c < n; ++c) dm[i * n + c] += tmp[c];
    }
    /* ---- correction velocity V_c = sum_l Fbar_l */
    double* Vc = calloc(3 * n, sizeof(double));
    double* gp = malloc(sizeof(double) * 3 * n);
    for (int j = 0; j < 3; ++j) or_deriv8_dir(FLD(F_P), nx, ny, nz, j, d1[j], gp + j * n);
    for (int l = 0; l < NSP; ++l)
      for (int j = 0; j < 3; ++j) {
        or_deriv8_dir(FLD(F_X + l), nx, ny, nz, j, d1[j], tmp);
        #pragma omp parallel for schedule(static) if (n > 4096)
        for (long long c = 0; c < n; ++c)
          Vc[j * n + c] -= FLD(F_D + l)[c] * tmp[c] + FLD(F_DP + l)[c] * gp[j * n + c];
      }
    /* div V_c = sum_l div Fbar_l = -sum_l (narrow part of species l) */
    double* divVc = malloc(sizeof(double) * n);
    #pragma omp parallel for schedule(static) if (n > 4096)
    for (long long c = 0; c < n; ++c) {
      double sdv = 0.0;
      for (int k = 0; k < NSP; ++k) sdv += dY[k * n + c];
      divVc[c] = -sdv;
    }
    /* species: -div F_k = -div Fbar_k + Y_k div V_c + V_c . grad Y_k */
    for (int k = 0; k < NSP && spec; ++k) {
      double* o = out + (5 + k) * n;
      #pragma omp parallel for schedule(static) if (n > 4096)
      for (long long c = 0; c < n; ++c) o[c] += dY[k * n + c] + FLD(F_Y + k)[c] * divVc[c];
      for (int j = 0; j < 3; ++j) {
        or_deriv8_dir(FLD(F_Y + k), nx, ny, nz, j, d1[j], tmp);
        #pragma omp parallel for schedule(static) if (n > 4096)
        for (long long c = 0; c < n; ++c) o[c] += Vc[j * n + c] * tmp[c];
      }
    }
    /* energy: div(lam grad T) + div(tau.u) - div sum F_k h_k */
    double* oE = out + 4 * n;
    #pragma omp parallel for schedule(static) if (n > 4096)
    for (long long c = 0; c < n; ++c) {
      double g[3][3];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) g[i][j] = G[(3 * i + j) * n + c];
      const double div = g[0][0] + g[1][1] + g[2][2];
      const double eta = FLD(F_ETA)[c], lam2 = FLD(F_LAM2)[c];
      double heat = 0.0; /* tau : grad u */
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          const double tau = eta * (g[i][j] + g[j][i]) + (i == j ? lam2 * div : 0.0);
          heat += tau * g[i][j];
        }
      double udivtau = 0.0;
      for (int i = 0; i < 3; ++i) udivtau += FLD(F_U + i)[c] * dm[i * n + c];
      double hyd = 0.0;
      for (int k = 0; k < NSP; ++k) hyd += FLD(F_HY + k)[c] * divVc[c];
      oE[c] += dE[c] + (visc ? heat : 0.0) + (visc ? udivtau : 0.0) + (enth ? hyd : 0.0);
    }
    for (int k = 0; k < NSP && enth; ++k)
      for (int j = 0; j < 3; ++j) {
        or_deriv8_dir(FLD(F_HY + k), nx, ny, nz, j, d1[j], tmp);
        #pragma omp parallel for schedule(static) if (n > 4096)
        for (long long c = 0; c < n; ++c) oE[c] += Vc[j * n + c] * tmp[c];
      }
    /* momentum: div tau */
    for (int i = 0; i < 3; ++i)
      #pragma omp parallel for schedule(static) if (n > 4096)
      for (long long c = 0; c < n; ++c) out[(1 + i) * n + c] += dm[i * n + c];
    free(tmp); free(flux); free(dm); free(dE); free(dY); free(G); free(Vc); free(gp); free(divVc);
  }
  if (part != OR_NS_ADVDIFF && (terms & OR_T_CHEM)) {
    /* wdot: rho omega_k */
    #pragma omp parallel for schedule(static) if (n > 4096)
    for (long long c = 0; c < n; ++c) {
      double Y[NSP], w[NSP];
      for (int k = 0; k < NSP; ++k) Y[k] = FLD(F_Y + k)[c];
      or_ns_wdot_cell(rho[c], FLD(F_T)[c], Y, w);
      for (int k = 0; k < NSP; ++k) out[(5 + k) * n + c] += w[k];
    }
  }
#undef FLD
  free(f);
  free(rho);
  return 0;
}

void or_ns_chem_gross(const double* U, long long n, double* gross) {
#pragma omp parallel for schedule(static) if (n > 4096)
  for (long long c = 0; c < n; ++c) {
    cellprim q;
    ctoprim_cell(U, n, c, &q);
    double g[NSP];
    wdot_gross_cell(q.rho, q.T, q.Y, g);
    for (int k = 0; k < NSP; ++k) gross[k * n + c] = g[k];
  }
}
