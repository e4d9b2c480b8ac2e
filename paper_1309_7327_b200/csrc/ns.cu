// NS right-hand side kernels (see ns.cuh).  The decomposition follows the CPU
// oracle (oracle/ns_oracle.c), so every intermediate is comparable:
//   prim      : ctoprim (Newton for T) + transport + coefficient fields
//   phase A   : per direction, the narrow diffusion terms, hyperbolic flux
//               derivatives, velocity gradients, V_c (ns_dir.inc)
//   phase B   : per direction, the mixed viscous derivatives of
//               eta d_i u_j and lam2 div u (formed while staging)
//   assemble2 : pointwise terms (tau:grad u, u . div tau, V_c) + wdot
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "ns.cuh"

namespace smc {

namespace {

constexpr int NSP = SMC_NSP;
constexpr int NV = SMC_NVAR;

// prim_ field indices (same roles as the oracle's F_* enum)
// The transport factor s (rhoD_k = rhoD0_k s) is stored once; rhoD_k,
// eta43 = (4/3 + xi/eta) eta and lam2 = (xi/eta - 2/3) eta are formed where
// they are used.
enum : int {
  F_U = 0, F_T = 3, F_P, F_ETA, F_LAM, F_DHP, F_HYS, F_S, F_RHO, F_Y,
  F_X = F_Y + NSP, F_DH = F_X + NSP, F_DP = F_DH + NSP, F_COUNT = F_DP + NSP
};
// acc_ fields (interior): the narrow momentum results (+ div tau, phase B)
// and sum over species of the narrow species results (for div V_c), each
// summed over the three directions in order
enum : int { A_DM = 0, A_DY = 3, A_COUNT };
// scratch_ blocks (interior arrays): NA_1 | HY_1 (phase A's x + y sums)
enum : int { SC_NA1 = 0, SC_HY1 = SC_NA1 + 4, SC_COUNT = SC_HY1 + SMC_NVAR };

struct Tables {
  double W[NSP], th[NSP][4], mu0[NSP], lam0[NSP], rhoD0[NSP];
  // derived on the host: R_k = R_u / W_k, 1 / W_k and the enthalpy
  // polynomial in Horner form {a0, a1/2, a2/3, a3}: no divisions per cell
  double R[NSP], Winv[NSP], hc[NSP][4], hcm1[NSP];
  double kf[SMC_NREAC][3], kr[SMC_NREAC][3];
  int reac[SMC_NREAC][3], prod[SMC_NREAC][3], tb[SMC_NREAC];
};
__constant__ Tables cT;

struct Geo {
  int nx, ny, nz, G;
  long long plane, flen;
  double d1[3], d2[3];
  double dc[3][4];  // the 8th-order first-derivative weights over the spacing, per direction
};

// 8th-order centred first derivative (stencil_kernel.hpp:48-54) from a
// 9-point window w[0..8] centred at w[4], with the weights already divided
// by the spacing (Geo::dc: kernel-parameter constants, no scaling multiply)
__device__ __forceinline__ double deriv8_c(const double* w, const double* c) {
  double r = c[0] * (w[5] - w[3]);
  r = __fma_rn(c[1], w[6] - w[2], r);
  r = __fma_rn(c[2], w[7] - w[1], r);
  return __fma_rn(c[3], w[8] - w[0], r);
}

// Device view of the conserved state (NsStateView): the three blocks as
// base pointers rebased so that block b's element of in-interior offset o
// (plane-0 relative, ghost planes negative) is p_b + o + v * fs_b.  Scalar
// members and selects: an indexed array would live in local memory.
struct UV {
  const double *p0, *p1, *p2;
  long long fs0, fs1, fs2;
  long long lim1;  // offset of plane nz (block 0 ends at offset 0)
  // address of field 0 of the cell at offset o, and that block's field stride
  __device__ __forceinline__ const double* at(long long o, long long& fs) const {
    const bool lo = o < 0, hi = o >= lim1;
    fs = lo ? fs0 : hi ? fs2 : fs1;
    return (lo ? p0 : hi ? p2 : p1) + o;
  }
};

__device__ __forceinline__ long long zo(const Geo& g, int k) {
  if (g.G == 0) k = wrap_near(k, g.nz);
  return static_cast<long long>(k) * g.plane;
}

// e_k, h_k, cv_k of the thermodynamic polynomial (smc_mechanism.h), Horner
// form with host-derived coefficients
__device__ __forceinline__ double spec_e(int k, double T) {
  const double* c = cT.hc[k];
  return cT.R[k] * (c[3] + T * ((c[0] - 1.0) + T * (c[1] + T * c[2])));
}
__device__ __forceinline__ double spec_h(int k, double T) {
  const double* c = cT.hc[k];
  return cT.R[k] * (c[3] + T * (c[0] + T * (c[1] + T * c[2])));
}

// T from e by Newton on the mixture's energy cubic: e(T) = sum_k Y_k e_k(T)
// = E0 + T (E1 + T (E2 + T E3)) with cv = de/dT = E1 + T (2 E2 + 3 E3 T), so
// an iteration costs two Horner evaluations instead of 2 x 9 species sums.
//
// The operation sequence is fixed with explicit roundings (_rn intrinsics,
// fused multiply-adds where written) and restated operation for operation
// by the oracle (oracle/ns_oracle.c temperature(), with C fma()), so T, and
// p below, are the same bits on both sides.  That matters: on fine grids of
// a nearly uniform-pressure state the momentum RHS is -grad p plus small
// terms, and a per-cell difference of a few ulps of p (~1e5 Pa) becomes
// eps p / dx ~ 1e-7 after differentiation, ~3e-10 of the momentum RHS at
// 256^3 (measured), above the single-RHS bar.
__device__ double temperature(const double* Y, double e) {
  double E0 = 0.0, E1 = 0.0, E2 = 0.0, E3 = 0.0;
#pragma unroll
  for (int k = 0; k < NSP; ++k) {
    const double yr = __dmul_rn(Y[k], cT.R[k]);
    const double* c = cT.hc[k];
    E0 = __fma_rn(yr, c[3], E0);
    E1 = __fma_rn(yr, cT.hcm1[k], E1);
    E2 = __fma_rn(yr, c[1], E2);
    E3 = __fma_rn(yr, c[2], E3);
  }
  E0 = __dsub_rn(E0, e);
  const double D2 = __dmul_rn(2.0, E2), D3 = __dmul_rn(3.0, E3);
  double T = 1000.0;
  for (int it = 0; it < 50; ++it) {
    const double f = __fma_rn(T, __fma_rn(T, __fma_rn(T, E3, E2), E1), E0);
    const double df = __fma_rn(T, __fma_rn(T, D3, D2), E1);
    const double dT = __ddiv_rn(f, df);
    T = __dsub_rn(T, dT);
    if (fabs(dT) <= __dmul_rn(1e-9, T)) break;
  }
  return T;
}

// Specific internal energy from the conserved state (canonical sequence,
// shared bit for bit with the oracle): e = rho E / rho - |u|^2 / 2.
__device__ __forceinline__ double internal_energy(double rhoE, double ri, const double* u) {
  const double k2 = __fma_rn(u[2], u[2], __fma_rn(u[1], u[1], __dmul_rn(u[0], u[0])));
  return __fma_rn(-0.5, k2, __dmul_rn(rhoE, ri));
}

// ---------------------------------------------------------------- prim
// planes [k0, k1) of the ghosted workspace (k in [-G, nz + G))
__global__ void __launch_bounds__(256, 3) prim_kernel(const UV U, double* __restrict__ F, Geo g,
                                                   int k0, int k1) {
  const long long n = g.flen;  // F: all planes incl. ghosts
  const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (r >= (k1 - k0) * g.plane) return;
  const long long o = r + k0 * g.plane;  // offset relative to interior plane 0
  const long long c = o + g.G * g.plane;
  long long fs;
  const double* uc = U.at(o, fs);
  const double rho = uc[0];
  const double ri = __ddiv_rn(1.0, rho);
  double u[3], Y[NSP], X[NSP];
  for (int i = 0; i < 3; ++i) u[i] = __dmul_rn(uc[(1 + i) * fs], ri);
  double wsum = 0.0;  // sum_k Y_k / W_k (canonical sequence, as the oracle)
#pragma unroll
  for (int k = 0; k < NSP; ++k) {
    Y[k] = __dmul_rn(uc[(5 + k) * fs], ri);
    wsum = __fma_rn(Y[k], cT.Winv[k], wsum);
  }
  const double e = internal_energy(uc[4 * fs], ri, u);
  const double T = temperature(Y, e);
  const double p = __dmul_rn(__dmul_rn(__dmul_rn(rho, SMC_RU), T), wsum);
  const double s = pow(T / SMC_T_REF, SMC_TRANSPORT_EXP);
  double eta = 0.0, lam = 0.0, dhp = 0.0, hys = 0.0;
  const double pinv = 1.0 / p, wsinv = 1.0 / wsum;
#pragma unroll
  for (int k = 0; k < NSP; ++k) {
    X[k] = (Y[k] * cT.Winv[k]) * wsinv;
    eta += X[k] * cT.mu0[k];
    lam += X[k] * cT.lam0[k];
  }
  eta *= s;
  lam *= s;
  for (int i = 0; i < 3; ++i) F[(F_U + i) * n + c] = u[i];
  F[F_T * n + c] = T;
  F[F_RHO * n + c] = rho;
  F[F_P * n + c] = p;
  F[F_ETA * n + c] = eta;
  F[F_LAM * n + c] = lam;
#pragma unroll
  for (int k = 0; k < NSP; ++k) {
    const double h = spec_h(k, T);
    const double rd = cT.rhoD0[k] * s;
    F[(F_Y + k) * n + c] = Y[k];
    F[(F_X + k) * n + c] = X[k];
    F[(F_DH + k) * n + c] = rd * h;
    F[(F_DP + k) * n + c] = rd * (X[k] - Y[k]) * pinv;
    dhp += rd * h * (X[k] - Y[k]) * pinv;
    hys += h * Y[k];
  }
  F[F_DHP * n + c] = dhp;
  F[F_HYS * n + c] = hys;
  F[F_S * n + c] = s;
}

// ------------------------------------------------------------ narrow
// v'_r of the interface whose window starts at u[0]: v_r with the sign of
// rows r >= S folded in (narrow_vsd, common.cuh), so the dot is plain.
template <int S>
__device__ __forceinline__ void narrow_v(const double* u, const StencilM& M, double* v) {
  narrow_vsd<S>(u, M, v);
}
template <int S>
__device__ __forceinline__ double narrow_dot(const double* a, const double* v) {
  return narrow_adot<S>(a, v);
}

// ------------------------------------------------------------- wdot
// Species indices of every reaction as compile-time constants (the
// mechanism's X-macro), so the concentration and production arrays stay in
// registers; the rate parameters come from the constant bank.
struct RxIdx {
  int r[3], p[3], tb;
};
#define SMC_RX_IDX(r0, r1, r2, p0, p1, p2, tb, af, bf, ef, ar, br, er) \
  RxIdx{{r0, r1, r2}, {p0, p1, p2}, tb},
constexpr RxIdx kRx[SMC_NREAC] = {SMC_REACTION_LIST(SMC_RX_IDX)};
#undef SMC_RX_IDX

// exp(x) for the Arrhenius factors (|x| well inside (-708, 709)): x = (32 n
// + j) ln2 / 32 + r with |r| <= ln2 / 64 (Cody-Waite, the split ln2 / 32 is
// exact for |32 n + j| < 2^21), exp(r) by its Taylor polynomial of degree 6
// (truncation 1.7e-17 relative), times 2^(j/32) from a 32-entry table
// (correctly rounded on the host) and 2^n added to the exponent bits: 11
// FP64 instructions and one L1-resident load per exponential (the degree-12
// reduction by ln2 took 16; the chemistry part 0.87 -> 0.80 ms at 256^3);
// max relative error 3.0e-16 against expl over [-700, 700] (1.4 ulp,
// measured on 2^20 points), and the chemistry part agrees with the oracle's
// glibc exp to ~1e-14.
__device__ double gExp2J[32];
__device__ __forceinline__ double arrhenius_exp(double x) {
  const double kd = rint(x * 46.166241308446828784);  // 32 / ln2
  const int k = static_cast<int>(kd);
  double r = __fma_rn(kd, -2.166084938653512e-02, x);     // ln2_hi / 32 (exact)
  r = __fma_rn(kd, -5.9631716539705865626e-12, r);         // ln2_lo / 32
  double q = 1.38888888888888888889e-03;                  // 1/6!
  q = __fma_rn(q, r, 8.33333333333333333333e-03);
  q = __fma_rn(q, r, 4.16666666666666666667e-02);
  q = __fma_rn(q, r, 1.66666666666666666667e-01);
  q = __fma_rn(q, r, 0.5);
  q = __fma_rn(q, r, 1.0);
  q = __fma_rn(q, r, 1.0);
  const double t = __dmul_rn(__ldg(&gExp2J[k & 31]), q);
  return __longlong_as_double(__double_as_longlong(t) + (static_cast<long long>(k >> 5) << 52));
}

// Temperature exponent and activation energy of every rate as compile-time
// constants: a rate with no activation energy and a temperature exponent of
// 0, -1 or -2 is A, A / T or A / T^2 (no exponential; 3 of the 26 rates of
// the built-in mechanism)
struct RxArr {
  double bf, ef, br, er;
};
#define SMC_RX_ARR(r0, r1, r2, p0, p1, p2, tb, af, bf, ef, ar, br, er) RxArr{bf, ef, br, er},
constexpr RxArr kArr[SMC_NREAC] = {SMC_REACTION_LIST(SMC_RX_ARR)};
#undef SMC_RX_ARR

template <int R, bool FWD>
__device__ __forceinline__ double rate(double lnT, double invRT) {
  constexpr double b = FWD ? kArr[R].bf : kArr[R].br, e = FWD ? kArr[R].ef : kArr[R].er;
  const double* k = FWD ? cT.kf[R] : cT.kr[R];
  if constexpr (e == 0.0 && b == 0.0) {
    return k[0];
  } else if constexpr (e == 0.0 && (b == -1.0 || b == -2.0)) {
    const double invT = invRT * SMC_RU;
    return b == -1.0 ? k[0] * invT : k[0] * (invT * invT);
  } else {
    return k[0] * arrhenius_exp(k[1] * lnT - k[2] * invRT);
  }
}

template <int R>
__device__ __forceinline__ void rx_step(const double* C, double M, double lnT, double invRT,
                                        double* om) {
  constexpr RxIdx x = kRx[R];
  const double kf = rate<R, true>(lnT, invRT);
  const double kr = rate<R, false>(lnT, invRT);
  double qf = kf, qr = kr;
  if constexpr (x.r[0] >= 0) qf *= C[x.r[0]];
  if constexpr (x.p[0] >= 0) qr *= C[x.p[0]];
  if constexpr (x.r[1] >= 0) qf *= C[x.r[1]];
  if constexpr (x.p[1] >= 0) qr *= C[x.p[1]];
  if constexpr (x.r[2] >= 0) qf *= C[x.r[2]];
  if constexpr (x.p[2] >= 0) qr *= C[x.p[2]];
  if constexpr (x.tb != 0) {
    qf *= M;
    qr *= M;
  }
  const double q = qf - qr;
  if constexpr (x.r[0] >= 0) om[x.r[0]] -= q;
  if constexpr (x.p[0] >= 0) om[x.p[0]] += q;
  if constexpr (x.r[1] >= 0) om[x.r[1]] -= q;
  if constexpr (x.p[1] >= 0) om[x.p[1]] += q;
  if constexpr (x.r[2] >= 0) om[x.r[2]] -= q;
  if constexpr (x.p[2] >= 0) om[x.p[2]] += q;
}
template <int... R>
__device__ __forceinline__ void rx_all(std::integer_sequence<int, R...>, const double* C,
                                       double M, double lnT, double invRT, double* om) {
  (rx_step<R>(C, M, lnT, invRT, om), ...);
}

// rho omega_k W_k of one cell (smc_mechanism.h kinetics)
__device__ __forceinline__ void wdot_cell(double rho, double T, const double* Y, double* w) {
  double C[NSP], M = 0.0, om[NSP];
#pragma unroll
  for (int s = 0; s < NSP; ++s) {
    C[s] = rho * Y[s] * cT.Winv[s];
    M += C[s];
    om[s] = 0.0;
  }
  const double lnT = log(T), invRT = 1.0 / (SMC_RU * T);
  rx_all(std::make_integer_sequence<int, SMC_NREAC>{}, C, M, lnT, invRT, om);
#pragma unroll
  for (int s = 0; s < NSP; ++s) w[s] = cT.W[s] * om[s];
}

// chemistry part alone (MRSDC f2): ctoprim's temperature + wdot fused, so the
// 32 chemistry calls of an MRSDC step read the 14 conserved fields and write
// the RHS without materialising the primitive workspace.
__device__ __forceinline__ void chem_cell(const double* Uc, double* o) {
  const double rho = Uc[0];
  const double ri = __ddiv_rn(1.0, rho);
  double u[3], Y[NSP], w[NSP];
  for (int i = 0; i < 3; ++i) u[i] = __dmul_rn(Uc[1 + i], ri);
#pragma unroll
  for (int k = 0; k < NSP; ++k) Y[k] = __dmul_rn(Uc[5 + k], ri);
  wdot_cell(rho, temperature(Y, internal_energy(Uc[4], ri, u)), Y, w);
  for (int v = 0; v < 5; ++v) o[v] = 0.0;
#pragma unroll
  for (int s = 0; s < NSP; ++s) o[5 + s] = w[s];
}

__global__ void __launch_bounds__(256) chem_kernel(const UV U, double* __restrict__ out,
                                                   long long out_fs, Geo g) {
  const long long n = g.plane * g.nz;
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  const double* uc = U.p1 + c;  // interior block
  double Uc[NV], o[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) Uc[v] = uc[v * U.fs1];
  chem_cell(Uc, o);
#pragma unroll
  for (int v = 0; v < NV; ++v) out[v * out_fs + c] = o[v];
}

// The MRSDC fine-node update fused with the chemistry part: per cell, the 14
// updated state values next = cur + sum_d dc_d (da_d - db_d) + pre (the
// arithmetic of sweep_update_kernel<ND, 0>) stay in registers for chem_cell,
// so the chemistry does not re-read the state the update just wrote.
struct ChemUpdP {
  double* next;
  const double *cur, *pre, *da[2], *db[2];
  double dc[2];
  double* out;
  long long n;
};
template <int ND>
__global__ void __launch_bounds__(256) chem_update_kernel(const ChemUpdP p) {
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (c >= p.n) return;
  double Uc[NV], o[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const long long i = v * p.n + c;
    double x = p.cur[i];
#pragma unroll
    for (int d = 0; d < ND; ++d) x = __fma_rn(p.dc[d], __dsub_rn(p.da[d][i], p.db[d][i]), x);
    x = __dadd_rn(x, p.pre[i]);
    p.next[i] = x;
    Uc[v] = x;
  }
  chem_cell(Uc, o);
#pragma unroll
  for (int v = 0; v < NV; ++v) p.out[v * p.n + c] = o[v];
}

// The chemistry part's FD Jacobian, one cell per thread: column j from the
// cell's state with component j perturbed, as DeviceNewton's column loop
// (fd_perturb_kernel, the chemistry evaluation, fd_column_kernel) forms it,
// without the 14 full-grid passes.  Periodic box (no ghost planes).
__global__ void __launch_bounds__(128, 4) chem_fd_jacobian_kernel(const double* __restrict__ U,
                                                               const double* __restrict__ FU,
                                                               double* __restrict__ jac, long long n,
                                                               double atol, double root_eps) {
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  double w[NV], fw[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) w[v] = U[v * n + c], fw[v] = FU[v * n + c];
#pragma unroll 1
  for (int j = 0; j < NV; ++j) {
    double wp[NV], fp[NV];
    double hv = 0.0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      wp[v] = w[v];
      if (v == j) {
        const double a = fabs(w[v]);
        hv = __dmul_rn(root_eps, (a < atol) ? atol : a);
        wp[v] = __dadd_rn(w[v], hv);
      }
    }
    chem_cell(wp, fp);
    const double inv = 1.0 / hv;
#pragma unroll
    for (int r = 0; r < NV; ++r) jac[(r * NV + j) * n + c] = __dmul_rn(__dsub_rn(fp[r], fw[r]), inv);
  }
}

__global__ void __launch_bounds__(256) tp_kernel(const double* __restrict__ F, double* T,
                                                 double* p, Geo g) {
  const long long n = g.plane * g.nz;
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  const long long cg = c + g.G * g.plane;
  T[c] = F[F_T * g.flen + cg];
  p[c] = F[F_P * g.flen + cg];
}

__global__ void __launch_bounds__(256) conserved_kernel(const double* __restrict__ T,
                                                        const double* __restrict__ p,
                                                        const double* __restrict__ uvw,
                                                        const double* __restrict__ Y, long long n,
                                                        double* __restrict__ U) {
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  double Yc[NSP], rinv = 0.0, e = 0.0;
#pragma unroll
  for (int s = 0; s < NSP; ++s) {
    Yc[s] = Y[s * n + c];
    rinv += Yc[s] * cT.Winv[s];
  }
  const double rho = p[c] / (SMC_RU * T[c] * rinv);
#pragma unroll
  for (int s = 0; s < NSP; ++s) e += Yc[s] * spec_e(s, T[c]);
  const double u = uvw[c], v = uvw[n + c], w = uvw[2 * n + c];
  U[c] = rho;
  U[n + c] = rho * u;
  U[2 * n + c] = rho * v;
  U[3 * n + c] = rho * w;
  U[4 * n + c] = rho * (e + 0.5 * (u * u + v * v + w * w));
#pragma unroll
  for (int s = 0; s < NSP; ++s) U[(5 + s) * n + c] = rho * Yc[s];
}

void upload_tables() {
  static bool done = false;
  if (done) return;
  Tables t{};
  for (int s = 0; s < NSP; ++s) {
    t.W[s] = SMC_W[s];
    for (int q = 0; q < 4; ++q) t.th[s][q] = SMC_THERMO[s][q];
    t.mu0[s] = SMC_MU0[s];
    t.lam0[s] = SMC_LAM0[s];
    t.rhoD0[s] = SMC_RHOD0[s];
    t.R[s] = SMC_RU / SMC_W[s];
    t.Winv[s] = 1.0 / SMC_W[s];
    t.hc[s][0] = SMC_THERMO[s][0];
    t.hc[s][1] = SMC_THERMO[s][1] / 2.0;
    t.hc[s][2] = SMC_THERMO[s][2] / 3.0;
    t.hc[s][3] = SMC_THERMO[s][3];
    t.hcm1[s] = SMC_THERMO[s][0] - 1.0;
  }
  for (int r = 0; r < SMC_NREAC; ++r) {
    for (int q = 0; q < 3; ++q) {
      t.kf[r][q] = SMC_REACTIONS[r].fwd[q];
      t.kr[r][q] = SMC_REACTIONS[r].rev[q];
      t.reac[r][q] = SMC_REACTIONS[r].reac[q];
      t.prod[r][q] = SMC_REACTIONS[r].prod[q];
    }
    t.tb[r] = SMC_REACTIONS[r].third_body;
  }
  SMC_CUDA(cudaMemcpyToSymbol(cT, &t, sizeof(t)));
  double e2[32];
  for (int j = 0; j < 32; ++j) e2[j] = static_cast<double>(exp2l(j / 32.0L));
  SMC_CUDA(cudaMemcpyToSymbol(gExp2J, e2, sizeof(e2)));
  done = true;
}

int blocks(long long n) { return static_cast<int>((n + 255) / 256); }

#include "ns_dir.inc"

#ifndef SMC_B3_WAVES
#define SMC_B3_WAVES 4  // fused phase B: about this many waves of z-chunk CTAs
#endif

template <class K>
void set_smem(K kern, std::size_t bytes) {
  SMC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
}

// The direction-split evaluation; `phase` selects the part that needs no
// ghost plane (kNsInterior: ctoprim and the x / y passes on the interior
// planes), the rest (kNsBoundary) or both (kNsAll).
template <int S>
void rhs_v2(const Geo& g, const UV& U, const double* F, double* A, double* GR, double* SC,
            double* out, long long ofs, const StencilM& M, int chem, int phase,
            cudaStream_t st, KernelMarks* marks) {
  auto mark = [&](const char* name) {
    if (marks) marks->mark(name, st);
  };
  static bool configured = false;
  const std::size_t sm0 = sizeof(DirSmem<0>), sm1 = sizeof(DirSmem<1>), sm2 = sizeof(DirSmem<2>);
  if (!configured) {
    set_smem(ns_phase_a<0, S>, sm0), set_smem(ns_phase_a<1, S>, sm1), set_smem(ns_phase_a<2, S>, sm2);
    const std::size_t smb = sizeof(PBSmem);
    set_smem(ns_phase_b<0>, smb), set_smem(ns_phase_b<1>, smb), set_smem(ns_phase_b<2>, smb);
    set_smem(ns_phase_b3, sizeof(B3Smem));
    configured = true;
  }
  const int allp = g.nz + 2 * g.G;
  const long long n = g.plane * g.nz;
  // scratch SC (SC_COUNT arrays of n): phase A of directions 1, 2 -> [NA |
  // HY] x 2, phase B of the three directions; ns_assemble2 adds them in
  double* na1 = SC + SC_NA1 * n;
  double* hy1 = SC + SC_HY1 * n;
  constexpr int NT0 = Tile<0, nr_a<0>()>::THREADS, NT1 = Tile<1, nr_a<1>()>::THREADS;
  // ctoprim + the x / y passes over planes [k0, k0 + np)
  auto planes = [&](int k0, int np) {
    if (np <= 0) return;
    prim_kernel<<<blocks(np * g.plane), 256, 0, st>>>(U, const_cast<double*>(F), g, k0, k0 + np);
    SMC_CHECK_LAUNCH();
    mark("prim");
    dim3 g0 = dir_grid<0, nr_a<0>()>(g, np), g1 = dir_grid<1, nr_a<1>()>(g, np);
    ns_phase_a<0, S><<<g0, NT0, sm0, st>>>(F, A, nullptr, GR, out, ofs, nullptr, 0, g, M, k0);
    SMC_CHECK_LAUNCH();
    mark("phase_a_x");
    ns_phase_a<1, S><<<g1, NT1, sm1, st>>>(F, na1, A, GR, hy1, n, out, ofs, g, M, k0);
    SMC_CHECK_LAUNCH();
    mark("phase_a_y");
  };
  if (phase == kNsAll) planes(-g.G, allp);
  if (phase == kNsInterior) planes(0, g.nz);
  if (phase == kNsInterior) return;
  if (phase == kNsBoundary) {
    planes(-g.G, g.G);
    planes(g.nz, g.G);
  }
  ns_phase_a<2, S><<<dir_grid<2, nr_a<2>()>(g, allp), NT1, sm2, st>>>(F, A, na1, GR, out, ofs, hy1, n, g, M, 0);
  SMC_CHECK_LAUNCH();
  mark("phase_a_z");
  if (g.nx % B3X == 0 && g.ny % B3Y == 0) {
    // all three directions in one z-march
    const int tiles = (g.nx / B3X) * (g.ny / B3Y);
    const int resident = 2 * num_sms();
    const int chunks = std::max(1, std::min(g.nz / 16, (SMC_B3_WAVES * resident + tiles - 1) / tiles));
    const int kc = (g.nz + chunks - 1) / chunks;
    ns_phase_b3<<<dim3(tiles, (g.nz + kc - 1) / kc), B3T, sizeof(B3Smem), st>>>(F, GR, A, g, kc);
    SMC_CHECK_LAUNCH();
    mark("phase_b");
    ns_assemble2<<<blocks(n), 256, 0, st>>>(F, GR, A, out, ofs, g, chem);
  } else {
    ns_phase_b<0><<<dir_grid<0>(g, g.nz), DT_THREADS, sizeof(PBSmem), st>>>(F, GR, A, g);
    SMC_CHECK_LAUNCH();
    mark("phase_b_x");
    ns_phase_b<1><<<dir_grid<1>(g, g.nz), DT_THREADS, sizeof(PBSmem), st>>>(F, GR, A, g);
    SMC_CHECK_LAUNCH();
    mark("phase_b_y");
    ns_phase_b<2><<<dir_grid<2>(g, g.nz), DT_THREADS, sizeof(PBSmem), st>>>(F, GR, A, g);
    SMC_CHECK_LAUNCH();
    mark("phase_b_z");
    ns_assemble2<<<blocks(n), 256, 0, st>>>(F, GR, A, out, ofs, g, chem);
  }
  SMC_CHECK_LAUNCH();
  mark(chem ? "assemble_wdot" : "assemble");
}

}  // namespace

void KernelMarks::mark(const char* name, cudaStream_t st) {
  cudaEvent_t e;
  SMC_CUDA(cudaEventCreate(&e));
  SMC_CUDA(cudaEventRecord(e, st));
  ev.emplace_back(name, e);
}

KernelMarks::~KernelMarks() {
  for (auto& p : ev) cudaEventDestroy(p.second);
  if (start) cudaEventDestroy(start);
}

NsWorkspace::NsWorkspace(const NsBox& box, double dx, double dy, double dz, const StencilM& M,
                         int s)
    : box_(box), M_(M), s_(s) {
  require(box.nx >= 9 && box.ny >= 9, "ns: need at least 9 cells in x and y");
  require(box.nx % 2 == 0, "ns: nx must be even (16-byte staging of x-contiguous pairs)");
  require(box.G == 0 ? box.nz >= 9 : (box.G >= 4 && box.nz >= 1),
          "ns: need nz >= 9 (periodic) or >= 4 ghost planes (slab)");
  require(s == 4 || s == 3, "ns: narrow half width must be 3 or 4");
  require(dx > 0 && dy > 0 && dz > 0, "ns: spacings must be positive");
  dx_[0] = dx, dx_[1] = dy, dx_[2] = dz;
  upload_tables();
  prim_.resize(static_cast<std::size_t>(F_COUNT) * box.field_len());
  acc_.resize(static_cast<std::size_t>(A_COUNT) * box.cells());
  grad_.resize(static_cast<std::size_t>(9) * box.field_len());
  scratch_.resize(static_cast<std::size_t>(SC_COUNT) * box.cells());
}

static Geo make_geo(const NsBox& b, const double* d) {
  Geo g;
  g.nx = b.nx, g.ny = b.ny, g.nz = b.nz, g.G = b.G;
  g.plane = b.plane();
  g.flen = b.field_len();
  for (int q = 0; q < 3; ++q) {
    g.d1[q] = 1.0 / d[q], g.d2[q] = 1.0 / (d[q] * d[q]);
    const double c[4] = {4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0};
    for (int j = 0; j < 4; ++j) g.dc[q][j] = c[j] / d[q];
  }
  return g;
}

static UV make_uv(const NsStateView& v, const NsBox& b) {
  UV u;
  const long long plane = b.plane(), n = b.cells();
  u.p1 = v.mid, u.fs1 = v.mid_fs;
  if (b.G == 0) {
    u.p0 = u.p2 = v.mid, u.fs0 = u.fs2 = v.mid_fs;
  } else {
    // rebase each block so that p + (plane-0 relative offset) addresses it
    u.p0 = v.lo + b.G * plane, u.fs0 = v.lo_fs;
    u.p2 = v.hi - n, u.fs2 = v.hi_fs;
  }
  u.lim1 = n;
  return u;
}

void NsWorkspace::rhs(const double* U, double* out, int part, cudaStream_t st) {
  rhs(NsStateView::ghosted(U, box_), out, box_.cells(), part, st, kNsAll);
}

void NsWorkspace::rhs(const NsStateView& U, double* out, long long out_fs, int part,
                      cudaStream_t st, int phase) {
  // the direction kernels stage U with 16-byte copies and write out with
  // 16-byte stores (x-contiguous cell pairs)
  auto al16 = [](const void* p) { return reinterpret_cast<std::uintptr_t>(p) % 16 == 0; };
  const bool ghosts = box_.G > 0;
  require(U.mid && (!ghosts || (U.lo && U.hi)), "ns rhs: missing state block");
  require(al16(U.mid) && al16(out) && (!ghosts || (al16(U.lo) && al16(U.hi))) &&
              U.mid_fs % 2 == 0 && (!ghosts || (U.lo_fs % 2 == 0 && U.hi_fs % 2 == 0)) &&
              out_fs % 2 == 0,
          "ns rhs: U and out must be 16-byte aligned device arrays");
  require(out_fs >= box_.cells() && U.mid_fs >= box_.cells(), "ns rhs: field stride too small");
  const Geo g = make_geo(box_, dx_);
  const UV uv = make_uv(U, box_);
  const long long n = box_.cells();
  if (part == kNsChem) {
    if (phase == kNsBoundary) return;  // pointwise: all of it is interior work
    chem_kernel<<<blocks(n), 256, 0, st>>>(uv, out, out_fs, g);
    SMC_CHECK_LAUNCH();
    if (marks_) marks_->mark("chem", st);
    return;
  }
  double* F = prim_.get();
  double* A = acc_.get();
  if (s_ == 4)
    rhs_v2<4>(g, uv, F, A, grad_.get(), scratch_.get(), out, out_fs, M_,
              part == kNsFull, phase, st, marks_);
  else
    rhs_v2<3>(g, uv, F, A, grad_.get(), scratch_.get(), out, out_fs, M_,
              part == kNsFull, phase, st, marks_);
}

std::shared_ptr<NsWorkspace> NsWorkspace::chunk_workspace(int nz_chunk) const {
  NsBox b = box_;
  b.nz = nz_chunk;
  b.G = 4;
  return std::make_shared<NsWorkspace>(b, dx_[0], dx_[1], dx_[2], M_, s_);
}

NsRhsOp::~NsRhsOp() {
  for (cudaEvent_t e : ev_in_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_done_) cudaEventDestroy(e);
  if (ev_halo_) cudaEventDestroy(ev_halo_);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (d2h_) cudaStreamDestroy(d2h_);
}

// Chunk boundaries of the host pipeline: short chunks at both ends (the
// pipeline's fill and drain), SMC_NS_E2E_CHUNK planes (default 16) in the
// middle; every chunk holds >= 8 planes (2 x the halo).  Empty when the box
// is too short to pipeline.
std::vector<int> ns_e2e_bounds(int nz) {
  static const int mid = [] {  // 16 / 32 / 64: 47.4 / 49.9 / 58.8 ms best-of-5 at 256^3
    const char* e = std::getenv("SMC_NS_E2E_CHUNK");
    return e ? std::max(8, std::atoi(e)) : 16;
  }();
  std::vector<int> b{0};
  if (nz < 2 * mid) return {};
  int lo = 0, hi = nz;
  std::vector<int> tail;
  for (int w : {8, 8, 16}) {  // ramp: 8, 8, 16 planes at each end
    if (hi - lo < 2 * w + mid) break;
    lo += w, b.push_back(lo);
    hi -= w, tail.push_back(hi);
  }
  const int nm = std::max(1, (hi - lo + mid - 1) / mid);
  for (int q = 1; q < nm; ++q) b.push_back(lo + static_cast<int>(1LL * (hi - lo) * q / nm));
  b.push_back(hi);
  for (auto it = tail.rbegin(); it != tail.rend(); ++it) b.push_back(*it == hi ? -1 : *it);
  b.erase(std::remove(b.begin(), b.end(), -1), b.end());
  if (b.back() != nz) b.push_back(nz);
  return b;
}

void NsRhsOp::eval_host(double t, const double* u, double* out) {
  const NsBox& b = ws_->box();
  const std::vector<int> bnd = b.G == 0 ? ns_e2e_bounds(b.nz) : std::vector<int>{};
  if (bnd.size() < 3) {
    RhsOp::eval_host(t, u, out);
    return;
  }
  const int nch = static_cast<int>(bnd.size()) - 1, G = 4;
  const long long n = b.cells(), plane = b.plane();
  stage_u_.resize(static_cast<std::size_t>(SMC_NVAR) * n);
  stage_out_.resize(static_cast<std::size_t>(SMC_NVAR) * n);
  auto ws_for = [&](int kc) -> NsWorkspace& {
    for (auto& w : chunk_ws_)
      if (w->box().nz == kc) return *w;
    chunk_ws_.push_back(ws_->chunk_workspace(kc));
    return *chunk_ws_.back();
  };
  if (!h2d_) {
    SMC_CUDA(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
    SMC_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
    SMC_CUDA(cudaEventCreateWithFlags(&ev_halo_, cudaEventDisableTiming));
  }
  while (static_cast<int>(ev_in_.size()) < nch) {
    cudaEvent_t a, c;
    SMC_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    SMC_CUDA(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
    ev_in_.push_back(a);
    ev_done_.push_back(c);
  }
  double* dU = stage_u_.get();
  double* dO = stage_out_.get();
  auto copy = [&](double* dst, const double* src, int k0, int k1, cudaMemcpyKind kind,
                  cudaStream_t st) {
    for (int v = 0; v < SMC_NVAR; ++v)
      SMC_CUDA(cudaMemcpyAsync(dst + v * n + k0 * plane, src + v * n + k0 * plane,
                               sizeof(double) * (k1 - k0) * plane, kind, st));
  };
  // the previous call's reads of the staging buffers precede this call's writes
  SMC_CUDA(cudaEventRecord(ev_halo_, stream_));
  SMC_CUDA(cudaStreamWaitEvent(h2d_, ev_halo_, 0));
  copy(dU, u, b.nz - G, b.nz, cudaMemcpyHostToDevice, h2d_);  // chunk 0's lower halo
  SMC_CUDA(cudaEventRecord(ev_halo_, h2d_));
  for (int c = 0; c < nch; ++c) {
    const int k0 = bnd[c], k1 = c + 1 == nch ? b.nz - G : bnd[c + 1];
    copy(dU, u, k0, k1, cudaMemcpyHostToDevice, h2d_);
    SMC_CUDA(cudaEventRecord(ev_in_[c], h2d_));
  }
  for (int c = 0; c < nch; ++c) {
    const int k0 = bnd[c], k1 = bnd[c + 1];
    if (c == 0) SMC_CUDA(cudaStreamWaitEvent(stream_, ev_halo_, 0));
    SMC_CUDA(cudaStreamWaitEvent(stream_, ev_in_[c], 0));
    if (c + 1 < nch) SMC_CUDA(cudaStreamWaitEvent(stream_, ev_in_[c + 1], 0));
    const NsStateView view{dU + ((k0 - G + b.nz) % b.nz) * plane, n, dU + k0 * plane, n,
                           dU + (k1 % b.nz) * plane, n};
    ws_for(k1 - k0).rhs(view, dO + k0 * plane, n, part_, stream_, kNsAll);
    SMC_CUDA(cudaEventRecord(ev_done_[c], stream_));
    SMC_CUDA(cudaStreamWaitEvent(d2h_, ev_done_[c], 0));
    copy(out, dO, k0, k1, cudaMemcpyDeviceToHost, d2h_);
  }
  SMC_CUDA(cudaStreamSynchronize(d2h_));
  ++evals_;
}

bool NsWorkspace::chem_after_update(double* next, const double* cur, int nd,
                                    const double* const* da, const double* const* db,
                                    const double* dc, const double* pre, double* out,
                                    cudaStream_t st) {
  if (nd < 0 || nd > 2 || !pre) return false;
  ChemUpdP p{};
  p.next = next, p.cur = cur, p.pre = pre, p.out = out, p.n = box_.cells();
  for (int d = 0; d < nd; ++d) p.da[d] = da[d], p.db[d] = db[d], p.dc[d] = dc[d];
  const unsigned nb = static_cast<unsigned>((p.n + 255) / 256);
  if (nd == 0)
    chem_update_kernel<0><<<nb, 256, 0, st>>>(p);
  else if (nd == 1)
    chem_update_kernel<1><<<nb, 256, 0, st>>>(p);
  else
    chem_update_kernel<2><<<nb, 256, 0, st>>>(p);
  SMC_CHECK_LAUNCH();
  if (marks_) marks_->mark("chem_update", st);
  return true;
}

bool NsWorkspace::chem_fd_jacobian(const double* U, const double* FU, double* jac, double atol,
                                   double root_eps, cudaStream_t st) {
  if (box_.G != 0) return false;
  const long long n = box_.cells();
  chem_fd_jacobian_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(U, FU, jac, n,
                                                                                  atol, root_eps);
  SMC_CHECK_LAUNCH();
  return true;
}

void NsWorkspace::temperature_pressure(const double* U, double* T, double* p, cudaStream_t st) {
  const Geo g = make_geo(box_, dx_);
  prim_kernel<<<blocks(g.flen), 256, 0, st>>>(make_uv(NsStateView::ghosted(U, box_), box_),
                                              prim_.get(), g, -g.G, g.nz + g.G);
  SMC_CHECK_LAUNCH();
  tp_kernel<<<blocks(box_.cells()), 256, 0, st>>>(prim_.get(), T, p, g);
  SMC_CHECK_LAUNCH();
}

void ns_conserved_from_primitives(const double* T, const double* p, const double* uvw,
                                  const double* Y, long long n, double* U, cudaStream_t st) {
  upload_tables();
  conserved_kernel<<<blocks(n), 256, 0, st>>>(T, p, uvw, Y, n, U);
  SMC_CHECK_LAUNCH();
}

}  // namespace smc
