/*
 * smc_mechanism.h — the BUILDER-DEFINED SYNTHETIC 9-species H2/O2/N2-shaped
 * mechanism, thermodynamics and transport used by the NS right-hand side.
 *
 * The reference (`nsdc`) contains no Navier-Stokes physics and no mechanism
 * (SURVEY.md §0); the paper cites a published 9-species H2/O2
 * mechanism and EGLIB transport that are not in
 * /root/reference.  Per the task rules no published mechanism is reproduced:
 * every rate, thermodynamic and transport coefficient below is SELF-CHOSEN.
 * Only the species set, their elemental composition (hence molecular
 * weights) and element-balanced reaction stoichiometry are physical facts.
 * This is input data (an "input deck") shared by the product kernels and the
 * CPU oracle, not an algorithm.
 *
 * Units: SI.  W [kg/mol]; cp_k/R_k = a0 + a1 T + a2 T^2;
 * h_k/R_k = a0 T + a1 T^2/2 + a2 T^3/3 + b  [K];  R_k = R_u / W_k.
 * Transport: eta_k = mu0_k s, lambda_k = lam0_k s, rhoD_k = rhoD0_k s with
 * s = (T / 300 K)^0.7; mixture eta = sum X_k eta_k, lambda = sum X_k
 * lambda_k; bulk viscosity xi = XI_OVER_ETA * eta.
 * Kinetics: k = A T^b exp(-Ea / (R_u T)) for forward and reverse
 * directions independently (no equilibrium constants), third body
 * [M] = sum_k C_k with unit efficiencies.  The prefactors are sized so that
 * at 1200-1800 K the fastest radical time scale is ~50-200 acoustic steps at
 * dx = 1e-4 m (CFL 0.5): explicit SDC on the full RHS (configs[2]) stays
 * well inside its stability region, and a 100x faster chemistry (which made
 * explicit SDC at CFL 0.5 blow up on the configs[3] hot spot) remains a
 * one-line change for MRSDC studies.
 */
#ifndef SMC_MECHANISM_H
#define SMC_MECHANISM_H

#define SMC_NSP 9
#define SMC_NREAC 13
#define SMC_NVAR (5 + SMC_NSP) /* rho, rho u, rho v, rho w, rho E, rho Y_k */

/* species order */
enum { SP_H2 = 0, SP_O2, SP_H2O, SP_H, SP_O, SP_OH, SP_HO2, SP_H2O2, SP_N2 };

#define SMC_RU 8.314462618      /* J / (mol K) */
#define SMC_T_REF 300.0
#define SMC_TRANSPORT_EXP 0.7
#define SMC_XI_OVER_ETA 0.25

static const double SMC_W[SMC_NSP] = {2.01588e-3, 31.9988e-3, 18.01528e-3, 1.00794e-3, 15.9994e-3,
                                      17.00734e-3, 33.00674e-3, 34.01468e-3, 28.0134e-3};

/* cp/R polynomial {a0, a1, a2} and enthalpy offset b [K] (self-chosen) */
static const double SMC_THERMO[SMC_NSP][4] = {
    {3.40, 1.0e-4, 1.0e-8, 0.0},      /* H2 */
    {3.30, 6.0e-4, -1.0e-7, 0.0},     /* O2 */
    {3.60, 9.0e-4, -1.0e-7, -29000.0},/* H2O */
    {2.50, 0.0, 0.0, 26000.0},        /* H */
    {2.60, -1.0e-4, 2.0e-8, 30000.0}, /* O */
    {3.50, 1.0e-4, 1.0e-8, 4500.0},   /* OH */
    {4.00, 1.2e-3, -2.0e-7, 1500.0},  /* HO2 */
    {4.50, 2.0e-3, -3.0e-7, -16000.0},/* H2O2 */
    {3.25, 5.0e-4, -8.0e-8, 0.0},     /* N2 */
};

/* transport prefactors at 300 K (self-chosen): mu0 [Pa s], lam0 [W/m/K],
 * rhoD0 [kg/m/s].  rhoD_k multiplies grad X_k in Fbar_k,
 * so it already carries the W_k / W factor of a mass-based mixture
 * coefficient: light species (H, H2) get small rhoD0 and every species'
 * effective mass diffusivity rhoD_k W / (rho W_k) stays ~1e-4..2e-3 m^2/s. */
static const double SMC_MU0[SMC_NSP] = {9.0e-6, 2.0e-5, 1.0e-5, 6.0e-6, 1.5e-5,
                                        1.5e-5, 2.0e-5, 1.9e-5, 1.8e-5};
static const double SMC_LAM0[SMC_NSP] = {0.18, 0.026, 0.018, 0.40, 0.05, 0.05, 0.027, 0.025, 0.026};
static const double SMC_RHOD0[SMC_NSP] = {5.7e-6, 2.5e-5, 1.7e-5, 4.3e-6, 2.0e-5,
                                          2.1e-5, 2.6e-5, 2.7e-5, 2.1e-5};

/* Reactions: up to 3 reactant / product species indices (-1 = none),
 * third-body flag, forward {A, b, Ea}, reverse {A, b, Ea} (self-chosen). */
typedef struct {
  int reac[3];
  int prod[3];
  int third_body;
  double fwd[3];
  double rev[3];
} smc_reaction;

/* The reaction list as an X-macro, so C code gets the table below and CUDA
 * code can unroll over compile-time species indices:
 * X(reactant0..2, product0..2, third_body, A_f, b_f, Ea_f, A_r, b_r, Ea_r). */
#define SMC_REACTION_LIST(X) \
  /* H + O2 = O + OH */ \
  X(SP_H, SP_O2, -1, SP_O, SP_OH, -1, 0, 2e+06, 0.0, 70000.0, 1.2e+05, 0.2, 2000.0) \
  /* O + H2 = H + OH */ \
  X(SP_O, SP_H2, -1, SP_H, SP_OH, -1, 0, 0.0005, 2.6, 26000.0, 0.00022, 2.6, 18000.0) \
  /* OH + H2 = H2O + H */ \
  X(SP_OH, SP_H2, -1, SP_H2O, SP_H, -1, 0, 2, 1.5, 14000.0, 9, 1.5, 77000.0) \
  /* O + H2O = OH + OH */ \
  X(SP_O, SP_H2O, -1, SP_OH, SP_OH, -1, 0, 0.03, 2.0, 56000.0, 0.01, 2.0, 3000.0) \
  /* H2 + M = H + H + M */ \
  X(SP_H2, -1, -1, SP_H, SP_H, -1, 1, 4.5e+11, -1.4, 436000.0, 1e+04, -1.0, 0.0) \
  /* O + O + M = O2 + M */ \
  X(SP_O, SP_O, -1, SP_O2, -1, -1, 1, 60, -0.5, 0.0, 2e+10, -0.9, 495000.0) \
  /* H + OH + M = H2O + M */ \
  X(SP_H, SP_OH, -1, SP_H2O, -1, -1, 1, 2.2e+08, -2.0, 0.0, 3e+15, -2.5, 500000.0) \
  /* H + O2 + M = HO2 + M */ \
  X(SP_H, SP_O2, -1, SP_HO2, -1, -1, 1, 6e+03, -0.8, 0.0, 2e+10, -0.6, 205000.0) \
  /* HO2 + H = OH + OH */ \
  X(SP_HO2, SP_H, -1, SP_OH, SP_OH, -1, 0, 7e+05, 0.0, 1200.0, 200, 0.6, 150000.0) \
  /* HO2 + H = H2 + O2 */ \
  X(SP_HO2, SP_H, -1, SP_H2, SP_O2, -1, 0, 2.8e+05, 0.0, 4500.0, 5e+04, 0.3, 230000.0) \
  /* HO2 + OH = H2O + O2 */ \
  X(SP_HO2, SP_OH, -1, SP_H2O, SP_O2, -1, 0, 2.9e+05, 0.0, 0.0, 1e+06, 0.2, 290000.0) \
  /* HO2 + HO2 = H2O2 + O2 */ \
  X(SP_HO2, SP_HO2, -1, SP_H2O2, SP_O2, -1, 0, 4e+04, 0.0, 5000.0, 1e+06, 0.0, 160000.0) \
  /* H2O2 + M = OH + OH + M */ \
  X(SP_H2O2, -1, -1, SP_OH, SP_OH, -1, 1, 1.2e+09, 0.0, 190000.0, 2.3e+04, -0.8, 0.0)

#define SMC_REACTION_ENTRY(r0, r1, r2, p0, p1, p2, tb, af, bf, ef, ar, br, er) \
  {{r0, r1, r2}, {p0, p1, p2}, tb, {af, bf, ef}, {ar, br, er}},
static const smc_reaction SMC_REACTIONS[SMC_NREAC] = {SMC_REACTION_LIST(SMC_REACTION_ENTRY)};
#undef SMC_REACTION_ENTRY

#endif /* SMC_MECHANISM_H */
