/* TEST INFRASTRUCTURE ONLY — see oracle.h for the usage rule.
 *
 * CPU restatement of the multicomponent reacting Navier-Stokes right-hand
 * side of PAPER.md:143-213 (equations), :215-249 (8th-order narrow stencil
 * for same-direction second derivatives, 8th-order centred first
 * derivatives elsewhere), :399-428 (correction velocity by the chain rule),
 * with the builder-defined synthetic mechanism of include/smc_mechanism.h.
 *
 * PARITY UNPINNED beyond its building blocks: the reference contains no NS
 * physics, so no reference test or golden vector pins these
 * results.  The building blocks are pinned: or_narrow_dir / or_deriv8_dir
 * equal the reference kernels bitwise (tests/test_oracle.py).  Physics-
 * independent checks (conservation, sum of mass production rates, order of
 * accuracy) are in tests/test_ns.py.
 *
 * State layout: U[v * N + cell], v = rho, rho u, rho v, rho w, rho E,
 * rho Y_1..9; cell = (k*ny + j)*nx + i, periodic box.
 */
#ifndef SMC_NS_ORACLE_H
#define SMC_NS_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

#define OR_NS_FULL 0
#define OR_NS_ADVDIFF 1 /* hypterm + diffterm: the MRSDC "f1" */
#define OR_NS_CHEM 2    /* wdot: the MRSDC "f2" */

/* ctoprim (+ transport): writes T and p of every cell (for tests). */
void or_ns_temperature_pressure(const double* U, long long n, double* T, double* p);

/* RHS of the 14 conserved equations (part: full / advection-diffusion /
 * chemistry).  m64/s: the narrow-stencil coupling matrix (or_build_narrow). */
int or_ns_rhs(const double* U, int nx, int ny, int nz, double dx, double dy, double dz,
              const double* m64, int s, int part, double* out);

/* Term selection for or_ns_rhs_terms (the manufactured-solution tests pin
 * each physical term separately against the exact calculus):
 *   HYP   -div of the Euler fluxes (all 14 equations)
 *   VISC  div tau (momentum) and div(tau . u) (energy)
 *   HEAT  div(lambda grad T) (energy)
 *   SPEC  -div F_k = -div Fbar_k + div(Y_k V_c) (species)
 *   ENTH  -div sum_k F_k h_k (energy)
 *   CHEM  rho omega_k (species) */
#define OR_T_HYP 1
#define OR_T_VISC 2
#define OR_T_HEAT 4
#define OR_T_SPEC 8
#define OR_T_ENTH 16
#define OR_T_CHEM 32
#define OR_T_ALL 63
int or_ns_rhs_terms(const double* U, int nx, int ny, int nz, double dx, double dy, double dz,
                    const double* m64, int s, int part, int terms, double* out);

/* rho omega_k W_k for one cell (mass production rates, kg/m^3/s). */
void or_ns_wdot_cell(double rho, double T, const double* Y, double* wdot);

/* Gross chemistry magnitudes W_k sum_r |nu_rk| (qf_r + qr_r) per cell
 * (gross[k * n + c]); diagnostics for the wdot cancellation (tests). */
void or_ns_chem_gross(const double* U, long long n, double* gross);

/* Conserved state from (rho-free) primitives: T, p, u, v, w, Y_k per cell. */
void or_ns_conserved(const double* T, const double* p, const double* uvw, const double* Y,
                     long long n, double* U);

#ifdef __cplusplus
}
#endif
#endif
