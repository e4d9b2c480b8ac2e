/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("oracle") of the reference
 * algorithm on the RHS hot path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as the
 * checker.  The product (paper_1309_7327_b200/) never links or calls it.
 *
 * Pinning: the stencil / heat / SDC / MRSDC functions are checked against the
 * reference itself (oracle/_ref, built from /root/reference sources) and
 * against the golden vectors in tests/golden/ (tests/test_oracle.py).  The NS
 * functions (ns_oracle.h) have no reference implementation: "parity unpinned"
 * beyond their narrow-stencil / first-derivative building blocks.
 *
 * Layout conventions: fields are x-fastest, v[(k*ny + j)*nx + i]; periodic in
 * every direction; no ghost cells (periodic wrap by modular indexing, as
 * proj/core/src/pde.cpp:79-83, :100).
 */
#ifndef SMC_ORACLE_H
#define SMC_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

/* stencil.cpp:117-132 + PAPER.md:263-300 (order 8) / :320-345 (order 6).
 * m64 is 8x8 row-major, top-left 2s x 2s used.  Returns 0 or 1 (bad args). */
int or_build_narrow(int order, const double* params, int nparams, double* m64, int* s);

/* stencil_kernel.hpp:13-25: h[i] = sum_mm a[i+mm] * (sum_nn M[mm][nn] u[i+nn]),
 * a/u valid on [-(s-1), n+s-1].  Fixed order: mm ascending outer, nn inner. */
void or_narrow_interfaces(int s, const double* a, const double* u, int n, const double* m64,
                          double* h);

/* stencil.cpp:134-155 (periodic 1-D operator). */
int or_apply_narrow(const double* m64, int s, const double* a, const double* u, int n,
                    double dx, double* out);

/* stencil.cpp:157-169 / stencil_kernel.hpp:48-54 (periodic 8th-order D). */
int or_first_derivative8(const double* u, int n, double dx, double* out);

/* Non-periodic lines with the boundary closure of PAPER.md:449-461 (see
 * oracle.c): m8 = the 8th-order matrix (or_build_narrow(8, ...)), m6 = the
 * 6th-order one for the fourth cells; n >= 8. */
int or_apply_narrow_bounded(const double* m8, const double* m6, const double* a, const double* u,
                            int n, double dx, double* out);
int or_first_derivative_bounded(const double* u, int n, double dx, double* out);
/* stencil.cpp:171-176 */
int or_apply_wide(const double* a, const double* u, int n, double dx, double* out);

/* One direction of the narrow operator on a periodic 3-D box:
 *   out (+)= (H_{i+1/2} - H_{i-1/2}) * inv_d2 along dir (0 = x, 1 = y, 2 = z)
 * with H from coefficient c and field u.  accumulate = 0 overwrites. */
void or_narrow_dir(const double* m64, int s, const double* c, const double* u, int nx, int ny,
                   int nz, int dir, double inv_d2, int accumulate, double* out);

/* Periodic 8th-order first derivative along dir, scaled by inv_d. */
void or_deriv8_dir(const double* u, int nx, int ny, int nz, int dir, double inv_d, double* out);

/* configs[1]: (a U_x)_x + (a U_y)_y + (a U_z)_z, summed x, y, z in that order. */
/* OpenMP thread count of the oracle's loops (0 = all host threads); results
 * are bitwise independent of it. */
void or_set_threads(int n);
int or_get_threads(void);

int or_narrow3d(const double* m64, int s, const double* a, const double* u, int nx, int ny,
                int nz, double dx, double dy, double dz, double* out);

/* HeatOperator::rhs (pde.cpp:85-205): kind 0/1 = narrow (m64, s), 2 = wide.
 * out = (a u_x)_x + (b u_y)_y + g0 * gt (g0 may be NULL). */
int or_heat2d_rhs(int kind, const double* m64, int s, const double* a, const double* b,
                  const double* g0, double gt, const double* u, int nx, int ny, double dx,
                  double dy, double* out);

typedef void (*or_rhs_cb)(double t, const double* u, double* out, long long n, void* ctx);

/* integrate_sdc (sdc.cpp:38-127) given the node set tau[0..M] and the
 * integration matrices q, s (M x (M+1), row-major). */
int or_integrate_sdc(or_rhs_cb f, void* ctx, long long dim, const double* u0, double t0,
                     double t1, int nsteps, int m, const double* tau, const double* q,
                     const double* smat, int iterations, double cutoff, int reuse_first,
                     double* u_out, double* residuals, int max_res, int* sweeps,
                     int* fresh_evals, int* early_stop);

/* integrate_mrsdc mode 1 (mrsdc.cpp:23-135, :227-259) given the hierarchy:
 * coarse nodes t1[0..m1], fine nodes t2[0..m2], s21/q21 m2 x (m1+1),
 * s22/q22 m2 x (m2+1), fine_of_coarse[0..m1], p_map[0..m2]. */
int or_integrate_mrsdc1(or_rhs_cb f1, void* c1, or_rhs_cb f2, void* c2, long long dim,
                        const double* u0, double t0, double tend, int nsteps, int m1,
                        const double* t1, int m2, const double* t2, const double* s21,
                        const double* q21, const double* s22, const double* q22,
                        const int* fine_of_coarse, const int* p_map, int iterations,
                        double cutoff, double* u_out, double* residuals, int max_res,
                        int* sweeps, int* f1_evals, int* f2_evals);

/* StiffOptions (core/include/nsdc/stiff.hpp:10-20) plus the block structure
 * the device solver exploits: f couples only the `block` components of one
 * block (block 0 = dense, the reference's case).  Component j of block b sits
 * at j*nb + b when `interleaved` (structure-of-arrays, the NS state) and at
 * b*block + j otherwise. */
typedef struct {
  double rtol, atol;
  int max_newton_iters;
  long long block;
  int interleaved;
} or_stiff;

/* NewtonReport (stiff.hpp:22-27) */
typedef struct {
  int iterations;
  double final_residual;
  int converged;
  int f_evals;
} or_newton_report;

/* solve_backward_euler (core/src/stiff.cpp:34-76, fd_jacobian :16-30,
 * lu_factor/lu_solve core/src/matrix.cpp:9-51): w = c + beta f(t, w) by
 * Newton from guess.  With block > 0 the finite-difference Jacobian is formed
 * one block column at a time (every block perturbed at once) and factored
 * per block; for a block-local f this equals the dense computation bit for
 * bit.  Returns 0, or 1 on bad arguments; convergence is in *rep. */
int or_solve_backward_euler(or_rhs_cb f, void* ctx, long long dim, double t, double beta,
                            const double* c, const double* guess, const or_stiff* opts,
                            double* w, or_newton_report* rep);

/* integrate_mrsdc, mode 2 (core/src/mrsdc.cpp:137-206, :227-259): f1 implicit
 * on the coarse nodes.  Returns 0, 1 on bad arguments, 2 when a Newton solve
 * fails (*fail_node = coarse node, *fail_sweep = sweep). */
int or_integrate_mrsdc2(or_rhs_cb f1, void* c1, or_rhs_cb f2, void* c2, long long dim,
                        const double* u0, double t0, double tend, int nsteps, int m1,
                        const double* t1, int m2, const double* t2, const double* s21,
                        const double* q21, const double* s22, const double* q22,
                        const int* fine_of_coarse, int iterations, double cutoff,
                        const or_stiff* opts, double* u_out, double* residuals, int max_res,
                        int* sweeps, int* f1_evals, int* f2_evals, int* implicit_solves,
                        int* newton_f1_evals, int* fail_node, int* fail_sweep);

/* integrate_stiff (core/src/stiff.cpp:80-188): adaptive backward Euler /
 * variable-step BDF2 with step doubling, over or_solve_backward_euler.
 * Returns 0, 1 on bad arguments (span < 0, bad tolerances), 2 when the step
 * size collapses (*t_fail = the time reached). */
int or_integrate_stiff(or_rhs_cb f, void* ctx, long long dim, const double* u0, double t0,
                       double t1, const or_stiff* opts, double initial_step_fraction,
                       double* u_out, int* accepted, int* rejected, double* t_fail);

#ifdef __cplusplus
}
#endif
#endif
