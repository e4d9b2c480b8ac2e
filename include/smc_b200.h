/*
 * smc_b200.h — C ABI of the B200-native RHS library (libsmc_b200.so).
 *
 * Drop-in boundary for the reference `nsdc` library's RHS hot path
 * (/root/reference/proj/core).  Every entry point below names the reference
 * interface it replaces (file:line, relative to /root/reference/proj).  The
 * ABI is plain C: pointers, sizes, status codes; no C++ or torch types.
 * The C++ mirror of the reference API (include/nsdc_b200/*.hpp) and the
 * Python bindings (paper_1309_7327_b200/_capi.py) are thin layers over it.
 *
 * Conventions
 *  - Fields are fp64, x fastest: v[(k*ny + j)*nx + i] (the reference Field2D
 *    flattening, core/include/nsdc/pde.hpp:24-35, extended by one axis).
 *  - `where` says where caller pointers live: SMC_HOST (staged through the
 *    library's device buffers, synchronous) or SMC_DEVICE (stream-ordered on
 *    the handle's stream, asynchronous).
 *  - Status: SMC_OK, SMC_EINVAL (reference: std::invalid_argument),
 *    SMC_EINTEGRATION (reference: nsdc::IntegrationError,
 *    core/include/nsdc/errors.hpp:16-19), SMC_ECUDA.  smc_last_error() gives
 *    the message of the last failure on the calling thread.
 *  - Handles are not thread-safe; use one per host thread (the reference
 *    steppers carry the same rule, core/include/nsdc/sdc.hpp:43-44).
 */
#ifndef SMC_B200_H
#define SMC_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMC_OK 0
#define SMC_EINVAL 1
#define SMC_EINTEGRATION 2
#define SMC_ECUDA 3

#define SMC_HOST 0
#define SMC_DEVICE 1

/* StencilChoice::Kind (core/include/nsdc/stencil.hpp:65-75) */
#define SMC_NARROW8 0
#define SMC_NARROW6 1
#define SMC_WIDE8 2

/* NodeKind families (core/include/nsdc/quadrature.hpp:9) */
#define SMC_GAUSS_LOBATTO 0
#define SMC_CLENSHAW_CURTIS 1

typedef struct smc_rhs smc_rhs;     /* a right-hand side f(t, u) on the device */
typedef struct smc_sdc smc_sdc;     /* device-resident single-rate SDC stepper */
typedef struct smc_mrsdc smc_mrsdc; /* device-resident multirate SDC stepper */
typedef struct smc_comm smc_comm;   /* one rank of a z-slab decomposition (NCCL or local) */

typedef void (*smc_rhs_fn)(double t, const double* u, double* out, long long n, void* ctx);
typedef double (*smc_time_fn)(double t, void* ctx);
typedef void (*smc_field_fn)(double t, double* field, void* ctx);
typedef double (*smc_reduce_fn)(double local, void* ctx);
/* device-side callback: u, out are device pointers, stream the handle's
 * cudaStream_t; must be stream-ordered on it */
typedef void (*smc_dev_rhs_fn)(double t, const double* u, double* out, long long n, void* stream,
                               void* ctx);

/* Sweep diagnostics: SweepDiagnostics (core/include/nsdc/sdc.hpp:30-35) and
 * MrsdcDiagnostics (core/include/nsdc/mrsdc.hpp:30-38).  `residuals` is a
 * caller buffer of `residual_capacity` doubles; n_residuals is the full
 * history length (entries past the capacity are dropped). */
typedef struct {
  int sweeps;
  int fresh_evals;
  int f1_evals;
  int f2_evals;
  int early_stop;
  int nonfinite;
  int n_residuals;
  int residual_capacity;
  double* residuals;
  int implicit_solves;  /* MRSDC mode 2 */
  int newton_f1_evals;  /* f1 evaluations inside Newton, counted apart */
} smc_diag;

/* StiffOptions (core/include/nsdc/stiff.hpp:10-20) plus the block structure
 * of the implicit term: f couples only the `block` components of one block
 * (0 = dense, the reference's case).  Component j of block b lives at
 * j*(n/block) + b when `interleaved` (structure-of-arrays, e.g. the 14 NS
 * fields of one cell), else at b*block + j.  The finite-difference Jacobian
 * then costs `block` evaluations per Newton step instead of n, and the LU is
 * batched per block; for a block-local f the result equals the dense
 * computation bit for bit. */
typedef struct {
  double rtol;          /* 1e-8 */
  double atol;          /* 1e-10 */
  int max_newton_iters; /* 16 */
  long long block;
  int interleaved;
  double initial_step_fraction; /* 1e-3: integrate_stiff's first step as a fraction of the span */
} smc_stiff;

/* NewtonReport (core/include/nsdc/stiff.hpp:22-27) */
typedef struct {
  int iterations;
  double final_residual;
  int converged;
  int f_evals;
} smc_newton_report;

/* ------------------------------------------------------------- library */
int smc_version(void);
const char* smc_last_error(void);
/* Number of kernel launches issued by this library since load (evidence
 * counter for bench.py's gpu_launches). */
long long smc_launch_count(void);
int smc_synchronize(void);
/* FP64 pipe peak of the current device (DFMA loop, TFLOP/s): the FP64
 * roofline denominator (no reference counterpart). */
int smc_measure_fp64_peak(int iters, double* tflops);
/* FP64 tensor path (mma.sync m8n8k4 f64) throughput; mode 1 mixes DMMA and
 * DFMA warps.  Diagnostic only. */
int smc_measure_dmma_peak(int iters, int mode, double* tflops);
/* TFLOP/s of up to n DFMA probe variants (chains per thread, operand
 * placement, warps per SM): the best of them and of the DMMA probe is the
 * FP64 roofline denominator (bench.py reports them all). */
int smc_measure_fp64_variants(int iters, double* tflops, int n);

/* ------------------------------------------------------------- stencil */
/* nsdc::build_narrow — core/src/stencil.cpp:117-132.  m64: 8x8 row-major. */
int smc_build_narrow(int order, const double* params, int nparams, double* m64, int* s);
/* nsdc::apply_narrow — core/src/stencil.cpp:134-155 (periodic 1-D, on device). */
int smc_apply_narrow(int order, const double* params, int nparams, const double* a,
                     const double* u, int n, double dx, double* out, int where);
/* nsdc::first_derivative8 — core/src/stencil.cpp:157-169. */
int smc_first_derivative8(const double* u, int n, double dx, double* out, int where);
/* Non-periodic lines (no reference counterpart: the reference's operators
 * are periodic; this is the physical-boundary closure of PAPER.md:449-461):
 * nlines contiguous lines of n >= 8 cells.  Diffusion (a u_x)_x: 8th-order
 * narrow stencils from the fifth cell in, 6th / 4th-order centred narrow
 * stencils at the fourth / third cells, centred 2nd order at the second and
 * completely biased 2nd order at the boundary cell.  params = {} (SMC
 * defaults), {m47, m48} or {m47, m48, m36} (the 6th-order matrix of the
 * fourth cells; default 281/3600, stencil.hpp:33). */
int smc_apply_narrow_bounded(const double* params, int nparams, const double* a, const double* u,
                             int n, int nlines, double dx, double* out, int where);
/* First derivative with the same closure: 8th / 6th / 4th-order centred,
 * biased 3rd order at the second cell and completely biased 3rd order at
 * the boundary cell. */
int smc_first_derivative_bounded(const double* u, int n, int nlines, double dx, double* out,
                                 int where);
/* nsdc::apply_wide — core/src/stencil.cpp:171-176. */
int smc_apply_wide(const double* a, const double* u, int n, double dx, double* out, int where);

/* --------------------------------------------------------- operators */
/* HeatOperator(const HeatProblem&, const Grid2D&, const StencilChoice&) —
 * core/include/nsdc/pde.hpp:69-84, core/src/pde.cpp:209-258.  a, b, g0 are
 * the problem's a(x,y), b(x,y), g_space(x,y) sampled on the nodes (host
 * arrays, nx*ny; g0 may be NULL).  params: {m47, m48} / {m36} / unused. */
int smc_heat_create(int nx, int ny, int kind, const double* params, const double* a,
                    const double* b, const double* g0, smc_rhs** out);
/* separable source g0 * g_time(t) (pde.cpp:107-108, :121-123) */
int smc_heat_set_time_source(smc_rhs* h, smc_time_fn g_time, void* ctx);
/* non-separable source g(t, x, y) filled on the grid per call (pde.cpp:124-126) */
int smc_heat_set_full_source(smc_rhs* h, smc_field_fn g_full, void* ctx);

/* 3-D narrow operator (a U_x)_x + (a U_y)_y + (a U_z)_z on a periodic box —
 * the composition of narrow_interfaces<S> / narrow_interfaces_rows<S>
 * (core/src/stencil_kernel.hpp:13-44) used by narrow_rhs_rows<S>
 * (core/src/pde.cpp:85-129), one axis up (BASELINE.json configs[1]). */
int smc_narrow3d_create(int nx, int ny, int nz, double dx, double dy, double dz, int order,
                        const double* params, int nparams, const double* a, int where,
                        smc_rhs** out);
/* The same operator on one z-slab of a block-decomposed periodic box
 * (multi-GPU): `a` (and every u passed to apply_planes)
 * holds nz + 2*zghost planes, zghost >= S ghost planes below and above the
 * interior, filled by the caller's halo exchange; out holds the nz interior
 * planes.  Device pointers; stream-ordered on the handle's stream. */
int smc_narrow3d_create_slab(int nx, int ny, int nz, int zghost, double dx, double dy, double dz,
                             int order, const double* params, int nparams, const double* a,
                             int where, smc_rhs** out);
/* Interior planes [kbeg, kend) only, so the interior can run while the halo
 * is in flight and the boundary planes after it lands. */
int smc_narrow3d_apply_planes(smc_rhs* op, const double* u, double* out, int kbeg, int kend);
/* Peer halo (multi-GPU without an exchange step): apply a slab operator
 * (smc_narrow3d_create_slab, zghost >= S, coefficient ghosts filled once) to
 * u holding only the nz interior planes; the S planes below / above are read
 * inside the kernel from the neighbours' interior arrays u_lo (nz_lo planes,
 * its top planes are used) and u_hi (its bottom planes).  The pointers are
 * device addresses valid in this process: a neighbour GPU's buffer opened
 * with smc_ipc_import (peer loads over NVLink) or another buffer on this
 * device.  The caller orders the neighbours' writes before the call (e.g. a
 * stream-ordered NCCL all-reduce of one element) and keeps the buffers alive. */
int smc_narrow3d_apply_peer(smc_rhs* h, const double* u, const double* u_lo, int nz_lo,
                            const double* u_hi, double* out, int kbeg, int kend);
/* CUDA IPC of device buffers between the processes of one node.  Export
 * whole allocations (e.g. from smc_device_alloc): the importer maps the
 * allocation base. */
#define SMC_IPC_HANDLE_BYTES 64
int smc_device_alloc(long long nbytes, void** dptr);
int smc_device_free(void* dptr);
int smc_ipc_export(const void* dptr, unsigned char* handle /* SMC_IPC_HANDLE_BYTES */);
int smc_ipc_import(const unsigned char* handle, void** dptr);
int smc_ipc_close(void* dptr);
/* z planes per CTA of the narrow kernel (tuning knob; 0 = heuristic). */
int smc_narrow3d_set_kc(smc_rhs* op, int kc);

/* Multicomponent reacting Navier-Stokes RHS (
 * no reference implementation) with the builder-defined
 * synthetic 9-species mechanism of include/smc_mechanism.h.  State: SMC_NVAR
 * (= 14) fields of nx*ny*nz cells, field-major (rho, rho u, rho v, rho w,
 * rho E, rho Y_1..9).  One workspace, three Rhs views: the full RHS, the
 * advection-diffusion part (MRSDC f1: hypterm + diffterm) and the chemistry
 * part (MRSDC f2: wdot) — the split of PAPER.md:732-735.  Any view pointer
 * may be NULL.  zghost = 0: periodic box (interior-only arrays); zghost >= 4:
 * one z-slab, arrays passed to smc_ns_rhs_ghosted carry the ghost planes.
 * nx must be even (the stencil kernels stage x-contiguous 16-byte pairs) and
 * nx, ny >= 9; otherwise SMC_EINVAL. */
int smc_ns_create(int nx, int ny, int nz, int zghost, double dx, double dy, double dz, int order,
                  const double* params, int nparams, smc_rhs** full, smc_rhs** advdiff,
                  smc_rhs** chem);
/* Slab mode: out (interior) = RHS of U (SMC_NVAR ghosted fields), device. */
int smc_ns_rhs_ghosted(smc_rhs* ns, const double* U, double* out);
/* One evaluation of a periodic NS view on device buffers with an event after
 * every kernel: ms[i] / names[i] (static strings) of the first cap kernels in
 * launch order, *count = kernels launched.  For bench.py's per-kernel table. */
int smc_ns_profile(smc_rhs* ns, const double* U, double* out, double* ms, const char** names,
                   int cap, int* count);
/* ctoprim: temperature and pressure of every interior cell. */
int smc_ns_temperature_pressure(smc_rhs* ns, const double* U, double* T, double* p, int where);
/* Conserved state from T, p, velocity (3 fields), Y (9 fields); n cells. */
int smc_ns_conserved(const double* T, const double* p, const double* uvw, const double* Y,
                     long long n, double* U, int where);

/* ---- multi-GPU: z-slab decomposition of the NS box ----
 * The reference is single-process (parallel_for over rows, parallel.cpp:20-36);
 * the paper decomposes the box into boxes with 4 ghost cells and recomputes
 * the coefficients on the ghosts.  A rank owns
 * nz interior planes of an nx x ny x (nz * size) periodic box; its RHS is an
 * smc_rhs of dim 14 nx ny nz that the device steppers advance unchanged (the
 * drop-in nsdc::Rhs contract, field.hpp:14-16), exchanging 4 ghost planes
 * of the conserved state with its two neighbours per evaluation (NCCL
 * send/recv on a communication stream, overlapped with ctoprim and the x / y
 * passes of the interior planes).  Results are bitwise independent of the
 * number of ranks. */
/* NCCL unique id (128 bytes) for smc_comm_init; created on one rank and
 * shared with the others by the caller.  SMC_ECUDA if libnccl is absent. */
int smc_comm_unique_id(char* id128);
/* This process's rank of an NCCL communicator of nranks on the current device. */
int smc_comm_init(const char* id128, int nranks, int rank, smc_comm** out);
/* nranks ranks of one in-process group on the current device (device copies
 * instead of NCCL): out[0..nranks).  For testing several slabs on one GPU;
 * each rank's state must be published (smc_ns_slab_publish) before a
 * neighbour evaluates. */
int smc_comm_init_local(int nranks, smc_comm** out);
int smc_comm_rank(const smc_comm* c, int* rank, int* size);
/* *v = max over ranks of *v (synchronous). */
int smc_comm_allreduce_max(smc_comm* c, double* v);
int smc_comm_destroy(smc_comm* c);
/* This rank's slab RHS views (full / advection-diffusion / chemistry, as
 * smc_ns_create) of the nx x ny x (nz * size) periodic box. */
int smc_ns_slab_create(smc_comm* c, int nx, int ny, int nz, double dx, double dy, double dz,
                       int order, const double* params, int nparams, smc_rhs** full,
                       smc_rhs** advdiff, smc_rhs** chem);
/* In-process groups: the device state u the neighbours read in their next
 * evaluation (an evaluation publishes its own input too).  No-op for NCCL. */
int smc_ns_slab_publish(smc_rhs* slab, const double* u);
/* The steppers' residual max-norm (sdc.cpp:20-30, mrsdc.cpp:23-35) and the
 * implicit solver's norms reduced over the communicator's ranks, so every
 * rank takes the same sweeps and Newton steps. */
int smc_sdc_set_comm(smc_sdc* s, smc_comm* c);
int smc_mrsdc_set_comm(smc_mrsdc* m, smc_comm* c);

/* Any host callback as an operator (nsdc::Rhs, core/include/nsdc/field.hpp:14-16). */
int smc_rhs_from_callback(long long dim, smc_rhs_fn f, void* ctx, smc_rhs** out);

/* A callback that works on device buffers itself (e.g. a multi-GPU RHS whose
 * halo exchange is issued by the host through NCCL) — lets the device
 * steppers drive any RHS without host round trips. */
int smc_rhs_from_device_callback(long long dim, smc_dev_rhs_fn f, void* ctx, smc_rhs** out);

/* Rhs call: out = f(t, u) — HeatOperator::rhs / as_rhs (pde.cpp:266-284). */
int smc_rhs_eval(smc_rhs* op, double t, const double* u, double* out, int where);
long long smc_rhs_dim(const smc_rhs* op);
/* cudaStream_t as void*; NULL = legacy default stream. */
int smc_rhs_set_stream(smc_rhs* op, void* stream);
int smc_rhs_destroy(smc_rhs* op);

/* solve_backward_euler — core/src/stiff.cpp:34-76: w = c + beta f(t, w) by
 * Newton from guess (n = the rhs dimension).  With report == NULL a
 * non-converged solve returns SMC_EINTEGRATION (the reference throws
 * IntegrationError); with a report the caller inspects report->converged. */
int smc_solve_backward_euler(smc_rhs* f, double t, double beta, const double* c,
                             const double* guess, double* w, int where, const smc_stiff* opts,
                             smc_newton_report* report);

/* integrate_stiff — core/src/stiff.cpp:115-188: u' = f(t, u) from t0 to t1 by
 * adaptive backward Euler / variable-step BDF2 with step doubling, every
 * implicit stage through the device Newton (block structure from opts).
 * SMC_EINVAL for t1 < t0 or bad tolerances, SMC_EINTEGRATION when the step
 * size collapses.  accepted / rejected (may be NULL) count the steps. */
int smc_integrate_stiff(smc_rhs* f, const double* u0, double t0, double t1, double* u_out,
                        int where, const smc_stiff* opts, int* accepted, int* rejected);

/* ------------------------------------------------------- quadrature */
/* gauss_lobatto / clenshaw_curtis — core/src/quadrature.cpp:101-132 */
int smc_nodes(int family, int n, double* t);
/* integration_matrices — core/src/quadrature.cpp:134-158; q, s: (n-1) x n */
int smc_integration_matrices(int family, int n, double* q, double* s);
/* build_hierarchy(coarse, TypeB{inner}) (repeats 1), TypeC{inner, repeats}
 * (repeats > 1) or TypeA{inner} (repeats 0: inner is the fine set and must
 * contain every coarse node) — core/src/quadrature.cpp:178-248.  *m2p1
 * receives the fine node count; arrays may be NULL (query), else sized for
 * m2p1 (1 + (nc-1)*repeats*(ni-1) for TypeB/C, ni for TypeA). */
int smc_build_hierarchy(int coarse_family, int coarse_nodes, int inner_family, int inner_nodes,
                        int repeats, int* m2p1, double* fine, double* q21, double* s21,
                        double* q22, double* s22, int* fine_of_coarse, int* p_map);

/* ---------------------------------------------------------- steppers */
/* SdcStepper(NodeSet, StepControls) — core/include/nsdc/sdc.hpp:45-69. */
int smc_sdc_create(int family, int num_nodes, int iterations, double residual_ratio_cutoff,
                   int reuse_first_eval, smc_sdc** out);
/* SdcStepper::step — core/src/sdc.cpp:38-96.  f0 / f_end may be NULL. */
int smc_sdc_step(smc_sdc* s, smc_rhs* f, const double* u0, double t_n, double dt,
                 const double* f0, double* u_out, double* f_end, int where, smc_diag* diag);
/* integrate_sdc — core/src/sdc.cpp:105-127 (state stays on the device). */
int smc_sdc_integrate(smc_sdc* s, smc_rhs* f, const double* u0, double t0, double t1,
                      int nsteps, double* u_out, int where, smc_diag* diag);
/* Cross-rank max of the per-sweep residual (multi-GPU; identity if unset). */
int smc_sdc_set_reducer(smc_sdc* s, smc_reduce_fn fn, void* ctx);
int smc_sdc_destroy(smc_sdc* s);

/* MrsdcStepper(MultirateHierarchy, StepControls) with the hierarchy
 * build_hierarchy(coarse, TypeA/TypeB/TypeC{inner}) (repeats as in
 * smc_build_hierarchy) — core/include/nsdc/mrsdc.hpp:51-82. */
int smc_mrsdc_create(int coarse_family, int coarse_nodes, int inner_family, int inner_nodes,
                     int repeats, int iterations, double residual_ratio_cutoff,
                     int reuse_first_eval, smc_mrsdc** out);
/* MrsdcStepper::step_mode1 — core/src/mrsdc.cpp:84-135. */
int smc_mrsdc_step_mode1(smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0, double t_n,
                         double dt, const double* f0_1, const double* f0_2, double* u_out,
                         double* f1_end, double* f2_end, int where, smc_diag* diag);
/* integrate_mrsdc, mode 1 — core/src/mrsdc.cpp:227-259. */
int smc_mrsdc_integrate_mode1(smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0,
                              double t0, double t1, int nsteps, double* u_out, int where,
                              smc_diag* diag);
/* StiffOptions of mode 2 (MrsdcStepper(h, controls, stiff), mrsdc.hpp:51). */
int smc_mrsdc_set_stiff(smc_mrsdc* m, const smc_stiff* opts);
/* MrsdcStepper::step_mode2 — core/src/mrsdc.cpp:137-206: f1 implicit on the
 * coarse nodes, one backward-Euler-form Newton solve per coarse interval.
 * Newton failure returns SMC_EINTEGRATION naming the coarse node and sweep. */
int smc_mrsdc_step_mode2(smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0, double t_n,
                         double dt, const double* f0_1, const double* f0_2, double* u_out,
                         double* f1_end, double* f2_end, int where, smc_diag* diag);
/* integrate_mrsdc with rhs.f1_stiffness == Implicit — core/src/mrsdc.cpp:227-259. */
int smc_mrsdc_integrate_mode2(smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0,
                              double t0, double t1, int nsteps, double* u_out, int where,
                              smc_diag* diag);
int smc_mrsdc_set_reducer(smc_mrsdc* m, smc_reduce_fn fn, void* ctx);
int smc_mrsdc_destroy(smc_mrsdc* m);

#ifdef __cplusplus
}
#endif
#endif /* SMC_B200_H */
