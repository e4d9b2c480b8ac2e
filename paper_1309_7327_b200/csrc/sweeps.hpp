// Device-resident SDC / MRSDC (modes 1 and 2) sweeps, host-orchestrated.
// Reference: SdcStepper::step / integrate_sdc (proj/core/src/sdc.cpp:38-127),
// MrsdcStepper::step_mode1 / integrate_mrsdc (proj/core/src/mrsdc.cpp:43-135,
// :227-259), MrsdcStepper::step_mode2 (mrsdc.cpp:137-206) with the device
// Newton of stiff.hpp.  Node values never leave HBM; per sweep the host only reads the
// residual (or, with early stop disabled, once per step).
#pragma once

#include <functional>
#include <vector>

#include "ops.hpp"
#include "quadrature.hpp"
#include "stiff.hpp"

namespace smc {

struct SweepDiag {
  std::vector<double> residuals;
  int sweeps = 0;
  int fresh_evals = 0;  // SDC
  int f1_evals = 0, f2_evals = 0;  // MRSDC
  int implicit_solves = 0, newton_f1_evals = 0;  // MRSDC mode 2 (mrsdc.hpp:30-38)
  bool early_stop = false;
  bool nonfinite = false;  // a non-finite residual was seen
  void add(const SweepDiag& o);
};

class DeviceSdc {
 public:
  DeviceSdc(Nodes nodes, int iterations, double cutoff, bool reuse_first);
  void step(RhsOp& f, const double* u0, double t_n, double dt, const double* f0, double* u_out,
            double* f_end, SweepDiag& d);
  void integrate(RhsOp& f, const double* u0, double t0, double t1, int nsteps, double* u_out,
                 SweepDiag& d);
  void set_reducer(Reducer r) { reduce_ = std::move(r); }
  const Nodes& nodes() const { return nodes_; }
  const SweepTables& tables() const { return tab_; }

 private:
  void ensure(long long dim);
  void run(RhsOp& f, double t_n, double dt, bool have_f0, SweepDiag& d);
  Nodes nodes_;
  SweepTables tab_;
  int iterations_;
  double cutoff_;
  bool reuse_first_;
  long long dim_ = -1;
  std::vector<DevBuf> U_, FA_, FB_;
  DevBuf F0_, res_;
  std::vector<double*> u_, fa_, fb_;
  double* f0_ = nullptr;
  double* f_last_ = nullptr;
  Reducer reduce_;
};

class DeviceMrsdc {
 public:
  DeviceMrsdc(Hierarchy h, int iterations, double cutoff, bool reuse_first);
  void step_mode1(RhsOp& f1, RhsOp& f2, const double* u0, double t_n, double dt,
                  const double* f01, const double* f02, double* u_out, double* f1_end,
                  double* f2_end, SweepDiag& d);
  void integrate_mode1(RhsOp& f1, RhsOp& f2, const double* u0, double t0, double t1, int nsteps,
                       double* u_out, SweepDiag& d);
  // f1 implicit: per coarse interval one backward-Euler-form Newton solve
  // (mrsdc.cpp:137-206); throws IntegrationFailure naming the coarse node.
  void step_mode2(RhsOp& f1, RhsOp& f2, const double* u0, double t_n, double dt,
                  const double* f01, const double* f02, double* u_out, double* f1_end,
                  double* f2_end, SweepDiag& d);
  void integrate_mode2(RhsOp& f1, RhsOp& f2, const double* u0, double t0, double t1, int nsteps,
                       double* u_out, SweepDiag& d);
  void set_reducer(Reducer r) {
    reduce_ = r;
    newton_.set_reducer(std::move(r));
  }
  void set_stiff(const StiffOpts& o) { stiff_ = o; }
  const StiffOpts& stiff() const { return stiff_; }
  const Hierarchy& hierarchy() const { return h_; }

 private:
  struct SweepResiduals;  // node integrals + per-sweep residuals (sweeps.cu)
  void ensure(long long dim);
  void run(RhsOp& f1, RhsOp& f2, double t_n, double dt, bool have_f01, bool have_f02,
           SweepDiag& d);
  void run2(RhsOp& f1, RhsOp& f2, double t_n, double dt, bool have_f01, bool have_f02,
            SweepDiag& d);
  void integrate(int mode, RhsOp& f1, RhsOp& f2, const double* u0, double t0, double t1,
                 int nsteps, double* u_out, SweepDiag& d);
  Hierarchy h_;
  int iterations_;
  double cutoff_;
  bool reuse_first_;
  long long dim_ = -1;
  std::vector<DevBuf> U_, F1A_, F1B_, F2A_, F2B_, SO_;
  DevBuf F10_, F20_, res_;
  std::vector<double*> u_, f1a_, f1b_, f2a_, f2b_, so_;
  double* f10_ = nullptr;
  double* f20_ = nullptr;
  double* f1_last_ = nullptr;
  double* f2_last_ = nullptr;
  Reducer reduce_;
  StiffOpts stiff_;
  DeviceNewton newton_;
  DevBuf C_, W_;  // mode 2: Newton right-hand side and solution
};

// Pointwise sweep kernels (exposed for tests / the NS path).
constexpr int kMaxTerms = 24;
constexpr int kMaxRows = 16;
// next = cur + sum_d c_d (a_d - b_d) + (pre ? pre : dt * sum_j w_j g_j)
void launch_sweep_update(double* next, const double* cur, int nd, const double* const* da,
                         const double* const* db, const double* dc, int ng,
                         const double* const* g, const double* w, double dt, const double* pre,
                         long long n, cudaStream_t st);
// rows r: out_r = dt * sum_j w[r][j] g_j
void launch_integrals(int rows, double* const* out, int ng, const double* const* g,
                      const double* w /*rows x ng*/, double dt, long long n, cudaStream_t st);
// c = (u + sum_q so_q) - dt1 * old  (mrsdc.cpp:165-169)
void launch_be_rhs(double* c, const double* u, int nso, const double* const* so, const double* old,
                   double dt1, long long n, cudaStream_t st);
// *slot = max_i |u0 + dt sum_j q_j g_j - um|  (slot must be zeroed; NaN -> +inf)
void launch_residual(const double* u0, const double* um, int ng, const double* const* g,
                     const double* q, double dt, long long n, double* slot, cudaStream_t st);
// launch_integrals for the next sweep fused with launch_residual of the last
// one (they read the same node values); two launches where the fused
// fixed-shape kernel does not apply.
void launch_integrals_residual(int rows, double* const* out, int ng, const double* const* g,
                               const double* w, double dt, const double* u0, const double* um,
                               const double* q, long long n, double* slot, cudaStream_t st);

}  // namespace smc
