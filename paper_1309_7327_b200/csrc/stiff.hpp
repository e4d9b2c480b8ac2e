// Device backward-Euler Newton: solve_backward_euler (proj/core/src/stiff.cpp:34-76,
// fd_jacobian :16-30, lu_factor / lu_solve proj/core/src/matrix.cpp:9-51) on
// device-resident state, for MRSDC mode 2 (proj/core/src/mrsdc.cpp:137-206).
//
// The reference forms a dense dim x dim finite-difference Jacobian (dim RHS
// evaluations per Newton step) and a dense LU — hopeless for a PDE state.
// Here f may declare a block structure: it couples only the `block`
// components of one block (the 14 conserved variables of one cell for the
// chemistry term).  Then one RHS evaluation with column j of EVERY block
// perturbed yields column j of every block's Jacobian (block evaluations per
// Newton step instead of dim), and the LU is batched, one block per thread.
// For a block-local f this is the dense computation bit for bit: the
// off-block entries are exact zeros, so the dense elimination and
// substitution reduce to the per-block ones (pinned in test_oracle_mode2.py).
// block = 0 means dense (one block of dim), the reference's own case.
#pragma once

#include "ops.hpp"

namespace smc {

// StiffOptions (proj/core/include/nsdc/stiff.hpp:10-20) + block structure.
struct StiffOpts {
  double rtol = 1e-8;
  double atol = 1e-10;
  int max_newton_iters = 16;
  long long block = 0;   // 0: dense
  int interleaved = 0;   // component j of block b at j*nb + b (else b*block + j)
  double initial_step_fraction = 1e-3;  // integrate_stiff's first step / span
};

// NewtonReport (stiff.hpp:22-27)
struct NewtonReport {
  int iterations = 0;
  double final_residual = 0.0;
  bool converged = false;
  int f_evals = 0;
};

class DeviceNewton {
 public:
  DeviceNewton();
  ~DeviceNewton();
  DeviceNewton(const DeviceNewton&) = delete;
  DeviceNewton& operator=(const DeviceNewton&) = delete;
  // w = c + beta f(t, w) from guess; device pointers of f.dim() doubles,
  // stream-ordered on f.stream().  Never throws for non-convergence: the
  // caller inspects rep.converged (stiff.cpp:71-75 with a report).
  void solve(RhsOp& f, double t, double beta, const double* c, const double* guess, double* w,
             const StiffOpts& o, NewtonReport& rep);
  // Multi-rank f (a slab of a decomposed box): the residual and solution
  // norms and the singular flag are reduced (max) over ranks, so every rank
  // takes the same number of Newton steps and calls f equally often.
  void set_reducer(Reducer r) { reduce_ = std::move(r); }

 private:
  void ensure(long long dim, long long block);
  long long dim_ = -1, block_ = -1;
  DevBuf fw_, fp_, wp_, delta_, jac_, h_, slots_;
  int* piv_ = nullptr;
  long long piv_n_ = 0;
  double* host_slots_ = nullptr;  // pinned readback
  Reducer reduce_;
};

// integrate_stiff (proj/core/src/stiff.cpp:80-188): adaptive backward Euler,
// then variable-step BDF2, error-controlled by step doubling, every implicit
// stage through DeviceNewton (so a block-local f gets the batched solver).
// Device pointers of f.dim() doubles; the step control runs on the host and
// reads two norms per attempted step.  Throws InvalidArgument for t1 < t0 or
// bad tolerances and IntegrationFailure when the step size collapses.
struct StiffStats {
  int accepted = 0, rejected = 0;
};
// With a reducer (multi-rank f) the error norms are reduced over ranks, so
// every rank accepts and rejects the same steps.
void integrate_stiff(RhsOp& f, const double* u0, double t0, double t1, double* u_out,
                     const StiffOpts& o, StiffStats* stats = nullptr,
                     const Reducer& reduce = Reducer());

}  // namespace smc
