// Drop-in demonstration + parity: the unmodified reference library (nsdc,
// built from /root/reference by oracle/Makefile) and the B200 library (via
// the C++ mirror include/nsdc_b200/nsdc_b200.hpp) in one binary.
//  * the reference's own integrate_sdc drives the GPU heat RHS (as_rhs());
//  * the device-resident nsdc_b200 steppers drive the reference's RHS and the
//    GPU RHS;
//  * every result is compared with the all-reference computation.
// Exit code = number of failed checks.  Built by tests/cpp/Makefile (needs
// the reference headers, so only where /root/reference exists); run by
// tests/test_gpu_cpp_shim.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "nsdc/mrsdc.hpp"
#include "nsdc/pde.hpp"
#include "nsdc/quadrature.hpp"
#include "nsdc/sdc.hpp"
#include "nsdc/stencil.hpp"
#include "nsdc_b200/nsdc_b200.hpp"

namespace B = nsdc_b200;

static int failures = 0;
static void check(bool ok, const std::string& what, double v = 0.0) {
  std::printf("%s  %s  %.3e\n", ok ? "PASS" : "FAIL", what.c_str(), v);
  if (!ok) ++failures;
}
static double relerr(const std::vector<double>& a, const std::vector<double>& b) {
  double e = 0.0, m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    e = std::max(e, std::fabs(a[i] - b[i]));
    m = std::max(m, std::fabs(b[i]));
  }
  return e / (m > 0 ? m : 1.0);
}

// the reference problems restated through the mirror's HeatProblem type
static B::HeatProblem mirror(const nsdc::HeatProblem& p) {
  B::HeatProblem q;
  q.a = p.a, q.b = p.b, q.g = p.g, q.g_space = p.g_space, q.g_time = p.g_time, q.u0 = p.u0;
  q.exact = p.exact, q.epsilon = p.epsilon;
  return q;
}

int main() {
  // coupling matrix (stencil.cpp:117-132)
  {
    auto r = nsdc::build_narrow(8, {nsdc::kSmcM47, nsdc::kSmcM48});
    auto g = B::build_narrow(8, {B::kSmcM47, B::kSmcM48});
    bool same = r.s == g.s;
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) same = same && r.m[i][j] == g.m[i][j];
    check(same, "build_narrow bitwise");
  }
  for (int pid = 1; pid <= 2; ++pid) {
    const nsdc::HeatProblem p = pid == 1 ? nsdc::make_t1() : nsdc::make_t2();
    const int n = 32;
    const nsdc::Grid2D g{n, n};
    nsdc::HeatOperator ref(p, g, nsdc::stencil_preset("SMC"));
    B::HeatOperator gpu(mirror(p), B::Grid2D{n, n}, B::stencil_preset("SMC"));
    const nsdc::Field2D u = nsdc::eval_on_grid(g, p.u0);
    nsdc::Field2D ro(n, n);
    ref.rhs(0.4, u, ro);
    B::Field2D gu(n, n), go;
    gu.v = u.v;
    gpu.rhs(0.4, gu, go);
    check(relerr(go.v, ro.v) <= 1e-12, "T" + std::to_string(pid) + " HeatOperator::rhs",
          relerr(go.v, ro.v));

    const double dt = nsdc::appendix_dt(g, p);
    nsdc::StepControls c;
    c.residual_ratio_cutoff = 0.0;
    B::StepControls bc;
    bc.residual_ratio_cutoff = 0.0;
    auto [u_ref, d_ref] = nsdc::integrate_sdc(ref.as_rhs(), u.v, 0.0, 10 * dt, 10,
                                              nsdc::gauss_lobatto(3), c);
    // 1) the reference integrator driving the GPU RHS (drop-in of the Rhs)
    auto [u_a, d_a] = nsdc::integrate_sdc(gpu.as_rhs(), u.v, 0.0, 10 * dt, 10,
                                          nsdc::gauss_lobatto(3), c);
    check(relerr(u_a, u_ref) <= 1e-9 && d_a.fresh_evals == d_ref.fresh_evals,
          "T" + std::to_string(pid) + " nsdc::integrate_sdc(gpu.as_rhs()) 10 steps",
          relerr(u_a, u_ref));
    // 2) device-resident stepper + GPU RHS
    auto [u_b, d_b] = B::integrate_sdc(gpu, u.v, 0.0, 10 * dt, 10, B::gauss_lobatto(3), bc);
    check(relerr(u_b, u_ref) <= 1e-9 && d_b.fresh_evals == d_ref.fresh_evals &&
              d_b.sweeps == d_ref.sweeps,
          "T" + std::to_string(pid) + " nsdc_b200::integrate_sdc(gpu) 10 steps",
          relerr(u_b, u_ref));
    // 3) device-resident stepper + the reference's own RHS (std::function)
    auto [u_c, d_c] = B::integrate_sdc(ref.as_rhs(), u.v, 0.0, 10 * dt, 10,
                                       B::gauss_lobatto(3), bc);
    check(relerr(u_c, u_ref) <= 1e-12, "T" + std::to_string(pid) +
                                           " nsdc_b200::integrate_sdc(ref.as_rhs())",
          relerr(u_c, u_ref));
  }
  // MRSDC mode 1 on the reference's split linear problem (pde.cpp:332-345)
  {
    auto prob = nsdc::make_split_linear(-1.0, -10.0);
    auto h = nsdc::build_hierarchy(nsdc::gauss_lobatto(3), nsdc::TypeB{nsdc::gauss_lobatto(5)});
    nsdc::StepControls c;
    c.residual_ratio_cutoff = 0.0;
    auto [u_ref, d_ref] = nsdc::integrate_mrsdc(prob.rhs, {1.0}, 0.0, 1.0, 8, h, c);
    B::SplitRHS s{prob.rhs.f1, prob.rhs.f2};
    B::StepControls bc;
    bc.residual_ratio_cutoff = 0.0;
    auto [u_b, d_b] = B::integrate_mrsdc(s, {1.0}, 0.0, 1.0, 8, B::gauss_lobatto(3),
                                         B::TypeB{B::gauss_lobatto(5)}, bc);
    check(std::fabs(u_b[0] - u_ref[0]) <= 1e-14 && d_b.f1_evals == d_ref.f1_evals &&
              d_b.f2_evals == d_ref.f2_evals,
          "integrate_mrsdc mode 1 split linear", std::fabs(u_b[0] - u_ref[0]));
  }
  // error behaviour mirrors the reference (pde_test.cpp:243-263)
  {
    bool threw = false;
    try {
      B::HeatOperator bad(mirror(nsdc::make_t1()), B::Grid2D{8, 20}, B::stencil_preset("SMC"));
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    check(threw, "grid too small -> std::invalid_argument");
    threw = false;
    try {
      B::stencil_preset("smc");
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    check(threw, "unknown preset -> std::invalid_argument");
  }
  std::printf("%d failures\n", failures);
  return failures;
}
