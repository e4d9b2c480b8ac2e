#include <algorithm>
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
#include "nsdc/stiff.hpp"
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
  // MRSDC mode 2 (f1 implicit, mrsdc.cpp:137-206) on the reference's stiff
  // Prothero-Robinson split (mrsdc_test.cpp:23-35, acceptance_test.cpp:357-371),
  // reference vs the mirror's drop-in signatures
  {
    const double sigma = 1.0e4;
    nsdc::SplitRHS r;
    r.f1 = [sigma](double t, const nsdc::Field& u, nsdc::Field& out) {
      out.resize(u.size());
      for (std::size_t i = 0; i < u.size(); ++i) out[i] = -sigma * (u[i] - std::cos(t));
    };
    r.f2 = [](double t, const nsdc::Field& u, nsdc::Field& out) {
      out.assign(u.size(), -std::sin(t));
    };
    r.f1_stiffness = nsdc::SplitRHS::Stiffness::Implicit;
    auto h = nsdc::build_hierarchy(nsdc::gauss_lobatto(3), nsdc::TypeB{nsdc::gauss_lobatto(5)});
    nsdc::StepControls c;
    c.num_iterations = 6;
    c.residual_ratio_cutoff = 0.0;
    nsdc::StiffOptions so;
    so.rtol = 1e-12;
    so.atol = 1e-13;
    auto [u_ref, d_ref] = nsdc::integrate_mrsdc(r, {1.0}, 0.0, 0.2, 10, h, c, so);

    B::SplitRHS s{r.f1, r.f2, B::SplitRHS::Stiffness::Implicit};
    auto bh = B::build_hierarchy(B::gauss_lobatto(3), B::TypeB{B::gauss_lobatto(5)});
    B::StepControls bc;
    bc.num_iterations = 6;
    bc.residual_ratio_cutoff = 0.0;
    B::StiffOptions bso;
    bso.rtol = 1e-12;
    bso.atol = 1e-13;
    auto [u_b, d_b] = B::integrate_mrsdc(s, {1.0}, 0.0, 0.2, 10, bh, bc, bso);
    check(std::fabs(u_b[0] - u_ref[0]) <= 1e-10 * std::fabs(u_ref[0]) &&
              d_b.implicit_solves == d_ref.implicit_solves && d_b.f1_evals == d_ref.f1_evals &&
              d_b.f2_evals == d_ref.f2_evals,
          "integrate_mrsdc mode 2 stiff oscillator", std::fabs(u_b[0] - u_ref[0]));
    // the mirror's tables come from an independent construction
    // (Golub-Welsch nodes, Chebyshev-moment weights): equal to rounding
    bool same_tables = bh.fine.nodes.size() == h.fine.nodes.size() &&
                       bh.fine_of_coarse == h.fine_of_coarse && bh.p_map == h.p_map;
    double table_diff = 0.0;
    for (std::size_t q = 0; same_tables && q < h.fine.nodes.size(); ++q)
      table_diff = std::max(table_diff, std::fabs(bh.fine.nodes[q] - h.fine.nodes[q]));
    for (int q = 0; same_tables && q < h.s22.rows; ++q)
      for (int j = 0; j < h.s22.cols; ++j)
        table_diff = std::max(table_diff, std::fabs(bh.s22(q, j) - h.s22(q, j)));
    check(same_tables && table_diff <= 1e-15, "build_hierarchy tables to rounding", table_diff);

    // Newton failure names the coarse node (mrsdc_test.cpp:215-228)
    B::SplitRHS bad{[](double, const B::Field& u, B::Field& out) { out = {u[0] * u[0]}; },
                    [](double, const B::Field& u, B::Field& out) { out.assign(u.size(), 0.0); },
                    B::SplitRHS::Stiffness::Implicit};
    std::string msg;
    try {
      B::mrsdc_step_mode2(bad, {5.0}, 0.0, 1.0,
                          B::build_hierarchy(B::gauss_lobatto(3), B::TypeB{B::gauss_lobatto(2)}),
                          bc, B::StiffOptions{});
    } catch (const B::IntegrationError& e) {
      msg = e.what();
    }
    check(msg.find("coarse node 1") != std::string::npos, "mode 2 Newton failure -> IntegrationError");

    // solve_backward_euler (stiff.cpp:34-76) with a report
    nsdc::NewtonReport rr;
    nsdc::Field wr = nsdc::solve_backward_euler(r.f1, 0.1, 0.05, {0.5}, {0.5}, so, &rr);
    B::NewtonReport br;
    B::Field wb = B::solve_backward_euler(s.f1, 0.1, 0.05, {0.5}, {0.5}, bso, &br);
    check(wb[0] == wr[0] && br.iterations == rr.iterations && br.f_evals == rr.f_evals &&
              br.converged == rr.converged,
          "solve_backward_euler bitwise", std::fabs(wb[0] - wr[0]));
  }
  // integrate_stiff (stiff.cpp:115-188) on the stiff forced oscillator
  {
    const double sigma = 1.0e4;
    nsdc::Rhs f = [sigma](double t, const nsdc::Field& u, nsdc::Field& out) {
      out.resize(u.size());
      for (std::size_t i = 0; i < u.size(); ++i) out[i] = -sigma * (u[i] - std::cos(t)) - std::sin(t);
    };
    nsdc::StiffOptions so;
    B::StiffOptions bso;
    const nsdc::Field ur = nsdc::integrate_stiff(f, {1.0}, 0.0, 1.0, so);
    const B::Field ub = B::integrate_stiff(f, {1.0}, 0.0, 1.0, bso);
    check(ub[0] == ur[0], "integrate_stiff bitwise", std::fabs(ub[0] - ur[0]));
  }
  // non-periodic lines (the paper's boundary closure; no reference
  // counterpart): away from the ends they are the reference's periodic
  // operators, and a too-short line throws like apply_narrow does
  {
    const int n = 96;
    std::vector<double> a(n), u(n);
    for (int i = 0; i < n; ++i) {
      a[i] = 1.0 + 0.3 * std::sin(0.37 * i);
      u[i] = std::cos(0.21 * i) + 0.1 * std::sin(1.3 * i);
    }
    const double dx = 1.0 / n;
    const auto m = nsdc::build_narrow(8, {nsdc::kSmcM47, nsdc::kSmcM48});
    const auto rp = nsdc::apply_narrow(m, a, u, dx);
    const auto gb = B::apply_narrow_bounded(a, u, dx);
    const auto rd = nsdc::first_derivative8(u, dx);
    const auto gd = B::first_derivative_bounded(u, dx);
    double e = 0.0, sc = 0.0, ed = 0.0, sd = 0.0;
    for (int i = 8; i < n - 8; ++i) {
      e = std::max(e, std::fabs(gb[i] - rp[i])), sc = std::max(sc, std::fabs(rp[i]));
      ed = std::max(ed, std::fabs(gd[i] - rd[i])), sd = std::max(sd, std::fabs(rd[i]));
    }
    check(e <= 1e-12 * sc && ed <= 1e-12 * sd, "bounded lines = periodic operators inside",
          std::max(e / sc, ed / sd));
    bool threw = false;
    try {
      B::apply_narrow_bounded(std::vector<double>(7, 1.0), std::vector<double>(7, 1.0), 0.1);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    check(threw, "bounded line too short -> std::invalid_argument");
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
