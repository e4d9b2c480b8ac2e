// Study harness parity: the reference's study module (nsdc::parse_study_config
// / run_study / to_csv / parse_csv, proj/core/src/study.cpp, compiled from
// the reference sources by tests/cpp/Makefile) against nsdc_b200/study.hpp,
// which runs the same studies on the GPU operator and the device steppers.
// Rows must agree to rounding (the error values are differences of the same
// states, computed on two different machines), console output of the cost
// model and every config error message must be identical, and the CSV
// writer / reader must be the same text.  Exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "nsdc/errors.hpp"
#include "nsdc/study.hpp"
#include "nsdc_b200/study.hpp"

namespace B = nsdc_b200;

static int failures = 0;
static void check(bool ok, const std::string& what, double v = 0.0) {
  std::printf("%s  %s  %.3e\n", ok ? "PASS" : "FAIL", what.c_str(), v);
  if (!ok) ++failures;
}

template <class F>
static std::string captured(F&& f) {
  std::ostringstream buf;
  auto* old = std::cout.rdbuf(buf.rdbuf());
  try {
    f();
  } catch (...) {
    std::cout.rdbuf(old);
    throw;
  }
  std::cout.rdbuf(old);
  return buf.str();
}

static void compare_study(const std::string& name, const std::string& json, double floor) {
  std::vector<nsdc::ConvergenceRow> r;
  std::vector<B::ConvergenceRow> b;
  captured([&] { r = nsdc::run_study(nsdc::parse_study_config(json)); });
  captured([&] { b = B::run_study(B::parse_study_config(json)); });
  bool ok = r.size() == b.size();
  double worst = 0.0;
  for (std::size_t i = 0; ok && i < r.size(); ++i) {
    ok = ok && r[i].resolution == b[i].resolution && r[i].dt == b[i].dt;
    for (auto [x, y] : {std::pair{r[i].linf, b[i].linf}, std::pair{r[i].l2, b[i].l2}}) {
      const double d = std::fabs(x - y);
      worst = std::max(worst, d / std::max(std::fabs(x), floor));
      ok = ok && d <= floor + 1e-6 * std::fabs(x);
    }
    ok = ok && r[i].linf_rate.has_value() == b[i].linf_rate.has_value();
    if (r[i].linf_rate && r[i].linf > 1e3 * floor)
      ok = ok && std::fabs(*r[i].linf_rate - *b[i].linf_rate) <= 1e-3;
  }
  check(ok, "run_study " + name + " (" + std::to_string(r.size()) + " rows)", worst);
}

static void compare_error(const std::string& json, bool prefix_only = false) {
  std::string er, eb;
  try {
    nsdc::parse_study_config(json);
  } catch (const nsdc::ConfigError& e) {
    er = e.what();
  }
  try {
    B::parse_study_config(json);
  } catch (const B::ConfigError& e) {
    eb = e.what();
  }
  const bool ok = !er.empty() && (prefix_only ? eb.rfind("invalid JSON", 0) == 0 &&
                                                    er.rfind("invalid JSON", 0) == 0
                                              : er == eb);
  check(ok, "ConfigError '" + er.substr(0, 60) + "' vs '" + eb.substr(0, 60) + "'");
}

int main() {
  // convergence studies (the acceptance tables' shapes, short horizons)
  compare_study("T1 SMC appendix dt", R"({"problem": "T1", "grids": [16, 32, 64],
      "t_final": 0.1, "residual_cutoff": 0.0})", 1e-13);
  compare_study("T1 NARROW6 fixed dt", R"({"problem": "T1", "stencil": "NARROW6",
      "grids": [16, 32], "t_final": 0.05, "dt_rule": "fixed", "dt": 0.002})", 1e-13);
  compare_study("T1 WIDE halving list", R"({"problem": "T1", "stencil": "WIDE",
      "grids": [16, 32], "t_final": 0.02, "dt_rule": "halving_list", "dt_list": [0.004, 0.002]})",
                1e-13);
  compare_study("T2 OPTIMAL highres reference", R"({"problem": "T2", "stencil": "OPTIMAL",
      "grids": [16, 32], "reference": "highres", "reference_n": 64, "t_final": 0.02,
      "residual_cutoff": 0.0})", 1e-13);
  compare_study("T1 m47/m48 override, clenshaw_curtis", R"({"problem": "T1", "grids": [16, 32],
      "stencil_m47": 0.08, "stencil_m48": -0.02, "node_family": "clenshaw_curtis",
      "num_nodes": 4, "t_final": 0.05})", 1e-13);
  compare_study("SdcOrderODE", R"({"problem": "SdcOrderODE", "grids": [2, 4, 8, 16],
      "lambda1": -1.0, "t_final": 1.0, "residual_cutoff": 0.0})", 1e-15);
  compare_study("MrsdcMode1ODE type_b", R"({"problem": "MrsdcMode1ODE", "grids": [2, 4, 8],
      "hierarchy": "type_b", "fine_nodes": 5, "residual_cutoff": 0.0})", 1e-15);
  compare_study("MrsdcMode1ODE type_a", R"({"problem": "MrsdcMode1ODE", "grids": [2, 4, 8],
      "hierarchy": "type_a", "fine_nodes": 5, "residual_cutoff": 0.0})", 1e-15);
  compare_study("MrsdcMode1ODE type_c", R"({"problem": "MrsdcMode1ODE", "grids": [2, 4],
      "hierarchy": "type_c", "fine_nodes": 3, "repeats": 2, "num_nodes": 5})", 1e-15);
  compare_study("MrsdcMode2ODE", R"({"problem": "MrsdcMode2ODE", "grids": [1, 2, 4],
      "hierarchy": "type_b", "fine_nodes": 5, "iterations": 8, "t_final": 0.1,
      "stiffness": 10000.0, "residual_cutoff": 0.0})", 1e-13);

  // cost model console line (costmodel.hpp; study.cpp:416-423)
  {
    const char* cm = R"({"problem": "CostModel", "N": 20, "flops": 1.0e12, "bandwidth": 2.0e11})";
    const std::string a = captured([&] { nsdc::run_study(nsdc::parse_study_config(cm)); });
    const std::string b = captured([&] { B::run_study(B::parse_study_config(cm)); });
    check(a == b && !a.empty(), "CostModel console line identical");
  }

  // CSV writer / reader (study.cpp:226-272)
  {
    auto r = nsdc::run_study(nsdc::parse_study_config(
        R"({"problem": "SdcOrderODE", "grids": [2, 4], "residual_cutoff": 0.0})"));
    std::vector<B::ConvergenceRow> b;
    for (const auto& x : r) b.push_back({x.resolution, x.dt, x.linf, x.linf_rate, x.l2, x.l2_rate});
    const std::string ca = nsdc::to_csv(r), cb = B::to_csv(b);
    check(ca == cb, "to_csv identical text");
    const auto back = B::parse_csv(cb);
    bool same = back.size() == r.size();
    for (std::size_t i = 0; same && i < back.size(); ++i)
      same = B::to_csv({back[i]}) == nsdc::to_csv({nsdc::parse_csv(ca)[i]});
    check(same, "parse_csv round trip");
  }

  // config errors: same messages, same validation order
  for (const char* bad : {
           R"({"grids": [8]})",
           R"({"problem": "T3", "grids": [8]})",
           R"({"problem": "T1", "grids": [8], "bogus": 1})",
           R"({"problem": "T1"})",
           R"({"problem": "T1", "grids": [16, 8]})",
           R"({"problem": "T1", "grids": [8, 1.5]})",
           R"({"problem": "T1", "grids": "8"})",
           R"({"problem": "T1", "grids": [8], "stencil": "smc"})",
           R"({"problem": "T1", "grids": [8], "stencil": "NARROW6", "stencil_m47": 0.1})",
           R"({"problem": "T1", "grids": [8], "stencil_m36": 0.1})",
           R"({"problem": "T1", "grids": [8], "node_family": "legendre"})",
           R"({"problem": "T1", "grids": [8], "num_nodes": 3.5})",
           R"({"problem": "T1", "grids": [8], "hierarchy": "type_d"})",
           R"({"problem": "T1", "grids": [8], "dt_rule": "cfl"})",
           R"({"problem": "T1", "grids": [8], "dt_rule": "fixed"})",
           R"({"problem": "T1", "grids": [8, 16], "dt_rule": "halving_list", "dt_list": [0.1]})",
           R"({"problem": "T1", "grids": [8], "dt_list": [0.1, "x"]})",
           R"({"problem": "T1", "grids": [8], "reference": "other"})",
           R"({"problem": "T1", "grids": [24], "reference": "highres", "reference_n": 64})",
           R"({"problem": "T1", "grids": [8], "t_final": "1"})",
           R"({"problem": "T1", "grids": [8], "output": 3})",
           R"([1, 2])",
       })
    compare_error(bad);
  compare_error(R"({"problem": "T1", "grids": [8])", true);
  compare_error(R"(not json)", true);

  // run-time errors of the multirate problems
  for (const char* bad : {
           R"({"problem": "MrsdcMode1ODE", "grids": [2]})",
           R"({"problem": "MrsdcMode1ODE", "grids": [2], "hierarchy": "type_b"})",
           R"({"problem": "SdcOrderODE", "grids": [0]})",
       }) {
    std::string er, eb;
    try {
      captured([&] { nsdc::run_study(nsdc::parse_study_config(bad)); });
    } catch (const nsdc::ConfigError& e) {
      er = e.what();
    }
    try {
      captured([&] { B::run_study(B::parse_study_config(bad)); });
    } catch (const B::ConfigError& e) {
      eb = e.what();
    }
    check(!er.empty() && er == eb, "run_study error '" + er + "'");
  }
  std::printf("%d failures\n", failures);
  return failures;
}
