// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrappers that expose the UNMODIFIED reference library
// (/root/reference/proj/core, compiled from its own sources by oracle/Makefile
// into oracle/_ref/) to the Python tests, the golden-vector generator and
// bench.py's `--impl reference` / cpu_baseline legs.  Nothing here
// re-implements reference arithmetic: every function forwards to a reference
// symbol, except ref_narrow3d, which composes the reference's own line
// kernels in 3-D exactly the way narrow_rhs_rows<S> composes them in 2-D
// (proj/core/src/pde.cpp:85-129; SURVEY.md §8(c) "oracle3d").
#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "nsdc/field.hpp"
#include "nsdc/mrsdc.hpp"
#include "nsdc/parallel.hpp"
#include "nsdc/pde.hpp"
#include "nsdc/quadrature.hpp"
#include "nsdc/sdc.hpp"
#include "nsdc/stencil.hpp"
#include "nsdc/stiff.hpp"
#include "stencil_kernel.hpp"  // proj/core/src (private kernels, -I on the src dir)

using namespace nsdc;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

StencilChoice choice_from(int kind, const double* params) {
  // kind: 0 = narrow8, 1 = narrow6, 2 = wide8 (StencilChoice::Kind order, stencil.hpp:65-75)
  if (kind == 0) return StencilChoice::narrow8(params[0], params[1]);
  if (kind == 1) return StencilChoice::narrow6(params[0]);
  return StencilChoice::wide8();
}

NodeSet nodes_from(int family, int n) {
  return family == 0 ? gauss_lobatto(n) : clenshaw_curtis(n);
}

// Heat problems addressable from C: 1 = T1, 2 = T2 (pde.cpp:21-50), 3 = the
// x-only problem of pde_test.cpp:17-25 restated as a HeatProblem, 0 = grid
// arrays supplied by the caller (a, b, g0 sampled on the nodes; g_time = 1).
struct ArrayProblem {
  int nx, ny;
  std::vector<double> a, b, g0;
};

HeatProblem make_problem(int id, ArrayProblem* arr) {
  if (id == 1) return make_t1();
  if (id == 2) return make_t2();
  if (id == 3) {
    HeatProblem p;
    p.a = [](double x, double y) { return 1.0 + 0.2 * std::cos(x) * std::cos(y); };
    p.b = [](double x, double) { return 1.0 + 0.3 * std::sin(x); };
    p.u0 = [](double x, double) { return std::sin(x); };
    return p;
  }
  // Node lookup: the operator only ever evaluates coefficients on grid nodes.
  HeatProblem p;
  auto idx = [arr](double x, double y) {
    const Grid2D g{arr->nx, arr->ny};
    int i = static_cast<int>(std::lround(x / g.dx()));
    int j = static_cast<int>(std::lround(y / g.dy()));
    i = ((i % arr->nx) + arr->nx) % arr->nx;
    j = ((j % arr->ny) + arr->ny) % arr->ny;
    return static_cast<std::size_t>(j) * arr->nx + i;
  };
  p.a = [arr, idx](double x, double y) { return arr->a[idx(x, y)]; };
  p.b = [arr, idx](double x, double y) { return arr->b[idx(x, y)]; };
  p.u0 = [](double, double) { return 0.0; };
  if (!arr->g0.empty()) {
    p.g_space = [arr, idx](double x, double y) { return arr->g0[idx(x, y)]; };
    p.g_time = [](double) { return 1.0; };
    p.g = [gs = p.g_space](double, double x, double y) { return gs(x, y); };
  }
  return p;
}

void copy_matrix(const Matrix& m, double* out) {
  if (out) std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
}

typedef void (*rhs_cb)(double t, const double* u, double* out, long long n, void* ctx);

Rhs wrap_cb(rhs_cb cb, void* ctx) {
  return [cb, ctx](double t, const Field& u, Field& out) {
    out.resize(u.size());
    cb(t, u.data(), out.data(), static_cast<long long>(u.size()), ctx);
  };
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_workers(int n) {
  if (n <= 0)
    unsetenv("NSDC_MAX_WORKERS");
  else
    setenv("NSDC_MAX_WORKERS", std::to_string(n).c_str(), 1);
}
int ref_worker_limit() { return worker_limit(); }

// stencil.cpp:117-132
int ref_build_narrow(int order, const double* params, int nparams, double* m64, int* s) {
  return guarded([&] {
    StencilMatrix m = build_narrow(order, std::vector<double>(params, params + nparams));
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) m64[i * 8 + j] = m.m[i][j];
    *s = m.s;
  });
}

// stencil.cpp:134-155
int ref_apply_narrow(int order, const double* params, int nparams, const double* a,
                     const double* u, int n, double dx, double* out) {
  return guarded([&] {
    StencilMatrix m = build_narrow(order, std::vector<double>(params, params + nparams));
    Field r = apply_narrow(m, Field(a, a + n), Field(u, u + n), dx);
    std::memcpy(out, r.data(), sizeof(double) * n);
  });
}

// stencil.cpp:157-176
int ref_first_derivative8(const double* u, int n, double dx, double* out) {
  return guarded([&] {
    Field r = first_derivative8(Field(u, u + n), dx);
    std::memcpy(out, r.data(), sizeof(double) * n);
  });
}
int ref_apply_wide(const double* a, const double* u, int n, double dx, double* out) {
  return guarded([&] {
    Field r = apply_wide(Field(a, a + n), Field(u, u + n), dx);
    std::memcpy(out, r.data(), sizeof(double) * n);
  });
}
double ref_truncation_bound(int order, const double* params, int nparams) {
  return truncation_bound(order, std::vector<double>(params, params + nparams));
}
int ref_optimize_params(int order, double* out) {
  return guarded([&] {
    auto p = optimize_params(order);
    for (std::size_t i = 0; i < p.size(); ++i) out[i] = p[i];
  });
}

// 3-D narrow operator (a U_x)_x + (a U_y)_y + (a U_z)_z on a periodic
// nx*ny*nz box, x fastest: v[(k*ny + j)*nx + i].  Same composition as
// narrow_rhs_rows<S> (pde.cpp:85-129): x interfaces from a periodically
// padded row via narrow_interfaces<S>; y and z interfaces from 2S row
// pointers via narrow_interfaces_rows<S>; out = dHx/dx^2 + dHy/dy^2 +
// dHz/dz^2 in that order.  Planes are distributed with the reference's own
// parallel_for (parallel.cpp:20-36).
int ref_narrow3d(const double* m64, int s, const double* a, const double* u, int nx, int ny,
                 int nz, double dx, double dy, double dz, double* out) {
  return guarded([&] {
    if (s != 4 && s != 3) throw std::invalid_argument("ref_narrow3d: s must be 3 or 4");
    if (nx < 2 * s || ny < 2 * s || nz < 2 * s)
      throw std::invalid_argument("ref_narrow3d: grid too small");
    std::array<std::array<double, 8>, 8> mm{};
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) mm[i][j] = m64[i * 8 + j];
    const double idx2 = 1.0 / (dx * dx), idy2 = 1.0 / (dy * dy), idz2 = 1.0 / (dz * dz);
    const std::size_t plane = static_cast<std::size_t>(nx) * ny;
    auto body = [&](int kb, int ke) {
      const int S = s;
      std::vector<double> ubuf(nx + 2 * S - 1), abuf(nx + 2 * S - 1);
      std::vector<double> hx(nx), hy_prev(nx), hy_cur(nx);
      // z interfaces are carried plane to plane like hy_prev/hy_cur in
      // pde.cpp:110-127, so each interface is computed once per band.
      std::vector<double> hz_prev(plane), hz_cur(plane);
      const double* ru[8];
      const double* ra[8];
      auto rows = [&](int k, int j, int dir, int ih, double* h) {
        // interface ih + 1/2 along dir (1 = y, 2 = z) for the x-line (j, k)
        for (int q = 0; q < 2 * S; ++q) {
          int jj = j, kk = k;
          if (dir == 1)
            jj = ((ih + q - (S - 1)) % ny + ny) % ny;
          else
            kk = ((ih + q - (S - 1)) % nz + nz) % nz;
          const std::size_t off = static_cast<std::size_t>(kk) * plane + static_cast<std::size_t>(jj) * nx;
          ru[q] = u + off;
          ra[q] = a + off;
        }
        if (S == 4)
          detail::narrow_interfaces_rows<4>(ra, ru, nx, mm, h);
        else
          detail::narrow_interfaces_rows<3>(ra, ru, nx, mm, h);
      };
      for (int j = 0; j < ny; ++j)
        rows(0, j, 2, (kb - 1 + nz) % nz, hz_prev.data() + static_cast<std::size_t>(j) * nx);
      for (int k = kb; k < ke; ++k) {
        for (int j = 0; j < ny; ++j) rows(0, j, 2, k, hz_cur.data() + static_cast<std::size_t>(j) * nx);
        rows(k, 0, 1, ny - 1, hy_prev.data());
        for (int j = 0; j < ny; ++j) {
          const std::size_t off = static_cast<std::size_t>(k) * plane + static_cast<std::size_t>(j) * nx;
          double* up = ubuf.data() + (S - 1);
          double* ap = abuf.data() + (S - 1);
          for (int i = 0; i < nx; ++i) {
            up[i] = u[off + i];
            ap[i] = a[off + i];
          }
          for (int i = 1; i <= S - 1; ++i) {
            up[-i] = u[off + nx - i];
            ap[-i] = a[off + nx - i];
          }
          for (int i = 0; i < S; ++i) {
            up[nx + i] = u[off + i];
            ap[nx + i] = a[off + i];
          }
          if (S == 4)
            detail::narrow_interfaces<4>(ap, up, nx, mm, hx.data());
          else
            detail::narrow_interfaces<3>(ap, up, nx, mm, hx.data());
          rows(k, j, 1, j, hy_cur.data());
          const double* zl = hz_prev.data() + static_cast<std::size_t>(j) * nx;
          const double* zh = hz_cur.data() + static_cast<std::size_t>(j) * nx;
          double* o = out + off;
          o[0] = (hx[0] - hx[nx - 1]) * idx2 + (hy_cur[0] - hy_prev[0]) * idy2 +
                 (zh[0] - zl[0]) * idz2;
          for (int i = 1; i < nx; ++i)
            o[i] = (hx[i] - hx[i - 1]) * idx2 + (hy_cur[i] - hy_prev[i]) * idy2 +
                   (zh[i] - zl[i]) * idz2;
          hy_prev.swap(hy_cur);
        }
        hz_prev.swap(hz_cur);
      }
    };
    parallel_for(nz, body);
  });
}

// ---------------------------------------------------------------- heat 2-D
// HeatOperator (pde.cpp:209-274) on problem `id`; a/b/g0 used when id == 0.
int ref_heat2d_rhs(int id, int nx, int ny, int kind, const double* params, const double* a,
                   const double* b, const double* g0, double t, const double* u, double* out) {
  return guarded([&] {
    ArrayProblem arr{nx, ny, {}, {}, {}};
    if (id == 0) {
      const std::size_t n = static_cast<std::size_t>(nx) * ny;
      arr.a.assign(a, a + n);
      arr.b.assign(b, b + n);
      if (g0) arr.g0.assign(g0, g0 + n);
    }
    HeatProblem p = make_problem(id, &arr);
    HeatOperator op(p, Grid2D{nx, ny}, choice_from(kind, params));
    Field2D uu(nx, ny);
    std::memcpy(uu.v.data(), u, sizeof(double) * uu.v.size());
    Field2D oo(nx, ny);
    op.rhs(t, uu, oo);
    std::memcpy(out, oo.v.data(), sizeof(double) * oo.v.size());
  });
}

// Best wall time of HeatOperator::rhs (pde.cpp:266-274) over `reps` calls on
// the problem's own u0 (operator built once; workers from ref_set_workers).
int ref_heat2d_time(int id, int nx, int ny, int kind, const double* params, int reps,
                    double* best_seconds) {
  return guarded([&] {
    ArrayProblem arr{nx, ny, {}, {}, {}};
    HeatProblem p = make_problem(id, &arr);
    const Grid2D g{nx, ny};
    HeatOperator op(p, g, choice_from(kind, params));
    Field2D uu = eval_on_grid(g, p.u0);
    Field2D oo(nx, ny);
    op.rhs(0.1, uu, oo);  // warm-up
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      op.rhs(0.1, uu, oo);
      const std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t0;
      best = std::min(best, dt.count());
    }
    *best_seconds = best;
  });
}

// eval_on_grid of the problem's a, b, g_space, u0 (pde.cpp:52-57)
int ref_heat2d_fields(int id, int nx, int ny, double* a, double* b, double* g0, double* u0) {
  return guarded([&] {
    ArrayProblem arr{nx, ny, {}, {}, {}};
    HeatProblem p = make_problem(id, &arr);
    const Grid2D g{nx, ny};
    auto put = [&](const std::function<double(double, double)>& f, double* dst) {
      if (!dst) return;
      if (!f) {
        std::fill(dst, dst + static_cast<std::size_t>(nx) * ny, 0.0);
        return;
      }
      Field2D v = eval_on_grid(g, f);
      std::memcpy(dst, v.v.data(), sizeof(double) * v.v.size());
    };
    put(p.a, a);
    put(p.b, b);
    put(p.g_space, g0);
    put(p.u0, u0);
  });
}

double ref_appendix_dt(int id, int nx, int ny) {
  ArrayProblem arr{nx, ny, {}, {}, {}};
  return appendix_dt(Grid2D{nx, ny}, make_problem(id, &arr));
}

// integrate_sdc (sdc.cpp:105-127) over the heat operator of problem id.
int ref_heat2d_integrate_sdc(int id, int nx, int ny, int kind, const double* params,
                             const double* u0, double t0, double t1, int nsteps, int family,
                             int num_nodes, int iterations, double cutoff, double* u_out,
                             double* residuals, int max_res, int* sweeps, int* fresh_evals) {
  return guarded([&] {
    ArrayProblem arr{nx, ny, {}, {}, {}};
    HeatProblem p = make_problem(id, &arr);
    HeatOperator op(p, Grid2D{nx, ny}, choice_from(kind, params));
    StepControls c;
    c.num_iterations = iterations;
    c.residual_ratio_cutoff = cutoff;
    const std::size_t n = static_cast<std::size_t>(nx) * ny;
    auto [u, diag] = integrate_sdc(op.as_rhs(), Field(u0, u0 + n), t0, t1, nsteps,
                                   nodes_from(family, num_nodes), c);
    std::memcpy(u_out, u.data(), sizeof(double) * n);
    if (residuals)
      for (int i = 0; i < std::min<int>(max_res, diag.residual_history.size()); ++i)
        residuals[i] = diag.residual_history[i];
    *sweeps = diag.sweeps;
    *fresh_evals = diag.fresh_evals;
  });
}

// Generic integrate_sdc with a C callback RHS.
int ref_integrate_sdc(rhs_cb cb, void* ctx, long long dim, const double* u0, double t0,
                      double t1, int nsteps, int family, int num_nodes, int iterations,
                      double cutoff, int reuse_first, double* u_out, double* residuals,
                      int max_res, int* sweeps, int* fresh_evals, int* early_stop) {
  return guarded([&] {
    StepControls c;
    c.num_iterations = iterations;
    c.residual_ratio_cutoff = cutoff;
    c.reuse_first_eval = reuse_first != 0;
    auto [u, diag] = integrate_sdc(wrap_cb(cb, ctx), Field(u0, u0 + dim), t0, t1, nsteps,
                                   nodes_from(family, num_nodes), c);
    std::memcpy(u_out, u.data(), sizeof(double) * dim);
    if (residuals)
      for (int i = 0; i < std::min<int>(max_res, diag.residual_history.size()); ++i)
        residuals[i] = diag.residual_history[i];
    *sweeps = diag.sweeps;
    *fresh_evals = diag.fresh_evals;
    *early_stop = diag.early_stop ? 1 : 0;
  });
}

// integrate_mrsdc mode 1 (mrsdc.cpp:227-259) with C callbacks; fine level
// TypeB{inner} (fine_type 1) or TypeC{inner, repeats} (fine_type 2).
int ref_integrate_mrsdc1(rhs_cb f1, void* ctx1, rhs_cb f2, void* ctx2, long long dim,
                         const double* u0, double t0, double t1, int nsteps, int coarse_family,
                         int coarse_nodes, int fine_type, int fine_family, int fine_nodes,
                         int repeats, int iterations, double cutoff, double* u_out,
                         double* residuals, int max_res, int* sweeps, int* f1_evals,
                         int* f2_evals) {
  return guarded([&] {
    StepControls c;
    c.num_iterations = iterations;
    c.residual_ratio_cutoff = cutoff;
    FineSpec spec = fine_type == 2 ? FineSpec{TypeC{nodes_from(fine_family, fine_nodes), repeats}}
                                   : FineSpec{TypeB{nodes_from(fine_family, fine_nodes)}};
    MultirateHierarchy h = build_hierarchy(nodes_from(coarse_family, coarse_nodes), spec);
    SplitRHS rhs;
    rhs.f1 = wrap_cb(f1, ctx1);
    rhs.f2 = wrap_cb(f2, ctx2);
    auto [u, diag] = integrate_mrsdc(rhs, Field(u0, u0 + dim), t0, t1, nsteps, h, c);
    std::memcpy(u_out, u.data(), sizeof(double) * dim);
    if (residuals)
      for (int i = 0; i < std::min<int>(max_res, diag.residual_history.size()); ++i)
        residuals[i] = diag.residual_history[i];
    *sweeps = diag.sweeps;
    *f1_evals = diag.f1_evals;
    *f2_evals = diag.f2_evals;
  });
}

// integrate_mrsdc with f1 implicit (mode 2, mrsdc.cpp:137-206, :227-259) and
// StiffOptions{rtol, atol, max_newton_iters} (stiff.hpp:10-20).  Returns 2
// with ref_last_error() on IntegrationError (e.g. Newton failure).
int ref_integrate_mrsdc2(rhs_cb f1, void* ctx1, rhs_cb f2, void* ctx2, long long dim,
                         const double* u0, double t0, double t1, int nsteps, int coarse_family,
                         int coarse_nodes, int fine_type, int fine_family, int fine_nodes,
                         int repeats, int iterations, double cutoff, double rtol, double atol,
                         int max_newton_iters, double* u_out, double* residuals, int max_res,
                         int* sweeps, int* f1_evals, int* f2_evals, int* implicit_solves,
                         int* newton_f1_evals) {
  return guarded([&] {
    StepControls c;
    c.num_iterations = iterations;
    c.residual_ratio_cutoff = cutoff;
    StiffOptions so;
    so.rtol = rtol;
    so.atol = atol;
    so.max_newton_iters = max_newton_iters;
    FineSpec spec = fine_type == 2 ? FineSpec{TypeC{nodes_from(fine_family, fine_nodes), repeats}}
                                   : FineSpec{TypeB{nodes_from(fine_family, fine_nodes)}};
    MultirateHierarchy h = build_hierarchy(nodes_from(coarse_family, coarse_nodes), spec);
    SplitRHS rhs;
    rhs.f1 = wrap_cb(f1, ctx1);
    rhs.f2 = wrap_cb(f2, ctx2);
    rhs.f1_stiffness = SplitRHS::Stiffness::Implicit;
    auto [u, diag] = integrate_mrsdc(rhs, Field(u0, u0 + dim), t0, t1, nsteps, h, c, so);
    std::memcpy(u_out, u.data(), sizeof(double) * dim);
    if (residuals)
      for (int i = 0; i < std::min<int>(max_res, diag.residual_history.size()); ++i)
        residuals[i] = diag.residual_history[i];
    *sweeps = diag.sweeps;
    *f1_evals = diag.f1_evals;
    *f2_evals = diag.f2_evals;
    *implicit_solves = diag.implicit_solves;
    *newton_f1_evals = diag.newton_f1_evals;
  });
}

// solve_backward_euler (stiff.cpp:34-76) with a report: out_int = {iterations,
// converged, f_evals}, *final_residual.
int ref_solve_backward_euler(rhs_cb f, void* ctx, long long dim, double t, double beta,
                             const double* c, const double* guess, double rtol, double atol,
                             int max_newton_iters, double* w, int* out_int,
                             double* final_residual) {
  return guarded([&] {
    StiffOptions so;
    so.rtol = rtol;
    so.atol = atol;
    so.max_newton_iters = max_newton_iters;
    NewtonReport rep;
    Field r = solve_backward_euler(wrap_cb(f, ctx), t, beta, Field(c, c + dim),
                                   Field(guess, guess + dim), so, &rep);
    std::memcpy(w, r.data(), sizeof(double) * dim);
    out_int[0] = rep.iterations;
    out_int[1] = rep.converged ? 1 : 0;
    out_int[2] = rep.f_evals;
    *final_residual = rep.final_residual;
  });
}

// integrate_stiff (stiff.cpp:115-188); returns 2 with ref_last_error() on
// IntegrationError (step size collapse), 1 on std::invalid_argument.
int ref_integrate_stiff(rhs_cb f, void* ctx, long long dim, const double* u0, double t0,
                        double t1, double rtol, double atol, int max_newton_iters,
                        double initial_step_fraction, double* u_out) {
  return guarded([&] {
    StiffOptions so;
    so.rtol = rtol;
    so.atol = atol;
    so.max_newton_iters = max_newton_iters;
    so.initial_step_fraction = initial_step_fraction;
    Field r = integrate_stiff(wrap_cb(f, ctx), Field(u0, u0 + dim), t0, t1, so);
    std::memcpy(u_out, r.data(), sizeof(double) * dim);
  });
}

// ------------------------------------------------------------- quadrature
int ref_nodes(int family, int n, double* out) {
  return guarded([&] {
    NodeSet s = nodes_from(family, n);
    std::memcpy(out, s.nodes.data(), sizeof(double) * s.nodes.size());
  });
}
// Q and S, each M x (M+1) row-major (quadrature.cpp:134-158)
int ref_integration_matrices(int family, int n, double* q, double* s) {
  return guarded([&] {
    IntegrationMatrices m = integration_matrices(nodes_from(family, n));
    copy_matrix(m.q, q);
    copy_matrix(m.s, s);
  });
}
// build_hierarchy (quadrature.cpp:178-248).  Returns fine count in *m2p1.
int ref_build_hierarchy(int coarse_family, int coarse_nodes, int fine_type, int fine_family,
                        int fine_nodes, int repeats, int* m2p1, double* fine, double* q21,
                        double* s21, double* q22, double* s22, int* fine_of_coarse, int* p_map) {
  return guarded([&] {
    FineSpec spec = fine_type == 2 ? FineSpec{TypeC{nodes_from(fine_family, fine_nodes), repeats}}
                                   : FineSpec{TypeB{nodes_from(fine_family, fine_nodes)}};
    MultirateHierarchy h = build_hierarchy(nodes_from(coarse_family, coarse_nodes), spec);
    *m2p1 = h.fine.count();
    if (fine) std::memcpy(fine, h.fine.nodes.data(), sizeof(double) * h.fine.nodes.size());
    copy_matrix(h.q21, q21);
    copy_matrix(h.s21, s21);
    copy_matrix(h.q22, q22);
    copy_matrix(h.s22, s22);
    if (fine_of_coarse)
      for (std::size_t i = 0; i < h.fine_of_coarse.size(); ++i) fine_of_coarse[i] = h.fine_of_coarse[i];
    if (p_map)
      for (std::size_t i = 0; i < h.p_map.size(); ++i) p_map[i] = h.p_map[i];
  });
}

}  // extern "C"
