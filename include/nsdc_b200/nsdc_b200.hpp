// nsdc_b200.hpp — C++ drop-in for the RHS hot path of the reference `nsdc`
// library (/root/reference/proj/core/include/nsdc), header-only over the C
// ABI of libsmc_b200.so (include/smc_b200.h).
//
// Same names, signatures, argument meaning and error behaviour as the
// reference (std::invalid_argument for bad arguments, IntegrationError for
// integration failures); the types Field and Rhs are the same std types, so
// an nsdc_b200 operator's as_rhs() plugs into the reference's own
// integrate_sdc / integrate_mrsdc unchanged, and the reference's Rhs plugs
// into the device-resident steppers here.  Namespace nsdc_b200 (not nsdc) so
// both libraries can be linked into one binary for parity testing; a user
// switching over writes `namespace nsdc = nsdc_b200;`.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <functional>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <variant>
#include <vector>

#include "../smc_b200.h"

namespace nsdc_b200 {

// ---------------------------------------------------------------- field.hpp
using Field = std::vector<double>;
using Rhs = std::function<void(double t, const Field& u, Field& out)>;

inline double max_norm(const Field& v) {
  double m = 0.0;
  for (double x : v) m = std::max(m, std::fabs(x));
  return m;
}
inline void axpy(double alpha, const Field& x, Field& y) {
  for (std::size_t i = 0; i < y.size(); ++i) y[i] += alpha * x[i];
}

// --------------------------------------------------------------- errors.hpp
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
class IntegrationError : public std::runtime_error {
 public:
  explicit IntegrationError(const std::string& w) : std::runtime_error(w) {}
};

namespace detail {
inline void check(int rc) {
  if (rc == SMC_OK) return;
  const std::string msg = smc_last_error();
  if (rc == SMC_EINVAL) throw std::invalid_argument(msg);
  if (rc == SMC_EINTEGRATION) throw IntegrationError(msg);
  throw std::runtime_error(msg);
}
struct RhsDeleter {
  void operator()(smc_rhs* h) const { smc_rhs_destroy(h); }
};
using RhsHandle = std::unique_ptr<smc_rhs, RhsDeleter>;
}  // namespace detail

// -------------------------------------------------------------- stencil.hpp
struct StencilMatrix {
  int s = 0;
  std::array<std::array<double, 8>, 8> m{};
  std::vector<double> params;
  double at(int mm, int nn) const { return m[mm + s - 1][nn + s - 1]; }
};

inline constexpr double kSmcM47 = 3557.0 / 44100.0;
inline constexpr double kSmcM48 = -2083.0 / 117600.0;
inline constexpr double kOptimalM47 = 1059283.0 / 13608000.0;
inline constexpr double kOptimalM48 = -856481.0 / 40824000.0;
inline constexpr double kDefaultM36 = 281.0 / 3600.0;

inline StencilMatrix build_narrow(int order, const std::vector<double>& params) {
  StencilMatrix out;
  double m64[64];
  detail::check(smc_build_narrow(order, params.data(), static_cast<int>(params.size()), m64,
                                 &out.s));
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) out.m[i][j] = m64[i * 8 + j];
  out.params = params;
  return out;
}

inline Field apply_narrow(const StencilMatrix& m, const Field& a, const Field& u, double dx) {
  if (a.size() != u.size()) throw std::invalid_argument("apply_narrow: size mismatch");
  Field out(u.size());
  detail::check(smc_apply_narrow(m.s == 4 ? 8 : 6, m.params.data(),
                                 static_cast<int>(m.params.size()), a.data(), u.data(),
                                 static_cast<int>(u.size()), dx, out.data(), SMC_HOST));
  return out;
}
inline Field first_derivative8(const Field& u, double dx) {
  Field out(u.size());
  detail::check(smc_first_derivative8(u.data(), static_cast<int>(u.size()), dx, out.data(),
                                      SMC_HOST));
  return out;
}
// Non-periodic lines with the paper's boundary closure (smc_b200.h
// smc_apply_narrow_bounded): one line of u.size() cells.
inline Field apply_narrow_bounded(const Field& a, const Field& u, double dx,
                                  const std::vector<double>& params = {}) {
  if (a.size() != u.size()) throw std::invalid_argument("apply_narrow_bounded: size mismatch");
  Field out(u.size());
  detail::check(smc_apply_narrow_bounded(params.data(), static_cast<int>(params.size()), a.data(),
                                         u.data(), static_cast<int>(u.size()), 1, dx, out.data(),
                                         SMC_HOST));
  return out;
}
inline Field first_derivative_bounded(const Field& u, double dx) {
  Field out(u.size());
  detail::check(smc_first_derivative_bounded(u.data(), static_cast<int>(u.size()), 1, dx,
                                             out.data(), SMC_HOST));
  return out;
}
inline Field apply_wide(const Field& a, const Field& u, double dx) {
  if (a.size() != u.size()) throw std::invalid_argument("apply_wide: size mismatch");
  Field out(u.size());
  detail::check(smc_apply_wide(a.data(), u.data(), static_cast<int>(u.size()), dx, out.data(),
                               SMC_HOST));
  return out;
}

struct StencilChoice {
  enum class Kind { Narrow8, Narrow6, Wide8 };
  Kind kind = Kind::Narrow8;
  std::array<double, 2> params{};
  static StencilChoice narrow8(double m47, double m48) { return {Kind::Narrow8, {m47, m48}}; }
  static StencilChoice narrow6(double m36) { return {Kind::Narrow6, {m36, 0.0}}; }
  static StencilChoice wide8() { return {Kind::Wide8, {0.0, 0.0}}; }
};

inline StencilChoice stencil_preset(std::string_view name) {
  if (name == "SMC") return StencilChoice::narrow8(kSmcM47, kSmcM48);
  if (name == "ZERO") return StencilChoice::narrow8(0.0, 0.0);
  if (name == "OPTIMAL") return StencilChoice::narrow8(kOptimalM47, kOptimalM48);
  if (name == "NARROW6") return StencilChoice::narrow6(kDefaultM36);
  if (name == "WIDE") return StencilChoice::wide8();
  throw std::invalid_argument("unknown stencil preset: " + std::string(name));
}

// ----------------------------------------------------------- quadrature.hpp
enum class NodeKind { GaussLobatto, ClenshawCurtis, Composite };
struct NodeSet {
  std::vector<double> nodes;
  NodeKind kind = NodeKind::GaussLobatto;
  int count() const { return static_cast<int>(nodes.size()); }
  int intervals() const { return count() - 1; }
};
inline NodeSet gauss_lobatto(int n) {
  if (n < 2) throw std::invalid_argument("gauss_lobatto: need at least 2 nodes");
  NodeSet s{std::vector<double>(n), NodeKind::GaussLobatto};
  detail::check(smc_nodes(SMC_GAUSS_LOBATTO, n, s.nodes.data()));
  return s;
}
inline NodeSet clenshaw_curtis(int n) {
  if (n < 2) throw std::invalid_argument("clenshaw_curtis: need at least 2 nodes");
  NodeSet s{std::vector<double>(n), NodeKind::ClenshawCurtis};
  detail::check(smc_nodes(SMC_CLENSHAW_CURTIS, n, s.nodes.data()));
  return s;
}
inline int family_of(const NodeSet& s) {
  if (s.kind == NodeKind::Composite)
    throw std::invalid_argument("device steppers take simple node sets");
  return s.kind == NodeKind::GaussLobatto ? SMC_GAUSS_LOBATTO : SMC_CLENSHAW_CURTIS;
}
struct TypeA {
  NodeSet fine;  // must contain every coarse node
};
struct TypeB {
  NodeSet inner;
};
struct TypeC {
  NodeSet inner;
  int repeats = 1;
};
using FineSpec = std::variant<TypeA, TypeB, TypeC>;

// matrix.hpp: dense row-major matrix
struct Matrix {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), a(static_cast<std::size_t>(r) * c) {}
  double& operator()(int r, int c) { return a[static_cast<std::size_t>(r) * cols + c]; }
  double operator()(int r, int c) const { return a[static_cast<std::size_t>(r) * cols + c]; }
};

// MultirateHierarchy (quadrature.hpp:70-77) from the library's builder
// (quadrature.cpp:178-248); `spec` records what the device stepper is built
// from (TypeB == TypeC with one repeat, TypeA == repeats 0 with the fine set
// as `inner`).
struct MultirateHierarchy {
  NodeSet coarse;
  NodeSet fine;
  Matrix q21, s21;
  Matrix q22, s22;
  std::vector<int> fine_of_coarse;
  std::vector<int> p_map;
  TypeC spec;
};
inline MultirateHierarchy build_hierarchy(const NodeSet& coarse, const FineSpec& fs) {
  const TypeC c = std::holds_alternative<TypeA>(fs)   ? TypeC{std::get<TypeA>(fs).fine, 0}
                  : std::holds_alternative<TypeB>(fs) ? TypeC{std::get<TypeB>(fs).inner, 1}
                                                      : std::get<TypeC>(fs);
  if (std::holds_alternative<TypeC>(fs) && std::get<TypeC>(fs).repeats < 1)
    throw std::invalid_argument("build_hierarchy: repeats must be >= 1");
  MultirateHierarchy h;
  h.coarse = coarse;
  h.spec = c;
  int m2p1 = 0;
  detail::check(smc_build_hierarchy(family_of(coarse), coarse.count(), family_of(c.inner),
                                    c.inner.count(), c.repeats, &m2p1, nullptr, nullptr, nullptr,
                                    nullptr, nullptr, nullptr, nullptr));
  const int m1 = coarse.intervals(), m2 = m2p1 - 1;
  h.fine = NodeSet{std::vector<double>(m2p1), NodeKind::Composite};
  h.q21 = Matrix(m2, m1 + 1), h.s21 = Matrix(m2, m1 + 1);
  h.q22 = Matrix(m2, m2p1), h.s22 = Matrix(m2, m2p1);
  h.fine_of_coarse.resize(coarse.count());
  h.p_map.resize(m2p1);
  detail::check(smc_build_hierarchy(family_of(coarse), coarse.count(), family_of(c.inner),
                                    c.inner.count(), c.repeats, &m2p1, h.fine.nodes.data(),
                                    h.q21.a.data(), h.s21.a.data(), h.q22.a.data(),
                                    h.s22.a.data(), h.fine_of_coarse.data(), h.p_map.data()));
  return h;
}

// ---------------------------------------------------------------- pde.hpp
inline constexpr double kTwoPi = 2.0 * std::numbers::pi;
struct Grid2D {  // pde.hpp:14-22: node-based periodic [0, 2pi)^2
  int nx = 0, ny = 0;
  double dx() const { return kTwoPi / nx; }
  double dy() const { return kTwoPi / ny; }
  double x(int i) const { return i * kTwoPi / nx; }
  double y(int j) const { return j * kTwoPi / ny; }
};
struct Field2D {
  int nx = 0, ny = 0;
  std::vector<double> v;
  Field2D() = default;
  Field2D(int nx_, int ny_) : nx(nx_), ny(ny_), v(static_cast<std::size_t>(nx_) * ny_, 0.0) {}
  double& at(int i, int j) { return v[static_cast<std::size_t>(j) * nx + i]; }
  double at(int i, int j) const { return v[static_cast<std::size_t>(j) * nx + i]; }
};
struct HeatProblem {
  std::function<double(double, double)> a, b;
  std::function<double(double, double, double)> g;
  std::function<double(double, double)> g_space;
  std::function<double(double)> g_time;
  std::function<double(double, double)> u0;
  std::function<double(double, double, double)> exact;
  double epsilon = 0.0;
};
inline Field2D eval_on_grid(const Grid2D& g, const std::function<double(double, double)>& fn) {
  Field2D out(g.nx, g.ny);
  for (int j = 0; j < g.ny; ++j)
    for (int i = 0; i < g.nx; ++i) out.at(i, j) = fn(g.x(i), g.y(j));
  return out;
}

// Heat RHS on the GPU (pde.hpp:69-84).  The problem's coefficient and source
// functions are host code: they are sampled on the grid at construction
// (pde.cpp:232-257); per call only g_time(t) runs on the host.
class HeatOperator {
 public:
  HeatOperator(const HeatProblem& p, const Grid2D& g, const StencilChoice& choice)
      : st_(std::make_unique<State>()) {
    st_->grid = g;
    const int min_n = choice.kind == StencilChoice::Kind::Wide8
                          ? 9
                          : (choice.kind == StencilChoice::Kind::Narrow8 ? 9 : 7);
    if (g.nx < min_n || g.ny < min_n)
      throw std::invalid_argument("HeatOperator: grid too small for the chosen stencil");
    if (!p.a || !p.b || !p.u0) throw std::invalid_argument("HeatOperator: incomplete problem");
    const Field2D a = eval_on_grid(g, p.a), b = eval_on_grid(g, p.b);
    Field2D g0;
    const bool separable = static_cast<bool>(p.g_space) && static_cast<bool>(p.g_time);
    if (separable) g0 = eval_on_grid(g, p.g_space);
    const int kind = static_cast<int>(choice.kind);
    smc_rhs* h = nullptr;
    detail::check(smc_heat_create(g.nx, g.ny, kind, choice.params.data(), a.v.data(), b.v.data(),
                                  separable ? g0.v.data() : nullptr, &h));
    st_->h.reset(h);
    if (separable) {
      st_->g_time = p.g_time;
      detail::check(smc_heat_set_time_source(h, &State::gtime, st_.get()));
    } else if (p.g) {
      st_->g_full = p.g;
      detail::check(smc_heat_set_full_source(h, &State::gfull, st_.get()));
    }
  }

  void rhs(double t, const Field2D& u, Field2D& out) const {
    if (u.nx != st_->grid.nx || u.ny != st_->grid.ny)
      throw std::invalid_argument("HeatOperator::rhs: field/grid shape mismatch");
    out.nx = u.nx, out.ny = u.ny;
    out.v.resize(u.v.size());
    detail::check(smc_rhs_eval(st_->h.get(), t, u.v.data(), out.v.data(), SMC_HOST));
  }
  Rhs as_rhs() const {
    State* s = st_.get();
    const std::size_t n = static_cast<std::size_t>(s->grid.nx) * s->grid.ny;
    return [s, n](double t, const Field& u, Field& out) {
      if (u.size() != n) throw std::invalid_argument("heat rhs: flat state has wrong size");
      out.resize(n);
      detail::check(smc_rhs_eval(s->h.get(), t, u.data(), out.data(), SMC_HOST));
    };
  }
  const Grid2D& grid() const { return st_->grid; }
  smc_rhs* handle() const { return st_->h.get(); }

 private:
  struct State {
    Grid2D grid;
    detail::RhsHandle h;
    std::function<double(double)> g_time;
    std::function<double(double, double, double)> g_full;
    static double gtime(double t, void* ctx) { return static_cast<State*>(ctx)->g_time(t); }
    static void gfull(double t, double* f, void* ctx) {
      auto* s = static_cast<State*>(ctx);
      for (int j = 0; j < s->grid.ny; ++j)
        for (int i = 0; i < s->grid.nx; ++i)
          f[static_cast<std::size_t>(j) * s->grid.nx + i] =
              s->g_full(t, s->grid.x(i), s->grid.y(j));
    }
  };
  std::unique_ptr<State> st_;
};

inline Field2D heat_rhs(const HeatProblem& p, const Grid2D& g, const StencilChoice& c, double t,
                        const Field2D& u) {
  HeatOperator op(p, g, c);
  Field2D out(g.nx, g.ny);
  op.rhs(t, u, out);
  return out;
}

// 3-D narrow operator (a U_x)_x + (a U_y)_y + (a U_z)_z (BASELINE configs[1]).
class Narrow3DOperator {
 public:
  Narrow3DOperator(int nx, int ny, int nz, double dx, double dy, double dz, const Field& a,
                   const StencilChoice& c = StencilChoice::narrow8(kSmcM47, kSmcM48)) {
    if (a.size() != static_cast<std::size_t>(nx) * ny * nz)
      throw std::invalid_argument("Narrow3DOperator: coefficient size mismatch");
    smc_rhs* h = nullptr;
    const int order = c.kind == StencilChoice::Kind::Narrow6 ? 6 : 8;
    detail::check(smc_narrow3d_create(nx, ny, nz, dx, dy, dz, order, c.params.data(),
                                      order == 8 ? 2 : 1, a.data(), SMC_HOST, &h));
    h_.reset(h);
  }
  Rhs as_rhs() const {
    smc_rhs* h = h_.get();
    return [h](double t, const Field& u, Field& out) {
      if (static_cast<long long>(u.size()) != smc_rhs_dim(h))
        throw std::invalid_argument("narrow3d rhs: flat state has wrong size");
      out.resize(u.size());
      detail::check(smc_rhs_eval(h, t, u.data(), out.data(), SMC_HOST));
    };
  }
  smc_rhs* handle() const { return h_.get(); }

 private:
  detail::RhsHandle h_;
};

// ---------------------------------------------------------------- mrsdc.hpp
struct SplitRHS {
  Rhs f1;
  Rhs f2;
  enum class Stiffness { Explicit, Implicit };
  Stiffness f1_stiffness = Stiffness::Explicit;
};

// Reacting-NS RHS (14 conserved fields, field-major) with the synthetic
// mechanism of include/smc_mechanism.h: full RHS, and the MRSDC split
// f1 = hypterm + diffterm, f2 = wdot.
class NsOperator {
 public:
  NsOperator(int nx, int ny, int nz, double dx,
             const StencilChoice& c = StencilChoice::narrow8(kSmcM47, kSmcM48)) {
    smc_rhs *f = nullptr, *a = nullptr, *ch = nullptr;
    const int order = c.kind == StencilChoice::Kind::Narrow6 ? 6 : 8;
    detail::check(smc_ns_create(nx, ny, nz, 0, dx, dx, dx, order, c.params.data(),
                                order == 8 ? 2 : 1, &f, &a, &ch));
    full_.reset(f), adv_.reset(a), chem_.reset(ch);
  }
  Rhs as_rhs() const { return wrap(full_.get()); }
  SplitRHS as_split() const { return SplitRHS{wrap(adv_.get()), wrap(chem_.get())}; }
  smc_rhs* full() const { return full_.get(); }
  smc_rhs* advdiff() const { return adv_.get(); }
  smc_rhs* chem() const { return chem_.get(); }

 private:
  static Rhs wrap(smc_rhs* h) {
    return [h](double t, const Field& u, Field& out) {
      out.resize(u.size());
      detail::check(smc_rhs_eval(h, t, u.data(), out.data(), SMC_HOST));
    };
  }
  detail::RhsHandle full_, adv_, chem_;
};

// ------------------------------------------------ multi-GPU (z-slab) NS
// One rank of an NCCL communicator (smc_comm_*): the unique id is created on
// one rank (unique_id()) and shared by the host program (MPI, a file, a
// socket), then every rank constructs Communicator(id, size, rank) on its
// own GPU.  A C++ host replaces the reference's single-process
// parallel_for (parallel.cpp:20-36) by one process per GPU.
class Communicator {
 public:
  static std::string unique_id() {
    std::string id(128, '\0');
    detail::check(smc_comm_unique_id(id.data()));
    return id;
  }
  Communicator(const std::string& id, int size, int rank) {
    if (id.size() != 128) throw std::invalid_argument("Communicator: the id holds 128 bytes");
    smc_comm* c = nullptr;
    detail::check(smc_comm_init(id.data(), size, rank, &c));
    c_.reset(c);
  }
  int rank() const {
    int r = 0, s = 0;
    detail::check(smc_comm_rank(c_.get(), &r, &s));
    return r;
  }
  int size() const {
    int r = 0, s = 0;
    detail::check(smc_comm_rank(c_.get(), &r, &s));
    return s;
  }
  double allreduce_max(double v) {
    detail::check(smc_comm_allreduce_max(c_.get(), &v));
    return v;
  }
  smc_comm* handle() const { return c_.get(); }

 private:
  struct Del {
    void operator()(smc_comm* c) const { smc_comm_destroy(c); }
  };
  std::unique_ptr<smc_comm, Del> c_;
};

// This rank's z-slab (nz planes) of the periodic nx x ny x (nz * size) NS
// box: the same Rhs / SplitRHS views as NsOperator over the rank's interior
// state; the 4-plane halo is exchanged inside every evaluation.
class NsSlabOperator {
 public:
  NsSlabOperator(Communicator& comm, int nx, int ny, int nz, double dx,
                 const StencilChoice& c = StencilChoice::narrow8(kSmcM47, kSmcM48)) {
    smc_rhs *f = nullptr, *a = nullptr, *ch = nullptr;
    const int order = c.kind == StencilChoice::Kind::Narrow6 ? 6 : 8;
    detail::check(smc_ns_slab_create(comm.handle(), nx, ny, nz, dx, dx, dx, order,
                                     c.params.data(), order == 8 ? 2 : 1, &f, &a, &ch));
    full_.reset(f), adv_.reset(a), chem_.reset(ch);
  }
  Rhs as_rhs() const { return wrap(full_.get()); }
  SplitRHS as_split() const { return SplitRHS{wrap(adv_.get()), wrap(chem_.get())}; }
  smc_rhs* full() const { return full_.get(); }
  smc_rhs* advdiff() const { return adv_.get(); }
  smc_rhs* chem() const { return chem_.get(); }

 private:
  static Rhs wrap(smc_rhs* h) {
    return [h](double t, const Field& u, Field& out) {
      out.resize(u.size());
      detail::check(smc_rhs_eval(h, t, u.data(), out.data(), SMC_HOST));
    };
  }
  detail::RhsHandle full_, adv_, chem_;
};

// ----------------------------------------------------------------- sdc.hpp
struct StepControls {
  int num_iterations = 4;
  double residual_ratio_cutoff = 0.05;
  bool reuse_first_eval = true;
};
struct SweepDiagnostics {
  std::vector<double> residual_history;
  int sweeps = 0;
  int fresh_evals = 0;
  bool early_stop = false;
};
struct MrsdcDiagnostics {
  std::vector<double> residual_history;
  int sweeps = 0;
  int f1_evals = 0;
  int f2_evals = 0;
  int implicit_solves = 0;
  int newton_f1_evals = 0;
  bool early_stop = false;
};

// stiff.hpp:10-27.  `block` / `interleaved` declare the block structure of
// the implicit term for the device Newton (0 = dense, the reference's case;
// see smc_stiff in smc_b200.h).  A user-supplied Jacobian is not on the
// device path.
struct StiffOptions {
  double rtol = 1e-8;
  double atol = 1e-10;
  int max_newton_iters = 16;
  double initial_step_fraction = 1e-3;
  enum class Jacobian { FiniteDifference, UserSupplied };
  Jacobian jacobian = Jacobian::FiniteDifference;
  std::function<void(double t, const Field& u, Matrix& j)> user_jacobian;
  long long block = 0;
  bool interleaved = false;
};
struct NewtonReport {
  int iterations = 0;
  double final_residual = 0.0;
  bool converged = false;
  int f_evals = 0;
};

namespace detail {
// Any nsdc::Rhs as a device operator (host round trip per call); the
// overloads below taking a GPU operator skip it.
struct CallbackRhs {
  Rhs f;
  RhsHandle h;
  std::size_t dim;
  CallbackRhs(const Rhs& fn, std::size_t n) : f(fn), dim(n) {
    smc_rhs* raw = nullptr;
    check(smc_rhs_from_callback(static_cast<long long>(n), &CallbackRhs::tramp, this, &raw));
    h.reset(raw);
  }
  static void tramp(double t, const double* u, double* out, long long n, void* ctx) {
    auto* self = static_cast<CallbackRhs*>(ctx);
    Field uu(u, u + n), oo(static_cast<std::size_t>(n));
    self->f(t, uu, oo);
    std::copy(oo.begin(), oo.end(), out);
  }
};
struct DiagBuf {
  std::vector<double> res = std::vector<double>(4096);
  smc_diag d{};
  DiagBuf() {
    d.residual_capacity = static_cast<int>(res.size());
    d.residuals = res.data();
  }
  std::vector<double> history() const {
    return {res.begin(), res.begin() + std::min(d.n_residuals, d.residual_capacity)};
  }
};
inline smc_stiff to_c(const StiffOptions& o) {
  if (o.jacobian == StiffOptions::Jacobian::UserSupplied)
    throw std::invalid_argument("StiffOptions: a user-supplied Jacobian is not on the device path");
  return smc_stiff{o.rtol, o.atol, o.max_newton_iters, o.block, o.interleaved ? 1 : 0,
                   o.initial_step_fraction};
}
struct SdcDeleter {
  void operator()(smc_sdc* s) const { smc_sdc_destroy(s); }
};
struct MrsdcDeleter {
  void operator()(smc_mrsdc* s) const { smc_mrsdc_destroy(s); }
};
}  // namespace detail

// Device-resident SdcStepper (sdc.hpp:45-69): node values stay in HBM.
class SdcStepper {
 public:
  SdcStepper(NodeSet nodes, StepControls c) : nodes_(std::move(nodes)), c_(c) {
    if (c.num_iterations < 1) throw std::invalid_argument("SdcStepper: need at least one sweep");
    smc_sdc* s = nullptr;
    detail::check(smc_sdc_create(family_of(nodes_), nodes_.count(), c.num_iterations,
                                 c.residual_ratio_cutoff, c.reuse_first_eval ? 1 : 0, &s));
    s_.reset(s);
  }
  struct Result {
    Field u;
    Field f_end;
    SweepDiagnostics diag;
  };
  Result step(const Rhs& f, const Field& u0, double t_n, double dt, const Field* f0 = nullptr) {
    detail::CallbackRhs cb(f, u0.size());
    return step(cb.h.get(), u0, t_n, dt, f0);
  }
  Result step(smc_rhs* op, const Field& u0, double t_n, double dt, const Field* f0 = nullptr) {
    Result r{Field(u0.size()), Field(u0.size()), {}};
    detail::DiagBuf db;
    detail::check(smc_sdc_step(s_.get(), op, u0.data(), t_n, dt, f0 ? f0->data() : nullptr,
                               r.u.data(), r.f_end.data(), SMC_HOST, &db.d));
    r.diag = {db.history(), db.d.sweeps, db.d.fresh_evals, db.d.early_stop != 0};
    return r;
  }
  std::pair<Field, SweepDiagnostics> integrate(smc_rhs* op, const Field& u0, double t0,
                                               double t1, int nsteps) {
    if (nsteps < 0) throw std::invalid_argument("integrate_sdc: negative step count");
    Field u(u0.size());
    detail::DiagBuf db;
    detail::check(smc_sdc_integrate(s_.get(), op, u0.data(), t0, t1, nsteps, u.data(), SMC_HOST,
                                    &db.d));
    return {std::move(u), {db.history(), db.d.sweeps, db.d.fresh_evals, db.d.early_stop != 0}};
  }
  const NodeSet& nodes() const { return nodes_; }
  // residual reduced over the ranks of a slab decomposition
  void set_communicator(const Communicator& c) { detail::check(smc_sdc_set_comm(s_.get(), c.handle())); }

 private:
  NodeSet nodes_;
  StepControls c_;
  std::unique_ptr<smc_sdc, detail::SdcDeleter> s_;
};

inline std::pair<Field, SweepDiagnostics> sdc_step(const Rhs& f, const Field& u0, double t_n,
                                                   double dt, const NodeSet& nodes,
                                                   const StepControls& c) {
  SdcStepper s(nodes, c);
  auto r = s.step(f, u0, t_n, dt);
  return {std::move(r.u), std::move(r.diag)};
}

// integrate_sdc (sdc.hpp:78-80) for any Rhs ...
inline std::pair<Field, SweepDiagnostics> integrate_sdc(const Rhs& f, const Field& u0, double t0,
                                                        double t1, int nsteps,
                                                        const NodeSet& nodes,
                                                        const StepControls& c) {
  if (nsteps < 0) throw std::invalid_argument("integrate_sdc: negative step count");
  detail::CallbackRhs cb(f, u0.size());
  SdcStepper s(nodes, c);
  return s.integrate(cb.h.get(), u0, t0, t1, nsteps);
}
// ... and without host round trips for a GPU operator
template <class Op>
inline auto integrate_sdc(const Op& op, const Field& u0, double t0, double t1, int nsteps,
                          const NodeSet& nodes, const StepControls& c)
    -> decltype(op.handle(), std::pair<Field, SweepDiagnostics>{}) {
  SdcStepper s(nodes, c);
  return s.integrate(op.handle(), u0, t0, t1, nsteps);
}

// Device-resident MrsdcStepper (mrsdc.hpp:51-82): mode 1 and mode 2 (f1
// implicit through the device Newton), hierarchy build_hierarchy(coarse,
// TypeB/TypeC{inner}).
class MrsdcStepper {
 public:
  MrsdcStepper(MultirateHierarchy h, StepControls c, StiffOptions stiff = {})
      : c_(c), h_(std::move(h)), stiff_(std::move(stiff)) {
    if (c.num_iterations < 1) throw std::invalid_argument("MrsdcStepper: need at least one sweep");
    smc_mrsdc* m = nullptr;
    detail::check(smc_mrsdc_create(family_of(h_.coarse), h_.coarse.count(),
                                   family_of(h_.spec.inner), h_.spec.inner.count(),
                                   h_.spec.repeats, c.num_iterations, c.residual_ratio_cutoff,
                                   c.reuse_first_eval ? 1 : 0, &m));
    m_.reset(m);
    const smc_stiff so = detail::to_c(stiff_);
    detail::check(smc_mrsdc_set_stiff(m_.get(), &so));
  }
  MrsdcStepper(const NodeSet& coarse, const TypeC& fine, StepControls c)
      : MrsdcStepper(build_hierarchy(coarse, fine), c) {}
  MrsdcStepper(const NodeSet& coarse, const TypeB& fine, StepControls c)
      : MrsdcStepper(coarse, TypeC{fine.inner, 1}, c) {}
  struct Result {
    Field u, f1_end, f2_end;
    MrsdcDiagnostics diag;
  };
  // residual and implicit-solver norms reduced over a slab decomposition
  void set_communicator(const Communicator& c) {
    detail::check(smc_mrsdc_set_comm(m_.get(), c.handle()));
  }
  Result step_mode1(smc_rhs* f1, smc_rhs* f2, const Field& u0, double t_n, double dt,
                    const Field* f01 = nullptr, const Field* f02 = nullptr) {
    return step(smc_mrsdc_step_mode1, f1, f2, u0, t_n, dt, f01, f02);
  }
  Result step_mode1(const SplitRHS& rhs, const Field& u0, double t_n, double dt,
                    const Field* f01 = nullptr, const Field* f02 = nullptr) {
    detail::CallbackRhs a(rhs.f1, u0.size()), b(rhs.f2, u0.size());
    return step_mode1(a.h.get(), b.h.get(), u0, t_n, dt, f01, f02);
  }
  // f1 implicit: one backward-Euler-form Newton solve per coarse interval
  // (mrsdc.cpp:137-206); throws IntegrationError naming the coarse node.
  Result step_mode2(smc_rhs* f1, smc_rhs* f2, const Field& u0, double t_n, double dt,
                    const Field* f01 = nullptr, const Field* f02 = nullptr) {
    return step(smc_mrsdc_step_mode2, f1, f2, u0, t_n, dt, f01, f02);
  }
  Result step_mode2(const SplitRHS& rhs, const Field& u0, double t_n, double dt,
                    const Field* f01 = nullptr, const Field* f02 = nullptr) {
    detail::CallbackRhs a(rhs.f1, u0.size()), b(rhs.f2, u0.size());
    return step_mode2(a.h.get(), b.h.get(), u0, t_n, dt, f01, f02);
  }
  std::pair<Field, MrsdcDiagnostics> integrate_mode1(smc_rhs* f1, smc_rhs* f2, const Field& u0,
                                                     double t0, double t1, int nsteps) {
    return integrate(smc_mrsdc_integrate_mode1, f1, f2, u0, t0, t1, nsteps);
  }
  std::pair<Field, MrsdcDiagnostics> integrate_mode2(smc_rhs* f1, smc_rhs* f2, const Field& u0,
                                                     double t0, double t1, int nsteps) {
    return integrate(smc_mrsdc_integrate_mode2, f1, f2, u0, t0, t1, nsteps);
  }
  const MultirateHierarchy& hierarchy() const { return h_; }

 private:
  using StepFn = int (*)(smc_mrsdc*, smc_rhs*, smc_rhs*, const double*, double, double,
                         const double*, const double*, double*, double*, double*, int,
                         smc_diag*);
  using IntFn = int (*)(smc_mrsdc*, smc_rhs*, smc_rhs*, const double*, double, double, int,
                        double*, int, smc_diag*);
  Result step(StepFn fn, smc_rhs* f1, smc_rhs* f2, const Field& u0, double t_n, double dt,
              const Field* f01, const Field* f02) {
    const std::size_t n = u0.size();
    Result r{Field(n), Field(n), Field(n), {}};
    detail::DiagBuf db;
    detail::check(fn(m_.get(), f1, f2, u0.data(), t_n, dt, f01 ? f01->data() : nullptr,
                     f02 ? f02->data() : nullptr, r.u.data(), r.f1_end.data(), r.f2_end.data(),
                     SMC_HOST, &db.d));
    r.diag = to_diag(db);
    return r;
  }
  std::pair<Field, MrsdcDiagnostics> integrate(IntFn fn, smc_rhs* f1, smc_rhs* f2,
                                               const Field& u0, double t0, double t1,
                                               int nsteps) {
    Field u(u0.size());
    detail::DiagBuf db;
    detail::check(fn(m_.get(), f1, f2, u0.data(), t0, t1, nsteps, u.data(), SMC_HOST, &db.d));
    return {std::move(u), to_diag(db)};
  }
  static MrsdcDiagnostics to_diag(const detail::DiagBuf& db) {
    MrsdcDiagnostics d;
    d.residual_history = db.history();
    d.sweeps = db.d.sweeps, d.f1_evals = db.d.f1_evals, d.f2_evals = db.d.f2_evals;
    d.implicit_solves = db.d.implicit_solves, d.newton_f1_evals = db.d.newton_f1_evals;
    d.early_stop = db.d.early_stop != 0;
    return d;
  }
  StepControls c_;
  MultirateHierarchy h_;
  StiffOptions stiff_;
  std::unique_ptr<smc_mrsdc, detail::MrsdcDeleter> m_;
};

// mrsdc.hpp:97-101: fixed-step integration, mode selected by f1_stiffness.
inline std::pair<Field, MrsdcDiagnostics> integrate_mrsdc(const SplitRHS& rhs, const Field& u0,
                                                          double t0, double t1, int nsteps,
                                                          const MultirateHierarchy& h,
                                                          const StepControls& c,
                                                          const StiffOptions& stiff = {}) {
  if (nsteps < 0) throw std::invalid_argument("integrate_mrsdc: negative step count");
  detail::CallbackRhs a(rhs.f1, u0.size()), b(rhs.f2, u0.size());
  MrsdcStepper m(h, c, stiff);
  return rhs.f1_stiffness == SplitRHS::Stiffness::Implicit
             ? m.integrate_mode2(a.h.get(), b.h.get(), u0, t0, t1, nsteps)
             : m.integrate_mode1(a.h.get(), b.h.get(), u0, t0, t1, nsteps);
}
inline std::pair<Field, MrsdcDiagnostics> integrate_mrsdc(const SplitRHS& rhs, const Field& u0,
                                                          double t0, double t1, int nsteps,
                                                          const NodeSet& coarse,
                                                          const TypeB& fine,
                                                          const StepControls& c) {
  return integrate_mrsdc(rhs, u0, t0, t1, nsteps, build_hierarchy(coarse, fine), c);
}
inline std::pair<Field, MrsdcDiagnostics> mrsdc_step_mode2(const SplitRHS& rhs, const Field& u0,
                                                           double t_n, double dt,
                                                           const MultirateHierarchy& h,
                                                           const StepControls& c,
                                                           const StiffOptions& stiff) {
  MrsdcStepper m(h, c, stiff);
  MrsdcStepper::Result r = m.step_mode2(rhs, u0, t_n, dt);
  return {std::move(r.u), std::move(r.diag)};
}

// stiff.hpp:42-49: adaptive BE/BDF2 integration on the device; throws
// IntegrationError when the step size collapses, std::invalid_argument for
// t1 < t0 or bad tolerances.
inline Field integrate_stiff(const Rhs& f, const Field& u0, double t0, double t1,
                             const StiffOptions& opts) {
  detail::CallbackRhs op(f, u0.size());
  Field u(u0.size());
  const smc_stiff so = detail::to_c(opts);
  detail::check(smc_integrate_stiff(op.h.get(), u0.data(), t0, t1, u.data(), SMC_HOST, &so,
                                    nullptr, nullptr));
  return u;
}

// stiff.hpp:29-40: w = c + beta f(t_eval, w) by Newton from guess, on the
// device.  Throws IntegrationError on non-convergence when report is null.
inline Field solve_backward_euler(const Rhs& f, double t_eval, double beta, const Field& c,
                                  const Field& guess, const StiffOptions& opts,
                                  NewtonReport* report = nullptr) {
  detail::CallbackRhs op(f, c.size());
  Field w(c.size());
  const smc_stiff so = detail::to_c(opts);
  smc_newton_report rep{};
  detail::check(smc_solve_backward_euler(op.h.get(), t_eval, beta, c.data(), guess.data(),
                                         w.data(), SMC_HOST, &so, report ? &rep : nullptr));
  if (report) *report = NewtonReport{rep.iterations, rep.final_residual, rep.converged != 0,
                                     rep.f_evals};
  return w;
}

}  // namespace nsdc_b200
