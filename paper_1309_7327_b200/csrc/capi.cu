// extern "C" entry points (include/smc_b200.h).  Exceptions never cross the
// boundary: they become status codes plus a thread-local message.
#include <cstring>
#include <string>
#include <vector>

#include "../../include/smc_b200.h"
#include "dist.hpp"
#include "narrow.cuh"
#include "ns.cuh"
#include "ops.hpp"
#include "quadrature.hpp"
#include "sweeps.hpp"

struct smc_rhs {
  std::unique_ptr<smc::RhsOp> op;
};
struct smc_comm {
  std::shared_ptr<smc::HaloTransport> t;
};
struct smc_sdc {
  std::unique_ptr<smc::DeviceSdc> s;
  smc_reduce_fn reduce = nullptr;
  void* reduce_ctx = nullptr;
};
struct smc_mrsdc {
  std::unique_ptr<smc::DeviceMrsdc> m;
  smc_reduce_fn reduce = nullptr;
  void* reduce_ctx = nullptr;
};

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SMC_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return SMC_EINVAL;
  } catch (const smc::IntegrationFailure& e) {
    g_error = e.what();
    return SMC_EINTEGRATION;
  } catch (const smc::CudaFailure& e) {
    g_error = e.what();
    return SMC_ECUDA;
  } catch (const std::exception& e) {
    g_error = e.what();
    return SMC_ECUDA;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw smc::InvalidArgument(std::string(what) + ": null pointer");
}

// Stage caller arrays to the device when they live on the host.
struct Staged {
  smc::DevBuf buf;
  const double* dev = nullptr;
  Staged(const double* p, long long n, int where, cudaStream_t st) {
    if (!p) return;
    if (where == SMC_DEVICE) {
      dev = p;
      return;
    }
    buf.resize(static_cast<std::size_t>(n));
    SMC_CUDA(cudaMemcpyAsync(buf.get(), p, n * sizeof(double), cudaMemcpyHostToDevice, st));
    dev = buf.get();
  }
};
struct StagedOut {
  smc::DevBuf buf;
  double* dev = nullptr;
  double* host = nullptr;
  long long n = 0;
  StagedOut(double* p, long long n_, int where) : n(n_) {
    if (!p) return;
    if (where == SMC_DEVICE) {
      dev = p;
      return;
    }
    buf.resize(static_cast<std::size_t>(n));
    dev = buf.get();
    host = p;
  }
  void finish(cudaStream_t st) {
    if (host)
      SMC_CUDA(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
};

void fill_diag(const smc::SweepDiag& d, smc_diag* out) {
  if (!out) return;
  out->sweeps = d.sweeps;
  out->fresh_evals = d.fresh_evals;
  out->f1_evals = d.f1_evals;
  out->f2_evals = d.f2_evals;
  out->early_stop = d.early_stop ? 1 : 0;
  out->nonfinite = d.nonfinite ? 1 : 0;
  out->n_residuals = static_cast<int>(d.residuals.size());
  out->implicit_solves = d.implicit_solves;
  out->newton_f1_evals = d.newton_f1_evals;
  if (out->residuals)
    for (int i = 0; i < out->residual_capacity && i < out->n_residuals; ++i)
      out->residuals[i] = d.residuals[i];
}

smc::RhsOp& op_of(smc_rhs* h) {
  need(h, "rhs handle");
  return *h->op;
}

}  // namespace

extern "C" {

int smc_version(void) { return 100; }
const char* smc_last_error(void) { return g_error.c_str(); }
long long smc_launch_count(void) { return smc::launch_counter().load(); }
int smc_synchronize(void) {
  return guarded([] { SMC_CUDA(cudaDeviceSynchronize()); });
}

// ------------------------------------------------------------- stencil
int smc_build_narrow(int order, const double* params, int nparams, double* m64, int* s) {
  return guarded([&] {
    need(params, "params");
    need(m64, "m64");
    smc::StencilM M = smc::make_stencil(order, params, nparams, s);
    std::memcpy(m64, &M.m[0][0], sizeof(double) * 64);
  });
}

int smc_apply_narrow(int order, const double* params, int nparams, const double* a,
                     const double* u, int n, double dx, double* out, int where) {
  return guarded([&] {
    need(a, "a"), need(u, "u"), need(out, "out");
    int s = 0;
    smc::StencilM M = smc::make_stencil(order, params, nparams, &s);
    smc::require(n >= 2 * s, "apply_narrow: grid too small for stencil");
    smc::require(dx > 0.0, "apply_narrow: dx must be positive");
    Staged da(a, n, where, nullptr), du(u, n, where, nullptr);
    StagedOut o(out, n, where);
    smc::NarrowArgs p;
    p.u = du.dev, p.cx = p.cy = p.cz = da.dev, p.out = o.dev;
    p.nx = n, p.ny = 1, p.nz = 1, p.dims = 1, p.kc = 1;
    p.idx2 = 1.0 / (dx * dx);
    smc::launch_narrow(p, s, M, nullptr);
    o.finish(nullptr);
    SMC_CUDA(cudaStreamSynchronize(nullptr));
  });
}

int smc_first_derivative8(const double* u, int n, double dx, double* out, int where) {
  return guarded([&] {
    need(u, "u"), need(out, "out");
    smc::require(n >= 9, "first_derivative8: need at least 9 points");
    smc::require(dx > 0.0, "first_derivative8: dx must be positive");
    Staged du(u, n, where, nullptr);
    StagedOut o(out, n, where);
    smc::launch_deriv8(du.dev, o.dev, n, 1, 1, 0, dx, nullptr);
    o.finish(nullptr);
    SMC_CUDA(cudaStreamSynchronize(nullptr));
  });
}

int smc_apply_narrow_bounded(const double* params, int nparams, const double* a, const double* u,
                             int n, int nlines, double dx, double* out, int where) {
  return guarded([&] {
    need(a, "a"), need(u, "u"), need(out, "out");
    smc::require(nparams == 0 || nparams == 2 || nparams == 3,
                 "apply_narrow_bounded: params are {} or {m47, m48} or {m47, m48, m36}");
    if (nparams) need(params, "params");
    const double p8[2] = {nparams ? params[0] : 3557.0 / 44100.0,
                          nparams ? params[1] : -2083.0 / 117600.0};
    const double p6[1] = {nparams == 3 ? params[2] : 281.0 / 3600.0};
    const smc::StencilM m8 = smc::make_stencil(8, p8, 2, nullptr);
    const smc::StencilM m6 = smc::make_stencil(6, p6, 1, nullptr);
    smc::require(n >= 8 && nlines >= 1, "apply_narrow_bounded: need n >= 8 and nlines >= 1");
    const long long total = static_cast<long long>(n) * nlines;
    Staged da(a, total, where, nullptr), du(u, total, where, nullptr);
    StagedOut o(out, total, where);
    smc::launch_narrow_bounded(m8, m6, da.dev, du.dev, o.dev, n, nlines, dx, nullptr);
    o.finish(nullptr);
    SMC_CUDA(cudaStreamSynchronize(nullptr));
  });
}

int smc_first_derivative_bounded(const double* u, int n, int nlines, double dx, double* out,
                                 int where) {
  return guarded([&] {
    need(u, "u"), need(out, "out");
    smc::require(n >= 8 && nlines >= 1,
                 "first_derivative_bounded: need n >= 8 and nlines >= 1");
    const long long total = static_cast<long long>(n) * nlines;
    Staged du(u, total, where, nullptr);
    StagedOut o(out, total, where);
    smc::launch_deriv_bounded(du.dev, o.dev, n, nlines, dx, nullptr);
    o.finish(nullptr);
    SMC_CUDA(cudaStreamSynchronize(nullptr));
  });
}

int smc_apply_wide(const double* a, const double* u, int n, double dx, double* out, int where) {
  return guarded([&] {
    need(a, "a"), need(u, "u"), need(out, "out");
    smc::require(n >= 9, "first_derivative8: need at least 9 points");
    smc::require(dx > 0.0, "first_derivative8: dx must be positive");
    Staged da(a, n, where, nullptr), du(u, n, where, nullptr);
    StagedOut o(out, n, where);
    smc::DevBuf w1(n);
    smc::launch_wide2d(du.dev, da.dev, nullptr, nullptr, 0.0, w1.get(), nullptr, o.dev, n, 1, dx,
                       1.0, nullptr);
    o.finish(nullptr);
    SMC_CUDA(cudaStreamSynchronize(nullptr));
  });
}

// ----------------------------------------------------------- operators
int smc_heat_create(int nx, int ny, int kind, const double* params, const double* a,
                    const double* b, const double* g0, smc_rhs** out) {
  return guarded([&] {
    need(out, "out");
    *out = nullptr;
    static const double zero[2] = {0.0, 0.0};
    auto h = std::make_unique<smc_rhs>();
    h->op = std::make_unique<smc::HeatOp>(nx, ny, kind, params ? params : zero, a, b, g0);
    *out = h.release();
  });
}

int smc_heat_set_time_source(smc_rhs* h, smc_time_fn g_time, void* ctx) {
  return guarded([&] {
    auto* op = dynamic_cast<smc::HeatOp*>(&op_of(h));
    smc::require(op != nullptr, "not a heat operator");
    op->set_time_source(g_time, ctx);
  });
}

int smc_heat_set_full_source(smc_rhs* h, smc_field_fn g_full, void* ctx) {
  return guarded([&] {
    auto* op = dynamic_cast<smc::HeatOp*>(&op_of(h));
    smc::require(op != nullptr, "not a heat operator");
    op->set_full_source(g_full, ctx);
  });
}

int smc_narrow3d_create(int nx, int ny, int nz, double dx, double dy, double dz, int order,
                        const double* params, int nparams, const double* a, int where,
                        smc_rhs** out) {
  return guarded([&] {
    need(out, "out");
    need(params, "params");
    *out = nullptr;
    auto h = std::make_unique<smc_rhs>();
    h->op = std::make_unique<smc::Narrow3DOp>(nx, ny, nz, dx, dy, dz, order, params, nparams, a,
                                              where);
    *out = h.release();
  });
}

int smc_narrow3d_create_slab(int nx, int ny, int nz, int zghost, double dx, double dy, double dz,
                             int order, const double* params, int nparams, const double* a,
                             int where, smc_rhs** out) {
  return guarded([&] {
    need(out, "out");
    need(params, "params");
    *out = nullptr;
    smc::require(zghost >= 1, "narrow3d slab: zghost must be positive");
    auto h = std::make_unique<smc_rhs>();
    h->op = std::make_unique<smc::Narrow3DOp>(nx, ny, nz, dx, dy, dz, order, params, nparams, a,
                                              where, zghost);
    *out = h.release();
  });
}

int smc_narrow3d_apply_planes(smc_rhs* h, const double* u, double* out, int kbeg, int kend) {
  return guarded([&] {
    auto* op = dynamic_cast<smc::Narrow3DOp*>(&op_of(h));
    smc::require(op != nullptr, "not a narrow3d operator");
    need(u, "u"), need(out, "out");
    op->eval_planes(u, out, kbeg, kend);
  });
}

int smc_narrow3d_apply_peer(smc_rhs* h, const double* u, const double* u_lo, int nz_lo,
                            const double* u_hi, double* out, int kbeg, int kend) {
  return guarded([&] {
    need(u, "u"), need(u_lo, "u_lo"), need(u_hi, "u_hi"), need(out, "out");
    auto* op = dynamic_cast<smc::Narrow3DOp*>(&op_of(h));
    if (!op) throw smc::InvalidArgument("smc_narrow3d_apply_peer: not a narrow3d operator");
    op->eval_planes_peer(u, u_lo, nz_lo, u_hi, out, kbeg, kend);
  });
}

int smc_ipc_export(const void* dptr, unsigned char* handle) {
  return guarded([&] {
    need(dptr, "dptr"), need(handle, "handle");
    cudaIpcMemHandle_t hd;
    SMC_CUDA(cudaIpcGetMemHandle(&hd, const_cast<void*>(dptr)));
    static_assert(sizeof(hd) == SMC_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &hd, sizeof(hd));
  });
}

int smc_ipc_import(const unsigned char* handle, void** dptr) {
  return guarded([&] {
    need(handle, "handle"), need(dptr, "dptr");
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle, sizeof(hd));
    SMC_CUDA(cudaIpcOpenMemHandle(dptr, hd, cudaIpcMemLazyEnablePeerAccess));
  });
}

int smc_ipc_close(void* dptr) {
  return guarded([&] { SMC_CUDA(cudaIpcCloseMemHandle(dptr)); });
}

int smc_device_alloc(long long nbytes, void** dptr) {
  return guarded([&] {
    need(dptr, "dptr");
    smc::require(nbytes > 0, "smc_device_alloc: size must be positive");
    SMC_CUDA(cudaMalloc(dptr, static_cast<std::size_t>(nbytes)));
  });
}

int smc_device_free(void* dptr) {
  return guarded([&] {
    if (dptr) SMC_CUDA(cudaFree(dptr));
  });
}

int smc_narrow3d_set_kc(smc_rhs* h, int kc) {
  return guarded([&] {
    auto* op = dynamic_cast<smc::Narrow3DOp*>(&op_of(h));
    smc::require(op != nullptr, "not a narrow3d operator");
    smc::require(kc >= 0, "kc must be >= 0");
    if (kc > 0) op->set_kc(kc);
  });
}

int smc_rhs_from_callback(long long dim, smc_rhs_fn f, void* ctx, smc_rhs** out) {
  return guarded([&] {
    need(out, "out");
    *out = nullptr;
    auto h = std::make_unique<smc_rhs>();
    h->op = std::make_unique<smc::HostCallbackOp>(dim, f, ctx);
    *out = h.release();
  });
}

int smc_rhs_from_device_callback(long long dim, smc_dev_rhs_fn f, void* ctx, smc_rhs** out) {
  return guarded([&] {
    need(out, "out");
    *out = nullptr;
    auto h = std::make_unique<smc_rhs>();
    h->op = std::make_unique<smc::DeviceCallbackOp>(dim, f, ctx);
    *out = h.release();
  });
}

int smc_rhs_eval(smc_rhs* h, double t, const double* u, double* out, int where) {
  return guarded([&] {
    need(u, "u"), need(out, "out");
    op_of(h).eval(t, u, out, where);
  });
}

long long smc_rhs_dim(const smc_rhs* h) { return h ? h->op->dim() : -1; }

int smc_rhs_set_stream(smc_rhs* h, void* stream) {
  return guarded([&] { op_of(h).set_stream(static_cast<cudaStream_t>(stream)); });
}

int smc_rhs_destroy(smc_rhs* h) {
  delete h;
  return SMC_OK;
}

// ------------------------------------------------------------ NS RHS
int smc_ns_create(int nx, int ny, int nz, int zghost, double dx, double dy, double dz, int order,
                  const double* params, int nparams, smc_rhs** full, smc_rhs** advdiff,
                  smc_rhs** chem) {
  return guarded([&] {
    need(params, "params");
    int s = 0;
    smc::StencilM M = smc::make_stencil(order, params, nparams, &s);
    smc::NsBox box;
    box.nx = nx, box.ny = ny, box.nz = nz, box.G = zghost;
    auto ws = std::make_shared<smc::NsWorkspace>(box, dx, dy, dz, M, s);
    smc_rhs** outs[3] = {full, advdiff, chem};
    for (int part = 0; part < 3; ++part) {
      if (!outs[part]) continue;
      auto h = std::make_unique<smc_rhs>();
      h->op = std::make_unique<smc::NsRhsOp>(ws, part);
      *outs[part] = h.release();
    }
  });
}

int smc_comm_unique_id(char* id128) {
  return guarded([&] {
    need(id128, "id");
    smc::nccl_unique_id(id128);
  });
}

int smc_comm_init(const char* id128, int nranks, int rank, smc_comm** out) {
  return guarded([&] {
    need(id128, "id"), need(out, "out");
    *out = nullptr;
    auto c = std::make_unique<smc_comm>();
    c->t = smc::make_nccl_transport(id128, nranks, rank);
    *out = c.release();
  });
}

int smc_comm_init_local(int nranks, smc_comm** out) {
  return guarded([&] {
    need(out, "out");
    auto group = smc::make_local_group(nranks);
    for (int r = 0; r < nranks; ++r) {
      auto c = std::make_unique<smc_comm>();
      c->t = group[r];
      out[r] = c.release();
    }
  });
}

int smc_comm_rank(const smc_comm* c, int* rank, int* size) {
  return guarded([&] {
    need(c, "comm"), need(rank, "rank"), need(size, "size");
    *rank = c->t->rank();
    *size = c->t->size();
  });
}

int smc_comm_allreduce_max(smc_comm* c, double* v) {
  return guarded([&] {
    need(c, "comm"), need(v, "v");
    *v = c->t->allreduce_max(*v, nullptr);
  });
}

int smc_comm_destroy(smc_comm* c) {
  delete c;
  return SMC_OK;
}

int smc_ns_slab_create(smc_comm* c, int nx, int ny, int nz, double dx, double dy, double dz,
                       int order, const double* params, int nparams, smc_rhs** full,
                       smc_rhs** advdiff, smc_rhs** chem) {
  return guarded([&] {
    need(c, "comm"), need(params, "params");
    int s = 0;
    smc::StencilM M = smc::make_stencil(order, params, nparams, &s);
    smc::NsBox box;
    box.nx = nx, box.ny = ny, box.nz = nz, box.G = 4;
    auto ws = std::make_shared<smc::NsWorkspace>(box, dx, dy, dz, M, s);
    smc_rhs** outs[3] = {full, advdiff, chem};
    for (int part = 0; part < 3; ++part) {
      if (!outs[part]) continue;
      auto h = std::make_unique<smc_rhs>();
      h->op = std::make_unique<smc::NsSlabOp>(c->t, ws, part);
      *outs[part] = h.release();
    }
  });
}

int smc_ns_slab_publish(smc_rhs* h, const double* u) {
  return guarded([&] {
    need(u, "u");
    auto* op = dynamic_cast<smc::NsSlabOp*>(&op_of(h));
    if (!op) throw smc::InvalidArgument("not an NS slab operator");
    op->publish(u);
  });
}

static smc::NsRhsOp& ns_of(smc_rhs* h) {
  auto* op = dynamic_cast<smc::NsRhsOp*>(&op_of(h));
  if (!op) throw smc::InvalidArgument("not an NS operator");
  return *op;
}

int smc_ns_rhs_ghosted(smc_rhs* h, const double* U, double* out) {
  return guarded([&] {
    need(U, "U"), need(out, "out");
    smc::NsRhsOp& op = ns_of(h);
    op.workspace().rhs(U, out, op.part(), op.stream());
  });
}

int smc_ns_profile(smc_rhs* h, const double* U, double* out, double* ms, const char** names,
                   int cap, int* count) {
  return guarded([&] {
    need(U, "U"), need(out, "out"), need(count, "count");
    smc::NsRhsOp& op = ns_of(h);
    cudaStream_t st = op.stream();
    smc::KernelMarks marks;
    SMC_CUDA(cudaEventCreate(&marks.start));
    SMC_CUDA(cudaEventRecord(marks.start, st));
    op.workspace().set_marks(&marks);
    try {
      op.eval_device(0.0, U, out);
    } catch (...) {
      op.workspace().set_marks(nullptr);
      throw;
    }
    op.workspace().set_marks(nullptr);
    SMC_CUDA(cudaStreamSynchronize(st));
    *count = static_cast<int>(marks.ev.size());
    cudaEvent_t prev = marks.start;
    for (int i = 0; i < *count && i < cap; ++i) {
      float t = 0.0f;
      SMC_CUDA(cudaEventElapsedTime(&t, prev, marks.ev[i].second));
      if (ms) ms[i] = t;
      if (names) names[i] = marks.ev[i].first;
      prev = marks.ev[i].second;
    }
  });
}

int smc_ns_temperature_pressure(smc_rhs* h, const double* U, double* T, double* p, int where) {
  return guarded([&] {
    need(U, "U"), need(T, "T"), need(p, "p");
    smc::NsRhsOp& op = ns_of(h);
    const smc::NsBox& b = op.workspace().box();
    cudaStream_t st = op.stream();
    Staged dU(U, SMC_NVAR * b.field_len(), where, st);
    StagedOut oT(T, b.cells(), where), op_(p, b.cells(), where);
    op.workspace().temperature_pressure(dU.dev, oT.dev, op_.dev, st);
    oT.finish(st), op_.finish(st);
    SMC_CUDA(cudaStreamSynchronize(st));
  });
}

int smc_ns_conserved(const double* T, const double* p, const double* uvw, const double* Y,
                     long long n, double* U, int where) {
  return guarded([&] {
    need(T, "T"), need(p, "p"), need(uvw, "uvw"), need(Y, "Y"), need(U, "U");
    Staged dT(T, n, where, nullptr), dp(p, n, where, nullptr), du(uvw, 3 * n, where, nullptr),
        dY(Y, SMC_NSP * n, where, nullptr);
    StagedOut oU(U, SMC_NVAR * n, where);
    smc::ns_conserved_from_primitives(dT.dev, dp.dev, du.dev, dY.dev, n, oU.dev, nullptr);
    oU.finish(nullptr);
    SMC_CUDA(cudaStreamSynchronize(nullptr));
  });
}

// ---------------------------------------------------------- quadrature
int smc_nodes(int family, int n, double* t) {
  return guarded([&] {
    need(t, "t");
    smc::Nodes s = smc::make_nodes(family, n);
    std::memcpy(t, s.t.data(), sizeof(double) * s.t.size());
  });
}

int smc_integration_matrices(int family, int n, double* q, double* s) {
  return guarded([&] {
    smc::SweepTables m = smc::integration_matrices(smc::make_nodes(family, n));
    if (q) std::memcpy(q, m.q.a.data(), sizeof(double) * m.q.a.size());
    if (s) std::memcpy(s, m.s.a.data(), sizeof(double) * m.s.a.size());
  });
}

int smc_build_hierarchy(int coarse_family, int coarse_nodes, int inner_family, int inner_nodes,
                        int repeats, int* m2p1, double* fine, double* q21, double* s21,
                        double* q22, double* s22, int* fine_of_coarse, int* p_map) {
  return guarded([&] {
    smc::Hierarchy h = smc::build_hierarchy(smc::make_nodes(coarse_family, coarse_nodes),
                                            smc::make_nodes(inner_family, inner_nodes), repeats);
    if (m2p1) *m2p1 = h.fine.count();
    auto put = [](const smc::Table& t, double* d) {
      if (d) std::memcpy(d, t.a.data(), sizeof(double) * t.a.size());
    };
    if (fine) std::memcpy(fine, h.fine.t.data(), sizeof(double) * h.fine.t.size());
    put(h.q21, q21), put(h.s21, s21), put(h.q22, q22), put(h.s22, s22);
    if (fine_of_coarse)
      std::memcpy(fine_of_coarse, h.fine_of_coarse.data(), sizeof(int) * h.fine_of_coarse.size());
    if (p_map) std::memcpy(p_map, h.p_map.data(), sizeof(int) * h.p_map.size());
  });
}

// ------------------------------------------------------------ steppers
int smc_sdc_create(int family, int num_nodes, int iterations, double cutoff, int reuse_first,
                   smc_sdc** out) {
  return guarded([&] {
    need(out, "out");
    *out = nullptr;
    auto s = std::make_unique<smc_sdc>();
    s->s = std::make_unique<smc::DeviceSdc>(smc::make_nodes(family, num_nodes), iterations, cutoff,
                                            reuse_first != 0);
    *out = s.release();
  });
}

int smc_sdc_set_reducer(smc_sdc* s, smc_reduce_fn fn, void* ctx) {
  return guarded([&] {
    need(s, "sdc handle");
    if (fn)
      s->s->set_reducer([fn, ctx](double v) { return fn(v, ctx); });
    else
      s->s->set_reducer(nullptr);
  });
}

int smc_sdc_step(smc_sdc* s, smc_rhs* f, const double* u0, double t_n, double dt,
                 const double* f0, double* u_out, double* f_end, int where, smc_diag* diag) {
  return guarded([&] {
    need(s, "sdc handle"), need(u0, "u0"), need(u_out, "u_out");
    smc::RhsOp& op = op_of(f);
    const long long n = op.dim();
    cudaStream_t st = op.stream();
    Staged du(u0, n, where, st), df0(f0, n, where, st);
    StagedOut ou(u_out, n, where), of(f_end, n, where);
    smc::SweepDiag d;
    s->s->step(op, du.dev, t_n, dt, df0.dev, ou.dev, of.dev, d);
    ou.finish(st);
    of.finish(st);
    if (where == SMC_HOST) SMC_CUDA(cudaStreamSynchronize(st));
    fill_diag(d, diag);
  });
}

int smc_sdc_integrate(smc_sdc* s, smc_rhs* f, const double* u0, double t0, double t1,
                      int nsteps, double* u_out, int where, smc_diag* diag) {
  return guarded([&] {
    need(s, "sdc handle"), need(u0, "u0"), need(u_out, "u_out");
    smc::RhsOp& op = op_of(f);
    const long long n = op.dim();
    cudaStream_t st = op.stream();
    Staged du(u0, n, where, st);
    StagedOut ou(u_out, n, where);
    smc::SweepDiag d;
    s->s->integrate(op, du.dev, t0, t1, nsteps, ou.dev, d);
    ou.finish(st);
    if (where == SMC_HOST) SMC_CUDA(cudaStreamSynchronize(st));
    fill_diag(d, diag);
  });
}

int smc_sdc_destroy(smc_sdc* s) {
  delete s;
  return SMC_OK;
}

int smc_mrsdc_create(int coarse_family, int coarse_nodes, int inner_family, int inner_nodes,
                     int repeats, int iterations, double cutoff, int reuse_first,
                     smc_mrsdc** out) {
  return guarded([&] {
    need(out, "out");
    *out = nullptr;
    auto m = std::make_unique<smc_mrsdc>();
    m->m = std::make_unique<smc::DeviceMrsdc>(
        smc::build_hierarchy(smc::make_nodes(coarse_family, coarse_nodes),
                             smc::make_nodes(inner_family, inner_nodes), repeats),
        iterations, cutoff, reuse_first != 0);
    *out = m.release();
  });
}

int smc_sdc_set_comm(smc_sdc* s, smc_comm* c) {
  return guarded([&] {
    need(s, "sdc handle"), need(c, "comm");
    std::shared_ptr<smc::HaloTransport> t = c->t;
    s->s->set_reducer([t](double v) { return t->allreduce_max(v, nullptr); });
  });
}

int smc_mrsdc_set_comm(smc_mrsdc* m, smc_comm* c) {
  return guarded([&] {
    need(m, "mrsdc handle"), need(c, "comm");
    std::shared_ptr<smc::HaloTransport> t = c->t;
    m->m->set_reducer([t](double v) { return t->allreduce_max(v, nullptr); });
  });
}

int smc_mrsdc_set_reducer(smc_mrsdc* m, smc_reduce_fn fn, void* ctx) {
  return guarded([&] {
    need(m, "mrsdc handle");
    if (fn)
      m->m->set_reducer([fn, ctx](double v) { return fn(v, ctx); });
    else
      m->m->set_reducer(nullptr);
  });
}

}  // extern "C"

namespace {

int mrsdc_step(int mode, smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0, double t_n,
               double dt, const double* f0_1, const double* f0_2, double* u_out, double* f1_end,
               double* f2_end, int where, smc_diag* diag) {
  return guarded([&] {
    need(m, "mrsdc handle"), need(u0, "u0"), need(u_out, "u_out");
    smc::RhsOp& a = op_of(f1);
    smc::RhsOp& b = op_of(f2);
    const long long n = a.dim();
    cudaStream_t st = b.stream();
    Staged du(u0, n, where, st), d1(f0_1, n, where, st), d2(f0_2, n, where, st);
    StagedOut ou(u_out, n, where), o1(f1_end, n, where), o2(f2_end, n, where);
    smc::SweepDiag d;
    if (mode == 2)
      m->m->step_mode2(a, b, du.dev, t_n, dt, d1.dev, d2.dev, ou.dev, o1.dev, o2.dev, d);
    else
      m->m->step_mode1(a, b, du.dev, t_n, dt, d1.dev, d2.dev, ou.dev, o1.dev, o2.dev, d);
    ou.finish(st), o1.finish(st), o2.finish(st);
    if (where == SMC_HOST) SMC_CUDA(cudaStreamSynchronize(st));
    fill_diag(d, diag);
  });
}

int mrsdc_integrate(int mode, smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0, double t0,
                    double t1, int nsteps, double* u_out, int where, smc_diag* diag) {
  return guarded([&] {
    need(m, "mrsdc handle"), need(u0, "u0"), need(u_out, "u_out");
    smc::RhsOp& a = op_of(f1);
    smc::RhsOp& b = op_of(f2);
    const long long n = a.dim();
    cudaStream_t st = b.stream();
    Staged du(u0, n, where, st);
    StagedOut ou(u_out, n, where);
    smc::SweepDiag d;
    if (mode == 2)
      m->m->integrate_mode2(a, b, du.dev, t0, t1, nsteps, ou.dev, d);
    else
      m->m->integrate_mode1(a, b, du.dev, t0, t1, nsteps, ou.dev, d);
    ou.finish(st);
    if (where == SMC_HOST) SMC_CUDA(cudaStreamSynchronize(st));
    fill_diag(d, diag);
  });
}

smc::StiffOpts stiff_of(const smc_stiff* o) {
  smc::StiffOpts s;
  if (o) {
    s.rtol = o->rtol, s.atol = o->atol, s.max_newton_iters = o->max_newton_iters;
    s.block = o->block, s.interleaved = o->interleaved;
    s.initial_step_fraction = o->initial_step_fraction;
  }
  smc::require(s.rtol >= 0.0 && s.atol >= 0.0, "StiffOptions: negative tolerance");
  smc::require(s.block >= 0, "StiffOptions: negative block size");
  return s;
}

}  // namespace

extern "C" {

int smc_mrsdc_step_mode1(smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0, double t_n,
                         double dt, const double* f0_1, const double* f0_2, double* u_out,
                         double* f1_end, double* f2_end, int where, smc_diag* diag) {
  return mrsdc_step(1, m, f1, f2, u0, t_n, dt, f0_1, f0_2, u_out, f1_end, f2_end, where, diag);
}

int smc_mrsdc_integrate_mode1(smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0,
                              double t0, double t1, int nsteps, double* u_out, int where,
                              smc_diag* diag) {
  return mrsdc_integrate(1, m, f1, f2, u0, t0, t1, nsteps, u_out, where, diag);
}

int smc_mrsdc_set_stiff(smc_mrsdc* m, const smc_stiff* opts) {
  return guarded([&] {
    need(m, "mrsdc handle");
    m->m->set_stiff(stiff_of(opts));
  });
}

int smc_mrsdc_step_mode2(smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0, double t_n,
                         double dt, const double* f0_1, const double* f0_2, double* u_out,
                         double* f1_end, double* f2_end, int where, smc_diag* diag) {
  return mrsdc_step(2, m, f1, f2, u0, t_n, dt, f0_1, f0_2, u_out, f1_end, f2_end, where, diag);
}

int smc_mrsdc_integrate_mode2(smc_mrsdc* m, smc_rhs* f1, smc_rhs* f2, const double* u0,
                              double t0, double t1, int nsteps, double* u_out, int where,
                              smc_diag* diag) {
  return mrsdc_integrate(2, m, f1, f2, u0, t0, t1, nsteps, u_out, where, diag);
}

int smc_integrate_stiff(smc_rhs* f, const double* u0, double t0, double t1, double* u_out,
                        int where, const smc_stiff* opts, int* accepted, int* rejected) {
  return guarded([&] {
    need(u0, "u0"), need(u_out, "u_out");
    smc::RhsOp& op = op_of(f);
    const long long n = op.dim();
    cudaStream_t st = op.stream();
    const smc::StiffOpts so = stiff_of(opts);
    Staged du(u0, n, where, st);
    StagedOut ou(u_out, n, where);
    smc::StiffStats stats;
    smc::integrate_stiff(op, du.dev, t0, t1, ou.dev, so, &stats);
    ou.finish(st);
    SMC_CUDA(cudaStreamSynchronize(st));
    if (accepted) *accepted = stats.accepted;
    if (rejected) *rejected = stats.rejected;
  });
}

int smc_solve_backward_euler(smc_rhs* f, double t, double beta, const double* c,
                             const double* guess, double* w, int where, const smc_stiff* opts,
                             smc_newton_report* report) {
  return guarded([&] {
    need(c, "c"), need(guess, "guess"), need(w, "w");
    smc::RhsOp& op = op_of(f);
    const long long n = op.dim();
    cudaStream_t st = op.stream();
    const smc::StiffOpts so = stiff_of(opts);
    Staged dc(c, n, where, st), dg(guess, n, where, st);
    StagedOut ow(w, n, where);
    smc::DeviceNewton newton;
    smc::NewtonReport rep;
    newton.solve(op, t, beta, dc.dev, dg.dev, ow.dev, so, rep);
    ow.finish(st);
    SMC_CUDA(cudaStreamSynchronize(st));
    if (report) {
      report->iterations = rep.iterations;
      report->final_residual = rep.final_residual;
      report->converged = rep.converged ? 1 : 0;
      report->f_evals = rep.f_evals;
    } else if (!rep.converged) {
      throw smc::IntegrationFailure("backward-Euler Newton failed: residual " +
                                    std::to_string(rep.final_residual) + " after " +
                                    std::to_string(rep.iterations) + " iterations");
    }
  });
}

int smc_mrsdc_destroy(smc_mrsdc* m) {
  delete m;
  return SMC_OK;
}

}  // extern "C"
