// Right-hand-side operators behind the C ABI.  Each one implements the
// reference's `nsdc::Rhs` contract (proj/core/include/nsdc/field.hpp:14-16:
// "writes f(t, u) into out ... out may alias nothing") on device buffers.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace smc {

// Owning device buffer of doubles.
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t n) { resize(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_, n_ = o.n_;
      o.p_ = nullptr, o.n_ = 0;
    }
    return *this;
  }
  void resize(std::size_t n) {
    if (n == n_) return;
    release();
    if (n) SMC_CUDA(cudaMalloc(&p_, n * sizeof(double)));
    n_ = n;
  }
  double* get() const { return p_; }
  std::size_t size() const { return n_; }

 private:
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  double* p_ = nullptr;
  std::size_t n_ = 0;
};

enum Where : int { kHost = 0, kDevice = 1 };

// Global max over ranks of a per-rank value (identity on one rank): the
// residual max-norms of the sweeps (sdc.cpp:20-30, mrsdc.cpp:23-35) and the
// Newton / step-control norms of the implicit solver (stiff.cpp:49-66).
using Reducer = std::function<double(double)>;

class RhsOp {
 public:
  virtual ~RhsOp() = default;
  virtual long long dim() const = 0;
  // out = f(t, u) on device buffers, stream-ordered on stream().
  virtual void eval_device(double t, const double* u, double* out) = 0;
  virtual const char* name() const = 0;

  // Host or device pointers; host calls stage through owned buffers and
  // synchronize before returning.
  void eval(double t, const double* u, double* out, int where);
  // Host-pointer evaluation (default: copy in, evaluate, copy out).
  virtual void eval_host(double t, const double* u, double* out);

  cudaStream_t stream() const { return stream_; }
  void set_stream(cudaStream_t s) { stream_ = s; }
  long long evals() const { return evals_; }

  // Optional fused finite-difference block Jacobian for DeviceNewton
  // (stiff.cpp:16-30 per block): jac[(r * block + j) * nb + b] =
  // (f(w + h e_j)_r - fw_r) * (1 / h), h = root_eps * max(|w_j|, atol), for
  // every block b of a block-local f, the same bits as perturbing column j of
  // every block and evaluating f.  Returns false when the operator has no
  // fused form for this layout (the caller then runs the column loop).
  virtual bool fd_block_jacobian(const double* /*w*/, const double* /*fw*/, double* /*jac*/,
                                 long long /*block*/, int /*interleaved*/, double /*atol*/,
                                 double /*root_eps*/) {
    return false;
  }

  // Optional fused sweep update + evaluation (MRSDC's fine nodes):
  // next = cur + sum_{d < nd} dc_d (da_d - db_d) + pre elementwise, with the
  // arithmetic of sweep_update_kernel<nd, 0>, then out = f(t, next), in one
  // pass for a pointwise f.  Returns false when the operator has no fused
  // form (the caller then launches the update and evaluates).
  virtual bool eval_after_update(double /*t*/, double* /*next*/, const double* /*cur*/,
                                 int /*nd*/, const double* const* /*da*/,
                                 const double* const* /*db*/, const double* /*dc*/,
                                 const double* /*pre*/, double* /*out*/) {
    return false;
  }

 protected:
  cudaStream_t stream_ = nullptr;
  long long evals_ = 0;
  DevBuf stage_u_, stage_out_;
};

// configs[1]: (a U_x)_x + (a U_y)_y + (a U_z)_z on a periodic box.
class Narrow3DOp final : public RhsOp {
 public:
  // zghost == 0: periodic box, arrays hold nz planes.  zghost >= S: a and u
  // carry zghost ghost planes below and above the nz interior planes (a
  // z-slab of a decomposed box, ghosts filled by the halo exchange); out
  // holds the nz interior planes.
  Narrow3DOp(int nx, int ny, int nz, double dx, double dy, double dz, int order,
             const double* params, int nparams, const double* a, int where, int zghost = 0);
  long long dim() const override { return static_cast<long long>(nx_) * ny_ * nz_; }
  void eval_device(double t, const double* u, double* out) override;
  const char* name() const override { return "narrow3d"; }
  void set_kc(int kc) { kc_ = kc; }
  int kc() const { return kc_; }
  int s() const { return s_; }
  int zghost() const { return zghost_; }
  // interior planes [kb, ke) only (overlap of halo exchange and compute)
  void eval_planes(const double* u, double* out, int kb, int ke);
  // slab operator, peer halo: u holds the nz interior planes, the S planes
  // below / above are read from the neighbours' interior arrays u_lo (nz_lo
  // planes) and u_hi in the kernel itself
  void eval_planes_peer(const double* u, const double* u_lo, int nz_lo, const double* u_hi,
                        double* out, int kb, int ke);
  // Host buffers: z-chunked pipeline, so the host->device copy of chunk c+1,
  // the stencil on chunk c and the device->host copy of chunk c-1 overlap
  // (the link is full duplex; the kernel is ~10x faster than either copy).
  void eval_host(double t, const double* u, double* out) override;
  ~Narrow3DOp() override;

 private:
  int nx_, ny_, nz_, s_ = 4, kc_ = 8, zghost_ = 0;
  double dx_, dy_, dz_;
  StencilM M_{};
  DevBuf a_;
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr;
  std::vector<cudaEvent_t> ev_in_, ev_done_;
};

// HeatOperator (proj/core/include/nsdc/pde.hpp:69-84): u_t = (a u_x)_x +
// (b u_y)_y + g on the periodic [0, 2pi)^2 grid, narrow8 / narrow6 / wide.
class HeatOp final : public RhsOp {
 public:
  using GTime = double (*)(double t, void* ctx);
  using GFull = void (*)(double t, double* field, void* ctx);

  HeatOp(int nx, int ny, int kind, const double* params, const double* a, const double* b,
         const double* g0);
  long long dim() const override { return static_cast<long long>(nx_) * ny_; }
  void eval_device(double t, const double* u, double* out) override;
  const char* name() const override { return "heat2d"; }
  void set_time_source(GTime f, void* ctx) { gtime_ = f, gtime_ctx_ = ctx; }
  void set_full_source(GFull f, void* ctx) { gfull_ = f, gfull_ctx_ = ctx; }

 private:
  int nx_, ny_, kind_, s_ = 0;
  StencilM M_{};
  DevBuf a_, b_, g0_, w1_, w2_, gfull_dev_;
  std::vector<double> gfull_host_;
  bool has_g0_ = false;
  GTime gtime_ = nullptr;
  void* gtime_ctx_ = nullptr;
  GFull gfull_ = nullptr;
  void* gfull_ctx_ = nullptr;
};

// A host callback wrapped as an operator (for ODE-sized problems and for
// driving the device steppers with any nsdc::Rhs, e.g. the reference's own).
class HostCallbackOp final : public RhsOp {
 public:
  using Cb = void (*)(double t, const double* u, double* out, long long n, void* ctx);
  HostCallbackOp(long long dim, Cb cb, void* ctx);
  long long dim() const override { return dim_; }
  void eval_device(double t, const double* u, double* out) override;
  const char* name() const override { return "host_callback"; }

 private:
  long long dim_;
  Cb cb_;
  void* ctx_;
  std::vector<double> hu_, ho_;
};

// A callback that computes on device buffers itself (e.g. a multi-GPU RHS
// whose halo exchange runs through torch.distributed / NCCL on the host).
class DeviceCallbackOp final : public RhsOp {
 public:
  using Cb = void (*)(double t, const double* u, double* out, long long n, void* stream,
                      void* ctx);
  DeviceCallbackOp(long long dim, Cb cb, void* ctx) : dim_(dim), cb_(cb), ctx_(ctx) {
    require(dim >= 1, "device callback rhs: dim must be positive");
    require(cb != nullptr, "device callback rhs: null callback");
  }
  long long dim() const override { return dim_; }
  void eval_device(double t, const double* u, double* out) override {
    cb_(t, u, out, dim_, static_cast<void*>(stream_), ctx_);
    ++evals_;
  }
  const char* name() const override { return "device_callback"; }

 private:
  long long dim_;
  Cb cb_;
  void* ctx_;
};

StencilM make_stencil(int order, const double* params, int nparams, int* s);
int num_sms();

}  // namespace smc
