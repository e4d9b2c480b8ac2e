#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "narrow.cuh"
#include "ops.hpp"

namespace smc {

// ------------------------------------------------------- coupling matrix
// M(i, j) = c + p*m47 + q*m48 for rows 1..s (order 8) or
// c + p*m36 (order 6); the lower rows follow from the
// central antisymmetry M(i, j) = -M(2s+1-i, 2s+1-j).  Equivalent to
// nsdc::build_narrow (proj/core/src/stencil.cpp:117-132).
namespace {
struct Aff {
  double c, p, q;
};
constexpr Aff kM8[4][8] = {
    {{5.0 / 336, 0, 1}, {-83.0 / 3600, -1.0 / 5, -14.0 / 5}, {299.0 / 50400, 2.0 / 5, 13.0 / 5},
     {17.0 / 12600, -1.0 / 5, -4.0 / 5}, {1.0 / 1120, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    {{-11.0 / 560, 0, -2}, {-31.0 / 360, 1, 3}, {41.0 / 200, -9.0 / 5, 4.0 / 5},
     {-5927.0 / 50400, 4.0 / 5, -9.0 / 5}, {17.0 / 600, -1.0 / 5, -4.0 / 5},
     {-503.0 / 50400, 1.0 / 5, 4.0 / 5}, {0, 0, 0}, {0, 0, 0}},
    {{-1.0 / 280, 0, 0}, {1097.0 / 5040, -2, 6}, {-1349.0 / 10080, 3, -12},
     {-887.0 / 5040, -1, 6}, {3613.0 / 50400, 4.0 / 5, -9.0 / 5},
     {467.0 / 25200, -3.0 / 5, 18.0 / 5}, {139.0 / 25200, -1.0 / 5, -9.0 / 5}, {0, 0, 0}},
    {{17.0 / 1680, 0, 2}, {-319.0 / 2520, 2, -8}, {-919.0 / 5040, -2, 6}, {-445.0 / 2016, 0, 0},
     {583.0 / 720, -1, 6}, {-65.0 / 224, 0, -7}, {0, 1, 0}, {0, 0, 1}},
};
constexpr Aff kM6[3][6] = {
    {{-11.0 / 180, 1, 0}, {1.0 / 9, -2, 0}, {-1.0 / 18, 1, 0}, {1.0 / 180, 0, 0}, {0, 0, 0},
     {0, 0, 0}},
    {{7.0 / 60, -3, 0}, {-1.0 / 120, 5, 0}, {-17.0 / 90, -2, 0}, {5.0 / 72, 1, 0},
     {1.0 / 90, -1, 0}, {0, 0, 0}},
    {{-1.0 / 15, 3, 0}, {-11.0 / 60, -3, 0}, {-101.0 / 360, 0, 0}, {137.0 / 180, -2, 0},
     {-83.0 / 360, 1, 0}, {0, 1, 0}},
};
}  // namespace

StencilM make_stencil(int order, const double* params, int nparams, int* s_out) {
  if (order == 8)
    require(nparams == 2, "order 8 takes two parameters {m47, m48}");
  else if (order == 6)
    require(nparams == 1, "order 6 takes one parameter {m36}");
  else
    throw InvalidArgument("stencil order must be 6 or 8, got " + std::to_string(order));
  StencilM M{};
  const int s = order == 8 ? 4 : 3;
  const double x = params[0], y = order == 8 ? params[1] : 0.0;
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < 2 * s; ++j) {
      const Aff& t = order == 8 ? kM8[i][j] : kM6[i][j];
      const double v = t.c + t.p * x + t.q * y;
      M.m[i][j] = v;
      M.m[2 * s - 1 - i][2 * s - 1 - j] = -v;
    }
  for (int r = 0; r < s; ++r)
    for (int j = 0; j < s; ++j) {
      M.p[r][j] = 0.5 * (M.m[r][j] + M.m[r][2 * s - 1 - j]);
      M.q[r][j] = 0.5 * (M.m[r][j] - M.m[r][2 * s - 1 - j]);
    }
  if (s_out) *s_out = s;
  return M;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    SMC_CUDA(cudaGetDevice(&dev));
    SMC_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

// ------------------------------------------------------------------ RhsOp
void RhsOp::eval(double t, const double* u, double* out, int where) {
  if (where == kDevice)
    eval_device(t, u, out);
  else
    eval_host(t, u, out);
}

void RhsOp::eval_host(double t, const double* u, double* out) {
  const std::size_t n = static_cast<std::size_t>(dim());
  stage_u_.resize(n);
  stage_out_.resize(n);
  SMC_CUDA(cudaMemcpyAsync(stage_u_.get(), u, n * sizeof(double), cudaMemcpyHostToDevice, stream_));
  eval_device(t, stage_u_.get(), stage_out_.get());
  SMC_CUDA(cudaMemcpyAsync(out, stage_out_.get(), n * sizeof(double), cudaMemcpyDeviceToHost,
                           stream_));
  SMC_CUDA(cudaStreamSynchronize(stream_));
}

// ------------------------------------------------------------- Narrow3D
Narrow3DOp::Narrow3DOp(int nx, int ny, int nz, double dx, double dy, double dz, int order,
                       const double* params, int nparams, const double* a, int where,
                       int zghost)
    : nx_(nx), ny_(ny), nz_(nz), zghost_(zghost), dx_(dx), dy_(dy), dz_(dz) {
  M_ = make_stencil(order, params, nparams, &s_);
  require(nx >= 2 * s_ && ny >= 2 * s_ && nz >= (zghost ? 1 : 2 * s_),
          "narrow3d: grid too small for the chosen stencil");
  require(zghost == 0 || zghost >= s_, "narrow3d: need at least S ghost planes");
  require(dx > 0 && dy > 0 && dz > 0, "narrow3d: spacings must be positive");
  require(a != nullptr, "narrow3d: coefficient field required");
  const std::size_t na = static_cast<std::size_t>(nx) * ny * (nz + 2 * zghost);
  a_.resize(na);
  SMC_CUDA(cudaMemcpy(a_.get(), a, na * sizeof(double),
                      where == kDevice ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  kc_ = narrow_default_kc(nx, ny, nz, 3, num_sms());
}

void Narrow3DOp::eval_planes(const double* u, double* out, int kb, int ke) {
  const long long plane = static_cast<long long>(nx_) * ny_;
  NarrowArgs p;
  p.u = u + zghost_ * plane;
  p.cx = p.cy = p.cz = a_.get() + zghost_ * plane;
  p.out = out;
  p.nx = nx_, p.ny = ny_, p.nz = nz_;
  p.dims = 3;
  p.kc = kc_;
  p.kbeg = kb, p.kend = ke;
  p.zwrap = zghost_ == 0;
  p.idx2 = 1.0 / (dx_ * dx_), p.idy2 = 1.0 / (dy_ * dy_), p.idz2 = 1.0 / (dz_ * dz_);
  launch_narrow(p, s_, M_, stream_);
}

void Narrow3DOp::eval_planes_peer(const double* u, const double* u_lo, int nz_lo,
                                  const double* u_hi, double* out, int kb, int ke) {
  require(zghost_ >= s_, "narrow3d: the peer halo needs a slab operator");
  require(nz_lo >= s_, "narrow3d: the lower neighbour holds fewer than S planes");
  require(nz_ >= s_, "narrow3d: the peer halo needs at least S interior planes");
  const long long plane = static_cast<long long>(nx_) * ny_;
  NarrowArgs p;
  p.u = u;
  p.cx = p.cy = p.cz = a_.get() + zghost_ * plane;
  p.out = out;
  p.nx = nx_, p.ny = ny_, p.nz = nz_;
  p.dims = 3;
  p.kc = kc_;
  p.kbeg = kb, p.kend = ke;
  p.zwrap = false;
  p.zpeer = true;
  p.u_lo = u_lo, p.u_hi = u_hi, p.lo_len = nz_lo * plane;
  p.idx2 = 1.0 / (dx_ * dx_), p.idy2 = 1.0 / (dy_ * dy_), p.idz2 = 1.0 / (dz_ * dz_);
  launch_narrow(p, s_, M_, stream_);
}

void Narrow3DOp::eval_device(double, const double* u, double* out) {
  require(zghost_ == 0, "narrow3d: a ghosted (slab) operator is applied with apply_planes");
  eval_planes(u, out, 0, nz_);
  ++evals_;
}

Narrow3DOp::~Narrow3DOp() {
  for (cudaEvent_t e : ev_in_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_done_) cudaEventDestroy(e);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (d2h_) cudaStreamDestroy(d2h_);
}

void Narrow3DOp::eval_host(double t, const double* u, double* out) {
  require(zghost_ == 0, "narrow3d: a ghosted (slab) operator is applied with apply_planes");
  // Chunk boundaries: short chunks at both ends (the pipeline's fill and
  // drain are one chunk each), SMC_E2E_CHUNK_PLANES (default 32) planes in
  // the middle; every chunk holds >= 8 >= S planes.
  static const int mid_planes = [] {
    const char* e = std::getenv("SMC_E2E_CHUNK_PLANES");
    return e ? std::max(8, std::atoi(e)) : 32;
  }();
  std::vector<int> bnd{0};
  if (nz_ >= 48 + mid_planes) {
    bnd.push_back(8);
    bnd.push_back(24);
    const int mid = nz_ - 48, nm = (mid + mid_planes - 1) / mid_planes;
    for (int i = 1; i <= nm; ++i) bnd.push_back(24 + static_cast<int>((1LL * mid * i) / nm));
    bnd.push_back(nz_ - 8);
    bnd.push_back(nz_);
  } else {
    const int n = std::min(8, nz_ / 8);
    for (int i = 1; i <= n; ++i) bnd.push_back(static_cast<int>((1LL * nz_ * i) / std::max(n, 1)));
  }
  const int nchunk = static_cast<int>(bnd.size()) - 1;
  if (nchunk < 2) {
    RhsOp::eval_host(t, u, out);
    return;
  }
  const std::size_t plane = static_cast<std::size_t>(nx_) * ny_;
  stage_u_.resize(plane * nz_);
  stage_out_.resize(plane * nz_);
  if (!h2d_) {
    SMC_CUDA(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
    SMC_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
  }
  while (static_cast<int>(ev_in_.size()) < nchunk) {
    cudaEvent_t a, b;
    SMC_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    SMC_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    ev_in_.push_back(a);
    ev_done_.push_back(b);
  }
  auto lo = [&](int c) { return bnd[c]; };
  auto h2d = [&](int k0, int k1) {
    const std::size_t off = plane * k0, cnt = plane * (k1 - k0);
    SMC_CUDA(cudaMemcpyAsync(stage_u_.get() + off, u + off, cnt * sizeof(double),
                             cudaMemcpyHostToDevice, h2d_));
  };
  // Host->device: first the top S planes (the periodic neighbours of plane
  // 0), then the chunks in order.  Once chunk c is resident, interior planes
  // [lo(c) - S, lo(c+1) - S) have their whole stencil (the last range runs to
  // nz and wraps onto chunk 0), so the stencil lags the copy by S planes and
  // the device->host copy of each range starts as soon as it is computed.
  // Enqueue order: per chunk in pipeline order (copy in, stencil, copy out
  // of the previous chunk) by default.  SMC_E2E_ORDER=0 enqueues all copies
  // in, then all stencils, then all copies out: the same dependencies, but in
  // some processes the two copy directions then stopped overlapping (4.5-4.8
  // ms per call instead of 3.4; measured in 2 of 3 fresh processes at 64-plane
  // chunks); the pipeline order ran 3.35-3.38 ms in 9 of 9.
  static const int order = [] {
    const char* e = std::getenv("SMC_E2E_ORDER");
    return e ? std::atoi(e) : 1;
  }();
  auto range = [&](int c, int& k0, int& k1) {
    k0 = c == 0 ? 0 : lo(c) - s_;
    k1 = c == nchunk - 1 ? nz_ : lo(c + 1) - s_;
  };
  auto in = [&](int c) {
    h2d(lo(c), c == nchunk - 1 ? nz_ - s_ : lo(c + 1));
    SMC_CUDA(cudaEventRecord(ev_in_[c], h2d_));
  };
  auto compute = [&](int c) {
    int k0, k1;
    range(c, k0, k1);
    SMC_CUDA(cudaStreamWaitEvent(stream_, ev_in_[c], 0));
    eval_planes(stage_u_.get(), stage_out_.get(), k0, k1);
    SMC_CUDA(cudaEventRecord(ev_done_[c], stream_));
  };
  auto outc = [&](int c) {
    int k0, k1;
    range(c, k0, k1);
    SMC_CUDA(cudaStreamWaitEvent(d2h_, ev_done_[c], 0));
    const std::size_t off = plane * k0, cnt = plane * (k1 - k0);
    SMC_CUDA(cudaMemcpyAsync(out + off, stage_out_.get() + off, cnt * sizeof(double),
                             cudaMemcpyDeviceToHost, d2h_));
  };
  h2d(nz_ - s_, nz_);
  if (order == 1) {
    // per chunk, in pipeline order
    for (int c = 0; c < nchunk; ++c) {
      in(c);
      compute(c);
      if (c > 0) outc(c - 1);
    }
    outc(nchunk - 1);
  } else {
    for (int c = 0; c < nchunk; ++c) in(c);
    for (int c = 0; c < nchunk; ++c) compute(c);
    for (int c = 0; c < nchunk; ++c) outc(c);
  }
  SMC_CUDA(cudaStreamSynchronize(d2h_));
  ++evals_;
}

// ----------------------------------------------------------------- Heat
HeatOp::HeatOp(int nx, int ny, int kind, const double* params, const double* a, const double* b,
               const double* g0)
    : nx_(nx), ny_(ny), kind_(kind) {
  require(kind >= 0 && kind <= 2, "HeatOperator: stencil kind must be narrow8, narrow6 or wide8");
  if (kind == 0)
    M_ = make_stencil(8, params, 2, &s_);
  else if (kind == 1)
    M_ = make_stencil(6, params, 1, &s_);
  const int min_n = kind == 2 ? 9 : 2 * s_ + 1;  // pde.cpp:227-229
  require(nx >= min_n && ny >= min_n, "HeatOperator: grid too small for the chosen stencil");
  require(a && b, "HeatOperator: incomplete problem");
  const std::size_t n = static_cast<std::size_t>(nx) * ny;
  for (std::size_t i = 0; i < n; ++i)
    require(a[i] > 0.0, "HeatOperator: coefficient a not positive");
  for (std::size_t i = 0; i < n; ++i)
    require(b[i] > 0.0, "HeatOperator: coefficient b not positive");
  a_.resize(n);
  b_.resize(n);
  SMC_CUDA(cudaMemcpy(a_.get(), a, n * sizeof(double), cudaMemcpyHostToDevice));
  SMC_CUDA(cudaMemcpy(b_.get(), b, n * sizeof(double), cudaMemcpyHostToDevice));
  if (g0) {
    g0_.resize(n);
    SMC_CUDA(cudaMemcpy(g0_.get(), g0, n * sizeof(double), cudaMemcpyHostToDevice));
    has_g0_ = true;
  }
  if (kind == 2) {
    w1_.resize(n);
    w2_.resize(n);
  }
}

void HeatOp::eval_device(double t, const double* u, double* out) {
  const double two_pi = 2.0 * 3.14159265358979323846;
  const double dx = two_pi / nx_, dy = two_pi / ny_;  // Grid2D (pde.cpp:16-19)
  const double* src = nullptr;
  double gt = 0.0;
  if (has_g0_ && gtime_) {
    src = g0_.get();
    gt = gtime_(t, gtime_ctx_);
  } else if (gfull_) {
    // non-separable source: the user's callback is host code; evaluate it on
    // the grid and upload (pde.cpp:124-126 calls it per cell per RHS).
    const std::size_t n = static_cast<std::size_t>(dim());
    gfull_host_.resize(n);
    gfull_dev_.resize(n);
    gfull_(t, gfull_host_.data(), gfull_ctx_);
    SMC_CUDA(cudaMemcpyAsync(gfull_dev_.get(), gfull_host_.data(), n * sizeof(double),
                             cudaMemcpyHostToDevice, stream_));
    SMC_CUDA(cudaStreamSynchronize(stream_));
    src = gfull_dev_.get();
    gt = 1.0;
  }
  if (kind_ == 2) {
    launch_wide2d(u, a_.get(), b_.get(), src, gt, w1_.get(), w2_.get(), out, nx_, ny_, dx, dy,
                  stream_);
  } else {
    NarrowArgs p;
    p.u = u;
    p.cx = a_.get();
    p.cy = b_.get();
    p.cz = nullptr;
    p.g0 = src;
    p.gt = gt;
    p.out = out;
    p.nx = nx_, p.ny = ny_, p.nz = 1;
    p.dims = 2;
    p.kc = 1;
    p.idx2 = 1.0 / (dx * dx), p.idy2 = 1.0 / (dy * dy);
    launch_narrow(p, s_, M_, stream_);
  }
  ++evals_;
}

// ---------------------------------------------------------- HostCallback
HostCallbackOp::HostCallbackOp(long long dim, Cb cb, void* ctx) : dim_(dim), cb_(cb), ctx_(ctx) {
  require(dim >= 1, "host callback rhs: dim must be positive");
  require(cb != nullptr, "host callback rhs: null callback");
}

void HostCallbackOp::eval_device(double t, const double* u, double* out) {
  const std::size_t n = static_cast<std::size_t>(dim_);
  hu_.resize(n);
  ho_.resize(n);
  SMC_CUDA(cudaMemcpyAsync(hu_.data(), u, n * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  SMC_CUDA(cudaStreamSynchronize(stream_));
  cb_(t, hu_.data(), ho_.data(), dim_, ctx_);
  SMC_CUDA(cudaMemcpyAsync(out, ho_.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream_));
  SMC_CUDA(cudaStreamSynchronize(stream_));
  ++evals_;
}

}  // namespace smc
