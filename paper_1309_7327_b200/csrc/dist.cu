// z-slab decomposition of the NS box: halo transports and the slab RHS
// (see dist.hpp).
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "dist.hpp"

namespace smc {

// ------------------------------------------------------------------ NCCL
// The few entry points used, resolved from libnccl.so.2 at run time (in a
// process that already loaded NCCL, e.g. through torch, dlopen returns that
// copy).  Types as in nccl.h.
namespace {

using ncclComm_t = struct ncclComm*;
using ncclResult_t = int;
constexpr int kNcclSuccess = 0;
constexpr int kNcclDouble = 8;  // ncclFloat64
constexpr int kNcclMax = 2;     // ncclMax
struct ncclUniqueId {
  char internal[128];
};

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) n.error = std::string("libnccl.so.2 lacks ") + name;
    };
    sym(n.GetUniqueId, "ncclGetUniqueId");
    sym(n.CommInitRank, "ncclCommInitRank");
    sym(n.CommDestroy, "ncclCommDestroy");
    sym(n.GroupStart, "ncclGroupStart");
    sym(n.GroupEnd, "ncclGroupEnd");
    sym(n.Send, "ncclSend");
    sym(n.Recv, "ncclRecv");
    sym(n.AllReduce, "ncclAllReduce");
    sym(n.GetErrorString, "ncclGetErrorString");
    n.ok = n.error.empty();
  });
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != kNcclSuccess)
    throw CudaFailure(std::string(what) + ": " + nccl().GetErrorString(r));
}

const Nccl& nccl_or_throw() {
  const Nccl& n = nccl();
  if (!n.ok) throw CudaFailure(n.error);
  return n;
}

class NcclTransport final : public HaloTransport {
 public:
  NcclTransport(const char* id, int nranks, int rank) : rank_(rank), size_(nranks) {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "comm: bad rank / size");
    const Nccl& n = nccl_or_throw();
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    nccl_check(n.CommInitRank(&comm_, nranks, uid, rank), "ncclCommInitRank");
    SMC_CUDA(cudaMalloc(&slot_, sizeof(double)));
  }
  ~NcclTransport() override {
    if (slot_) cudaFree(slot_);
    if (comm_) nccl().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void exchange(const double* u, long long ufs, double* lo, double* hi, long long plane, int G,
                int nz, int nvar, cudaStream_t st) override {
    const Nccl& n = nccl();
    const size_t cnt = static_cast<size_t>(G) * plane;
    const long long hs = G * plane;
    // per field: up (top planes -> next, prev's top -> lo), then down; with
    // prev == next (two ranks, or one) the k-th send to a peer meets the
    // k-th receive from it, so the order matches the planes' roles
    nccl_check(n.GroupStart(), "ncclGroupStart");
    for (int v = 0; v < nvar; ++v) {
      const double* uv = u + v * ufs;
      nccl_check(n.Send(uv + (nz - G) * plane, cnt, kNcclDouble, next(), comm_, st), "ncclSend");
      nccl_check(n.Recv(lo + v * hs, cnt, kNcclDouble, prev(), comm_, st), "ncclRecv");
      nccl_check(n.Send(uv, cnt, kNcclDouble, prev(), comm_, st), "ncclSend");
      nccl_check(n.Recv(hi + v * hs, cnt, kNcclDouble, next(), comm_, st), "ncclRecv");
    }
    nccl_check(n.GroupEnd(), "ncclGroupEnd");
  }
  double allreduce_max(double v, cudaStream_t st) override {
    SMC_CUDA(cudaMemcpyAsync(slot_, &v, sizeof(double), cudaMemcpyHostToDevice, st));
    nccl_check(nccl().AllReduce(slot_, slot_, 1, kNcclDouble, kNcclMax, comm_, st),
               "ncclAllReduce");
    double r = 0.0;
    SMC_CUDA(cudaMemcpyAsync(&r, slot_, sizeof(double), cudaMemcpyDeviceToHost, st));
    SMC_CUDA(cudaStreamSynchronize(st));
    return r;
  }

 private:
  int rank_, size_;
  ncclComm_t comm_ = nullptr;
  double* slot_ = nullptr;
};

// ------------------------------------------------------- in-process group
struct LocalGroup {
  std::vector<const double*> u;
  std::vector<long long> ufs;
};

class LocalTransport final : public HaloTransport {
 public:
  LocalTransport(std::shared_ptr<LocalGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
  int rank() const override { return rank_; }
  int size() const override { return static_cast<int>(g_->u.size()); }
  void publish(const double* u, long long ufs) override {
    g_->u[rank_] = u;
    g_->ufs[rank_] = ufs;
  }
  void exchange(const double* u, long long ufs, double* lo, double* hi, long long plane, int G,
                int nz, int nvar, cudaStream_t st) override {
    publish(u, ufs);
    const double* up = g_->u[prev()];
    const double* un = g_->u[next()];
    require(up && un, "local comm: a neighbour has not published its state");
    const size_t bytes = sizeof(double) * G * plane;
    for (int v = 0; v < nvar; ++v) {
      SMC_CUDA(cudaMemcpyAsync(lo + v * G * plane, up + v * g_->ufs[prev()] + (nz - G) * plane,
                               bytes, cudaMemcpyDeviceToDevice, st));
      SMC_CUDA(cudaMemcpyAsync(hi + v * G * plane, un + v * g_->ufs[next()], bytes,
                               cudaMemcpyDeviceToDevice, st));
    }
  }
  double allreduce_max(double v, cudaStream_t) override { return v; }
  bool remote() const override { return false; }

 private:
  std::shared_ptr<LocalGroup> g_;
  int rank_;
};

}  // namespace

bool nccl_available() { return nccl().ok; }

void nccl_unique_id(char* id128) {
  ncclUniqueId uid;
  nccl_check(nccl_or_throw().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(id128, uid.internal, sizeof(uid.internal));
}

std::shared_ptr<HaloTransport> make_nccl_transport(const char* id, int nranks, int rank) {
  return std::make_shared<NcclTransport>(id, nranks, rank);
}

std::vector<std::shared_ptr<HaloTransport>> make_local_group(int nranks) {
  require(nranks >= 1, "local comm: need at least one rank");
  auto g = std::make_shared<LocalGroup>();
  g->u.assign(nranks, nullptr);
  g->ufs.assign(nranks, 0);
  std::vector<std::shared_ptr<HaloTransport>> out;
  for (int r = 0; r < nranks; ++r) out.push_back(std::make_shared<LocalTransport>(g, r));
  return out;
}

// ------------------------------------------------------------- slab RHS
NsSlabOp::NsSlabOp(std::shared_ptr<HaloTransport> tr, std::shared_ptr<NsWorkspace> ws, int part)
    : tr_(std::move(tr)), ws_(std::move(ws)), part_(part) {
  const NsBox& b = ws_->box();
  require(b.G >= 4, "ns slab: the workspace needs >= 4 ghost planes");
  require(b.nz >= b.G, "ns slab: a rank needs at least as many planes as the halo is deep");
  const std::size_t hb = static_cast<std::size_t>(SMC_NVAR) * b.G * b.plane();
  lo_.resize(hb);
  hi_.resize(hb);
  SMC_CUDA(cudaStreamCreateWithFlags(&comm_, cudaStreamNonBlocking));
  SMC_CUDA(cudaEventCreateWithFlags(&ev_in_, cudaEventDisableTiming));
  SMC_CUDA(cudaEventCreateWithFlags(&ev_halo_, cudaEventDisableTiming));
}

NsSlabOp::~NsSlabOp() {
  if (ev_in_) cudaEventDestroy(ev_in_);
  if (ev_halo_) cudaEventDestroy(ev_halo_);
  if (ev_bnd_) cudaEventDestroy(ev_bnd_);
  if (ev_prev_) cudaEventDestroy(ev_prev_);
  for (cudaEvent_t e : ev_chunk_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_done_) cudaEventDestroy(e);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (d2h_) cudaStreamDestroy(d2h_);
  if (comm_) cudaStreamDestroy(comm_);
}

void NsSlabOp::eval_host(double t, const double* u, double* out) {
  const NsBox& b = ws_->box();
  const std::vector<int> bnd = ns_e2e_bounds(b.nz);
  if (!tr_->remote() || part_ == kNsChem || bnd.size() < 3) {
    RhsOp::eval_host(t, u, out);
    return;
  }
  const int nch = static_cast<int>(bnd.size()) - 1, G = b.G;
  const long long n = b.cells(), plane = b.plane();
  stage_u_.resize(static_cast<std::size_t>(SMC_NVAR) * n);
  stage_out_.resize(static_cast<std::size_t>(SMC_NVAR) * n);
  auto ws_for = [&](int kc) -> NsWorkspace& {
    for (auto& w : chunk_ws_)
      if (w->box().nz == kc) return *w;
    chunk_ws_.push_back(ws_->chunk_workspace(kc));
    return *chunk_ws_.back();
  };
  if (!h2d_) {
    SMC_CUDA(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
    SMC_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
    SMC_CUDA(cudaEventCreateWithFlags(&ev_bnd_, cudaEventDisableTiming));
    SMC_CUDA(cudaEventCreateWithFlags(&ev_prev_, cudaEventDisableTiming));
  }
  while (static_cast<int>(ev_chunk_.size()) < nch) {
    cudaEvent_t a, c;
    SMC_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    SMC_CUDA(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
    ev_chunk_.push_back(a);
    ev_done_.push_back(c);
  }
  double* dU = stage_u_.get();
  double* dO = stage_out_.get();
  auto copy = [&](double* dst, const double* src, int k0, int k1, cudaMemcpyKind kind,
                  cudaStream_t st) {
    if (k1 <= k0) return;
    for (int v = 0; v < SMC_NVAR; ++v)
      SMC_CUDA(cudaMemcpyAsync(dst + v * n + k0 * plane, src + v * n + k0 * plane,
                               sizeof(double) * (k1 - k0) * plane, kind, st));
  };
  // the previous evaluation's reads of the staging and halo buffers come first
  SMC_CUDA(cudaEventRecord(ev_prev_, stream_));
  SMC_CUDA(cudaStreamWaitEvent(h2d_, ev_prev_, 0));
  SMC_CUDA(cudaStreamWaitEvent(comm_, ev_prev_, 0));
  copy(dU, u, 0, G, cudaMemcpyHostToDevice, h2d_);           // the planes the
  copy(dU, u, b.nz - G, b.nz, cudaMemcpyHostToDevice, h2d_);  // neighbours need
  SMC_CUDA(cudaEventRecord(ev_bnd_, h2d_));
  SMC_CUDA(cudaStreamWaitEvent(comm_, ev_bnd_, 0));
  tr_->exchange(dU, n, lo_.get(), hi_.get(), plane, G, b.nz, SMC_NVAR, comm_);
  SMC_CUDA(cudaEventRecord(ev_halo_, comm_));
  for (int c = 0; c < nch; ++c) {
    const int k0 = std::max(bnd[c], G), k1 = std::min(bnd[c + 1], b.nz - G);
    copy(dU, u, k0, k1, cudaMemcpyHostToDevice, h2d_);
    SMC_CUDA(cudaEventRecord(ev_chunk_[c], h2d_));
  }
  SMC_CUDA(cudaStreamWaitEvent(stream_, ev_bnd_, 0));
  for (int c = 0; c < nch; ++c) {
    const int k0 = bnd[c], k1 = bnd[c + 1];
    SMC_CUDA(cudaStreamWaitEvent(stream_, ev_chunk_[c], 0));
    if (c + 1 < nch) SMC_CUDA(cudaStreamWaitEvent(stream_, ev_chunk_[c + 1], 0));
    if (c == 0 || c + 1 == nch) SMC_CUDA(cudaStreamWaitEvent(stream_, ev_halo_, 0));
    const long long hs = G * plane;
    const NsStateView view{c == 0 ? lo_.get() : dU + (k0 - G) * plane, c == 0 ? hs : n,
                           dU + k0 * plane, n,
                           c + 1 == nch ? hi_.get() : dU + k1 * plane, c + 1 == nch ? hs : n};
    ws_for(k1 - k0).rhs(view, dO + k0 * plane, n, part_, stream_, kNsAll);
    SMC_CUDA(cudaEventRecord(ev_done_[c], stream_));
    SMC_CUDA(cudaStreamWaitEvent(d2h_, ev_done_[c], 0));
    copy(out, dO, k0, k1, cudaMemcpyDeviceToHost, d2h_);
  }
  SMC_CUDA(cudaStreamSynchronize(d2h_));
  ++evals_;
}

void NsSlabOp::eval_device(double, const double* u, double* out) {
  const NsBox& b = ws_->box();
  const long long n = b.cells();
  const NsStateView view{lo_.get(), b.G * b.plane(), u, n, hi_.get(), b.G * b.plane()};
  if (part_ == kNsChem) {  // pointwise: no halo
    ws_->rhs(view, out, n, part_, stream_, kNsAll);
    ++evals_;
    return;
  }
  // the exchange waits for the state (and for the previous evaluation's
  // reads of the halo blocks) and overlaps the interior work
  SMC_CUDA(cudaEventRecord(ev_in_, stream_));
  SMC_CUDA(cudaStreamWaitEvent(comm_, ev_in_, 0));
  tr_->exchange(u, n, lo_.get(), hi_.get(), b.plane(), b.G, b.nz, SMC_NVAR, comm_);
  SMC_CUDA(cudaEventRecord(ev_halo_, comm_));
  ws_->rhs(view, out, n, part_, stream_, kNsInterior);
  SMC_CUDA(cudaStreamWaitEvent(stream_, ev_halo_, 0));
  ws_->rhs(view, out, n, part_, stream_, kNsBoundary);
  ++evals_;
}

}  // namespace smc
