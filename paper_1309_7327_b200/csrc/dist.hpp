// Block decomposition of the periodic NS box into z-slabs, one per GPU
// (the paper's box decomposition with ghost cells and
// ghost-cell coefficient recompute).
//
// A rank owns nz interior planes of an nx x ny x (nz * world) periodic box,
// field-major like the periodic state (so the device steppers advance it
// unchanged).  Its RHS needs G = 4 planes of the neighbours' state below and
// above: they arrive in two small halo blocks (14 fields x G planes each)
// through a HaloTransport while ctoprim and the x / y passes run on the
// interior planes; the kernels read the halo blocks in place (NsStateView),
// so the state is never copied into a ghosted array.
//
// Transports: NCCL (ncclSend / ncclRecv over NVLink / NVSwitch, one
// communicator per rank from an ncclUniqueId; libnccl is loaded at run time,
// so the library itself has no link dependency on it), and an in-process
// group of ranks on one device (device copies; tests of the slab logic with
// several ranks on one GPU, where ranks must not wait on each other).
#pragma once

#include <memory>
#include <vector>

#include "ns.cuh"
#include "ops.hpp"

namespace smc {

class HaloTransport {
 public:
  virtual ~HaloTransport() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  int prev() const { return (rank() + size() - 1) % size(); }
  int next() const { return (rank() + 1) % size(); }
  // Stream-ordered on st: for every field v, the G bottom interior planes of
  // u (field stride ufs) go to prev() and its G top planes to next(); lo
  // receives prev()'s top planes and hi next()'s bottom planes (field stride
  // G * plane in both halo blocks).
  virtual void exchange(const double* u, long long ufs, double* lo, double* hi, long long plane,
                        int G, int nz, int nvar, cudaStream_t st) = 0;
  // Global max over ranks of a per-rank value (the sweeps' residual, the
  // Newton norms): synchronous.
  virtual double allreduce_max(double v, cudaStream_t st) = 0;
  // In-process groups: the state this rank's neighbours read in their next
  // exchange (the NCCL transport sends instead and ignores it).
  virtual void publish(const double* /*u*/, long long /*ufs*/) {}
  // true when the neighbours' halo arrives by messages (NCCL), false for an
  // in-process group reading published device states
  virtual bool remote() const { return true; }
};

// NCCL: `id` is NCCL_UNIQUE_ID_BYTES (128) bytes from nccl_unique_id() on one
// rank, shared with the others by the caller (e.g. torch.distributed).
std::shared_ptr<HaloTransport> make_nccl_transport(const char* id, int nranks, int rank);
void nccl_unique_id(char* id128);
bool nccl_available();
// nranks transports of one in-process group on the current device
std::vector<std::shared_ptr<HaloTransport>> make_local_group(int nranks);

// The RHS of one rank's slab (dim = 14 * nx * ny * nz): full, advection-
// diffusion (MRSDC f1) or chemistry (f2; pointwise, no exchange).
class NsSlabOp final : public RhsOp {
 public:
  NsSlabOp(std::shared_ptr<HaloTransport> tr, std::shared_ptr<NsWorkspace> ws, int part);
  ~NsSlabOp() override;
  long long dim() const override { return SMC_NVAR * ws_->box().cells(); }
  void eval_device(double t, const double* u, double* out) override;
  // the chemistry part is pointwise: the MRSDC fine-node update fused with it
  // (the slab state is the rank's interior planes, 14 fields)
  bool eval_after_update(double, double* next, const double* cur, int nd,
                         const double* const* da, const double* const* db, const double* dc,
                         const double* pre, double* out) override {
    if (part_ != kNsChem || !ws_->chem_after_update(next, cur, nd, da, db, dc, pre, out, stream_))
      return false;
    ++evals_;
    return true;
  }
  const char* name() const override { return "ns_slab"; }
  HaloTransport& transport() { return *tr_; }
  void publish(const double* u) { tr_->publish(u, ws_->box().cells()); }
  // Host buffers: the rank's 4 bottom and 4 top planes go H2D first and to
  // the neighbours while the rest of the state streams in chunk by chunk;
  // each chunk's RHS (halo read in place: the neighbouring chunks, or the
  // received blocks at the slab's ends) runs as soon as its planes landed,
  // and its result goes D2H meanwhile (NsRhsOp::eval_host's pipeline with
  // the exchange folded in).  In-process groups take the plain path.
  void eval_host(double t, const double* u, double* out) override;

 private:
  std::vector<std::shared_ptr<NsWorkspace>> chunk_ws_;
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr;
  std::vector<cudaEvent_t> ev_chunk_, ev_done_;
  cudaEvent_t ev_bnd_ = nullptr, ev_prev_ = nullptr;
  std::shared_ptr<HaloTransport> tr_;
  std::shared_ptr<NsWorkspace> ws_;
  int part_;
  DevBuf lo_, hi_;
  cudaStream_t comm_ = nullptr;
  cudaEvent_t ev_in_ = nullptr, ev_halo_ = nullptr;
};

}  // namespace smc
