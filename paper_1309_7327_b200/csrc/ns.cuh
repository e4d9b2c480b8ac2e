// Multicomponent reacting Navier-Stokes RHS on
// sm_100a: ctoprim + transport, hypterm, diffterm (narrow stencil for
// same-direction second derivatives, 8th-order first derivatives for mixed
// and correction terms), wdot with the synthetic mechanism of
// include/smc_mechanism.h.  The reference has no NS code;
// oracle/ns_oracle.c is the CPU restatement the kernels are checked against.
#pragma once

#include "../../include/smc_mechanism.h"
#include "common.cuh"
#include "ops.hpp"

#include <utility>
#include <vector>

namespace smc {

// Periodic box or one z-slab with G ghost planes per field (multi-GPU).
struct NsBox {
  int nx = 0, ny = 0, nz = 0;  // interior
  int G = 0;                   // ghost planes below/above (0: periodic wrap in z)
  long long plane() const { return static_cast<long long>(nx) * ny; }
  long long cells() const { return plane() * nz; }
  long long field_len() const { return plane() * (nz + 2 * G); }
};

enum NsPart : int { kNsFull = 0, kNsAdvDiff = 1, kNsChem = 2 };

// Where the conserved state of a box with G ghost planes lives: planes
// [-G, 0) (lower halo), [0, nz) (interior) and [nz, nz + G) (upper halo) are
// three field-major blocks, each with its own base pointer (its first plane)
// and field stride.  They may be one ghosted array (field stride
// field_len()), an interior array plus two separate halo buffers (a rank's
// state and the planes received from its neighbours: no ghost copy of the
// state), or three windows of one larger array (z-chunks of a box).  The
// periodic box (G = 0) uses the interior block only and wraps z.
struct NsStateView {
  const double* lo = nullptr;
  long long lo_fs = 0;
  const double* mid = nullptr;
  long long mid_fs = 0;
  const double* hi = nullptr;
  long long hi_fs = 0;
  // one contiguous array of nz + 2G planes per field
  static NsStateView ghosted(const double* U, const NsBox& b) {
    const long long fl = b.field_len();
    return {U, fl, U + b.G * b.plane(), fl, U + (b.G + b.nz) * b.plane(), fl};
  }
};

// Plane range of the RHS evaluation (for the overlap of a halo exchange
// with the interior work).  kAll: the whole evaluation; kInterior: the work
// that needs no ghost plane (ctoprim and the x / y direction passes of the
// interior planes); kBoundary: the rest, after the ghosts have arrived.
enum NsPhase : int { kNsAll = 0, kNsInterior = 1, kNsBoundary = 2 };

// Optional per-kernel timing of one evaluation (smc_ns_profile): an event is
// recorded after every kernel, named by the kernel.
struct KernelMarks {
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  cudaEvent_t start = nullptr;
  void mark(const char* name, cudaStream_t st);
  ~KernelMarks();
};

// Device workspace shared by the three RHS views (full / f1 / f2).
class NsWorkspace {
 public:
  NsWorkspace(const NsBox& box, double dx, double dy, double dz, const StencilM& M, int s);
  // out (interior, SMC_NVAR fields) = part of the RHS at state U.  U holds
  // SMC_NVAR fields of box.field_len() each (ghosts filled by the caller
  // when box.G > 0).
  void rhs(const double* U, double* out, int part, cudaStream_t st);
  // The general form: U through a state view, out with field stride out_fs
  // (>= cells()), optionally one phase of the evaluation.
  void rhs(const NsStateView& U, double* out, long long out_fs, int part, cudaStream_t st,
           int phase = kNsAll);
  // Fused FD Jacobian of the chemistry part (RhsOp::fd_block_jacobian) for
  // the cell-block layout (block SMC_NVAR, field-major); false when the box
  // has ghost planes (the state is then not cell-block shaped).
  // MRSDC fine node: the sweep update of the state (RhsOp::eval_after_update)
  // fused with the chemistry part at the updated state; the state is the
  // box's interior cells, 14 fields (a slab's own planes)
  bool chem_after_update(double* next, const double* cur, int nd, const double* const* da,
                         const double* const* db, const double* dc, const double* pre,
                         double* out, cudaStream_t st);
  bool chem_fd_jacobian(const double* U, const double* FU, double* jac, double atol,
                        double root_eps, cudaStream_t st);
  // T and p of every interior cell (ctoprim), for tests / diagnostics.
  void temperature_pressure(const double* U, double* T, double* p, cudaStream_t st);
  const NsBox& box() const { return box_; }
  void set_marks(KernelMarks* m) { marks_ = m; }
  // A workspace for nz_chunk-plane z-chunks of this box (4 ghost planes,
  // same spacings and stencil): the host-buffer pipeline evaluates chunks.
  std::shared_ptr<NsWorkspace> chunk_workspace(int nz_chunk) const;

 private:
  KernelMarks* marks_ = nullptr;
  NsBox box_;
  double dx_[3];
  StencilM M_;
  int s_;
  DevBuf prim_;   // primitive + coefficient fields (all planes)
  DevBuf acc_;    // direction sums: narrow momentum + div tau, sum_k narrow species (interior)
  DevBuf grad_;   // d_j u_i (all planes)
  DevBuf scratch_;  // phase A's x + y sums (18 interior arrays)
};

// Chunk boundaries of the host-buffer pipelines (0 = b[0] < ... < b.back() =
// nz): 8, 8, 16-plane chunks at both ends, ~32 in the middle; empty when nz
// is too short to pipeline.
std::vector<int> ns_e2e_bounds(int nz);

// Conserved state from primitives (T, p, u, v, w, Y_k), n cells, device ptrs.
void ns_conserved_from_primitives(const double* T, const double* p, const double* uvw,
                                  const double* Y, long long n, double* U, cudaStream_t st);

class NsRhsOp final : public RhsOp {
 public:
  NsRhsOp(std::shared_ptr<NsWorkspace> ws, int part) : ws_(std::move(ws)), part_(part) {}
  long long dim() const override { return SMC_NVAR * ws_->box().cells(); }
  // The Rhs view is the periodic box only: a ghosted workspace (zghost > 0)
  // reads 14 fields of field_len() each, which a caller's state of dim()
  // doubles does not hold (smc_ns_rhs_ghosted and the slab RHS take those).
  void eval_device(double, const double* u, double* out) override {
    require(ws_->box().G == 0,
            "ns: a ghosted (zghost > 0) operator has no plain Rhs view; use "
            "smc_ns_rhs_ghosted or the slab RHS (smc_ns_slab_*)");
    ws_->rhs(u, out, part_, stream_);
    ++evals_;
  }
  const char* name() const override { return "ns"; }
  bool eval_after_update(double, double* next, const double* cur, int nd,
                         const double* const* da, const double* const* db, const double* dc,
                         const double* pre, double* out) override {
    if (part_ != kNsChem || ws_->box().G != 0 ||
        !ws_->chem_after_update(next, cur, nd, da, db, dc, pre, out, stream_))
      return false;
    ++evals_;
    return true;
  }
  bool fd_block_jacobian(const double* w, const double* fw, double* jac, long long block,
                         int interleaved, double atol, double root_eps) override {
    if (part_ != kNsChem || block != SMC_NVAR || !interleaved) return false;
    if (!ws_->chem_fd_jacobian(w, fw, jac, atol, root_eps, stream_)) return false;
    evals_ += block;
    return true;
  }
  NsWorkspace& workspace() { return *ws_; }
  int part() const { return part_; }
  // Host buffers (smc_rhs_eval with SMC_HOST): a z-chunk pipeline.  The
  // state goes H2D chunk by chunk (the box's top 4 planes first: the first
  // chunk's lower halo); each chunk's RHS runs as soon as it and the next
  // chunk's first planes have landed, reading its halo in place from the
  // neighbouring chunks (NsStateView), and its result goes D2H while later
  // chunks are still arriving (the link is full duplex).
  void eval_host(double t, const double* u, double* out) override;
  ~NsRhsOp() override;

 private:
  std::shared_ptr<NsWorkspace> ws_;
  int part_;
  std::vector<std::shared_ptr<NsWorkspace>> chunk_ws_;  // one per chunk size
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr;
  std::vector<cudaEvent_t> ev_in_, ev_done_;
  cudaEvent_t ev_halo_ = nullptr;
};

}  // namespace smc
