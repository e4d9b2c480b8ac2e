#pragma once
#include "common.cuh"

namespace smc {

// Arguments of the narrow-operator kernel.  Fields are x-fastest,
// v[(k*ny + j)*nx + i] (the reference Field / Field2D flattening,
// proj/core/include/nsdc/pde.hpp:24-35 extended by one axis).  With zwrap the
// z index wraps periodically over [0, nz); without it the pointers address
// plane 0 of an array that carries S ghost planes on both sides (multi-GPU
// slabs, filled by the halo exchange).
struct NarrowArgs {
  const double* u = nullptr;
  const double* cx = nullptr;  // coefficient for the x sweep (a)
  const double* cy = nullptr;  // ... y sweep (b in the 2-D heat operator)
  const double* cz = nullptr;  // ... z sweep
  const double* g0 = nullptr;  // separable source factor, may be null
  double* out = nullptr;
  int nx = 0, ny = 1, nz = 1;
  int dims = 3;                // 1, 2 or 3 active directions
  int kc = 1;                  // z planes per CTA
  int kbeg = 0, kend = -1;     // plane range [kbeg, kend) to compute (kend < 0: nz)
  bool zwrap = true;
  bool use_fast = true;         // allow the narrow3d_fast kernel
  // Peer halo (multi-GPU, narrow3d_fast only): u holds the nz interior planes
  // and the planes below / above come straight from the neighbours' interior
  // arrays (device pointers valid here: CUDA IPC / peer access over NVLink,
  // or another buffer on this device), so no exchange step precedes the
  // kernel.  u_lo + lo_len is the end of the lower neighbour's interior.
  const double* u_lo = nullptr;
  const double* u_hi = nullptr;
  long long lo_len = 0;
  bool zpeer = false;
  double idx2 = 0, idy2 = 0, idz2 = 0, gt = 0;
};

void launch_narrow(const NarrowArgs& p, int s, const StencilM& M, cudaStream_t st);
int narrow_default_kc(int nx, int ny, int nz, int dims, int num_sms);

// FP64-issue-optimised 3-D kernel (narrow3d_fast.cu) for nx % 64 == 0,
// ny % 8 == 0; launch_narrow dispatches to it when applicable.
bool narrow3d_fast_applicable(const NarrowArgs& p);
void launch_narrow3d_fast(const NarrowArgs& p, int s, const StencilM& M, cudaStream_t st);
int narrow3d_fast_default_kc(int nx, int ny, int nz, int num_sms);

// 2-D heat operator tiles (narrow2d_fast.cu) for nx % 32 == 0, ny % 8 == 0.
bool narrow2d_fast_applicable(const NarrowArgs& p);
void launch_narrow2d_fast(const NarrowArgs& p, int s, const StencilM& M, cudaStream_t st);

// Wide route D(a D u) (+ y term when w2/b given) + g0*gt; w1/w2 scratch.
void launch_wide2d(const double* u, const double* a, const double* b, const double* g0, double gt,
                   double* w1, double* w2, double* out, int nx, int ny, double dx, double dy,
                   cudaStream_t st);
void launch_deriv8(const double* u, double* out, int nx, int ny, int nz, int dir, double dx,
                   cudaStream_t st);

// Non-periodic lines with the paper's boundary closure (bounded.cu): nlines
// contiguous lines of n cells; m8 / m6 from make_stencil(8 / 6, ...).
void launch_narrow_bounded(const StencilM& m8, const StencilM& m6, const double* a,
                           const double* u, double* out, int n, int nlines, double dx,
                           cudaStream_t st);
void launch_deriv_bounded(const double* u, double* out, int n, int nlines, double dx,
                          cudaStream_t st);

}  // namespace smc
