#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <utility>

#include "sweeps.hpp"

namespace smc {

// ---------------------------------------------------------------- kernels
namespace {

struct UpdateP {
  double* next;
  const double* cur;
  const double* da[2];
  const double* db[2];
  double dc[2];
  const double* g[kMaxTerms];
  double w[kMaxTerms];
  const double* pre;
  double dt;
  long long n;
  int nd, ng;
};

// Grid-stride, HBM-bound.  Summation order per element follows
// sdc.cpp:73-78 / mrsdc.cpp:110-112: cur + dtm (F_new - F_old) [+ ...] + I,
// with I = dt * (sum_j w_j F_j) as sdc.cpp:61-68 / mrsdc.cpp:69-82.
template <int ND, int NG>
__global__ void __launch_bounds__(256) sweep_update_kernel(const UpdateP p) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.n;
       i += stride) {
    double integ;
    if (NG == 0) {
      integ = p.pre[i];
    } else {
      double acc = p.w[0] * p.g[0][i];
#pragma unroll
      for (int j = 1; j < NG; ++j) acc = __fma_rn(p.w[j], p.g[j][i], acc);
      integ = __dmul_rn(p.dt, acc);
    }
    double v = p.cur[i];
#pragma unroll
    for (int d = 0; d < ND; ++d) v = __fma_rn(p.dc[d], __dsub_rn(p.da[d][i], p.db[d][i]), v);
    p.next[i] = __dadd_rn(v, integ);
  }
}

struct IntegralP {
  double* out[kMaxRows];
  const double* g[kMaxTerms];
  double w[kMaxRows][kMaxTerms];
  double dt;
  long long n;
  int rows, ng;
};

// The weight table is copied to shared memory once per block: indexed by the
// runtime row it would otherwise be a dependent constant-bank load per FMA.
__global__ void __launch_bounds__(256) integrals_kernel(const IntegralP p) {
  __shared__ double ws[kMaxRows][kMaxTerms];
  for (int t = threadIdx.x; t < kMaxRows * kMaxTerms; t += blockDim.x)
    ws[t / kMaxTerms][t % kMaxTerms] = p.w[t / kMaxTerms][t % kMaxTerms];
  __syncthreads();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.n;
       i += stride) {
    double gv[kMaxTerms];
#pragma unroll
    for (int j = 0; j < kMaxTerms; ++j)
      if (j < p.ng) gv[j] = p.g[j][i];
    for (int r = 0; r < p.rows; ++r) {
      double acc = ws[r][0] * gv[0];
#pragma unroll
      for (int j = 1; j < kMaxTerms; ++j)
        if (j < p.ng) acc = __fma_rn(ws[r][j], gv[j], acc);
      p.out[r][i] = __dmul_rn(p.dt, acc);
    }
  }
}

// Fixed-shape variant (the hierarchies the benchmarks use: MRSDC GL(3) /
// TypeB GL(5) is 8 rows x 12 terms, SDC GL(3) 2 x 3): trip counts known, the
// weights read straight from the parameter bank, two elements per thread as
// 16-byte loads and stores.  Same sums in the same order as integrals_kernel.
template <int ROWS, int NG>
__global__ void __launch_bounds__(256) integrals_fixed_kernel(const IntegralP p) {
  const long long n2 = p.n / 2;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n2;
       i += stride) {
    double2 gv[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) gv[j] = __ldg(reinterpret_cast<const double2*>(p.g[j]) + i);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      double a0 = p.w[r][0] * gv[0].x, a1 = p.w[r][0] * gv[0].y;
#pragma unroll
      for (int j = 1; j < NG; ++j) a0 = __fma_rn(p.w[r][j], gv[j].x, a0), a1 = __fma_rn(p.w[r][j], gv[j].y, a1);
      reinterpret_cast<double2*>(p.out[r])[i] = make_double2(__dmul_rn(p.dt, a0), __dmul_rn(p.dt, a1));
    }
  }
  if (p.n & 1) {  // odd tail element
    const long long i = p.n - 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        double acc = p.w[r][0] * p.g[0][i];
#pragma unroll
        for (int j = 1; j < NG; ++j) acc = __fma_rn(p.w[r][j], p.g[j][i], acc);
        p.out[r][i] = __dmul_rn(p.dt, acc);
      }
    }
  }
}

struct ResidualP {
  const double* u0;
  const double* um;
  const double* g[kMaxTerms];
  double q[kMaxTerms];
  double dt;
  long long n;
  int ng;
  unsigned long long* slot;  // [0] max as bits, [1] non-finite flag
};

// sdc.cpp:20-30 / mrsdc.cpp:23-35.  Non-negative doubles order like their
// bit patterns, so the block maxima combine with an integer atomicMax.  A
// NaN is skipped by the max (as std::max(r, NaN) == r in the reference) but
// raises the non-finite flag.
__global__ void __launch_bounds__(256) residual_kernel(const ResidualP p) {
  double r = 0.0;
  unsigned long long bad = 0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.n;
       i += stride) {
    double acc = p.q[0] * p.g[0][i];
    for (int j = 1; j < p.ng; ++j) acc = __fma_rn(p.q[j], p.g[j][i], acc);
    const double v = fabs(__dsub_rn(__fma_rn(p.dt, acc, p.u0[i]), p.um[i]));
    if (!isfinite(v)) bad = 1;
    if (v > r) r = v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ double wr[8];
  __shared__ unsigned long long wb[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    wr[warp] = r;
    wb[warp] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      r = fmax(r, wr[w]);
      bad |= wb[w];
    }
    if (isinf(r)) bad = 1;
    atomicMax(p.slot, static_cast<unsigned long long>(__double_as_longlong(r)));
    if (bad) atomicMax(p.slot + 1, 1ull);
  }
}

// integrals_fixed_kernel fused with the residual of the previous sweep
// (MRSDC): both read the same node values F, so one pass serves the next
// sweep's node integrals and the last sweep's residual.  The per-element
// residual arithmetic and the block reduction are residual_kernel's.
template <int ROWS, int NG>
__global__ void __launch_bounds__(256) integrals_residual_kernel(const IntegralP p,
                                                                 const ResidualP rp) {
  const long long n2 = p.n / 2;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  double r = 0.0;
  unsigned long long bad = 0;
  auto res1 = [&](double acc, double u0, double um) {
    const double v = fabs(__dsub_rn(__fma_rn(rp.dt, acc, u0), um));
    if (!isfinite(v)) bad = 1;
    if (v > r) r = v;
  };
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n2;
       i += stride) {
    double2 gv[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) gv[j] = __ldg(reinterpret_cast<const double2*>(p.g[j]) + i);
    const double2 u0 = __ldg(reinterpret_cast<const double2*>(rp.u0) + i);
    const double2 um = __ldg(reinterpret_cast<const double2*>(rp.um) + i);
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr) {
      double a0 = p.w[rr][0] * gv[0].x, a1 = p.w[rr][0] * gv[0].y;
#pragma unroll
      for (int j = 1; j < NG; ++j) a0 = __fma_rn(p.w[rr][j], gv[j].x, a0), a1 = __fma_rn(p.w[rr][j], gv[j].y, a1);
      reinterpret_cast<double2*>(p.out[rr])[i] = make_double2(__dmul_rn(p.dt, a0), __dmul_rn(p.dt, a1));
    }
    double q0 = rp.q[0] * gv[0].x, q1 = rp.q[0] * gv[0].y;
#pragma unroll
    for (int j = 1; j < NG; ++j) q0 = __fma_rn(rp.q[j], gv[j].x, q0), q1 = __fma_rn(rp.q[j], gv[j].y, q1);
    res1(q0, u0.x, um.x);
    res1(q1, u0.y, um.y);
  }
  if ((p.n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail element
    const long long i = p.n - 1;
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr) {
      double acc = p.w[rr][0] * p.g[0][i];
#pragma unroll
      for (int j = 1; j < NG; ++j) acc = __fma_rn(p.w[rr][j], p.g[j][i], acc);
      p.out[rr][i] = __dmul_rn(p.dt, acc);
    }
    double acc = rp.q[0] * p.g[0][i];
#pragma unroll
    for (int j = 1; j < NG; ++j) acc = __fma_rn(rp.q[j], p.g[j][i], acc);
    res1(acc, rp.u0[i], rp.um[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ double wr[8];
  __shared__ unsigned long long wb[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    wr[warp] = r;
    wb[warp] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      r = fmax(r, wr[w]);
      bad |= wb[w];
    }
    if (isinf(r)) bad = 1;
    atomicMax(rp.slot, static_cast<unsigned long long>(__double_as_longlong(r)));
    if (bad) atomicMax(rp.slot + 1, 1ull);
  }
}

// SDC: the first node update of sweep k (no F difference, sdc.cpp:74) fused
// with the residual of sweep k - 1: both read u0 and the same node values F.
// Per element the update is sweep_update_kernel<0, NG>'s and the residual
// residual_kernel's; the block reduction is residual_kernel's.  um must not
// alias next (the caller falls back to two launches for one-interval nodes).
template <int NG>
__global__ void __launch_bounds__(256) update_residual_kernel(const UpdateP p, const ResidualP rp) {
  double r = 0.0;
  unsigned long long bad = 0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.n;
       i += stride) {
    double gv[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) gv[j] = p.g[j][i];
    const double cur = p.cur[i];
    double acc = p.w[0] * gv[0];
#pragma unroll
    for (int j = 1; j < NG; ++j) acc = __fma_rn(p.w[j], gv[j], acc);
    p.next[i] = __dadd_rn(cur, __dmul_rn(p.dt, acc));
    double q = rp.q[0] * gv[0];
#pragma unroll
    for (int j = 1; j < NG; ++j) q = __fma_rn(rp.q[j], gv[j], q);
    const double v = fabs(__dsub_rn(__fma_rn(rp.dt, q, cur), rp.um[i]));
    if (!isfinite(v)) bad = 1;
    if (v > r) r = v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ double wr[8];
  __shared__ unsigned long long wb[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    wr[warp] = r;
    wb[warp] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      r = fmax(r, wr[w]);
      bad |= wb[w];
    }
    if (isinf(r)) bad = 1;
    atomicMax(rp.slot, static_cast<unsigned long long>(__double_as_longlong(r)));
    if (bad) atomicMax(rp.slot + 1, 1ull);
  }
}

struct BeRhsP {
  double* c;
  const double* u;
  const double* so[kMaxRows];
  const double* old;
  double dt1;
  long long n;
  int nso;
};

__global__ void __launch_bounds__(256) be_rhs_kernel(const BeRhsP p) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.n;
       i += stride) {
    double acc = 0.0;
    for (int q = 0; q < p.nso; ++q) acc = __dadd_rn(acc, p.so[q][i]);
    p.c[i] = __dsub_rn(__dadd_rn(p.u[i], acc), __dmul_rn(p.dt1, p.old[i]));
  }
}

int blocks_for(long long n) {
  const long long want = (n + 255) / 256;
  const long long cap = static_cast<long long>(num_sms()) * 8;
  return static_cast<int>(std::max(1LL, std::min(want, cap)));
}

}  // namespace

void launch_sweep_update(double* next, const double* cur, int nd, const double* const* da,
                         const double* const* db, const double* dc, int ng,
                         const double* const* g, const double* w, double dt, const double* pre,
                         long long n, cudaStream_t st) {
  require(nd >= 0 && nd <= 2 && ng >= 0 && ng <= kMaxTerms, "sweep update: too many terms");
  require(ng > 0 || pre, "sweep update: no integral");
  UpdateP p{};
  p.next = next, p.cur = cur, p.pre = pre, p.dt = dt, p.n = n, p.nd = nd, p.ng = pre ? 0 : ng;
  for (int d = 0; d < nd; ++d) p.da[d] = da[d], p.db[d] = db[d], p.dc[d] = dc[d];
  for (int j = 0; j < p.ng; ++j) p.g[j] = g[j], p.w[j] = w[j];
  const int blocks = blocks_for(n);
#define SMC_UPD(ND, NG) \
  sweep_update_kernel<ND, NG><<<blocks, 256, 0, st>>>(p)
#define SMC_UPD_ND(NG)          \
  do {                          \
    if (nd == 0) SMC_UPD(0, NG); \
    else if (nd == 1) SMC_UPD(1, NG); \
    else SMC_UPD(2, NG);        \
  } while (0)
  switch (p.ng) {
    case 0: SMC_UPD_ND(0); break;
    case 1: SMC_UPD_ND(1); break;
    case 2: SMC_UPD_ND(2); break;
    case 3: SMC_UPD_ND(3); break;
    case 4: SMC_UPD_ND(4); break;
    case 5: SMC_UPD_ND(5); break;
    case 6: SMC_UPD_ND(6); break;
    case 7: SMC_UPD_ND(7); break;
    case 8: SMC_UPD_ND(8); break;
    case 9: SMC_UPD_ND(9); break;
    default: throw InvalidArgument("sweep update: use precomputed integrals beyond 9 nodes");
  }
#undef SMC_UPD_ND
#undef SMC_UPD
  SMC_CHECK_LAUNCH();
}

void launch_integrals(int rows, double* const* out, int ng, const double* const* g,
                      const double* w, double dt, long long n, cudaStream_t st) {
  require(rows >= 1 && rows <= kMaxRows && ng >= 1 && ng <= kMaxTerms,
          "integrals: table too large");
  IntegralP p{};
  p.rows = rows, p.ng = ng, p.dt = dt, p.n = n;
  for (int r = 0; r < rows; ++r) {
    p.out[r] = out[r];
    for (int j = 0; j < ng; ++j) p.w[r][j] = w[r * ng + j];
  }
  for (int j = 0; j < ng; ++j) p.g[j] = g[j];
  bool aligned = true;
  for (int j = 0; j < ng; ++j) aligned = aligned && (reinterpret_cast<std::uintptr_t>(g[j]) & 15) == 0;
  for (int r = 0; r < rows; ++r)
    aligned = aligned && (reinterpret_cast<std::uintptr_t>(out[r]) & 15) == 0;
  const int fb = static_cast<int>(std::max(
      1LL, std::min((n / 2 + 255) / 256, static_cast<long long>(num_sms()) * 16)));
  if (aligned && rows == 8 && ng == 12)
    integrals_fixed_kernel<8, 12><<<fb, 256, 0, st>>>(p);
  else if (aligned && rows == 2 && ng == 3)
    integrals_fixed_kernel<2, 3><<<fb, 256, 0, st>>>(p);
  else
    integrals_kernel<<<blocks_for(n), 256, 0, st>>>(p);
  SMC_CHECK_LAUNCH();
}

void launch_be_rhs(double* c, const double* u, int nso, const double* const* so, const double* old,
                   double dt1, long long n, cudaStream_t st) {
  require(nso >= 1 && nso <= kMaxRows, "mrsdc mode 2: too many fine sub-steps per coarse interval");
  BeRhsP p{};
  p.c = c, p.u = u, p.old = old, p.dt1 = dt1, p.n = n, p.nso = nso;
  for (int q = 0; q < nso; ++q) p.so[q] = so[q];
  be_rhs_kernel<<<blocks_for(n), 256, 0, st>>>(p);
  SMC_CHECK_LAUNCH();
}

void launch_residual(const double* u0, const double* um, int ng, const double* const* g,
                     const double* q, double dt, long long n, double* slot, cudaStream_t st) {
  require(ng >= 1 && ng <= kMaxTerms, "residual: too many terms");
  ResidualP p{};
  p.u0 = u0, p.um = um, p.dt = dt, p.n = n, p.ng = ng;
  p.slot = reinterpret_cast<unsigned long long*>(slot);
  for (int j = 0; j < ng; ++j) p.g[j] = g[j], p.q[j] = q[j];
  residual_kernel<<<blocks_for(n), 256, 0, st>>>(p);
  SMC_CHECK_LAUNCH();
}

void launch_integrals_residual(int rows, double* const* out, int ng, const double* const* g,
                               const double* w, double dt, const double* u0, const double* um,
                               const double* q, long long n, double* slot, cudaStream_t st) {
  bool aligned = (reinterpret_cast<std::uintptr_t>(u0) & 15) == 0 &&
                 (reinterpret_cast<std::uintptr_t>(um) & 15) == 0;
  for (int j = 0; j < ng; ++j) aligned = aligned && (reinterpret_cast<std::uintptr_t>(g[j]) & 15) == 0;
  for (int r = 0; r < rows; ++r)
    aligned = aligned && (reinterpret_cast<std::uintptr_t>(out[r]) & 15) == 0;
  if (!(aligned && rows == 8 && ng == 12)) {
    launch_residual(u0, um, ng, g, q, dt, n, slot, st);
    launch_integrals(rows, out, ng, g, w, dt, n, st);
    return;
  }
  IntegralP p{};
  p.rows = rows, p.ng = ng, p.dt = dt, p.n = n;
  for (int r = 0; r < rows; ++r) {
    p.out[r] = out[r];
    for (int j = 0; j < ng; ++j) p.w[r][j] = w[r * ng + j];
  }
  ResidualP rp{};
  rp.u0 = u0, rp.um = um, rp.dt = dt, rp.n = n, rp.ng = ng;
  rp.slot = reinterpret_cast<unsigned long long*>(slot);
  for (int j = 0; j < ng; ++j) p.g[j] = g[j], rp.g[j] = g[j], rp.q[j] = q[j];
  const int fb = static_cast<int>(std::max(
      1LL, std::min((n / 2 + 255) / 256, static_cast<long long>(num_sms()) * 16)));
  integrals_residual_kernel<8, 12><<<fb, 256, 0, st>>>(p, rp);
  SMC_CHECK_LAUNCH();
}

void launch_update_residual(double* next, const double* u0, const double* um, int ng,
                            const double* const* g, const double* w, const double* q, double dt,
                            long long n, double* slot, cudaStream_t st) {
  require(um != next, "update_residual: the residual's end state is the updated node");
  if (ng < 2 || ng > 5) {
    launch_residual(u0, um, ng, g, q, dt, n, slot, st);
    launch_sweep_update(next, u0, 0, nullptr, nullptr, nullptr, ng, g, w, dt, nullptr, n, st);
    return;
  }
  UpdateP p{};
  p.next = next, p.cur = u0, p.dt = dt, p.n = n, p.ng = ng;
  ResidualP rp{};
  rp.u0 = u0, rp.um = um, rp.dt = dt, rp.n = n, rp.ng = ng;
  rp.slot = reinterpret_cast<unsigned long long*>(slot);
  for (int j = 0; j < ng; ++j) p.g[j] = g[j], p.w[j] = w[j], rp.g[j] = g[j], rp.q[j] = q[j];
  const int blocks = blocks_for(n);
  switch (ng) {
    case 2: update_residual_kernel<2><<<blocks, 256, 0, st>>>(p, rp); break;
    case 3: update_residual_kernel<3><<<blocks, 256, 0, st>>>(p, rp); break;
    case 4: update_residual_kernel<4><<<blocks, 256, 0, st>>>(p, rp); break;
    default: update_residual_kernel<5><<<blocks, 256, 0, st>>>(p, rp); break;
  }
  SMC_CHECK_LAUNCH();
}

void SweepDiag::add(const SweepDiag& o) {
  residuals.insert(residuals.end(), o.residuals.begin(), o.residuals.end());
  sweeps += o.sweeps;
  fresh_evals += o.fresh_evals;
  f1_evals += o.f1_evals;
  f2_evals += o.f2_evals;
  implicit_solves += o.implicit_solves;
  newton_f1_evals += o.newton_f1_evals;
  early_stop = early_stop || o.early_stop;
  nonfinite = nonfinite || o.nonfinite;
}

namespace {

// sdc.cpp:9-16 / mrsdc.cpp:9-16
bool stalled(const std::vector<double>& h, double cutoff) {
  if (cutoff <= 0.0 || h.size() < 2) return false;
  const double prev = h[h.size() - 2], cur = h.back();
  if (cur == 0.0) return true;
  const double ratio = prev / cur;
  return ratio >= 1.0 - cutoff && ratio <= 1.0 + cutoff;
}

void d2d(double* dst, const double* src, long long n, cudaStream_t st) {
  if (dst != src)
    SMC_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

// Reads the residual slots of sweeps [first, first + count) and applies the
// cross-rank reduction; slots are (max bits, flag) pairs.
void collect(const DevBuf& res, int first, int count, cudaStream_t st, const Reducer& reduce,
             SweepDiag& d) {
  std::vector<double> h(2 * count);
  SMC_CUDA(cudaMemcpyAsync(h.data(), res.get() + 2 * first, 2 * count * sizeof(double),
                           cudaMemcpyDeviceToHost, st));
  SMC_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < count; ++i) {
    double r = h[2 * i];
    unsigned long long flag;
    std::memcpy(&flag, &h[2 * i + 1], sizeof(flag));
    if (flag) d.nonfinite = true;
    if (reduce) r = reduce(r);
    d.residuals.push_back(r);
  }
}

}  // namespace

// ------------------------------------------------------------- DeviceSdc
DeviceSdc::DeviceSdc(Nodes nodes, int iterations, double cutoff, bool reuse_first)
    : nodes_(std::move(nodes)), iterations_(iterations), cutoff_(cutoff), reuse_first_(reuse_first) {
  require(iterations >= 1, "SdcStepper: need at least one sweep");
  tab_ = integration_matrices(nodes_);
  require(nodes_.intervals() <= 8, "SdcStepper: at most 9 nodes on the device path");
}

void DeviceSdc::ensure(long long dim) {
  if (dim == dim_) return;
  const int m = nodes_.intervals();
  U_.clear(), FA_.clear(), FB_.clear();
  for (int i = 0; i <= m; ++i) U_.emplace_back(dim);
  for (int i = 0; i < m; ++i) FA_.emplace_back(dim), FB_.emplace_back(dim);
  F0_.resize(dim);
  res_.resize(2 * static_cast<std::size_t>(iterations_));
  u_.clear(), fa_.clear(), fb_.clear();
  for (auto& b : U_) u_.push_back(b.get());
  for (auto& b : FA_) fa_.push_back(b.get());
  for (auto& b : FB_) fb_.push_back(b.get());
  f0_ = F0_.get();
  dim_ = dim;
}

// One SdcStepper::step (sdc.cpp:38-96) on the internal buffers: u_[0] holds
// u0; F0 is valid when have_f0.  Leaves the end state in u_[M] and the final
// node's F in f_last_.
void DeviceSdc::run(RhsOp& f, double t_n, double dt, bool have_f0, SweepDiag& d) {
  const int m = nodes_.intervals();
  const long long n = dim_;
  const auto& tau = nodes_.t;
  cudaStream_t st = f.stream();
  if (!have_f0) {
    f.eval_device(t_n, u_[0], f0_);
    ++d.fresh_evals;
  }
  std::vector<const double*> fold(m + 1, f0_), fnew(m + 1, f0_);
  SMC_CUDA(cudaMemsetAsync(res_.get(), 0, res_.size() * sizeof(double), st));
  const double* qrow = &tab_.q.a[static_cast<std::size_t>(m - 1) * (m + 1)];
  int collected = 0, formed = 0;
  // the residual of sweep k was formed: read it back when early stopping is
  // on; false when the step ends there (sdc.cpp:84-91)
  auto check = [&](int k) {
    formed = k;
    if (cutoff_ <= 0.0) return true;
    collect(res_, k - 1, 1, st, reduce_, d);
    collected = k;
    if (!stalled(d.residuals, cutoff_)) return true;
    d.early_stop = true;
    return false;
  };
  // one-interval nodes: u_[m] is node 1's buffer, so the residual is formed
  // at the end of its own sweep
  const bool fuse = m > 1;
  bool stop = false;
  for (int k = 1; k <= iterations_ && !stop; ++k) {
    std::vector<double*>& set = (k % 2) ? fa_ : fb_;
    for (int j = 1; j <= m; ++j) fnew[j] = set[j - 1];
    for (int r = 0; r < m; ++r) {
      const double dtm = (tau[r + 1] - tau[r]) * dt;
      const double* da[1] = {fnew[r]};
      const double* db[1] = {fold[r]};
      const double dc[1] = {dtm};
      const int nd = (r == 0 || fnew[r] == fold[r]) ? 0 : 1;  // m == 0 branch, sdc.cpp:74
      const double* srow = &tab_.s.a[static_cast<std::size_t>(r) * (m + 1)];
      if (fuse && r == 0 && k > 1) {
        // node 1 of sweep k with the residual of sweep k - 1 (same u0 and F;
        // u_[m] is not written here for m > 1, so a stop leaves sweep k - 1's
        // end state)
        launch_update_residual(u_[1], u_[0], u_[m], m + 1, fold.data(), srow, qrow, dt, n,
                               res_.get() + 2 * (k - 2), st);
        if (!check(k - 1)) {
          stop = true;
          break;
        }
      } else {
        launch_sweep_update(u_[r + 1], u_[r], nd, da, db, dc, m + 1, fold.data(), srow, dt,
                            nullptr, n, st);
      }
      f.eval_device(t_n + tau[r + 1] * dt, u_[r + 1], set[r]);
      ++d.fresh_evals;
    }
    if (stop) break;
    d.sweeps = k;
    fold = fnew;
    if (!fuse) {
      launch_residual(u_[0], u_[m], m + 1, fold.data(), qrow, dt, n, res_.get() + 2 * (k - 1), st);
      if (!check(k)) break;
    }
  }
  if (formed < d.sweeps) {
    launch_residual(u_[0], u_[m], m + 1, fold.data(), qrow, dt, n, res_.get() + 2 * (d.sweeps - 1), st);
    check(d.sweeps);
  }
  if (collected < d.sweeps) collect(res_, collected, d.sweeps - collected, st, reduce_, d);
  f_last_ = const_cast<double*>(fold[m]);
}

void DeviceSdc::step(RhsOp& f, const double* u0, double t_n, double dt, const double* f0,
                     double* u_out, double* f_end, SweepDiag& d) {
  ensure(f.dim());
  const long long n = dim_;
  cudaStream_t st = f.stream();
  d2d(u_[0], u0, n, st);
  const bool have = f0 && reuse_first_;
  if (have) d2d(f0_, f0, n, st);
  run(f, t_n, dt, have, d);
  d2d(u_out, u_[nodes_.intervals()], n, st);
  if (f_end) d2d(f_end, f_last_, n, st);
}

void DeviceSdc::integrate(RhsOp& f, const double* u0, double t0, double t1, int nsteps,
                          double* u_out, SweepDiag& total) {
  require(nsteps >= 0, "integrate_sdc: negative step count");
  ensure(f.dim());
  const long long n = dim_;
  const int m = nodes_.intervals();
  cudaStream_t st = f.stream();
  d2d(u_[0], u0, n, st);
  const double dt = (t1 - t0) / std::max(nsteps, 1);
  for (int step = 0; step < nsteps; ++step) {
    SweepDiag d;
    run(f, t0 + step * dt, dt, step > 0 && reuse_first_, d);
    // recycle: next u0 = U_M, next F0 = F at the last node (sdc.cpp:116-118)
    std::swap(u_[0], u_[m]);
    for (auto* set : {&fa_, &fb_})
      for (auto& p : *set)
        if (p == f_last_) std::swap(p, f0_);
    total.add(d);
  }
  d2d(u_out, u_[0], n, st);
}

// ----------------------------------------------------------- DeviceMrsdc
DeviceMrsdc::DeviceMrsdc(Hierarchy h, int iterations, double cutoff, bool reuse_first)
    : h_(std::move(h)), iterations_(iterations), cutoff_(cutoff), reuse_first_(reuse_first) {
  require(iterations >= 1, "MrsdcStepper: need at least one sweep");
  require(h_.fine.intervals() <= kMaxRows, "MrsdcStepper: at most 16 fine intervals on device");
  require(h_.coarse.count() + h_.fine.count() <= kMaxTerms,
          "MrsdcStepper: hierarchy too large for the device path");
}

void DeviceMrsdc::ensure(long long dim) {
  if (dim == dim_) return;
  const int m1 = h_.coarse.intervals(), m2 = h_.fine.intervals();
  U_.clear(), F1A_.clear(), F1B_.clear(), F2A_.clear(), F2B_.clear(), SO_.clear();
  for (int i = 0; i <= m2; ++i) U_.emplace_back(dim);
  for (int i = 0; i < m1; ++i) F1A_.emplace_back(dim), F1B_.emplace_back(dim);
  for (int i = 0; i < m2; ++i) F2A_.emplace_back(dim), F2B_.emplace_back(dim), SO_.emplace_back(dim);
  F10_.resize(dim);
  F20_.resize(dim);
  res_.resize(2 * static_cast<std::size_t>(iterations_));
  auto ptrs = [](std::vector<DevBuf>& v) {
    std::vector<double*> p;
    for (auto& b : v) p.push_back(b.get());
    return p;
  };
  u_ = ptrs(U_), f1a_ = ptrs(F1A_), f1b_ = ptrs(F1B_), f2a_ = ptrs(F2A_), f2b_ = ptrs(F2B_);
  so_ = ptrs(SO_);
  f10_ = F10_.get(), f20_ = F20_.get();
  dim_ = dim;
}

// MrsdcStepper::step_mode1 (mrsdc.cpp:84-135) on the internal buffers.
// The node integrals at the start of sweep k and the residual of sweep k - 1
// read the same node values, so they are formed in one pass
// (launch_integrals_residual).  With early stopping the residual of sweep
// k - 1 is read back there and a stall ends the step before sweep k changes
// any state, as mrsdc.cpp:120-131 stops after sweep k - 1.
struct DeviceMrsdc::SweepResiduals {
  DeviceMrsdc& m;
  SweepDiag& d;
  cudaStream_t st;
  int m2, ng;
  const std::vector<double>& w;
  const std::vector<double>& qrow;
  double dt;
  long long n;
  int formed = 0, collected = 0;

  static std::vector<const double*> cat(const std::vector<const double*>& a,
                                        const std::vector<const double*>& b) {
    std::vector<const double*> g(a.begin(), a.end());
    g.insert(g.end(), b.begin(), b.end());
    return g;
  }
  // the residual of sweep k was formed: false when early stopping ends here
  bool check(int k) {
    formed = k;
    if (m.cutoff_ <= 0.0) return true;
    collect(m.res_, k - 1, 1, st, m.reduce_, d);
    collected = k;
    if (!stalled(d.residuals, m.cutoff_)) return true;
    d.early_stop = true;
    return false;
  }
  bool begin(int k, const std::vector<const double*>& o1, const std::vector<const double*>& o2) {
    const std::vector<const double*> g = cat(o1, o2);
    if (k == 1) {
      launch_integrals(m2, m.so_.data(), ng, g.data(), w.data(), dt, n, st);
      return true;
    }
    launch_integrals_residual(m2, m.so_.data(), ng, g.data(), w.data(), dt, m.u_[0], m.u_[m2],
                              qrow.data(), n, m.res_.get() + 2 * (k - 2), st);
    return check(k - 1);
  }
  void end(const std::vector<const double*>& o1, const std::vector<const double*>& o2) {
    if (formed < d.sweeps) {
      const std::vector<const double*> g = cat(o1, o2);
      launch_residual(m.u_[0], m.u_[m2], ng, g.data(), qrow.data(), dt, n,
                      m.res_.get() + 2 * (d.sweeps - 1), st);
      check(d.sweeps);
    }
    if (collected < d.sweeps) collect(m.res_, collected, d.sweeps - collected, st, m.reduce_, d);
  }
};

void DeviceMrsdc::run(RhsOp& f1, RhsOp& f2, double t_n, double dt, bool have1, bool have2,
                      SweepDiag& d) {
  const int m1 = h_.coarse.intervals(), m2 = h_.fine.intervals();
  const long long n = dim_;
  const auto& t1 = h_.coarse.t;
  const auto& t2 = h_.fine.t;
  cudaStream_t st = f2.stream();
  require(f1.stream() == st, "mrsdc: f1 and f2 must share a stream");
  if (!have1) {
    f1.eval_device(t_n, u_[0], f10_);
    ++d.f1_evals;
  }
  if (!have2) {
    f2.eval_device(t_n, u_[0], f20_);
    ++d.f2_evals;
  }
  std::vector<int> coarse_at(m2 + 1, -1);
  for (int p = 0; p <= m1; ++p) coarse_at[h_.fine_of_coarse[p]] = p;
  std::vector<const double*> o1(m1 + 1, f10_), n1(m1 + 1, f10_), o2(m2 + 1, f20_),
      n2(m2 + 1, f20_);
  // integral weights: row q = [s21(q, :), s22(q, :)] against [F1_old, F2_old]
  const int ng = m1 + 1 + m2 + 1;
  std::vector<double> w(static_cast<std::size_t>(m2) * ng);
  for (int q = 0; q < m2; ++q) {
    for (int j = 0; j <= m1; ++j) w[q * ng + j] = h_.s21(q, j);
    for (int j = 0; j <= m2; ++j) w[q * ng + m1 + 1 + j] = h_.s22(q, j);
  }
  std::vector<double> qrow(ng);
  for (int j = 0; j <= m1; ++j) qrow[j] = h_.q21(m2 - 1, j);
  for (int j = 0; j <= m2; ++j) qrow[m1 + 1 + j] = h_.q22(m2 - 1, j);
  SMC_CUDA(cudaMemsetAsync(res_.get(), 0, res_.size() * sizeof(double), st));
  SweepResiduals rs{*this, d, st, m2, ng, w, qrow, dt, n};
  for (int k = 1; k <= iterations_; ++k) {
    std::vector<double*>& s1 = (k % 2) ? f1a_ : f1b_;
    std::vector<double*>& s2 = (k % 2) ? f2a_ : f2b_;
    // accumulate_node_terms (mrsdc.cpp:69-82) from the previous sweep's values
    // (with the previous sweep's residual, mrsdc.cpp:23-35, in the same pass)
    if (!rs.begin(k, o1, o2)) break;
    for (int p = 1; p <= m1; ++p) n1[p] = o1[p];  // refreshed when the sweep reaches node p
    for (int q = 0; q < m2; ++q) {
      const double dtq = (t2[q + 1] - t2[q]) * dt;
      const int p = h_.p_map[q];
      const double* da[2];
      const double* db[2];
      double dc[2];
      int nd = 0;
      if (n1[p] != o1[p]) da[nd] = n1[p], db[nd] = o1[p], dc[nd] = dtq, ++nd;
      if (n2[q] != o2[q]) da[nd] = n2[q], db[nd] = o2[q], dc[nd] = dtq, ++nd;
      // the update of node q + 1 and f2 there, fused when f2 is pointwise
      // (the NS chemistry part), else two passes
      if (!f2.eval_after_update(t_n + t2[q + 1] * dt, u_[q + 1], u_[q], nd, da, db, dc, so_[q],
                                s2[q])) {
        launch_sweep_update(u_[q + 1], u_[q], nd, da, db, dc, 0, nullptr, nullptr, dt, so_[q], n,
                            st);
        f2.eval_device(t_n + t2[q + 1] * dt, u_[q + 1], s2[q]);
      }
      n2[q + 1] = s2[q];
      ++d.f2_evals;
      if (const int pc = coarse_at[q + 1]; pc > 0) {
        f1.eval_device(t_n + t1[pc] * dt, u_[q + 1], s1[pc - 1]);
        n1[pc] = s1[pc - 1];
        ++d.f1_evals;
      }
    }
    d.sweeps = k;
    o1 = n1;
    o2 = n2;
  }
  rs.end(o1, o2);
  f1_last_ = const_cast<double*>(o1[m1]);
  f2_last_ = const_cast<double*>(o2[m2]);
}

void DeviceMrsdc::step_mode1(RhsOp& f1, RhsOp& f2, const double* u0, double t_n, double dt,
                             const double* f01, const double* f02, double* u_out, double* f1_end,
                             double* f2_end, SweepDiag& d) {
  require(f1.dim() == f2.dim(), "mrsdc: f1/f2 dimension mismatch");
  ensure(f1.dim());
  const long long n = dim_;
  cudaStream_t st = f2.stream();
  d2d(u_[0], u0, n, st);
  const bool h1 = f01 && reuse_first_, h2 = f02 && reuse_first_;
  if (h1) d2d(f10_, f01, n, st);
  if (h2) d2d(f20_, f02, n, st);
  run(f1, f2, t_n, dt, h1, h2, d);
  d2d(u_out, u_[h_.fine.intervals()], n, st);
  if (f1_end) d2d(f1_end, f1_last_, n, st);
  if (f2_end) d2d(f2_end, f2_last_, n, st);
}

// MrsdcStepper::step_mode2 (mrsdc.cpp:137-206) on the internal buffers.
void DeviceMrsdc::run2(RhsOp& f1, RhsOp& f2, double t_n, double dt, bool have1, bool have2,
                       SweepDiag& d) {
  const int m1 = h_.coarse.intervals(), m2 = h_.fine.intervals();
  const long long n = dim_;
  const auto& t1 = h_.coarse.t;
  const auto& t2 = h_.fine.t;
  cudaStream_t st = f2.stream();
  require(f1.stream() == st, "mrsdc: f1 and f2 must share a stream");
  C_.resize(n);
  W_.resize(n);
  // provisional U at every fine node (mrsdc.cpp:49): mode 2 reads U_q1 as the
  // Newton guess before the sweep has written it
  for (int q = 1; q <= m2; ++q) d2d(u_[q], u_[0], n, st);
  if (!have1) {
    f1.eval_device(t_n, u_[0], f10_);
    ++d.f1_evals;
  }
  if (!have2) {
    f2.eval_device(t_n, u_[0], f20_);
    ++d.f2_evals;
  }
  std::vector<const double*> o1(m1 + 1, f10_), n1(m1 + 1, f10_), o2(m2 + 1, f20_),
      n2(m2 + 1, f20_);
  const int ng = m1 + 1 + m2 + 1;
  std::vector<double> w(static_cast<std::size_t>(m2) * ng);
  for (int q = 0; q < m2; ++q) {
    for (int j = 0; j <= m1; ++j) w[q * ng + j] = h_.s21(q, j);
    for (int j = 0; j <= m2; ++j) w[q * ng + m1 + 1 + j] = h_.s22(q, j);
  }
  std::vector<double> qrow(ng);
  for (int j = 0; j <= m1; ++j) qrow[j] = h_.q21(m2 - 1, j);
  for (int j = 0; j <= m2; ++j) qrow[m1 + 1 + j] = h_.q22(m2 - 1, j);
  SMC_CUDA(cudaMemsetAsync(res_.get(), 0, res_.size() * sizeof(double), st));
  SweepResiduals rs{*this, d, st, m2, ng, w, qrow, dt, n};
  for (int k = 1; k <= iterations_; ++k) {
    std::vector<double*>& s1 = (k % 2) ? f1a_ : f1b_;
    std::vector<double*>& s2 = (k % 2) ? f2a_ : f2b_;
    if (!rs.begin(k, o1, o2)) break;
    for (int p = 0; p < m1; ++p) {
      const int q0 = h_.fine_of_coarse[p], q1 = h_.fine_of_coarse[p + 1];
      const double dt1 = (t1[p + 1] - t1[p]) * dt;
      const double t_right = t_n + t1[p + 1] * dt;
      // backward-Euler-form correction at the right coarse node
      launch_be_rhs(C_.get(), u_[q0], q1 - q0, so_.data() + q0, o1[p + 1], dt1, n, st);
      NewtonReport rep;
      newton_.solve(f1, t_right, dt1, C_.get(), u_[q1], W_.get(), stiff_, rep);
      ++d.implicit_solves;
      d.newton_f1_evals += rep.f_evals;
      if (!rep.converged)
        throw IntegrationFailure("mrsdc mode 2: Newton failed at coarse node " +
                                 std::to_string(p + 1) + ", sweep " + std::to_string(k) +
                                 ", residual " + std::to_string(rep.final_residual));
      f1.eval_device(t_right, W_.get(), s1[p]);
      n1[p + 1] = s1[p];
      ++d.f1_evals;
      for (int q = q0; q < q1; ++q) {
        const double dtq = (t2[q + 1] - t2[q]) * dt;
        const double* da[2];
        const double* db[2];
        double dc[2];
        int nd = 0;
        da[nd] = n1[p + 1], db[nd] = o1[p + 1], dc[nd] = dtq, ++nd;
        if (n2[q] != o2[q]) da[nd] = n2[q], db[nd] = o2[q], dc[nd] = dtq, ++nd;
        launch_sweep_update(u_[q + 1], u_[q], nd, da, db, dc, 0, nullptr, nullptr, dt, so_[q], n,
                            st);
        f2.eval_device(t_n + t2[q + 1] * dt, u_[q + 1], s2[q]);
        n2[q + 1] = s2[q];
        ++d.f2_evals;
      }
    }
    d.sweeps = k;
    o1 = n1;
    o2 = n2;
  }
  rs.end(o1, o2);
  f1_last_ = const_cast<double*>(o1[m1]);
  f2_last_ = const_cast<double*>(o2[m2]);
}

void DeviceMrsdc::step_mode2(RhsOp& f1, RhsOp& f2, const double* u0, double t_n, double dt,
                             const double* f01, const double* f02, double* u_out, double* f1_end,
                             double* f2_end, SweepDiag& d) {
  require(f1.dim() == f2.dim(), "mrsdc: f1/f2 dimension mismatch");
  ensure(f1.dim());
  const long long n = dim_;
  cudaStream_t st = f2.stream();
  d2d(u_[0], u0, n, st);
  const bool h1 = f01 && reuse_first_, h2 = f02 && reuse_first_;
  if (h1) d2d(f10_, f01, n, st);
  if (h2) d2d(f20_, f02, n, st);
  run2(f1, f2, t_n, dt, h1, h2, d);
  d2d(u_out, u_[h_.fine.intervals()], n, st);
  if (f1_end) d2d(f1_end, f1_last_, n, st);
  if (f2_end) d2d(f2_end, f2_last_, n, st);
}

void DeviceMrsdc::integrate(int mode, RhsOp& f1, RhsOp& f2, const double* u0, double t0,
                            double t1, int nsteps, double* u_out, SweepDiag& total) {
  require(nsteps >= 0, "integrate_mrsdc: negative step count");
  require(f1.dim() == f2.dim(), "mrsdc: f1/f2 dimension mismatch");
  ensure(f1.dim());
  const long long n = dim_;
  const int m2 = h_.fine.intervals();
  cudaStream_t st = f2.stream();
  d2d(u_[0], u0, n, st);
  const double dt = (t1 - t0) / std::max(nsteps, 1);
  for (int step = 0; step < nsteps; ++step) {
    SweepDiag d;
    const bool reuse = step > 0 && reuse_first_;
    if (mode == 2)
      run2(f1, f2, t0 + step * dt, dt, reuse, reuse, d);
    else
      run(f1, f2, t0 + step * dt, dt, reuse, reuse, d);
    std::swap(u_[0], u_[m2]);
    for (auto* set : {&f1a_, &f1b_})
      for (auto& p : *set)
        if (p == f1_last_) std::swap(p, f10_);
    for (auto* set : {&f2a_, &f2b_})
      for (auto& p : *set)
        if (p == f2_last_) std::swap(p, f20_);
    total.add(d);
  }
  d2d(u_out, u_[0], n, st);
}

void DeviceMrsdc::integrate_mode1(RhsOp& f1, RhsOp& f2, const double* u0, double t0, double t1,
                                  int nsteps, double* u_out, SweepDiag& total) {
  integrate(1, f1, f2, u0, t0, t1, nsteps, u_out, total);
}

void DeviceMrsdc::integrate_mode2(RhsOp& f1, RhsOp& f2, const double* u0, double t0, double t1,
                                  int nsteps, double* u_out, SweepDiag& total) {
  integrate(2, f1, f2, u0, t0, t1, nsteps, u_out, total);
}

}  // namespace smc
