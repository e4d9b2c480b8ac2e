// Device backward-Euler Newton with a block-structured finite-difference
// Jacobian (see stiff.hpp).  Arithmetic follows the reference operation by
// operation without contraction (explicit _rn intrinsics), so the dense case
// reproduces stiff.cpp / matrix.cpp exactly.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>

#include "stiff.hpp"

namespace smc {
namespace {

struct BlockMap {
  long long B, nb;
  int inter;
  __device__ __forceinline__ long long at(long long b, long long j) const {
    return inter ? j * nb + b : b * B + j;
  }
};

int grid_for(long long n) {
  const long long want = (n + 255) / 256;
  const long long cap = static_cast<long long>(num_sms()) * 8;
  return static_cast<int>(std::max(1LL, std::min(want, cap)));
}

// delta = w - beta f(w) - c (stiff.cpp:54-58); slots[0] = max |delta|,
// slots[1] = max |w| (field.hpp:18-22).  A NaN never wins the max, as with
// std::max(r, NaN) == r in the reference.
__global__ void __launch_bounds__(256) be_residual_kernel(const double* w, const double* fw,
                                                          const double* c, double beta,
                                                          double* delta, long long n,
                                                          unsigned long long* slots) {
  double r = 0.0, m = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double d = __dsub_rn(__dsub_rn(w[i], __dmul_rn(beta, fw[i])), c[i]);
    delta[i] = d;
    const double ad = fabs(d), aw = fabs(w[i]);
    if (ad > r) r = ad;
    if (aw > m) m = aw;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(slots, static_cast<unsigned long long>(__double_as_longlong(r)));
    atomicMax(slots + 1, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// Column j of every block: h_b = sqrt(eps) max(|w|, atol), wp += h
// (fd_jacobian, stiff.cpp:19-24).
__global__ void __launch_bounds__(256) fd_perturb_kernel(const double* w, double* wp, double* h,
                                                         long long j, BlockMap bm, double atol,
                                                         double root_eps) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long b = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; b < bm.nb;
       b += stride) {
    const long long i = bm.at(b, j);
    const double a = fabs(w[i]);
    const double hv = __dmul_rn(root_eps, (a < atol) ? atol : a);
    h[b] = hv;
    wp[i] = __dadd_rn(w[i], hv);
  }
}

// J_b(r, j) = (f(wp) - f(w)) * (1 / h_b) (stiff.cpp:25-28); jac laid out
// [r][c][b] so the per-block threads of the LU read it coalesced.  Restores
// wp for the next column.
__global__ void __launch_bounds__(256) fd_column_kernel(const double* fp, const double* fw,
                                                        const double* w, double* wp,
                                                        const double* h, double* jac, long long j,
                                                        BlockMap bm) {
  const long long total = bm.B * bm.nb;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += stride) {
    const long long r = t / bm.nb, b = t - r * bm.nb;
    const long long k = bm.at(b, r);
    const double inv = 1.0 / h[b];
    jac[(r * bm.B + j) * bm.nb + b] = __dmul_rn(__dsub_rn(fp[k], fw[k]), inv);
    if (r == 0) {
      const long long i = bm.at(b, j);
      wp[i] = w[i];
    }
  }
}

// jg = I - beta J (stiff.cpp:63-65), then lu_factor (matrix.cpp:9-33) per
// block; a zero pivot in any block raises *flag.
__global__ void __launch_bounds__(128) lu_factor_kernel(double* jac, int* piv, double beta,
                                                        BlockMap bm, unsigned long long* flag) {
  const long long B = bm.B, nb = bm.nb;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long b = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; b < nb;
       b += stride) {
    auto m = [&](long long r, long long c) -> double& { return jac[(r * B + c) * nb + b]; };
    for (long long r = 0; r < B; ++r)
      for (long long c = 0; c < B; ++c)
        m(r, c) = __dsub_rn(r == c ? 1.0 : 0.0, __dmul_rn(beta, m(r, c)));
    for (long long col = 0; col < B; ++col) {
      long long best = col;
      double best_mag = fabs(m(col, col));
      for (long long r = col + 1; r < B; ++r) {
        const double mag = fabs(m(r, col));
        if (mag > best_mag) {
          best = r;
          best_mag = mag;
        }
      }
      piv[col * nb + b] = static_cast<int>(best);
      if (best_mag == 0.0) {
        atomicMax(flag, 1ull);
        break;
      }
      if (best != col)
        for (long long c = 0; c < B; ++c) {
          const double tmp = m(col, c);
          m(col, c) = m(best, c);
          m(best, c) = tmp;
        }
      const double inv = 1.0 / m(col, col);
      for (long long r = col + 1; r < B; ++r) {
        const double l = __dmul_rn(m(r, col), inv);
        m(r, col) = l;
        for (long long c = col + 1; c < B; ++c)
          m(r, c) = __dsub_rn(m(r, c), __dmul_rn(l, m(col, c)));
      }
    }
  }
}

// lu_solve (matrix.cpp:35-51) on each block of delta, then w -= delta
// (stiff.cpp:68).
__global__ void __launch_bounds__(128) lu_solve_update_kernel(const double* jac, const int* piv,
                                                              double* delta, double* w,
                                                              BlockMap bm) {
  const long long B = bm.B, nb = bm.nb;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long b = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; b < nb;
       b += stride) {
    auto m = [&](long long r, long long c) { return jac[(r * B + c) * nb + b]; };
    auto x = [&](long long r) -> double& { return delta[bm.at(b, r)]; };
    for (long long i = 0; i < B; ++i) {
      const long long p = piv[i * nb + b];
      if (p != i) {
        const double tmp = x(i);
        x(i) = x(p);
        x(p) = tmp;
      }
    }
    for (long long i = 1; i < B; ++i) {
      double s = x(i);
      for (long long j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(m(i, j), x(j)));
      x(i) = s;
    }
    for (long long i = B - 1; i >= 0; --i) {
      double s = x(i);
      for (long long j = i + 1; j < B; ++j) s = __dsub_rn(s, __dmul_rn(m(i, j), x(j)));
      x(i) = s / m(i, i);
    }
    for (long long r = 0; r < B; ++r) {
      const long long k = bm.at(b, r);
      w[k] = __dsub_rn(w[k], delta[k]);
    }
  }
}

// Small blocks (block <= 16): one thread per block, the block's iteration
// matrix staged in shared memory laid out [entry][thread] (conflict-free),
// factored and solved there: the Jacobian is read once and nothing but the
// solution is written back (the global-memory factor + solve pair above
// re-reads and re-writes every entry O(block) times).  B is a template
// parameter so every loop is unrolled at its exact trip count: a row's
// loads are issued together instead of one dependent shared-memory round
// trip per entry.  delta is replaced by the Newton update; w is updated by a
// separate kernel once the host has seen that no block was singular
// (stiff.cpp:66 breaks before it).
//
// Kept as the fallback (SMC_LU_LANES=0).  Measured on the NS chemistry at
// 128^3 (block 14): 7.8 ms per factor-and-solve with run-time B, 7.3 ms
// unrolled; the global pair about 9 ms.  It holds four warps per SM (54 KB
// of shared memory per warp).  lu_lane_kernel below takes 4.9 ms.
constexpr int kLuThreads = 32;
constexpr int kLuMaxB = 16;

template <int B>
__global__ void __launch_bounds__(kLuThreads) lu_smem_kernel(const double* jac, double* delta,
                                                             double beta, BlockMap bm,
                                                             unsigned long long* flag) {
  extern __shared__ double sh[];
  const long long nb = bm.nb;
  const int t = threadIdx.x;
  const long long b = blockIdx.x * static_cast<long long>(kLuThreads) + t;
  double* mat = sh;                     // [B*B][32]
  double* x = sh + B * B * kLuThreads;  // [B][32]
  auto m = [&](int r, int c) -> double& { return mat[(r * B + c) * kLuThreads + t]; };
  auto xv = [&](int r) -> double& { return x[r * kLuThreads + t]; };
  if (b >= nb) return;
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c < B; ++c)
      m(r, c) = __dsub_rn(r == c ? 1.0 : 0.0,
                          __dmul_rn(beta, jac[(static_cast<long long>(r) * B + c) * nb + b]));
#pragma unroll
  for (int r = 0; r < B; ++r) xv(r) = delta[bm.at(b, r)];
  unsigned long long piv = 0;  // 4 bits per column
#pragma unroll 1
  for (int col = 0; col < B; ++col) {
    int best = col;
    double best_mag = fabs(m(col, col));
#pragma unroll 1
    for (int r = col + 1; r < B; ++r) {
      const double mag = fabs(m(r, col));
      if (mag > best_mag) {
        best = r;
        best_mag = mag;
      }
    }
    piv |= static_cast<unsigned long long>(best) << (4 * col);
    if (best_mag == 0.0) {
      atomicMax(flag, 1ull);
      return;
    }
    double* rc = mat + (col * B) * kLuThreads + t;
    if (best != col) {
      double* rb = mat + (best * B) * kLuThreads + t;
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const double tmp = rc[c * kLuThreads];
        rc[c * kLuThreads] = rb[c * kLuThreads];
        rb[c * kLuThreads] = tmp;
      }
    }
    // the pivot row in registers (entries left of col are not used)
    double prow[B];
#pragma unroll
    for (int c = 0; c < B; ++c) prow[c] = c >= col ? rc[c * kLuThreads] : 0.0;
    double inv = 0.0;
#pragma unroll
    for (int c = 0; c < B; ++c)
      if (c == col) inv = 1.0 / prow[c];
#pragma unroll 1
    for (int r = col + 1; r < B; ++r) {
      double* rr = mat + (r * B) * kLuThreads + t;
      double row[B];
#pragma unroll
      for (int c = 0; c < B; ++c) row[c] = c >= col ? rr[c * kLuThreads] : 0.0;
      double l = 0.0;
#pragma unroll
      for (int c = 0; c < B; ++c)
        if (c == col) l = __dmul_rn(row[c], inv);
#pragma unroll
      for (int c = 0; c < B; ++c) {
        if (c == col) rr[c * kLuThreads] = l;
        if (c > col) rr[c * kLuThreads] = __dsub_rn(row[c], __dmul_rn(l, prow[c]));
      }
    }
  }
  // lu_solve (matrix.cpp:35-51), x in registers
  double xr[B];
#pragma unroll
  for (int i = 0; i < B; ++i) xr[i] = xv(i);
#pragma unroll
  for (int i = 0; i < B; ++i) {
    const int p = static_cast<int>((piv >> (4 * i)) & 15u);
    if (p != i) {  // x_i <-> x_p, p > i (a select chain keeps xr in registers)
      const double xi = xr[i];
      double xp = xi;
#pragma unroll
      for (int q = i + 1; q < B; ++q) xp = p == q ? xr[q] : xp;
#pragma unroll
      for (int q = i + 1; q < B; ++q) xr[q] = p == q ? xi : xr[q];
      xr[i] = xp;
    }
  }
#pragma unroll
  for (int i = 1; i < B; ++i) {
    double s = xr[i];
#pragma unroll
    for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(m(i, j), xr[j]));
    xr[i] = s;
  }
#pragma unroll
  for (int i = B - 1; i >= 0; --i) {
    double s = xr[i];
#pragma unroll
    for (int j = i + 1; j < B; ++j) s = __dsub_rn(s, __dmul_rn(m(i, j), xr[j]));
    xr[i] = s / m(i, i);
  }
#pragma unroll
  for (int r = 0; r < B; ++r) delta[bm.at(b, r)] = xr[r];
}

// 16 lanes per block, one row of the iteration matrix per lane in registers,
// 16 blocks per 256-thread CTA.
//   * The CTA stages its 16 blocks' Jacobian entries through shared memory
//     (each entry's 16 consecutive blocks are one 128-byte read).
//   * Rows never move: each lane tracks the position of its row in the
//     current order (a swap exchanges two positions).
//   * Pivot search (matrix.cpp:13-20): a 4-round shuffle max of the 64-bit
//     pattern of |m(., col)| (monotonic for non-negative doubles; NaN and
//     positions above col excluded), then a 4-round min of the position
//     among the rows holding it: the first maximum, as the reference's
//     strict '>' scan finds; a NaN diagonal keeps col.
//   * The pivot row goes through a shared-memory slot; every row below
//     eliminates itself against it: the reference's operations on the same
//     operands (matrix.cpp:21-31).
//   * lu_solve (matrix.cpp:35-51): the swaps of x are the row swaps, so the
//     lane of original row r starts from delta_r; forward and backward
//     substitution broadcast each finished x_j by shuffle and every row
//     subtracts in ascending j as the reference does.
constexpr int kLuCells = 16;
template <int B>
__global__ void __launch_bounds__(256, 4) lu_lane_kernel(const double* jac, double* delta,
                                                      double beta, BlockMap bm,
                                                      unsigned long long* flag) {
  __shared__ double stage[B * B][kLuCells + 1];
  __shared__ __align__(16) double slot[8][2][16];  // [warp][group][entry]
  const long long nb = bm.nb;
  const long long b0 = blockIdx.x * static_cast<long long>(kLuCells);
  const int ncell = static_cast<int>(nb - b0 < kLuCells ? nb - b0 : kLuCells);
  {
    constexpr int NE = B * B * kLuCells;
    double v[(NE + 255) / 256];
#pragma unroll
    for (int q = 0; q < (NE + 255) / 256; ++q) {
      const int e = threadIdx.x + 256 * q;
      const int rc = e / kLuCells, cc = e - rc * kLuCells;
      v[q] = e < NE && cc < ncell ? jac[rc * nb + b0 + cc] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < (NE + 255) / 256; ++q) {
      const int e = threadIdx.x + 256 * q;
      const int rc = e / kLuCells, cc = e - rc * kLuCells;
      if (e < NE) stage[rc][cc] = v[q];
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = lane >> 4, gl = gw * 16;
  const int g = warp * 2 + gw;
  const int r = lane & 15;
  const bool live = g < ncell;
  const long long b = b0 + g;
  double m[B];
#pragma unroll
  for (int c = 0; c < B; ++c)
    m[c] = r < B ? __dsub_rn(r == c ? 1.0 : 0.0, __dmul_rn(beta, stage[r * B + c][g])) : 0.0;
  double x = live && r < B ? delta[bm.at(b, r)] : 0.0;
  int pos = r < B ? r : 16;  // padding lanes never take part
  bool dead = !live;
  double* ps = slot[warp][gw];
  auto lane_of = [&](int p) {
    const unsigned bits = (__ballot_sync(0xffffffffu, pos == p) >> gl) & 0xffffu;
    return gl + __ffs(static_cast<int>(bits)) - 1;
  };
#pragma unroll
  for (int col = 0; col < B; ++col) {
    const double mg = fabs(m[col]);
    const bool cand = pos >= col && pos < B;
    const unsigned long long key =
        cand && !isnan(mg) ? static_cast<unsigned long long>(__double_as_longlong(mg)) + 1ull : 0ull;
    unsigned long long km = key;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, km, o, 16);
      km = ok > km ? ok : km;
    }
    int kp = cand && key == km ? pos : 16;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) kp = min(kp, __shfl_xor_sync(0xffffffffu, kp, o, 16));
    const bool nan_diag = ((__ballot_sync(0xffffffffu, pos == col && isnan(mg)) >> gl) & 0xffffu) != 0;
    const int best = nan_diag ? col : kp;
    if (!nan_diag && km == 1ull && !dead) {  // best_mag == 0: singular
      if (r == 0) atomicMax(flag, 1ull);
      dead = true;
    }
    if (pos == best) {
#pragma unroll
      for (int c = 0; c < B; ++c)
        if (c >= col) ps[c] = m[c];
    }
    if (pos == col)
      pos = best;
    else if (pos == best)
      pos = col;
    __syncwarp();
    double p[B];
#pragma unroll
    for (int c = 0; c < B; ++c) p[c] = c >= col ? ps[c] : 0.0;
    __syncwarp();
    const double inv = 1.0 / p[col];
    if (pos > col && pos < B) {
      const double l = __dmul_rn(m[col], inv);
      m[col] = l;
#pragma unroll
      for (int c = col + 1; c < B; ++c) m[c] = __dsub_rn(m[c], __dmul_rn(l, p[c]));
    }
  }
  // forward substitution with the unit lower factor
#pragma unroll
  for (int j = 0; j + 1 < B; ++j) {
    const double xj = __shfl_sync(0xffffffffu, x, lane_of(j));
    if (pos > j && pos < B) x = __dsub_rn(x, __dmul_rn(m[j], xj));
  }
  // backward substitution (the row at position k needs x_{k+1..B-1})
  double xs[B];
#pragma unroll
  for (int k = B - 1; k >= 0; --k) {
    double sk = x;
#pragma unroll
    for (int j = k + 1; j < B; ++j) sk = __dsub_rn(sk, __dmul_rn(m[j], xs[j]));
    const double xk = sk / m[k];
    xs[k] = __shfl_sync(0xffffffffu, xk, lane_of(k));
    if (pos == k && !dead) delta[bm.at(b, k)] = xk;
  }
}

// SMC_FD_FUSED=0 forces DeviceNewton's column loop even when f offers a
// fused block Jacobian (the two must agree bit for bit; see the tests).
bool fd_fused() {
  static const bool v = [] {
    const char* e = std::getenv("SMC_FD_FUSED");
    return !(e && std::atoi(e) == 0);
  }();
  return v;
}

// SMC_LU_LANES=0 selects the thread-per-block shared-memory kernel.
bool lu_lanes() {
  static const bool v = [] {
    const char* e = std::getenv("SMC_LU_LANES");
    return !(e && std::atoi(e) == 0);
  }();
  return v;
}

template <int B>
void launch_lu_b(const double* jac, double* delta, double beta, BlockMap bm,
                 unsigned long long* flag, cudaStream_t st) {
  const std::size_t shm = sizeof(double) * (B * B + B) * kLuThreads;
  static bool attr = false;
  if (!attr) {
    SMC_CUDA(cudaFuncSetAttribute(lu_smem_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(shm)));
    attr = true;
  }
  if (lu_lanes()) {
    lu_lane_kernel<B><<<static_cast<unsigned>((bm.nb + kLuCells - 1) / kLuCells), 256, 0, st>>>(
        jac, delta, beta, bm, flag);
  } else {
    lu_smem_kernel<B><<<static_cast<unsigned>((bm.nb + kLuThreads - 1) / kLuThreads), kLuThreads,
                        shm, st>>>(jac, delta, beta, bm, flag);
  }
  SMC_CHECK_LAUNCH();
}
template <int... Bs>
void launch_lu_any(int B, const double* jac, double* delta, double beta, BlockMap bm,
                   unsigned long long* flag, cudaStream_t st, std::integer_sequence<int, Bs...>) {
  ((B == Bs + 1 ? launch_lu_b<Bs + 1>(jac, delta, beta, bm, flag, st) : void()), ...);
}
void launch_lu_smem(int B, const double* jac, double* delta, double beta, BlockMap bm,
                     unsigned long long* flag, cudaStream_t st) {
  launch_lu_any(B, jac, delta, beta, bm, flag, st, std::make_integer_sequence<int, kLuMaxB>{});
}

// w -= delta (stiff.cpp:68)
__global__ void __launch_bounds__(256) sub_kernel(double* w, const double* delta, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    w[i] = __dsub_rn(w[i], delta[i]);
}

// bdf2_solve's right-hand side and guess (stiff.cpp:94-99)
__global__ void __launch_bounds__(256) bdf2_prep_kernel(const double* u_nm1, const double* u_n,
                                                        double rho, double denom, double* c,
                                                        double* guess, long long n) {
  const double a = __dmul_rn(__dadd_rn(1.0, rho), __dadd_rn(1.0, rho)), b = __dmul_rn(rho, rho);
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    c[i] = __dsub_rn(__dmul_rn(a, u_n[i]), __dmul_rn(b, u_nm1[i])) / denom;
    guess[i] = __dadd_rn(u_n[i], __dmul_rn(rho, __dsub_rn(u_n[i], u_nm1[i])));
  }
}

// slots[0] = max |full - half| (diff_norm), slots[1] = max |half| (max_norm)
__global__ void __launch_bounds__(256) stiff_norms_kernel(const double* full, const double* half,
                                                          long long n,
                                                          unsigned long long* slots) {
  double d = 0.0, m = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double a = fabs(__dsub_rn(full[i], half[i])), b = fabs(half[i]);
    if (a > d) d = a;
    if (b > m) m = b;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(slots, static_cast<unsigned long long>(__double_as_longlong(d)));
    atomicMax(slots + 1, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// Richardson correction on acceptance: half += w (half - full) (stiff.cpp:171-172)
__global__ void __launch_bounds__(256) stiff_correct_kernel(double* half, const double* full,
                                                            double w, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    half[i] = __dadd_rn(half[i], __dmul_rn(w, __dsub_rn(half[i], full[i])));
}

double bits_to_double(unsigned long long u) {
  double d;
  std::memcpy(&d, &u, sizeof(d));
  return d;
}

}  // namespace

DeviceNewton::DeviceNewton() {
  SMC_CUDA(cudaMallocHost(&host_slots_, 4 * sizeof(double)));
}

DeviceNewton::~DeviceNewton() {
  if (piv_) cudaFree(piv_);
  if (host_slots_) cudaFreeHost(host_slots_);
}

void DeviceNewton::ensure(long long dim, long long block) {
  if (dim == dim_ && block == block_) return;
  const long long nb = dim / block;
  fw_.resize(dim), fp_.resize(dim), wp_.resize(dim), delta_.resize(dim);
  jac_.resize(static_cast<std::size_t>(block) * block * nb);
  h_.resize(nb);
  slots_.resize(4);
  if (piv_n_ != block * nb) {
    if (piv_) cudaFree(piv_);
    piv_ = nullptr;
    SMC_CUDA(cudaMalloc(&piv_, sizeof(int) * block * nb));
    piv_n_ = block * nb;
  }
  dim_ = dim, block_ = block;
}

void DeviceNewton::solve(RhsOp& f, double t, double beta, const double* c, const double* guess,
                         double* w, const StiffOpts& o, NewtonReport& rep) {
  const long long dim = f.dim();
  const long long B = o.block > 0 ? o.block : dim;
  require(dim >= 1 && dim % B == 0, "solve_backward_euler: block must divide the dimension");
  require(o.max_newton_iters >= 0, "solve_backward_euler: negative iteration limit");
  ensure(dim, B);
  const BlockMap bm{B, dim / B, o.block > 0 && o.interleaved ? 1 : 0};
  cudaStream_t st = f.stream();
  const double root_eps = std::sqrt(DBL_EPSILON);  // stiff.cpp:19
  auto* slots = reinterpret_cast<unsigned long long*>(slots_.get());
  auto read_slots = [&](int n) {
    SMC_CUDA(cudaMemcpyAsync(host_slots_, slots_.get(), n * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
    SMC_CUDA(cudaStreamSynchronize(st));
  };
  if (w != guess)
    SMC_CUDA(cudaMemcpyAsync(w, guess, dim * sizeof(double), cudaMemcpyDeviceToDevice, st));
  rep = NewtonReport{};
  for (int iter = 0; iter < o.max_newton_iters; ++iter) {
    f.eval_device(t, w, fw_.get());
    ++rep.f_evals;
    SMC_CUDA(cudaMemsetAsync(slots_.get(), 0, 3 * sizeof(double), st));
    be_residual_kernel<<<grid_for(dim), 256, 0, st>>>(w, fw_.get(), c, beta, delta_.get(), dim,
                                                     slots);
    SMC_CHECK_LAUNCH();
    read_slots(2);
    unsigned long long u[2];
    std::memcpy(u, host_slots_, sizeof(u));
    double rnorm = bits_to_double(u[0]), wnorm = bits_to_double(u[1]);
    if (reduce_) rnorm = reduce_(rnorm), wnorm = reduce_(wnorm);
    rep.final_residual = rnorm;
    if (rnorm <= o.atol + o.rtol * wnorm) {
      rep.converged = true;
      break;
    }
    if (o.block > 0 && fd_fused() &&
        f.fd_block_jacobian(w, fw_.get(), jac_.get(), B, bm.inter, o.atol, root_eps)) {
      rep.f_evals += static_cast<int>(B);
    } else {
      SMC_CUDA(cudaMemcpyAsync(wp_.get(), w, dim * sizeof(double), cudaMemcpyDeviceToDevice, st));
      for (long long j = 0; j < B; ++j) {
        fd_perturb_kernel<<<grid_for(bm.nb), 256, 0, st>>>(w, wp_.get(), h_.get(), j, bm, o.atol,
                                                          root_eps);
        SMC_CHECK_LAUNCH();
        f.eval_device(t, wp_.get(), fp_.get());
        ++rep.f_evals;
        fd_column_kernel<<<grid_for(B * bm.nb), 256, 0, st>>>(fp_.get(), fw_.get(), w, wp_.get(),
                                                             h_.get(), jac_.get(), j, bm);
        SMC_CHECK_LAUNCH();
      }
    }
    unsigned long long flag;
    if (B <= kLuMaxB) {
      launch_lu_smem(static_cast<int>(B), jac_.get(), delta_.get(), beta, bm, slots + 2, st);
      read_slots(3);
      std::memcpy(&flag, host_slots_ + 2, sizeof(flag));
      if (reduce_) flag = reduce_(flag ? 1.0 : 0.0) > 0.0;
      if (flag) break;  // singular iteration matrix (stiff.cpp:66)
      sub_kernel<<<grid_for(dim), 256, 0, st>>>(w, delta_.get(), dim);
      SMC_CHECK_LAUNCH();
    } else {
      const int lu_grid = static_cast<int>(std::max(
          1LL, std::min((bm.nb + 127) / 128, static_cast<long long>(num_sms()) * 16)));
      lu_factor_kernel<<<lu_grid, 128, 0, st>>>(jac_.get(), piv_, beta, bm, slots + 2);
      SMC_CHECK_LAUNCH();
      read_slots(3);
      std::memcpy(&flag, host_slots_ + 2, sizeof(flag));
      if (reduce_) flag = reduce_(flag ? 1.0 : 0.0) > 0.0;
      if (flag) break;  // singular iteration matrix (stiff.cpp:66)
      lu_solve_update_kernel<<<lu_grid, 128, 0, st>>>(jac_.get(), piv_, delta_.get(), w, bm);
      SMC_CHECK_LAUNCH();
    }
    rep.iterations = iter + 1;
  }
}

namespace {

double bdf2_coeff(double rho) {  // stiff.cpp:118-121
  return -(1.0 + rho) * (1.0 + rho) / (6.0 * rho * (1.0 + 2.0 * rho));
}

}  // namespace

// The host step controller below follows stiff.cpp:115-188 statement for
// statement (rho_full / rho_mid / c_half / weight / the clamps): bitwise
// agreement with the reference's accepted-step sequence needs the same
// scalar arithmetic in the same order.  What is new is the device side:
// every implicit stage is a DeviceNewton solve (batched per-block LU, fused
// FD Jacobian) and the norms are device reductions read back once per step.
void integrate_stiff(RhsOp& f, const double* u0, double t0, double t1, double* u_out,
                     const StiffOpts& o, StiffStats* stats, const Reducer& reduce) {
  const long long dim = f.dim();
  cudaStream_t st = f.stream();
  StiffStats local;
  StiffStats& ss = stats ? *stats : local;
  ss = StiffStats{};
  const double span = t1 - t0;
  if (span == 0.0) {
    if (u_out != u0)
      SMC_CUDA(cudaMemcpyAsync(u_out, u0, dim * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return;
  }
  require(!(span < 0.0), "integrate_stiff: t1 must be >= t0");
  require(!(o.rtol <= 0.0 || o.atol < 0.0), "integrate_stiff: bad tolerances");
  DevBuf U(dim), Up(dim), Yf(dim), Ym(dim), Yh(dim), C(dim), Gs(dim), slots(2);
  double* u = U.get();
  double* u_prev = Up.get();
  double* y_half = Yh.get();
  SMC_CUDA(cudaMemcpyAsync(u, u0, dim * sizeof(double), cudaMemcpyDeviceToDevice, st));
  DeviceNewton newton;
  if (reduce) newton.set_reducer(reduce);
  auto be = [&](double t_new, double h, const double* un, double* out) {
    NewtonReport rep;
    newton.solve(f, t_new, h, un, un, out, o, rep);
    return rep.converged;
  };
  auto bdf2 = [&](double t_new, double h, double rho, const double* unm1, const double* un,
                  double* out) {
    const double denom = 1.0 + 2.0 * rho;
    bdf2_prep_kernel<<<grid_for(dim), 256, 0, st>>>(unm1, un, rho, denom, C.get(), Gs.get(), dim);
    SMC_CHECK_LAUNCH();
    NewtonReport rep;
    newton.solve(f, t_new, h * (1.0 + rho) / denom, C.get(), Gs.get(), out, o, rep);
    return rep.converged;
  };
  double host[2];
  double t = t0, h_prev = 0.0;
  double h = std::clamp(o.initial_step_fraction, 1e-12, 1.0) * span;
  const double h_min = 1e-14 * span;
  bool have_history = false;
  while (t < t1) {
    h = std::min(h, t1 - t);
    if (h < h_min)
      throw IntegrationFailure("integrate_stiff: step size collapsed at t = " + std::to_string(t));
    bool ok;
    double weight;
    if (!have_history) {
      ok = be(t + h, h, u, Yf.get()) && be(t + 0.5 * h, 0.5 * h, u, Ym.get()) &&
           be(t + h, 0.5 * h, Ym.get(), y_half);
      weight = 1.0;
    } else {
      const double rho_full = h / h_prev;
      const double rho_mid = 0.5 * h / h_prev;
      ok = bdf2(t + h, h, rho_full, u_prev, u, Yf.get()) &&
           bdf2(t + 0.5 * h, 0.5 * h, rho_mid, u_prev, u, Ym.get()) &&
           bdf2(t + h, 0.5 * h, 1.0, u, Ym.get(), y_half);
      const double c_full = bdf2_coeff(rho_full);
      const double c_half = ((4.0 / 3.0) * bdf2_coeff(rho_mid) + bdf2_coeff(1.0)) / 8.0;
      weight = std::clamp(c_half / (c_full - c_half), 0.05, 2.0);
    }
    if (!ok) {
      h *= 0.5;
      ++ss.rejected;
      continue;
    }
    SMC_CUDA(cudaMemsetAsync(slots.get(), 0, 2 * sizeof(double), st));
    stiff_norms_kernel<<<grid_for(dim), 256, 0, st>>>(
        Yf.get(), y_half, dim, reinterpret_cast<unsigned long long*>(slots.get()));
    SMC_CHECK_LAUNCH();
    SMC_CUDA(cudaMemcpyAsync(host, slots.get(), sizeof(host), cudaMemcpyDeviceToHost, st));
    SMC_CUDA(cudaStreamSynchronize(st));
    if (reduce) host[0] = reduce(host[0]), host[1] = reduce(host[1]);
    const double err = weight * host[0];
    const double p = have_history ? 3.0 : 2.0;
    const double tol = o.rtol * host[1] + o.atol;
    if (err <= tol) {
      stiff_correct_kernel<<<grid_for(dim), 256, 0, st>>>(y_half, Yf.get(), weight, dim);
      SMC_CHECK_LAUNCH();
      std::swap(u_prev, u);
      std::swap(u, y_half);
      t += h;
      h_prev = h;
      have_history = true;
      ++ss.accepted;
    } else {
      ++ss.rejected;
    }
    double factor = err > 0.0 ? 0.9 * std::pow(tol / err, 1.0 / p) : 5.0;
    factor = std::clamp(factor, 0.2, 5.0);
    h *= factor;
  }
  SMC_CUDA(cudaMemcpyAsync(u_out, u, dim * sizeof(double), cudaMemcpyDeviceToDevice, st));
  SMC_CUDA(cudaStreamSynchronize(st));
}

}  // namespace smc
