// Shared device/host helpers for the sm_100a RHS library.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace smc {

// Status codes of the C ABI (include/smc_b200.h).
enum Status : int { kOk = 0, kInvalid = 1, kIntegration = 2, kCuda = 3 };

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct IntegrationFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define SMC_CUDA(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::smc::CudaFailure(std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" + \
                               __FILE__ + ":" + std::to_string(__LINE__) + ")");          \
  } while (0)

// Kernel launches issued by the library (exported as smc_launch_count()).
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}

#define SMC_CHECK_LAUNCH()                 \
  do {                                     \
    ::smc::launch_counter().fetch_add(1);  \
    SMC_CUDA(cudaGetLastError());          \
  } while (0)

inline void require(bool ok, const std::string& what) {
  if (!ok) throw InvalidArgument(what);
}

// The 8x8 coupling matrix of the narrow operator (stencil.hpp:20-27), laid
// out [mm + S - 1][nn + S - 1].  Passed by value as a kernel parameter so
// every launch carries its own copy (kernel parameters live in the constant
// bank; DFMA reads them as c[0x0][...] operands at no issue cost).
struct StencilM {
  double m[8][8];
};

// Structural nonzeros of row r (PAPER.md:263-300 / :320-345): rows of the
// upper half start at column 0 and end at S + r; the lower half mirrors
// (row S is full, row S+1 starts at column 1, ...).
template <int S>
__host__ __device__ constexpr int row_lo(int r) {
  return r < S ? 0 : r - S;
}
template <int S>
__host__ __device__ constexpr int row_hi(int r) {
  return r < S ? S + r : 2 * S - 1;
}

__host__ __device__ inline int wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

#ifdef __CUDACC__
// H_{i+1/2} = sum_mm a_{i+mm} (sum_nn M[mm][nn] u_{i+nn}) for one interface.
// a[w], u[w] hold offsets w - (S - 1), w = 0 .. 2S-1.  Order fixed as in
// stencil_kernel.hpp:13-25 (mm ascending outer, nn ascending inner); explicit
// fma so the instruction sequence (and hence the bits) is the same no matter
// which thread or tiling computes the interface.
//
// Only the upper half of M is read: the lower rows are taken through the
// central antisymmetry M[r][c] = -M[2S-1-r][2S-1-c], so a
// kernel needs 26 (S = 4) distinct constants, which fit the uniform register
// file, instead of 52.  The products and their order are unchanged.
template <int S>
__device__ __forceinline__ double mcoef(const StencilM& M, int r, int c) {
  return M.m[r][c];
}
template <int S>
__device__ __forceinline__ double narrow_iface(const double* a, const double* u,
                                               const StencilM& M) {
  double acc;
#pragma unroll
  for (int r = 0; r < 2 * S; ++r) {
    constexpr int L = 2 * S - 1;
    const int lo = row_lo<S>(r), hi = row_hi<S>(r);
    double v;
    if (r < S) {
      v = M.m[r][lo] * u[lo];
#pragma unroll
      for (int c = lo + 1; c <= hi; ++c) v = __fma_rn(M.m[r][c], u[c], v);
      acc = (r == 0) ? a[0] * v : __fma_rn(a[r], v, acc);
    } else {
      // v_r = sum_c M[r][c] u_c = -sum_c M[L-r][L-c] u_c
      v = M.m[L - r][L - lo] * u[lo];
#pragma unroll
      for (int c = lo + 1; c <= hi; ++c) v = __fma_rn(M.m[L - r][L - c], u[c], v);
      acc = __fma_rn(-a[r], v, acc);
    }
  }
  return acc;
}

// Two independent interfaces in lockstep (same arithmetic as narrow_iface for
// each): every M entry is used by two adjacent, independent FMAs, which
// doubles the instruction-level parallelism of the dependent row chains.
template <int S>
__device__ __forceinline__ void narrow_iface2(const double* a0, const double* u0, const double* a1,
                                              const double* u1, const StencilM& M, double& h0,
                                              double& h1) {
  double acc0, acc1;
#pragma unroll
  for (int r = 0; r < 2 * S; ++r) {
    constexpr int L = 2 * S - 1;
    const int lo = row_lo<S>(r), hi = row_hi<S>(r);
    double v0, v1;
    if (r < S) {
      v0 = M.m[r][lo] * u0[lo];
      v1 = M.m[r][lo] * u1[lo];
#pragma unroll
      for (int c = lo + 1; c <= hi; ++c) {
        v0 = __fma_rn(M.m[r][c], u0[c], v0);
        v1 = __fma_rn(M.m[r][c], u1[c], v1);
      }
      if (r == 0) {
        acc0 = a0[0] * v0;
        acc1 = a1[0] * v1;
      } else {
        acc0 = __fma_rn(a0[r], v0, acc0);
        acc1 = __fma_rn(a1[r], v1, acc1);
      }
    } else {
      v0 = M.m[L - r][L - lo] * u0[lo];
      v1 = M.m[L - r][L - lo] * u1[lo];
#pragma unroll
      for (int c = lo + 1; c <= hi; ++c) {
        v0 = __fma_rn(M.m[L - r][L - c], u0[c], v0);
        v1 = __fma_rn(M.m[L - r][L - c], u1[c], v1);
      }
      acc0 = __fma_rn(-a0[r], v0, acc0);
      acc1 = __fma_rn(-a1[r], v1, acc1);
    }
  }
  h0 = acc0;
  h1 = acc1;
}

// 8th-order centred first derivative (stencil_kernel.hpp:48-54) from a
// 9-point window w[0..8] centred at w[4].
__device__ __forceinline__ double deriv8_w(const double* w, double inv_d) {
  const double c1 = 4.0 / 5.0, c2 = -1.0 / 5.0, c3 = 4.0 / 105.0, c4 = -1.0 / 280.0;
  double r = c1 * (w[5] - w[3]);
  r = __fma_rn(c2, w[6] - w[2], r);
  r = __fma_rn(c3, w[7] - w[1], r);
  r = __fma_rn(c4, w[8] - w[0], r);
  return r * inv_d;
}

#endif  // __CUDACC__

}  // namespace smc
