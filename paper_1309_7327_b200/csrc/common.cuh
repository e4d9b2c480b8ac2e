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
  // Symmetric / antisymmetric halves of the upper rows (filled by
  // make_stencil): p[r][j] = (m[r][j] + m[r][L-j]) / 2,
  // q[r][j] = (m[r][j] - m[r][L-j]) / 2, r, j < S, L = 2S - 1; p[r][S-1] is
  // implied by the zero row sum and not read.
  double p[4][4];
  double q[4][4];
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
// wrap for indices a stencil reach away from [0, n): selects instead of the
// integer division (which costs a dependent multiply-high chain per call)
__host__ __device__ inline int wrap_near(int i, int n) {
  if (i < -n || i >= 2 * n) return wrap(i, n);
  return i < 0 ? i + n : i >= n ? i - n : i;
}

#ifdef __CUDACC__
// H_{i+1/2} = sum_mm a_{i+mm} (sum_nn M[mm][nn] u_{i+nn}) for one interface
// (stencil_kernel.hpp:13-25).  a[w], u[w] hold offsets w - (S - 1),
// w = 0 .. 2S-1.
//
// Evaluated through the central antisymmetry M[L-r][L-c] = -M[r][c]
// (L = 2S - 1): with the window's symmetric and
// antisymmetric parts s_j = u_j + u_{L-j}, d_j = u_j - u_{L-j} (j < S),
//   v_r     = sum_c M[r][c] u_c   = P_r + Q_r,
//   v_{L-r} = -sum_c M[r][c] u_{L-c} = Q_r - P_r,   r < S,
// with P_r = sum_j p[r][j] s_j and Q_r = sum_j q[r][j] d_j (StencilM::p, q).
// Each row of M sums to zero (constants are annihilated), so do the rows of
// p and P_r = sum_{j<S-1} p[r][j] (s_j - s_{S-1}).  That is 3S - 1 adds,
// S(2S - 1) multiply-adds and 2S adds for the 2S values v_r (47 FP64
// instructions for S = 4, 28 constants) instead of the 52 structural
// nonzeros, and the dot with a stays 2S: 55 per interface instead of 60.  The rounding
// differs from the reference's row order by a few ulps of the interface sum
// (~1e-13 of the field, inside the 1e-12 single-RHS bar the tests hold);
// the sequence is fixed, so every thread, tiling and kernel that forms an
// interface gets the same bits.
// s'_j = s_j - s_{S-1} (j < S-1; the rows of p sum to zero, so P_r needs
// only these) and d_j (j < S) of a window.
template <int S>
__device__ __forceinline__ void sd_parts(const double* u, double* sj, double* dj) {
  constexpr int L = 2 * S - 1;
  const double sl = __dadd_rn(u[S - 1], u[S]);
#pragma unroll
  for (int j = 0; j < S - 1; ++j) sj[j] = __dsub_rn(__dadd_rn(u[j], u[L - j]), sl);
#pragma unroll
  for (int j = 0; j < S; ++j) dj[j] = __dsub_rn(u[j], u[L - j]);
}
template <int S>
__device__ __forceinline__ void narrow_vsd(const double* u, const StencilM& M, double* v) {
  constexpr int L = 2 * S - 1;
  double sj[S], dj[S];
  sd_parts<S>(u, sj, dj);
#pragma unroll
  for (int r = 0; r < S; ++r) {
    double pr = __dmul_rn(M.p[r][0], sj[0]), qr = __dmul_rn(M.q[r][0], dj[0]);
#pragma unroll
    for (int j = 1; j < S - 1; ++j) pr = __fma_rn(M.p[r][j], sj[j], pr);
#pragma unroll
    for (int j = 1; j < S; ++j) qr = __fma_rn(M.q[r][j], dj[j], qr);
    v[r] = __dadd_rn(qr, pr);
    v[L - r] = __dsub_rn(qr, pr);
  }
}
template <int S>
__device__ __forceinline__ double narrow_adot(const double* a, const double* v) {
  double acc = __dmul_rn(a[0], v[0]);
#pragma unroll
  for (int r = 1; r < 2 * S; ++r) acc = __fma_rn(a[r], v[r], acc);
  return acc;
}
// Interface sum with the dot taken in row-pair order r, L-r (r < S), so each
// pair (P_r, Q_r) is consumed as soon as it is formed.
template <int S>
__device__ __forceinline__ double narrow_iface(const double* a, const double* u,
                                               const StencilM& M) {
  constexpr int L = 2 * S - 1;
  double sj[S], dj[S];
  sd_parts<S>(u, sj, dj);
  double acc;
#pragma unroll
  for (int r = 0; r < S; ++r) {
    double pr = __dmul_rn(M.p[r][0], sj[0]), qr = __dmul_rn(M.q[r][0], dj[0]);
#pragma unroll
    for (int j = 1; j < S - 1; ++j) pr = __fma_rn(M.p[r][j], sj[j], pr);
#pragma unroll
    for (int j = 1; j < S; ++j) qr = __fma_rn(M.q[r][j], dj[j], qr);
    acc = r == 0 ? __dmul_rn(a[0], __dadd_rn(qr, pr)) : __fma_rn(a[r], __dadd_rn(qr, pr), acc);
    acc = __fma_rn(a[L - r], __dsub_rn(qr, pr), acc);
  }
  return acc;
}

// The coefficient-side form of the same interface sum, for one coefficient
// window a shared by several fields (the NS velocities and eta):
//   H = sum_c u_c w_c,  w_c = sum_r M[r][c] a_r.
// By the central antisymmetry, with sigma_r = a_r + a_{L-r} and
// delta_r = a_r - a_{L-r} (r < S), w_c + w_{L-c} = 2 A_c and
// w_c - w_{L-c} = 2 B_c where A_c = sum_r p[r][c] delta_r and
// B_c = sum_r q[r][c] sigma_r.  Since the rows of p sum to zero so do the
// A_c, and H = sum_{c<S-1} A_c s'_c + sum_{c<S} B_c d_c with the same s'_c,
// d_c of the field window as narrow_vsd: constants in u are annihilated
// exactly.  The transform costs 2S + (S-1)S + S^2 = 36 operations (S = 4)
// once per coefficient window, each field then 11 + 7 = 18 instead of 55.
template <int S>
__device__ __forceinline__ void narrow_wform(const double* a, const StencilM& M, double* A,
                                             double* B) {
  constexpr int L = 2 * S - 1;
  double sg[S], dl[S];
#pragma unroll
  for (int r = 0; r < S; ++r) sg[r] = __dadd_rn(a[r], a[L - r]), dl[r] = __dsub_rn(a[r], a[L - r]);
#pragma unroll
  for (int c = 0; c < S - 1; ++c) {
    double x = __dmul_rn(M.p[0][c], dl[0]);
#pragma unroll
    for (int r = 1; r < S; ++r) x = __fma_rn(M.p[r][c], dl[r], x);
    A[c] = x;
  }
#pragma unroll
  for (int c = 0; c < S; ++c) {
    double x = __dmul_rn(M.q[0][c], sg[0]);
#pragma unroll
    for (int r = 1; r < S; ++r) x = __fma_rn(M.q[r][c], sg[r], x);
    B[c] = x;
  }
}
template <int S>
__device__ __forceinline__ double narrow_wdot(const double* A, const double* B, const double* u) {
  double sj[S], dj[S];
  sd_parts<S>(u, sj, dj);
  double acc = __dmul_rn(B[0], dj[0]);
#pragma unroll
  for (int c = 1; c < S; ++c) acc = __fma_rn(B[c], dj[c], acc);
#pragma unroll
  for (int c = 0; c < S - 1; ++c) acc = __fma_rn(A[c], sj[c], acc);
  return acc;
}

// Two independent interfaces in lockstep (same arithmetic as narrow_iface for
// each): every constant is used by two adjacent, independent instructions,
// which doubles the instruction-level parallelism of the chains.
template <int S>
__device__ __forceinline__ void narrow_iface2(const double* a0, const double* u0, const double* a1,
                                              const double* u1, const StencilM& M, double& h0,
                                              double& h1) {
  constexpr int L = 2 * S - 1;
  double s0[S], d0[S], s1[S], d1[S];
  sd_parts<S>(u0, s0, d0);
  sd_parts<S>(u1, s1, d1);
  double acc0, acc1;
#pragma unroll
  for (int r = 0; r < S; ++r) {
    double p0 = __dmul_rn(M.p[r][0], s0[0]), q0 = __dmul_rn(M.q[r][0], d0[0]);
    double p1 = __dmul_rn(M.p[r][0], s1[0]), q1 = __dmul_rn(M.q[r][0], d1[0]);
#pragma unroll
    for (int j = 1; j < S - 1; ++j) p0 = __fma_rn(M.p[r][j], s0[j], p0), p1 = __fma_rn(M.p[r][j], s1[j], p1);
#pragma unroll
    for (int j = 1; j < S; ++j) q0 = __fma_rn(M.q[r][j], d0[j], q0), q1 = __fma_rn(M.q[r][j], d1[j], q1);
    if (r == 0) {
      acc0 = __dmul_rn(a0[0], __dadd_rn(q0, p0));
      acc1 = __dmul_rn(a1[0], __dadd_rn(q1, p1));
    } else {
      acc0 = __fma_rn(a0[r], __dadd_rn(q0, p0), acc0);
      acc1 = __fma_rn(a1[r], __dadd_rn(q1, p1), acc1);
    }
    acc0 = __fma_rn(a0[L - r], __dsub_rn(q0, p0), acc0);
    acc1 = __fma_rn(a1[L - r], __dsub_rn(q1, p1), acc1);
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
