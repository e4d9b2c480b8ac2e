// Non-periodic lines: the narrow diffusion operator (a u_x)_x and the first
// derivative with the physical-boundary closure of PAPER.md:449-461
// (SURVEY.md §8(f) 4).  The periodic kernels stay the hot path; these close a
// line at both ends the way the paper describes for walls and open
// boundaries:
//   cells 4 .. n-5        8th order (the periodic stencils)
//   cells 3, n-4          6th-order centred (narrow: the 6th-order matrix)
//   cells 2, n-3          4th-order centred (narrow: the zero-corner member
//                         of the 4th-order family; a = 1 gives the classic
//                         (-1, 16, -30, 16, -1) / 12)
//   cells 1, n-2          centred 2nd order (diffusion), biased 3rd order
//                         (advection)
//   cells 0, n-1          completely biased 2nd (diffusion) / 3rd
//                         (advection) order
// Characteristic boundary conditions themselves (which state the boundary
// cells are driven to) are the caller's; the closure is the discretisation.
// The CPU restatement is oracle/oracle.c or_apply_narrow_bounded /
// or_first_derivative_bounded (the parity checker of tests/test_gpu_bounded.py).
//
// Layout: nlines contiguous lines of n cells (line-major).  One thread per
// cell; operands come through the read-only cache (a line's 17-cell window is
// reused by its neighbours), so the kernel streams a, u once and writes out
// once: 24 B per cell (diffusion), 16 B (derivative).
#include "common.cuh"
#include "narrow.cuh"

namespace smc {

namespace {

struct BoundedM {
  double m8[8][8];  // [mm + 3][nn + 3]
  double m6[6][6];  // [mm + 2][nn + 2]
};

__device__ __forceinline__ double m4b(int r, int c) {
  // zero-corner 4th-order narrow matrix, [mm + 1][nn + 1]
  constexpr double k = 1.0 / 12.0;
  const double rows[4][4] = {{0.0, k, -k, 0.0},
                             {k, -0.75, 2.0 / 3.0, 0.0},
                             {0.0, -2.0 / 3.0, 0.75, -k},
                             {0.0, k, -k, 0.0}};
  return rows[r][c];
}

template <int S>
__device__ __forceinline__ double iface(const BoundedM& M, const double* __restrict__ a,
                                        const double* __restrict__ u, int i) {
  double acc = 0.0;
#pragma unroll
  for (int mm = -S + 1; mm <= S; ++mm) {
    double v = 0.0;
#pragma unroll
    for (int nn = -S + 1; nn <= S; ++nn) {
      const double c = S == 4   ? M.m8[mm + 3][nn + 3]
                       : S == 3 ? M.m6[mm + 2][nn + 2]
                                : m4b(mm + 1, nn + 1);
      if (c != 0.0 || S == 4) v = fma(c, __ldg(u + i + nn), v);
    }
    acc = fma(__ldg(a + i + mm), v, acc);
  }
  return acc;
}

__device__ __forceinline__ double iface_at(const BoundedM& M, const double* a, const double* u,
                                           int d, int i) {
  if (d >= 4) return iface<4>(M, a, u, i);
  if (d == 3) return iface<3>(M, a, u, i);
  if (d == 2) return iface<2>(M, a, u, i);
  return 0.5 * (__ldg(a + i) + __ldg(a + i + 1)) * (__ldg(u + i + 1) - __ldg(u + i));
}

__global__ void narrow_bounded_kernel(BoundedM M, const double* __restrict__ a,
                                      const double* __restrict__ u, double* __restrict__ out,
                                      int n, long long total, double dx) {
  const double id2 = 1.0 / (dx * dx);
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < total;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long base = c - c % n;
    const int i = static_cast<int>(c - base);
    const double* al = a + base;
    const double* ul = u + base;
    const int d = min(i, n - 1 - i);
    double r;
    if (d == 0) {
      const int s = i == 0 ? 1 : -1;  // one-sided towards the interior
      const double* ua = ul + i;
      const double* aa = al + i;
      const double ux = s * (-3.0 * __ldg(ua) + 4.0 * __ldg(ua + s) - __ldg(ua + 2 * s)) / (2.0 * dx);
      const double ax = s * (-3.0 * __ldg(aa) + 4.0 * __ldg(aa + s) - __ldg(aa + 2 * s)) / (2.0 * dx);
      const double uxx = (2.0 * __ldg(ua) - 5.0 * __ldg(ua + s) + 4.0 * __ldg(ua + 2 * s) -
                          __ldg(ua + 3 * s)) * id2;
      r = __ldg(aa) * uxx + ax * ux;
    } else {
      r = (iface_at(M, al, ul, d, i) - iface_at(M, al, ul, d, i - 1)) * id2;
    }
    out[c] = r;
  }
}

__global__ void deriv_bounded_kernel(const double* __restrict__ u, double* __restrict__ out, int n,
                                     long long total, double dx) {
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < total;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(c % n);
    const double* w = u + c;
    const int d = min(i, n - 1 - i);
    const int s = i < n - 1 - i ? 1 : -1;
    double v;
    if (d >= 4)
      v = (4.0 / 5.0) * (__ldg(w + 1) - __ldg(w - 1)) - (1.0 / 5.0) * (__ldg(w + 2) - __ldg(w - 2)) +
          (4.0 / 105.0) * (__ldg(w + 3) - __ldg(w - 3)) -
          (1.0 / 280.0) * (__ldg(w + 4) - __ldg(w - 4));
    else if (d == 3)
      v = 0.75 * (__ldg(w + 1) - __ldg(w - 1)) - 0.15 * (__ldg(w + 2) - __ldg(w - 2)) +
          (1.0 / 60.0) * (__ldg(w + 3) - __ldg(w - 3));
    else if (d == 2)
      v = (2.0 / 3.0) * (__ldg(w + 1) - __ldg(w - 1)) - (1.0 / 12.0) * (__ldg(w + 2) - __ldg(w - 2));
    else if (d == 1)
      v = s * (-2.0 * __ldg(w - s) - 3.0 * __ldg(w) + 6.0 * __ldg(w + s) - __ldg(w + 2 * s)) / 6.0;
    else
      v = s * (-11.0 * __ldg(w) + 18.0 * __ldg(w + s) - 9.0 * __ldg(w + 2 * s) +
               2.0 * __ldg(w + 3 * s)) / 6.0;
    out[c] = v / dx;
  }
}

int bounded_grid(long long total) {
  const long long b = (total + 255) / 256;
  return static_cast<int>(b < 148LL * 16 ? (b > 0 ? b : 1) : 148LL * 16);
}

}  // namespace

void launch_narrow_bounded(const StencilM& m8, const StencilM& m6, const double* a,
                           const double* u, double* out, int n, int nlines, double dx,
                           cudaStream_t st) {
  require(n >= 8, "narrow_bounded: need at least 8 cells per line");
  require(nlines >= 1, "narrow_bounded: nlines must be positive");
  require(dx > 0.0, "narrow_bounded: dx must be positive");
  BoundedM M;
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) M.m8[r][c] = m8.m[r][c];
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) M.m6[r][c] = m6.m[r][c];
  const long long total = static_cast<long long>(n) * nlines;
  narrow_bounded_kernel<<<bounded_grid(total), 256, 0, st>>>(M, a, u, out, n, total, dx);
  SMC_CHECK_LAUNCH();
}

void launch_deriv_bounded(const double* u, double* out, int n, int nlines, double dx,
                          cudaStream_t st) {
  require(n >= 8, "first_derivative_bounded: need at least 8 cells per line");
  require(nlines >= 1, "first_derivative_bounded: nlines must be positive");
  require(dx > 0.0, "first_derivative_bounded: dx must be positive");
  const long long total = static_cast<long long>(n) * nlines;
  deriv_bounded_kernel<<<bounded_grid(total), 256, 0, st>>>(u, out, n, total, dx);
  SMC_CHECK_LAUNCH();
}

}  // namespace smc
