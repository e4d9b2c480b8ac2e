// Narrow-stencil variable-coefficient diffusion  sum_d (c_d U_d)_d  on sm_100a.
//
// Reference: the interface sums of nsdc::detail::narrow_interfaces<S> /
// narrow_interfaces_rows<S> (proj/core/src/stencil_kernel.hpp:13-44) composed
// as narrow_rhs_rows<S> composes them (proj/core/src/pde.cpp:85-129): every
// interface H_{i+1/2} is computed once and differenced, the y (and z)
// interface is carried from one row (plane) to the next.
//
// B200 mapping ("2.5-D" z-march, SURVEY.md §7 "Carried interface"):
//   * a CTA owns a TX x TY (x, y) tile and marches along z over KC planes;
//   * the z window (2S planes of U and c_z for the CTA's own columns) lives
//     in registers, so every z interface is computed once and carried;
//   * the current plane, with a 4-cell halo in x and y, is staged in shared
//     memory by cp.async (LDGSTS), double-buffered so plane k+1 lands while
//     plane k is being differenced;
//   * x and y interfaces of plane k are computed once each into shared
//     memory (TX+1 resp. TY+1 per line, the extra one by an idle lane group),
//     then differenced; the periodic wrap is folded into the load addresses,
//     so the product keeps the reference's ghost-free Field layout.
// The work is FP64-bound (341 flop / 24 B per cell); there
// is nothing GEMM-shaped here, so no tensor cores.
#include "common.cuh"
#include <algorithm>
#include <cstdlib>
#include <string>

#include "narrow.cuh"

namespace smc {

namespace {

constexpr int TX = 32;            // x extent of a tile (one warp row)
constexpr int TYW = 8;            // warps per CTA
constexpr int RPT = 2;            // rows per thread
constexpr int TY = TYW * RPT;     // y extent of a tile
constexpr int NTHREADS = TX * TYW;

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <int S, bool HAS_Y, bool SAME>
struct Smem {
  static constexpr int W = TX + 2 * S;                 // tile columns incl. halo
  static constexpr int H = HAS_Y ? TY + 2 * S : TY;    // tile rows incl. halo
  static constexpr int CELLS = W * H;
  static constexpr int FIELDS = SAME ? 2 : 3;          // u, c_x(, c_y)
  double tile[2][FIELDS][CELLS];
  double hx[TY][TX + 1];
  double hy[HAS_Y ? TY + 1 : 1][TX];
};

// In-plane source offsets of the tile cells this thread stages; identical
// for every plane, so computed once per CTA (wrap folded in).
template <int S, bool HAS_Y, bool SAME>
struct StagePlan {
  static constexpr int N = (Smem<S, HAS_Y, SAME>::CELLS + NTHREADS - 1) / NTHREADS;
  int off[N];
  __device__ void init(int x0, int y0, int nx, int ny) {
    using SM = Smem<S, HAS_Y, SAME>;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int e = threadIdx.x + i * NTHREADS;
      const int row = e / SM::W, col = e - row * SM::W;
      const int gx = wrap(x0 - S + col, nx);
      const int gy = HAS_Y ? wrap(y0 - S + row, ny) : wrap(y0 + row, ny);
      off[i] = e < SM::CELLS ? gy * nx + gx : -1;
    }
  }
};

template <int S, bool HAS_Y, bool SAME>
__device__ __forceinline__ void stage_plane(Smem<S, HAS_Y, SAME>& sm, int buf, const NarrowArgs& p,
                                            const StagePlan<S, HAS_Y, SAME>& plan,
                                            long long plane_off) {
  using SM = Smem<S, HAS_Y, SAME>;
  const double* u = p.u + plane_off;
  const double* cx = p.cx + plane_off;
  const double* cy = p.cy + plane_off;
#pragma unroll
  for (int i = 0; i < plan.N; ++i) {
    const int e = threadIdx.x + i * NTHREADS;
    if (i + 1 < plan.N || e < SM::CELLS) {
      const int g = plan.off[i];
      cp_async8(&sm.tile[buf][0][e], u + g);
      cp_async8(&sm.tile[buf][1][e], cx + g);
      if constexpr (!SAME) cp_async8(&sm.tile[buf][SM::FIELDS - 1][e], cy + g);
    }
  }
  cp_async_commit();
}

template <int S, bool HAS_Y, bool HAS_Z, bool SAME, bool HAS_SRC>
__global__ void __launch_bounds__(NTHREADS, 1)
    narrow_kernel(const NarrowArgs p, const StencilM M) {
  using SM = Smem<S, HAS_Y, SAME>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

  const int tiles_x = (p.nx + TX - 1) / TX;
  const int x0 = (blockIdx.x % tiles_x) * TX;
  const int y0 = (blockIdx.x / tiles_x) * TY;
  const int tx = threadIdx.x % TX;
  const int ty = threadIdx.x / TX;
  const int kend = p.kend < 0 ? p.nz : p.kend;
  const int k0 = p.kbeg + blockIdx.y * p.kc;
  const int k1 = min(k0 + p.kc, kend);
  const long long plane = static_cast<long long>(p.nx) * p.ny;

  // Own columns (wrapped so partial tiles stay in bounds; stores predicated).
  long long col_off[RPT];
  bool col_ok[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int gx = x0 + tx, gy = y0 + ty + TYW * j;
    col_ok[j] = gx < p.nx && gy < p.ny;
    col_off[j] = static_cast<long long>(wrap(gy, p.ny)) * p.nx + wrap(gx, p.nx);
  }
  auto zplane = [&](int k) -> long long {
    return static_cast<long long>(p.zwrap ? wrap(k, p.nz) : k) * plane;
  };

  // z window: offsets k-(S-1) .. k+S of U and c_z for the own columns.
  double wu[RPT][2 * S], wc[RPT][2 * S], hz_prev[RPT], pf_u[RPT], pf_c[RPT];
  if constexpr (HAS_Z) {
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
#pragma unroll
      for (int w = 0; w < 2 * S; ++w) {  // planes k0-S .. k0+S-1 (window of k0-1)
        const long long o = zplane(k0 - S + w) + col_off[j];
        wu[j][w] = __ldg(p.u + o);
        wc[j][w] = __ldg(p.cz + o);
      }
      hz_prev[j] = narrow_iface<S>(wc[j], wu[j], M);  // interface k0 - 1/2
      const long long o = zplane(k0 + S) + col_off[j];
      pf_u[j] = __ldg(p.u + o);
      pf_c[j] = __ldg(p.cz + o);
    }
  }

  StagePlan<S, HAS_Y, SAME> plan;
  plan.init(x0, y0, p.nx, p.ny);
  int buf = 0;
  stage_plane<S, HAS_Y, SAME>(sm, 0, p, plan, zplane(k0));

  for (int k = k0; k < k1; ++k) {
    cp_async_wait_all();
    __syncthreads();  // tile[buf] complete; hx/hy of the previous plane consumed
    if (k + 1 < k1) stage_plane<S, HAS_Y, SAME>(sm, buf ^ 1, p, plan, zplane(k + 1));

    double hz[RPT];
    if constexpr (HAS_Z) {
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
#pragma unroll
        for (int w = 0; w < 2 * S - 1; ++w) {
          wu[j][w] = wu[j][w + 1];
          wc[j][w] = wc[j][w + 1];
        }
        wu[j][2 * S - 1] = pf_u[j];
        wc[j][2 * S - 1] = pf_c[j];
        if (k + 1 < k1) {
          const long long o = zplane(k + 1 + S) + col_off[j];
          pf_u[j] = __ldg(p.u + o);
          pf_c[j] = __ldg(p.cz + o);
        }
      }
    }

    const double* tu = sm.tile[buf][0];
    const double* tcx = sm.tile[buf][1];
    const double* tcy = sm.tile[buf][SM::FIELDS - 1];
    constexpr int RY = HAS_Y ? S : 0;  // row offset of the tile interior

    // x interfaces x0+tx+1/2 of rows ty + 8j
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int r = ty + TYW * j;
      double a[2 * S], u[2 * S];
#pragma unroll
      for (int w = 0; w < 2 * S; ++w) {
        a[w] = tcx[(r + RY) * SM::W + tx + 1 + w];
        u[w] = tu[(r + RY) * SM::W + tx + 1 + w];
      }
      sm.hx[r][tx + 1] = narrow_iface<S>(a, u, M);
    }
    // the extra interface x0-1/2 of every row (one half-warp)
    if (ty == 0 && tx < TY) {
      const int r = tx;
      double a[2 * S], u[2 * S];
#pragma unroll
      for (int w = 0; w < 2 * S; ++w) {
        a[w] = tcx[(r + RY) * SM::W + w];
        u[w] = tu[(r + RY) * SM::W + w];
      }
      sm.hx[r][0] = narrow_iface<S>(a, u, M);
    }
    if constexpr (HAS_Y) {
      // y interfaces y0+r+1/2 of column tx
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int r = ty + TYW * j;
        double a[2 * S], u[2 * S];
#pragma unroll
        for (int w = 0; w < 2 * S; ++w) {
          a[w] = tcy[(r + 1 + w) * SM::W + tx + S];
          u[w] = tu[(r + 1 + w) * SM::W + tx + S];
        }
        sm.hy[r + 1][tx] = narrow_iface<S>(a, u, M);
      }
      if (ty == 1) {  // the extra interface y0-1/2 of every column
        double a[2 * S], u[2 * S];
#pragma unroll
        for (int w = 0; w < 2 * S; ++w) {
          a[w] = tcy[w * SM::W + tx + S];
          u[w] = tu[w * SM::W + tx + S];
        }
        sm.hy[0][tx] = narrow_iface<S>(a, u, M);
      }
    }
    if constexpr (HAS_Z) {
#pragma unroll
      for (int j = 0; j < RPT; ++j) hz[j] = narrow_iface<S>(wc[j], wu[j], M);
    }
    __syncthreads();

    const long long po = zplane(k);
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int r = ty + TYW * j;
      // (dHx)/dx^2 + (dHy)/dy^2 + (dHz)/dz^2 [+ g0 g(t)], pde.cpp:118-126 order
      double o = __dmul_rn(__dsub_rn(sm.hx[r][tx + 1], sm.hx[r][tx]), p.idx2);
      if constexpr (HAS_Y)
        o = __dadd_rn(o, __dmul_rn(__dsub_rn(sm.hy[r + 1][tx], sm.hy[r][tx]), p.idy2));
      if constexpr (HAS_Z) {
        o = __dadd_rn(o, __dmul_rn(__dsub_rn(hz[j], hz_prev[j]), p.idz2));
        hz_prev[j] = hz[j];
      }
      if (col_ok[j]) {
        if constexpr (HAS_SRC) o = __dadd_rn(o, __dmul_rn(p.g0[po + col_off[j]], p.gt));
        p.out[po + col_off[j]] = o;
      }
    }
    buf ^= 1;
  }
}

template <int S, bool HAS_Y, bool HAS_Z, bool SAME, bool HAS_SRC>
void launch_t(const NarrowArgs& p, const StencilM& M, cudaStream_t st) {
  using SM = Smem<S, HAS_Y, SAME>;
  auto kern = narrow_kernel<S, HAS_Y, HAS_Z, SAME, HAS_SRC>;
  static bool configured = false;
  if (!configured) {
    SMC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(SM))));
    configured = true;
  }
  const int tiles = ((p.nx + TX - 1) / TX) * ((p.ny + TY - 1) / TY);
  const int kend = p.kend < 0 ? p.nz : p.kend;
  if (kend <= p.kbeg) return;
  const dim3 grid(tiles, (kend - p.kbeg + p.kc - 1) / p.kc);
  kern<<<grid, NTHREADS, sizeof(SM), st>>>(p, M);
  SMC_CHECK_LAUNCH();
}

template <int S>
void launch_s(const NarrowArgs& p, const StencilM& M, cudaStream_t st) {
  const bool same = p.cx == p.cy && p.cy == p.cz;
  if (p.dims == 3) {
    require(same, "narrow3d: one coefficient field shared by all directions");
    require(p.g0 == nullptr, "narrow3d: no source term");
    if (p.use_fast && narrow3d_fast_applicable(p))
      launch_narrow3d_fast(p, S, M, st);
    else
      launch_t<S, true, true, true, false>(p, M, st);
  } else if (p.dims == 2) {
    if (p.use_fast && narrow2d_fast_applicable(p))
      launch_narrow2d_fast(p, S, M, st);
    else if (p.g0)
      launch_t<S, true, false, false, true>(p, M, st);
    else
      launch_t<S, true, false, false, false>(p, M, st);
  } else {
    launch_t<S, false, false, true, false>(p, M, st);
  }
}

}  // namespace

int narrow_default_kc(int nx, int ny, int nz, int dims, int num_sms) {
  if (dims < 3) return 1;
  if (nx % 64 == 0 && ny % 8 == 0) return narrow3d_fast_default_kc(nx, ny, nz, num_sms);
  const long long tiles = static_cast<long long>((nx + TX - 1) / TX) * ((ny + TY - 1) / TY);
  // ~8 CTAs per SM slot pair in flight over the run, but at least 8 planes
  // per CTA so the 2S-plane window warm-up stays below ~50% extra z loads.
  const long long target = 8LL * 2 * num_sms;
  long long kc = (tiles * nz + target - 1) / target;
  if (kc < 8) kc = 8;
  if (kc > nz) kc = nz;
  return static_cast<int>(kc);
}

void launch_narrow(const NarrowArgs& p, int s, const StencilM& M, cudaStream_t st) {
  require(s == 3 || s == 4, "narrow: half width must be 3 or 4");
  require(p.kc >= 1, "narrow: kc >= 1");
  require(!p.zpeer || (p.use_fast && narrow3d_fast_applicable(p) && p.u_lo && p.u_hi),
          "narrow: the peer halo needs the fast 3-D kernel (nx % 32, ny % 8, 16-byte "
          "aligned fields) and both neighbour arrays");
  if (s == 4)
    launch_s<4>(p, M, st);
  else
    launch_s<3>(p, M, st);
}

// ----------------------------------------------------------- wide route
// D(a D u) as two passes of the 8th-order first derivative
// (pde.cpp:131-194, stencil.cpp:171-176).  Memory-bound, one thread per cell.
namespace {

__device__ __forceinline__ double d8_line(const double* f, long long base, int q, int n,
                                          long long stride, double inv_d) {
  double w[9];
#pragma unroll
  for (int d = -4; d <= 4; ++d) w[d + 4] = __ldg(f + base + static_cast<long long>(wrap(q + d, n)) * stride);
  return deriv8_w(w, inv_d);
}

__global__ void wide_pass1(const double* __restrict__ u, const double* __restrict__ a,
                           const double* __restrict__ b, double* __restrict__ w1,
                           double* __restrict__ w2, int nx, int ny, double inv_dx,
                           double inv_dy) {
  const long long n = static_cast<long long>(nx) * ny;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(c % nx), j = static_cast<int>(c / nx);
    w1[c] = a[c] * d8_line(u, static_cast<long long>(j) * nx, i, nx, 1, inv_dx);
    if (w2) w2[c] = b[c] * d8_line(u, i, j, ny, nx, inv_dy);
  }
}

__global__ void wide_pass2(const double* __restrict__ w1, const double* __restrict__ w2,
                           const double* __restrict__ g0, double gt, double* __restrict__ out,
                           int nx, int ny, double inv_dx, double inv_dy) {
  const long long n = static_cast<long long>(nx) * ny;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(c % nx), j = static_cast<int>(c / nx);
    double o = d8_line(w1, static_cast<long long>(j) * nx, i, nx, 1, inv_dx);
    if (w2) o = __dadd_rn(o, d8_line(w2, i, j, ny, nx, inv_dy));
    if (g0) o = __dadd_rn(o, __dmul_rn(g0[c], gt));
    out[c] = o;
  }
}

__global__ void deriv8_kernel(const double* __restrict__ u, double* __restrict__ out, int nx,
                              int ny, int nz, int dir, double inv_d) {
  const long long n = static_cast<long long>(nx) * ny * nz;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(c % nx);
    const long long jk = c / nx;
    const int j = static_cast<int>(jk % ny), k = static_cast<int>(jk / ny);
    const int q = dir == 0 ? i : dir == 1 ? j : k;
    const int len = dir == 0 ? nx : dir == 1 ? ny : nz;
    const long long stride = dir == 0 ? 1 : dir == 1 ? nx : static_cast<long long>(nx) * ny;
    out[c] = d8_line(u, c - q * stride, q, len, stride, inv_d);
  }
}

int grid_for(long long n) {
  long long b = (n + 255) / 256;
  return static_cast<int>(b > 148 * 64 ? 148 * 64 : (b < 1 ? 1 : b));
}

// Single-pass wide route: a CTA owns a WX x WY tile, stages u with an 8-cell
// halo (w1 = a D_x u is needed 4 cells past the tile in x, and D_x of u 4
// further), a (x halo 4) and b (y halo 4), forms w1 / w2 on the tile's
// extended rows / columns in shared memory and differences them: one read
// of u, a, b and one write per point (32 B) instead of two passes with two
// temporaries (the reference's wide_pass1 / wide_pass2, pde.cpp:131-194,
// whose arithmetic and order it keeps, so the results are the same bits).
constexpr int WX = 32, WY = 32, WH = 4, WT = 512;
constexpr int UW = WX + 4 * WH, UH = WY + 4 * WH;  // u over [x0-8, x0+40) x [y0-8, y0+40)
struct WideSmem {  // a and b are read once each, straight from global memory
  double u[UH][UW];
  double w1[WY][WX + 2 * WH];  // x in [x0-4, x0+36), tile rows
  double w2[WY + 2 * WH][WX];  // tile columns, y in [y0-4, y0+36)
};

__device__ __forceinline__ double d8_at(const double* p, int stride, double inv_d) {
  double w[9];
#pragma unroll
  for (int d = -4; d <= 4; ++d) w[d + 4] = d == 0 ? 0.0 : p[d * stride];
  return deriv8_w(w, inv_d);
}

// rows [r0, r0 + nr) x columns [c0, c0 + nc) of field f (periodic) into the
// shared block dst (pitch nc): 16-byte loads when the rows do not wrap in x
// (every interior tile; x0 and the offsets are even), element loads else.
template <int NC>
__device__ __forceinline__ void stage(double* dst, const double* __restrict__ f, int r0, int nr,
                                      int c0, int nx, int ny) {
  const bool inside = c0 >= 0 && c0 + NC <= nx;
  if (inside) {
    for (int e = threadIdx.x; e < nr * (NC / 2); e += WT) {
      const int r = e / (NC / 2), c = 2 * (e % (NC / 2));
      const double2 v = __ldg(reinterpret_cast<const double2*>(
          f + static_cast<long long>(wrap(r0 + r, ny)) * nx + c0 + c));
      dst[r * NC + c] = v.x, dst[r * NC + c + 1] = v.y;
    }
  } else {
    for (int e = threadIdx.x; e < nr * NC; e += WT) {
      const int r = e / NC, c = e % NC;
      dst[e] = __ldg(f + static_cast<long long>(wrap(r0 + r, ny)) * nx + wrap(c0 + c, nx));
    }
  }
}

__global__ void __launch_bounds__(WT) wide_tiled(const double* __restrict__ u,
                                                 const double* __restrict__ a,
                                                 const double* __restrict__ b,
                                                 const double* __restrict__ g0, double gt,
                                                 double* __restrict__ out, int nx, int ny,
                                                 double inv_dx, double inv_dy) {
  extern __shared__ __align__(16) unsigned char wide_raw[];
  WideSmem& sm = *reinterpret_cast<WideSmem*>(wide_raw);
  const int x0 = blockIdx.x * WX, y0 = blockIdx.y * WY;
  const int tid = threadIdx.x;
  stage<UW>(&sm.u[0][0], u, y0 - 2 * WH, UH, x0 - 2 * WH, nx, ny);
  __syncthreads();
  // w1 = a D_x u on the tile rows, x in [x0-4, x0+36); w2 = b D_y u on the
  // tile columns, y in [y0-4, y0+36)
  for (int e = tid; e < WY * (WX + 2 * WH); e += WT) {
    const int r = e / (WX + 2 * WH), c = e % (WX + 2 * WH);
    const double ac = __ldg(a + static_cast<long long>(y0 + r) * nx + wrap(x0 - WH + c, nx));
    sm.w1[r][c] = ac * d8_at(&sm.u[r + 2 * WH][c + WH], 1, inv_dx);
  }
  for (int e = tid; e < (WY + 2 * WH) * WX; e += WT) {
    const int r = e / WX, c = e % WX;
    const double bc = __ldg(b + static_cast<long long>(wrap(y0 - WH + r, ny)) * nx + x0 + c);
    sm.w2[r][c] = bc * d8_at(&sm.u[r + WH][c + 2 * WH], UW, inv_dy);
  }
  __syncthreads();
  for (int e = tid; e < WX * WY; e += WT) {
    const int r = e / WX, c = e % WX;
    double o = d8_at(&sm.w1[r][c + WH], 1, inv_dx);
    o = __dadd_rn(o, d8_at(&sm.w2[r + WH][c], WX, inv_dy));
    const long long gi = static_cast<long long>(y0 + r) * nx + x0 + c;
    if (g0) o = __dadd_rn(o, __dmul_rn(g0[gi], gt));
    out[gi] = o;
  }
}

// Wide route as a y-march (the heat RHS's narrow2d_march layout): a CTA owns
// a segment of YW = 256 columns (128 threads, two adjacent columns each) and
// a chunk of rows.  Per row k:
//   x: w1 = a D_x u of row k goes to a shared row (own columns plus a
//      4-column halo each side, formed by two lanes of every warp) and, after
//      the row's barrier, D_x w1 at the own columns;
//   y: the thread's two columns of u rows k .. k+8 and of w2 = b D_y u rows
//      k-4 .. k+4 live in registers; each step shifts in u row k+8 and w2
//      row k+4.
// Staging (16-byte cp.async, YD rows ahead): u rows in a ring of 9 + YD rows
// with an 8-column halo -- a row arrives once, feeds the y windows as their
// leading row and eight steps later the x stencil as the centre row --, a
// rows (4-column halo), b rows (four rows ahead of a) and g0 rows in rings of
// YD + 1.  One read of u, a, b (and g0) and one write per point; the same
// arithmetic and order as wide_pass1 / wide_pass2 (the same bits as the two
// passes and as wide_tiled).
constexpr int YW = 256, YT = YW / 2, YH = 2 * WH;   // segment, threads, u halo (8)
constexpr int YUW = YW + 2 * YH;                    // staged u row: 272
constexpr int YW1 = YW + 2 * WH;                    // a / w1 row: 264
template <int D, bool SRC>
struct YMarchSmem {
  static constexpr int NU = 9 + D, NA = D + 1;  // ring depths
  double u[NU][YUW];          // u row r, columns x0-8 ..      (slot r % NU)
  double a[NA][YW1];          // a row r, columns x0-4 ..      (slot r % NA)
  double b[NA][YW];           // b row r + 4, own columns      (slot r % NA)
  double g[SRC ? NA : 1][YW]; // g0 row r, own columns
  double w1[2][YW1];          // w1 of rows of even / odd parity
};

__device__ __forceinline__ void cp16w(double* dst, const double* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}

template <int V>
struct YRot {
  static constexpr int value = V;
};

// D = staging distance in rows (one cp.async group per row).  Step k forms
// out row k from w1 row k (formed in step k - 1) and the y windows, then w1
// row k + 1, then stages row k + D; one barrier per row.  The y windows are
// register rings: a step of rotation R writes the new row into slot R and
// reads logical entry j from slot (j + R + 1) % 9, so the march is unrolled
// by nine and nothing is shifted.
template <int D, bool SRC>
__global__ void __launch_bounds__(YT, 4)
    wide_march(const double* __restrict__ u, const double* __restrict__ a,
               const double* __restrict__ b, const double* __restrict__ g0, double gt,
               double* __restrict__ out, int nx, int ny, int kc, double inv_dx, double inv_dy) {
  using Sm = YMarchSmem<D, SRC>;
  constexpr int NU = Sm::NU, NA = Sm::NA;
  extern __shared__ __align__(16) unsigned char ym_raw[];
  Sm& sm = *reinterpret_cast<Sm*>(ym_raw);
  const int segs = nx / YW;
  const int x0 = (blockIdx.x % segs) * YW;
  const int k0 = static_cast<int>(blockIdx.x / segs) * kc;
  const int k1 = min(k0 + kc, ny);
  const int cp = threadIdx.x, lane = cp & 31, wid = cp >> 5;
  const int col = x0 + 2 * cp;
  const long long plane = static_cast<long long>(nx) * ny;
  auto roff = [&](int k) { return static_cast<long long>(wrap(k, ny)) * nx; };
  auto ld2 = [&](const double* f, int k) {
    return __ldg(reinterpret_cast<const double2*>(f + roff(k) + col));
  };
  auto adv = [&](long long& ro) {  // next row, periodic
    ro += nx;
    if (ro >= plane) ro -= plane;
  };

  // this thread's 16-byte chunks: u (136 per row: threads 0..7 take two), a
  // (132: threads 0..3 take two), b and g0 (one each)
  const int uo0 = wrap(x0 - YH + 2 * cp, nx), uo1 = wrap(x0 - YH + 2 * (cp + YT), nx);
  const int ao0 = wrap(x0 - WH + 2 * cp, nx), ao1 = wrap(x0 - WH + 2 * (cp + YT), nx);
  const bool u2 = cp + YT < YUW / 2, a2 = cp + YT < YW1 / 2;
  auto stage_u = [&](int s, long long ro) {
    double* d = sm.u[s];
    cp16w(d + 2 * cp, u + ro + uo0);
    if (u2) cp16w(d + 2 * (cp + YT), u + ro + uo1);
  };
  // one group per row r: u row r + 8, a / g0 row r, b row r + 4 (slots and
  // row offsets advanced incrementally)
  int st_r = k0, st_su = (k0 + 8) % NU, st_sa = k0 % NA;
  long long st_ru = roff(k0 + 8), st_ra = roff(k0), st_rb = roff(k0 + 4);
  auto stage_next = [&]() {
    if (st_r < k1) {
      stage_u(st_su, st_ru);
      cp16w(sm.a[st_sa] + 2 * cp, a + st_ra + ao0);
      if (a2) cp16w(sm.a[st_sa] + 2 * (cp + YT), a + st_ra + ao1);
      cp16w(sm.b[st_sa] + 2 * cp, b + st_rb + col);
      if constexpr (SRC) cp16w(sm.g[st_sa] + 2 * cp, g0 + st_ra + col);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    ++st_r;
    st_su = st_su + 1 == NU ? 0 : st_su + 1;
    st_sa = st_sa + 1 == NA ? 0 : st_sa + 1;
    adv(st_ru), adv(st_ra), adv(st_rb);
  };
  // the w1 halo column of this lane (lanes 0, 1 of every warp: 8 columns)
  const int h = 2 * wid + lane;                            // 0 .. 7 for lane < 2
  const int hc = h < WH ? h : YW + h;                      // w1 row index (0..3, 260..263)
  // w1 = a D_x u of a staged row into w1[par]
  auto form_w1 = [&](int su, int sa, int par) {
    const double* ur = sm.u[su];
    const double* ar = sm.a[sa];
    double* w1 = sm.w1[par];
    const double2 ak = *reinterpret_cast<const double2*>(ar + WH + 2 * cp);
    double w[10];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const double2 v = *reinterpret_cast<const double2*>(ur + 2 * cp + WH + 2 * j);
      w[2 * j] = v.x, w[2 * j + 1] = v.y;
    }
    *reinterpret_cast<double2*>(w1 + WH + 2 * cp) =
        make_double2(ak.x * deriv8_w(w, inv_dx), ak.y * deriv8_w(w + 1, inv_dx));
    if (lane < 2) {
      double wh[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) wh[j] = ur[hc + j];
      w1[hc] = ar[hc] * deriv8_w(wh, inv_dx);
    }
  };

  // prologue: the centre rows k0 .. k0+7 (one group), then rows k0 .. k0+D-1
  {
    long long ro = roff(k0);
    for (int r = k0; r < k0 + 8; ++r) {
      stage_u(r % NU, ro);
      adv(ro);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
#pragma unroll
  for (int i = 0; i < D; ++i) stage_next();

  // y rings: after the warm-up (rotation 8 -- eight pushes from rotation 0),
  // logical uw[j] = u row k + j, ww[j] = w2 row k - 4 + j at the next push
  double2 pu[9], pw[9];
  auto w2_of = [&](const double2* w, int rot, double2 bv) {  // b * D_y u, logical window
    double tx[9], ty[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) tx[j] = w[(j + rot) % 9].x, ty[j] = w[(j + rot) % 9].y;
    return make_double2(bv.x * deriv8_w(tx, inv_dy), bv.y * deriv8_w(ty, inv_dy));
  };
  // warm-up from global memory: u rows k0-8 .. k0+7 -> w2 rows k0-4 .. k0+3;
  // the loads are issued together
#pragma unroll
  for (int j = 1; j < 9; ++j) pu[j] = ld2(u, k0 - 9 + j);
  pu[0] = pw[0] = make_double2(0.0, 0.0);
  {
    double2 wu8[8], wb8[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) wu8[r] = ld2(u, k0 + r), wb8[r] = ld2(b, k0 - 4 + r);
#pragma unroll
    for (int r = 0; r < 8; ++r) {  // push of rotation r
      pu[r] = wu8[r];
      pw[r] = w2_of(pu, r + 1, wb8[r]);
    }
  }
  // row k0's group landed everywhere -> w1 row k0; then rows through k0 + 1
  asm volatile("cp.async.wait_group %0;\n" ::"n"(D - 1) : "memory");
  __syncthreads();
  form_w1(k0 % NU, k0 % NA, 0);
  asm volatile("cp.async.wait_group %0;\n" ::"n"(D - 2) : "memory");
  __syncthreads();

  int su8 = (k0 + 8) % NU, sa = k0 % NA, su1 = (k0 + 1) % NU, sa1 = (k0 + 1) % NA;
  long long oo = static_cast<long long>(k0) * nx + col;
  auto step = [&](auto rc, int k) {
    constexpr int R = decltype(rc)::value;
    const int par = (k - k0) & 1;
    // ---- y: push u row k+8 and w2 row k+4 (b row k+4), both staged
    pu[R] = *reinterpret_cast<const double2*>(&sm.u[su8][YH + 2 * cp]);
    pw[R] = w2_of(pu, R + 1, *reinterpret_cast<const double2*>(&sm.b[sa][2 * cp]));
    // ---- out row k = D_x w1 + D_y w2 (+ g0 g(t)), wide_pass2's order
    {
      const double* w1 = sm.w1[par];
      double w[10];
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(w1 + 2 * cp + 2 * j);
        w[2 * j] = v.x, w[2 * j + 1] = v.y;
      }
      double tx[9], ty[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) tx[j] = pw[(j + R + 1) % 9].x, ty[j] = pw[(j + R + 1) % 9].y;
      double o0 = __dadd_rn(deriv8_w(w, inv_dx), deriv8_w(tx, inv_dy));
      double o1 = __dadd_rn(deriv8_w(w + 1, inv_dx), deriv8_w(ty, inv_dy));
      if constexpr (SRC) {
        const double2 g = *reinterpret_cast<const double2*>(&sm.g[sa][2 * cp]);
        o0 = __dadd_rn(o0, __dmul_rn(g.x, gt));
        o1 = __dadd_rn(o1, __dmul_rn(g.y, gt));
      }
      *reinterpret_cast<double2*>(out + oo) = make_double2(o0, o1);
    }
    // ---- w1 row k + 1 (its rows landed at the last barrier); stage row k +
    //      D into the slots of row k - 1, all read before the last barrier
    if (k + 1 < k1) form_w1(su1, sa1, par ^ 1);
    stage_next();
    asm volatile("cp.async.wait_group %0;\n" ::"n"(D - 2) : "memory");
    __syncthreads();
    su8 = su8 + 1 == NU ? 0 : su8 + 1;
    su1 = su1 + 1 == NU ? 0 : su1 + 1;
    sa = sa + 1 == NA ? 0 : sa + 1;
    sa1 = sa1 + 1 == NA ? 0 : sa1 + 1;
    oo += nx;
  };
  int k = k0;
#pragma unroll 1
  for (; k + 9 <= k1; k += 9) {
    step(YRot<8>{}, k), step(YRot<0>{}, k + 1), step(YRot<1>{}, k + 2);
    step(YRot<2>{}, k + 3), step(YRot<3>{}, k + 4), step(YRot<4>{}, k + 5);
    step(YRot<5>{}, k + 6), step(YRot<6>{}, k + 7), step(YRot<7>{}, k + 8);
  }
  // the last < 9 rows
  if (k < k1) step(YRot<8>{}, k++);
  if (k < k1) step(YRot<0>{}, k++);
  if (k < k1) step(YRot<1>{}, k++);
  if (k < k1) step(YRot<2>{}, k++);
  if (k < k1) step(YRot<3>{}, k++);
  if (k < k1) step(YRot<4>{}, k++);
  if (k < k1) step(YRot<5>{}, k++);
  if (k < k1) step(YRot<6>{}, k++);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// SMC_WIDE = 2pass / tiled / march forces a route; by default the y-march
// where nx % 256 == 0 and the grid fills two waves, else the tiles.
int wide_mode() {
  static const int m = [] {
    const char* e = std::getenv("SMC_WIDE");
    if (!e) return 0;
    const std::string v(e);
    return v == "2pass" ? 1 : v == "tiled" ? 2 : v == "march" ? 3 : 0;
  }();
  return m;
}
bool wide_tiled_on() { return wide_mode() != 1; }


}  // namespace

void launch_wide2d(const double* u, const double* a, const double* b, const double* g0, double gt,
                   double* w1, double* w2, double* out, int nx, int ny, double dx, double dy,
                   cudaStream_t st) {
  const long long n = static_cast<long long>(nx) * ny;
  if (b && nx % YW == 0 && ny >= 9 && wide_mode() != 1 && wide_mode() != 2) {
    int dev = 0, sms = 0;
    SMC_CUDA(cudaGetDevice(&dev));
    SMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long long segs = nx / YW;
    if (wide_mode() == 3 || segs * (ny / 16) >= sms) {
      // one wave of four CTAs per SM (4096^2: 37 chunks of 111 rows; chunks of
      // 32 / 37 / 56 / 64 / 111 rows: 0.126 / 0.116 / 0.113 / 0.122 / 0.105 ms),
      // chunks of at least 16 rows
      long long chunks = std::max(1LL, 4LL * sms / segs);
      chunks = std::max(1LL, std::min(chunks, static_cast<long long>(ny) / 16));
      int kc = static_cast<int>((ny + chunks - 1) / chunks);
      if (const char* e = std::getenv("SMC_WIDE_KC")) kc = std::max(1, std::atoi(e));
      const unsigned grid = static_cast<unsigned>(segs * ((ny + kc - 1) / kc));
      auto go = [&](auto kern, std::size_t sh) {
        static bool configured = false;  // one per instantiation
        if (!configured) {
          SMC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sh)));
          configured = true;
        }
        kern<<<grid, YT, sh, st>>>(u, a, b, g0, gt, out, nx, ny, kc, 1.0 / dx, 1.0 / dy);
      };
      // staging distance 3 rows (4 measured the same, and takes more shared memory)
      g0 ? go(wide_march<3, true>, sizeof(YMarchSmem<3, true>))
         : go(wide_march<3, false>, sizeof(YMarchSmem<3, false>));
      SMC_CHECK_LAUNCH();
      return;
    }
  }
  if (b && nx % WX == 0 && ny % WY == 0 && nx >= UW && wide_tiled_on()) {
    static bool configured = false;
    if (!configured) {
      SMC_CUDA(cudaFuncSetAttribute(wide_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sizeof(WideSmem))));
      configured = true;
    }
    wide_tiled<<<dim3(nx / WX, ny / WY), WT, sizeof(WideSmem), st>>>(u, a, b, g0, gt, out, nx,
                                                                     ny, 1.0 / dx, 1.0 / dy);
    SMC_CHECK_LAUNCH();
    return;
  }
  wide_pass1<<<grid_for(n), 256, 0, st>>>(u, a, b, w1, w2, nx, ny, 1.0 / dx, 1.0 / dy);
  SMC_CHECK_LAUNCH();
  wide_pass2<<<grid_for(n), 256, 0, st>>>(w1, w2, g0, gt, out, nx, ny, 1.0 / dx, 1.0 / dy);
  SMC_CHECK_LAUNCH();
}

void launch_deriv8(const double* u, double* out, int nx, int ny, int nz, int dir, double dx,
                   cudaStream_t st) {
  const long long n = static_cast<long long>(nx) * ny * nz;
  deriv8_kernel<<<grid_for(n), 256, 0, st>>>(u, out, nx, ny, nz, dir, 1.0 / dx);
  SMC_CHECK_LAUNCH();
}

}  // namespace smc
