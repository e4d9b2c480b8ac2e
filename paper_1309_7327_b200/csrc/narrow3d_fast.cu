// 3-D narrow operator, FP64-issue-optimised z-march (configs[1] hot kernel).
//
// Same arithmetic as narrow_kernel (narrow.cu) — every interface
// H_{i+1/2} = sum_m a_{i+m} sum_n M_mn u_{i+n} computed once in the fixed
// order of stencil_kernel.hpp:13-25, then differenced as pde.cpp:118-120 —
// laid out so that the FP64 pipe, not the issue slot, is the limit:
//   * CTA tile 32 (x) x 8 (y) of 128 threads (default; 64 x 8 of 256 threads
//     with SMC_NARROW_FX=64), a thread owns 2 adjacent x cells, so its x
//     window comes from 5 conflict-free 16-byte LDS per field and its y
//     window from 8 LDS.128 that serve both columns; at <= 168 registers
//     three CTAs (12 warps) share an SM;
//   * only the 26 upper-half entries of M are read (antisymmetry, see
//     narrow_iface), so they stay in uniform registers; the two cells'
//     interfaces are formed in lockstep (narrow_iface2) for ILP;
//   * the z window (2S planes of U and a for the 2 columns) lives in
//     registers and is shifted by moves: a compact loop body keeps the
//     instruction cache warm (the 2S-fold unrolled variant measured slower);
//   * the centre plane (with a 4-cell halo) is staged by 16-byte cp.async
//     two planes ahead (triple buffer); the z window's leading plane is
//     prefetched two planes ahead with LDG.128; all addresses are
//     precomputed, the z offset advances incrementally;
//   * one CTA barrier per plane (it publishes the y interfaces and, as every
//     thread first waits for its own copies of plane k+1, the next tile);
//   * x neighbours' interfaces come by warp shuffle, y neighbours' through
//     shared memory (double-buffered by plane parity); the tile-edge
//     interfaces (x0-1/2 of each row, y0-1/2 of each column) are packed into
//     warps 1-3.
// Measured variants kept out: 2 CTAs/SM at 128 registers
// with the y window split (spills), z interfaces formed last with the
// leading-plane load issued at the step start, a persistent grid.
// Requirements (else narrow.cu's general kernel runs): nx % tile width == 0,
// ny % 8 == 0, 16-byte aligned fields.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "narrow.cuh"

namespace smc {
namespace {

// Tile geometry.  FXT = tile width in x: 64 (256 threads, one CTA per SM at
// up to 255 registers) or 32 (128 threads, three CTAs per SM at <= 168
// registers: 12 warps per SM instead of 8).  A thread owns 2 adjacent x
// cells; LPR threads cover one tile row.
template <int FXT>
struct NG {
  static constexpr int FX = FXT;
  static constexpr int FY = 8;
  static constexpr int LPR = FX / 2;
  static constexpr int FT = LPR * FY;
  static constexpr int HALO = 4;                       // staged halo (>= S)
  static constexpr int SW = FX + 2 * HALO;             // tile columns
  static constexpr int SH = FY + 2 * HALO;             // tile rows
  static constexpr int CHUNKS = SH * SW / 2;           // 16-byte chunks per field per plane
  static constexpr int CPT = (CHUNKS + FT - 1) / FT;   // per thread (last partial)
  static constexpr int NBUF = 3;
  static constexpr int OCC = FXT == 64 ? 1 : 3;
};

template <int FXT>
struct FastSmem {
  using G = NG<FXT>;
  double tile[G::NBUF][2][G::SH * G::SW];  // u, a
  double hy[2][G::FY + 1][G::FX];          // y interfaces, double-buffered by plane parity
  double hxe[2][G::FY];                    // x0 - 1/2 interfaces
};

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_groups() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ double2 lds2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}

// One (tile, [k0, k1)) segment of the z-march.  PEER: ghost planes of U come
// from the neighbours' arrays (a separate instantiation, so the common path
// carries no per-plane pointer selection).
template <int S, int FXT, bool PEER>
__device__ __forceinline__ void march_segment(FastSmem<FXT>& sm, const NarrowArgs& p,
                                              const StencilM& M, int tile, int k0, int k1) {
  using G = NG<FXT>;
  constexpr int FX = G::FX, FY = G::FY, FT = G::FT, HALO = G::HALO, SW = G::SW;
  constexpr int CHUNKS = G::CHUNKS, CPT = G::CPT, NBUF = G::NBUF, LPR = G::LPR;
  constexpr int WIN = 2 * S;
  const int tiles_x = p.nx / FX;
  const int x0 = (tile % tiles_x) * FX;
  const int y0 = (tile / tiles_x) * FY;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int row = threadIdx.x / LPR;  // tile row of my cells
  const int cp = threadIdx.x % LPR;   // my column pair
  const long long plane = static_cast<long long>(p.nx) * p.ny;
  const long long zspan = plane * p.nz;

  // plane offset helpers (periodic wrap or ghosted slab)
  auto zoff = [&](int k) -> long long {
    if (p.zwrap) {
      k %= p.nz;
      if (k < 0) k += p.nz;
    }
    return static_cast<long long>(k) * plane;
  };
  auto zadv = [&](long long o) -> long long {
    o += plane;
    if (p.zwrap && o >= zspan) o -= zspan;
    return o;
  };

  // plane base of U (offset o = k * plane from the interior start): the peer
  // halo reads ghost planes from the neighbours' arrays
  auto ub = [&](long long o) -> const double* {
    if constexpr (!PEER) return p.u + o;
    if (o < 0) return p.u_lo + (p.lo_len + o);
    if (o >= zspan) return p.u_hi + (o - zspan);
    return p.u + o;
  };

  // staging plan: in-plane offsets of this thread's 16-byte chunks
  int soff[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = threadIdx.x + i * FT;
    const int r = c / (SW / 2), col = 2 * (c - r * (SW / 2));
    const int gx = wrap(x0 - HALO + col, p.nx);
    const int gy = wrap(y0 - HALO + r, p.ny);
    soff[i] = c < CHUNKS ? gy * p.nx + gx : 0;
  }
  auto stage = [&](int buf, long long po) {
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int c = threadIdx.x + i * FT;
      if (i + 1 < CPT || c < CHUNKS) {
        cp16(&sm.tile[buf][0][2 * c], ub(po) + soff[i]);
        cp16(&sm.tile[buf][1][2 * c], p.cz + po + soff[i]);
      }
    }
    commit();
  };

  // own columns: x0 + 2*cp + {0, 1}, row y0 + row
  const int col_off = (y0 + row) * p.nx + x0 + 2 * cp;
  auto ld2 = [&](const double* base, long long o) {
    return __ldg(reinterpret_cast<const double2*>(base + o + col_off));
  };
  auto ld2u = [&](long long o) {
    return __ldg(reinterpret_cast<const double2*>(ub(o) + col_off));
  };

  // z window (2 columns): slot j holds plane k - S + 1 + j at step k
  double2 wu[WIN], wa[WIN];
  double2 pf_u[2], pf_a[2];  // leading planes prefetched two ahead
  {
    long long o = zoff(k0 - S);
#pragma unroll
    for (int j = 0; j < WIN; ++j) {
      wu[j] = ld2u(o);
      wa[j] = ld2(p.cz, o);
      o = zadv(o);
    }
  }
  // leading planes k0 + S, k0 + S + 1 (never past k1 - 1 + S: a ghosted
  // slab has only S planes above its interior)
  long long o_pf = zoff(k0 + S);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    if (k0 + j < k1) {
      pf_u[j] = ld2u(o_pf);
      pf_a[j] = ld2(p.cz, o_pf);
    }
    o_pf = zadv(o_pf);
  }
  // centre-plane staging: planes k0, k0 + 1 now (buffers 0, 1)
  long long o_st = zoff(k0);
  stage(0, o_st);
  o_st = zadv(o_st);
  if (k0 + 1 < k1)
    stage(1, o_st);
  else
    commit();
  o_st = zadv(o_st);
  long long o_out = zoff(k0);

  // z interface k0 - 1/2 from the initial window (planes k0 - S .. k0 + S - 1)
  double hzp0, hzp1;
  {
    double a0[WIN], u0[WIN], a1[WIN], u1[WIN];
#pragma unroll
    for (int j = 0; j < WIN; ++j) a0[j] = wa[j].x, u0[j] = wu[j].x, a1[j] = wa[j].y, u1[j] = wu[j].y;
    hzp0 = narrow_iface<S>(a0, u0, M);
    hzp1 = narrow_iface<S>(a1, u1, M);
  }
  // plane k0's tile must be visible to every thread before the first step
  wait_groups<1>();
  __syncthreads();

  const double idx2 = p.idx2, idy2 = p.idy2, idz2 = p.idz2;

  // (dHx)/dx^2 + (dHy)/dy^2 + (dHz)/dz^2 of plane (parity hb), pde.cpp:118-120
  auto finish = [&](int hb, double hx0, double hx1, double hz0, double hz1, double hzl0,
                    double hzl1, long long oo) {
    double hxl = __shfl_up_sync(0xffffffffu, hx1, 1);
    if (cp == 0) hxl = sm.hxe[hb][row];
    const double2 yu = lds2(&sm.hy[hb][row][2 * cp]);
    const double2 yd = lds2(&sm.hy[hb][row + 1][2 * cp]);
    // x, y, z differences scaled and summed with two fused multiply-adds
    double o0 = __dmul_rn(__dsub_rn(hx0, hxl), idx2);
    double o1 = __dmul_rn(__dsub_rn(hx1, hx0), idx2);
    o0 = __fma_rn(__dsub_rn(yd.x, yu.x), idy2, o0);
    o1 = __fma_rn(__dsub_rn(yd.y, yu.y), idy2, o1);
    o0 = __fma_rn(__dsub_rn(hz0, hzl0), idz2, o0);
    o1 = __fma_rn(__dsub_rn(hz1, hzl1), idz2, o1);
    *reinterpret_cast<double2*>(p.out + oo + col_off) = make_double2(o0, o1);
  };

#pragma unroll 1
  for (int k = k0; k < k1; ++k) {
    const int t = k - k0;
    const int buf = t % NBUF;
    const int hb = t & 1;
    // z window: shift in the plane prefetched two steps ago
#pragma unroll
    for (int j = 0; j + 1 < WIN; ++j) wu[j] = wu[j + 1], wa[j] = wa[j + 1];
    wu[WIN - 1] = pf_u[0];
    wa[WIN - 1] = pf_a[0];
    pf_u[0] = pf_u[1];
    pf_a[0] = pf_a[1];
    if (k + 2 < k1) {
      pf_u[1] = ld2u(o_pf);
      pf_a[1] = ld2(p.cz, o_pf);
      o_pf = zadv(o_pf);
    }
    const double* tu = sm.tile[buf][0];
    const double* ta = sm.tile[buf][1];
    double hz0, hz1;
    {
      double a0[WIN], u0[WIN], a1[WIN], u1[WIN];
#pragma unroll
      for (int j = 0; j < WIN; ++j) a0[j] = wa[j].x, u0[j] = wu[j].x, a1[j] = wa[j].y, u1[j] = wu[j].y;
      narrow_iface2<S>(a0, u0, a1, u1, M, hz0, hz1);
    }
    // ---- x interfaces x+1/2 for my two cells (row HALO + row)
    double hx0, hx1;
    {
      // values at tile columns 2*cp + HALO - S + 1 + j
      constexpr int NV = WIN + 2;  // loaded in pairs
      constexpr int BASE = HALO - S + 1 - ((HALO - S + 1) & 1);  // even start
      constexpr int OFF = (HALO - S + 1) - BASE;                 // 0 or 1
      double ua[NV], aa[NV];
      const double* ru = tu + (HALO + row) * SW + 2 * cp + BASE;
      const double* ra = ta + (HALO + row) * SW + 2 * cp + BASE;
#pragma unroll
      for (int j = 0; j < NV / 2; ++j) {
        const double2 vu = lds2(ru + 2 * j), va = lds2(ra + 2 * j);
        ua[2 * j] = vu.x, ua[2 * j + 1] = vu.y;
        aa[2 * j] = va.x, aa[2 * j + 1] = va.y;
      }
      narrow_iface2<S>(aa + OFF, ua + OFF, aa + OFF + 1, ua + OFF + 1, M, hx0, hx1);
    }
    // ---- y interfaces y+1/2 for my two columns
    {
      double u0[WIN], a0[WIN], u1[WIN], a1[WIN];
#pragma unroll
      for (int j = 0; j < WIN; ++j) {
        const int r = HALO + row - S + 1 + j;
        const double2 vu = lds2(tu + r * SW + HALO + 2 * cp);
        const double2 va = lds2(ta + r * SW + HALO + 2 * cp);
        u0[j] = vu.x, u1[j] = vu.y, a0[j] = va.x, a1[j] = va.y;
      }
      double y0v, y1v;
      narrow_iface2<S>(a0, u0, a1, u1, M, y0v, y1v);
      *reinterpret_cast<double2*>(&sm.hy[hb][row + 1][2 * cp]) = make_double2(y0v, y1v);
    }
    // ---- extra interfaces: y0 - 1/2 of every column (warps 1 .. FX/32, one
    //      column per lane), x0 - 1/2 of each row (the next warp): FX/32 + 1
    //      warp issues of an interface (two half warps and an eighth of a
    //      warp measured 0.268-0.270 ms at 256^3)
    if (wid >= 1 && wid <= FX / 32) {
      const int c = (wid - 1) * 32 + lane;
      double uu[WIN], aa[WIN];
#pragma unroll
      for (int j = 0; j < WIN; ++j) {
        uu[j] = tu[(HALO - S + j) * SW + HALO + c];
        aa[j] = ta[(HALO - S + j) * SW + HALO + c];
      }
      sm.hy[hb][0][c] = narrow_iface<S>(aa, uu, M);
    } else if (wid == FX / 32 + 1 && lane < FY) {
      double uu[WIN], aa[WIN];
#pragma unroll
      for (int j = 0; j < WIN; ++j) {
        uu[j] = tu[(HALO + lane) * SW + HALO - S + j];
        aa[j] = ta[(HALO + lane) * SW + HALO - S + j];
      }
      sm.hxe[hb][lane] = narrow_iface<S>(aa, uu, M);
    }
    // ---- stage plane k + 2 into the buffer of plane k - 1 (all of its
    //      readers passed the previous barrier), then make plane k + 1 ready
    if (k + 2 < k1) {
      stage((t + 2) % NBUF, o_st);
      o_st = zadv(o_st);
    } else {
      commit();  // keep the group count uniform
    }
    wait_groups<1>();
    __syncthreads();
    finish(hb, hx0, hx1, hz0, hz1, hzp0, hzp1, o_out);
    o_out = zadv(o_out);
    hzp0 = hz0;
    hzp1 = hz1;
  }
  // drain the (empty) trailing groups; the next segment reuses the buffers
  wait_groups<0>();
  __syncthreads();
}

// Chunked grid (default): tile = blockIdx.x, planes [kbeg + y*kc, +kc), so
// co-scheduled CTAs are x/y neighbours at the same z and tile halos hit in
// L2.  Persistent grid: CTA b owns the contiguous range [b*L/G, (b+1)*L/G)
// of L = tile * nplanes + plane (one wave, equal work to within a plane).
template <int S, int FXT, bool PEER>
__global__ void __launch_bounds__(NG<FXT>::FT, NG<FXT>::OCC)
    narrow3d_fast(const NarrowArgs p, const StencilM M, int chunked) {
  using G = NG<FXT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FastSmem<FXT>& sm = *reinterpret_cast<FastSmem<FXT>*>(smem_raw);
  const int kend = p.kend < 0 ? p.nz : p.kend;
  if (chunked) {
    const int k0 = p.kbeg + blockIdx.y * p.kc;
    march_segment<S, FXT, PEER>(sm, p, M, blockIdx.x, k0, min(k0 + p.kc, kend));
    return;
  }
  const long long np = kend - p.kbeg;
  const long long total = static_cast<long long>(p.nx / G::FX) * (p.ny / G::FY) * np;
  const long long lo = total * blockIdx.x / gridDim.x;
  const long long hi = total * (blockIdx.x + 1) / gridDim.x;
  for (long long l = lo; l < hi;) {
    const int tile = static_cast<int>(l / np);
    const int kk = static_cast<int>(l - tile * np);
    const int len = static_cast<int>(min(np - kk, hi - l));
    march_segment<S, FXT, PEER>(sm, p, M, tile, p.kbeg + kk, p.kbeg + kk + len);
    l += len;
  }
}

// SMC_NARROW_GRID=persistent selects the one-wave persistent grid (tuning
// knob).  Both measure 0.295 ms at 256^3; the chunked grid keeps co-resident
// CTAs on neighbouring tiles, so it moves 2.9x fewer DRAM bytes (388 vs
// 925 MB per launch), which is the default.
bool chunked_grid() {
  static bool c = [] {
    const char* e = std::getenv("SMC_NARROW_GRID");
    return !(e && std::string(e) == "persistent");
  }();
  return c;
}

int num_sms_cached() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// SMC_NARROW_FX=32|64 selects the tile width (tuning knob); see NG.  32 (three
// CTAs of 4 warps per SM) measured 0.278 ms at 256^3 against 0.296 ms for 64
// (one CTA of 8 warps), so it is the default.
int fast_fx() {
  static int f = [] {
    const char* e = std::getenv("SMC_NARROW_FX");
    return (e && std::atoi(e) == 64) ? 64 : 32;
  }();
  return f;
}

template <int S, int FXT, bool PEER>
void launch_fast_s(const NarrowArgs& p, const StencilM& M, cudaStream_t st) {
  using G = NG<FXT>;
  static bool configured = false;
  if (!configured) {
    SMC_CUDA(cudaFuncSetAttribute(narrow3d_fast<S, FXT, PEER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(FastSmem<FXT>))));
    configured = true;
  }
  const int kend = p.kend < 0 ? p.nz : p.kend;
  if (kend <= p.kbeg) return;
  const int tiles = (p.nx / G::FX) * (p.ny / G::FY);
  if (chunked_grid()) {
    const dim3 grid(tiles, (kend - p.kbeg + p.kc - 1) / p.kc);
    narrow3d_fast<S, FXT, PEER><<<grid, G::FT, sizeof(FastSmem<FXT>), st>>>(p, M, 1);
  } else {
    const long long work = static_cast<long long>(tiles) * (kend - p.kbeg);
    const long long by_kc = (work + p.kc - 1) / p.kc;
    const int grid =
        static_cast<int>(std::max(1LL, std::min<long long>(num_sms_cached() * G::OCC, by_kc)));
    narrow3d_fast<S, FXT, PEER><<<grid, G::FT, sizeof(FastSmem<FXT>), st>>>(p, M, 0);
  }
  SMC_CHECK_LAUNCH();
}

}  // namespace

bool narrow3d_fast_applicable(const NarrowArgs& p) {
  const auto al = [](const void* q) { return (reinterpret_cast<std::uintptr_t>(q) & 15) == 0; };
  const int fx = fast_fx();
  return p.dims == 3 && p.nx % fx == 0 && p.ny % NG<64>::FY == 0 && p.nx >= fx &&
         p.cx == p.cz && p.cy == p.cz && p.g0 == nullptr && al(p.u) && al(p.cz) && al(p.out) &&
         (!p.zpeer || (al(p.u_lo) && al(p.u_hi)));
}

void launch_narrow3d_fast(const NarrowArgs& p, int s, const StencilM& M, cudaStream_t st) {
  if (fast_fx() == 32) {
    if (p.zpeer)
      s == 4 ? launch_fast_s<4, 32, true>(p, M, st) : launch_fast_s<3, 32, true>(p, M, st);
    else
      s == 4 ? launch_fast_s<4, 32, false>(p, M, st) : launch_fast_s<3, 32, false>(p, M, st);
  } else {
    if (p.zpeer)
      s == 4 ? launch_fast_s<4, 64, true>(p, M, st) : launch_fast_s<3, 64, true>(p, M, st);
    else
      s == 4 ? launch_fast_s<4, 64, false>(p, M, st) : launch_fast_s<3, 64, false>(p, M, st);
  }
}

int narrow3d_fast_default_kc(int nx, int ny, int nz, int num_sms) {
  const int fx = fast_fx();
  const int occ = fx == 32 ? NG<32>::OCC : NG<64>::OCC;
  const long long tiles = static_cast<long long>(nx / fx) * (ny / NG<64>::FY);
  const long long resident = static_cast<long long>(num_sms) * occ;
  // chunked grid: equal z chunks of about 32 planes (256^3, 32-wide tiles:
  // kc 8 / 16 / 21 / 32 / 64 measured 0.291 / 0.284 / 0.280 / 0.279 / 0.284
  // ms), more and shorter (>= 8 planes) while the grid is under two waves
  long long chunks = std::max(1LL, (nz + 16LL) / 32);
  while (tiles * chunks < 2 * resident && (nz + chunks) / (chunks + 1) >= 8) ++chunks;
  return static_cast<int>((nz + chunks - 1) / chunks);
}

}  // namespace smc
