// 2-D heat operator RHS (HeatOperator::rhs, proj/core/src/pde.cpp:85-129:
// (a u_x)_x + (b u_y)_y + g0 g(t) on the periodic grid), FP64-issue-optimised
// like narrow3d_fast.cu's per-plane step, without the z march:
//   * a CTA owns a 32 x 16 tile (256 threads; 32 x 8 when ny % 16 != 0), 2
//     adjacent x cells per thread,
//     stages u, a and b with a 4-cell halo by 16-byte cp.async;
//   * x interfaces of a thread's two cells from 5 LDS.128 per field, y
//     interfaces of its two columns from 8 LDS.128 per field, each pair
//     formed in lockstep (narrow_iface2) from the 26 upper-half M entries;
//   * the tile-edge interfaces (x0 - 1/2 of each row, y0 - 1/2 of each
//     column) are packed into warps 1-3, neighbours' interfaces come by
//     shuffle (x) and through shared memory (y);
//   * 27.5 KB (17.7 KB) of shared memory and no z window: four (eight) CTAs
//     per SM.
// Same interface sums and differencing order as the general kernel
// (narrow.cu); requires nx % 32 == 0, ny % 8 == 0 and 16-byte aligned fields.
// Large grids (nx % 256 == 0) take the y-march below instead (same bits).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "narrow.cuh"

namespace smc {
namespace {

constexpr int TX2 = 32;
constexpr int LPR2 = TX2 / 2;          // threads per tile row
constexpr int HALO2 = 4;
constexpr int SW2 = TX2 + 2 * HALO2;   // 40

// Tile of 32 x TY rows: TY = 16 (256 threads, four CTAs per SM) when ny %
// 16 == 0, else 8 (128 threads, eight CTAs per SM).  The extra interfaces
// per tile (x0 - 1/2 of each row, y0 - 1/2 of each column) are 40 per 256
// cells for TY = 8, 48 per 512 for TY = 16.  At 4096^2: TY = 8 0.197 ms,
// 16 0.192 ms, 32 (two CTAs of 16 warps per SM) 0.216 ms.
template <int TY>
struct T2 {
  static constexpr int FT = LPR2 * TY;              // threads
  static constexpr int SH = TY + 2 * HALO2;
  static constexpr int CH = SH * SW2 / 2;           // 16-byte chunks per field
  static constexpr int CPT = (CH + FT - 1) / FT;
  static constexpr int OCC = 64 / TY;
};

template <int TY>
struct Smem2 {
  double t[3][T2<TY>::SH * SW2];  // u, a (x sweep), b (y sweep)
  double hy[TY + 1][TX2];
  double hxe[TY];
};

__device__ __forceinline__ void cp16_2(void* dst, const void* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}

__device__ __forceinline__ double2 lds2_2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}

template <int S, bool SRC, int TY>
__global__ void __launch_bounds__(T2<TY>::FT, S == 4 ? T2<TY>::OCC : T2<TY>::OCC * 3 / 4)
    narrow2d_fast(const NarrowArgs p, const StencilM M) {
  constexpr int WIN = 2 * S;
  constexpr int TY2 = TY, FT2 = T2<TY>::FT, CH2 = T2<TY>::CH, CPT2 = T2<TY>::CPT;
  __shared__ __align__(16) Smem2<TY> sm;
  const int tiles_x = p.nx / TX2;
  const int x0 = (blockIdx.x % tiles_x) * TX2;
  const int y0 = (blockIdx.x / tiles_x) * TY2;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int row = threadIdx.x / LPR2, cp = threadIdx.x % LPR2;

  // stage u, a, b (periodic wrap folded into the chunk offsets)
#pragma unroll
  for (int i = 0; i < CPT2; ++i) {
    const int c = threadIdx.x + i * FT2;
    if (i + 1 < CPT2 || c < CH2) {
      const int r = c / (SW2 / 2), col = 2 * (c - r * (SW2 / 2));
      const long long off = static_cast<long long>(wrap(y0 - HALO2 + r, p.ny)) * p.nx +
                            wrap(x0 - HALO2 + col, p.nx);
      cp16_2(&sm.t[0][2 * c], p.u + off);
      cp16_2(&sm.t[1][2 * c], p.cx + off);
      cp16_2(&sm.t[2][2 * c], p.cy + off);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  const double* tu = sm.t[0];
  const double* ta = sm.t[1];
  const double* tb = sm.t[2];
  // ---- x interfaces x+1/2 of my two cells (row HALO2 + row)
  double hx0, hx1;
  {
    constexpr int NV = WIN + 2;
    constexpr int BASE = HALO2 - S + 1 - ((HALO2 - S + 1) & 1);
    constexpr int OFF = (HALO2 - S + 1) - BASE;
    double ua[NV], aa[NV];
    const double* ru = tu + (HALO2 + row) * SW2 + 2 * cp + BASE;
    const double* ra = ta + (HALO2 + row) * SW2 + 2 * cp + BASE;
#pragma unroll
    for (int j = 0; j < NV / 2; ++j) {
      const double2 vu = lds2_2(ru + 2 * j), va = lds2_2(ra + 2 * j);
      ua[2 * j] = vu.x, ua[2 * j + 1] = vu.y;
      aa[2 * j] = va.x, aa[2 * j + 1] = va.y;
    }
    narrow_iface2<S>(aa + OFF, ua + OFF, aa + OFF + 1, ua + OFF + 1, M, hx0, hx1);
  }
  // ---- y interfaces y+1/2 of my two columns
  {
    double u0[WIN], b0[WIN], u1[WIN], b1[WIN];
#pragma unroll
    for (int j = 0; j < WIN; ++j) {
      const int r = HALO2 + row - S + 1 + j;
      const double2 vu = lds2_2(tu + r * SW2 + HALO2 + 2 * cp);
      const double2 vb = lds2_2(tb + r * SW2 + HALO2 + 2 * cp);
      u0[j] = vu.x, u1[j] = vu.y, b0[j] = vb.x, b1[j] = vb.y;
    }
    double y0v, y1v;
    narrow_iface2<S>(b0, u0, b1, u1, M, y0v, y1v);
    *reinterpret_cast<double2*>(&sm.hy[row + 1][2 * cp]) = make_double2(y0v, y1v);
  }
  // ---- tile-edge interfaces: y0 - 1/2 of the even columns (warp 1), of the
  //      odd columns (warp 2), x0 - 1/2 of each row (warp 3)
  if ((wid == 1 || wid == 2) && lane < LPR2) {
    const int col = HALO2 + 2 * lane + (wid - 1);
    double uu[WIN], bb[WIN];
#pragma unroll
    for (int j = 0; j < WIN; ++j) {
      uu[j] = tu[(HALO2 - S + j) * SW2 + col];
      bb[j] = tb[(HALO2 - S + j) * SW2 + col];
    }
    sm.hy[0][2 * lane + (wid - 1)] = narrow_iface<S>(bb, uu, M);
  } else if (wid == 3 && lane < TY2) {
    double uu[WIN], aa[WIN];
#pragma unroll
    for (int j = 0; j < WIN; ++j) {
      uu[j] = tu[(HALO2 + lane) * SW2 + HALO2 - S + j];
      aa[j] = ta[(HALO2 + lane) * SW2 + HALO2 - S + j];
    }
    sm.hxe[lane] = narrow_iface<S>(aa, uu, M);
  }
  __syncthreads();
  // ---- (dHx)/dx^2 + (dHy)/dy^2 (+ g0 g(t)), pde.cpp:118-124
  double hxl = __shfl_up_sync(0xffffffffu, hx1, 1);
  if (cp == 0) hxl = sm.hxe[row];
  const double2 yu = lds2_2(&sm.hy[row][2 * cp]);
  const double2 yd = lds2_2(&sm.hy[row + 1][2 * cp]);
  double o0 = __dmul_rn(__dsub_rn(hx0, hxl), p.idx2);
  double o1 = __dmul_rn(__dsub_rn(hx1, hx0), p.idx2);
  o0 = __dadd_rn(o0, __dmul_rn(__dsub_rn(yd.x, yu.x), p.idy2));
  o1 = __dadd_rn(o1, __dmul_rn(__dsub_rn(yd.y, yu.y), p.idy2));
  const long long oo = static_cast<long long>(y0 + row) * p.nx + x0 + 2 * cp;
  if constexpr (SRC) {
    const double2 g = __ldg(reinterpret_cast<const double2*>(p.g0 + oo));
    o0 = __dadd_rn(o0, __dmul_rn(g.x, p.gt));
    o1 = __dadd_rn(o1, __dmul_rn(g.y, p.gt));
  }
  *reinterpret_cast<double2*>(p.out + oo) = make_double2(o0, o1);
}

template <int S, bool SRC>
void launch2(const NarrowArgs& p, const StencilM& M, cudaStream_t st) {
  if (p.ny % 16 == 0) {
    narrow2d_fast<S, SRC, 16><<<(p.nx / TX2) * (p.ny / 16), T2<16>::FT, 0, st>>>(p, M);
  } else {
    narrow2d_fast<S, SRC, 8><<<(p.nx / TX2) * (p.ny / 8), T2<8>::FT, 0, st>>>(p, M);
  }
  SMC_CHECK_LAUNCH();
}


// ---------------------------------------------------------------- y-march
// The heat RHS as the 3-D kernel's z-march with y as the march axis (no
// in-plane y): a CTA owns a segment of MW = 256 columns (128 threads, two
// adjacent cells each) and a chunk of rows.  Per row it stages u and a with
// a 4-cell x halo (16-byte cp.async, two rows ahead, triple buffer) for the
// x interfaces; the y window (2S rows of u and b for the thread's two
// columns) lives in registers, its leading row prefetched two rows ahead.
// Each interface is formed once: x neighbours' by shuffle, across warps
// through shared memory, the segment's x0 - 1/2 of every row of the chunk
// up front by all four warps; the y interface below the chunk once per chunk.  Same interface sums and
// differencing order as the tiled kernel (pde.cpp:118-124).
constexpr int MW = 256;
constexpr int MT = MW / 2;               // 128 threads
constexpr int MSW = MW + 2 * HALO2;      // staged row width
constexpr int MCH = MSW / 2;             // 16-byte chunks per field per row
constexpr int MCPT = (MCH + MT - 1) / MT;

constexpr int MKC = 128;                 // rows per chunk at most
struct MarchSmem {
  double row[3][2][MSW];  // u, a
  double xs[2][MT / 32];  // last x interface of each warp
  double hxe[MKC];        // x0 - 1/2 of every row of the chunk
};

template <int S, bool SRC, int OCCM>
__global__ void __launch_bounds__(MT, OCCM) narrow2d_march(const NarrowArgs p, const StencilM M) {
  constexpr int WIN = 2 * S;
  __shared__ __align__(16) MarchSmem sm;
  const int segs = p.nx / MW;
  const int x0 = (blockIdx.x % segs) * MW;
  const int k0 = static_cast<int>(blockIdx.x / segs) * p.kc;
  const int k1 = min(k0 + p.kc, p.ny);
  const int cp = threadIdx.x, lane = cp & 31, wid = cp >> 5;
  const int nx = p.nx, ny = p.ny;
  auto roff = [&](int k) { return static_cast<long long>(wrap(k, ny)) * nx; };

  int soff[MCPT];
#pragma unroll
  for (int i = 0; i < MCPT; ++i) {
    const int c = cp + i * MT;
    soff[i] = c < MCH ? wrap(x0 - HALO2 + 2 * c, nx) : 0;
  }
  auto stage = [&](int buf, int k) {
    const long long ro = roff(k);
#pragma unroll
    for (int i = 0; i < MCPT; ++i) {
      const int c = cp + i * MT;
      if (i + 1 < MCPT || c < MCH) {
        cp16_2(&sm.row[buf][0][2 * c], p.u + ro + soff[i]);
        cp16_2(&sm.row[buf][1][2 * c], p.cx + ro + soff[i]);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  const int col = x0 + 2 * cp;
  auto ld2 = [&](const double* base, int k) {
    return __ldg(reinterpret_cast<const double2*>(base + roff(k) + col));
  };

  // y window: slot j holds row k - S + 1 + j at step k
  double2 wu[WIN], wb[WIN], pf_u[2], pf_b[2];
#pragma unroll
  for (int j = 0; j < WIN; ++j) wu[j] = ld2(p.u, k0 - S + j), wb[j] = ld2(p.cy, k0 - S + j);
#pragma unroll
  for (int j = 0; j < 2; ++j)
    if (k0 + j < k1) pf_u[j] = ld2(p.u, k0 + S + j), pf_b[j] = ld2(p.cy, k0 + S + j);
  stage(0, k0);
  if (k0 + 1 < k1)
    stage(1, k0 + 1);
  else
    asm volatile("cp.async.commit_group;\n" ::);
  // y interface k0 - 1/2
  double hyp0, hyp1;
  {
    double b0[WIN], u0[WIN], b1[WIN], u1[WIN];
#pragma unroll
    for (int j = 0; j < WIN; ++j) b0[j] = wb[j].x, u0[j] = wu[j].x, b1[j] = wb[j].y, u1[j] = wu[j].y;
    hyp0 = narrow_iface<S>(b0, u0, M);
    hyp1 = narrow_iface<S>(b1, u1, M);
  }
  // x0 - 1/2 of every row of the chunk, up front: row r goes to warp r % 4
  // (lane r / 4), so the four warps -- one per scheduler -- share the edge
  // work evenly instead of warp 0 forming one extra interface per row
  for (int r = 4 * lane + wid; r < k1 - k0; r += MT) {
    const long long ro = roff(k0 + r);
    double uu[WIN], aa[WIN];
#pragma unroll
    for (int j = 0; j < WIN; ++j) {
      const int c = wrap(x0 - S + j, nx);
      uu[j] = __ldg(p.u + ro + c), aa[j] = __ldg(p.cx + ro + c);
    }
    sm.hxe[r] = narrow_iface<S>(aa, uu, M);
  }
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  __syncthreads();
  const double idx2 = p.idx2, idy2 = p.idy2;

#pragma unroll 1
  for (int k = k0; k < k1; ++k) {
    const int t = k - k0, buf = t % 3, hb = t & 1;
#pragma unroll
    for (int j = 0; j + 1 < WIN; ++j) wu[j] = wu[j + 1], wb[j] = wb[j + 1];
    wu[WIN - 1] = pf_u[0];
    wb[WIN - 1] = pf_b[0];
    pf_u[0] = pf_u[1];
    pf_b[0] = pf_b[1];
    if (k + 2 < k1) pf_u[1] = ld2(p.u, k + 2 + S), pf_b[1] = ld2(p.cy, k + 2 + S);
    // ---- y interfaces k + 1/2 of my two columns
    double hy0, hy1;
    {
      double b0[WIN], u0[WIN], b1[WIN], u1[WIN];
#pragma unroll
      for (int j = 0; j < WIN; ++j) b0[j] = wb[j].x, u0[j] = wu[j].x, b1[j] = wb[j].y, u1[j] = wu[j].y;
      narrow_iface2<S>(b0, u0, b1, u1, M, hy0, hy1);
    }
    // ---- x interfaces x+1/2 of my two cells (staged row k)
    const double* tu = sm.row[buf][0];
    const double* ta = sm.row[buf][1];
    double hx0, hx1;
    {
      constexpr int NV = WIN + 2;
      constexpr int BASE = HALO2 - S + 1 - ((HALO2 - S + 1) & 1);
      constexpr int OFF = (HALO2 - S + 1) - BASE;
      double ua[NV], aa[NV];
      const double* ru = tu + 2 * cp + BASE;
      const double* ra = ta + 2 * cp + BASE;
#pragma unroll
      for (int j = 0; j < NV / 2; ++j) {
        const double2 vu = lds2_2(ru + 2 * j), va = lds2_2(ra + 2 * j);
        ua[2 * j] = vu.x, ua[2 * j + 1] = vu.y;
        aa[2 * j] = va.x, aa[2 * j + 1] = va.y;
      }
      narrow_iface2<S>(aa + OFF, ua + OFF, aa + OFF + 1, ua + OFF + 1, M, hx0, hx1);
    }
    if (lane == 31) sm.xs[hb][wid] = hx1;
    if (k + 2 < k1)
      stage((t + 2) % 3, k + 2);
    else
      asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    // ---- (dHx)/dx^2 + (dHy)/dy^2 (+ g0 g(t)), pde.cpp:118-124
    double hxl = __shfl_up_sync(0xffffffffu, hx1, 1);
    if (lane == 0) hxl = wid == 0 ? sm.hxe[t] : sm.xs[hb][wid - 1];
    double o0 = __dmul_rn(__dsub_rn(hx0, hxl), idx2);
    double o1 = __dmul_rn(__dsub_rn(hx1, hx0), idx2);
    o0 = __dadd_rn(o0, __dmul_rn(__dsub_rn(hy0, hyp0), idy2));
    o1 = __dadd_rn(o1, __dmul_rn(__dsub_rn(hy1, hyp1), idy2));
    const long long oo = static_cast<long long>(k) * nx + col;
    if constexpr (SRC) {
      const double2 g = __ldg(reinterpret_cast<const double2*>(p.g0 + oo));
      o0 = __dadd_rn(o0, __dmul_rn(g.x, p.gt));
      o1 = __dadd_rn(o1, __dmul_rn(g.y, p.gt));
    }
    *reinterpret_cast<double2*>(p.out + oo) = make_double2(o0, o1);
    hyp0 = hy0;
    hyp1 = hy1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <int S, bool SRC>
void launch_march(NarrowArgs p, const StencilM& M, cudaStream_t st) {
  // equal row chunks of about 32 rows, more and shorter (>= 8 rows) while
  // the grid is under two waves of three CTAs per SM
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long segs = p.nx / MW;
  long long chunks = std::max(1LL, (p.ny + 16LL) / 32);
  while (segs * chunks < 2LL * 3 * sms && (p.ny + chunks) / (chunks + 1) >= 8) ++chunks;
  p.kc = static_cast<int>((p.ny + chunks - 1) / chunks);
  if (const char* e = std::getenv("SMC_HEAT2D_KC")) p.kc = std::max(1, std::atoi(e));
  p.kc = std::min(p.kc, MKC);
  const long long grid = segs * ((p.ny + p.kc - 1) / p.kc);
  static const int occ = [] {
    const char* e = std::getenv("SMC_HEAT2D_OCC");
    return e ? std::atoi(e) : 3;
  }();
  if (occ == 4)
    narrow2d_march<S, SRC, 4><<<static_cast<unsigned>(grid), MT, 0, st>>>(p, M);
  else
    narrow2d_march<S, SRC, 3><<<static_cast<unsigned>(grid), MT, 0, st>>>(p, M);
  SMC_CHECK_LAUNCH();
}

// The y-march is the default where it fills the GPU (nx % 256 == 0 and at
// least two waves of 32-row chunks): 4096^2 0.187 ms against 0.192 ms for the
// tiles (FP64 pipe 60 % at 2.8 warps per scheduler, 156 registers; row chunks
// of 16 / 24 / 32 / 37 / 48: 0.191 / 0.190 / 0.187 / 0.186 / 0.199 ms; four
// CTAs per SM at 128 registers spill and gain < 1 %).  Smaller grids take the
// one-shot tiles.  SMC_HEAT2D=march / tiled forces either (same bits).
int heat2d_mode() {
  static int m = [] {
    const char* e = std::getenv("SMC_HEAT2D");
    if (e && std::string(e) == "march") return 1;
    if (e && std::string(e) == "tiled") return 2;
    return 0;
  }();
  return m;
}
bool use_march(const NarrowArgs& p, int s) {
  if (p.nx % MW != 0 || p.ny < 2 * s) return false;
  const int mode = heat2d_mode();
  if (mode) return mode == 1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return static_cast<long long>(p.nx / MW) * (p.ny / 32) >= 2LL * 3 * sms;
}

}  // namespace

bool narrow2d_fast_applicable(const NarrowArgs& p) {
  const auto al = [](const void* q) { return (reinterpret_cast<std::uintptr_t>(q) & 15) == 0; };
  return p.dims == 2 && p.nx % TX2 == 0 && p.ny % 8 == 0 && p.nx >= TX2 && p.ny >= 8 &&
         al(p.u) && al(p.cx) && al(p.cy) && al(p.out) && (p.g0 == nullptr || al(p.g0));
}

void launch_narrow2d_fast(const NarrowArgs& p, int s, const StencilM& M, cudaStream_t st) {
  if (use_march(p, s)) {
    if (p.g0)
      s == 4 ? launch_march<4, true>(p, M, st) : launch_march<3, true>(p, M, st);
    else
      s == 4 ? launch_march<4, false>(p, M, st) : launch_march<3, false>(p, M, st);
    return;
  }
  if (p.g0)
    s == 4 ? launch2<4, true>(p, M, st) : launch2<3, true>(p, M, st);
  else
    s == 4 ? launch2<4, false>(p, M, st) : launch2<3, false>(p, M, st);
}

}  // namespace smc
