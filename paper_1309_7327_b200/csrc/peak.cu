// FP64 pipe peak on this device: a dependent-chain-free DFMA loop (8
// independent accumulators per thread, 148 x 8 CTAs of 256 threads), timed
// with CUDA events.  MEASURED_PEAKS.json carries HBM and bf16 only; this is
// the denominator of the FP64 roofline (SURVEY.md §8(d) note).
#include "../../include/smc_b200.h"
#include "common.cuh"

namespace smc {
namespace {

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
  double r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5,
         r6 = r0 + 6, r7 = r0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      r0 = __fma_rn(r0, a, b);
      r1 = __fma_rn(r1, a, b);
      r2 = __fma_rn(r2, a, b);
      r3 = __fma_rn(r3, a, b);
      r4 = __fma_rn(r4, a, b);
      r5 = __fma_rn(r5, a, b);
      r6 = __fma_rn(r6, a, b);
      r7 = __fma_rn(r7, a, b);
    }
  }
  const double s = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
  if (s == 1234.5678) out[0] = s;  // keep the chain alive
}

// Variants of the DFMA probe (smc_measure_fp64_variants): CH independent
// chains per thread; KIND 0: multiplier and addend in registers shared by
// the chains (as dfma_loop), 1: a distinct multiplier register per chain,
// 2: compile-time constants (operands from the constant bank, no register
// reads for them).  The probe that issues the most DFMA per second is the
// FP64 roofline's denominator (the DMMA path shares the pipe).
template <int CH, int KIND>
__global__ void __launch_bounds__(256) dfma_variant(double* out, int iters, double a, double b) {
  double r[CH], m[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) r[c] = threadIdx.x + c, m[c] = a + c * 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 128 / CH; ++u) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if constexpr (KIND == 0) r[c] = __fma_rn(r[c], a, b);
        else if constexpr (KIND == 1) r[c] = __fma_rn(r[c], m[c], b);
        else r[c] = __fma_rn(r[c], 0.999999999, 1.0e-7);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += r[c];
  if (s == 1234.5678) out[0] = s;
}

// FP64 tensor path (mma.sync m8n8k4 f64, DMMA): 4 independent accumulator
// tiles per warp.  mode 0: DMMA only; mode 1: even warps DMMA, odd warps DFMA
// (does the tensor path add to the FP64 pipe?).
__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters, int mode) {
  const bool dmma = mode == 0 || ((threadIdx.x >> 5) & 1) == 0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  double r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5,
         r6 = r0 + 6, r7 = r0 + 7;
  if (dmma) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(c[t][0]), "+d"(c[t][1])
              : "d"(a), "d"(b));
      }
    }
  } else {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        r0 = __fma_rn(r0, a, b), r1 = __fma_rn(r1, a, b), r2 = __fma_rn(r2, a, b);
        r3 = __fma_rn(r3, a, b), r4 = __fma_rn(r4, a, b), r5 = __fma_rn(r5, a, b);
        r6 = __fma_rn(r6, a, b), r7 = __fma_rn(r7, a, b);
      }
    }
  }
  double s = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 1234.5678) out[0] = s;
}

}  // namespace
}  // namespace smc

extern "C" int smc_measure_fp64_peak(int iters, double* tflops) {
  try {
    int dev = 0, sms = 0;
    SMC_CUDA(cudaGetDevice(&dev));
    SMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* d = nullptr;
    SMC_CUDA(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t e0, e1;
    SMC_CUDA(cudaEventCreate(&e0));
    SMC_CUDA(cudaEventCreate(&e1));
    const int blocks = sms * 8;
    smc::dfma_loop<<<blocks, 256>>>(d, 16, 0.999999, 1e-7);  // warm-up
    SMC_CHECK_LAUNCH();
    SMC_CUDA(cudaEventRecord(e0));
    smc::dfma_loop<<<blocks, 256>>>(d, iters, 0.999999, 1e-7);
    SMC_CHECK_LAUNCH();
    SMC_CUDA(cudaEventRecord(e1));
    SMC_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SMC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * 256;
    *tflops = flops / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return SMC_OK;
  } catch (const std::exception&) {
    return SMC_ECUDA;
  }
}

// mode 0: DMMA-only TFLOP/s; mode 1: mixed DMMA (even warps) + DFMA (odd
// warps), TFLOP/s of both combined.  Diagnostic for the FP64 roofline.
extern "C" int smc_measure_dmma_peak(int iters, int mode, double* tflops) {
  try {
    int dev = 0, sms = 0;
    SMC_CUDA(cudaGetDevice(&dev));
    SMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* d = nullptr;
    SMC_CUDA(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t e0, e1;
    SMC_CUDA(cudaEventCreate(&e0));
    SMC_CUDA(cudaEventCreate(&e1));
    const int blocks = sms * 8;
    smc::dmma_loop<<<blocks, 256>>>(d, 4, mode);
    SMC_CHECK_LAUNCH();
    SMC_CUDA(cudaEventRecord(e0));
    smc::dmma_loop<<<blocks, 256>>>(d, iters, mode);
    SMC_CHECK_LAUNCH();
    SMC_CUDA(cudaEventRecord(e1));
    SMC_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SMC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double warps = blocks * 8.0;
    // one m8n8k4 = 2*8*8*4 = 512 flop per warp; DFMA warp-iteration = 16*8*32*2
    const double f_dmma = 512.0 * 32 * iters;
    const double f_dfma = 2.0 * 8 * 16 * 32 * iters;
    const double flops = mode == 0 ? warps * f_dmma : warps / 2 * (f_dmma + f_dfma);
    *tflops = flops / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return SMC_OK;
  } catch (const std::exception&) {
    return SMC_ECUDA;
  }
}

// TFLOP/s of the DFMA probe variants (up to n of them): 0: 8 chains, shared
// operand registers; 1: 16 chains; 2: 8 chains, a multiplier register per
// chain; 3: 8 chains, constant-bank operands; 4: variant 3 at 4 CTAs of 256
// threads per SM (half the warps).  Each is timed after a warm-up launch.
extern "C" int smc_measure_fp64_variants(int iters, double* tflops, int n) {
  try {
    int dev = 0, sms = 0;
    SMC_CUDA(cudaGetDevice(&dev));
    SMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* d = nullptr;
    SMC_CUDA(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t e0, e1;
    SMC_CUDA(cudaEventCreate(&e0));
    SMC_CUDA(cudaEventCreate(&e1));
    using K = void (*)(double*, int, double, double);
    const K kern[5] = {smc::dfma_variant<8, 0>, smc::dfma_variant<16, 0>, smc::dfma_variant<8, 1>,
                       smc::dfma_variant<8, 2>, smc::dfma_variant<8, 2>};
    const int per_sm[5] = {8, 8, 8, 8, 4};
    for (int v = 0; v < n && v < 5; ++v) {
      const int blocks = sms * per_sm[v];
      kern[v]<<<blocks, 256>>>(d, 16, 0.999999, 1e-7);
      SMC_CHECK_LAUNCH();
      SMC_CUDA(cudaEventRecord(e0));
      kern[v]<<<blocks, 256>>>(d, iters, 0.999999, 1e-7);
      SMC_CHECK_LAUNCH();
      SMC_CUDA(cudaEventRecord(e1));
      SMC_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      SMC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      tflops[v] = 2.0 * 128 * static_cast<double>(iters) * blocks * 256 / (ms * 1e-3) / 1e12;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return SMC_OK;
  } catch (const std::exception&) {
    return SMC_ECUDA;
  }
}
