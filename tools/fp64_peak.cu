// FP64 vector-pipe throughput on sm_100a (B200): DFMA, DMUL and DADD issue rates.
//
// Configs 4 and 5 of the Chebyshev filter put FP64 on the critical path next to HBM (the real
// kernels issue one DMUL + one DADD per product: bitwise parity with the reference's unfused
// SSE2 arithmetic; the complex ones four DFMA per complex MAC). This measures the pipe's peak so
// the C5 line can report a fraction of a MEASURED FP64 roofline.
//
// Every thread runs 8 independent dependency chains (enough ILP to cover the pipe latency at
// 16 warps / SM); 148 x 8 CTAs of 256 threads; best of 5 timed launches (CUDA events) after a
// warm-up. Output: one JSON line. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

constexpr int kChains = 8;

template <int OP>
__global__ void __launch_bounds__(256) fp64_loop(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) x[j] = 1.0 + 1e-3 * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
      if (OP == 0) x[j] = __fma_rn(x[j], a, b);
      else if (OP == 1) x[j] = __dmul_rn(x[j], a);
      else x[j] = __dadd_rn(x[j], b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += x[j];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keeps the chains alive
}

template <int OP>
double run(int sms, double* out, int iters) {
  const int grid = sms * 8, block = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp64_loop<OP><<<grid, block>>>(out, iters, 0.999999, 1e-9);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fp64_loop<OP><<<grid, block>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double ops = static_cast<double>(grid) * block * iters * kChains;
  return ops / (best * 1e-3);  // instructions (per lane) per second
}

// Sustained mode (`fp64_peak <seconds>`): DFMA launches back to back for that long, one event pair around
// the whole run -- the throughput the pipe holds under the board's power cap (tools/fp64_power.py samples
// power and SM clock beside it).
double sustained(int sms, double* out, double seconds) {
  const int grid = sms * 8, block = 256, iters = 200000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp64_loop<0><<<grid, block>>>(out, iters, 0.999999, 1e-9);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  int launches = 0;
  float ms = 0.f;
  cudaEventRecord(e0);
  while (ms < seconds * 1e3) {
    for (int k = 0; k < 4; ++k, ++launches) fp64_loop<0><<<grid, block>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double ops = static_cast<double>(grid) * block * iters * kChains * launches;
  return ops / (ms * 1e-3);
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaSetDevice(dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * sms * 8 * 256) != cudaSuccess) {
    std::printf("{\"error\": \"cudaMalloc failed\"}\n");
    return 1;
  }
  if (argc > 1) {
    const double secs = std::atof(argv[1]);
    const double fma_s = sustained(sms, out, secs > 0.5 ? secs : 0.5);
    std::printf("{\"dfma_sustained_tflops\": %.3f, \"seconds\": %.1f}\n", 2.0 * fma_s / 1e12, secs);
    cudaFree(out);
    return 0;
  }
  const int iters = 20000;
  const double fma = run<0>(sms, out, iters);
  const double mul = run<1>(sms, out, iters);
  const double add = run<2>(sms, out, iters);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
    return 1;
  }
  const double lanes_per_sm_clk = fma / sms / (clk_khz * 1e3);
  std::printf(
      "{\"dfma_tflops\": %.3f, \"dmul_tops\": %.3f, \"dadd_tops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
      "\"dfma_lanes_per_sm_per_max_clock\": %.2f, \"how\": \"tools/fp64_peak.cu: 8 independent chains per thread, "
      "%d x 256 threads, best of 5 CUDA-event timed launches; DFMA = 2 flops\"}\n",
      2.0 * fma / 1e12, mul / 1e12, add / 1e12, sms, clk_khz / 1e3, lanes_per_sm_clk, sms * 8);
  cudaFree(out);
  return 0;
}
