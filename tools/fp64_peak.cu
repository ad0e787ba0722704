// FP64 pipe peak microbenchmark (measurement tool, not product code).
//
// MEASURED_PEAKS.json has no FP64 entry, so the FP64 roof
// used by bench.py's roofline is measured here: independent DFMA / DADD chains
// (8 per thread, enough ILP to cover the FP64 pipe latency) on every SM.
// Prints one JSON line: instructions/s per opcode and the implied lanes/clk/SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fma_rn(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // defeat DCE
}

__global__ void dadd_loop(double* out, int iters, double a) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __dadd_rn(x[c], a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms_fma = 1e30f, ms_add = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    float ms;
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < ms_fma) ms_fma = ms;
    cudaEventRecord(e0);
    dadd_loop<<<blocks, threads>>>(out, iters, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < ms_add) ms_add = ms;
  }
  double n_instr = (double)blocks * threads * iters * CHAINS;
  double fma_per_s = n_instr / (ms_fma * 1e-3), add_per_s = n_instr / (ms_add * 1e-3);
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"clock_rate_mhz_attr\": %.0f, \"dfma_per_s\": %.4e, \"dadd_per_s\": %.4e, "
         "\"dfma_tflops\": %.3f, \"ms_fma\": %.3f, \"ms_add\": %.3f, \"err\": \"%s\"}\n",
         sms, clk_khz / 1e3, fma_per_s, add_per_s, 2 * fma_per_s / 1e12, ms_fma, ms_add,
         cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
