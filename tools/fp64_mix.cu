// FP64 pipe / issue-mix microbenchmark (measurement tool, not product code).
//
// The EFT query body issues ~312 FP64 instructions and ~250 others per query; this measures,
// in SM cycles (clock64), how the B200 SM overlaps them: per-SM FP64 lanes/clk for pure DADD
// streams at several warp counts, DADD mixed 1:1 with 32-bit selects, the ordered-TwoSum
// pattern (FSETP + 4 FSEL + 3 DADD), Knuth's TwoSum (6 DADD), and the DADD dependent latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8

__device__ __forceinline__ float hif(double x) { return __int_as_float(__double2hiint(x)); }

// kind 0: pure DADD (CH independent chains)
// kind 1: DADD + one independent 32-bit FSEL per DADD
// kind 2: ordered TwoSum per chain: FSETP, 4 FSEL, 3 DADD
// kind 3: Knuth TwoSum per chain: 6 DADD
// kind 4: single dependent DADD chain (latency)
// kind 5: DFMA with three distinct sources (one a loop constant)
// kind 6: DADD of two live chains (both operands fresh registers, no reuse)
// kind 7: DFMA of three live chains (all operands fresh registers)
template <int KIND>
__global__ void mix(double* out, long long* cyc, int iters, double a, double b) {
  double x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * 1e-3 + c; y[c] = 1e-9 * (c + 1); }
  float f = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (KIND == 0) {
#pragma unroll
      for (int c = 0; c < CH; ++c) x[c] = __dadd_rn(x[c], a);
    } else if (KIND == 1) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        x[c] = __dadd_rn(x[c], a);
        f = (__float_as_int(f) & (1 << c)) ? f : __int_as_float(__float_as_int(f) ^ c);
      }
    } else if (KIND == 2) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const double p = x[c], q = y[c];
        const bool sw = fabsf(hif(p)) < fabsf(hif(q));
        const double big = sw ? q : p, small = sw ? p : q;
        const double s = __dadd_rn(p, q);
        const double e = __dsub_rn(small, __dsub_rn(s, big));
        x[c] = s; y[c] = __dmul_rn(e, a) ;  // keep e live (1 DMUL); y stays tiny
      }
    } else if (KIND == 3) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const double p = x[c], q = y[c];
        const double s = __dadd_rn(p, q);
        const double v = __dsub_rn(s, p);
        const double e = __dadd_rn(__dsub_rn(p, __dsub_rn(s, v)), __dsub_rn(q, v));
        x[c] = s; y[c] = __dmul_rn(e, a);
      }
    } else if (KIND == 4) {
      x[0] = __dadd_rn(x[0], a);
    } else if (KIND == 5) {
#pragma unroll
      for (int c = 0; c < CH; ++c) x[c] = __fma_rn(x[c], y[c], b);
    } else if (KIND == 6) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const double t = __dadd_rn(x[c], y[c]);
        y[c] = __dadd_rn(y[c], x[(c + 1) % CH]);
        x[c] = t;
      }
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const double t = __fma_rn(x[c], y[c], x[(c + 3) % CH]);
        y[c] = __fma_rn(y[c], x[(c + 1) % CH], y[(c + 2) % CH]);
        x[c] = t;
      }
    }
  }
  long long t1 = clock64();
  double s = f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c] + y[c];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, int threads, int blocks_per_sm, double fp64_per_iter,
         double other_per_iter) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, sizeof(long long) * sms * blocks_per_sm);
  const int iters = 4000;
  const int blocks = sms * blocks_per_sm;
  mix<KIND><<<blocks, threads>>>(out, cyc, 10, 1e-7, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<KIND><<<blocks, threads>>>(out, cyc, iters, 1e-7, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[4096];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  // per SM: warps * 32 threads * iters * ops
  const double thr_per_sm = (double)threads * blocks_per_sm;
  const double fp64_lanes = thr_per_sm * iters * fp64_per_iter / mx;
  const double warp_inst_other = thr_per_sm / 32 * iters * other_per_iter / mx;
  printf("%-26s warps/SM=%3d  FP64 lanes/clk/SM=%6.2f  other warp-inst/clk/SM=%5.2f  cyc/iter=%.1f"
         "  (%.3f ms, eff clock %.0f MHz) %s\n",
         name, (int)(thr_per_sm / 32), fp64_lanes, warp_inst_other, mx / iters, ms,
         mx / (ms * 1e3), cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16, 32}) run<0>("dadd", w * 32, 1, CH, 0);
  for (int w : {8, 16, 32}) run<1>("dadd+fsel", w * 32, 1, CH, CH);
  for (int w : {8, 16, 32}) run<2>("ordered twosum (+dmul)", w * 32, 1, CH * 4, CH * 5);
  for (int w : {8, 16, 32}) run<3>("knuth twosum (+dmul)", w * 32, 1, CH * 7, 0);
  run<4>("dadd dependent latency", 32, 1, 1, 0);
  for (int w : {16, 32}) run<5>("dfma 3 sources", w * 32, 1, CH, 0);
  for (int w : {16, 32}) run<6>("dadd 2 live operands", w * 32, 1, 2 * CH, 0);
  for (int w : {16, 32}) run<7>("dfma 3 live operands", w * 32, 1, 2 * CH, 0);
  return 0;
}
