// Compute-only throughput of the per-query device code (tools, not product): each thread runs
// the EFT query on register-resident synthetic arcs (perturbed each iteration so nothing is
// hoisted), folding the outputs into a checksum; no HBM traffic.  Prints ns per query for a
// few occupancies, to separate FP64/issue efficiency from memory effects.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I include -o tools/compute_only tools/compute_only.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2510_09892_b200/csrc/sgi_query.cuh"

template <int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) bench(int iters, double* sink) {
  double x1 = 0.6 + threadIdx.x * 1e-5, y1 = 0.3, z1 = 0.74, x2 = 0.59, y2 = 0.31 + blockIdx.x * 1e-7;
  double z2 = 0.745, z0 = 0.742;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    sgi::RegIn in = {{x1, y1, z1, x2, y2, z2}};
    sgi::QueryOut o;
    bool ok = sgi::query_fast<MODE>(in, z0, o);
    acc += o.p0x + (ok ? 0.0 : 1.0) + o.count;
    x1 = __dadd_rn(x1, 1e-9); y2 = __dadd_rn(y2, 1e-9);
  }
  if (acc == 12345.0) sink[0] = acc;
}

// two independent queries per iteration (ILP 2): does the body gain from more independent work
// per warp than the scheduler finds across warps?
template <int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) bench2(int iters, double* sink) {
  double x1 = 0.6 + threadIdx.x * 1e-5, y1 = 0.3, z1 = 0.74, x2 = 0.59, y2 = 0.31 + blockIdx.x * 1e-7;
  double z2 = 0.745, z0 = 0.742;
  double u1 = 0.2 + threadIdx.x * 1e-5, v1 = 0.6, w1 = 0.77, u2 = 0.21, v2 = 0.59 + blockIdx.x * 1e-7;
  double w2 = 0.775, zz = 0.771;
  double acc = 0.0;
  for (int it = 0; it < iters; it += 2) {
    sgi::RegIn in = {{x1, y1, z1, x2, y2, z2}};
    sgi::RegIn in2 = {{u1, v1, w1, u2, v2, w2}};
    sgi::QueryOut o, o2;
    bool ok = sgi::query_fast<MODE>(in, z0, o);
    bool ok2 = sgi::query_fast<MODE>(in2, zz, o2);
    acc += o.p0x + (ok ? 0.0 : 1.0) + o.count + o2.p0x + (ok2 ? 0.0 : 1.0) + o2.count;
    x1 = __dadd_rn(x1, 1e-9); y2 = __dadd_rn(y2, 1e-9);
    u1 = __dadd_rn(u1, 1e-9); v2 = __dadd_rn(v2, 1e-9);
  }
  if (acc == 12345.0) sink[0] = acc;
}

// lane type W2: the production pair kernel's body (two queries interleaved op by op)
template <int MODE>
__global__ void __launch_bounds__(512, 1) bench_w2(int iters, double* sink) {
  sgi::W2 x1 = {0.6 + threadIdx.x * 1e-5, 0.2 + threadIdx.x * 1e-5}, y1 = {0.3, 0.6}, z1 = {0.74, 0.77};
  sgi::W2 x2 = {0.59, 0.21}, y2 = {0.31 + blockIdx.x * 1e-7, 0.59 + blockIdx.x * 1e-7};
  sgi::W2 z2 = {0.745, 0.775}, z0 = {0.742, 0.771};
  double acc = 0.0;
  for (int it = 0; it < iters; it += 2) {
    struct In {
      sgi::W2 v[6];
      __device__ sgi::W2 operator()(int c) const { return v[c]; }
    } in = {{x1, y1, z1, x2, y2, z2}};
    sgi::QueryOut2 o;
    sgi::B2 ok = sgi::query_fast2<MODE>(in, z0, o);
    acc += o.p0x.x + o.p0x.y + (ok.x ? 0.0 : 1.0) + (ok.y ? 0.0 : 1.0) + o.count[0] + o.count[1];
    x1.x = __dadd_rn(x1.x, 1e-9); x1.y = __dadd_rn(x1.y, 1e-9);
    y2.x = __dadd_rn(y2.x, 1e-9); y2.y = __dadd_rn(y2.y, 1e-9);
  }
  if (acc == 12345.0) sink[0] = acc;
}

template <int MODE>
void run_w2(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 8);
  int iters = 2000;
  dim3 grid(sms);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  bench_w2<MODE><<<grid, 512>>>(10, sink);
  cudaEventRecord(a);
  bench_w2<MODE><<<grid, 512>>>(iters, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double q = (double)grid.x * 512 * iters;
  printf("%-22s 16 warps/SM  %.4f ns/query  -> 2^24 queries in %.4f ms  (%s)\n", name,
         ms * 1e6 / q, ms * 1e6 / q * 16777216 / 1e6, cudaGetErrorString(cudaGetLastError()));
}

template <int MODE, int MINB>
void run2(const char* name, int blocks_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 8);
  int iters = 2000;
  dim3 grid(sms * blocks_per_sm);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  bench2<MODE, MINB><<<grid, 256>>>(10, sink);
  cudaEventRecord(a);
  bench2<MODE, MINB><<<grid, 256>>>(iters, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double q = (double)grid.x * 256 * iters;
  printf("%-22s blocks/SM=%d  %.4f ns/query  -> 2^24 queries in %.4f ms  (%s)\n", name,
         blocks_per_sm, ms * 1e6 / q, ms * 1e6 / q * 16777216 / 1e6, cudaGetErrorString(cudaGetLastError()));
}

template <int MODE, int MINB>
void run(const char* name, int blocks_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 8);
  int iters = 2000;
  dim3 grid(sms * blocks_per_sm);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  bench<MODE, MINB><<<grid, 256>>>(10, sink);
  cudaEventRecord(a);
  bench<MODE, MINB><<<grid, 256>>>(iters, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double q = (double)grid.x * 256 * iters;
  printf("%-22s blocks/SM=%d  %.4f ns/query  -> 2^24 queries in %.4f ms  (%s)\n", name,
         blocks_per_sm, ms * 1e6 / q, ms * 1e6 / q * 16777216 / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<sgi::MODE_EFT, 1>("eft", 1);
  run<sgi::MODE_EFT, 1>("eft", 2);
  run<sgi::MODE_EFT, 1>("eft", 3);
  run<sgi::MODE_EFT, 4>("eft minb4", 4);
  run<sgi::MODE_NAIVE, 1>("naive", 3);
  run_w2<sgi::MODE_EFT>("eft W2 (production)");
  run2<sgi::MODE_EFT, 1>("eft ilp2", 1);
  run2<sgi::MODE_EFT, 1>("eft ilp2", 2);
  run<sgi::MODE_EFT, 1>("eft", 1);
  return 0;
}
