// sgi_inputs/gen_device.cu — device build of gen.h (nvcc -fmad=false).  Same SoA layout and
// bit-identical arcs as gen_host.c; lets the bench build 2^24..2^30-arc workloads in HBM in
// milliseconds instead of copying them from the host.
#include <stdint.h>
#include <cuda_runtime.h>
#include "gen.h"

__global__ void sgi_gen_kernel(int config, uint64_t seed, int64_t offset, int64_t n, int64_t ld,
                               double* __restrict__ a, double* __restrict__ b,
                               double* __restrict__ z0) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    double pa[3], pb[3], z;
    gen_arc(config, seed, (uint64_t)(offset + j), pa, pb, &z);
#pragma unroll
    for (int c = 0; c < 3; ++c) { a[c * ld + j] = pa[c]; b[c * ld + j] = pb[c]; }
    z0[j] = z;
  }
}

extern "C" int sgi_gen_device(int config, uint64_t seed, int64_t offset, int64_t n, int64_t ld,
                              double* a, double* b, double* z0, void* stream) {
  if (n < 0 || ld < n || offset < 0) return 1;
  if ((config < GEN_C1 || config > GEN_SECONDARY || config == 4)) return 1;
  if (n == 0) return 0;
  if (!a || !b || !z0) return 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = (n + 255) / 256, cap = (int64_t)sms * 16;
  int grid = (int)(want < cap ? want : cap);
  sgi_gen_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(config, seed, offset, n, ld, a, b, z0);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
