/* examples/c_abi_demo.c — calling libsgi.so from plain C99 (no Python, no torch).
 *
 *   nvcc -o c_abi_demo examples/c_abi_demo.c -Iinclude -Lpaper_2510_09892_b200 -lsgi -lcudart \
 *        -Xlinker -rpath=$PWD/paper_2510_09892_b200
 *
 * The meridian arc (1,0,0) -> (0,0,1) against three latitudes: z0 = 0.5 gives one point
 * (sqrt(3)/2, 0, 0.5); z0 = 1 touches the pole; z0 = 1 + 2^-50 misses. */
#include <stdio.h>
#include <string.h>
#include <cuda_runtime_api.h>

#include "sgi.h"

int main(void) {
  enum { N = 3 };
  const double a[3 * N] = {1, 1, 1, 0, 0, 0, 0, 0, 0};          /* planes x, y, z */
  const double b[3 * N] = {0, 0, 0, 0, 0, 0, 1, 1, 1};
  const double z0[N] = {0.5, 1.0, 1.0 + 0x1p-50};
  double out[6 * N];
  unsigned char cnt[N];
  double *da, *db, *dz, *dout;
  unsigned char* dcnt;
  if (cudaMalloc((void**)&da, sizeof a) || cudaMalloc((void**)&db, sizeof b) ||
      cudaMalloc((void**)&dz, sizeof z0) || cudaMalloc((void**)&dout, sizeof out) ||
      cudaMalloc((void**)&dcnt, sizeof cnt)) {
    fprintf(stderr, "no CUDA device\n");
    return 1;
  }
  cudaMemcpy(da, a, sizeof a, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b, sizeof b, cudaMemcpyHostToDevice);
  cudaMemcpy(dz, z0, sizeof z0, cudaMemcpyHostToDevice);
  sgi_status st = sgi_intersect_arc_lat(da, db, dz, N, N, dout, dcnt, SGI_MODE_EFT, NULL);
  if (st != SGI_OK) {
    fprintf(stderr, "%s: %s\n", sgi_status_str(st), sgi_last_error());
    return 1;
  }
  cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost);
  cudaMemcpy(cnt, dcnt, sizeof cnt, cudaMemcpyDeviceToHost);
  for (int i = 0; i < N; ++i)
    printf("z0 = %a: count %d, P = (%a, %a, %a)\n", z0[i], cnt[i], out[0 * N + i], out[1 * N + i],
           out[2 * N + i]);
  return 0;
}
