/* sgi_inputs/gen_host.c — host build of gen.h (gcc -O2 -ffp-contract=off -fopenmp).
 * Fills SoA planes a[c*ld + j], b[c*ld + j] (c = x,y,z), z0[j] with arcs of global index
 * offset + j, 0 <= j < n.  Bit-identical to the device build (gen_device.cu). */
#include <stdint.h>
#include "gen.h"

int sgi_gen_host(int config, uint64_t seed, int64_t offset, int64_t n, int64_t ld,
                 double* a, double* b, double* z0) {
  if (n < 0 || ld < n || offset < 0) return 1;
  if ((config < GEN_C1 || config > GEN_SECONDARY || config == 4)) return 1;
  if (n > 0 && (!a || !b || !z0)) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    double pa[3], pb[3], z;
    gen_arc(config, seed, (uint64_t)(offset + j), pa, pb, &z);
    for (int c = 0; c < 3; ++c) { a[c * ld + j] = pa[c]; b[c * ld + j] = pb[c]; }
    z0[j] = z;
  }
  return 0;
}
