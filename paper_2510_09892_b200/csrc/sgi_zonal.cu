// sgi_zonal.cu — fused zonal-mean pass: mesh edges x latitude table -> compacted intersections
// (the paper's motivating application, zonal means on regridding meshes).
//
// Three launches over tiles of kEdges consecutive edges:
//   filter per edge, from an accurate normal (each component within 2 ulps), the arc's z-range: the
//          endpoints' z/|x| and, when the great circle's extremum lies strictly inside the arc
//          (dz/dt changes sign: g1 = (n x a)_z > 0 > g2 = (n x b)_z for a maximum), the apex
//          height sqrt(|n_xy|^2/|n|^2); widened by delta = 2^-40 (far above its rounding error);
//          a search in the latitude table (shared memory) gives the candidate latitudes
//          [klo, klo + kcnt), stored per edge (8 B) with each tile's candidate sum;
//   scan   one CTA turns the tile sums into output bases (and the total);
//   emit   warps walk tiles in any order (each tile knows its base), 128 edges at a time: a
//          warp scan of the stored kcnt numbers the segment's pairs (edge-major, latitude
//          ascending, deterministic), each pair's endpoints are gathered by cp.async into a
//          warp-private queue, and every 64 queued pairs run as 32 two-query lanes of the
//          batch kernel's W2 path (AccuX lines 2-25 + containment) while the other queue's
//          gathers are in flight; no CTA barriers.
// A pair's result is bit-identical to sgi_intersect_arc_lat on the same (a, b, z0): both run
// the same device code.  Candidate pairs whose latitude only touches the widened range
// come out with count 0; every pair with a nonzero count is a candidate (tests/test_gpu_zonal.py).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "sgi.h"
#include "sgi_query.cuh"
#include "sgi_tma.cuh"

#if SGI_ZONAL_COUNT_FALLBACKS     // measurement only (tools/zonal_variants.py): emit_exact calls
__device__ unsigned long long g_zonal_fallbacks = 0;
extern "C" unsigned long long sgi_debug_zonal_fallbacks(int reset) {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, g_zonal_fallbacks, sizeof(v));
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_zonal_fallbacks, &z, sizeof(z));
  }
  return v;
}
#endif

#if SGI_CERT_DEBUG_REASONS
extern "C" void sgi_debug_cert_reasons(unsigned long long* out5, int reset) {
  cudaMemcpyFromSymbol(out5, ::g_cert_reasons, 5 * sizeof(unsigned long long));
  if (reset) {
    const unsigned long long z[5] = {0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(::g_cert_reasons, z, sizeof(z));
  }
}
#endif

namespace sgi_internal {
void set_error_msg(const char* msg, cudaError_t e);   // sgi_capi.cu: sgi_last_error() text
}

namespace {

// the queries' policy: a two-point pair's second root goes to the fallback (sgi_eft.cuh
// CertDefer; an edge cuts one latitude twice only near its z-extremum)
#ifndef SGI_ZONAL_DEFER_TWO
#define SGI_ZONAL_DEFER_TWO 1
#endif
#if SGI_ZONAL_DEFER_TWO
using ZCert = sgi::CertDefer;
#else
using ZCert = sgi::Cert;
#endif

// the fused kernel draws a one-round tile's next ticket before storing the parked tile (the
// atomic in flight under that look-back and the stores) and loads the parked tile's first
// look-back window while its next tile's bulk copies are in flight
#ifndef SGI_ZONAL_EARLY_TK
#define SGI_ZONAL_EARLY_TK 1
#endif
#ifndef SGI_ZONAL_LB
#define SGI_ZONAL_LB 1     // tiles per lane per look-back step (4: 0.3485 ms, 2: 0.3446, 1: 0.3412)
#endif
// a pair whose certificates fail: Fast policy first (1; measured 0.363 vs 0.345 ms — C4's 0.12%
// fallback pairs are the ones whose Fast guards fail too) or the Exact policy at once (0)
// the filter's edges per thread consecutive, counts kept in registers and one barrier fewer (1;
// measured 0.348 vs 0.339 ms: 2-way bank conflicts on the 128-bit reads and longer live ranges)
// or strided (0)
#ifndef SGI_ZONAL_CONSEC_FILTER
#define SGI_ZONAL_CONSEC_FILTER 0
#endif
#ifndef SGI_ZONAL_L2_PREFETCH    // tile t + gridDim prefetched into L2 under tile t's arithmetic
#define SGI_ZONAL_L2_PREFETCH 1
#endif
#ifndef SGI_ZONAL_ONE_BARRIER    // one barrier between tiles instead of two back to back
#define SGI_ZONAL_ONE_BARRIER 1
#endif
#ifndef SGI_ZONAL_FALLBACK_FAST
#define SGI_ZONAL_FALLBACK_FAST 0
#endif
#ifndef SGI_ZONAL_EARLY_TMA     // ... and issues that ticket's bulk copies once the tile is free
#define SGI_ZONAL_EARLY_TMA 1
#endif
#ifndef SGI_ZONAL_LB_PREFETCH
#define SGI_ZONAL_LB_PREFETCH 1
#endif

// the filter takes an endpoint's z as its height when |x|^2 is within 2^-44 of 1 (zrange)
#ifndef SGI_ZONAL_UNIT_Z
#define SGI_ZONAL_UNIT_Z 1
#endif

#ifndef SGI_ZONAL_THREADS
#define SGI_ZONAL_THREADS 256
#endif
#ifndef SGI_ZONAL_FILTER_PREFETCH
#define SGI_ZONAL_FILTER_PREFETCH 0   // next tile's edges: 0 none, 1 registers, 2 cp.async to smem
#endif
#ifndef SGI_ZONAL_FILTER_MINB
#define SGI_ZONAL_FILTER_MINB 3     // <= 80 regs (64 used: 4 CTAs, 32 warps/SM; latency-bound)
#endif
constexpr int kThreads = SGI_ZONAL_THREADS;       // threads per CTA
constexpr int kEdges = 2 * kThreads;              // edges per tile (two adjacent per thread)
constexpr int kLatSmem = 4096;                    // latitude tables up to this length live in smem
constexpr double kDelta = 9.094947017729282e-13;  // 2^-40

__device__ __forceinline__ int lower_bound(const double* t, int n, double x) {  // first t[k] >= x
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (t[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int upper_bound(const double* t, int n, double x) {  // first t[k] > x
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (t[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}


// A bucket index over z in [-1, 1] turns each table search into one shared-memory lookup plus a
// look at the few entries of one bucket (SGI_ZONAL_EXACT_BKT, build_buckets below).  The older
// bracket form (SGI_ZONAL_EXACT_BKT=0): bkt[b] = lower_bound(tab, -1 + 2b/kBuckets) for
// b = 0..kBuckets (the boundaries are exact binary fractions); for x in bucket b (computed up to
// one bucket of rounding) the answer lies between the bounds of buckets b-1 and b+2; outside
// [-1, 1] the bracket opens to the table's ends.  Either handles any strictly increasing table.
#ifndef SGI_ZONAL_BUCKETS
#define SGI_ZONAL_BUCKETS 2048
#endif
constexpr int kBuckets = SGI_ZONAL_BUCKETS;

#ifndef SGI_ZONAL_EXACT_BKT
#define SGI_ZONAL_EXACT_BKT 1
#endif

// The bucket of x: floor((x + 1) kBuckets / 2) in float32, clamped to [0, kBuckets - 1].  Every
// step (the conversion, the addition, the power-of-two scaling, floor, the clamp) is monotone
// non-decreasing, so bucket(x) < bucket(y) implies x < y — which is all the exact index needs.
__device__ __forceinline__ int bucket_of(double x) {
  const float f = fminf(fmaxf(__fmul_rn(__fadd_rn(__double2float_rn(x), 1.0f), (float)(kBuckets / 2)),
                              0.0f), (float)(kBuckets - 1));
  return (int)f;
}

__device__ __forceinline__ void build_buckets(int* bkt, const double* tab, int nlat) {
#if SGI_ZONAL_EXACT_BKT
  // bkt[b] = the first k with bucket(tab[k]) >= b (tab increasing, so bucket(tab[k]) is too):
  // for x with bucket(x) = b, every k < bkt[b] has tab[k] < x and every k >= bkt[b + 1] has
  // tab[k] > x, so both searches of x only look at the entries of bucket b
  for (int b = threadIdx.x; b <= kBuckets; b += blockDim.x) {
    int lo = 0, hi = nlat;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (bucket_of(tab[mid]) < b) lo = mid + 1; else hi = mid;
    }
    bkt[b] = lo;
  }
#else
  for (int b = threadIdx.x; b <= kBuckets; b += blockDim.x)
    bkt[b] = lower_bound(tab, nlat, -1.0 + (double)b * (2.0 / kBuckets));
#endif
  __syncthreads();
}

template <bool UPPER>   // false: first k with tab[k] >= x; true: first k with tab[k] > x
__device__ __forceinline__ int bucket_search(const int* bkt, const double* tab, int nlat, double x) {
#if SGI_ZONAL_EXACT_BKT
  // the entries of x's bucket only (build_buckets); most buckets hold at most two latitudes,
  // counted without a loop
  const int b = bucket_of(x);
  const int lo = bkt[b], n = bkt[b + 1] - lo;
  if (n <= 2) {
    int k = lo;
    if (n >= 1 && (UPPER ? tab[lo] <= x : tab[lo] < x)) ++k;
    if (n == 2 && (UPPER ? tab[lo + 1] <= x : tab[lo + 1] < x)) ++k;
    return k;
  }
  return lo + (UPPER ? upper_bound(tab + lo, n, x) : lower_bound(tab + lo, n, x));
#else
  // the bucket only has to be right to within one (the bracket spans b-1 .. b+2): float32 is
  // far more than enough (NaN never reaches here: the caller screens it)
  const float f = fminf(fmaxf(__fmul_rn(__fadd_rn((float)x, 1.0f), (float)(kBuckets / 2)), 0.0f),
                        (float)(kBuckets - 1));
  const int b = (int)f;
  const int lo = b >= 1 ? bkt[b - 1] : 0;
  const int hi = b + 2 <= kBuckets - 1 ? bkt[b + 2] : nlat;
  return lo + (UPPER ? upper_bound(tab + lo, hi - lo, x) : lower_bound(tab + lo, hi - lo, x));
#endif
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

struct EdgeX {
  double x[6];
};

__device__ __forceinline__ void load_edge(EdgeX& r, const double* __restrict__ va,
                                          const double* __restrict__ vb, int64_t lde, int64_t e) {
  r.x[0] = __ldg(va + e); r.x[1] = __ldg(va + lde + e); r.x[2] = __ldg(va + 2 * lde + e);
  r.x[3] = __ldg(vb + e); r.x[4] = __ldg(vb + lde + e); r.x[5] = __ldg(vb + 2 * lde + e);
}

// 1/sqrt(x) for a normal positive x: the MUFU seed and two Newton steps (relative error a few
// ulps) — the filter's heights only need to be far inside delta = 2^-40, and this avoids the
// special-case branches of the library rsqrt.
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = __dmul_rn(0.5, x);
  y = __fma_rn(y, __fma_rn(-h, __dmul_rn(y, y), 0.5), y);
  y = __fma_rn(y, __fma_rn(-h, __dmul_rn(y, y), 0.5), y);
  return y;
}

// a*b - c*d within 2 ulps of the exact value (Kahan's difference of products with FMA: w = RN(cd),
// e = w - cd exactly, result RN(RN(ab - w) + e)) — the filter's normal, accurate in direction
// for any arc length, in 4 operations and a 3-deep chain.
__device__ __forceinline__ double kahan_dop(double a, double b, double c, double d) {
  const double w = __dmul_rn(c, d);
  const double e = __fma_rn(-c, d, w);
  const double f = __fma_rn(a, b, -w);
  return __dadd_rn(f, e);
}

// Candidate latitudes [klo, klo + kcnt) of one edge (see the file comment).  The filter needs the
// direction of n only to a few ulps: each component within 2 ulps of the exact one (kahan_dop, so
// short arcs keep their accuracy) and heights from the device rsqrt (a few ulps, deterministic) —
// errors ~1e-15, far below delta.
// The arc's widened z-range: lo = zlo - delta, hi = zhi + delta; mode 0 = no candidates (NaN
// inputs), 1 = search the table, 2 = every latitude (n = 0: degenerate at every latitude).
struct ZRange {
  double lo, hi;
  int mode;
};
__device__ __forceinline__ ZRange zrange(const double* x) {
  const double nx = kahan_dop(x[1], x[5], x[2], x[4]);
  const double ny = kahan_dop(x[2], x[3], x[0], x[5]);
  const double nz = kahan_dop(x[0], x[4], x[1], x[3]);
  const double ra2 = __dadd_rn(__dadd_rn(__dmul_rn(x[0], x[0]), __dmul_rn(x[1], x[1])), __dmul_rn(x[2], x[2]));
  const double rb2 = __dadd_rn(__dadd_rn(__dmul_rn(x[3], x[3]), __dmul_rn(x[4], x[4])), __dmul_rn(x[5], x[5]));
#if SGI_ZONAL_UNIT_Z
  // endpoints on the unit sphere to 2^-44 (|x|^2 as computed: within 2^-44 + 4u of 1, so
  // |z/|x| - z| <= 2^-44.9, far inside delta): z itself, no rsqrt (the usual mesh input)
  // (the high words compared as float32 bit patterns: 0x3D300000 is 2^-44's)
  const float lim = __int_as_float(0x3D300000);
  const bool unit = fabsf(sgi::hi_as_float(__dadd_rn(ra2, -1.0))) < lim &&
                    fabsf(sgi::hi_as_float(__dadd_rn(rb2, -1.0))) < lim;
  double za = x[2], zb = x[5];
  if (!unit) {
    za = __dmul_rn(x[2], fast_rsqrt(ra2));
    zb = __dmul_rn(x[5], fast_rsqrt(rb2));
  }
#else
  const double za = __dmul_rn(x[2], fast_rsqrt(ra2)), zb = __dmul_rn(x[5], fast_rsqrt(rb2));
#endif

  const double g1 = __dsub_rn(__dmul_rn(nx, x[1]), __dmul_rn(ny, x[0]));
  const double g2 = __dsub_rn(__dmul_rn(nx, x[4]), __dmul_rn(ny, x[3]));
  const bool zbig = zb > za;                         // (NaN inputs are screened below)
  double zhi = zbig ? zb : za, zlo = zbig ? za : zb;
  const bool finite = za == za && zb == zb;
  const bool top_inside = g1 > 0.0 && g2 < 0.0, bottom_inside = g1 < 0.0 && g2 > 0.0;
  if (top_inside || bottom_inside) {                 // the circle's extremum is on the arc
    const double s2 = __dadd_rn(__dmul_rn(nx, nx), __dmul_rn(ny, ny));
    const double s3 = __dadd_rn(s2, __dmul_rn(nz, nz));
    const double h = s2 > 0.0 ? __dmul_rn(__dmul_rn(s2, fast_rsqrt(s2)), fast_rsqrt(s3)) : 0.0;
    if (top_inside) zhi = fmax(zhi, h);
    else zlo = fmin(zlo, -h);
  }
  ZRange r;
  r.lo = __dsub_rn(zlo, kDelta);
  r.hi = __dadd_rn(zhi, kDelta);
  // every latitude when the endpoints are parallel or nearly so — (|nx| + |ny| + |nz|)^2 <=
  // 2^-80 |a|^2 |b|^2 (n = 0: degenerate at every latitude; an arc shorter than ~1e-12 rad,
  // or a ~ -b) — where the plain query's rounded containment may accept points anywhere on the
  // circle (e.g. the antipode of a one-ulp arc), so the candidates stay a superset of its
  // nonzero pairs (the comparison on the high words, ties counted as thin)
  const double n1 = __dadd_rn(__dadd_rn(fabs(nx), fabs(ny)), fabs(nz));
  const bool thin = sgi::hi_as_float(__dmul_rn(__dmul_rn(n1, n1), 0x1p80)) <=
                    sgi::hi_as_float(__dmul_rn(ra2, rb2));
  r.mode = thin ? 2 : (finite && zhi == zhi && zlo == zlo) ? 1 : 0;
  return r;
}

// Candidate latitudes [klo, klo + kcnt) of a z-range: first k with tab[k] >= lo, then the first
// with tab[k] > hi — mesh edges span a latitude or two, so the kStep entries after klo are tested
// at once (the table is increasing: k = klo + the number of them <= hi) before a second search.
__device__ __forceinline__ void range_search(const ZRange& r, const double* tab, const int* bkt,
                                             int nlat, int& klo, int& kcnt) {
  klo = 0;
  kcnt = r.mode == 2 ? nlat : 0;
  if (r.mode != 1) return;
  klo = bucket_search<false>(bkt, tab, nlat, r.lo);
#if SGI_ZONAL_EXACT_BKT
  kcnt = bucket_search<true>(bkt, tab, nlat, r.hi) - klo;   // lo <= hi: never negative
#else
  constexpr int kStep = 3;
  int k = klo;
#pragma unroll
  for (int s = 0; s < kStep; ++s) k += (klo + s < nlat && tab[klo + s] <= r.hi) ? 1 : 0;
  if (k == klo + kStep && k < nlat && tab[k] <= r.hi) k = bucket_search<true>(bkt, tab, nlat, r.hi);
  kcnt = k - klo;
#endif
}

// Candidate latitudes [klo, klo + kcnt) of one edge (see the file comment).  The filter needs the
// direction of n only to a few ulps: each component within 2 ulps of the exact one (kahan_dop, so
// short arcs keep their accuracy) and heights from the device rsqrt (a few ulps, deterministic) —
// errors ~1e-15, far below delta.
__device__ __forceinline__ void candidates(const double* x, const double* tab, const int* bkt,
                                           int nlat, int& klo, int& kcnt) {
  range_search(zrange(x), tab, bkt, nlat, klo, kcnt);
}


// Pass 1: candidate latitudes of every edge, cand[e] = (klo, kcnt), and each tile's sum.
// Persistent CTAs stride over the tiles (the latitude table and its bucket index are staged
// once per CTA); thread tid owns edges 2 tid and 2 tid + 1 of a tile, the next tile's loads in
// flight while it works on this one.  SMEM: the latitude table fits in shared memory (the
// searches then compile to LDS).
template <bool SMEM>
__global__ void __launch_bounds__(kThreads, SGI_ZONAL_FILTER_MINB)
sgi_zonal_filter_kernel(const double* __restrict__ va, const double* __restrict__ vb, int64_t ne,
                        int64_t lde, const double* __restrict__ lat, int nlat,
                        int2* __restrict__ cand, unsigned long long* __restrict__ tile_sum) {
  extern __shared__ __align__(16) double s_lat[];
  __shared__ unsigned s_red[2][kThreads / 32];
  __shared__ int s_bkt[kBuckets + 1];
  if (SMEM) {
    for (int k = threadIdx.x; k < nlat; k += kThreads) s_lat[k] = lat[k];
    __syncthreads();
  }
  const double* tab = SMEM ? s_lat : lat;
  build_buckets(s_bkt, tab, nlat);
  const int64_t ntiles = (ne + kEdges - 1) / kEdges;
  const int64_t G = gridDim.x;
  // candidates of the thread's two edges of tile t; per-warp sums (32-bit: <= 64 x 2^23) meet in
  // s_red[parity] behind one barrier, which also keeps the warps within one tile of each other
  auto finish = [&](int64_t t, int parity, const EdgeX (&cur)[2]) {
    const int64_t e0 = t * kEdges + 2 * threadIdx.x;
    unsigned sum = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (e0 + j < ne) {
        int klo, kcnt;
        candidates(cur[j].x, tab, s_bkt, nlat, klo, kcnt);
        cand[e0 + j] = make_int2(klo, kcnt);
        sum += (unsigned)kcnt;
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
    if ((threadIdx.x & 31) == 0) s_red[parity][threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long acc = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) acc += s_red[parity][w];
      tile_sum[t] = acc;
    }
  };
#if SGI_ZONAL_FILTER_PREFETCH == 2
  // the next tile's endpoints by cp.async into a shared double buffer (each thread copies and
  // later reads only its own two edges, so no barrier guards the buffer)
  double* stage = s_lat + (SMEM ? ((size_t)nlat + 1) / 2 * 2 : 0);
  auto slot = [&](int buf, int c, int l) { return stage + ((size_t)buf * 6 + c) * kEdges + l; };
  auto issue = [&](int64_t t, int buf) {
    if (t < ntiles) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int l = 2 * threadIdx.x + j;
        const int64_t e = t * kEdges + l;
        if (e < ne) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            cp_async8(slot(buf, c, l), va + c * lde + e);
            cp_async8(slot(buf, 3 + c, l), vb + c * lde + e);
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(blockIdx.x, 0);
  int buf = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += G, buf ^= 1) {
    issue(t + G, buf ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    EdgeX cur[2];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 6; ++c) cur[j].x[c] = *slot(buf, c, 2 * threadIdx.x + j);
    finish(t, buf, cur);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
#elif SGI_ZONAL_FILTER_PREFETCH == 1
  // the next tile's edges load into registers during this one (ping-pong, no register copies)
  EdgeX A[2], B[2];
  auto step = [&](int64_t t, int parity, EdgeX (&cur)[2], EdgeX (&nxt)[2]) {
    const int64_t en = t * kEdges + 2 * threadIdx.x + G * kEdges;
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (en + j < ne) load_edge(nxt[j], va, vb, lde, en + j);
    finish(t, parity, cur);
  };
  int64_t t = blockIdx.x;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int64_t e = t * kEdges + 2 * threadIdx.x + j;
    if (t < ntiles && e < ne) load_edge(A[j], va, vb, lde, e);
  }
  for (; t < ntiles; t += 2 * G) {
    step(t, 0, A, B);
    if (t + G < ntiles) step(t + G, 1, B, A);
  }
#else
  int parity = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += G, parity ^= 1) {
    EdgeX cur[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t e = t * kEdges + 2 * threadIdx.x + j;
      if (e < ne) load_edge(cur[j], va, vb, lde, e);
    }
    finish(t, parity, cur);
  }
#endif
}

// Pass 2: exclusive scan of the tile sums in place, the total to *d_total (one CTA).  Rounds of
// kScanRound entries (one round covers 12.8 M edges): a coalesced load of every entry into
// shared memory at once, a serial scan of kScanPer contiguous entries per thread (odd stride, so
// the 8-byte reads are bank-conflict free), a block scan of the thread totals, a coalesced store.
constexpr int kScanThreads = 1024, kScanPer = 25, kScanRound = kScanThreads * kScanPer;
constexpr size_t kScanSmem = (size_t)kScanRound * sizeof(unsigned long long);
__global__ void __launch_bounds__(kScanThreads)
sgi_zonal_scan_kernel(unsigned long long* __restrict__ tile_sum, int64_t ntiles,
                      unsigned long long* __restrict__ d_total) {
  extern __shared__ unsigned long long s[];
  __shared__ unsigned long long s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long carry = 0;
  for (int64_t r0 = 0; r0 < ntiles; r0 += kScanRound) {
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      const int64_t i = r0 + k * kScanThreads + tid;
      s[k * kScanThreads + tid] = i < ntiles ? tile_sum[i] : 0;
    }
    __syncthreads();
    unsigned long long sum = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) sum += s[tid * kScanPer + k];
    unsigned long long x = sum;                      // block scan of the thread totals
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned long long w = s_warp[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += y;
      }
      s_warp[lane] = w;
    }
    __syncthreads();
    unsigned long long run = carry + x - sum + (warp > 0 ? s_warp[warp - 1] : 0);
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      const unsigned long long v = s[tid * kScanPer + k];
      s[tid * kScanPer + k] = run;
      run += v;
    }
    const unsigned long long round_total = s_warp[31];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      const int64_t i = r0 + k * kScanThreads + tid;
      if (i < ntiles) tile_sum[i] = s[k * kScanThreads + tid];
    }
    carry += round_total;
    __syncthreads();
  }
  if (tid == 0) *d_total = carry;
}

// Pair j of the output: (edge, k), its count and both slots (unused slots: canonical NaN).
__device__ __forceinline__ void store_pair(const sgi::QueryOut& o, double z0, int64_t edge, int k,
                                           int64_t j, int64_t cap,
                                           int64_t* __restrict__ out_edge,
                                           int32_t* __restrict__ out_lat,
                                           uint8_t* __restrict__ out_count,
                                           double* __restrict__ out_xyz) {
  const bool deg = o.count == sgi::kDegenerate;
  const double nan = sgi::qnan();
  out_edge[j] = edge;
  out_lat[j] = k;
  out_count[j] = o.count;
  __stcs(out_xyz + 0 * cap + j, o.p0x);
  __stcs(out_xyz + 1 * cap + j, o.p0y);
  __stcs(out_xyz + 2 * cap + j, (!deg && o.count >= 1) ? z0 : nan);
  __stcs(out_xyz + 3 * cap + j, o.p1x);
  __stcs(out_xyz + 4 * cap + j, o.p1y);
  __stcs(out_xyz + 5 * cap + j, (!deg && o.count == 2) ? z0 : nan);
}

// Pass 3: emit every candidate pair at its ordered output slot; no CTA barriers.  Each warp owns whole 512-edge tiles (grid
// stride over warps) and walks them kSegEdges = 128 edges at a time; lane L owns the four
// adjacent edges 4L .. 4L + 3 (candidate ranges prefetched one segment ahead in registers,
// their kcnt summed locally, one warp scan per segment) and appends their pairs, in output
// order, to a warp-private queue laid out for two-query lanes: item i sits in column i mod 32,
// half i / 32, so lane L later reads items L and L + 32 with one 128-bit shared load per
// coordinate (SmemIn2, the same W2 path as the batch kernel) and the output stores stay
// coalesced.  Endpoints are gathered into the queue by cp.async as pairs are appended; two
// queues alternate, so one queue's gathers fly while the other is computed.  The head is
// recomputed for every pair (mesh edges rarely span two latitudes); a long candidate range
// just fills several queues, so lanes stay balanced.
#ifndef SGI_ZONAL_WTHREADS
#define SGI_ZONAL_WTHREADS 256   // 2 CTAs per SM (0.489 ms per C4 pass vs 0.496 at 512)
#endif
#ifndef SGI_ZONAL_EMIT_REVERSE
#define SGI_ZONAL_EMIT_REVERSE 1   // emit tiles in the reverse of the filter's order (L2 reuse)
#endif
#ifndef SGI_ZONAL_EMIT_W2
#define SGI_ZONAL_EMIT_W2 1        // 1: two queries per lane (W2); 0: one per lane, more warps
#endif
constexpr int kHalves = SGI_ZONAL_EMIT_W2 ? 2 : 1;
constexpr int kWThreads = SGI_ZONAL_WTHREADS, kWarpsPerCta = kWThreads / 32, kBatch = 32 * kHalves;
constexpr int kEmitMinB = (SGI_ZONAL_EMIT_W2 ? 512 : 768) / kWThreads;
constexpr int kSegEdges = 128;
static_assert(kEdges % kSegEdges == 0, "a tile is a whole number of segments");
struct alignas(16) WarpQueue {
  double v[6][32][kHalves];        // planes a_x .. b_z; [column][half]
  long long edge[kBatch];
  long long slot[kBatch];
  int lat[kBatch];
};
constexpr int kCandRing = 3;       // candidate-range segments in flight per warp (bulk copies)
struct alignas(16) WarpSmem {
  WarpQueue q[2];
  int2 cand[kCandRing][kSegEdges];
  uint64_t full[kCandRing];        // mbarrier per ring slot (bytes of the bulk copy)
};

// Rare path: pair (e, k) recomputed from HBM with the IEEE intrinsics and stored at slot j.
// Out of line so the fast path carries none of its state.
template <int MODE>
__device__ __noinline__ void emit_exact(const double* __restrict__ va,
                                        const double* __restrict__ vb, int64_t lde,
                                        const double* tab, int64_t e, int k, int64_t j,
                                        int64_t cap, int64_t* __restrict__ out_edge,
                                        int32_t* __restrict__ out_lat,
                                        uint8_t* __restrict__ out_count,
                                        double* __restrict__ out_xyz) {
  const sgi::RegIn r = {{va[e], va[lde + e], va[2 * lde + e], vb[e], vb[lde + e], vb[2 * lde + e]}};
  const double z0 = tab[k];
#if SGI_ZONAL_COUNT_FALLBACKS
  atomicAdd(&::g_zonal_fallbacks, 1ull);
#endif
  sgi::QueryOut o;
#if SGI_ZONAL_FALLBACK_FAST
  // the listing's sequence with the branch-free division/sqrt (policy Fast), the IEEE
  // intrinsics only if one of its guards fails — as the batch kernel's fallback queue
  if (!sgi::query_with<MODE, sgi::Fast>(r, z0, o)) sgi::query_exact<MODE>(r, z0, o);
#else
  sgi::query_exact<MODE>(r, z0, o);
#endif
  store_pair(o, z0, e, k, j, cap, out_edge, out_lat, out_count, out_xyz);
}

// One queue of n <= kBatch pairs: lane runs items lane and lane + 32 as one W2 query pair (EFT
// modes) or one after the other.  Items >= n are stale or unset and are never stored.
template <int MODE>
__device__ __forceinline__ void run_batch(const WarpQueue& q, int n, const double* tab,
                                          const double* __restrict__ va,
                                          const double* __restrict__ vb, int64_t lde,
                                          int64_t cap, int64_t* __restrict__ out_edge,
                                          int32_t* __restrict__ out_lat,
                                          uint8_t* __restrict__ out_count,
                                          double* __restrict__ out_xyz) {
  const int lane = threadIdx.x & 31;
  SGI_CHECK(n >= 0 && n <= kBatch);
  auto store = [&](const sgi::QueryOut& o, double z0, bool ok, int r) {
    if (r >= n) return;
    SGI_CHECK(q.lat[r] >= 0 && q.slot[r] >= 0 && q.edge[r] >= 0);
    const int64_t j = q.slot[r];
    if (j >= cap) return;
    if (ok) store_pair(o, z0, q.edge[r], q.lat[r], j, cap, out_edge, out_lat, out_count, out_xyz);
    else emit_exact<MODE>(va, vb, lde, tab, q.edge[r], q.lat[r], j, cap, out_edge, out_lat,
                          out_count, out_xyz);
  };
  if constexpr (kHalves == 2 && (MODE == sgi::MODE_EFT || MODE == sgi::MODE_EFT_LITERAL)) {
    const sgi::SmemIn2 in = {smem_u32(&q.v[0][lane][0]), (uint32_t)sizeof(q.v[0])};
    // items >= n hold stale or never-written latitude indices: read the table only for live
    // items (entry 0 otherwise; their results are never stored)
    const sgi::W2 zz = {tab[lane < n ? q.lat[lane] : 0], tab[lane + 32 < n ? q.lat[lane + 32] : 0]};
    sgi::QueryOut2 o;
    const sgi::B2 ok = sgi::query_fast2<MODE, ZCert>(in, zz, o);
    store({o.p0x.x, o.p0y.x, o.p1x.x, o.p1y.x, o.count[0]}, zz.x, ok.x, lane);
    store({o.p0x.y, o.p0y.y, o.p1x.y, o.p1y.y, o.count[1]}, zz.y, ok.y, lane + 32);
  } else {
#pragma unroll
    for (int h = 0; h < kHalves; ++h) {
      const sgi::SmemIn in1 = {smem_u32(&q.v[0][lane][h]), (uint32_t)sizeof(q.v[0])};
      const double z0 = tab[lane + 32 * h < n ? q.lat[lane + 32 * h] : 0];
      sgi::QueryOut o;
      const bool ok = sgi::query_fast<MODE, ZCert>(in1, z0, o);
      store(o, z0, ok, lane + 32 * h);
    }
  }
}

template <int MODE>
__device__ __noinline__ void run_batch_tail(const WarpQueue& q, int n, const double* tab,
                                            const double* __restrict__ va,
                                            const double* __restrict__ vb, int64_t lde,
                                            int64_t cap, int64_t* __restrict__ out_edge,
                                            int32_t* __restrict__ out_lat,
                                            uint8_t* __restrict__ out_count,
                                            double* __restrict__ out_xyz) {
  run_batch<MODE>(q, n, tab, va, vb, lde, cap, out_edge, out_lat, out_count, out_xyz);
}

template <int MODE, bool SMEM>
__global__ void __launch_bounds__(kWThreads, kEmitMinB)
sgi_zonal_emit_warp_kernel(const double* __restrict__ va, const double* __restrict__ vb,
                           int64_t ne, int64_t lde, const double* __restrict__ lat, int nlat,
                           int64_t cap, int64_t* __restrict__ out_edge,
                           int32_t* __restrict__ out_lat, uint8_t* __restrict__ out_count,
                           double* __restrict__ out_xyz, const int2* __restrict__ cand,
                           const unsigned long long* __restrict__ tile_base) {
  extern __shared__ __align__(16) double s_dyn[];
  const size_t lat_words = SMEM ? ((size_t)nlat + 1) / 2 * 2 : 0;
  if (SMEM) {
    for (int k = threadIdx.x; k < nlat; k += kWThreads) s_dyn[k] = lat[k];
    __syncthreads();
  }
  const double* tab = SMEM ? s_dyn : lat;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem& W = reinterpret_cast<WarpSmem*>(s_dyn + lat_words)[warp];
#if SGI_DEBUG_CHECKS
  if (SMEM) __syncthreads();      // the table copy is complete before the scratch is poisoned
  sgi_poison_smem(reinterpret_cast<WarpSmem*>(s_dyn + lat_words), kWarpsPerCta * sizeof(WarpSmem));
  __syncthreads();
#endif
  // this warp's tiles t0, t0 + nwarps, ... (grid stride: at any time the warps of the grid
  // work on neighbouring tiles, which measured faster than contiguous per-warp ranges)
  const int64_t ntiles = (ne + kEdges - 1) / kEdges;
  const int64_t t0 = (int64_t)blockIdx.x * kWarpsPerCta + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerCta;
  const int mytiles = t0 < ntiles ? (int)((ntiles - t0 + nwarps - 1) / nwarps) : 0;
  constexpr int kSegs = kEdges / kSegEdges;
  const int nseg = mytiles * kSegs;                    // this warp's segments, in order
  const int l0 = 4 * lane;
  // this warp's i-th tile; in reverse order the first tiles are the filter's last ones, whose
  // endpoints and candidate ranges are still in L2
  auto tile_of = [&](int i) {
    const int64_t t = t0 + (int64_t)i * nwarps;
    return SGI_ZONAL_EMIT_REVERSE ? ntiles - 1 - t : t;
  };
  auto seg_edge0 = [&](int g) {
    return tile_of(g / kSegs) * kEdges + (g % kSegs) * kSegEdges;
  };
  // candidate ranges of segment g -> ring slot g % kCandRing by one bulk copy (lane 0), so the
  // next kCandRing - 1 segments are in flight without holding registers
  if (lane == 0) {
    for (int r = 0; r < kCandRing; ++r) mbar_init(&W.full[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int g) {
    if (lane != 0 || g >= nseg) return;
    const int64_t e0 = seg_edge0(g);
    const int64_t nv = ne - e0 < kSegEdges ? ne - e0 : kSegEdges;
    if (nv <= 0) {                                     // past the last edge: complete the phase
      mbar_expect_tx(&W.full[g % kCandRing], 0);
      return;
    }
    // whole 16-B units (an odd count reads 8 B of the tile sums that follow cand in d_work)
    const uint32_t bytes = (uint32_t)((nv + 1) / 2 * 16);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&W.full[g % kCandRing], bytes);
    bulk_g2s(&W.cand[g % kCandRing][0], cand + e0, bytes, &W.full[g % kCandRing]);
  };
  for (int g = 0; g < kCandRing - 1; ++g) issue(g);
  unsigned long long nbase = nseg > 0 ? tile_base[tile_of(0)] : 0;
  int cur = 0, qn = 0;                                 // filling queue, its queued pairs
  bool pending = false;                                // queue cur ^ 1 gathered, not yet run
  int64_t base = 0;                                    // first slot of the current segment
  for (int g = 0; g < nseg; ++g) {
    issue(g + kCandRing - 1);
    const int64_t e0 = seg_edge0(g);
    if (g % kSegs == 0) base = (int64_t)nbase;
    if ((g + 1) % kSegs == 0 && g + 1 < nseg)
      nbase = tile_base[tile_of((g + 1) / kSegs)];
    mbar_wait(&W.full[g % kCandRing], (uint32_t)((g / kCandRing) & 1));
    int4 ca = *reinterpret_cast<const int4*>(&W.cand[g % kCandRing][l0]);
    int4 cb = *reinterpret_cast<const int4*>(&W.cand[g % kCandRing][l0 + 2]);
    if (e0 + l0 + 3 >= ne) {                           // entries beyond ne: no candidates
      if (e0 + l0 >= ne) ca.y = 0;
      if (e0 + l0 + 1 >= ne) ca.w = 0;
      if (e0 + l0 + 2 >= ne) cb.y = 0;
      cb.w = 0;
    }
    const unsigned k0 = (unsigned)ca.y, k1 = (unsigned)ca.w, k2 = (unsigned)cb.y;
    const unsigned mine = k0 + k1 + k2 + (unsigned)cb.w;
    unsigned incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    const unsigned excl = incl - mine;
    const unsigned segtot = __shfl_sync(0xffffffffu, incl, 31);
    for (unsigned cursor = 0; cursor < segtot;) {      // queue slots [qn, qn + m) <- pairs [cursor, ...)
      const unsigned m = min((unsigned)(kBatch - qn), segtot - cursor);
      WarpQueue& q = W.q[cur];
      // slot-major fill: lane L fills slots L and L + 32; pair p's owner lane is the last lane
      // with excl <= p (found by a shuffle binary search), then one of its four edges
#pragma unroll
      for (int h = 0; h < kHalves; ++h) {
        const int at = lane + 32 * h;
        const bool valid = at >= qn && at < qn + (int)m;
        const unsigned p = min(cursor + (unsigned)(at - qn), segtot - 1);   // clamped when idle
        int own = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const unsigned x = __shfl_sync(0xffffffffu, excl, own + step);
          if (x <= p) own += step;
        }
        unsigned off = p - __shfl_sync(0xffffffffu, excl, own);
        const unsigned o0 = __shfl_sync(0xffffffffu, k0, own);
        const unsigned o1 = __shfl_sync(0xffffffffu, k1, own);
        const unsigned o2 = __shfl_sync(0xffffffffu, k2, own);
        const int q0 = __shfl_sync(0xffffffffu, ca.x, own), q1 = __shfl_sync(0xffffffffu, ca.z, own);
        const int q2 = __shfl_sync(0xffffffffu, cb.x, own), q3 = __shfl_sync(0xffffffffu, cb.z, own);
        int i = 0, klo = q0;                           // the owner's edge holding pair p
        if (off >= o0) { off -= o0; i = 1; klo = q1;
          if (off >= o1) { off -= o1; i = 2; klo = q2;
            if (off >= o2) { off -= o2; i = 3; klo = q3; } } }
        if (valid) {
          const int64_t e = e0 + 4 * own + i;
          const int k = klo + (int)off;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            cp_async8(&q.v[c][lane][h], va + c * lde + e);
            cp_async8(&q.v[3 + c][lane][h], vb + c * lde + e);
          }
          q.edge[at] = e;
          q.lat[at] = k;
          q.slot[at] = base + p;
        }
      }
      qn += (int)m;
      cursor += m;
      if (qn == kBatch) {                              // queue cur is full: run the other one
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (pending) {
          asm volatile("cp.async.wait_group 1;" ::: "memory");
          run_batch<MODE>(W.q[cur ^ 1], kBatch, tab, va, vb, lde, cap, out_edge, out_lat,
                          out_count, out_xyz);
        }
        pending = true;
        cur ^= 1;
        qn = 0;
      }
    }
    base += segtot;
    __syncwarp();                                      // ring slot g % kCandRing is reissued next
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
  // the last one or two queues: one out-of-line copy of the batch code (instruction cache)
  if (pending)
    run_batch_tail<MODE>(W.q[cur ^ 1], kBatch, tab, va, vb, lde, cap, out_edge, out_lat, out_count,
                         out_xyz);
  if (qn > 0)
    run_batch_tail<MODE>(W.q[cur], qn, tab, va, vb, lde, cap, out_edge, out_lat, out_count, out_xyz);
}

// ------------------------------------------------------------------ single-pass fused kernel
// One launch instead of filter + scan + emit (zonal): persistent CTAs take tiles
// of kFE consecutive edges in ticket order; per tile the six endpoint planes arrive in shared
// memory by bulk copies (TMA), the filter writes each edge's candidate range to shared memory,
// a block scan numbers the tile's pairs, and the tile's output base comes from a decoupled
// look-back over the preceding tiles' published counts (aggregate / inclusive flags in the
// workspace; tickets make every earlier tile's CTA resident, so the look-back always
// completes).  The pairs then run as two-query lanes straight from the staged endpoints and are
// stored at base + pair index: each edge is read from HBM once and no candidate range leaves
// the SM.  Pair results are the batch kernel's (same query code).
#ifndef SGI_ZONAL_FUSED
#define SGI_ZONAL_FUSED 1
#endif
#ifndef SGI_ZONAL_PARK
#define SGI_ZONAL_PARK 1     // park one-round tiles' results, store them after the next look-back
#endif                       // (0.389 vs 0.397 ms with the final filter; 0.434 vs 0.421 before it)
#ifndef SGI_ZONAL_STATIC
#define SGI_ZONAL_STATIC 0   // 1: static tiles + cooperative launch (0.478 ms vs 0.44: look-back waits)
#endif
#ifndef SGI_ZONAL_FT
#define SGI_ZONAL_FT 256
#endif
constexpr int kFT = SGI_ZONAL_FT;          // threads per CTA (256: 2 CTAs per SM at <= 128 registers)
constexpr int kFE = 4 * kFT;               // edges per tile
static_assert(kFT >= 64, "warp 1 draws the early ticket");
#ifndef SGI_ZONAL_MINB
#define SGI_ZONAL_MINB (512 / SGI_ZONAL_FT)      // 16 warps per SM at <= 128 registers
#endif
constexpr int kFMinB = SGI_ZONAL_MINB > 0 ? SGI_ZONAL_MINB : 1;
constexpr int kFPer = kFE / kFT;           // edges per thread in the filter
constexpr int kFP = 2 * kFT;               // pairs per round (two per thread)
constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kValMask = (1ull << 62) - 1;

struct FusedSmem {
  alignas(16) int kcnt[kFE];
  alignas(16) int excl[kFE + 4];
  alignas(16) int klo[kFE];
  int bkt[kBuckets + 1];
  unsigned short pmap[2 * kFT];
  unsigned wsum[kFT / 32];
  long long prefix;
  long long ticket;
  uint64_t full;
  unsigned long long lbpre[32 * SGI_ZONAL_LB];   // warp 0's prefetched first look-back window
};

// A tile's status word carries all that is published (flag and count in one aligned 64-bit
// word, single-copy atomic), so relaxed GPU-scope accesses suffice: no other data is ordered
// by it.  (Acquire loads would invalidate L1 — CCTL.IVALL — on every poll.)
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Two pairs' endpoints in the staged tile (lane type W2): coordinate c of edges l0 and l1.
struct SmemInTwo {
  uint32_t a0, a1, stride;
  __device__ __forceinline__ sgi::W2 operator()(int c) const {
    sgi::W2 v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v.x) : "r"(a0 + (uint32_t)c * stride));
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v.y) : "r"(a1 + (uint32_t)c * stride));
    return v;
  }
};

// The edge of tile pair p: the last e with excl[e] <= p (excl[kFE] = the tile's total).
template <int kE = kFE>
__device__ __forceinline__ int pair_edge(const int* excl, int p) {
  int lo = 0, hi = kE;                       // excl[lo] <= p < excl[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (excl[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}

// Exclusive output base of tile t: warp-wide look-back over the published tile counts, kLB
// tiles per lane per step, all loads in flight at once (32 kLB tiles per L2 round trip).  The
// walk is bound by waiting for predecessors that have not published their counts yet, not by
// round trips: wider windows poll more unpublished words and measured slower.
constexpr int kLB = SGI_ZONAL_LB;
// The first window's words as look_back loads them (lane L: tiles t-1-kLB L-j), into pre[] —
// issued early, they are consumed (and re-polled where still missing) by look_back(..., pre).
// A status word only moves forward (missing, aggregate, inclusive), so any value seen is usable.
__device__ __forceinline__ void look_back_prefetch(const unsigned long long* status, int64_t t,
                                                   unsigned long long* pre) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kLB; ++j) {
    const int64_t q = t - 1 - kLB * lane - j;
    pre[lane * kLB + j] = q >= 0 ? ld_status(status + q) : kInc;
  }
}

__device__ __forceinline__ long long look_back(const unsigned long long* status, int64_t t,
                                               const unsigned long long* pre = nullptr) {
  const int lane = threadIdx.x & 31;
  long long prefix = 0;
  for (int64_t p = t - 1;; p -= 32 * kLB) {
    unsigned long long v[kLB];
    // lane L covers tiles p - kLB L .. p - kLB L - kLB + 1 (nearest first)
#pragma unroll
    for (int j = 0; j < kLB; ++j) {
      const int64_t q = p - kLB * lane - j;
      SGI_CHECK(q < t);
      v[j] = pre && p == t - 1 ? pre[lane * kLB + j] : q >= 0 ? ld_status(status + q) : kInc;
    }
    // the nearest inclusive entry (lowest lane, then lowest j) ends the walk; only the entries
    // before it must have been published (a missing one further back does not matter)
    int jinc, first;
    unsigned inc;
    for (;;) {
      jinc = kLB;
#pragma unroll
      for (int j = kLB - 1; j >= 0; --j)
        if ((v[j] >> 62) == 2) jinc = j;
      inc = __ballot_sync(0xffffffffu, jinc < kLB);
      first = inc ? __ffs(inc) - 1 : 32;
      bool missing = false;
#pragma unroll
      for (int j = 0; j < kLB; ++j)
        missing |= (lane < first || (lane == first && j < jinc)) && (v[j] >> 62) == 0;
      if (!__any_sync(0xffffffffu, missing)) break;
#pragma unroll
      for (int j = 0; j < kLB; ++j) {
        const int64_t q = p - kLB * lane - j;
        if ((v[j] >> 62) == 0) v[j] = ld_status(status + q);
      }
    }
    long long mine = 0;
#pragma unroll
    for (int j = 0; j < kLB; ++j)
      if (lane < first || (lane == first && j <= jinc)) mine += (long long)(v[j] & kValMask);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, d);
    prefix += mine;
    if (inc) break;
  }
  return prefix;
}

template <int MODE>
__global__ void __launch_bounds__(kFT, kFMinB)
sgi_zonal_fused_kernel(const double* __restrict__ va, const double* __restrict__ vb, int64_t ne,
                       int64_t lde, const double* __restrict__ lat, int nlat, int64_t cap,
                       int64_t* __restrict__ out_edge, int32_t* __restrict__ out_lat,
                       uint8_t* __restrict__ out_count, double* __restrict__ out_xyz,
                       unsigned long long* __restrict__ status, unsigned long long* d_total,
                       bool tma) {
  extern __shared__ __align__(128) double s_fused[];
  __shared__ FusedSmem S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t lat_words = ((size_t)nlat + 15) / 16 * 16;       // 128-B aligned tile after it
  double* tab = s_fused;
  double* tile = s_fused + lat_words;                             // [6][kFE]
  sgi_poison_smem(&S, sizeof(S));
  sgi_poison_smem(s_fused + lat_words, 6 * kFE * sizeof(double));
  __syncthreads();
  for (int k = tid; k < nlat; k += kFT) tab[k] = lat[k];
  if (tid == 0) {
    mbar_init(&S.full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  build_buckets(S.bkt, tab, nlat);
  const int64_t ntiles = (ne + kFE - 1) / kFE;
  unsigned long long* ticket_ctr = status + ntiles;
  auto plane = [&](int c) { return (c < 3 ? va : vb) + (c % 3) * lde; };
  constexpr bool kW2 = MODE == sgi::MODE_EFT || MODE == sgi::MODE_EFT_LITERAL;
  uint32_t phase = 0;
  // parked results of the previous one-round tile: 4 coordinates per pair slot + packed
  // (edge in tile, latitude, count, ok, valid)
  double* park = tile + 6 * kFE;                                // [4][kFP]
  unsigned* park_meta = reinterpret_cast<unsigned*>(park + 4 * kFP);
  int64_t prev_t = 0;
  int prev_T = 0;
  bool have_prev = false;
  // look back for the parked tile, publish its inclusive count, store its results
  bool lb_ready = false;                 // S.lbpre holds prev_t's first look-back window
  bool pre_issued = false;               // the current tile's copies were issued by flush_parked
  // tile tt's six bulk copies (one thread; the tile buffer must be free)
  auto full_tile = [&](int64_t tt) { return tma && tt < ntiles && ne - tt * kFE >= kFE; };
  auto issue_tile = [&](int64_t tt) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&S.full, 6 * kFE * 8);
#pragma unroll
    for (int c = 0; c < 6; ++c) bulk_g2s(tile + c * kFE, plane(c) + tt * kFE, kFE * 8, &S.full);
  };
  // issue_t: the next tile, whose copies thread 32 issues once every thread is past this tile's
  // queries (the first barrier below); -1: none
  auto flush_parked = [&](long long issue_t) {
    if (warp == 0) {
      const long long pre = prev_t == 0 ? 0 : look_back(status, prev_t, lb_ready ? S.lbpre : nullptr);
      if (lane == 0) {
        if (prev_t > 0) st_status(status + prev_t, kInc | (unsigned long long)(pre + prev_T));
        S.prefix = pre;
        if (prev_t == ntiles - 1) *d_total = (unsigned long long)(pre + prev_T);
      }
    }
    __syncthreads();
    if (tid == 32 && issue_t >= 0 && full_tile(issue_t)) issue_tile(issue_t);
    const long long base = S.prefix;
    const int64_t pe0 = prev_t * kFE;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sl = h * kFT + tid;
      const unsigned m = park_meta[sl];
      if (!(m >> 31)) continue;
      const int64_t j = base + sl;
      if (j >= cap) continue;
      const int le = (int)(m & 1023u), kk = (int)((m >> 10) & 4095u);
      const sgi::QueryOut o = {park[0 * kFP + sl], park[1 * kFP + sl], park[2 * kFP + sl],
                               park[3 * kFP + sl], (uint8_t)((m >> 22) & 255u)};
      if ((m >> 30) & 1u) store_pair(o, tab[kk], pe0 + le, kk, j, cap, out_edge, out_lat,
                                     out_count, out_xyz);
      else emit_exact<MODE>(va, vb, lde, tab, pe0 + le, kk, j, cap, out_edge, out_lat, out_count,
                            out_xyz);
    }
    __syncthreads();                   // S.prefix and the parked slots are free again
  };
#if SGI_ZONAL_STATIC
  // static assignment (tiles blockIdx.x, + gridDim.x, ...): the cooperative launch makes every
  // CTA resident, so every earlier tile's CTA runs and the look-back completes; each CTA knows
  // its next tile and prefetches it into L2 under the current tile's arithmetic
  (void)ticket_ctr;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
#else
  // the first ticket here; each later one is drawn while the previous tile's results are being
  // stored, so its atomic round trip is off the critical path
  if (tid == 0) S.ticket = (long long)atomicAdd(ticket_ctr, 1ull);
  for (;;) {
    __syncthreads();
    const int64_t t = S.ticket;
    if (t >= ntiles) break;
#endif
    const int64_t e0 = t * kFE;
    const int nv = (int)(ne - e0 < kFE ? ne - e0 : kFE);
    // ---- endpoints of the tile -> shared memory
    if (tma && nv == kFE) {
      if (tid == 0 && !pre_issued) issue_tile(t);
#if SGI_ZONAL_LB_PREFETCH
      // the parked tile's first look-back window, loaded under the bulk copies
      if (warp == 0 && have_prev && prev_t > 0) look_back_prefetch(status, prev_t, S.lbpre);
      lb_ready = have_prev && prev_t > 0;
#endif
      mbar_wait(&S.full, phase);
      phase ^= 1;
    } else {
      for (int i = tid; i < 6 * kFE; i += kFT) {
        const int c = i / kFE, l = i % kFE;
        tile[i] = l < nv ? plane(c)[e0 + l] : 0.0;
      }
      __syncthreads();
    }
#if SGI_ZONAL_CONSEC_FILTER
    // ---- filter: candidate range of each edge (thread tid: edges 4 tid .. 4 tid + 3, read as
    // 128-bit pairs; the counts stay in registers for the scan, so no barrier between them)
    // (the four z-ranges first — independent FP64 chains the scheduler can interleave — then the
    // four table searches)
    static_assert(kFPer == 4, "four consecutive edges per thread");
    ZRange zr[kFPer];
    {
      double xs[6][kFPer];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const double2 u = *reinterpret_cast<const double2*>(&tile[c * kFE + kFPer * tid]);
        const double2 v = *reinterpret_cast<const double2*>(&tile[c * kFE + kFPer * tid + 2]);
        xs[c][0] = u.x; xs[c][1] = u.y; xs[c][2] = v.x; xs[c][3] = v.y;
      }
#pragma unroll
      for (int j = 0; j < kFPer; ++j) {
        double x[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) x[c] = xs[c][j];
        zr[j] = zrange(x);
        if (kFPer * tid + j >= nv) zr[j].mode = 0;
      }
    }
    int klo4[kFPer], c4a[kFPer];
#pragma unroll
    for (int j = 0; j < kFPer; ++j) range_search(zr[j], tab, S.bkt, nlat, klo4[j], c4a[j]);
    *reinterpret_cast<int4*>(&S.klo[kFPer * tid]) = make_int4(klo4[0], klo4[1], klo4[2], klo4[3]);
    const int4 c4 = make_int4(c4a[0], c4a[1], c4a[2], c4a[3]);
#else
    // ---- filter: candidate range of each edge (thread tid: edges tid, tid + kFT, ...)
    // (the four z-ranges first — independent FP64 chains the scheduler can interleave — then the
    // four table searches)
    ZRange zr[kFPer];
#pragma unroll
    for (int j = 0; j < kFPer; ++j) {
      const int l = tid + j * kFT;
      double x[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) x[c] = tile[c * kFE + l];
      zr[j] = zrange(x);
      if (l >= nv) zr[j].mode = 0;
    }
#pragma unroll
    for (int j = 0; j < kFPer; ++j) {
      const int l = tid + j * kFT;
      int klo, kcnt;
      range_search(zr[j], tab, S.bkt, nlat, klo, kcnt);
      S.klo[l] = klo;
      S.kcnt[l] = kcnt;
    }
    __syncthreads();
#endif
    // tile t + gridDim.x (about the ticket some CTA draws next) into L2 under this tile's
    // arithmetic, so that CTA's bulk copies hit L2
    if (SGI_ZONAL_L2_PREFETCH && tid == 0 && tma && t + gridDim.x < ntiles &&
        ne - (t + gridDim.x) * kFE >= kFE) {
#pragma unroll
      for (int c = 0; c < 6; ++c)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(plane(c) + (t + gridDim.x) * kFE),
                     "r"(kFE * 8) : "memory");
    }
    // ---- block scan of the counts (thread tid: edges 4 tid .. 4 tid + 3)
#if !SGI_ZONAL_CONSEC_FILTER
    const int4 c4 = *reinterpret_cast<const int4*>(&S.kcnt[kFPer * tid]);
#endif
    const unsigned mine = (unsigned)(c4.x + c4.y + c4.z + c4.w);
    unsigned incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane == 31) S.wsum[warp] = incl;
    __syncthreads();
    unsigned before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kFT / 32; ++w) {
      const unsigned x = S.wsum[w];
      before += w < warp ? x : 0;
      total += x;
    }
    {
      const int b = (int)(before + incl - mine);
      *reinterpret_cast<int4*>(&S.excl[kFPer * tid]) =
          make_int4(b, b + c4.x, b + c4.x + c4.y, b + c4.x + c4.y + c4.z);
      if (tid == kFT - 1) S.excl[kFE] = (int)total;
      // pair -> edge map of the first round (the pairs of later rounds search excl)
      const int cs[4] = {c4.x, c4.y, c4.z, c4.w};
      int o = b;
#pragma unroll
      for (int j = 0; j < kFPer; ++j) {
        const unsigned short e = (unsigned short)(kFPer * tid + j);
        if (cs[j] == 1) {                            // the usual case: one latitude
          if (o < kFP) S.pmap[o] = e;
        } else if (cs[j] > 1) {
          const int stop = min(o + cs[j], kFP);
          for (int q = o; q < stop; ++q) S.pmap[q] = e;
        }
        o += cs[j];
      }
    }
    // publish this tile's count (its aggregate; tile 0's is already inclusive)
    if (tid == 0) st_status(status + t, (t == 0 ? kInc : kAgg) | (unsigned long long)total);
    __syncthreads();
    const int T = (int)total;
    // ---- the tile's pairs, 2 kFT per round (thread tid: pairs r0 + tid, r0 + kFT + tid).  A
    // one-round tile (the usual case) parks its results in shared memory and stores them one tile
    // later, after the look-back for it — by then its predecessors have long published, so the
    // look-back is one L2 round trip instead of a wait; a larger tile flushes the parked one and
    // stores at once.
    const bool multi = !SGI_ZONAL_PARK || T > 2 * kFT;
    pre_issued = false;
#if !SGI_ZONAL_STATIC && SGI_ZONAL_EARLY_TK >= 2
    // the next ticket, drawn before this tile's queries (warp 1): its atomic round trip is hidden
    // under them, and the tile it names starts right after this one either way
    long long tk = 0;
    if (!multi && tid == 32) tk = (long long)atomicAdd(ticket_ctr, 1ull);
#endif
    if (multi && have_prev) {
      flush_parked(-1);
      have_prev = false;
    }
    bool have_prefix = !multi;
    for (int r0 = 0; r0 < T || !have_prefix || r0 == 0; r0 += 2 * kFT) {
      const int p0 = r0 + tid, p1 = r0 + kFT + tid;
      const bool v0 = p0 < T, v1 = p1 < T;
      sgi::QueryOut o[2];
      bool ok[2] = {true, true};
      int le[2] = {0, 0}, kk[2] = {0, 0};
      double zz[2] = {0.0, 0.0};
      if (v0) {
        SGI_CHECK(S.excl[0] == 0 && S.excl[kFE] == T);
        le[0] = p0 < kFP ? (int)S.pmap[p0] : pair_edge(S.excl, p0);
        kk[0] = S.klo[le[0]] + (p0 - S.excl[le[0]]);
        le[1] = le[0];
        kk[1] = kk[0];
        if (v1) {
          le[1] = p1 < kFP ? (int)S.pmap[p1] : pair_edge(S.excl, p1);
          kk[1] = S.klo[le[1]] + (p1 - S.excl[le[1]]);
        }
        SGI_CHECK(le[0] >= 0 && le[0] < nv && le[1] >= 0 && le[1] < nv);
        SGI_CHECK(kk[0] >= 0 && kk[0] < nlat && kk[1] >= 0 && kk[1] < nlat);
        SGI_CHECK(p0 >= S.excl[le[0]] && p0 < S.excl[le[0] + 1]);
        zz[0] = tab[kk[0]];
        zz[1] = tab[kk[1]];
        if constexpr (kW2) {
          const SmemInTwo in = {smem_u32(tile + le[0]), smem_u32(tile + le[1]), kFE * 8};
          sgi::QueryOut2 q;
          const sgi::B2 okb = sgi::query_fast2<MODE, ZCert>(in, sgi::W2{zz[0], zz[1]}, q);
          o[0] = {q.p0x.x, q.p0y.x, q.p1x.x, q.p1y.x, q.count[0]};
          o[1] = {q.p0x.y, q.p0y.y, q.p1x.y, q.p1y.y, q.count[1]};
          ok[0] = okb.x;
          ok[1] = okb.y;
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !v1) break;
            const sgi::SmemIn in = {smem_u32(tile + le[h]), kFE * 8};
            ok[h] = sgi::query_fast<MODE, ZCert>(in, zz[h], o[h]);
          }
        }
      }
      if (!multi) {
#if !SGI_ZONAL_STATIC && SGI_ZONAL_EARLY_TK
#if SGI_ZONAL_EARLY_TK == 1
        long long tk = 0;               // the next ticket, in flight under the flush (warp 1)
        if (tid == 32) tk = (long long)atomicAdd(ticket_ctr, 1ull);
#endif
#endif
        // store the parked tile (look-back for it first), then park this one
#if !SGI_ZONAL_STATIC && SGI_ZONAL_EARLY_TK && SGI_ZONAL_EARLY_TMA
        if (have_prev) flush_parked(tk);
        pre_issued = have_prev;
#else
        if (have_prev) flush_parked(-1);
#endif
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int sl = h * kFT + tid;
          park[0 * kFP + sl] = o[h].p0x;
          park[1 * kFP + sl] = o[h].p0y;
          park[2 * kFP + sl] = o[h].p1x;
          park[3 * kFP + sl] = o[h].p1y;
          park_meta[sl] = (unsigned)le[h] | ((unsigned)kk[h] << 10) | ((unsigned)o[h].count << 22) |
                          ((unsigned)ok[h] << 30) | ((unsigned)(h == 0 ? v0 : v1) << 31);
        }
        prev_t = t;
        prev_T = T;
        have_prev = true;
        lb_ready = false;
#if !SGI_ZONAL_STATIC && SGI_ZONAL_EARLY_TK
        if (tid == 32) S.ticket = tk;
#elif !SGI_ZONAL_STATIC
        if (tid == 0) S.ticket = (long long)atomicAdd(ticket_ctr, 1ull);
#endif
        break;
      }
      if (!have_prefix) {
        if (warp == 0) {
          const long long pre = t == 0 ? 0 : look_back(status, t);
          if (lane == 0) {
            if (t > 0) st_status(status + t, kInc | (unsigned long long)(pre + T));
            S.prefix = pre;
            if (t == ntiles - 1) *d_total = (unsigned long long)(pre + T);
          }
        }
        __syncthreads();
        have_prefix = true;
      }
      const long long base = S.prefix;
#if !SGI_ZONAL_STATIC
      if (tid == 0 && r0 + 2 * kFT >= T) S.ticket = (long long)atomicAdd(ticket_ctr, 1ull);
#endif
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!(h == 0 ? v0 : v1)) continue;
        const int64_t j = base + (h == 0 ? p0 : p1);
        if (j >= cap) continue;
        if (ok[h]) store_pair(o[h], zz[h], e0 + le[h], kk[h], j, cap, out_edge, out_lat, out_count,
                              out_xyz);
        else emit_exact<MODE>(va, vb, lde, tab, e0 + le[h], kk[h], j, cap, out_edge, out_lat,
                              out_count, out_xyz);
      }
    }
#if SGI_ZONAL_STATIC || !SGI_ZONAL_ONE_BARRIER
    __syncthreads();                   // the tile buffer and S are reused by the next tile
#endif
    // (otherwise the loop top's barrier, right after, is the one that guards that reuse)
  }
  if (have_prev) flush_parked(-1);
}

// ------------------------------------------------------- warp-specialised single-pass kernel
// The fused kernel's work split between 8 compute warps and one control warp (288 threads,
// 2 CTAs per SM at <= 112 registers), so the decoupled look-back leaves the compute warps'
// critical path: the control warp draws the tickets and issues each tile's bulk copies as soon
// as the compute warps release the tile buffer, then — once the compute warps have published the
// tile's count — walks back over the preceding tiles' status words and hands the output base
// over, while the compute warps run the tile's pairs.  Hand-offs are mbarriers (full: the
// tile's bytes / its ticket; agg: the tile's count is published; prefix: the base is known;
// free: the compute warps are done reading the tile buffer); the compute warps synchronise among
// themselves with named barrier 1.  Results equal the fused kernel's (same filter, scan and
// query code).
#ifndef SGI_ZONAL_WS
#define SGI_ZONAL_WS 0   // 1: this kernel instead of the fused one (0.47 vs 0.40 ms on C4: the
#endif                   // compute warps wait ~20% for the control warp's look-back, and 7
                         // compute warps leave tiles of 896 edges often needing a second round)
#ifndef SGI_ZONAL_WS_WARPS
#define SGI_ZONAL_WS_WARPS 7     // compute warps: 7 + 1 = 8 warps per CTA, 4 per sub-partition at
#endif                           // 2 CTAs per SM, so 128 registers (8 + 1 would cap them at 96)
constexpr int kWS = 32 * SGI_ZONAL_WS_WARPS; // compute threads
constexpr int kWSThreads = kWS + 32;        // plus the control warp
constexpr int kWSE = kFPer * kWS;           // edges per tile
constexpr int kWSP = 2 * kWS;               // pairs per round

struct WsSmem {
  alignas(16) int kcnt[kWSE];
  alignas(16) int excl[kWSE + 4];
  alignas(16) int klo[kWSE];
  int bkt[kBuckets + 1];
  unsigned short pmap[kWSP];
  unsigned wsum[kWS / 32];
  long long ticket[2];
  long long prefix;
  int total;
  uint64_t full, agg, pre, free_;
};

[[maybe_unused]] __device__ __forceinline__ void compute_sync() {   // (SGI_ZONAL_WS only)
  asm volatile("bar.sync 1, %0;" ::"n"(kWS) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(kWSThreads, 2)
sgi_zonal_ws_kernel(const double* __restrict__ va, const double* __restrict__ vb, int64_t ne,
                    int64_t lde, const double* __restrict__ lat, int nlat, int64_t cap,
                    int64_t* __restrict__ out_edge, int32_t* __restrict__ out_lat,
                    uint8_t* __restrict__ out_count, double* __restrict__ out_xyz,
                    unsigned long long* __restrict__ status, unsigned long long* d_total,
                    bool tma) {
  extern __shared__ __align__(128) double s_ws[];
  __shared__ WsSmem S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t lat_words = ((size_t)nlat + 15) / 16 * 16;
  double* tab = s_ws;
  double* tile = s_ws + lat_words;                                // [6][kWSE]
  sgi_poison_smem(&S, sizeof(S));
  sgi_poison_smem(s_ws + lat_words, 6 * kWSE * sizeof(double));
  __syncthreads();
  for (int k = tid; k < nlat; k += kWSThreads) tab[k] = lat[k];
  if (tid == 0) {
    mbar_init(&S.full, 1);
    mbar_init(&S.agg, 1);
    mbar_init(&S.pre, 1);
    mbar_init(&S.free_, kWS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  build_buckets(S.bkt, tab, nlat);                    // ends with a CTA barrier
  const int64_t ntiles = (ne + kWSE - 1) / kWSE;
  unsigned long long* ticket_ctr = status + ntiles;
  auto plane = [&](int c) { return (c < 3 ? va : vb) + (c % 3) * lde; };
  auto bulk_ok = [&](int64_t t) { return tma && t < ntiles && ne - t * kWSE >= kWSE; };
  constexpr bool kW2 = MODE == sgi::MODE_EFT || MODE == sgi::MODE_EFT_LITERAL;

  if (warp == kWS / 32) {
    // ------------------------------------------------------------------ control warp
    for (uint32_t i = 0;; ++i) {
      const uint32_t ph = i & 1;
      if (i > 0) mbar_wait(&S.free_, ph ^ 1);         // compute warps done with tile i - 1's buffer
      long long t = 0;
      if (lane == 0) {
        t = (long long)atomicAdd(ticket_ctr, 1ull);
        S.ticket[ph] = t;
        if (bulk_ok(t)) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&S.full, 6 * kWSE * 8);
#pragma unroll
          for (int c = 0; c < 6; ++c) bulk_g2s(tile + c * kWSE, plane(c) + t * kWSE, kWSE * 8, &S.full);
        } else {
          mbar_arrive(&S.full);                       // ticket only: the compute warps load it
        }
        // the tile a CTA draws next (about t + gridDim) into L2 under this one's arithmetic
        const int64_t tn = t + gridDim.x;
        if (bulk_ok(tn)) {
#pragma unroll
          for (int c = 0; c < 6; ++c)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(plane(c) + tn * kWSE),
                         "r"(kWSE * 8) : "memory");
        }
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntiles) break;
      mbar_wait(&S.agg, ph);                          // the tile's count is published
      const int T = S.total;
      const long long pre = t == 0 ? 0 : look_back(status, t);
      if (lane == 0) {
        if (t > 0) st_status(status + t, kInc | (unsigned long long)(pre + T));
        S.prefix = pre;
        if (t == ntiles - 1) *d_total = (unsigned long long)(pre + T);
        mbar_arrive(&S.pre);
      }
    }
    return;
  }

  // -------------------------------------------------------------------- compute warps
  for (uint32_t i = 0;; ++i) {
    const uint32_t ph = i & 1;
    mbar_wait(&S.full, ph);
    const int64_t t = S.ticket[ph];
    if (t >= ntiles) break;
    const int64_t e0 = t * kWSE;
    const int nv = (int)(ne - e0 < kWSE ? ne - e0 : kWSE);
    if (!bulk_ok(t)) {
      for (int q = tid; q < 6 * kWSE; q += kWS) {
        const int c = q / kWSE, l = q % kWSE;
        tile[q] = l < nv ? plane(c)[e0 + l] : 0.0;
      }
      compute_sync();
    }
    // filter: the four z-ranges of the thread's edges, then their table searches
    ZRange zr[kFPer];
#pragma unroll
    for (int j = 0; j < kFPer; ++j) {
      const int l = tid + j * kWS;
      double x[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) x[c] = tile[c * kWSE + l];
      zr[j] = zrange(x);
      if (l >= nv) zr[j].mode = 0;
    }
#pragma unroll
    for (int j = 0; j < kFPer; ++j) {
      const int l = tid + j * kWS;
      int klo, kcnt;
      range_search(zr[j], tab, S.bkt, nlat, klo, kcnt);
      S.klo[l] = klo;
      S.kcnt[l] = kcnt;
    }
    compute_sync();
    // block scan of the counts (thread tid: edges 4 tid .. 4 tid + 3) and the pair -> edge map
    const int4 c4 = *reinterpret_cast<const int4*>(&S.kcnt[kFPer * tid]);
    const unsigned mine = (unsigned)(c4.x + c4.y + c4.z + c4.w);
    unsigned incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane == 31) S.wsum[warp] = incl;
    compute_sync();
    unsigned before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWS / 32; ++w) {
      const unsigned x = S.wsum[w];
      before += w < warp ? x : 0;
      total += x;
    }
    {
      const int b = (int)(before + incl - mine);
      *reinterpret_cast<int4*>(&S.excl[kFPer * tid]) =
          make_int4(b, b + c4.x, b + c4.x + c4.y, b + c4.x + c4.y + c4.z);
      if (tid == kWS - 1) S.excl[kWSE] = (int)total;
      const int cs[4] = {c4.x, c4.y, c4.z, c4.w};
      int o = b;
#pragma unroll
      for (int j = 0; j < kFPer; ++j) {
        const unsigned short e = (unsigned short)(kFPer * tid + j);
        if (cs[j] == 1) {
          if (o < kWSP) S.pmap[o] = e;
        } else if (cs[j] > 1) {
          const int stop = min(o + cs[j], kWSP);
          for (int q = o; q < stop; ++q) S.pmap[q] = e;
        }
        o += cs[j];
      }
    }
    if (tid == 0) {
      st_status(status + t, (t == 0 ? kInc : kAgg) | (unsigned long long)total);
      S.total = (int)total;
      mbar_arrive(&S.agg);
    }
    compute_sync();
    const int T = (int)total;
    // the tile's pairs, kWSP per round (thread tid: pairs r0 + tid, r0 + kWS + tid)
    bool have_prefix = false;
    for (int r0 = 0; r0 < T || !have_prefix; r0 += kWSP) {
      const int p0 = r0 + tid, p1 = r0 + kWS + tid;
      const bool v0 = p0 < T, v1 = p1 < T;
      sgi::QueryOut o[2];
      bool ok[2] = {true, true};
      int le[2] = {0, 0}, kk[2] = {0, 0};
      double zz[2] = {0.0, 0.0};
      if (v0) {
        SGI_CHECK(S.excl[0] == 0 && S.excl[kWSE] == T);
        le[0] = p0 < kWSP ? (int)S.pmap[p0] : pair_edge<kWSE>(S.excl, p0);
        kk[0] = S.klo[le[0]] + (p0 - S.excl[le[0]]);
        le[1] = le[0];
        kk[1] = kk[0];
        if (v1) {
          le[1] = p1 < kWSP ? (int)S.pmap[p1] : pair_edge<kWSE>(S.excl, p1);
          kk[1] = S.klo[le[1]] + (p1 - S.excl[le[1]]);
        }
        SGI_CHECK(le[0] >= 0 && le[0] < nv && le[1] >= 0 && le[1] < nv);
        SGI_CHECK(kk[0] >= 0 && kk[0] < nlat && kk[1] >= 0 && kk[1] < nlat);
        zz[0] = tab[kk[0]];
        zz[1] = tab[kk[1]];
        if constexpr (kW2) {
          const SmemInTwo in = {smem_u32(tile + le[0]), smem_u32(tile + le[1]), kWSE * 8};
          sgi::QueryOut2 q;
          const sgi::B2 okb = sgi::query_fast2<MODE, ZCert>(in, sgi::W2{zz[0], zz[1]}, q);
          o[0] = {q.p0x.x, q.p0y.x, q.p1x.x, q.p1y.x, q.count[0]};
          o[1] = {q.p0x.y, q.p0y.y, q.p1x.y, q.p1y.y, q.count[1]};
          ok[0] = okb.x;
          ok[1] = okb.y;
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !v1) break;
            const sgi::SmemIn in = {smem_u32(tile + le[h]), kWSE * 8};
            ok[h] = sgi::query_fast<MODE, ZCert>(in, zz[h], o[h]);
          }
        }
      }
      if (r0 + kWSP >= T) {                          // the last round: the tile buffer is free
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.free_);
      }
      if (!have_prefix) {
        mbar_wait(&S.pre, ph);
        have_prefix = true;
      }
      const long long base = S.prefix;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!(h == 0 ? v0 : v1)) continue;
        const int64_t j = base + (h == 0 ? p0 : p1);
        if (j >= cap) continue;
        if (ok[h]) store_pair(o[h], zz[h], e0 + le[h], kk[h], j, cap, out_edge, out_lat, out_count,
                              out_xyz);
        else emit_exact<MODE>(va, vb, lde, tab, e0 + le[h], kk[h], j, cap, out_edge, out_lat,
                              out_count, out_xyz);
      }
    }
    compute_sync();                                  // S (excl, klo, prefix) reused by the next tile
  }
}

}  // namespace

extern "C" {

size_t sgi_zonal_workspace_bytes(int64_t n_edges) {
  if (n_edges < 0) return 0;
  const int64_t ntiles = (n_edges + kEdges - 1) / kEdges;
  return (size_t)n_edges * sizeof(int2) + (size_t)(ntiles + 1) * sizeof(unsigned long long);
}

sgi_status sgi_zonal_intersect(const double* va, const double* vb, int64_t n_edges, int64_t ld_e,
                               const double* lat_z0, int32_t n_lat, int64_t cap,
                               int64_t* out_edge, int32_t* out_lat, uint8_t* out_count,
                               double* out_xyz, unsigned long long* d_total, void* d_work,
                               size_t work_bytes, int mode, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_edges < 0 || ld_e < n_edges || n_lat < 0 || n_lat > (1 << 23) || cap < 0 || mode < SGI_MODE_NAIVE ||
      mode > SGI_MODE_NAIVE_KAHAN || !d_total) {
    sgi_internal::set_error_msg("sgi_zonal_intersect: invalid arguments", cudaSuccess);
    return SGI_E_INVALID;
  }
  if (n_edges > 0 && (!va || !vb || (n_lat > 0 && !lat_z0) || !d_work ||
                      ((uintptr_t)d_work & 15) != 0 ||
                      work_bytes < sgi_zonal_workspace_bytes(n_edges))) {
    sgi_internal::set_error_msg(
        "sgi_zonal_intersect: null pointer, workspace not 16-B aligned or too small", cudaSuccess);
    return SGI_E_INVALID;
  }
  if (cap > 0 && (!out_edge || !out_lat || !out_count || !out_xyz)) {
    sgi_internal::set_error_msg("sgi_zonal_intersect: null output with cap > 0", cudaSuccess);
    return SGI_E_INVALID;
  }
  cudaError_t e = cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) {
    sgi_internal::set_error_msg("sgi_zonal_intersect: cudaMemsetAsync", e);
    return SGI_E_CUDA;
  }
  if (n_edges == 0) return SGI_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t lat_smem = n_lat <= kLatSmem ? (size_t)n_lat * sizeof(double) : 0;
  const size_t lat_smem_even = n_lat <= kLatSmem ? ((size_t)n_lat + 1) / 2 * 2 * sizeof(double) : 0;
  const int64_t ntiles = (n_edges + kEdges - 1) / kEdges;
  int2* cand = (int2*)d_work;
  unsigned long long* tile = (unsigned long long*)((char*)d_work + (size_t)n_edges * sizeof(int2));
  // persistent grids: resident CTAs per SM x SMs, capped by the tile count
  auto grid_for = [&](auto kernel, size_t smem) {
    int occ = 1;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
    int64_t g = (int64_t)sms * (occ < 1 ? 1 : occ);
    return (int)(g < ntiles ? g : ntiles);
  };
  const bool smem_tab = n_lat <= kLatSmem;
  const int64_t ntiles_f = (n_edges + kFE - 1) / kFE;
  // status words of the single-pass kernels' tiles (+ the ticket counter)
  const int64_t nstatus = (SGI_ZONAL_WS ? (n_edges + kWSE - 1) / kWSE : ntiles_f) + 1;
  const bool fused = SGI_ZONAL_FUSED && cap > 0 && smem_tab &&
                     work_bytes >= (size_t)nstatus * sizeof(unsigned long long);
  if (fused) {
    // status words of the tiles and the ticket counter, zeroed for this call
    unsigned long long* status = (unsigned long long*)d_work;
    e = cudaMemsetAsync(status, 0, (size_t)nstatus * sizeof(unsigned long long), st);
    if (e != cudaSuccess) {
      sgi_internal::set_error_msg("sgi_zonal_intersect: cudaMemsetAsync", e);
      return SGI_E_CUDA;
    }
    const bool tma = ((((uintptr_t)va | (uintptr_t)vb) & 15) == 0) && (ld_e % 2 == 0);
    const size_t smem = ((size_t)n_lat + 15) / 16 * 16 * sizeof(double) + 6 * kFE * sizeof(double) +
                        (SGI_ZONAL_PARK ? 4 * kFP * sizeof(double) + kFP * sizeof(unsigned) : 0);
    auto fk = [&](auto kernel) {
      int occ = 1;
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kFT, smem);
      const int64_t g = (int64_t)sms * (occ < 1 ? 1 : occ);
      const int grid = (int)(g < ntiles_f ? g : ntiles_f);
#if SGI_ZONAL_STATIC
      // cooperative launch: all CTAs co-resident (the static look-back relies on it)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(kFT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      e = cudaLaunchKernelEx(&cfg, kernel, va, vb, n_edges, ld_e, lat_z0, (int)n_lat, cap, out_edge,
                             out_lat, out_count, out_xyz, status, d_total, tma);
#else
      kernel<<<grid, kFT, smem, st>>>(va, vb, n_edges, ld_e, lat_z0, n_lat, cap, out_edge, out_lat,
                                      out_count, out_xyz, status, d_total, tma);
#endif
    };
#if SGI_ZONAL_WS
    const size_t wsmem = ((size_t)n_lat + 15) / 16 * 16 * sizeof(double) + 6 * kWSE * sizeof(double);
    const int64_t ntiles_w = (n_edges + kWSE - 1) / kWSE;
    auto wk = [&](auto kernel) {
      const size_t smem = wsmem;
      int occ = 1;
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kWSThreads, smem);
      const int64_t g = (int64_t)sms * (occ < 1 ? 1 : occ);
      kernel<<<(int)(g < ntiles_w ? g : ntiles_w), kWSThreads, smem, st>>>(
          va, vb, n_edges, ld_e, lat_z0, (int)n_lat, cap, out_edge, out_lat, out_count, out_xyz,
          status, d_total, tma);
    };
    switch (mode) {
      case SGI_MODE_NAIVE: wk(sgi_zonal_ws_kernel<sgi::MODE_NAIVE>); break;
      case SGI_MODE_EFT: wk(sgi_zonal_ws_kernel<sgi::MODE_EFT>); break;
      case SGI_MODE_EFT_LITERAL: wk(sgi_zonal_ws_kernel<sgi::MODE_EFT_LITERAL>); break;
      case SGI_MODE_YAC: wk(sgi_zonal_ws_kernel<sgi::MODE_YAC>); break;
      case SGI_MODE_BASE: wk(sgi_zonal_ws_kernel<sgi::MODE_BASE>); break;
      default: wk(sgi_zonal_ws_kernel<sgi::MODE_NAIVE_KAHAN>); break;
    }
    if (false)
#endif
    switch (mode) {
      case SGI_MODE_NAIVE: fk(sgi_zonal_fused_kernel<sgi::MODE_NAIVE>); break;
      case SGI_MODE_EFT: fk(sgi_zonal_fused_kernel<sgi::MODE_EFT>); break;
      case SGI_MODE_EFT_LITERAL: fk(sgi_zonal_fused_kernel<sgi::MODE_EFT_LITERAL>); break;
      case SGI_MODE_YAC: fk(sgi_zonal_fused_kernel<sgi::MODE_YAC>); break;
      case SGI_MODE_BASE: fk(sgi_zonal_fused_kernel<sgi::MODE_BASE>); break;
      default: fk(sgi_zonal_fused_kernel<sgi::MODE_NAIVE_KAHAN>); break;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) {
      sgi_internal::set_error_msg("sgi_zonal_fused_kernel launch", e);
      return SGI_E_CUDA;
    }
    return SGI_OK;
  }
  const size_t filter_smem = (SGI_ZONAL_FILTER_PREFETCH == 2 ? lat_smem_even : lat_smem) +
                             (SGI_ZONAL_FILTER_PREFETCH == 2 ? 2 * 6 * kEdges * sizeof(double) : 0);
  if (smem_tab) {
    const int gf = grid_for(sgi_zonal_filter_kernel<true>, filter_smem);
    sgi_zonal_filter_kernel<true><<<gf, kThreads, filter_smem, st>>>(va, vb, n_edges, ld_e, lat_z0,
                                                                     n_lat, cand, tile);
  } else {
    const int gf = grid_for(sgi_zonal_filter_kernel<false>, filter_smem);
    sgi_zonal_filter_kernel<false><<<gf, kThreads, filter_smem, st>>>(va, vb, n_edges, ld_e, lat_z0,
                                                                      n_lat, cand, tile);
  }
  cudaFuncSetAttribute(sgi_zonal_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kScanSmem);
  sgi_zonal_scan_kernel<<<1, kScanThreads, kScanSmem, st>>>(tile, ntiles, d_total);
  if (cap > 0) {
    auto emit = [&](auto kernel) {
      int occ = 1;
      const size_t smem = lat_smem_even + kWarpsPerCta * sizeof(WarpSmem);
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kWThreads, smem);
      const int64_t want = (ntiles + kWarpsPerCta - 1) / kWarpsPerCta;
      const int64_t g = (int64_t)sms * (occ < 1 ? 1 : occ);
      kernel<<<(int)(g < want ? g : want), kWThreads, smem, st>>>(
          va, vb, n_edges, ld_e, lat_z0, n_lat, cap, out_edge, out_lat, out_count, out_xyz, cand,
          tile);
    };
#define SGI_EMIT(M) (smem_tab ? emit(sgi_zonal_emit_warp_kernel<M, true>) : emit(sgi_zonal_emit_warp_kernel<M, false>))
    switch (mode) {
      case SGI_MODE_NAIVE: SGI_EMIT(sgi::MODE_NAIVE); break;
      case SGI_MODE_EFT: SGI_EMIT(sgi::MODE_EFT); break;
      case SGI_MODE_EFT_LITERAL: SGI_EMIT(sgi::MODE_EFT_LITERAL); break;
      case SGI_MODE_YAC: SGI_EMIT(sgi::MODE_YAC); break;
      case SGI_MODE_BASE: SGI_EMIT(sgi::MODE_BASE); break;
      default: SGI_EMIT(sgi::MODE_NAIVE_KAHAN); break;
    }
#undef SGI_EMIT
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    sgi_internal::set_error_msg("sgi_zonal kernels launch", e);
    return SGI_E_CUDA;
  }
  return SGI_OK;
}

}  // extern "C"
