// sgi_zonal.cu — fused zonal-mean pass: mesh edges x latitude table -> compacted intersections
// (the paper's motivating application, zonal means on regridding meshes).
//
// Three launches over tiles of kEdges consecutive edges:
//   filter per edge, from the accurate (AccuDOP) normal rounded once, the arc's z-range: the
//          endpoints' z/|x| and, when the great circle's extremum lies strictly inside the arc
//          (dz/dt changes sign: g1 = (n x a)_z > 0 > g2 = (n x b)_z for a maximum), the apex
//          height sqrt(|n_xy|^2/|n|^2); widened by delta = 2^-40 (far above its rounding error);
//          a search in the latitude table (shared memory) gives the candidate latitudes
//          [klo, klo + kcnt), stored per edge (8 B) with each tile's candidate sum;
//   scan   one CTA turns the tile sums into output bases (and the total);
//   emit   CTAs walk tiles in any order (each tile knows its base): a block scan of the stored
//          kcnt orders the tile's candidates (edge-major, latitude ascending, deterministic)
//          and compacts the candidate edges; only those are read again, one per thread, and
//          get the query's z0-independent AccuX head (accurate normal pairs, |n_xy|^2, |n|^2 —
//          lines 2-6), staged in shared memory; the tile's pairs are then processed
//          densely (pair c -> thread c mod kThreads,
//          so lanes are not idle on edges that span no latitude), running the z0-dependent tail
//          of the query (AccuX lines 7-25 + containment).
// A pair's result is bit-identical to sgi_intersect_arc_lat on the same (a, b, z0): head and
// tail are the same device code.  Candidate pairs whose latitude only touches the widened range
// come out with count 0; every pair with a nonzero count is a candidate (tests/test_gpu_zonal.py).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "sgi.h"
#include "sgi_query.cuh"

namespace sgi_internal {
void set_error_msg(const char* msg, cudaError_t e);   // sgi_capi.cu: sgi_last_error() text
}

namespace {

#ifndef SGI_ZONAL_THREADS
#define SGI_ZONAL_THREADS 256
#endif
#ifndef SGI_ZONAL_FILTER_MINB
#define SGI_ZONAL_FILTER_MINB 1
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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// A bucket index over z in [-1, 1] turns each table search into one shared-memory lookup plus a
// short binary search: bkt[b] = lower_bound(tab, -1 + 2b/kBuckets) for b = 0..kBuckets (the
// boundaries are exact binary fractions).  For x in bucket b (computed up to one bucket of
// rounding) the answer lies between the bounds of buckets b-1 and b+2; outside [-1, 1] the
// bracket opens to the table's ends, so any strictly increasing table is handled.
constexpr int kBuckets = 2048;

__device__ __forceinline__ void build_buckets(int* bkt, const double* tab, int nlat) {
  for (int b = threadIdx.x; b <= kBuckets; b += blockDim.x)
    bkt[b] = lower_bound(tab, nlat, -1.0 + (double)b * (2.0 / kBuckets));
  __syncthreads();
}

template <bool UPPER>   // false: first k with tab[k] >= x; true: first k with tab[k] > x
__device__ __forceinline__ int bucket_search(const int* bkt, const double* tab, int nlat, double x) {
  // the bucket only has to be right to within one (the bracket spans b-1 .. b+2): float32 is
  // far more than enough (NaN never reaches here: the caller screens it)
  const float f = fminf(fmaxf(__fmul_rn(__fadd_rn((float)x, 1.0f), (float)(kBuckets / 2)), 0.0f),
                        (float)(kBuckets - 1));
  const int b = (int)f;
  const int lo = b >= 1 ? bkt[b - 1] : 0;
  const int hi = b + 2 <= kBuckets - 1 ? bkt[b + 2] : nlat;
  return lo + (UPPER ? upper_bound(tab + lo, hi - lo, x) : lower_bound(tab + lo, hi - lo, x));
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

// Candidate latitudes [klo, klo + kcnt) of one edge (see the file comment).  The filter needs the
// direction of n only to a few ulps: it takes the renormalised EFT normal's high parts (RN of the
// exact n, so short arcs keep their accuracy) and evaluates heights with the device rsqrt (a few
// ulps, deterministic) — errors ~1e-15, far below delta.
__device__ __forceinline__ void candidates(const double* x, const double* tab, const int* bkt,
                                           int nlat, int& klo, int& kcnt) {
  klo = 0;
  kcnt = 0;
  const sgi::dd nxp = sgi::accu_dop(x[1], x[5], x[2], x[4]);
  const sgi::dd nyp = sgi::accu_dop(x[2], x[3], x[0], x[5]);
  const sgi::dd nzp = sgi::accu_dop(x[0], x[4], x[1], x[3]);
  const double nx = __dadd_rn(nxp.hi, nxp.lo), ny = __dadd_rn(nyp.hi, nyp.lo);
  const double nz = __dadd_rn(nzp.hi, nzp.lo);
  const double ra2 = __dadd_rn(__dadd_rn(__dmul_rn(x[0], x[0]), __dmul_rn(x[1], x[1])), __dmul_rn(x[2], x[2]));
  const double rb2 = __dadd_rn(__dadd_rn(__dmul_rn(x[3], x[3]), __dmul_rn(x[4], x[4])), __dmul_rn(x[5], x[5]));
  const double za = __dmul_rn(x[2], fast_rsqrt(ra2)), zb = __dmul_rn(x[5], fast_rsqrt(rb2));
  const double g1 = __dsub_rn(__dmul_rn(nx, x[1]), __dmul_rn(ny, x[0]));
  const double g2 = __dsub_rn(__dmul_rn(nx, x[4]), __dmul_rn(ny, x[3]));
  double zhi = fmax(za, zb), zlo = fmin(za, zb);
  const bool top_inside = g1 > 0.0 && g2 < 0.0, bottom_inside = g1 < 0.0 && g2 > 0.0;
  if (top_inside || bottom_inside) {                 // the circle's extremum is on the arc
    const double s2 = __dadd_rn(__dmul_rn(nx, nx), __dmul_rn(ny, ny));
    const double s3 = __dadd_rn(s2, __dmul_rn(nz, nz));
    const double h = s2 > 0.0 ? __dmul_rn(__dmul_rn(s2, fast_rsqrt(s2)), fast_rsqrt(s3)) : 0.0;
    if (top_inside) zhi = fmax(zhi, h);
    else zlo = fmin(zlo, -h);
  }
  if (nx == 0.0 && ny == 0.0 && nz == 0.0) {
    kcnt = nlat;                                     // n = 0: degenerate at every latitude
  } else if (zhi == zhi && zlo == zlo) {             // NaN inputs: no candidates
    klo = bucket_search<false>(bkt, tab, nlat, __dsub_rn(zlo, kDelta));
    kcnt = bucket_search<true>(bkt, tab, nlat, __dadd_rn(zhi, kDelta)) - klo;
  }
}


// Block-wide inclusive scan of one 64-bit value per thread (kThreads threads); returns the
// inclusive value and leaves the block total in *total.
__device__ __forceinline__ unsigned long long block_scan(unsigned long long v,
                                                         unsigned long long* s_warp,
                                                         unsigned long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += y;
  }
  if (lane == 31) s_warp[warp] = v;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < kThreads / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < kThreads / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const unsigned long long incl = v + (warp > 0 ? s_warp[warp - 1] : 0);
  *total = s_warp[kThreads / 32 - 1];
  return incl;
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
  __shared__ unsigned long long s_red[kThreads / 32];
  __shared__ int s_bkt[kBuckets + 1];
  if (SMEM) {
    for (int k = threadIdx.x; k < nlat; k += kThreads) s_lat[k] = lat[k];
    __syncthreads();
  }
  const double* tab = SMEM ? s_lat : lat;
  build_buckets(s_bkt, tab, nlat);
  const int64_t ntiles = (ne + kEdges - 1) / kEdges;
  int64_t t = blockIdx.x;
  EdgeX cur[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int64_t e = t * kEdges + 2 * threadIdx.x + j;
    if (t < ntiles && e < ne) load_edge(cur[j], va, vb, lde, e);
  }
  for (; t < ntiles; t += gridDim.x) {
    const int64_t e0 = t * kEdges + 2 * threadIdx.x, en = e0 + (int64_t)gridDim.x * kEdges;
    EdgeX nxt[2];
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (en + j < ne) load_edge(nxt[j], va, vb, lde, en + j);
    unsigned long long sum = 0;
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
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long acc = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) acc += s_red[w];
      tile_sum[t] = acc;
    }
    __syncthreads();
    cur[0] = nxt[0];
    cur[1] = nxt[1];
  }
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

// Pass 3: emit every candidate pair of each tile at its ordered output slot.
//
// Each tile's endpoint planes and candidate ranges are staged in shared memory by cp.async one
// tile ahead (double buffer), so the compute never waits on a gather.  A block scan of the
// stored kcnt compacts the tile's candidate edges in edge order; then, when every candidate
// spans at most kFuseMax latitudes (the common case: mesh edges are short), one thread per
// candidate runs the query's z0-independent AccuX head (lines 2-6) once and the z0-dependent
// tail (lines 7-25 + containment) for each of its latitudes.  Tiles with a long candidate range
// process their pairs densely instead (pair c -> thread c mod kThreads, head recomputed per
// pair), so no lane idles behind one long edge.
constexpr int kFuseMax = 4;
struct EmitStage {                 // one tile's inputs
  double x[6][kEdges];             // endpoint planes a_x, a_y, a_z, b_x, b_y, b_z
  int2 cand[kEdges];               // (klo, kcnt) per edge
};
struct EmitList {                  // the tile's compacted candidate edges
  int edge[kEdges];                // tile-local edge index of candidate c
  int klo[kEdges];                 // first candidate latitude of candidate c
  int kcnt[kEdges];                // number of candidate latitudes of candidate c
  long long off[kEdges];           // first pair of candidate c within the tile
};
struct EmitSmem {
  EmitStage stage[2];
  EmitList list[2];
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

// Thread tid stages edges 2 tid, 2 tid + 1 of tile t (those below ne) and commits the group.
__device__ __forceinline__ void stage_tile(EmitStage& S, int64_t t, int64_t ne, int64_t lde,
                                           const double* __restrict__ va,
                                           const double* __restrict__ vb,
                                           const int2* __restrict__ cand) {
  const int l0 = 2 * threadIdx.x;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int64_t e = t * kEdges + l0 + j;
    if (e < ne) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        cp_async8(&S.x[c][l0 + j], va + c * lde + e);
        cp_async8(&S.x[3 + c][l0 + j], vb + c * lde + e);
      }
      cp_async8(&S.cand[l0 + j], cand + e);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int MODE, class IN>
__device__ __forceinline__ void emit_pair(const sgi::EdgePre& pre, const IN& in, int64_t edge,
                                          int k, const double* tab, int64_t j, int64_t cap,
                                          int64_t* __restrict__ out_edge,
                                          int32_t* __restrict__ out_lat,
                                          uint8_t* __restrict__ out_count,
                                          double* __restrict__ out_xyz) {
  const double z0 = tab[k];
  sgi::QueryOut o;
  if (!sgi::lat_query<MODE, sgi::Fast>(pre, in, z0, o)) {
    const sgi::RegIn r = {{in(0), in(1), in(2), in(3), in(4), in(5)}};
    sgi::query_exact<MODE>(r, z0, o);
  }
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

template <int MODE, bool SMEM>
__global__ void __launch_bounds__(kThreads, 512 / kThreads)
sgi_zonal_emit_kernel(const double* __restrict__ va, const double* __restrict__ vb, int64_t ne,
                      int64_t lde, const double* __restrict__ lat, int nlat, int64_t cap,
                      int64_t* __restrict__ out_edge, int32_t* __restrict__ out_lat,
                      uint8_t* __restrict__ out_count, double* __restrict__ out_xyz,
                      const int2* __restrict__ cand,
                      const unsigned long long* __restrict__ tile_base) {
  extern __shared__ __align__(16) double s_dyn[];
  __shared__ unsigned long long s_warp[kThreads / 32];
  const int tid = threadIdx.x;
  const size_t lat_words = SMEM ? ((size_t)nlat + 1) / 2 * 2 : 0;
  EmitSmem& S = *reinterpret_cast<EmitSmem*>(s_dyn + lat_words);
  if (SMEM) {
    for (int k = threadIdx.x; k < nlat; k += kThreads) s_dyn[k] = lat[k];
    __syncthreads();
  }
  const double* tab = SMEM ? s_dyn : lat;
  const int64_t ntiles = (ne + kEdges - 1) / kEdges;
  int buf = 0;
  if ((int64_t)blockIdx.x < ntiles) stage_tile(S.stage[0], blockIdx.x, ne, lde, va, vb, cand);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, buf ^= 1) {
    asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's copies of tile t
    EmitStage& G = S.stage[buf];
    EmitList& L = S.list[buf];
    const int64_t base = (int64_t)tile_base[t];
    const int l0 = 2 * tid;
    const int64_t e0 = t * kEdges + l0;
    const int2 c0 = e0 < ne ? G.cand[l0] : make_int2(0, 0);
    const int2 c1 = e0 + 1 < ne ? G.cand[l0 + 1] : make_int2(0, 0);
    // pairs (high 40 bits) and candidate flags (low 24 bits) of this thread's two edges
    const unsigned long long pairs = (unsigned long long)(unsigned)c0.y + (unsigned)c1.y;
    const unsigned flags = (c0.y > 0) + (c1.y > 0);
    const unsigned long long mine = (pairs << 24) | flags;
    unsigned long long tot;
    const unsigned long long excl = block_scan(mine, s_warp, &tot) - mine;  // (barriers)
    const int ncand = (int)(tot & 0xFFFFFF);
    const int64_t npairs = (int64_t)(tot >> 24);
    int slot = (int)(excl & 0xFFFFFF);
    int64_t poff = (int64_t)(excl >> 24);
    if (c0.y > 0) {
      L.edge[slot] = l0; L.klo[slot] = c0.x; L.kcnt[slot] = c0.y; L.off[slot] = poff; ++slot;
    }
    poff += c0.y;
    if (c1.y > 0) { L.edge[slot] = l0 + 1; L.klo[slot] = c1.x; L.kcnt[slot] = c1.y; L.off[slot] = poff; }
    // the list is complete, every thread's tile-t data is visible, and every thread is done
    // with tile t - gridDim.x, whose buffer the next tile's copies now overwrite
    const bool dense = __syncthreads_or(c0.y > kFuseMax || c1.y > kFuseMax);
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) stage_tile(S.stage[buf ^ 1], tn, ne, lde, va, vb, cand);
    const uint32_t gx = smem_u32(&G.x[0][0]);
    if (!dense) {
      for (int c = tid; c < ncand; c += kThreads) {     // head once, then its latitudes
        const int le = L.edge[c];
        const sgi::SmemIn in = {gx + (uint32_t)le * 8u, (uint32_t)(kEdges * 8)};
        const sgi::EdgePre pre = sgi::edge_pre<MODE>(in);
        const int kc = L.kcnt[c], k0 = L.klo[c];
        const int64_t j0 = base + L.off[c];
        for (int q = 0; q < kc && j0 + q < cap; ++q)
          emit_pair<MODE>(pre, in, t * kEdges + le, k0 + q, tab, j0 + q, cap, out_edge, out_lat,
                          out_count, out_xyz);
      }
    } else {
      for (int64_t p = tid; p < npairs && base + p < cap; p += kThreads) {
        int l = 0, h = ncand;                            // owner candidate: last off[l] <= p
        while (h - l > 1) {
          const int mid = (l + h) >> 1;
          if (L.off[mid] <= p) l = mid; else h = mid;
        }
        const int le = L.edge[l];
        const sgi::SmemIn in = {gx + (uint32_t)le * 8u, (uint32_t)(kEdges * 8)};
        emit_pair<MODE>(sgi::edge_pre<MODE>(in), in, t * kEdges + le,
                        L.klo[l] + (int)(p - L.off[l]), tab, base + p, cap, out_edge, out_lat,
                        out_count, out_xyz);
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
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
                      work_bytes < sgi_zonal_workspace_bytes(n_edges))) {
    sgi_internal::set_error_msg("sgi_zonal_intersect: null pointer or workspace too small",
                                cudaSuccess);
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
  const size_t emit_smem = lat_smem_even + sizeof(EmitSmem);
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
  const size_t filter_smem = lat_smem;
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
      const int ge = grid_for(kernel, emit_smem);
      kernel<<<ge, kThreads, emit_smem, st>>>(va, vb, n_edges, ld_e, lat_z0, n_lat, cap, out_edge,
                                              out_lat, out_count, out_xyz, cand, tile);
    };
#define SGI_EMIT(M) (smem_tab ? emit(sgi_zonal_emit_kernel<M, true>) : emit(sgi_zonal_emit_kernel<M, false>))
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
