// sgi_zonal.cu — fused zonal-mean pass: mesh edges x latitude table -> compacted intersections
// (the paper's motivating application, zonal means on regridding meshes).
//
// Every CTA owns one contiguous range of edges (equal sizes, rounded to tiles of kTile edges),
// and the pass runs as three launches:
//   count  per edge, from the accurate (AccuDOP) normal rounded once, the arc's z-range: the
//          endpoints' z/|x| and, when the great circle's extremum lies strictly inside the arc
//          (dz/dt changes sign: g1 = (n x a)_z > 0 > g2 = (n x b)_z for a maximum), the apex
//          height sqrt(|n_xy|^2/|n|^2); widened by delta = 2^-40 (far above its rounding error);
//          a binary search in the latitude table (shared memory) gives the candidate latitudes;
//          each CTA sums its candidates;
//   scan   one CTA turns the per-CTA sums into output bases (and the total);
//   emit   each CTA re-walks its range tile by tile: the same filter, plus the query's
//          z0-independent AccuX head (accurate normal pairs, |n_xy|^2, |n|^2 — lines 2-6,
//          P:746-750), staged in shared memory with the endpoints; a block scan orders the tile's candidates (edge-major, latitude
//          ascending, deterministic), and the tile's pairs are processed densely (pair c ->
//          thread c mod kTile, so lanes are not idle on edges that span no latitude), running the
//          z0-dependent tail of the query (AccuX lines 7-25 + containment).
// Edges are read twice (48 B each, 2 x 0.6 GB for the C4 mesh) instead of paying a device-wide
// decoupled look-back per tile, whose frontier propagation limited a single-pass version to a
// fraction of this throughput.  A pair's result is bit-identical to
// sgi_intersect_arc_lat on the same (a, b, z0): head and tail are the same device code.
// Candidate pairs whose latitude only touches the widened range come out with count 0; every
// pair with a nonzero count is a candidate (tests/test_gpu_zonal.py).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "sgi.h"
#include "sgi_query.cuh"

namespace sgi_internal {
void set_error_msg(const char* msg, cudaError_t e);   // sgi_capi.cu: sgi_last_error() text
}

namespace {

constexpr int kTile = 256;                        // threads per CTA = edges per tile
constexpr int kLatSmem = 4096;                    // latitude tables up to this length live in smem
constexpr int kMaxCtas = 4096;                    // per-CTA sums held in the workspace
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

struct SmemEdge {   // endpoint coordinates of one staged edge, read by pair threads
  const double* p;  // 6 doubles, contiguous
  __device__ __forceinline__ double operator()(int c) const { return p[c]; }
};

struct EdgeX {
  double x[6];
};

__device__ __forceinline__ void load_edge(EdgeX& r, const double* __restrict__ va,
                                          const double* __restrict__ vb, int64_t lde, int64_t e) {
  r.x[0] = __ldg(va + e); r.x[1] = __ldg(va + lde + e); r.x[2] = __ldg(va + 2 * lde + e);
  r.x[3] = __ldg(vb + e); r.x[4] = __ldg(vb + lde + e); r.x[5] = __ldg(vb + 2 * lde + e);
}

// Candidate latitudes [klo, klo + kcnt) of one edge (see the file comment).  The filter needs the
// direction of n only to a few ulps: it takes the renormalised EFT normal's high parts (RN of the
// exact n, so short arcs keep their accuracy) and evaluates heights with the device rsqrt (a few
// ulps, deterministic) — errors ~1e-15, far below delta.  count and emit run this same code.
__device__ __forceinline__ void candidates(const double* x, const double* tab, int nlat, int& klo,
                                           int& kcnt) {
  klo = 0;
  kcnt = 0;
  const sgi::dd nxp = sgi::accu_dop(x[1], x[5], x[2], x[4]);
  const sgi::dd nyp = sgi::accu_dop(x[2], x[3], x[0], x[5]);
  const sgi::dd nzp = sgi::accu_dop(x[0], x[4], x[1], x[3]);
  const double nx = __dadd_rn(nxp.hi, nxp.lo), ny = __dadd_rn(nyp.hi, nyp.lo);
  const double nz = __dadd_rn(nzp.hi, nzp.lo);
  const double ra2 = __dadd_rn(__dadd_rn(__dmul_rn(x[0], x[0]), __dmul_rn(x[1], x[1])), __dmul_rn(x[2], x[2]));
  const double rb2 = __dadd_rn(__dadd_rn(__dmul_rn(x[3], x[3]), __dmul_rn(x[4], x[4])), __dmul_rn(x[5], x[5]));
  const double za = __dmul_rn(x[2], rsqrt(ra2)), zb = __dmul_rn(x[5], rsqrt(rb2));
  const double g1 = __dsub_rn(__dmul_rn(nx, x[1]), __dmul_rn(ny, x[0]));
  const double g2 = __dsub_rn(__dmul_rn(nx, x[4]), __dmul_rn(ny, x[3]));
  const double s2 = __dadd_rn(__dmul_rn(nx, nx), __dmul_rn(ny, ny));
  const double s3 = __dadd_rn(s2, __dmul_rn(nz, nz));
  const double h = s3 > 0.0 ? __dmul_rn(__dsqrt_rn(s2), rsqrt(s3)) : 0.0;
  double zhi = fmax(za, zb), zlo = fmin(za, zb);
  if (g1 > 0.0 && g2 < 0.0) zhi = fmax(zhi, h);
  if (g1 < 0.0 && g2 > 0.0) zlo = fmin(zlo, -h);
  if (nx == 0.0 && ny == 0.0 && nz == 0.0) {
    kcnt = nlat;                                     // n = 0: degenerate at every latitude
  } else if (zhi == zhi && zlo == zlo) {             // NaN inputs: no candidates
    klo = lower_bound(tab, nlat, __dsub_rn(zlo, kDelta));
    kcnt = upper_bound(tab, nlat, __dadd_rn(zhi, kDelta)) - klo;
  }
}

__device__ __forceinline__ void cta_range(int64_t ne, int64_t& lo, int64_t& hi) {
  const int64_t per = ((ne + gridDim.x - 1) / gridDim.x + kTile - 1) / kTile * kTile;
  lo = (int64_t)blockIdx.x * per;
  hi = lo + per < ne ? lo + per : ne;
}

__device__ __forceinline__ const double* stage_lat(double* s_lat, const double* lat, int nlat) {
  if (nlat <= kLatSmem) {
    for (int k = threadIdx.x; k < nlat; k += kTile) s_lat[k] = lat[k];
    __syncthreads();
    return s_lat;
  }
  return lat;
}

// Block-wide inclusive scan of one int per thread (kTile threads); returns the inclusive value
// and leaves the block total in *total.
__device__ __forceinline__ int block_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += y;
  }
  if (lane == 31) s_warp[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kTile / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < kTile / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const int incl = v + (warp > 0 ? s_warp[warp - 1] : 0);
  *total = s_warp[kTile / 32 - 1];
  return incl;
}

// Pass 1: candidate count of every CTA's edge range.
__global__ void __launch_bounds__(kTile)
sgi_zonal_count_kernel(const double* __restrict__ va, const double* __restrict__ vb, int64_t ne,
                       int64_t lde, const double* __restrict__ lat, int nlat,
                       unsigned long long* __restrict__ cta_sum) {
  extern __shared__ __align__(16) double s_lat[];
  const double* tab = stage_lat(s_lat, lat, nlat);
  int64_t lo, hi;
  cta_range(ne, lo, hi);
  unsigned long long acc = 0;
  EdgeX cur;
  int64_t e = lo + threadIdx.x;
  if (e < hi) load_edge(cur, va, vb, lde, e);
  for (; e - threadIdx.x < hi; e += kTile) {
    EdgeX nxt;
    if (e + kTile < hi) load_edge(nxt, va, vb, lde, e + kTile);
    if (e < hi) {
      int klo, kcnt;
      candidates(cur.x, tab, nlat, klo, kcnt);
      acc += (unsigned long long)kcnt;
    }
    cur = nxt;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  __shared__ unsigned long long s_acc;
  if (threadIdx.x == 0) s_acc = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_acc, acc);
  __syncthreads();
  if (threadIdx.x == 0) cta_sum[blockIdx.x] = s_acc;
}

// Pass 2: exclusive scan of the per-CTA sums (one CTA), total to *d_total.
__global__ void __launch_bounds__(1024)
sgi_zonal_scan_kernel(unsigned long long* __restrict__ cta_sum, int nctas,
                      unsigned long long* __restrict__ d_total) {
  __shared__ unsigned long long s[kMaxCtas];
  for (int i = threadIdx.x; i < nctas; i += blockDim.x) s[i] = cta_sum[i];
  __syncthreads();
  if (threadIdx.x == 0) {                       // <= 4096 entries: a serial scan is ~microseconds
    unsigned long long run = 0;
    for (int i = 0; i < nctas; ++i) {
      const unsigned long long v = s[i];
      s[i] = run;
      run += v;
    }
    *d_total = run;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nctas; i += blockDim.x) cta_sum[i] = s[i];
}

// Pass 3: emit every candidate pair of the CTA's range at its ordered output slot.
constexpr size_t kEmitSmem = 0;

template <int MODE>
__global__ void __launch_bounds__(kTile)
sgi_zonal_emit_kernel(const double* __restrict__ va, const double* __restrict__ vb, int64_t ne,
                      int64_t lde, const double* __restrict__ lat, int nlat, int64_t cap,
                      int64_t* __restrict__ out_edge, int32_t* __restrict__ out_lat,
                      uint8_t* __restrict__ out_count, double* __restrict__ out_xyz,
                      const unsigned long long* __restrict__ cta_base) {
  extern __shared__ __align__(16) double s_lat[];
  __shared__ double s_xyz[kTile][6];
  __shared__ sgi::EdgePre s_pre[kTile];
  __shared__ int s_klo[kTile], s_off[kTile];
  __shared__ int s_warp[kTile / 32];
  const int tid = threadIdx.x;
  const double* tab = stage_lat(s_lat, lat, nlat);
  int64_t lo, hi;
  cta_range(ne, lo, hi);
  int64_t base = (int64_t)cta_base[blockIdx.x];
  EdgeX cur;
  if (lo + tid < hi) load_edge(cur, va, vb, lde, lo + tid);
  for (int64_t t0 = lo; t0 < hi && base < cap; t0 += kTile) {
    const int64_t e = t0 + tid;
    EdgeX nxt;
    if (e + kTile < hi) load_edge(nxt, va, vb, lde, e + kTile);
    int klo = 0, kcnt = 0;
    if (e < hi) {
      candidates(cur.x, tab, nlat, klo, kcnt);
#pragma unroll
      for (int c = 0; c < 6; ++c) s_xyz[tid][c] = cur.x[c];
      if (kcnt > 0) {
        const sgi::RegIn in = {{cur.x[0], cur.x[1], cur.x[2], cur.x[3], cur.x[4], cur.x[5]}};
        s_pre[tid] = sgi::edge_pre<MODE>(in);
      }
    }
    s_klo[tid] = klo;
    int total;
    const int incl = block_scan(kcnt, s_warp, &total);
    s_off[tid] = incl - kcnt;
    __syncthreads();                                 // staging and offsets complete
    for (int c = tid; c < total; c += kTile) {
      const int64_t j = base + c;
      if (j >= cap) break;
      int l = 0, h = kTile;                          // owner edge: last s_off[t] <= c
      while (h - l > 1) {
        int mid = (l + h) >> 1;
        if (s_off[mid] <= c) l = mid; else h = mid;
      }
      const int t = l;
      const int k = s_klo[t] + (c - s_off[t]);
      const double z0 = tab[k];
      const SmemEdge in = {s_xyz[t]};
      sgi::QueryOut o;
      if (!sgi::lat_query<MODE, sgi::Fast>(s_pre[t], in, z0, o)) {
        const sgi::RegIn r = {{in(0), in(1), in(2), in(3), in(4), in(5)}};
        sgi::query_exact<MODE>(r, z0, o);
      }
      const bool deg = o.count == sgi::kDegenerate;
      const double nan = sgi::qnan();
      out_edge[j] = t0 + t;
      out_lat[j] = k;
      out_count[j] = o.count;
      __stcs(out_xyz + 0 * cap + j, o.p0x);
      __stcs(out_xyz + 1 * cap + j, o.p0y);
      __stcs(out_xyz + 2 * cap + j, (!deg && o.count >= 1) ? z0 : nan);
      __stcs(out_xyz + 3 * cap + j, o.p1x);
      __stcs(out_xyz + 4 * cap + j, o.p1y);
      __stcs(out_xyz + 5 * cap + j, (!deg && o.count == 2) ? z0 : nan);
    }
    base += total;
    cur = nxt;
    __syncthreads();                                 // smem of this tile is free
  }
}

}  // namespace

extern "C" {

size_t sgi_zonal_workspace_bytes(int64_t n_edges) {
  if (n_edges < 0) return 0;
  return (size_t)kMaxCtas * sizeof(unsigned long long);
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
  const int64_t tiles = (n_edges + kTile - 1) / kTile;
  unsigned long long* cta = (unsigned long long*)d_work;
  const size_t emit_smem = kEmitSmem + lat_smem;
  auto grid_for = [&](auto kernel, size_t smem) {
    int occ = 1;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kEmitSmem + kLatSmem * sizeof(double)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kTile, smem);
    int64_t g = (int64_t)sms * (occ < 1 ? 1 : occ);
    if (g > tiles) g = tiles;
    if (g > kMaxCtas) g = kMaxCtas;
    return (int)g;
  };
  // both passes use the same grid so each CTA walks the same edge range
  int grid = 0;
  switch (mode) {
    case SGI_MODE_NAIVE: grid = grid_for(sgi_zonal_emit_kernel<sgi::MODE_NAIVE>, emit_smem); break;
    case SGI_MODE_EFT: grid = grid_for(sgi_zonal_emit_kernel<sgi::MODE_EFT>, emit_smem); break;
    case SGI_MODE_EFT_LITERAL: grid = grid_for(sgi_zonal_emit_kernel<sgi::MODE_EFT_LITERAL>, emit_smem); break;
    case SGI_MODE_YAC: grid = grid_for(sgi_zonal_emit_kernel<sgi::MODE_YAC>, emit_smem); break;
    case SGI_MODE_BASE: grid = grid_for(sgi_zonal_emit_kernel<sgi::MODE_BASE>, emit_smem); break;
    default: grid = grid_for(sgi_zonal_emit_kernel<sgi::MODE_NAIVE_KAHAN>, emit_smem); break;
  }
  grid_for(sgi_zonal_count_kernel, lat_smem);
  sgi_zonal_count_kernel<<<grid, kTile, lat_smem, st>>>(va, vb, n_edges, ld_e, lat_z0, n_lat, cta);
  sgi_zonal_scan_kernel<<<1, 1024, 0, st>>>(cta, grid, d_total);
  if (cap > 0) {
    auto emit = [&](auto kernel) {
      kernel<<<grid, kTile, emit_smem, st>>>(va, vb, n_edges, ld_e, lat_z0, n_lat, cap, out_edge,
                                             out_lat, out_count, out_xyz, cta);
    };
    switch (mode) {
      case SGI_MODE_NAIVE: emit(sgi_zonal_emit_kernel<sgi::MODE_NAIVE>); break;
      case SGI_MODE_EFT: emit(sgi_zonal_emit_kernel<sgi::MODE_EFT>); break;
      case SGI_MODE_EFT_LITERAL: emit(sgi_zonal_emit_kernel<sgi::MODE_EFT_LITERAL>); break;
      case SGI_MODE_YAC: emit(sgi_zonal_emit_kernel<sgi::MODE_YAC>); break;
      case SGI_MODE_BASE: emit(sgi_zonal_emit_kernel<sgi::MODE_BASE>); break;
      default: emit(sgi_zonal_emit_kernel<sgi::MODE_NAIVE_KAHAN>); break;
    }
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    sgi_internal::set_error_msg("sgi_zonal kernels launch", e);
    return SGI_E_CUDA;
  }
  return SGI_OK;
}

}  // extern "C"
