/* sgi.h — C ABI of libsgi.so: batched great-circle-arc / constant-latitude intersections on
 * NVIDIA B200 (sm_100a), after Chen, Ullrich & Panetta, "Fast and Accurate Intersections on a
 * Sphere" (arXiv 2510.09892; /root/reference/PAPER.md, cited as P:<line>).
 *
 * The operation (problem definition): for each query i, the great circle through
 * the arc endpoints a_i, b_i (normal n = a_i x b_i) meets the plane z = z0_i in
 * 0, 1 or 2 points, given by the closed form Eq.FINAL
 *     P(+-) = ( -(z0 nx nz +- s ny) / |n_xy|^2 , -(z0 ny nz -+ s nx) / |n_xy|^2 , z0 ),
 *     s = sqrt(|n_xy|^2 - |n|^2 z0^2).
 * Points are kept only if they lie on the closed minor arc from a_i to b_i.
 * Endpoints need not be unit length: the formula is invariant to |a| and |b|.
 *
 * Modes:
 *   SGI_MODE_EFT          AccuX (Alg.8) with error-free transformations, both roots,
 *                         each AccuDOP normal pair renormalised (reading R6).
 *                         Error bound 3 sqrt(1 - z0^2) u, u = 2^-53 (Eq.BOUND).
 *   SGI_MODE_EFT_LITERAL  AccuX exactly as listed (no renormalisation).
 *   SGI_MODE_NAIVE        Eq.FINAL in plain binary64 (§4).
 *   SGI_MODE_YAC          Eq.YAC in plain binary64: normalised normal n/|n|.
 *   SGI_MODE_BASE         Eq.BASE in plain binary64: divisor 1 - n^z^2.
 *   SGI_MODE_NAIVE_KAHAN  Eq.FINAL in binary64 with Kahan's DiffOfProd normal (Alg.3).
 * (the last three are the paper's comparison formulas)
 * Results are bit-identical to the CPU oracle's op sequence (oracle/eft_oracle.c) up to the sign
 * of zero, independent of grid shape, stream or sharding.
 *
 * Layout (all arrays caller-owned; SoA planes with leading dimension ld >= n):
 *   a[c*ld + i], b[c*ld + i]   endpoint coordinates, c = 0,1,2 = x,y,z        (float64)
 *   z0[i]                      latitude plane height                         (float64)
 *   out_xyz[(k*3 + c)*ld + i]  slot k = 0,1 of query i, coordinates c        (float64)
 *   out_count[i]               0, 1, 2, or SGI_DEGENERATE                    (uint8)
 * Slots hold the in-arc points in arc order (the first met travelling from a to b); unused
 * slots are the canonical quiet NaN 0x7FF8000000000000.  out_xyz z-coordinates are bit copies
 * of z0.  SGI_DEGENERATE (0xFF): n = 0 exactly (equal, antipodal or zero endpoints), or
 * n_xy = 0 with z0 = 0 (arc on the equator, which is the latitude).  n_xy = 0 with z0 != 0
 * gives count 0 (z0 compared with 0 exactly, subnormals included).  Contract: finite inputs
 * whose endpoint components and z0 are 0 or of magnitude in [2^-120, 2^120]; then every nonzero
 * term of the EFT chain lies in [2^-940, 2^800] (an exact cross-product component is a
 * multiple of 2^-345; |n|^2 z0^2 >= 2^-930 is the smallest product) and every error term stays
 * normal, so none underflows or overflows (the analysis ignores the exponent range,
 * P:461) and the device's certified shortcuts are exact (A13).  Outside it the
 * outputs are still computed, and NaN inputs give count 0.  No per-element condition fails a
 * call.
 *
 * Count correctness (readings R7, R7'): containment is decided by the paper-free
 * identity P.(n x x_k) = (|n|^2/S)(z0 g_k -+ s z_k) evaluated as rounded products compared
 * exactly (the paper only says the check is needed).  out_count equals the exact
 * count of the closed arc except when an endpoint lies on the latitude to within rounding: a
 * deciding comparison A >= B with |A - B| < 4u(|A| + |B|), u = 2^-53 (e.g. z0 equal to an
 * endpoint's height, as in the near-polar third of config 3: 25 of 20,000 sampled queries there,
 * none in configs 1, 2, 4, 5); there the count may differ from the exact one by that endpoint's
 * point, counted or not as the rounding falls.  A tangent point (s^2 = 0) counts once.
 *
 * Errors: SGI_E_INVALID (nothing is launched) for a null pointer with n > 0, n < 0, ld < n,
 * an unknown mode, or output arrays overlapping input arrays.  SGI_E_CUDA when a launch or
 * copy fails; sgi_last_error() then returns the CUDA message (thread-local).  n == 0 returns
 * SGI_OK without launching.
 */
#ifndef SGI_H
#define SGI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGI_ABI_VERSION 1
#define SGI_DEGENERATE ((uint8_t)0xFF)

typedef enum {
  SGI_MODE_NAIVE = 0,
  SGI_MODE_EFT = 1,
  SGI_MODE_EFT_LITERAL = 2,
  SGI_MODE_YAC = 3,
  SGI_MODE_BASE = 4,
  SGI_MODE_NAIVE_KAHAN = 5
} sgi_mode;
typedef enum { SGI_OK = 0, SGI_E_INVALID = 1, SGI_E_CUDA = 2 } sgi_status;

/* Device entry point.  a, b, z0, out_xyz, out_count are CUDA device pointers.  Enqueues one
 * kernel on `stream` (a cudaStream_t; NULL = legacy default stream) and returns without
 * synchronising; performs no allocation and keeps no state, so it is thread-safe. */
sgi_status sgi_intersect_arc_lat(const double* a, const double* b, const double* z0,
                                 int64_t n, int64_t ld, double* out_xyz, uint8_t* out_count,
                                 int mode, void* stream);

/* Host-buffer entry point (the end-to-end path).  a, b, z0, out_xyz, out_count are HOST
 * pointers in the layout above (page-locked memory lets the copies overlap; pageable works).
 * d_work is a caller-owned device buffer of work_bytes >= sgi_host_workspace_bytes(chunk)
 * bytes for some chunk >= 1; the batch is streamed through it in chunks, copies and kernels
 * pipelined over `stream` and two internal streams (three buffers).  Blocks until the results
 * are on the host. */
sgi_status sgi_intersect_arc_lat_host(const double* a, const double* b, const double* z0,
                                      int64_t n, int64_t ld, double* out_xyz,
                                      uint8_t* out_count, int mode, void* d_work,
                                      size_t work_bytes, void* stream);

/* Device bytes sgi_intersect_arc_lat_host needs for a given chunk length (three buffers). */
size_t sgi_host_workspace_bytes(int64_t chunk);

/* Histogram of out_count (device pointers): d_hist5[0..2] += number of queries with 0/1/2
 * points, d_hist5[3] += number of SGI_DEGENERATE, d_hist5[4] += total points.  Accumulates
 * into d_hist5 (the caller zeroes it); asynchronous on `stream`. */
sgi_status sgi_count_histogram(const uint8_t* out_count, int64_t n,
                               unsigned long long* d_hist5, void* stream);

/* Fused zonal-mean pass (zonal means on regridding meshes): every mesh
 * edge (va_e, vb_e) against a latitude table, compacted.  Edges are SoA planes va[c*ld_e + e],
 * vb[c*ld_e + e] (device); lat_z0[n_lat] is strictly increasing (device).  For each edge, the
 * candidate latitudes are those within delta = 2^-40 of the arc's z-range (endpoint heights
 * z/|x| and, when the great circle's extremum lies inside the arc, the apex height
 * sqrt(|n_xy|^2/|n|^2), from a normal accurate to 2 ulps per component); an edge with n = 0
 * (degenerate at every latitude) or nearly parallel endpoints ((|nx|+|ny|+|nz|)^2 <=
 * 2^-80 |a|^2 |b|^2, where the query's rounded containment may accept points far from the arc)
 * has every latitude as a candidate.  Every (edge, latitude) whose query has a nonzero count is
 * a candidate; candidates within delta of the range (and those of such edges) may have count 0.
 * Candidate pair j (edge-major, latitude ascending; deterministic) is written to out_edge[j],
 * out_lat[j], out_count[j] and out_xyz[(slot*3 + c)*cap + j], bit-identical to
 * sgi_intersect_arc_lat on (va_e, vb_e, lat_z0[k]) in `mode`.  Pairs j >= cap are not written;
 * *d_total (device) receives the number of candidate pairs, so cap = 0 is a count-only call.
 * d_work: caller-owned device workspace of sgi_zonal_workspace_bytes(n_edges) bytes (8 B per
 * edge for its candidate range plus 8 B per 512-edge tile, plus 8 B), 16-byte aligned
 * (SGI_E_INVALID otherwise; cudaMalloc and PyTorch allocations are).  n_lat <= 2^23.
 * Asynchronous on `stream`: with cap > 0 and n_lat <= 4096 one single-pass launch (tiles of
 * 1,024 edges staged by bulk copies, a decoupled look-back over per-tile counts kept in d_work,
 * which is zeroed by a memset on `stream` first); otherwise (a count-only call, or a larger
 * table) three launches: filter, scan, emit.  Both give the same pairs in the same order.
 * Errors as for sgi_intersect_arc_lat. */
sgi_status sgi_zonal_intersect(const double* va, const double* vb, int64_t n_edges,
                               int64_t ld_e, const double* lat_z0, int32_t n_lat, int64_t cap,
                               int64_t* out_edge, int32_t* out_lat, uint8_t* out_count,
                               double* out_xyz, unsigned long long* d_total, void* d_work,
                               size_t work_bytes, int mode, void* stream);
size_t sgi_zonal_workspace_bytes(int64_t n_edges);

/* Double-word points (reading R11 — an extension: the paper rounds each
 * coordinate once).  As sgi_intersect_arc_lat in an EFT mode (out_xyz and out_count
 * are bit-identical to it), plus out_lo[(slot*2 + c)*ld + i], c = 0,1 = x,y: a low part with
 * P ~ out_xyz + out_lo, from the root's numerator before CompDot's final rounding (the CompDotC
 * pair, Alg.1) and |n_xy|^2 as a pair (Alg.7):  lo = -((fma(hi, S2, X) + ((p - X) +
 * sigma)) + hi s2) / S2.  z needs no low part (P_z = z0 exactly).  Unused slots: canonical NaN.
 * mode must be SGI_MODE_EFT or SGI_MODE_EFT_LITERAL (else SGI_E_INVALID); other errors as for
 * sgi_intersect_arc_lat.  Device pointers, one launch on `stream` (TMA-staged when the batch is
 * large and 16-B aligned, as for sgi_intersect_arc_lat). */
sgi_status sgi_intersect_arc_lat_dw(const double* a, const double* b, const double* z0, int64_t n,
                                    int64_t ld, double* out_xyz, double* out_lo,
                                    uint8_t* out_count, int mode, void* stream);

/* Output statistics (the per-rank quantities the multi-GPU run reduces with NCCL).
 * Over the stored points of out_xyz/out_count (device; layout as above, n queries, leading
 * dimension ld): d_stats2[0] = max |(|P~|) - 1| / u (Eq.FINAL's points lie on the unit sphere,
 * P:307-308; |P~|^2 evaluated in double-word arithmetic), d_counts2[0] += number of points whose
 * z is not a bit copy of z0.  If ref_xyz/ref_count (another result for the same queries, e.g.
 * SGI_MODE_NAIVE) are given: d_counts2[1] += queries whose counts differ, d_stats2[1] = max over
 * the others' points of |P~ - P~ref| / u (the paper's distance).  Both buffers are
 * device memory the caller zeroes; maxima accumulate (atomic max), counts add.  Asynchronous on
 * `stream`.  Errors: SGI_E_INVALID for n < 0, ld < n, a null pointer with n > 0, or only one of
 * ref_xyz / ref_count. */
sgi_status sgi_output_stats(const double* out_xyz, const uint8_t* out_count, const double* z0,
                            int64_t n, int64_t ld, const double* ref_xyz,
                            const uint8_t* ref_count, double* d_stats2,
                            unsigned long long* d_counts2, void* stream);

/* Appendix-A instrumentation (Appendix A: "we recorded these results as
 * pairs of doubles (the leading term and compensation term)").  For each query i, every
 * intermediate of the mode's op sequence — computed with the IEEE intrinsics, i.e. the values
 * sgi_intersect_arc_lat reproduces — is written to out_trace[f * ld + i] for the
 * SGI_TRACE_FIELDS fields f below, and the count to out_count[i].  In the EFT modes each
 * (hi, lo) pair is the pair AccuX holds: the normal after AccuDOP (and the
 * renormalisation of SGI_MODE_EFT), |n_xy|^2 and |n|^2 (SumOfSquaresC), z0^2 (TwoProd),
 * |n|^2 z0^2 (CompDotC), s^2, s (AccSqrt), n_x n_z and n_y n_z, the four numerators after
 * CompDot's final rounding and as CompDotC pairs before it, and both points.  The plain
 * binary64 modes fill their own values (lo = 0; unused fields 0; Eq.YAC/BASE numerators use
 * the normalised normal).  Points are both roots of the great circle, before containment.
 * Device pointers, one launch on `stream`; a debug path, not tuned.  Errors as for
 * sgi_intersect_arc_lat (out_trace must not overlap the inputs). */
#define SGI_TRACE_FIELDS 38
enum {
  SGI_TRACE_NX, SGI_TRACE_EX, SGI_TRACE_NY, SGI_TRACE_EY, SGI_TRACE_NZ, SGI_TRACE_EZ,
  SGI_TRACE_S2, SGI_TRACE_S2_LO, SGI_TRACE_S3, SGI_TRACE_S3_LO, SGI_TRACE_C, SGI_TRACE_C_LO,
  SGI_TRACE_D, SGI_TRACE_D_LO, SGI_TRACE_SIGMA, SGI_TRACE_SIGMA_LO, SGI_TRACE_S, SGI_TRACE_S_LO,
  SGI_TRACE_FX, SGI_TRACE_FX_LO, SGI_TRACE_FY, SGI_TRACE_FY_LO,
  SGI_TRACE_XP, SGI_TRACE_YP, SGI_TRACE_XM, SGI_TRACE_YM,
  SGI_TRACE_PPX, SGI_TRACE_PPY, SGI_TRACE_PMX, SGI_TRACE_PMY,
  SGI_TRACE_XP_PAIR, SGI_TRACE_XP_PAIR_LO, SGI_TRACE_YP_PAIR, SGI_TRACE_YP_PAIR_LO,
  SGI_TRACE_XM_PAIR, SGI_TRACE_XM_PAIR_LO, SGI_TRACE_YM_PAIR, SGI_TRACE_YM_PAIR_LO
};
sgi_status sgi_intersect_trace(const double* a, const double* b, const double* z0, int64_t n,
                               int64_t ld, double* out_trace, uint8_t* out_count, int mode,
                               void* stream);
int sgi_trace_fields(void);                                    /* SGI_TRACE_FIELDS */

const char* sgi_status_str(sgi_status s);
const char* sgi_last_error(void);
int sgi_abi_version(void);

/* Which kernel a call with these arguments launches (introspection for tests and profiling;
 * no launch, no device access).  entry 0 = sgi_intersect_arc_lat, 1 = sgi_intersect_arc_lat_dw.
 * SGI_PATH_LDG: the grid-stride kernel (batches below 2^19 queries, an odd ld, or inputs not
 * 16-B aligned); SGI_PATH_TMA: the TMA-staged kernel, one query per thread; SGI_PATH_TMA_PAIR:
 * the TMA-staged kernel with two adjacent queries per thread (EFT modes, entry 0, outputs
 * 16-B aligned and out_count 2-B aligned).  SGI_PATH_NONE for n == 0 or arguments the entry
 * would reject.  Every path gives the same outputs bit for bit (up to the sign of zero). */
enum { SGI_PATH_NONE = 0, SGI_PATH_LDG = 1, SGI_PATH_TMA = 2, SGI_PATH_TMA_PAIR = 3 };
int sgi_dispatch_path(const double* a, const double* b, const double* z0, int64_t n, int64_t ld,
                      const double* out_xyz, const uint8_t* out_count, int mode, int entry);

#ifdef __cplusplus
}
#endif

#endif /* SGI_H */
