/* oracle/eft_oracle.c — ORACLE (a): plain, sequential CPU evaluation of the paper's EFT method.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code with the CUDA path
 * (paper_2510_09892_b200/csrc) and includes nothing from it.
 *
 * Source of truth: /root/reference/PAPER.md ("Fast and Accurate Intersections on a Sphere").
 * Each function cites the PAPER.md line range (P:nnn) and algorithm it restates.  The op order is
 * exactly the listing's; every fl(.) is one IEEE binary64 round-to-nearest-even operation
 * (P:464-482), FMA is C99 fma() (one rounding), and the file is compiled with
 * -O2 -ffp-contract=off -fno-fast-math so the compiler adds no contraction.
 *
 * Readings where the paper is silent or garbled (DESIGN.md §2 lists them all):
 *   R1  AccuDOP residual is r1 - r2, not the printed r1 + r2 (Alg.4 line 5).
 *   R2  AccuX's AccuDOP calls use the a*b - c*d argument convention; the cross product is
 *       n = x1 x x2.
 *   R3  AccSqrt (not printed; P:757 cites Rump2023): s = RN(sqrt(H)), r = fma(-s,s,H),
 *       lo = RN(RN(r + h) / RN(s + s)); H <= 0 gives (0, 0).
 *   R4  Garbled P:754 / P:765 read as e = fl(fl(s2 - eD) + eE) and eFy3 = fl(nz * e_ny).
 *   R5  Second root = the first with the s-terms negated, same leading minus.
 *   R6  Mode SGI_MODE_EFT renormalises each AccuDOP pair with TwoSum before use (SumOfSquaresC
 *       and the F products drop e*e terms and assume |e| <~ u|x|); SGI_MODE_EFT_LITERAL
 *       is the listing verbatim.
 *   R7  Containment (P:448-449 only says it must be checked) uses the exact identity
 *       P.(n x x_k) = (|n|^2/S)(z0 g_k -+ s z_k), g_k = nx y_k - ny x_k, evaluated as rounded
 *       products compared exactly; inclusive boundary.  Slots in arc order: with two points,
 *       P+ (ascending crossing) comes first iff g1 >= 0.
 *   R8  Naive mode ("pure floating-point implementation"; analysed in S1): plain cross
 *       product, no FMA, left-to-right products, 4 divisions.
 *   R9  Comparison formulas Eq.YAC / Eq.BASE / Kahan-normal naive: the same plain, left-to-right
 *       translation, normalising n with one sqrt and three divisions.
 *   parity unpinned: SGI_MODE_EFT_LITERAL on near-coincident endpoints (separation < 1e-7 rad)
 *   is outside the paper's nondegeneracy assumption; only bit-equality with the
 *   CUDA path is checked there, not the error bound.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct { double hi, lo; } pair;

/* TwoSum (Knuth).  s = fl(a+b), s + e = a + b exactly. */
static pair two_sum(double a, double b) {
  double s = a + b;
  double v = s - a;
  double e = (a - (s - v)) + (b - v);
  pair r = {s, e};
  return r;
}

/* FastTwoSum (Dekker).  Requires |a| >= |b| or a = 0. */
static pair fast_two_sum(double a, double b) {
  double s = a + b;
  double z = s - a;
  double e = b - z;
  pair r = {s, e};
  return r;
}

/* TwoProd via FMA.  p = fl(a*b), e = fma(a, b, -p), p + e = a*b exactly. */
static pair two_prod(double a, double b) {
  double p = a * b;
  double e = fma(a, b, -p);
  pair r = {p, e};
  return r;
}

/* Alg.1 CompDotC. */
static pair comp_dot_c(const double* x, const double* y, int n) {
  pair ps = two_prod(x[0], y[0]);
  double p = ps.hi, s = ps.lo;
  for (int i = 1; i < n; ++i) {
    pair hr = two_prod(x[i], y[i]);
    pair pq = two_sum(p, hr.hi);
    p = pq.hi;
    s = s + (pq.lo + hr.lo);
  }
  pair r = {p, s};
  return r;
}

/* Alg.2 CompDot: fl(p + s) of CompDotC. */
static double comp_dot(const double* x, const double* y, int n) {
  pair ps = comp_dot_c(x, y, n);
  return ps.hi + ps.lo;
}

/* Alg.3 Kahan DiffOfProd: a*d - b*c. */
static double kahan_dop(double a, double b, double c, double d) {
  double bc = b * c;
  double err = fma(-b, c, bc);
  double dop = fma(a, d, -bc);
  return dop + err;
}

/* Alg.4 AccuDOP: a*d - b*c as an unevaluated pair.  Reading R1: err = s + (r1 - r2). */
static pair accu_dop(double a, double b, double c, double d) {
  pair p1 = two_prod(a, d);
  pair p2 = two_prod(b, c);
  pair ds = two_sum(p1.hi, -p2.hi);
  double err = ds.lo + (p1.lo - p2.lo);
  pair r = {ds.hi, err};
  return r;
}

/* Alg.6 SumNonNeg. */
static pair sum_non_neg(pair A, pair B) {
  pair Hh = two_sum(A.hi, B.hi);
  double c = A.lo + B.lo;
  double d = Hh.lo + c;
  return fast_two_sum(Hh.hi, d);
}

/* Alg.5 SumOfSquares, starting from (0, 0) as printed. */
static pair sum_of_squares(const double* x, int n) {
  pair S = {0.0, 0.0};
  for (int j = 0; j < n; ++j) S = sum_non_neg(S, two_prod(x[j], x[j]));
  return S;
}

/* Alg.7 SumOfSquaresC. */
static pair sum_of_squares_c(const double* x, const double* e, int n) {
  pair Ss = sum_of_squares(x, n);
  double Rstar = comp_dot(x, e, n);
  double R = fma(2.0, Rstar, Ss.lo);
  return fast_two_sum(Ss.hi, R);
}

/* AccSqrt (bound P:826; algorithm not printed — reading R3). */
static pair acc_sqrt(double H, double h) {
  if (!(H > 0.0)) { pair z = {0.0, 0.0}; return z; }
  double s = sqrt(H);
  double r = fma(-s, s, H);
  double t = r + h;
  pair out = {s, t / (s + s)};
  return out;
}

/* ------------------------------------------------------------------------------------------- */
/* Modes, identical numbering to include/sgi.h (declared independently here). */
enum { OR_MODE_NAIVE = 0, OR_MODE_EFT = 1, OR_MODE_EFT_LITERAL = 2, OR_MODE_YAC = 3,
       OR_MODE_BASE = 4, OR_MODE_NAIVE_KAHAN = 5 };
#define OR_DEGENERATE 0xFF

/* Trace of every AccuX intermediate, for the Appendix-A style pins. */
typedef struct {
  double nx, ex, ny, ey, nz, ez;      /* normal pairs (after renormalisation in EFT mode) */
  double S2, s2, S3, s3;              /* |n_xy|^2, |n|^2 */
  double C, eC, D, eD;                /* z0^2, |n|^2 z0^2 */
  double sh, sl;                      /* s^2 */
  double s, es;                       /* s */
  double Fx, eFx, Fy, eFy;            /* n_x n_z, n_y n_z */
  double Xp, Yp, Xm, Ym;              /* numerators of both roots */
  double Pp[2], Pm[2];                /* both points' x, y */
  double Xpp[2], Ypp[2], Xmp[2], Ymp[2]; /* the numerators before CompDot's final rounding: the
                                          CompDotC pairs (p, sigma) of lines 17/22 (Appendix A
                                          analyses z0 nx nz + s ny as a pair);
                                          (value, 0) in the plain-binary64 modes */
} accux_trace;

/* Alg.8 AccuX, both roots (reading R5). */
static void accux(const double x1[3], const double x2[3], double z0, int renorm, accux_trace* t) {
  /* lines 2-4: n = x1 x x2 with AccuDOP (readings R1, R2) */
  pair nx = accu_dop(x1[1], x1[2], x2[1], x2[2]);   /* y1*z2 - z1*y2 */
  pair ny = accu_dop(x1[2], x1[0], x2[2], x2[0]);   /* z1*x2 - x1*z2 */
  pair nz = accu_dop(x1[0], x1[1], x2[0], x2[1]);   /* x1*y2 - y1*x2 */
  if (renorm) { nx = two_sum(nx.hi, nx.lo); ny = two_sum(ny.hi, ny.lo); nz = two_sum(nz.hi, nz.lo); }
  /* lines 5-6 */
  double v2[2] = {nx.hi, ny.hi}, e2[2] = {nx.lo, ny.lo};
  double v3[3] = {nx.hi, ny.hi, nz.hi}, e3[3] = {nx.lo, ny.lo, nz.lo};
  pair S2 = sum_of_squares_c(v2, e2, 2);
  pair S3 = sum_of_squares_c(v3, e3, 3);
  /* lines 7-8 */
  pair C = two_prod(z0, z0);
  double dx[4] = {S3.hi, S3.hi, S3.lo, S3.lo}, dy[4] = {C.hi, C.lo, C.hi, C.lo};
  pair D = comp_dot_c(dx, dy, 4);
  /* lines 9-11 (reading R4) */
  pair E = two_sum(S2.hi, -D.hi);
  double e = (S2.lo - D.lo) + E.lo;
  pair sq = fast_two_sum(E.hi, e);
  /* line 12 */
  pair s = acc_sqrt(sq.hi, sq.lo);
  /* lines 13-16 */
  pair Fx1 = two_prod(nx.hi, nz.hi);
  double eFx2 = nx.hi * nz.lo;
  double eFx3 = nz.hi * nx.lo;
  double eFx = (Fx1.lo + eFx2) + eFx3;
  /* lines 18-21 */
  pair Fy1 = two_prod(ny.hi, nz.hi);
  double eFy2 = ny.hi * nz.lo;
  double eFy3 = nz.hi * ny.lo;
  double eFy = (Fy1.lo + eFy2) + eFy3;
  /* lines 17 and 22, both roots */
  double w[6] = {z0, z0, s.hi, s.hi, s.lo, s.lo};
  double xp[6] = {Fx1.hi, eFx, ny.hi, ny.lo, ny.hi, ny.lo};
  double yp[6] = {Fy1.hi, eFy, -nx.hi, -nx.lo, -nx.hi, -nx.lo};
  double xm[6] = {Fx1.hi, eFx, -ny.hi, -ny.lo, -ny.hi, -ny.lo};
  double ym[6] = {Fy1.hi, eFy, nx.hi, nx.lo, nx.hi, nx.lo};
  double Xp = comp_dot(xp, w, 6), Yp = comp_dot(yp, w, 6);
  double Xm = comp_dot(xm, w, 6), Ym = comp_dot(ym, w, 6);
  pair Xpp = comp_dot_c(xp, w, 6), Ypp = comp_dot_c(yp, w, 6);
  pair Xmp = comp_dot_c(xm, w, 6), Ymp = comp_dot_c(ym, w, 6);
  t->Xpp[0] = Xpp.hi; t->Xpp[1] = Xpp.lo; t->Ypp[0] = Ypp.hi; t->Ypp[1] = Ypp.lo;
  t->Xmp[0] = Xmp.hi; t->Xmp[1] = Xmp.lo; t->Ymp[0] = Ymp.hi; t->Ymp[1] = Ymp.lo;
  /* lines 23-25 */
  t->Pp[0] = -(Xp / S2.hi); t->Pp[1] = -(Yp / S2.hi);
  t->Pm[0] = -(Xm / S2.hi); t->Pm[1] = -(Ym / S2.hi);
  t->nx = nx.hi; t->ex = nx.lo; t->ny = ny.hi; t->ey = ny.lo; t->nz = nz.hi; t->ez = nz.lo;
  t->S2 = S2.hi; t->s2 = S2.lo; t->S3 = S3.hi; t->s3 = S3.lo;
  t->C = C.hi; t->eC = C.lo; t->D = D.hi; t->eD = D.lo;
  t->sh = sq.hi; t->sl = sq.lo; t->s = s.hi; t->es = s.lo;
  t->Fx = Fx1.hi; t->eFx = eFx; t->Fy = Fy1.hi; t->eFy = eFy;
  t->Xp = Xp; t->Yp = Yp; t->Xm = Xm; t->Ym = Ym;
}

/* Naive Eq.FINAL in plain binary64 (reading R8). */
static void naive(const double x1[3], const double x2[3], double z0, accux_trace* t) {
  double nx = (x1[1] * x2[2]) - (x1[2] * x2[1]);
  double ny = (x1[2] * x2[0]) - (x1[0] * x2[2]);
  double nz = (x1[0] * x2[1]) - (x1[1] * x2[0]);
  double S2 = (nx * nx) + (ny * ny);
  double S3 = S2 + (nz * nz);
  double sh = S2 - (S3 * (z0 * z0));
  double s = sh > 0.0 ? sqrt(sh) : 0.0;
  double Xp = ((z0 * nx) * nz) + (s * ny), Xm = ((z0 * nx) * nz) - (s * ny);
  double Yp = ((z0 * ny) * nz) - (s * nx), Ym = ((z0 * ny) * nz) + (s * nx);
  memset(t, 0, sizeof(*t));
  t->nx = nx; t->ny = ny; t->nz = nz; t->S2 = S2; t->S3 = S3; t->sh = sh; t->s = s;
  t->Xp = Xp; t->Yp = Yp; t->Xm = Xm; t->Ym = Ym;
  t->Xpp[0] = Xp; t->Ypp[0] = Yp; t->Xmp[0] = Xm; t->Ymp[0] = Ym;
  t->Pp[0] = -(Xp / S2); t->Pp[1] = -(Yp / S2);
  t->Pm[0] = -(Xm / S2); t->Pm[1] = -(Ym / S2);
}

/* The paper's comparison formulas in plain binary64 (reading R9):
 *   YAC  Eq.YAC: hat n = n/|n|, s^ = sqrt(hx^2 + hy^2 - z0^2), divisor hx^2 + hy^2;
 *   BASE Eq.BASE: divisor 1 - hz^2, s* = sqrt(1 - hz^2 - z0^2);
 *   NAIVE_KAHAN  Eq.FINAL with each normal component by Kahan's DiffOfProd (Alg.3).
 * hx, hy, hz return the normal the containment test uses (hat n; n itself for NAIVE_KAHAN). */
static void variant(int mode, const double x1[3], const double x2[3], double z0, accux_trace* t,
                    double* hx, double* hy, double* hz) {
  double nx, ny, nz;
  if (mode == OR_MODE_NAIVE_KAHAN) {
    nx = kahan_dop(x1[1], x1[2], x2[1], x2[2]);   /* y1*z2 - z1*y2 */
    ny = kahan_dop(x1[2], x1[0], x2[2], x2[0]);   /* z1*x2 - x1*z2 */
    nz = kahan_dop(x1[0], x1[1], x2[0], x2[1]);   /* x1*y2 - y1*x2 */
  } else {
    nx = (x1[1] * x2[2]) - (x1[2] * x2[1]);
    ny = (x1[2] * x2[0]) - (x1[0] * x2[2]);
    nz = (x1[0] * x2[1]) - (x1[1] * x2[0]);
  }
  double S2 = (nx * nx) + (ny * ny);
  double S3 = S2 + (nz * nz);
  memset(t, 0, sizeof(*t));
  t->nx = nx; t->ny = ny; t->nz = nz; t->S2 = S2; t->S3 = S3;
  double ux = nx, uy = ny, uz = nz, den = S2, sh;
  if (mode != OR_MODE_NAIVE_KAHAN) {
    double N = sqrt(S3 > 0.0 ? S3 : 1.0);
    ux = nx / N; uy = ny / N; uz = nz / N;
    den = mode == OR_MODE_YAC ? (ux * ux) + (uy * uy) : 1.0 - (uz * uz);
    sh = den - (z0 * z0);
  } else {
    sh = S2 - (S3 * (z0 * z0));
  }
  double s = sh > 0.0 ? sqrt(sh) : 0.0;
  double bx = (z0 * ux) * uz, by = (z0 * uy) * uz;
  double Xp = bx + (s * uy), Xm = bx - (s * uy);
  double Yp = by - (s * ux), Ym = by + (s * ux);
  t->sh = sh; t->s = s; t->Xp = Xp; t->Yp = Yp; t->Xm = Xm; t->Ym = Ym;
  t->Xpp[0] = Xp; t->Ypp[0] = Yp; t->Xmp[0] = Xm; t->Ymp[0] = Ym;
  t->Pp[0] = -(Xp / den); t->Pp[1] = -(Yp / den);
  t->Pm[0] = -(Xm / den); t->Pm[1] = -(Ym / den);
  *hx = nx == 0.0 ? 0.0 : ux;
  *hy = ny == 0.0 ? 0.0 : uy;
  *hz = nz == 0.0 ? 0.0 : uz;
}

static double canonical_nan(void) {
  union { uint64_t u; double d; } c;
  c.u = 0x7FF8000000000000ull;
  return c.d;
}

/* One query: count in {0,1,2,0xFF} and the two slots (x,y) in arc order (reading R7). */
static uint8_t intersect_one(int mode, const double x1[3], const double x2[3], double z0,
                             double slot[2][2], accux_trace* tr, int* plus_first) {
  accux_trace t;
  double hx, hy, hz;
  if (mode == OR_MODE_NAIVE) {
    naive(x1, x2, z0, &t);
    hx = t.nx; hy = t.ny; hz = t.nz;
  } else if (mode >= OR_MODE_YAC) {
    variant(mode, x1, x2, z0, &t, &hx, &hy, &hz);
  } else {
    accux(x1, x2, z0, mode == OR_MODE_EFT, &t);
    if (mode == OR_MODE_EFT) { hx = t.nx; hy = t.ny; hz = t.nz; }
    else { hx = t.nx + t.ex; hy = t.ny + t.ey; hz = t.nz + t.ez; }
  }
  if (tr) *tr = t;
  double nan = canonical_nan();
  slot[0][0] = slot[0][1] = slot[1][0] = slot[1][1] = nan;
  uint8_t count;
  if (hx == 0.0 && hy == 0.0 && hz == 0.0) return OR_DEGENERATE;
  if (hx == 0.0 && hy == 0.0) return z0 == 0.0 ? OR_DEGENERATE : 0;
  if (t.sh < 0.0) return 0;
  double g1 = (hx * x1[1]) - (hy * x1[0]);
  double g2 = (hx * x2[1]) - (hy * x2[0]);
  double A1 = z0 * g1, B1 = t.s * x1[2];
  double A2 = z0 * g2, B2 = t.s * x2[2];
  int inp = (A1 >= B1) && (A2 <= B2);
  int inm = (t.sh > 0.0) && (A1 >= -B1) && (A2 <= -B2);
  count = (uint8_t)(inp + inm);
  if (plus_first) *plus_first = count == 2 ? g1 >= 0.0 : inp;
  if (count == 2) {
    const double* first = g1 >= 0.0 ? t.Pp : t.Pm;
    const double* second = g1 >= 0.0 ? t.Pm : t.Pp;
    slot[0][0] = first[0]; slot[0][1] = first[1];
    slot[1][0] = second[0]; slot[1][1] = second[1];
  } else if (count == 1) {
    const double* p = inp ? t.Pp : t.Pm;
    slot[0][0] = p[0]; slot[0][1] = p[1];
  }
  return count;
}

/* ------------------------------------------------------------------------ exported (ctypes) */
#ifdef _OPENMP
#include <omp.h>
#endif

/* Batch over SoA planes, same layout as the C-ABI: a[c*ld+i], b[c*ld+i], z0[i];
 * out_xyz[(slot*3 + c)*ld + i], out_count[i].  nthreads <= 0 means 1 (sequential). */
int oracle_intersect_batch(int mode, const double* a, const double* b, const double* z0,
                           int64_t n, int64_t ld, double* out_xyz, uint8_t* out_count,
                           int nthreads) {
  if (mode < 0 || mode > 5 || n < 0 || ld < n) return 1;
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t i = 0; i < n; ++i) {
    double x1[3] = {a[i], a[ld + i], a[2 * ld + i]};
    double x2[3] = {b[i], b[ld + i], b[2 * ld + i]};
    double slot[2][2];
    uint8_t c = intersect_one(mode, x1, x2, z0[i], slot, 0, 0);
    double nan = canonical_nan();
    for (int k = 0; k < 2; ++k) {
      int used = (c != OR_DEGENERATE) && (k < c);
      out_xyz[(k * 3 + 0) * ld + i] = slot[k][0];
      out_xyz[(k * 3 + 1) * ld + i] = slot[k][1];
      out_xyz[(k * 3 + 2) * ld + i] = used ? z0[i] : nan;
    }
    out_count[i] = c;
  }
  return 0;
}

/* Double-word points (reading R11): for each stored slot, the low part
 * `lo` with P ~ hi + lo, hi the stored (rounded) coordinate.  From the numerator's CompDotC pair
 * (p, sigma) (Alg.1) of the root in that slot, its CompDot X = RN(p + sigma), and
 * the pair (S2, s2) of |n_xy|^2 (Alg.7):
 *   t  = fma(hi, S2, X)          exact remainder of the rounded division
 *   dl = (p - X) + sigma         the numerator's low part
 *   r  = (t + dl) + hi * s2      N + hi D  (N = p + sigma, D = S2 + s2)
 *   lo = -(r / S2)               since -N/D = hi - (N + hi D)/D
 * Unused slots hold the canonical NaN in both planes.  EFT modes only. */
static double dw_lo(double hi, const double num_pair[2], double X, double S2, double s2) {
  double t = fma(hi, S2, X);
  double dl = (num_pair[0] - X) + num_pair[1];
  double r = (t + dl) + (hi * s2);
  return -(r / S2);
}

int oracle_intersect_dw_batch(int mode, const double* a, const double* b, const double* z0,
                              int64_t n, int64_t ld, double* out_xyz, double* out_lo,
                              uint8_t* out_count, int nthreads) {
  if ((mode != OR_MODE_EFT && mode != OR_MODE_EFT_LITERAL) || n < 0 || ld < n) return 1;
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t i = 0; i < n; ++i) {
    double x1[3] = {a[i], a[ld + i], a[2 * ld + i]};
    double x2[3] = {b[i], b[ld + i], b[2 * ld + i]};
    double slot[2][2];
    accux_trace t;
    int plus_first = 1;
    uint8_t c = intersect_one(mode, x1, x2, z0[i], slot, &t, &plus_first);
    double nan = canonical_nan();
    for (int k = 0; k < 2; ++k) {
      int used = (c != OR_DEGENERATE) && (k < c);
      out_xyz[(k * 3 + 0) * ld + i] = slot[k][0];
      out_xyz[(k * 3 + 1) * ld + i] = slot[k][1];
      out_xyz[(k * 3 + 2) * ld + i] = used ? z0[i] : nan;
      double lx = nan, ly = nan;
      if (used) {
        int plus = (k == 0) == plus_first;
        lx = dw_lo(slot[k][0], plus ? t.Xpp : t.Xmp, plus ? t.Xp : t.Xm, t.S2, t.s2);
        ly = dw_lo(slot[k][1], plus ? t.Ypp : t.Ymp, plus ? t.Yp : t.Ym, t.S2, t.s2);
      }
      out_lo[(k * 2 + 0) * ld + i] = lx;
      out_lo[(k * 2 + 1) * ld + i] = ly;
    }
    out_count[i] = c;
  }
  return 0;
}

/* Every intermediate of one query (Appendix-A instrumentation).  Fills 38 doubles
 * in the field order of accux_trace and returns the count. */
int oracle_trace(int mode, const double x1[3], const double x2[3], double z0, double* out30) {
  accux_trace t;
  double slot[2][2];
  int c = intersect_one(mode, x1, x2, z0, slot, &t, 0);
  memcpy(out30, &t, sizeof(t));
  return c;
}

/* Primitive batches for the operator pins.  op codes:
 *  0 two_sum(a,b)        1 fast_two_sum(a,b)     2 two_prod(a,b)
 *  3 kahan_dop(a,b,c,d)  4 accu_dop(a,b,c,d)     5 sum_non_neg((a,b),(c,d))
 *  6 sum_of_squares(x[k])                        7 sum_of_squares_c(x[k], e[k])
 *  8 acc_sqrt(H,h)       9 comp_dot_c(x[k],y[k]) 10 comp_dot(x[k], y[k])
 * `in` is row-major [n][width]; `out` is [n][2] (hi, lo; lo = 0 for scalar results).
 * For ops 6/7/9/10 the row holds x then e (or y), each of length k. */
int oracle_prim_batch(int op, int k, const double* in, int width, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double* r = in + i * width;
    pair p = {0.0, 0.0};
    switch (op) {
      case 0: p = two_sum(r[0], r[1]); break;
      case 1: p = fast_two_sum(r[0], r[1]); break;
      case 2: p = two_prod(r[0], r[1]); break;
      case 3: p.hi = kahan_dop(r[0], r[1], r[2], r[3]); break;
      case 4: p = accu_dop(r[0], r[1], r[2], r[3]); break;
      case 5: { pair A = {r[0], r[1]}, B = {r[2], r[3]}; p = sum_non_neg(A, B); } break;
      case 6: p = sum_of_squares(r, k); break;
      case 7: p = sum_of_squares_c(r, r + k, k); break;
      case 8: p = acc_sqrt(r[0], r[1]); break;
      case 9: p = comp_dot_c(r, r + k, k); break;
      case 10: p.hi = comp_dot(r, r + k, k); break;
      default: return 1;
    }
    out[2 * i] = p.hi;
    out[2 * i + 1] = p.lo;
  }
  return 0;
}
