/* sgi_inputs/gen.h — seeded, counter-based synthetic arc generators (configs C1-C3, C5, and
 * the paper's primary / secondary accuracy datasets, configs 6 and 7).
 *
 * A module of its own: it builds INPUTS only (endpoint pairs a, b and latitude z0) and holds
 * none of the method's arithmetic (no AccuX, no EFT, no intersection formula).  The same source
 * is compiled for the host (gcc, -ffp-contract=off) and for the device (nvcc, -fmad=false), and
 * uses only integer ops plus correctly rounded IEEE +,-,*,/,sqrt — no libm transcendentals —
 * so the host and device builds produce bit-identical arcs.  That lets CPU-only tests and the
 * oracles regenerate exactly the arcs the GPU bench and parity tests consume.
 *
 * Workload shapes follow BASELINE.json `configs` (read as in SURVEY.md §8(d)); DESIGN.md §3
 * states the recipe.  Paper context: the paper's own datasets are self-generated random arcs
 * (§7, lines 949-953 and 1040); none of its data is reproduced here.
 *
 * RNG: Philox4x32-10 keyed by the 64-bit seed, counter = (global arc index lo/hi, draw block,
 * config tag).  One Philox block yields two 53-bit uniforms.  Arc i depends only on
 * (config, seed, i), so any sharding of the index range reproduces the same arcs.
 */
#ifndef SGI_INPUTS_GEN_H
#define SGI_INPUTS_GEN_H

#include <stdint.h>

#ifdef __CUDACC__
#define GEN_HD __device__ __forceinline__
#define GEN_SQRT(x) __dsqrt_rn(x)
#define GEN_ADD(a, b) __dadd_rn(a, b)
#define GEN_SUB(a, b) __dsub_rn(a, b)
#define GEN_MUL(a, b) __dmul_rn(a, b)
#define GEN_DIV(a, b) __ddiv_rn(a, b)
#else
#include <math.h>
#define GEN_HD static inline
#define GEN_SQRT(x) sqrt(x)
#define GEN_ADD(a, b) ((a) + (b))
#define GEN_SUB(a, b) ((a) - (b))
#define GEN_MUL(a, b) ((a) * (b))
#define GEN_DIV(a, b) ((a) / (b))
#endif

/* ---------------------------------------------------------------- Philox4x32-10 */
typedef struct { uint32_t v[4]; } gen_u32x4;

GEN_HD uint32_t gen_mulhilo(uint32_t a, uint32_t b, uint32_t* hi) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  return (uint32_t)p;
}

GEN_HD gen_u32x4 gen_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, hi1;
    uint32_t lo0 = gen_mulhilo(0xD2511F53u, c0, &hi0);
    uint32_t lo1 = gen_mulhilo(0xCD9E8D57u, c2, &hi1);
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  gen_u32x4 out = {{c0, c1, c2, c3}};
  return out;
}

/* Per-arc draw stream: block b of arc i yields two uniforms in [0,1) with 53 random bits. */
typedef struct {
  uint64_t seed, index;
  uint32_t tag, block;
  double buf[2];
  int avail;
} gen_stream;

GEN_HD void gen_stream_init(gen_stream* s, uint64_t seed, uint64_t index, uint32_t tag) {
  s->seed = seed; s->index = index; s->tag = tag; s->block = 0; s->avail = 0;
}

GEN_HD double gen_u53(uint32_t hi, uint32_t lo) {
  /* (hi>>5)*2^26 + (lo>>6) is an exact 53-bit integer; scaling by 2^-53 is exact. */
  return GEN_MUL(GEN_ADD((double)(hi >> 5) * 67108864.0, (double)(lo >> 6)), 1.1102230246251565e-16);
}

GEN_HD double gen_uniform(gen_stream* s) {
  if (s->avail == 0) {
    gen_u32x4 r = gen_philox((uint32_t)s->index, (uint32_t)(s->index >> 32), s->block, s->tag, s->seed);
    s->block++;
    s->buf[0] = gen_u53(r.v[0], r.v[1]);
    s->buf[1] = gen_u53(r.v[2], r.v[3]);
    s->avail = 2;
  }
  return s->buf[2 - (s->avail--)];
}

/* ------------------------------------------------------- exact-op helper functions */
/* 2^k for -1022 <= k <= 1023, built from the exponent field (exact). */
GEN_HD double gen_pow2i(int k) {
  union { uint64_t u; double d; } c;
  c.u = (uint64_t)(k + 1023) << 52;
  return c.d;
}

/* 10^x for x in [-20, 0] from +,*,floor only (Horner Taylor series of 2^f on [0,1)).
 * Accuracy ~1e-16 relative — irrelevant for a log-uniform sampler; what matters is that
 * host and device evaluate the identical op sequence. */
GEN_HD double gen_exp10(double x) {
  double y = GEN_MUL(x, 3.321928094887362);   /* log2(10) */
  double fl = (double)(int64_t)y;
  if (fl > y) fl = GEN_SUB(fl, 1.0);           /* floor for negative y */
  double f = GEN_MUL(GEN_SUB(y, fl), 0.6931471805599453); /* f*ln2 in [0, ln2) */
  double p = 1.0;
  for (int k = 22; k >= 1; --k) p = GEN_ADD(1.0, GEN_DIV(GEN_MUL(p, f), (double)k));
  return GEN_MUL(p, gen_pow2i((int)fl));
}

/* log-uniform in [10^lo, 10^hi) */
GEN_HD double gen_logu(gen_stream* s, double lo, double hi) {
  double u = gen_uniform(s);
  return gen_exp10(GEN_ADD(lo, GEN_MUL(u, GEN_SUB(hi, lo))));
}

GEN_HD void gen_normalize3(double v[3]) {
  double r2 = GEN_ADD(GEN_ADD(GEN_MUL(v[0], v[0]), GEN_MUL(v[1], v[1])), GEN_MUL(v[2], v[2]));
  double r = GEN_SQRT(r2);
  v[0] = GEN_DIV(v[0], r); v[1] = GEN_DIV(v[1], r); v[2] = GEN_DIV(v[2], r);
}

/* Uniform direction on S^2 by rejection from the cube [-1,1]^3 (no transcendentals). */
GEN_HD void gen_unit3(gen_stream* s, double v[3]) {
  for (int attempt = 0; attempt < 256; ++attempt) {
    double x = GEN_SUB(GEN_MUL(2.0, gen_uniform(s)), 1.0);
    double y = GEN_SUB(GEN_MUL(2.0, gen_uniform(s)), 1.0);
    double z = GEN_SUB(GEN_MUL(2.0, gen_uniform(s)), 1.0);
    double r2 = GEN_ADD(GEN_ADD(GEN_MUL(x, x), GEN_MUL(y, y)), GEN_MUL(z, z));
    if (r2 <= 1.0 && r2 > 1e-4) { v[0] = x; v[1] = y; v[2] = z; gen_normalize3(v); return; }
  }
  v[0] = 0.0; v[1] = 0.0; v[2] = 1.0; /* unreachable in practice (p ~ 0.48^256) */
}

/* Uniform direction on S^1 by rejection from the square. */
GEN_HD void gen_unit2(gen_stream* s, double* cx, double* cy) {
  for (int attempt = 0; attempt < 256; ++attempt) {
    double x = GEN_SUB(GEN_MUL(2.0, gen_uniform(s)), 1.0);
    double y = GEN_SUB(GEN_MUL(2.0, gen_uniform(s)), 1.0);
    double r2 = GEN_ADD(GEN_MUL(x, x), GEN_MUL(y, y));
    if (r2 <= 1.0 && r2 > 1e-4) { double r = GEN_SQRT(r2); *cx = GEN_DIV(x, r); *cy = GEN_DIV(y, r); return; }
  }
  *cx = 1.0; *cy = 0.0;
}

/* Unit tangent at unit vector m: Gram-Schmidt of a random direction against m. */
GEN_HD void gen_tangent(gen_stream* s, const double m[3], double d[3]) {
  for (int attempt = 0; attempt < 64; ++attempt) {
    double g[3];
    gen_unit3(s, g);
    double gm = GEN_ADD(GEN_ADD(GEN_MUL(g[0], m[0]), GEN_MUL(g[1], m[1])), GEN_MUL(g[2], m[2]));
    d[0] = GEN_SUB(g[0], GEN_MUL(gm, m[0]));
    d[1] = GEN_SUB(g[1], GEN_MUL(gm, m[1]));
    d[2] = GEN_SUB(g[2], GEN_MUL(gm, m[2]));
    double r2 = GEN_ADD(GEN_ADD(GEN_MUL(d[0], d[0]), GEN_MUL(d[1], d[1])), GEN_MUL(d[2], d[2]));
    if (r2 > 1e-4) { gen_normalize3(d); return; }
  }
  d[0] = 1.0; d[1] = 0.0; d[2] = 0.0;
}

/* z0 uniform between the endpoint z values, clamped to that closed interval. */
GEN_HD double gen_z0_between(gen_stream* s, double za, double zb) {
  double lo = za < zb ? za : zb, hi = za < zb ? zb : za;
  double z = GEN_ADD(lo, GEN_MUL(gen_uniform(s), GEN_SUB(hi, lo)));
  if (z < lo) z = lo;
  if (z > hi) z = hi;
  return z;
}

/* Endpoints m -/+ h*d, normalised: a short arc of length 2*atan(h) ~ 2h centred on m. */
GEN_HD void gen_short_arc(const double m[3], const double d[3], double h, double a[3], double b[3]) {
  for (int c = 0; c < 3; ++c) {
    a[c] = GEN_SUB(m[c], GEN_MUL(h, d[c]));
    b[c] = GEN_ADD(m[c], GEN_MUL(h, d[c]));
  }
  gen_normalize3(a);
  gen_normalize3(b);
}

/* sin and cos of x in [-4, 8] (radians) from +,-,*,/ only: Cody-Waite reduction by pi/2 to
 * |r| <= pi/4 (two-part pi/2), Taylor series to degree 23/22, quadrant rotation.  Accuracy
 * ~1 ulp — irrelevant for a sampler (inputs need not be unit length); what matters
 * is that host and device evaluate the identical op sequence. */
GEN_HD void gen_sincos(double x, double* sn, double* cs) {
  double kq = (double)(int64_t)GEN_ADD(GEN_MUL(x, 0.6366197723675814), 8.5);  /* round(x*2/pi)+8 */
  kq = GEN_SUB(kq, 8.0);
  double r = GEN_SUB(GEN_SUB(x, GEN_MUL(kq, 1.5707963267948966)), GEN_MUL(kq, 6.123233995736766e-17));
  double r2 = GEN_MUL(r, r);
  double ps = 1.0, pc = 1.0;
  for (int k = 23; k >= 3; k -= 2) ps = GEN_SUB(1.0, GEN_DIV(GEN_MUL(ps, r2), (double)(k * (k - 1))));
  for (int k = 22; k >= 2; k -= 2) pc = GEN_SUB(1.0, GEN_DIV(GEN_MUL(pc, r2), (double)(k * (k - 1))));
  double s0 = GEN_MUL(r, ps), c0 = pc;
  int q = ((int)kq) & 3;
  if (q == 0) { *sn = s0; *cs = c0; }
  else if (q == 1) { *sn = c0; *cs = -s0; }
  else if (q == 2) { *sn = -s0; *cs = -c0; }
  else { *sn = -c0; *cs = s0; }
}

#define GEN_DEG 0.017453292519943295   /* pi/180 */

/* Point at latitude lat_deg in [0, 90] and longitude lon_deg: z = cos(colatitude) and
 * |p_xy| = sin(colatitude), with the colatitude 90 - lat formed exactly near the pole. */
GEN_HD void gen_latlon(double lat_deg, double lon_deg, double p[3]) {
  double sc, cc, sl, cl;
  gen_sincos(GEN_MUL(GEN_SUB(90.0, lat_deg), GEN_DEG), &sc, &cc);
  gen_sincos(GEN_MUL(lon_deg, GEN_DEG), &sl, &cl);
  p[0] = GEN_MUL(sc, cl); p[1] = GEN_MUL(sc, sl); p[2] = cc;
}

/* The paper's primary accuracy dataset: northern-hemisphere latitude bands, narrower
 * near the equator and the pole.  The paper does not print its band edges; these are SPEC's
 * default schedule, in degrees: 17 bands. */
#define GEN_NBANDS 17
GEN_HD double gen_band_edge(int k) {
  const double e[GEN_NBANDS + 1] = {0.0, 1e-4, 1e-3, 1e-2, 0.1, 1.0, 11.0, 21.0, 31.0, 41.0, 51.0,
                                    61.0, 71.0, 81.0, 89.0, 89.9, 89.99, 89.999};
  return e[k];
}
/* The paper's secondary dataset groups by the decade of the offset r: 13 decades
 * [1e-15, 1e-14) ... [1e-3, 1e-2). */
#define GEN_NDECADES 13

/* ------------------------------------------------------------------ configs */
enum { GEN_C1 = 1, GEN_C2 = 2, GEN_C3 = 3, GEN_C5 = 5, GEN_PRIMARY = 6, GEN_SECONDARY = 7 };

/* C1: a, b i.i.d. uniform on the sphere; z0 uniform between a_z and b_z. */
GEN_HD void gen_arc_uniform(gen_stream* s, double a[3], double b[3], double* z0) {
  gen_unit3(s, a);
  gen_unit3(s, b);
  *z0 = gen_z0_between(s, a[2], b[2]);
}

/* C2: short arcs — midpoint uniform, length log-uniform in [1e-4, 1e-2] rad, random
 * orientation (0.1-0.5 degree climate-mesh edges); z0 between the endpoint z values. */
GEN_HD void gen_arc_short(gen_stream* s, double a[3], double b[3], double* z0) {
  double m[3], d[3];
  gen_unit3(s, m);
  gen_tangent(s, m, d);
  double L = gen_logu(s, -4.0, -2.0);
  gen_short_arc(m, d, GEN_MUL(0.5, L), a, b);
  *z0 = gen_z0_between(s, a[2], b[2]);
}

/* C3 class 0: near-tangent.  Random unit normal nh; apex A (antapex for odd i/3) is the
 * highest (lowest) point of its great circle, at height +-|nh_xy|; the arc spans
 * theta in [1e-2, 1e-1] rad on both sides of it; z0 = z_ext * (1 - delta), delta log-uniform
 * in [1e-15, 1e-6]. */
GEN_HD void gen_arc_tangent(gen_stream* s, uint64_t i, double a[3], double b[3], double* z0) {
  double nh[3];
  for (int attempt = 0; attempt < 64; ++attempt) {
    gen_unit3(s, nh);
    if (GEN_ADD(GEN_MUL(nh[0], nh[0]), GEN_MUL(nh[1], nh[1])) > 1e-6) break;
  }
  double rxy = GEN_SQRT(GEN_ADD(GEN_MUL(nh[0], nh[0]), GEN_MUL(nh[1], nh[1])));
  double sgn = ((i / 3) & 1) ? -1.0 : 1.0;
  double A[3] = {GEN_MUL(sgn, GEN_DIV(GEN_MUL(-nh[0], nh[2]), rxy)),
                 GEN_MUL(sgn, GEN_DIV(GEN_MUL(-nh[1], nh[2]), rxy)), GEN_MUL(sgn, rxy)};
  double T[3] = {GEN_SUB(GEN_MUL(nh[1], A[2]), GEN_MUL(nh[2], A[1])),
                 GEN_SUB(GEN_MUL(nh[2], A[0]), GEN_MUL(nh[0], A[2])),
                 GEN_SUB(GEN_MUL(nh[0], A[1]), GEN_MUL(nh[1], A[0]))};
  double theta = gen_logu(s, -2.0, -1.0);
  gen_short_arc(A, T, theta, a, b);
  double delta = gen_logu(s, -15.0, -6.0);
  double zext = GEN_MUL(sgn, rxy);
  *z0 = GEN_SUB(zext, GEN_MUL(zext, delta));
}

/* C3 class 1: near-polar endpoints, |z| = RN(1 - t), t log-uniform in [2^-52, 1e-10]; the
 * hemisphere alternates with i/3; z0 between the endpoint z values. */
GEN_HD void gen_polar_point(gen_stream* s, double sgn, double p[3]) {
  double t = gen_logu(s, -15.653559774527022, -10.0); /* log10(2^-52) */
  double az = GEN_SUB(1.0, t);
  double r = GEN_SQRT(GEN_MUL(GEN_SUB(1.0, az), GEN_ADD(1.0, az)));
  double cx, cy;
  gen_unit2(s, &cx, &cy);
  p[0] = GEN_MUL(r, cx); p[1] = GEN_MUL(r, cy); p[2] = GEN_MUL(sgn, az);
}

GEN_HD void gen_arc_polar(gen_stream* s, uint64_t i, double a[3], double b[3], double* z0) {
  double sgn = ((i / 3) & 1) ? -1.0 : 1.0;
  gen_polar_point(s, sgn, a);
  gen_polar_point(s, sgn, b);
  *z0 = gen_z0_between(s, a[2], b[2]);
}

/* C3 class 2: near-coincident endpoints, separation log-uniform in [1e-12, 1e-7] rad. */
GEN_HD void gen_arc_coincident(gen_stream* s, double a[3], double b[3], double* z0) {
  double d[3];
  gen_unit3(s, a);
  gen_tangent(s, a, d);
  double th = gen_logu(s, -12.0, -7.0);
  for (int c = 0; c < 3; ++c) b[c] = GEN_ADD(a[c], GEN_MUL(th, d[c]));
  gen_normalize3(b);
  *z0 = gen_z0_between(s, a[2], b[2]);
}

/* C5 class 3: endpoints uniform on the sphere, z0 uniform in [-1, 1] (0/1/2 points all occur). */
GEN_HD void gen_arc_free(gen_stream* s, double a[3], double b[3], double* z0) {
  gen_unit3(s, a);
  gen_unit3(s, b);
  *z0 = GEN_SUB(GEN_MUL(2.0, gen_uniform(s)), 1.0);
}

/* Primary dataset, band k = i mod 17: both endpoints at latitudes uniform in the band
 * and longitudes uniform in [0, 360) degrees; z0 uniform between the endpoint z values. */
GEN_HD void gen_arc_primary(gen_stream* s, uint64_t i, double a[3], double b[3], double* z0) {
  const int k = (int)(i % GEN_NBANDS);
  const double lo = gen_band_edge(k), hi = gen_band_edge(k + 1);
  const double w = GEN_SUB(hi, lo);
  double la = GEN_ADD(lo, GEN_MUL(gen_uniform(s), w)), lb = GEN_ADD(lo, GEN_MUL(gen_uniform(s), w));
  if (la <= 0.0) la = hi;      /* the band is (lo, hi]: u = 0 maps to its top */
  if (lb <= 0.0) lb = hi;
  gen_latlon(la, GEN_MUL(360.0, gen_uniform(s)), a);
  gen_latlon(lb, GEN_MUL(360.0, gen_uniform(s)), b);
  *z0 = gen_z0_between(s, a[2], b[2]);
}

/* Secondary dataset, decade d = i mod 13: shallow arcs near the equator, endpoints
 * in the latitude band (0, 1e-4 deg], and z0 = (top of the great circle) - r with r
 * log-uniform in [10^(d-15), 10^(d-14)).  Built from a designed circle, so no intersection
 * arithmetic runs here (reading R10): its top height h = sin(tau) is log-uniform in
 * [h0, 10 h0], h0 = max(sin(1e-4 deg), 2r) (the circle must reach above z0 = h - r > -h);
 * apex A = (cos tau cos lam, cos tau sin lam, h), horizontal tangent T = (-sin lam, cos lam, 0);
 * each endpoint c A -+ sqrt(1 - c^2) T sits on either side of the apex at height z = c h drawn
 * uniform in (0, min(sin(1e-4 deg), z0 (1 - 1e-3))], so both intersection points lie on the
 * arc.  z0 uses the designed h, not a height recomputed from the rounded endpoints. */
GEN_HD void gen_arc_secondary(gen_stream* s, uint64_t i, double a[3], double b[3], double* z0) {
  const int d = (int)(i % GEN_NDECADES);
  const double r = gen_logu(s, (double)(d - 15), (double)(d - 14));
  const double zband = 1.7453292519057202e-06;          /* sin(1e-4 deg) */
  const double h0 = GEN_MUL(2.0, r) > zband ? GEN_MUL(2.0, r) : zband;
  const double top = GEN_MUL(h0, gen_exp10(gen_uniform(s)));   /* log-uniform in [h0, 10 h0) */
  const double ct = GEN_SQRT(GEN_MUL(GEN_SUB(1.0, top), GEN_ADD(1.0, top)));
  double sl, cl;
  gen_sincos(GEN_MUL(GEN_MUL(360.0, gen_uniform(s)), GEN_DEG), &sl, &cl);
  const double A[3] = {GEN_MUL(ct, cl), GEN_MUL(ct, sl), top};
  const double T[3] = {-sl, cl, 0.0};
  *z0 = GEN_SUB(top, r);
  double zmax = GEN_MUL(*z0, 0.999);
  if (zmax > zband) zmax = zband;
  for (int e = 0; e < 2; ++e) {
    double u = gen_uniform(s);
    double z = GEN_MUL(GEN_SUB(1.0, u), zmax);         /* (0, zmax] */
    double c = GEN_DIV(z, top);
    double sn = GEN_SQRT(GEN_MUL(GEN_SUB(1.0, c), GEN_ADD(1.0, c)));
    double* p = e == 0 ? a : b;
    double sg = e == 0 ? -1.0 : 1.0;
    for (int k = 0; k < 3; ++k) p[k] = GEN_ADD(GEN_MUL(c, A[k]), GEN_MUL(GEN_MUL(sg, sn), T[k]));
  }
}

/* Group of arc i in the paper-shaped configs: band (primary) or decade (secondary). */
GEN_HD int gen_group(int config, uint64_t i) {
  if (config == GEN_PRIMARY) return (int)(i % GEN_NBANDS);
  if (config == GEN_SECONDARY) return (int)(i % GEN_NDECADES);
  return 0;
}

/* Arc `i` (global index) of `config`.  Returns 0 on success, -1 for an unknown config. */
GEN_HD int gen_arc(int config, uint64_t seed, uint64_t i, double a[3], double b[3], double* z0) {
  gen_stream s;
  gen_stream_init(&s, seed, i, (uint32_t)config);
  switch (config) {
    case GEN_C1: gen_arc_uniform(&s, a, b, z0); return 0;
    case GEN_C2: gen_arc_short(&s, a, b, z0); return 0;
    case GEN_C3:
      switch (i % 3) {
        case 0: gen_arc_tangent(&s, i, a, b, z0); return 0;
        case 1: gen_arc_polar(&s, i, a, b, z0); return 0;
        default: gen_arc_coincident(&s, a, b, z0); return 0;
      }
    case GEN_C5:
      switch (i % 4) {
        case 0: case 1: gen_arc_uniform(&s, a, b, z0); return 0;
        case 2: gen_arc_short(&s, a, b, z0); return 0;
        default: gen_arc_free(&s, a, b, z0); return 0;
      }
    case GEN_PRIMARY: gen_arc_primary(&s, i, a, b, z0); return 0;
    case GEN_SECONDARY: gen_arc_secondary(&s, i, a, b, z0); return 0;
    default: return -1;
  }
}

#endif /* SGI_INPUTS_GEN_H */
