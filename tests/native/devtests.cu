// tests/native/devtests.cu — device unit tests of the EFT primitives in csrc/sgi_eft.cuh.
// Test-only library (libsgi_devtest.so); checks the value-preserving rewrites of DESIGN.md §5
// against the reference formulations ON THE DEVICE, bit for bit, over counter-based random
// inputs with adversarial exponent spreads, cancellations, zeros and guard-boundary values:
//   two_sum (ordered FastTwoSum)  vs  two_sum_knuth (6-op TwoSum)     values, and e == a+b-s
//   div_fast with a shared div_recip  vs  __ddiv_rn                   (when its guard passes)
//   sqrt_fast                         vs  __dsqrt_rn                  (when its guard passes)
// and counts how often each guard fails (the Exact recomputation rate).
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_09892_b200/csrc/sgi_eft.cuh"
#include "../../paper_2510_09892_b200/csrc/sgi_query.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

// random double with exponent in [emin, emax], random sign; some specials
__device__ double rnd(uint64_t key, int emin, int emax) {
  uint64_t r = mix(key);
  uint64_t sel = r & 63;
  if (sel == 0) return 0.0;
  if (sel == 1) return -0.0;
  uint64_t mant = mix(r + 0x9e3779b97f4a7c15ull) & 0xFFFFFFFFFFFFFull;
  int e = emin + (int)((r >> 8) % (uint64_t)(emax - emin + 1));
  uint64_t sign = (r >> 7) & 1;
  uint64_t bits = (sign << 63) | ((uint64_t)(e + 1023) << 52) | mant;
  return __longlong_as_double((long long)bits);
}

__device__ bool same_bits_or_zero(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b) || (a == 0.0 && b == 0.0);
}

// out[0]: two_sum value mismatches; out[1]: zero-sign-only differences; out[2]: exactness
// failures (e != a + b - s checked with a second TwoSum); out[3]: div mismatches (guard ok);
// out[4]: div guard failures; out[5]: sqrt mismatches (guard ok); out[6]: sqrt guard failures;
// out[7]: AccuDOP renormalisation, FastTwoSum(hi, lo) != Knuth TwoSum(hi, lo) (values);
// out[8]: AccuDOP quadruples that cancelled (Sterbenz case exercised); out[9]: is_zero /
// is_pos / is_neg / is_nonneg disagreeing with the double comparisons
extern "C" __global__ void devtest_kernel(uint64_t seed, int64_t n, unsigned long long* out) {
  unsigned long long c[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = seed * 0x100000001b3ull + (uint64_t)i * 8;
    double a = rnd(k, -200, 200);
    double b;
    uint64_t mode = mix(k + 1) % 4;
    if (mode == 0) b = rnd(k + 2, -200, 200);
    else if (mode == 1) b = -a * (1.0 + (double)((int)(mix(k + 3) % 9) - 4) * 1.1102230246251565e-16);
    else if (mode == 2) b = rnd(k + 2, -60, 60) * a;
    else b = a * 0.5 + rnd(k + 2, -120, -40);
    sgi::dd x = sgi::two_sum(a, b), y = sgi::two_sum_knuth(a, b);
    if (x.hi != y.hi || x.lo != y.lo) c[0]++;
    else if (__double_as_longlong(x.lo) != __double_as_longlong(y.lo)) c[1]++;
    // exactness: s + e == a + b  <=>  TwoSum(s, e) reproduces (s, e) and a - s + b == e exactly
    sgi::dd z = sgi::two_sum_knuth(x.hi, x.lo);
    if (z.hi != x.hi || z.lo != x.lo) c[2]++;
    // division with a shared reciprocal (numerators spread over many magnitudes, some tiny)
    double den = fabs(rnd(k + 4, -100, 100)) + 1e-300;
    double y0 = sgi::div_recip(den);
    for (int j = 0; j < 4; ++j) {
      double num = rnd(k + 5 + j, (j == 3) ? -1070 : -200, 200);
      bool ok = true;
      double q = sgi::div_fast(num, den, y0, ok);
      if (!ok) { c[4]++; continue; }
      if (!same_bits_or_zero(q, __ddiv_rn(num, den))) c[3]++;
    }
    double sx = fabs(rnd(k + 9, (mode == 3) ? -1074 : -300, 300));
    bool oks = true;
    double r = sgi::sqrt_fast(sx, oks);
    if (!oks) c[6]++;
    else if (!same_bits_or_zero(r, __dsqrt_rn(sx))) c[5]++;
    // AccuDOP a*b - c*d and its renormalisation (sgi_query.cuh accux_edge): c*d near a*b
    {
      double pa = rnd(k + 11, -100, 100), pb = rnd(k + 12, -100, 100);
      double pc = rnd(k + 13, -100, 100), pd;
      uint64_t m2 = mix(k + 14) % 4;
      if (m2 == 0 || pc == 0.0) pd = rnd(k + 15, -100, 100);
      else if (m2 == 1) pd = __ddiv_rn(__dmul_rn(pa, pb), pc);            // near-exact cancel
      else if (m2 == 2) pd = __dadd_rn(__ddiv_rn(__dmul_rn(pa, pb), pc),  // a few ulps off
                                       __dmul_rn(rnd(k + 16, -56, -50), __ddiv_rn(__dmul_rn(pa, pb), pc)));
      else pd = __dmul_rn(__ddiv_rn(__dmul_rn(pa, pb), pc), 0.5 + (double)(mix(k + 17) & 7) * 0.25);
      sgi::dd h = sgi::accu_dop(pa, pb, pc, pd);
      sgi::dd f = sgi::fast_two_sum(h.hi, h.lo), g = sgi::two_sum_knuth(h.hi, h.lo);
      if (f.hi != g.hi || f.lo != g.lo) c[7]++;
      const double p1 = __dmul_rn(pa, pb), p2 = __dmul_rn(pc, pd);
      if (p1 != 0.0 && p1 == __dadd_rn(__dsub_rn(p1, p2), p2) && fabs(p2) <= 2 * fabs(p1) &&
          fabs(p1) <= 2 * fabs(p2)) c[8]++;
      // sign / zero helpers against the double comparisons on the same spread of values
      const double v[4] = {h.hi, h.lo, a, -b};
      for (int j = 0; j < 4; ++j) {
        const double x = v[j];
        if (sgi::is_zero(x) != (x == 0.0) || sgi::is_pos(x) != (x > 0.0) ||
            sgi::is_neg(x) != (x < 0.0) || sgi::is_nonneg(x) != (x >= 0.0)) c[9]++;
      }
    }
  }
  for (int j = 0; j < 10; ++j)
    if (c[j]) atomicAdd(out + j, c[j]);
}

extern "C" int sgi_devtest(uint64_t seed, int64_t n, unsigned long long* d_out) {
  cudaMemset(d_out, 0, 10 * sizeof(unsigned long long));
  devtest_kernel<<<148 * 8, 256>>>(seed, n, d_out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}

// ------------------------------------------------------------------------------------------
// The device primitives one by one, in the op numbering of oracle_prim_batch (oracle (a)), so a
// test can compare each against the CPU oracle bit for bit on the same rows.  SumOfSquares starts
// from its first TwoProd as the production code does (reading A12: the first SumNonNeg with (0,0)
// is an exact identity); CompDotC/CompDot are the CompDotC step of sgi_eft.cuh in a loop;
// AccSqrt runs the Exact policy, or the Fast policy (then out[2i+1] is NaN where its guard
// failed, i.e. where the production code would recompute).
__global__ void devprim_kernel(int op, int k, const double* in, int width, int64_t n,
                               double* out, int fast) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* r = in + i * width;
    sgi::dd p = {0.0, 0.0};
    switch (op) {
      case 0: p = sgi::two_sum(r[0], r[1]); break;
      case 1: p = sgi::fast_two_sum(r[0], r[1]); break;
      case 2: p = sgi::two_prod(r[0], r[1]); break;
      case 3: p.hi = sgi::kahan_dop(r[0], r[1], r[2], r[3]); break;
      case 4: p = sgi::accu_dop(r[0], r[3], r[1], r[2]); break;   // oracle order: a*d - b*c
      case 5: p = sgi::sum_non_neg(sgi::dd{r[0], r[1]}, sgi::dd{r[2], r[3]}); break;
      case 6: case 7: {
        sgi::dd S = sgi::two_prod(r[0], r[0]);
        for (int j = 1; j < k; ++j) S = sgi::sum_non_neg(S, sgi::two_prod(r[j], r[j]));
        if (op == 6) { p = S; break; }
        sgi::dd R = sgi::two_prod(r[0], r[k]);
        for (int j = 1; j < k; ++j) sgi::cdc_step(R.hi, R.lo, r[j], r[k + j]);
        p = sgi::fast_two_sum(S.hi, sgi::fma(2.0, sgi::add(R.hi, R.lo), S.lo));
      } break;
      case 8: {
        bool ok_root = true, ok_div = true;
        if (fast) {
          p = sgi::acc_sqrt<sgi::Fast>(r[0], r[1], ok_root, ok_div);
          if (!(ok_root && ok_div)) p.lo = sgi::qnan();
        } else {
          p = sgi::acc_sqrt<sgi::Exact>(r[0], r[1], ok_root, ok_div);
        }
      } break;
      case 9: case 10: {
        sgi::dd P = sgi::two_prod(r[0], r[k]);
        for (int j = 1; j < k; ++j) sgi::cdc_step(P.hi, P.lo, r[j], r[k + j]);
        p = op == 9 ? P : sgi::dd{sgi::add(P.hi, P.lo), 0.0};
      } break;
      case 11: {   // certified numerators (policy Cert): row [F, eF, v, ev, z0, s, es]
        double Xp, Xm;
        bool ok = true;
        sgi::numerators_cert(r[0], r[1], r[2], r[3], r[4], r[5], r[6], Xp, Xm, ok);
        p = ok ? sgi::dd{Xp, Xm} : sgi::dd{sgi::qnan(), sgi::qnan()};
      } break;
      case 12: {   // the same through the two-lane type (rows i and i + n/2 as one W2 pair)
        if (i >= n / 2) break;
        const double* q = in + (i + n / 2) * width;
        sgi::W2 Xp, Xm;
        sgi::B2 ok = {true, true};
        sgi::numerators_cert(sgi::W2{r[0], q[0]}, sgi::W2{r[1], q[1]}, sgi::W2{r[2], q[2]},
                             sgi::W2{r[3], q[3]}, sgi::W2{r[4], q[4]}, sgi::W2{r[5], q[5]},
                             sgi::W2{r[6], q[6]}, Xp, Xm, ok);
        out[2 * (i + n / 2)] = ok.y ? Xp.y : sgi::qnan();
        out[2 * (i + n / 2) + 1] = ok.y ? Xm.y : sgi::qnan();
        p = ok.x ? sgi::dd{Xp.x, Xm.x} : sgi::dd{sgi::qnan(), sgi::qnan()};
      } break;
      case 14: {   // one root at a time (policy Cert's stored-roots path): + then - root
        bool okp = true, okm = true;
        const double Xp = sgi::numerator_cert_one(r[0], r[1], r[2], r[3], r[4], r[5], r[6], okp, 0.0);
        const double Xm = sgi::numerator_cert_one(r[0], r[1], r[2], r[3], r[4], sgi::flip_if(r[5], true),
                                                  sgi::flip_if(r[6], true), okm, 0.0);
        p = sgi::dd{okp ? Xp : sgi::qnan(), okm ? Xm : sgi::qnan()};
      } break;
      case 13: {   // policy Cert's front: row [nx, ex, ny, ey, nz, ez, z0] -> (S2, sigma_h)
        sgi::EdgePreT<double> e;
        e.nx = {r[0], r[1]}; e.ny = {r[2], r[3]}; e.nz = {r[4], r[5]};
        sgi::cert_sums(e);
        bool ok = true;
        const sgi::CertFront<double> f = sgi::cert_sigma(e, r[6], ok);
        p = ok ? sgi::dd{f.S2, f.sh} : sgi::dd{sgi::qnan(), sgi::qnan()};
      } break;
      default: break;
    }
    if (op == 12 && i >= n / 2) continue;
    out[2 * i] = p.hi;
    out[2 * i + 1] = p.lo;
  }
}

extern "C" int sgi_devprim(int op, int k, const double* d_in, int width, int64_t n, double* d_out,
                           int fast) {
  devprim_kernel<<<148 * 4, 256>>>(op, k, d_in, width, n, d_out, fast);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
