// Double-double natural logarithm, __host__ __device__, for the polar sampler.
//
// The reference draws normals with libstdc++'s Marsaglia polar method
// (libstdc++ random.tcc:1810-1843), whose multiplier is
// sqrt(-2 log(r2) / r2).  Everything in that formula except log is correctly
// rounded IEEE arithmetic, so the device stream equals the host stream bit for
// bit exactly where the device log equals glibc's log.  glibc 2.39 log is not
// correctly rounded (0.081% of polar inputs differ from the correctly rounded
// value, and its bits depend on the host CPU's FMA ifunc), so the best a
// host-independent device implementation can do is the correctly rounded
// result: this routine evaluates log(x) to ~2^-75 relative in double-double
// and rounds once.  tests/test_rng_log.py measures the agreement with glibc.
//
// Method: x = 2^e * m, m in [sqrt(1/2), sqrt(2)); c_i ~ 1/m from a 256-entry
// table (9 significant bits, c = 1 exactly around m = 1); r = m*c_i - 1 exact
// as a double-double (two-product); log x = e*ln2 - log(c_i) + log1p(r), the
// first three log1p terms in double-double, the rest (|r| < 2^-8) in double.
#pragma once
#include <cmath>
#include <cstdint>

#ifndef __CUDACC__
#define RSVD_HD
#else
#define RSVD_HD __host__ __device__
#endif

namespace rsvdb {
namespace ddlog {

struct dd {
  double hi, lo;
};

RSVD_HD inline dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
RSVD_HD inline dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
RSVD_HD inline dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
RSVD_HD inline dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
RSVD_HD inline dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
RSVD_HD inline dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return quick_two_sum(p.hi, p.lo);
}
RSVD_HD inline dd dd_div_d(dd a, double b) {
  const double q1 = a.hi / b;
  dd p = two_prod(q1, b);
  const double r = ((a.hi - p.hi) - p.lo + a.lo) / b;
  return quick_two_sum(q1, r);
}

constexpr int kTableBits = 8;
constexpr int kTableSize = 256;  // index i = round((m - 0.5) * 256), m in [0.70, 1.42)

// Table entry: c_i (9-bit) and -log(c_i) as double-double.
struct Entry {
  double c, nlog_hi, nlog_lo;
};

RSVD_HD inline double table_c(int i) {
  // c = 1 / (0.5 + i/256), rounded to 9 significant bits.
  const double v = 1.0 / (0.5 + double(i) / 256.0);
  int e;
  const double f = frexp(v, &e);  // v = f * 2^e, f in [0.5, 1)
  return ldexp(nearbyint(f * 512.0), e - 9);
}

// log(c) for c in (0.7, 1.42) to ~2^-104: 2*atanh(s), s = (c-1)/(c+1).
inline dd host_log_dd(double c) {
  // s as double-double: (c - 1) exact, (c + 1) exact for 9-bit c.
  const double num = c - 1.0, den = c + 1.0;
  dd s = dd_div_d(dd{num, 0.0}, den);
  dd s2 = dd_mul(s, s);
  dd term = s;
  dd sum = s;
  for (int k = 3; k < 80; k += 2) {
    term = dd_mul(term, s2);
    const dd add = dd_div_d(term, double(k));
    sum = dd_add(sum, add);
    if (std::fabs(add.hi) < 1e-40) break;
  }
  return dd_add(sum, sum);
}

inline void build_table(Entry* t) {
  for (int i = 0; i < kTableSize; ++i) {
    const double c = (i >= 40 && i <= 240) ? table_c(i) : 1.0;
    const dd l = host_log_dd(c);
    t[i] = {c, -l.hi, -l.lo};
  }
}

constexpr double kLn2Hi = 0.6931471805599453094;   // RN(ln 2)
constexpr double kLn2Lo = 2.319046813846299558e-17; // ln 2 - kLn2Hi

// Natural log of a positive normal double (the polar sampler's r2 in (0,1])
// as a normalized double-double (|lo| <= ulp(hi)/2).
RSVD_HD inline dd log_dd(double x, const Entry* table) {
  int e;
  double m = frexp(x, &e);  // x = m * 2^e, m in [0.5, 1)
  m *= 2.0;
  e -= 1;                    // m in [1, 2)
  if (m >= 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const int i = int(nearbyint((m - 0.5) * 256.0));
  const Entry en = table[i];
  // r = m*c - 1 exactly as double-double
  const dd p = two_prod(m, en.c);
  dd r = quick_two_sum(p.hi - 1.0, p.lo);
  // log1p(r) = r - r^2/2 + r^3/3 - r^4/4 + ...
  const dd r2 = dd_mul(r, r);
  const dd r3 = dd_mul(r2, r);
  const double rh = r.hi;
  // tail in double: -r^4/4 + r^5/5 - ... - r^12/12
  double tail = 0.0;
  {
    double pw = r2.hi * r2.hi;  // r^4
    double acc = 0.0;
    const double coef[9] = {-1.0 / 4, 1.0 / 5, -1.0 / 6, 1.0 / 7, -1.0 / 8,
                            1.0 / 9,  -1.0 / 10, 1.0 / 11, -1.0 / 12};
    // Horner in r: acc = sum coef[k] r^k, k=0..8, times r^4
    for (int k = 8; k >= 0; --k) acc = acc * rh + coef[k];
    tail = acc * pw;
  }
  dd s = dd_add(r, dd_mul_d(r2, -0.5));
  s = dd_add(s, dd_div_d(r3, 3.0));
  s = dd_add(s, dd{tail, 0.0});
  // + (-log c_i)
  s = dd_add(s, dd{en.nlog_hi, en.nlog_lo});
  // + e * ln2 (e * kLn2Hi exact via two_prod)
  if (e != 0) {
    dd el = two_prod(double(e), kLn2Hi);
    el.lo += double(e) * kLn2Lo;
    el = quick_two_sum(el.hi, el.lo);
    s = dd_add(s, el);
  }
  return s;
}

// Correctly rounded log.
RSVD_HD inline double log_cr(double x, const Entry* table) {
  const dd s = log_dd(x, table);
  return s.hi + s.lo;
}

// Distance, in ulps of v = RN(s.hi + s.lo), from the exact value s to the
// nearest rounding midpoint (0.5 = s is representable, 0 = s is a midpoint).
// A log with error bound 0.5 + w ulps can differ from v only where this
// distance is below w.  *pow2 is set when |v| is a power of two (the spacing
// below v is half an ulp; callers treat those as near a midpoint).
RSVD_HD inline double midpoint_distance(dd s, double v, bool* pow2) {
  if (v == 0.0) {
    *pow2 = false;
    return 0.5;
  }
  int e;
  const double f = frexp(v, &e);  // v = f * 2^e, |f| in [0.5, 1)
  *pow2 = fabs(f) == 0.5;
  const double ulp = ldexp(1.0, e - 53);
  const double resid = (s.hi - v) + s.lo;  // s.hi - v is exact (v in {hi, hi +- ulp})
  return 0.5 - fabs(resid) / ulp;
}

// Exact-mode flag test for the polar sampler: true where glibc's log may
// round log(x) differently from v = RN(s).  glibc 2.39's log (both the FMA and
// the SSE2 ifunc variants) differs from the correctly rounded value only when
// the exact value lies within ~0.02 ulp of a rounding midpoint, and that
// distance bound scales like an ABSOLUTE error near |log x| ~ 1/16 (the
// table path's largest term), falling by ~2x per binade on either side.
// Window, in ulps of v, for |v| = f * 2^e (|f| in [0.5, 1)):
//   w(e) = 0.04 * 2^-|e + 3|
// i.e. >= 2x the largest midpoint distance of any glibc mismatch observed per
// binade over 1e9 reference polar inputs per ifunc variant
// (tools/logwindow.cpp; profiles/r02_logwindow.txt).  Flags ~1.7 % of inputs.
RSVD_HD inline bool log_near_midpoint(dd s, double v) {
  bool p2;
  const double d = midpoint_distance(s, v, &p2);
  if (p2) return true;
  int e;
  frexp(v, &e);
  const int k = e + 3 < 0 ? -(e + 3) : e + 3;
  const double w = k > 60 ? 0.0 : ldexp(0.04, -k);
  return d < w;
}

}  // namespace ddlog
}  // namespace rsvdb
