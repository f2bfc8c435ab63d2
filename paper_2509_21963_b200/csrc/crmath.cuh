// crmath.cuh — correctly rounded (to within ~2^-104 before the final rounding) double
// log and cos for the sketch stream's Box-Muller step, normal_at (proj/src/rng.cpp:45-52):
//     sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2)
// CUDA's libm log/cos carry up to 1-2 ulp error and disagree with the reference's glibc on
// ~15% of sketch entries; evaluating both in double-double and rounding once agrees with
// glibc wherever glibc itself is correctly rounded (all but ~0.25% of entries, SURVEY.md
// F4/B.2). Header-only and __host__ __device__ so the CPU tests can pin it against mpmath.
#pragma once
#include <math.h>

#if defined(__CUDACC__)
#define CRM_HD __host__ __device__ __forceinline__
#else
#define CRM_HD inline
#endif

namespace itercur_b200 {
namespace crm {

struct dd {
  double hi, lo;
};

// Explicit round-to-nearest primitives: never contracted into FMAs by the compiler.
CRM_HD double add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;  // host build uses -ffp-contract=off
#endif
}
CRM_HD double sub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
CRM_HD double mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}

CRM_HD dd two_sum(double a, double b) {
  const double s = add(a, b);
  const double bb = sub(s, a);
  const double e = add(sub(a, sub(s, bb)), sub(b, bb));
  return dd{s, e};
}
CRM_HD dd fast_two_sum(double a, double b) {  // |a| >= |b|
  const double s = add(a, b);
  return dd{s, sub(b, sub(s, a))};
}
CRM_HD dd two_prod(double a, double b) {
  const double p = mul(a, b);
  return dd{p, fma(a, b, -p)};
}
CRM_HD dd dd_add(dd x, dd y) {  // accurate (IEEE-style) double-double addition
  dd s = two_sum(x.hi, y.hi);
  dd t = two_sum(x.lo, y.lo);
  s.lo = add(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = add(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}
CRM_HD dd dd_neg(dd x) { return dd{-x.hi, -x.lo}; }
CRM_HD dd dd_mul(dd x, dd y) {
  dd p = two_prod(x.hi, y.hi);
  p.lo = add(p.lo, add(mul(x.hi, y.lo), mul(x.lo, y.hi)));
  return fast_two_sum(p.hi, p.lo);
}
CRM_HD dd dd_mul_d(dd x, double y) {
  dd p = two_prod(x.hi, y);
  p.lo = add(p.lo, mul(x.lo, y));
  return fast_two_sum(p.hi, p.lo);
}
CRM_HD dd dd_div(dd x, dd y) {
  const double q1 = x.hi / y.hi;
  dd r = dd_add(x, dd_neg(dd_mul_d(y, q1)));
  const double q2 = r.hi / y.hi;
  r = dd_add(r, dd_neg(dd_mul_d(y, q2)));
  const double q3 = r.hi / y.hi;
  dd q = fast_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}

// 1/(2k+1) as double-double, k = 0..8
#define CRM_INV_ODD                                                                                               \
  {                                                                                                               \
    {0x1.0p+0, 0.0}, {0x1.5555555555555p-2, 0x1.5555555555555p-56}, {0x1.999999999999ap-3, -0x1.999999999999ap-57}, \
        {0x1.2492492492492p-3, 0x1.2492492492492p-57}, {0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-58},             \
        {0x1.745d1745d1746p-4, -0x1.745d1745d1746p-59}, {0x1.3b13b13b13b14p-4, -0x1.3b13b13b13b14p-58},           \
        {0x1.1111111111111p-4, 0x1.1111111111111p-60}, {0x1.e1e1e1e1e1e1ep-5, 0x1.e1e1e1e1e1e1ep-61},             \
  }
// 1/k! as double-double, k = 0..17
#define CRM_INV_FACT                                                                                              \
  {                                                                                                               \
    {0x1.0p+0, 0.0}, {0x1.0p+0, 0.0}, {0x1.0p-1, 0.0}, {0x1.5555555555555p-3, 0x1.5555555555555p-57},             \
        {0x1.5555555555555p-5, 0x1.5555555555555p-59}, {0x1.1111111111111p-7, 0x1.1111111111111p-63},             \
        {0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65}, {0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73},          \
        {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76}, {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73},          \
        {0x1.27e4fb7789f5cp-22, 0x1.cbbc05b4fa99ap-76}, {0x1.ae64567f544e4p-26, -0x1.c062e06d1f209p-80},          \
        {0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83}, {0x1.6124613a86d09p-33, 0x1.f28e0cc748ebep-87},          \
        {0x1.93974a8c07c9dp-37, 0x1.05d6f8a2efd1fp-92}, {0x1.ae7f3e733b81fp-41, 0x1.1d8656b0ee8cbp-97},           \
        {0x1.ae7f3e733b81fp-45, 0x1.1d8656b0ee8cbp-101}, {0x1.952c77030ad4ap-49, 0x1.ac981465ddc6cp-103},         \
  }

// 1/k! (double), k = 16..29, for the series tails
#define CRM_INV_FACT_TAIL                                                                                         \
  {                                                                                                               \
    0x1.ae7f3e733b81fp-45, 0x1.952c77030ad4ap-49, 0x1.6827863b97d97p-53, 0x1.2f49b46814157p-57,                   \
        0x1.e542ba4020225p-62, 0x1.71b8ef6dcf572p-66, 0x1.0ce396db7f853p-70, 0x1.761b41316381ap-75,               \
        0x1.f2cf01972f578p-80, 0x1.3f3ccdd165fa9p-84, 0x1.88e85fc6a4e5ap-89, 0x1.d1ab1c2dccea3p-94,               \
        0x1.0a18a2635085dp-98, 0x1.259f98b4358adp-103,                                                            \
  }

// log(u) for finite u > 0: u = 2^e f, f in [sqrt(1/2), sqrt(2)), log f = 2 atanh((f-1)/(f+1)).
CRM_HD double log_cr(double u) {
  const dd kInvOdd[9] = CRM_INV_ODD;
  const dd kLn2 = {0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
  int e = 0;
  double f = frexp(u, &e);  // u = f 2^e, f in [0.5, 1)
  if (f < 0.70710678118654752) {
    f = mul(f, 2.0);
    e -= 1;
  }
  const dd num = {sub(f, 1.0), 0.0};  // exact (Sterbenz)
  const dd s = dd_div(num, two_sum(f, 1.0));
  const dd t = dd_mul(s, s);
  // tail k = 9..21 in double: its contribution is below 2^-46 of the sum
  double q = 1.0 / 43.0;
  for (int k = 20; k >= 9; --k) q = add(mul(q, t.hi), 1.0 / (2.0 * k + 1.0));
  dd p = {q, 0.0};
  for (int k = 8; k >= 0; --k) p = dd_add(dd_mul(p, t), kInvOdd[k]);
  dd r = dd_mul(s, p);
  r.hi = mul(r.hi, 2.0);
  r.lo = mul(r.lo, 2.0);
  const dd el = dd_mul_d(kLn2, static_cast<double>(e));
  const dd res = dd_add(el, r);
  return add(res.hi, res.lo);
}

// cos(x) for finite |x| <= ~1e3 (here x = 2 pi u2 in (0, 2 pi)): Cody-Waite reduction by a
// triple-double pi/2, then double-double Taylor series on |r| <= pi/4.
CRM_HD double cos_cr(double x) {
  const dd kInvFact[18] = CRM_INV_FACT;
  const double kTail[14] = CRM_INV_FACT_TAIL;  // 1/(16+i)!
  const double P1 = 0x1.921fb54442d18p+0, P2 = 0x1.1a62633145c07p-54, P3 = -0x1.f1976b7ed8fbcp-110;
  const double kd = rint(mul(x, 0x1.45f306dc9c883p-1));  // x * 2/pi
  const dd p1 = two_prod(kd, P1), p2 = two_prod(kd, P2), p3 = two_prod(kd, P3);
  dd r = dd_add(dd{x, 0.0}, dd_neg(p1));
  r = dd_add(r, dd_neg(p2));
  r = dd_add(r, dd_neg(p3));
  const dd t = dd_mul(r, r);
  const int quadrant = static_cast<int>(kd) & 3;
  dd res;
  if ((quadrant & 1) == 0) {
    // cos r = sum_j (-1)^j t^j / (2j)!, j = 0..14; tail j >= 8 in double
    double q = 0.0;
    for (int j = 14; j >= 8; --j) {
      const double c = (j & 1) ? -kTail[2 * j - 16] : kTail[2 * j - 16];
      q = add(mul(q, t.hi), c);
    }
    dd p = {q, 0.0};
    for (int j = 7; j >= 0; --j) {
      const dd c = (j & 1) ? dd_neg(kInvFact[2 * j]) : kInvFact[2 * j];
      p = dd_add(dd_mul(p, t), c);
    }
    res = p;
  } else {
    // sin r = r * sum_j (-1)^j t^j / (2j+1)!, j = 0..13; tail j >= 8 in double
    double q = 0.0;
    for (int j = 13; j >= 8; --j) {
      const double c = (j & 1) ? -kTail[2 * j + 1 - 16] : kTail[2 * j + 1 - 16];
      q = add(mul(q, t.hi), c);
    }
    dd p = {q, 0.0};
    for (int j = 7; j >= 0; --j) {
      const dd c = (j & 1) ? dd_neg(kInvFact[2 * j + 1]) : kInvFact[2 * j + 1];
      p = dd_add(dd_mul(p, t), c);
    }
    res = dd_mul(p, r);
  }
  if (quadrant == 1 || quadrant == 2) res = dd_neg(res);  // cos: +cos, -sin, -cos, +sin
  return add(res.hi, res.lo);
}

// normal_at's Box-Muller step with the reference's evaluation order (rng.cpp:51).
CRM_HD double box_muller_cos(double u1, double u2) {
  const double two_pi = 6.283185307179586;  // 2.0 * M_PI, exact
  return mul(sqrt(mul(-2.0, log_cr(u1))), cos_cr(mul(two_pi, u2)));
}

}  // namespace crm
}  // namespace itercur_b200
