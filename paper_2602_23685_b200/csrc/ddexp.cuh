// ddexp.cuh -- exp(x) rounded correctly to fp64, for the SA acceptance test
// `rng.random() < math.exp(-(z_c - z) / T)` (alns.py:588).
//
// CUDA's exp() is accurate to <= 1 ulp, so its result can sit one ulp away
// from the host libm's; the comparison with the uniform draw then differs
// whenever the draw lands in between.  This version evaluates exp in
// double-double (~2^-93 relative error before the final rounding) and rounds
// once, so it returns the correctly rounded value except when exp(x) lies
// within 2^-93 of a rounding midpoint.
//
// Note on the host side: glibc's exp (what CPython's math.exp calls) is not
// correctly rounded either -- measured here, it differs from the correctly
// rounded value on 139 of 200,000 inputs in [-30, 0] (0.07 %).  A device/host
// disagreement of the SA decision therefore needs BOTH a glibc misrounding at
// x AND a uniform draw inside that one ulp (p ~ 2^-53): < 2^-63 per test.
//
// Method: k = rint(x / ln2), r = x - k ln2 with ln2 split into three parts
// (40 + 40 + 53 bits: k*L1 and k*L2 are exact), r' = r / 2^10, expm1(r') by a
// degree-9 Taylor polynomial in double-double, ten squarings in expm1 form
// (E <- 2E + E^2), then 1 + E scaled by 2^k.
#pragma once
#include <math.h>

namespace ddexp {

struct dd {
    double h, l;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd add(dd a, dd b) {
    dd s = two_sum(a.h, b.h);
    const dd t = two_sum(a.l, b.l);
    s.l = __dadd_rn(s.l, t.h);
    s = quick_two_sum(s.h, s.l);
    s.l = __dadd_rn(s.l, t.l);
    return quick_two_sum(s.h, s.l);
}
__device__ __forceinline__ dd mul(dd a, dd b) {
    dd p = two_prod(a.h, b.h);
    p.l = __dadd_rn(p.l, __dadd_rn(__dmul_rn(a.h, b.l), __dmul_rn(a.l, b.h)));
    return quick_two_sum(p.h, p.l);
}

// 1/n! for n = 2..9 as double-double (hi, lo)
__device__ __constant__ const double kInvFact[8][2] = {
    {0x1.0000000000000p-1, 0.0},
    {0x1.5555555555555p-3, 0x1.5555555555555p-57},
    {0x1.5555555555555p-5, 0x1.5555555555555p-59},
    {0x1.1111111111111p-7, 0x1.1111111111111p-63},
    {0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65},
    {0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73},
    {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76},
    {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73},
};

__device__ inline double exp_cr(double x) {
    // outside the normal-result range (and NaN / inf) the libdevice result is
    // what any uniform draw compares against identically: 0 < u only if u == 0
    if (!(x > -708.0) || !(x < 709.0)) return exp(x);
    const double L1 = 0x1.62e42fefa2000p-1, L2 = 0x1.9ef35793c6000p-41, L3 = 0x1.673007e5ed5e8p-81;
    const double k = rint(__dmul_rn(x, 0x1.71547652b82fep+0));
    const double s = __dsub_rn(x, __dmul_rn(k, L1));     // exact (Sterbenz)
    dd r = two_sum(s, -__dmul_rn(k, L2));                 // k*L2 exact
    r = add(r, dd{-__dmul_rn(k, L3), 0.0});
    r.h = ldexp(r.h, -10);
    r.l = ldexp(r.l, -10);
    // expm1(r) = r + r^2/2! + ... + r^9/9!  (Horner on the 1/n! tail)
    dd p = {kInvFact[7][0], kInvFact[7][1]};
    for (int i = 6; i >= 0; --i) p = add(mul(p, r), dd{kInvFact[i][0], kInvFact[i][1]});
    dd e = add(mul(mul(p, r), r), r);
    for (int i = 0; i < 10; ++i) e = add(add(e, e), mul(e, e));
    const dd one_e = add(dd{1.0, 0.0}, e);
    const int ki = (int)k;
    return ldexp(__dadd_rn(one_e.h, one_e.l), ki);
}

}  // namespace ddexp
