// rk_ddmath.cuh — double-double pow for the device-resident step-size controller.
//
// The host controller (R-12) computes dt * (0.9 * pow(E, -1/p)) with libm's pow,
// which is correctly rounded except within ~2^-15 ulp of a rounding midpoint.  CUDA's pow is
// only 2-ulp accurate, so a device copy of the controller would drift from the host (and the
// oracle) by an ulp of dt now and then.  pow_dd evaluates x^y = exp(y*log x) in double-double
// (~100 bits) and rounds once, so it returns the correctly rounded value except in the same
// astronomically rare near-midpoint cases (R-27).  Only the controller's arguments
// occur: x >= 5^-8 or x > 1 (x = +inf allowed), y in [-1, -1/8].
#pragma once
#include <cuda_runtime.h>

namespace rkb {

struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd dd_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd dd_quick(double a, double b) {  // |a| >= |b|
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd dd_two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = dd_two_sum(a.hi, b.hi);
    const dd t = dd_two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = dd_quick(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return dd_quick(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = dd_two_prod(a.hi, b.hi);
    p.lo = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
    return dd_quick(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = dd_two_prod(a.hi, b);
    p.lo = __dadd_rn(p.lo, __dmul_rn(a.lo, b));
    return dd_quick(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
    const double q1 = __ddiv_rn(a.hi, b.hi);
    dd r = dd_add(a, dd_neg(dd_mul_d(b, q1)));
    const double q2 = __ddiv_rn(r.hi, b.hi);
    r = dd_add(r, dd_neg(dd_mul_d(b, q2)));
    const double q3 = __ddiv_rn(r.hi, b.hi);
    return dd_add(dd_quick(q1, q2), dd{q3, 0.0});
}

__device__ __forceinline__ dd dd_ln2() { return {0.6931471805599453094, 2.319046813846299558e-17}; }

// log x for finite x > 0 (normal): x = m 2^e, m in [1/sqrt2, sqrt2),
// log m = 2 atanh(s) = 2 s (1 + s^2/3 + s^4/5 + ...), s = (m-1)/(m+1), |s| <= 0.1716.
__device__ inline dd dd_log(double x) {
    int e;
    double m = frexp(x, &e);  // m in [0.5, 1)
    if (m < 0.70710678118654752440) {
        m = __dmul_rn(m, 2.0);
        --e;
    }
    const dd s = dd_div(dd{__dsub_rn(m, 1.0), 0.0}, dd_two_sum(m, 1.0));
    const dd s2 = dd_mul(s, s);
    constexpr dd ODD[25] = {  // 1/(2n+1) as double-doubles (exact rationals, rounded twice)
        {1.0, 0.0},
        {0.3333333333333333, 1.850371707708594e-17},
        {0.2, -1.1102230246251566e-17},
        {0.14285714285714285, 7.93016446160826e-18},
        {0.1111111111111111, 6.1679056923619804e-18},
        {0.09090909090909091, -2.523234146875356e-18},
        {0.07692307692307693, -4.270088556250602e-18},
        {0.06666666666666667, 9.251858538542971e-19},
        {0.058823529411764705, 8.163404592832033e-19},
        {0.05263157894736842, 2.921639538487254e-18},
        {0.047619047619047616, 2.64338815386942e-18},
        {0.043478260869565216, 1.206764157201257e-18},
        {0.04, -8.326672684688674e-19},
        {0.037037037037037035, 2.05596856412066e-18},
        {0.034482758620689655, 4.785444071660157e-19},
        {0.03225806451612903, 8.953411488912552e-19},
        {0.030303030303030304, -8.410780489584519e-19},
        {0.02857142857142857, 8.921435019309293e-19},
        {0.02702702702702703, -1.50030138462859e-18},
        {0.02564102564102564, 8.896017825522087e-19},
        {0.024390243902439025, -8.46206573647223e-19},
        {0.023255813953488372, 3.2273925134452225e-19},
        {0.022222222222222223, -8.480870326997723e-19},
        {0.02127659574468085, 5.167261417803255e-19},
        {0.02040816326530612, 1.6285159162231251e-18}};
    dd P = ODD[24];  // 25 terms: s2^25/51 < 2^-128
#pragma unroll
    for (int n = 23; n >= 0; --n) P = dd_add(dd_mul(P, s2), ODD[n]);
    const dd lm = dd_mul_d(dd_mul(s, P), 2.0);
    return dd_add(dd_mul_d(dd_ln2(), (double)e), lm);
}

// exp z for a double-double z with z.hi in about [-745, 709]: z = k ln2 + r, r' = r/2^10,
// exp(r') - 1 by Taylor (11 terms), then 10 squarings of (1 + m) in the form 2m + m^2.
__device__ inline double dd_exp_round(dd z) {
    const double k = rint(__ddiv_rn(z.hi, 0.6931471805599453094));
    dd r = dd_add(z, dd_neg(dd_mul_d(dd_ln2(), k)));
    r = {ldexp(r.hi, -10), ldexp(r.lo, -10)};
    constexpr dd INV[12] = {  // 1/n, n = 1..12, as double-doubles
        {1.0, 0.0},
        {0.5, 0.0},
        {0.3333333333333333, 1.850371707708594e-17},
        {0.25, 0.0},
        {0.2, -1.1102230246251566e-17},
        {0.16666666666666666, 9.25185853854297e-18},
        {0.14285714285714285, 7.93016446160826e-18},
        {0.125, 0.0},
        {0.1111111111111111, 6.1679056923619804e-18},
        {0.1, -5.551115123125783e-18},
        {0.09090909090909091, -2.523234146875356e-18},
        {0.08333333333333333, 4.625929269271485e-18}};
    dd Q = {1.0, 0.0};
#pragma unroll
    for (int n = 12; n >= 2; --n) Q = dd_add(dd{1.0, 0.0}, dd_mul(dd_mul(r, Q), INV[n - 1]));
    dd m = dd_mul(r, Q);  // exp(r') - 1
    for (int i = 0; i < 10; ++i) m = dd_add(dd_mul_d(m, 2.0), dd_mul(m, m));
    const dd v = dd_add(dd{1.0, 0.0}, m);
    // scale by 2^k: exact unless the result is subnormal (not reached by the controller)
    return ldexp(__dadd_rn(v.hi, v.lo), (int)k);
}

// x^y rounded once from ~100 bits (the controller's arguments: x > 0, y < 0).
__device__ inline double pow_dd(double x, double y) {
    if (isinf(x)) return 0.0;
    if (x == 1.0) return 1.0;
    return dd_exp_round(dd_mul_d(dd_log(x), y));
}

// The host step adjusters (rk_runtime.cu step_adjust / step_adjust_spec; R-12, R-28)
// on the device, with pow_dd for libm's pow: e_rej / e_acc are the host-computed exponents,
// emin = 5^-p (Odeint's clamp).  Used by the device-resident adaptive loops (vector: K1 loop,
// grid: K5 loop); every thread of a grid evaluates it on the same inputs -> the same decision.
static __device__ __noinline__ double step_adjust_dev(double E, double e_rej, double e_acc, double emin, int ctrl,
                                                      double dt, int* ok) {
    if (ctrl == 1) {  // SPEC's elementary controller (R-28): always rescale
        if (E <= 1.0) {
            double fac = E == 0.0 ? 5.0 : __dmul_rn(0.9, pow_dd(E, e_acc));
            if (fac < 0.2) fac = 0.2;
            if (fac > 5.0) fac = 5.0;
            *ok = 1;
            return __dmul_rn(dt, fac);
        }
        double fac = __dmul_rn(0.9, pow_dd(E, e_rej));
        if (fac < 0.2) fac = 0.2;
        *ok = 0;
        return __dmul_rn(dt, fac);
    }
    if (E > 1.0) {
        double fac = __dmul_rn(0.9, pow_dd(E, e_rej));
        if (fac < 0.2) fac = 0.2;
        *ok = 0;
        return __dmul_rn(dt, fac);
    }
    *ok = 1;
    if (E < 0.5) {
        double Ec = emin;
        if (E > Ec) Ec = E;
        return __dmul_rn(dt, __dmul_rn(0.9, pow_dd(Ec, e_acc)));
    }
    return dt;
}

}  // namespace rkb
