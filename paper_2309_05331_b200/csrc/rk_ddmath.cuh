// rk_ddmath.cuh — correctly rounded pow for the step-size controller (host AND device).
//
// The controller (R-12 / R-28) computes dt * (0.9 * pow(E, -1/p)).  Its pow is read
// as the correctly rounded x^y (R-27): libm's pow is not always correctly rounded (glibc 2.39
// misses ~0.05-0.1 % of controller arguments by an ulp) and CUDA's device pow is 2-ulp
// accurate, so either would let the host loop, the device-resident loops and the oracle drift
// apart by an ulp of dt.  pow_dd evaluates x^y = exp(y*log x) in double-double (~100 bits,
// relative error below ~2^-98 for the controller's arguments) and rounds once, so it returns
// the correctly rounded value unless x^y lies within ~2^-98 of a rounding midpoint.  The same
// code runs on the host (rk_runtime.cu's controller) and on the device (K1 / K5 loops), with
// IEEE operations in the same order on both: identical bits.  The oracle computes the same
// reading independently (binary128 powq in the test oracle).  Only the controller's
// arguments occur: x >= 5^-8 or x > 1 (x = +inf, x = 0 allowed), y in [-1, -1/8].
#pragma once
#include <cuda_runtime.h>

#include <cmath>

namespace rkb {

// IEEE round-to-nearest operations: device intrinsics (never contracted), host operators
// (compiled with -ffp-contract=off, SSE2 doubles) and the C library's exact fma.
#ifdef __CUDA_ARCH__
#define DD_ADD(a, b) __dadd_rn(a, b)
#define DD_SUB(a, b) __dsub_rn(a, b)
#define DD_MUL(a, b) __dmul_rn(a, b)
#define DD_DIV(a, b) __ddiv_rn(a, b)
#define DD_FMA(a, b, c) __fma_rn(a, b, c)
#else
#define DD_ADD(a, b) ((a) + (b))
#define DD_SUB(a, b) ((a) - (b))
#define DD_MUL(a, b) ((a) * (b))
#define DD_DIV(a, b) ((a) / (b))
#define DD_FMA(a, b, c) ::fma(a, b, c)
#endif
#define DD_HD __host__ __device__

struct dd {
    double hi, lo;
};

DD_HD inline dd dd_two_sum(double a, double b) {
    const double s = DD_ADD(a, b);
    const double bb = DD_SUB(s, a);
    const double e = DD_ADD(DD_SUB(a, DD_SUB(s, bb)), DD_SUB(b, bb));
    return {s, e};
}
DD_HD inline dd dd_quick(double a, double b) {  // |a| >= |b|
    const double s = DD_ADD(a, b);
    return {s, DD_SUB(b, DD_SUB(s, a))};
}
DD_HD inline dd dd_two_prod(double a, double b) {
    const double p = DD_MUL(a, b);
    return {p, DD_FMA(a, b, -p)};
}
DD_HD inline dd dd_add(dd a, dd b) {
    dd s = dd_two_sum(a.hi, b.hi);
    const dd t = dd_two_sum(a.lo, b.lo);
    s.lo = DD_ADD(s.lo, t.hi);
    s = dd_quick(s.hi, s.lo);
    s.lo = DD_ADD(s.lo, t.lo);
    return dd_quick(s.hi, s.lo);
}
DD_HD inline dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
DD_HD inline dd dd_mul(dd a, dd b) {
    dd p = dd_two_prod(a.hi, b.hi);
    p.lo = DD_ADD(p.lo, DD_ADD(DD_MUL(a.hi, b.lo), DD_MUL(a.lo, b.hi)));
    return dd_quick(p.hi, p.lo);
}
DD_HD inline dd dd_mul_d(dd a, double b) {
    dd p = dd_two_prod(a.hi, b);
    p.lo = DD_ADD(p.lo, DD_MUL(a.lo, b));
    return dd_quick(p.hi, p.lo);
}
DD_HD inline dd dd_div(dd a, dd b) {
    const double q1 = DD_DIV(a.hi, b.hi);
    dd r = dd_add(a, dd_neg(dd_mul_d(b, q1)));
    const double q2 = DD_DIV(r.hi, b.hi);
    r = dd_add(r, dd_neg(dd_mul_d(b, q2)));
    const double q3 = DD_DIV(r.hi, b.hi);
    return dd_add(dd_quick(q1, q2), dd{q3, 0.0});
}

DD_HD inline dd dd_ln2() { return {0.6931471805599453094, 2.319046813846299558e-17}; }

// log x for finite x > 0 (normal): x = m 2^e, m in [1/sqrt2, sqrt2),
// log m = 2 atanh(s) = 2 s (1 + s^2/3 + s^4/5 + ...), s = (m-1)/(m+1), |s| <= 0.1716.
DD_HD inline dd dd_log(double x) {
    int e;
    double m = frexp(x, &e);  // m in [0.5, 1)
    if (m < 0.70710678118654752440) {
        m = DD_MUL(m, 2.0);
        --e;
    }
    const dd s = dd_div(dd{DD_SUB(m, 1.0), 0.0}, dd_two_sum(m, 1.0));
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
DD_HD inline double dd_exp_round(dd z) {
    const double k = rint(DD_DIV(z.hi, 0.6931471805599453094));
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
    return ldexp(DD_ADD(v.hi, v.lo), (int)k);
}

// x^y rounded once from ~100 bits (the controller's arguments: x >= 0, y < 0).
DD_HD inline double pow_dd(double x, double y) {
    if (isinf(x)) return 0.0;
    if (x == 0.0) return INFINITY;  // y < 0 (SPEC's E = 0: the grow cap applies)
    if (x == 1.0) return 1.0;
    return dd_exp_round(dd_mul_d(dd_log(x), y));
}

// The step adjusters (R-12 Odeint, R-28 SPEC) with the correctly rounded pow:
// e_rej / e_acc are the exponents -1/(q-1) (SPEC: -1/(p-1)) and -1/p, emin = 5^-p (Odeint's
// clamp, pow_dd(5, -p)).  Used by the host loop (rk_runtime.cu) and the device-resident loops
// (vector: K1 loop, grid: K5 loop; every thread evaluates it on the same inputs -> the same
// decision).
#ifdef __CUDA_ARCH__
#define DD_NOINLINE __noinline__
#else
#define DD_NOINLINE
#endif
static DD_HD DD_NOINLINE double step_adjust_dev(double E, double e_rej, double e_acc, double emin, int ctrl,
                                                      double dt, int* ok) {
    if (ctrl == 1) {  // SPEC's elementary controller (R-28): always rescale
        if (E <= 1.0) {
            double fac = E == 0.0 ? 5.0 : DD_MUL(0.9, pow_dd(E, e_acc));
            if (fac < 0.2) fac = 0.2;
            if (fac > 5.0) fac = 5.0;
            *ok = 1;
            return DD_MUL(dt, fac);
        }
        double fac = DD_MUL(0.9, pow_dd(E, e_rej));
        if (fac < 0.2) fac = 0.2;
        *ok = 0;
        return DD_MUL(dt, fac);
    }
    if (E > 1.0) {
        double fac = DD_MUL(0.9, pow_dd(E, e_rej));
        if (fac < 0.2) fac = 0.2;
        *ok = 0;
        return DD_MUL(dt, fac);
    }
    *ok = 1;
    if (E < 0.5) {
        double Ec = emin;
        if (E > Ec) Ec = E;
        return DD_MUL(dt, DD_MUL(0.9, pow_dd(Ec, e_acc)));
    }
    return dt;
}

}  // namespace rkb
