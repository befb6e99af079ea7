// rk_tableau.h — Butcher tableaux of the library (Table 1).
//
// The paper delegates the coefficients to Odeint; these are the standard
// published tables: explicit Euler, classic Runge–Kutta 4, Cash & Karp (1990) 5(4),
// Dormand & Prince (1980) 5(4) with FSAL.  Typed here independently of oracle/ (the two
// share no code); tests/test_abi.py cross-checks the two tables bit for bit.
#pragma once
#include <cstdint>

namespace rkb {

struct Rat {
    long long n, d;
};

struct Tableau {
    int s;          // stages
    int order;      // order of the propagated (b) solution
    int err_order;  // order of the embedded (bhat) solution, 0 if none
    Rat c[13];
    Rat a[13][13];  // strictly lower triangular
    Rat b[13];
    Rat bh[13];
};

__host__ __device__ constexpr Tableau tableau_of(int scheme) {
    switch (scheme) {
    case 0:  // explicit Euler
        return Tableau{1, 1, 0, {{0, 1}}, {{{0, 1}}}, {{1, 1}}, {{0, 1}}};
    case 1:  // classic RK4
        return Tableau{4, 4, 0,
                       {{0, 1}, {1, 2}, {1, 2}, {1, 1}},
                       {{{0, 1}}, {{1, 2}}, {{0, 1}, {1, 2}}, {{0, 1}, {0, 1}, {1, 1}}},
                       {{1, 6}, {1, 3}, {1, 3}, {1, 6}},
                       {{0, 1}}};
    case 2:  // Cash–Karp 5(4)
        return Tableau{6, 5, 4,
                       {{0, 1}, {1, 5}, {3, 10}, {3, 5}, {1, 1}, {7, 8}},
                       {{{0, 1}},
                        {{1, 5}},
                        {{3, 40}, {9, 40}},
                        {{3, 10}, {-9, 10}, {6, 5}},
                        {{-11, 54}, {5, 2}, {-70, 27}, {35, 27}},
                        {{1631, 55296}, {175, 512}, {575, 13824}, {44275, 110592}, {253, 4096}}},
                       {{37, 378}, {0, 1}, {250, 621}, {125, 594}, {0, 1}, {512, 1771}},
                       {{2825, 27648}, {0, 1}, {18575, 48384}, {13525, 55296}, {277, 14336}, {1, 4}}};
    case 3:  // Dormand–Prince 5(4), FSAL
        return Tableau{7, 5, 4,
                       {{0, 1}, {1, 5}, {3, 10}, {4, 5}, {8, 9}, {1, 1}, {1, 1}},
                       {{{0, 1}},
                        {{1, 5}},
                        {{3, 40}, {9, 40}},
                        {{44, 45}, {-56, 15}, {32, 9}},
                        {{19372, 6561}, {-25360, 2187}, {64448, 6561}, {-212, 729}},
                        {{9017, 3168}, {-355, 33}, {46732, 5247}, {49, 176}, {-5103, 18656}},
                        {{35, 384}, {0, 1}, {500, 1113}, {125, 192}, {-2187, 6784}, {11, 84}}},
                       {{35, 384}, {0, 1}, {500, 1113}, {125, 192}, {-2187, 6784}, {11, 84}, {0, 1}},
                       {{5179, 57600}, {0, 1}, {7571, 16695}, {393, 640}, {-92097, 339200}, {187, 2100}, {1, 40}}};
    case 4:  // Runge–Kutta–Fehlberg 7(8): b = 8th order (propagated), bh = 7th
        return Tableau{
            13, 8, 7,
            {{0, 1}, {2, 27}, {1, 9}, {1, 6}, {5, 12}, {1, 2}, {5, 6}, {1, 6}, {2, 3}, {1, 3}, {1, 1}, {0, 1}, {1, 1}},
            {{},
             {{2, 27}},
             {{1, 36}, {1, 12}},
             {{1, 24}, {0, 1}, {1, 8}},
             {{5, 12}, {0, 1}, {-25, 16}, {25, 16}},
             {{1, 20}, {0, 1}, {0, 1}, {1, 4}, {1, 5}},
             {{-25, 108}, {0, 1}, {0, 1}, {125, 108}, {-65, 27}, {125, 54}},
             {{31, 300}, {0, 1}, {0, 1}, {0, 1}, {61, 225}, {-2, 9}, {13, 900}},
             {{2, 1}, {0, 1}, {0, 1}, {-53, 6}, {704, 45}, {-107, 9}, {67, 90}, {3, 1}},
             {{-91, 108}, {0, 1}, {0, 1}, {23, 108}, {-976, 135}, {311, 54}, {-19, 60}, {17, 6}, {-1, 12}},
             {{2383, 4100}, {0, 1}, {0, 1}, {-341, 164}, {4496, 1025}, {-301, 82}, {2133, 4100}, {45, 82},
              {45, 164}, {18, 41}},
             {{3, 205}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {-6, 41}, {-3, 205}, {-3, 41}, {3, 41}, {6, 41}, {0, 1}},
             {{-1777, 4100}, {0, 1}, {0, 1}, {-341, 164}, {4496, 1025}, {-289, 82}, {2193, 4100}, {51, 82},
              {33, 164}, {12, 41}, {0, 1}, {1, 1}}},
            {{0, 1}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {34, 105}, {9, 35}, {9, 35}, {9, 280}, {9, 280}, {0, 1},
             {41, 840}, {41, 840}},
            {{41, 840}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {34, 105}, {9, 35}, {9, 35}, {9, 280}, {9, 280},
             {41, 840}, {0, 1}, {0, 1}}};
    case 5:  // explicit midpoint rule, order 2 (R-22)
        return Tableau{2, 2, 0, {{0, 1}, {1, 2}}, {{}, {{1, 2}}}, {{0, 1}, {1, 1}}, {{0, 1}}};
    case 6:  // modified midpoint = Odeint's modified_midpoint, Gragg with 2 substeps
             // h = dt/2: x1 = u + hF(u), x2 = u + 2hF(x1), u_new = (x1 + x2 + hF(x2))/2, i.e. the
             // 3-stage Butcher form c = (0, 1/2, 1), a21 = 1/2, a32 = 1, b = (1/4, 1/2, 1/4) (R-22)
        return Tableau{3, 2, 0, {{0, 1}, {1, 2}, {1, 1}}, {{}, {{1, 2}}, {{0, 1}, {1, 1}}},
                       {{1, 4}, {1, 2}, {1, 4}}, {{0, 1}}};
    default:
        return Tableau{0, 0, 0, {}, {}, {}, {}};
    }
}

__host__ __device__ constexpr bool rat_nz(Rat r) { return r.n != 0 && r.d != 0; }

// Exact e_j = b_j - bhat_j as a rational (rounded to double once by the caller, R-11).
__host__ __device__ constexpr long long gcd_ll(long long a, long long b) {
    a = a < 0 ? -a : a;
    b = b < 0 ? -b : b;
    while (b) {
        long long t = a % b;
        a = b;
        b = t;
    }
    return a ? a : 1;
}
__host__ __device__ constexpr Rat err_weight(const Tableau& T, int j) {
    if (T.err_order == 0) return Rat{0, 1};
    Rat x = T.b[j], y = T.bh[j];
    if (x.d == 0) x = Rat{0, 1};
    if (y.d == 0) y = Rat{0, 1};
    long long n = x.n * y.d - y.n * x.d, d = x.d * y.d;
    long long g = gcd_ll(n, d);
    return Rat{n / g, d / g};
}

inline double rat_double(Rat r) { return r.d == 0 ? 0.0 : (double)r.n / (double)r.d; }

// Adams–Bashforth k-step weights beta_j (j = 0 newest .. k-1 oldest), Table 1 multi-step row
// (P:L68): u_{n+1} = u_n + dt * sum_j beta_j f_{n-j}.  Standard values, reduced fractions.
__host__ __device__ constexpr Rat ab_beta(int k, int j) {
    constexpr Rat T[8][8] = {
        {{1, 1}},
        {{3, 2}, {-1, 2}},
        {{23, 12}, {-4, 3}, {5, 12}},
        {{55, 24}, {-59, 24}, {37, 24}, {-3, 8}},
        {{1901, 720}, {-1387, 360}, {109, 30}, {-637, 360}, {251, 720}},
        {{4277, 1440}, {-2641, 480}, {4991, 720}, {-3649, 720}, {959, 480}, {-95, 288}},
        {{198721, 60480}, {-18637, 2520}, {235183, 20160}, {-10754, 945}, {135713, 20160},
         {-5603, 2520}, {19087, 60480}},
        {{16083, 4480}, {-1152169, 120960}, {242653, 13440}, {-296053, 13440}, {2102243, 120960},
         {-115747, 13440}, {32863, 13440}, {-5257, 17280}},
    };
    return (k >= 1 && k <= 8 && j >= 0 && j < k) ? T[k - 1][j] : Rat{0, 1};
}

// Adams–Moulton k-term weights m_j (j = 0 weighs f_{n+1}, then f_n, f_{n-1} ...), the corrector
// of the Adams–Bashforth–Moulton row (R-26).  Standard values, reduced.
__host__ __device__ constexpr Rat am_beta(int k, int j) {
    constexpr Rat T[8][8] = {
        {{1, 1}},
        {{1, 2}, {1, 2}},
        {{5, 12}, {2, 3}, {-1, 12}},
        {{3, 8}, {19, 24}, {-5, 24}, {1, 24}},
        {{251, 720}, {323, 360}, {-11, 30}, {53, 360}, {-19, 720}},
        {{95, 288}, {1427, 1440}, {-133, 240}, {241, 720}, {-173, 1440}, {3, 160}},
        {{19087, 60480}, {2713, 2520}, {-15487, 20160}, {586, 945}, {-6737, 20160}, {263, 2520},
         {-863, 60480}},
        {{5257, 17280}, {139849, 120960}, {-4511, 4480}, {123133, 120960}, {-88547, 120960},
         {1537, 4480}, {-11351, 120960}, {275, 24192}},
    };
    return (k >= 1 && k <= 8 && j >= 0 && j < k) ? T[k - 1][j] : Rat{0, 1};
}

}  // namespace rkb
