/*
 * rk_oracle.c — plain fp64 CPU oracle.  TEST INFRASTRUCTURE ONLY (see rk_oracle.h):
 * only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may use it.
 *
 * Each function cites the passage it follows.  The method computes (up to rounding
 * order) a textbook explicit Runge–Kutta step of the semi-discrete ODE system, so the
 * oracle is that definition written out: every stage value Y_i and every k_i is
 * materialised over the whole global array, sums run left to right and skip zero
 * coefficients (R-17), no blocking, fusion or reordering.
 *
 * Pins: tests/test_oracle_*.py (closed forms, order conditions, invariants).
 * Controller constants: "parity unpinned" against Odeint itself (R-12);
 * pinned internally by the SURVEY App. B accept/reject magnitudes and tie-break tests.
 */
#include "rk_oracle.h"

#include <float.h>
#include <math.h>
#include <quadmath.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------
 * Butcher tableaux (exact rationals).  Table 1 names the schemes; the
 * paper delegates the coefficients to Odeint, so these are the standard
 * published tables (Euler; classic RK4; Cash & Karp 1990; Dormand & Prince 1980),
 * typed here independently of the CUDA library's copy.
 * --------------------------------------------------------------------------- */
typedef struct { int64_t n, d; } rat;
#define MAXS 13
typedef struct {
    int s, order, err_order, has_err;
    rat c[MAXS];
    rat a[MAXS][MAXS];
    rat b[MAXS];
    rat bh[MAXS]; /* embedded (lower-order) weights, zero if !has_err */
} tableau;

static const tableau TAB_EULER = {
    1, 1, 0, 0,
    {{0, 1}},
    {{{0, 1}}},
    {{1, 1}},
    {{0, 1}},
};

/* Explicit midpoint rule (order 2): an Euler half step, then the full step with the midpoint
 * slope.  Kept under its own name; Table 1's "modified midpoint" is TAB_MODIFIED_MIDPOINT
 * below (R-22). */
static const tableau TAB_MIDPOINT = {
    2, 2, 0, 0,
    {{0, 1}, {1, 2}},
    {{{0, 1}},
     {{1, 2}}},
    {{0, 1}, {1, 1}},
    {{0, 1}},
};

/* Modified midpoint (Table 1, order 2) = Odeint's modified_midpoint, Gragg's scheme with
 * its default n = 2 substeps of h = dt/2 (R-22):
 *     x1 = u + h F(u),  x2 = u + 2h F(x1),  u_new = (x1 + x2 + h F(x2)) / 2.
 * Substituting x1 and x2 gives the 3-stage Butcher form used here (R-17 arithmetic):
 *     Y2 = u + (dt/2) k1,  Y3 = u + dt k2,  u_new = u + (dt/4) k1 + (dt/2) k2 + (dt/4) k3. */
static const tableau TAB_MODIFIED_MIDPOINT = {
    3, 2, 0, 0,
    {{0, 1}, {1, 2}, {1, 1}},
    {{{0, 1}},
     {{1, 2}},
     {{0, 1}, {1, 1}}},
    {{1, 4}, {1, 2}, {1, 4}},
    {{0, 1}},
};

static const tableau TAB_RK4 = {
    4, 4, 0, 0,
    {{0, 1}, {1, 2}, {1, 2}, {1, 1}},
    {{{0, 1}},
     {{1, 2}},
     {{0, 1}, {1, 2}},
     {{0, 1}, {0, 1}, {1, 1}}},
    {{1, 6}, {1, 3}, {1, 3}, {1, 6}},
    {{0, 1}},
};

static const tableau TAB_CK54 = {
    6, 5, 4, 1,
    {{0, 1}, {1, 5}, {3, 10}, {3, 5}, {1, 1}, {7, 8}},
    {{{0, 1}},
     {{1, 5}},
     {{3, 40}, {9, 40}},
     {{3, 10}, {-9, 10}, {6, 5}},
     {{-11, 54}, {5, 2}, {-70, 27}, {35, 27}},
     {{1631, 55296}, {175, 512}, {575, 13824}, {44275, 110592}, {253, 4096}}},
    {{37, 378}, {0, 1}, {250, 621}, {125, 594}, {0, 1}, {512, 1771}},
    {{2825, 27648}, {0, 1}, {18575, 48384}, {13525, 55296}, {277, 14336}, {1, 4}},
};

static const tableau TAB_DOPRI5 = {
    7, 5, 4, 1,
    {{0, 1}, {1, 5}, {3, 10}, {4, 5}, {8, 9}, {1, 1}, {1, 1}},
    {{{0, 1}},
     {{1, 5}},
     {{3, 40}, {9, 40}},
     {{44, 45}, {-56, 15}, {32, 9}},
     {{19372, 6561}, {-25360, 2187}, {64448, 6561}, {-212, 729}},
     {{9017, 3168}, {-355, 33}, {46732, 5247}, {49, 176}, {-5103, 18656}},
     {{35, 384}, {0, 1}, {500, 1113}, {125, 192}, {-2187, 6784}, {11, 84}}},
    {{35, 384}, {0, 1}, {500, 1113}, {125, 192}, {-2187, 6784}, {11, 84}, {0, 1}},
    {{5179, 57600}, {0, 1}, {7571, 16695}, {393, 640}, {-92097, 339200}, {187, 2100}, {1, 40}},
};

/* Runge–Kutta–Fehlberg 7(8) (Fehlberg 1968).  b = 8th-order weights
 * (propagated, R-11), bh = 7th-order embedded weights. */
static const tableau TAB_RKF78 = {
    13, 8, 7, 1,
    {{0, 1}, {2, 27}, {1, 9}, {1, 6}, {5, 12}, {1, 2}, {5, 6}, {1, 6}, {2, 3}, {1, 3}, {1, 1}, {0, 1}, {1, 1}},
    {{{0, 1}},
     {{2, 27}},
     {{1, 36}, {1, 12}},
     {{1, 24}, {0, 1}, {1, 8}},
     {{5, 12}, {0, 1}, {-25, 16}, {25, 16}},
     {{1, 20}, {0, 1}, {0, 1}, {1, 4}, {1, 5}},
     {{-25, 108}, {0, 1}, {0, 1}, {125, 108}, {-65, 27}, {125, 54}},
     {{31, 300}, {0, 1}, {0, 1}, {0, 1}, {61, 225}, {-2, 9}, {13, 900}},
     {{2, 1}, {0, 1}, {0, 1}, {-53, 6}, {704, 45}, {-107, 9}, {67, 90}, {3, 1}},
     {{-91, 108}, {0, 1}, {0, 1}, {23, 108}, {-976, 135}, {311, 54}, {-19, 60}, {17, 6}, {-1, 12}},
     {{2383, 4100}, {0, 1}, {0, 1}, {-341, 164}, {4496, 1025}, {-301, 82}, {2133, 4100}, {45, 82}, {45, 164}, {18, 41}},
     {{3, 205}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {-6, 41}, {-3, 205}, {-3, 41}, {3, 41}, {6, 41}, {0, 1}},
     {{-1777, 4100}, {0, 1}, {0, 1}, {-341, 164}, {4496, 1025}, {-289, 82}, {2193, 4100}, {51, 82}, {33, 164}, {12, 41}, {0, 1}, {1, 1}}},
    {{0, 1}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {34, 105}, {9, 35}, {9, 35}, {9, 280}, {9, 280}, {0, 1}, {41, 840}, {41, 840}},
    {{41, 840}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {34, 105}, {9, 35}, {9, 35}, {9, 280}, {9, 280}, {41, 840}, {0, 1}, {0, 1}},
};

static const tableau* get_tableau(int scheme) {
    switch (scheme) {
    case ORC_EULER: return &TAB_EULER;
    case ORC_RK4: return &TAB_RK4;
    case ORC_CASH_KARP54: return &TAB_CK54;
    case ORC_DOPRI5: return &TAB_DOPRI5;
    case ORC_RKF78: return &TAB_RKF78;
    case ORC_MIDPOINT: return &TAB_MIDPOINT;
    case ORC_MODIFIED_MIDPOINT: return &TAB_MODIFIED_MIDPOINT;
    default: return NULL;
    }
}

static double rat_to_double(rat r) { return r.d == 0 ? 0.0 : (double)r.n / (double)r.d; }

/* gcd for the exact error weight e_j = b_j - bhat_j (rounded once, R-11). */
static int64_t gcd64(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a ? a : 1;
}
static rat rat_sub(rat x, rat y) {
    /* denominators here are < 2^20, so the cross products fit in int64 */
    int64_t n = x.n * y.d - y.n * x.d, d = x.d * y.d;
    int64_t g = gcd64(n, d);
    rat r = {n / g, d / g};
    if (r.d < 0) { r.n = -r.n; r.d = -r.d; }
    return r;
}

int orc_tableau(int scheme, int64_t* a_num, int64_t* a_den, int64_t* b_num, int64_t* b_den,
                int64_t* bh_num, int64_t* bh_den, int64_t* c_num, int64_t* c_den, int* order,
                int* err_order) {
    const tableau* T = get_tableau(scheme);
    if (!T) return -1;
    int s = T->s;
    for (int i = 0; i < s; ++i) {
        for (int j = 0; j < s; ++j) {
            rat r = (j < i) ? T->a[i][j] : (rat){0, 1};
            if (r.d == 0) r = (rat){0, 1};
            a_num[i * s + j] = r.n;
            a_den[i * s + j] = r.d;
        }
        b_num[i] = T->b[i].n; b_den[i] = T->b[i].d;
        rat bh = T->has_err ? T->bh[i] : (rat){0, 1};
        bh_num[i] = bh.n; bh_den[i] = bh.d ? bh.d : 1;
        c_num[i] = T->c[i].n; c_den[i] = T->c[i].d;
    }
    *order = T->order;
    *err_order = T->err_order;
    return s;
}

/* ------------------------------------------------------------------------------
 * Right-hand sides.
 * --------------------------------------------------------------------------- */

/* Eq. 1a: df/dt = f; generalised to du/dt = lambda*u (R-9). */
static void rhs_exp(int64_t count, const double* u, double* f, double lambda) {
    for (int64_t i = 0; i < count; ++i) f[i] = lambda * u[i];
}

/* Eq. 1b: df/dt = f(1 - f). */
static void rhs_logistic(int64_t count, const double* u, double* f) {
    for (int64_t i = 0; i < count; ++i) f[i] = u[i] * (1.0 - u[i]);
}

/* Gray–Scott, Listing 2 lines 25-26, parameters P:L150 (R-1, R-2):
 *   f0 = d1*Lap(C0) - C0*C1*C1 + F - F*C0
 *   f1 = d2*Lap(C1) + C0*C1*C1 - (F+K)*C1
 * evaluated in C++ left-to-right order.  Lap = 7-point second-order central
 * difference in difference form (R-3), periodic in x, y, z. */
static void rhs_gray_scott(const orc_problem* p, const double* u, double* f) {
    const int64_t nx = p->nx, ny = p->ny, nz = p->nz;
    const int64_t plane = nx * ny;       /* one component of one z-plane */
    const int64_t zstride = 2 * plane;   /* layout [z][c][y][x] */
    const double inv_h2 = 1.0 / (p->h * p->h);
    const double FK = p->F + p->K;
    for (int64_t z = 0; z < nz; ++z) {
        const int64_t zm = (z + nz - 1) % nz, zp = (z + 1) % nz;
        for (int64_t y = 0; y < ny; ++y) {
            const int64_t ym = (y + ny - 1) % ny, yp = (y + 1) % ny;
            for (int64_t x = 0; x < nx; ++x) {
                const int64_t xm = (x + nx - 1) % nx, xp = (x + 1) % nx;
                double L[2], cc[2];
                for (int c = 0; c < 2; ++c) {
                    const double* v = u + c * plane;
                    const double ctr = v[z * zstride + y * nx + x];
                    double s = (v[z * zstride + y * nx + xm] - ctr) + (v[z * zstride + y * nx + xp] - ctr);
                    s = s + ((v[z * zstride + ym * nx + x] - ctr) + (v[z * zstride + yp * nx + x] - ctr));
                    s = s + ((v[zm * zstride + y * nx + x] - ctr) + (v[zp * zstride + y * nx + x] - ctr));
                    L[c] = s * inv_h2;
                    cc[c] = ctr;
                }
                const double C0 = cc[0], C1 = cc[1];
                const double r = C0 * C1 * C1;                     /* (C0*C1)*C1 */
                const int64_t o = z * zstride + y * nx + x;
                f[o] = p->d1 * L[0] - r + p->F - p->F * C0;         /* ((d1*L0 - r) + F) - F*C0 */
                f[o + plane] = p->d2 * L[1] + r - FK * C1;          /* ((d2*L1) + r) - (F+K)*C1 */
            }
        }
    }
}

void orc_rhs(const orc_problem* p, const double* u, double* f) {
    const int64_t count = p->n * p->ncomp;
    switch (p->kind) {
    case ORC_RHS_EXP: rhs_exp(count, u, f, p->lambda); break;
    case ORC_RHS_LOGISTIC: rhs_logistic(count, u, f); break;
    case ORC_RHS_GRAY_SCOTT: rhs_gray_scott(p, u, f); break;
    default: break;
    }
}

/* ------------------------------------------------------------------------------
 * One explicit RK step, textbook form ("extrapolate the state ... update it
 * in-place", P:L42 error steppers).  Coefficients prepared once per
 * (scheme, dt): g_ij = dt*a_ij, beta_j = dt*b_j, delta_j = dt*(b_j - bhat_j).
 * --------------------------------------------------------------------------- */
int orc_step(const orc_problem* p, int scheme, double t, double dt, const double* u,
             double* u_new, double* err) {
    (void)t; /* all three systems are autonomous */
    const tableau* T = get_tableau(scheme);
    if (!T) return ORC_ERR_ARG;
    if (err && !T->has_err) return ORC_ERR_UNSUPPORTED;
    const int64_t count = p->n * p->ncomp;
    const int s = T->s;

    double g[MAXS][MAXS], beta[MAXS], delta[MAXS];
    for (int i = 0; i < s; ++i) {
        for (int j = 0; j < i; ++j) g[i][j] = dt * rat_to_double(T->a[i][j]);
        beta[i] = dt * rat_to_double(T->b[i]);
        delta[i] = T->has_err ? dt * rat_to_double(rat_sub(T->b[i], T->bh[i])) : 0.0;
    }
    /* stages needed: up to the last j with b_j != 0 (or delta_j != 0 if err wanted) */
    int s_eff = 0;
    for (int i = 0; i < s; ++i)
        if (T->b[i].n != 0 || (err && delta[i] != 0.0)) s_eff = i + 1;

    double* k[MAXS] = {0};
    double* Y = (double*)malloc(sizeof(double) * (size_t)count);
    for (int i = 0; i < s_eff; ++i) {
        k[i] = (double*)malloc(sizeof(double) * (size_t)count);
        /* Y_i = u + sum_{j<i, a_ij != 0} g_ij k_j, left to right */
        for (int64_t e = 0; e < count; ++e) {
            double y = u[e];
            for (int j = 0; j < i; ++j)
                if (T->a[i][j].n != 0) y = y + g[i][j] * k[j][e];
            Y[e] = y;
        }
        orc_rhs(p, Y, k[i]); /* k_i = F(t + c_i dt, Y_i) */
    }
    /* u_new = u + sum_{b_j != 0} beta_j k_j */
    for (int64_t e = 0; e < count; ++e) {
        double w = u[e];
        for (int j = 0; j < s_eff; ++j)
            if (T->b[j].n != 0) w = w + beta[j] * k[j][e];
        u_new[e] = w;
    }
    /* err = sum_{delta_j != 0} delta_j k_j, first term not added to zero */
    if (err) {
        for (int64_t e = 0; e < count; ++e) {
            double acc = 0.0;
            int first = 1;
            for (int j = 0; j < s_eff; ++j) {
                if (delta[j] == 0.0) continue;
                if (first) { acc = delta[j] * k[j][e]; first = 0; }
                else acc = acc + delta[j] * k[j][e];
            }
            err[e] = acc;
        }
    }
    for (int i = 0; i < s_eff; ++i) free(k[i]);
    free(Y);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------
 * Error control (P:L46 norm requirement; P:L135 for_each_norm).
 * --------------------------------------------------------------------------- */
double orc_error_ratio_max(int64_t count, const double* err, const double* u, const double* k1,
                           double dt, double atol, double rtol) {
    double E = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        const double r = fabs(err[i]) / (atol + rtol * (fabs(u[i]) + dt * fabs(k1[i])));
        if (isnan(r)) return NAN;
        if (r > E) E = r;
    }
    return E;
}

/* The controller's x^y, correctly rounded (R-27): evaluated in binary128
 * (libquadmath powq, 113-bit significand) and rounded once to double.  Double rounding can
 * only differ from the correctly rounded value when x^y lies within ~2^-110 (relative) of a
 * double rounding midpoint.  Pinned against 60-digit decimal arithmetic
 * (tests/test_oracle_adaptive.py::test_controller_pow_correctly_rounded). */
static double cr_pow(double x, double y) {
    return (double)powq((__float128)x, (__float128)y);
}

int orc_controller(double E, int p, int q, double* dt) {
    if (E > 1.0) {
        /* reject: decrease_step */
        double fac = (9.0 / 10.0) * cr_pow(E, -1.0 / (double)(q - 1));
        if (fac < 1.0 / 5.0) fac = 1.0 / 5.0;
        *dt = *dt * fac;
        return 0;
    }
    /* accept: increase_step */
    if (E < 0.5) {
        double Ec = cr_pow(5.0, -(double)p);
        if (E > Ec) Ec = E;
        *dt = *dt * ((9.0 / 10.0) * cr_pow(Ec, -1.0 / (double)p));
    }
    return 1;
}

/* ------------------------------------------------------------------------------
 * Drivers (P:L198 integrate_const, P:L201 do_step / integrate_adaptive).
 * --------------------------------------------------------------------------- */
int orc_integrate_const(const orc_problem* p, int scheme, double* u, double t0, double t1,
                        double dt, int64_t* steps) {
    if (!(dt > 0.0) || !(t1 > t0)) return ORC_ERR_ARG;
    const int64_t count = p->n * p->ncomp;
    double* un = (double*)malloc(sizeof(double) * (size_t)count);
    int64_t n = 0;
    double t = t0;
    while ((t + dt) - t1 <= DBL_EPSILON) {
        int rc = orc_step(p, scheme, t, dt, u, un, NULL);
        if (rc != ORC_OK) { free(un); return rc; }
        memcpy(u, un, sizeof(double) * (size_t)count);
        ++n;
        t = t0 + (double)n * dt;
    }
    free(un);
    *steps = n;
    return ORC_OK;
}

/* SPEC's elementwise_err_ratio, reading R-28. */
double orc_error_ratio_max_spec(int64_t count, const double* err, const double* u_old,
                                const double* u_new, double atol, double rtol) {
    double E = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        const double a = fabs(u_old[i]), b = fabs(u_new[i]);
        const double m = a >= b ? a : b;
        const double r = fabs(err[i]) / (atol + rtol * m);
        if (isnan(r)) return NAN;
        if (r > E) E = r;
    }
    return E;
}

/* SPEC's try_step step-size rule, reading R-28. */
int orc_controller_spec(double E, int p, double* dt) {
    if (E <= 1.0) {
        /* accepted: dt_next = dt*min(grow_cap, max(shrink_floor, safety*err^(-1/p))) */
        double fac = (9.0 / 10.0) * cr_pow(E, -1.0 / (double)p);
        if (fac < 1.0 / 5.0) fac = 1.0 / 5.0;
        if (fac > 5.0) fac = 5.0;
        *dt = *dt * fac;
        return 1;
    }
    /* rejected: dt_next = dt*max(shrink_floor, safety*err^(-1/(p-1))) */
    double fac = (9.0 / 10.0) * cr_pow(E, -1.0 / (double)(p - 1));
    if (fac < 1.0 / 5.0) fac = 1.0 / 5.0;
    *dt = *dt * fac;
    return 0;
}

int orc_integrate_adaptive_ctrl(const orc_problem* p, int scheme, double* u, double t0,
                                double t1, double dt0, double atol, double rtol, int controller,
                                int max_tries, int64_t* accepted, int64_t* rejected) {
    const tableau* T = get_tableau(scheme);
    if (!T) return ORC_ERR_ARG;
    if (!T->has_err) return ORC_ERR_UNSUPPORTED;
    if (!(dt0 > 0.0) || !(t1 > t0) || !(atol > 0.0) || !(rtol >= 0.0) || max_tries < 1 ||
        (controller != ORC_CTRL_ODEINT && controller != ORC_CTRL_SPEC))
        return ORC_ERR_ARG;
    const int64_t count = p->n * p->ncomp;
    double* un = (double*)malloc(sizeof(double) * (size_t)count);
    double* er = (double*)malloc(sizeof(double) * (size_t)count);
    double* k1 = (double*)malloc(sizeof(double) * (size_t)count);
    int64_t acc = 0, rej = 0;
    int rc = ORC_OK;
    double t = t0, dt = dt0;
    while (t1 - t > DBL_EPSILON) {
        if ((t + dt) - t1 > DBL_EPSILON) dt = t1 - t;
        if (controller == ORC_CTRL_ODEINT)
            orc_rhs(p, u, k1); /* dxdt at the start of the step (ratio denominator) */
        int tries = 0;
        for (;;) {
            /* step-size floor (SURVEY §8b RK_ERR_DT_UNDERFLOW; R-29): a try with
             * dt < 16 eps max(|t|, 1) cannot advance t meaningfully */
            if (dt < 16.0 * DBL_EPSILON * fmax(fabs(t), 1.0)) { rc = ORC_ERR_DT_UNDERFLOW; goto done; }
            rc = orc_step(p, scheme, t, dt, u, un, er);
            if (rc != ORC_OK) goto done;
            const double E = controller == ORC_CTRL_ODEINT
                                 ? orc_error_ratio_max(count, er, u, k1, dt, atol, rtol)
                                 : orc_error_ratio_max_spec(count, er, u, un, atol, rtol);
            if (isnan(E)) { rc = ORC_ERR_DIVERGED; goto done; }
            const double dt_used = dt;
            const int ok = controller == ORC_CTRL_ODEINT
                               ? orc_controller(E, T->order, T->err_order, &dt)
                               : orc_controller_spec(E, T->order, &dt);
            if (ok) {
                memcpy(u, un, sizeof(double) * (size_t)count);
                t = t + dt_used;
                ++acc;
                break;
            }
            ++rej;
            if (++tries >= max_tries) { rc = ORC_ERR_STALL; goto done; }
        }
    }
done:
    free(un); free(er); free(k1);
    *accepted = acc;
    *rejected = rej;
    return rc;
}

int orc_integrate_adaptive(const orc_problem* p, int scheme, double* u, double t0, double t1,
                           double dt0, double atol, double rtol, int64_t* accepted,
                           int64_t* rejected) {
    return orc_integrate_adaptive_ctrl(p, scheme, u, t0, t1, dt0, atol, rtol, ORC_CTRL_ODEINT,
                                       500, accepted, rejected);
}

/* ------------------------------------------------------------------------------
 * Adams–Bashforth (Table 1 multi-step row; Fig. 2c/d).
 * Published coefficients over a common denominator (newest first), e.g. Hairer, Norsett &
 * Wanner I, III.1; pinned in tests against the Lagrange-integral definition.
 * --------------------------------------------------------------------------- */
static const int64_t AB_NUM[8][8] = {
    {1},
    {3, -1},
    {23, -16, 5},
    {55, -59, 37, -9},
    {1901, -2774, 2616, -1274, 251},
    {4277, -7923, 9982, -7298, 2877, -475},
    {198721, -447288, 705549, -688256, 407139, -134472, 19087},
    {434241, -1152169, 2183877, -2664477, 2102243, -1041723, 295767, -36799},
};
static const int64_t AB_DEN[8] = {1, 2, 12, 24, 720, 1440, 60480, 120960};

int orc_ab_coefficients(int k, int64_t* num, int64_t* den) {
    if (k < 1 || k > 8) return -1;
    for (int j = 0; j < k; ++j) {
        num[j] = AB_NUM[k - 1][j];
        den[j] = AB_DEN[k - 1];
    }
    return k;
}

int orc_ab_integrate(const orc_problem* p, int k, double* u, double t0, double dt, int64_t nsteps,
                     double* traj) {
    if (k < 1 || k > 8 || !(dt > 0.0) || nsteps < 0) return ORC_ERR_ARG;
    const int64_t count = p->n * p->ncomp;
    double g[8];
    for (int j = 0; j < k; ++j) g[j] = dt * ((double)AB_NUM[k - 1][j] / (double)AB_DEN[k - 1]);
    double* f[8];
    for (int j = 0; j < k; ++j) f[j] = (double*)malloc(sizeof(double) * (size_t)count);
    double* un = (double*)malloc(sizeof(double) * (size_t)count);
    int rc = ORC_OK;
    for (int64_t n = 0; n < nsteps; ++n) {
        const double t = t0 + (double)n * dt;
        orc_rhs(p, u, f[n % k]); /* f_n = F(t_n, u_n) */
        if (n < k - 1) {
            rc = orc_step(p, ORC_RKF78, t, dt, u, un, NULL); /* bootstrap (R-23) */
            if (rc != ORC_OK) break;
        } else {
            for (int64_t e = 0; e < count; ++e) {
                double w = u[e];
                for (int j = 0; j < k; ++j) w = w + g[j] * f[(n - j) % k][e];
                un[e] = w;
            }
        }
        memcpy(u, un, sizeof(double) * (size_t)count);
        if (traj) memcpy(traj + n * count, u, sizeof(double) * (size_t)count);
    }
    for (int j = 0; j < k; ++j) free(f[j]);
    free(un);
    return rc;
}

/* Adams–Moulton k-term coefficients m_0..m_{k-1} (m_0 weighs f_{n+1}, then f_n, f_{n-1} ...),
 * the corrector of Table 1's "Adams-Bashforth-Moulton 1..8" row: the integrals over
 * [t_n, t_{n+1}] of the Lagrange basis on t_{n+1}, t_n, ..., t_{n-k+2} (textbook values). */
static const int64_t AM_NUM[8][8] = {
    {1},
    {1, 1},
    {5, 8, -1},
    {9, 19, -5, 1},
    {251, 646, -264, 106, -19},
    {475, 1427, -798, 482, -173, 27},
    {19087, 65112, -46461, 37504, -20211, 6312, -863},
    {36799, 139849, -121797, 123133, -88547, 41499, -11351, 1375},
};
static const int64_t AM_DEN[8] = {1, 2, 12, 24, 720, 1440, 60480, 120960};

int orc_am_coefficients(int k, int64_t* num, int64_t* den) {
    if (k < 1 || k > 8) return -1;
    for (int j = 0; j < k; ++j) {
        num[j] = AM_NUM[k - 1][j];
        den[j] = AM_DEN[k - 1];
    }
    return k;
}

int orc_abm_integrate(const orc_problem* p, int k, double* u, double t0, double dt, int64_t nsteps,
                      double* traj) {
    if (k < 1 || k > 8 || !(dt > 0.0) || nsteps < 0) return ORC_ERR_ARG;
    const int64_t count = p->n * p->ncomp;
    double g[8], m[8];
    for (int j = 0; j < k; ++j) {
        g[j] = dt * ((double)AB_NUM[k - 1][j] / (double)AB_DEN[k - 1]);
        m[j] = dt * ((double)AM_NUM[k - 1][j] / (double)AM_DEN[k - 1]);
    }
    double* f[8];
    for (int j = 0; j < k; ++j) f[j] = (double*)malloc(sizeof(double) * (size_t)count);
    double* un = (double*)malloc(sizeof(double) * (size_t)count);
    double* fp = (double*)malloc(sizeof(double) * (size_t)count);
    int rc = ORC_OK;
    for (int64_t n = 0; n < nsteps; ++n) {
        const double t = t0 + (double)n * dt;
        orc_rhs(p, u, f[n % k]); /* E: f_n = F(t_n, u_n) */
        if (n < k - 1) {
            rc = orc_step(p, ORC_RKF78, t, dt, u, un, NULL); /* bootstrap (R-23) */
            if (rc != ORC_OK) break;
        } else {
            /* P: predictor u_p = u_n + sum_{j<k} (dt*beta_j) f_{n-j}, newest first (R-24) */
            for (int64_t e = 0; e < count; ++e) {
                double w = u[e];
                for (int j = 0; j < k; ++j) w = w + g[j] * f[(n - j) % k][e];
                un[e] = w;
            }
            orc_rhs(p, un, fp); /* E: f_p = F(t_{n+1}, u_p) */
            /* C: u_{n+1} = u_n + (dt*m_0) f_p + sum_{j=1}^{k-1} (dt*m_j) f_{n-j+1}, newest first */
            for (int64_t e = 0; e < count; ++e) {
                double w = u[e] + m[0] * fp[e];
                for (int j = 1; j < k; ++j) w = w + m[j] * f[(n - j + 1) % k][e];
                un[e] = w;
            }
        }
        memcpy(u, un, sizeof(double) * (size_t)count);
        if (traj) memcpy(traj + n * count, u, sizeof(double) * (size_t)count);
    }
    for (int j = 0; j < k; ++j) free(f[j]);
    free(un);
    free(fp);
    return rc;
}

/* ------------------------------------------------------------------------------
 * Algebra ops.
 * --------------------------------------------------------------------------- */
int orc_lincomb(int64_t count, double* out, int k, const double* coef, const double* const* in) {
    if (k < 1 || k > 14) return ORC_ERR_ARG;
    for (int64_t i = 0; i < count; ++i) {
        double acc = coef[0] * in[0][i];
        for (int j = 1; j < k; ++j) acc = acc + coef[j] * in[j][i];
        out[i] = acc;
    }
    return ORC_OK;
}

double orc_norm_inf(int64_t count, const double* u) {
    double m = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        const double a = fabs(u[i]);
        if (isnan(a)) return NAN;
        if (a > m) m = a;
    }
    return m;
}
