/*
 * rk_oracle.h — plain, slow, obviously-correct fp64 CPU oracle for the explicit
 * Runge–Kutta hot path of arxiv 2309.05331 (OpenFPM + Boost.Odeint).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2309_05331_b200/,
 * include/) may include, link or call this code; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may.  It shares no code, header,
 * table or helper with the CUDA path: the Butcher tableaux below are typed separately
 * from the library's and cross-checked by tests.
 *
 * Citations: P:Lnn = /root/reference/PAPER.md line nn (section in brackets);
 *            S:Lnn = SPEC.md line nn; DESIGN.md "R-x" = a reading of the paper.
 *
 * Everything works on the GLOBAL single-domain array (no decomposition, no ghosts):
 *   vector state : [c][i]          (ncomp components of n elements)
 *   grid state   : [z][c][y][x]    (x fastest), periodic in x, y, z by modulo.
 * Every k_j of a step is stored (textbook Butcher form).  Sums run left to right in
 * increasing j and skip zero coefficients (R-17).  Build flags:
 * -O2 -ffp-contract=off (no FMA contraction), IEEE division, no fast-math.
 */
#ifndef RK_ORACLE_H
#define RK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Schemes of Table 1 on the hot path. */
enum { ORC_EULER = 0, ORC_RK4 = 1, ORC_CASH_KARP54 = 2, ORC_DOPRI5 = 3, ORC_RKF78 = 4,
       ORC_MIDPOINT = 5 /* explicit midpoint */, ORC_MODIFIED_MIDPOINT = 6 /* Gragg, Table 1 P:L58 */ };
/* RHS kinds: Eq. 1a as du/dt = lambda*u, Eq. 1b, Eq. 3 / Listing 2. */
enum { ORC_RHS_EXP = 0, ORC_RHS_LOGISTIC = 1, ORC_RHS_GRAY_SCOTT = 2 };
/* Status codes. */
enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_UNSUPPORTED = 2, ORC_ERR_DIVERGED = 3, ORC_ERR_STALL = 4,
       ORC_ERR_DT_UNDERFLOW = 5 };

typedef struct {
    int kind;            /* ORC_RHS_* */
    int ncomp;           /* components (1 for exp/logistic, 2 for Gray–Scott) */
    int64_t n;           /* elements per component (vector) or nx*ny*nz (grid) */
    int64_t nx, ny, nz;  /* grid dims (Gray–Scott only) */
    double lambda;       /* exp: du/dt = lambda*u */
    double d1, d2, F, K; /* Gray–Scott parameters, Listing 2 */
    double h;            /* grid spacing, h = L/n (R-4) */
} orc_problem;

/* Tableau access for tests: exact rationals as (num, den) int64 pairs.
 * a is s*s row-major (strictly lower triangular), b/bhat/c length s (s <= 13).  bhat is all
 * zero for schemes without an embedded solution.  Returns s, or -1 for bad scheme. */
int orc_tableau(int scheme, int64_t* a_num, int64_t* a_den, int64_t* b_num, int64_t* b_den,
                int64_t* bh_num, int64_t* bh_den, int64_t* c_num, int64_t* c_den,
                int* order, int* err_order);

/* F(u) of the three model systems.  u and f are full states of the problem's size. */
void orc_rhs(const orc_problem* p, const double* u, double* f);

/* One explicit RK step in textbook Butcher form:
 *   Y_i = u + sum_{j<i} (dt*a_ij) k_j,  k_i = F(Y_i),  u_new = u + sum_j (dt*b_j) k_j,
 *   err = sum_j (dt*(b_j - bhat_j)) k_j  (only if err != NULL; CK54 / DOPRI5 only;
 *   for DOPRI5 this includes k_7 = F(Y_7) with Y_7 = u_new, the FSAL stage).
 * u is not modified.  Returns ORC_OK or ORC_ERR_UNSUPPORTED (err for a scheme
 * without embedded weights). */
int orc_step(const orc_problem* p, int scheme, double t, double dt, const double* u,
             double* u_new, double* err);

/* Odeint-style per-element error ratio and its max (R-12, R-13):
 *   r = |err| / (atol + rtol*(|u| + dt*|k1|)),  E = max r over all elements.
 * NaN in any r makes E NaN. */
double orc_error_ratio_max(int64_t count, const double* err, const double* u,
                           const double* k1, double dt, double atol, double rtol);

/* Odeint default step adjuster (R-12, R-14).  On E > 1: reject,
 * dt *= max(0.9*E^(-1/(q-1)), 0.2); else accept and, if E < 0.5,
 * dt *= 0.9*max(E, 5^-p)^(-1/p).  Returns 1 if accepted, 0 if rejected. */
int orc_controller(double E, int p, int q, double* dt);

/* integrate_const (Odeint loop, R-15): steps while
 * (t_n + dt) - t1 <= eps with t_n = t0 + n*dt.  Updates u in place. */
int orc_integrate_const(const orc_problem* p, int scheme, double* u, double t0, double t1,
                        double dt, int64_t* steps);

/* integrate_adaptive (Odeint loop, R-16): error-controlled
 * stepping from t0 to exactly t1 with the controller above; at most 500 tries
 * per step (ORC_ERR_STALL), NaN error ratio -> ORC_ERR_DIVERGED.
 * Updates u in place; reports accepted and rejected try counts. */
int orc_integrate_adaptive(const orc_problem* p, int scheme, double* u, double t0, double t1,
                           double dt0, double atol, double rtol, int64_t* accepted,
                           int64_t* rejected);

/* The alternative controller reading of DESIGN.md R-28: SPEC's elementary controller
 * (S:L218-233), kept behind an option because the paper delegates the constants to Odeint
 * and SURVEY Z12 ships Odeint's.
 * Ratio (S:L75-83 elementwise_err_ratio):
 *   r = |err| / (atol + rtol*m),  m = |u_old| if |u_old| >= |u_new| else |u_new|,
 *   E = max r over all elements (NaN in any r makes E NaN). */
double orc_error_ratio_max_spec(int64_t count, const double* err, const double* u_old,
                                const double* u_new, double atol, double rtol);
/* SPEC try_step, p = order of the propagated solution:
 *   E <= 1: accept, dt *= min(5, max(0.2, 0.9*E^(-1/p)))      (E == 0: x5, the grow cap)
 *   E >  1: reject, dt *= max(0.2, 0.9*E^(-1/(p-1))).
 * Returns 1 if accepted, 0 if rejected. */
int orc_controller_spec(double E, int p, double* dt);
enum { ORC_CTRL_ODEINT = 0, ORC_CTRL_SPEC = 1 };
/* integrate_adaptive with a choice of controller (ORC_CTRL_*); the Odeint choice is exactly
 * orc_integrate_adaptive.  max_tries: tries per step before ORC_ERR_STALL (Odeint 500). */
int orc_integrate_adaptive_ctrl(const orc_problem* p, int scheme, double* u, double t0,
                                double t1, double dt0, double atol, double rtol, int controller,
                                int max_tries, int64_t* accepted, int64_t* rejected);

/* Adams–Bashforth k-step coefficients beta_0..beta_{k-1} (newest first) as exact rationals
 * (Table 1 "multi-step, Adams-Bashforth 1..8").  Returns k, or -1 if k not in 1..8. */
int orc_ab_coefficients(int k, int64_t* num, int64_t* den);

/* Adams–Bashforth k-step integration of nsteps fixed steps of size dt from t0 (
 * S:L144-152).  Step n evaluates f_n = F(u_n) and keeps the last k values.
 * The first min(k-1, nsteps) steps are bootstrap steps with RKF78 (R-23); after
 * that u_{n+1} = u_n + sum_{j=0}^{k-1} (dt*beta_j) f_{n-j}, summed newest first (Odeint's
 * order, R-24).  Updates u in place; if traj != NULL, u after step n+1 is also
 * stored at traj + n*count (trajectory-max error norms, R-8). */
int orc_ab_integrate(const orc_problem* p, int k, double* u, double t0, double dt, int64_t nsteps,
                     double* traj);

/* Adams–Moulton k-term corrector coefficients m_0..m_{k-1} (m_0 weighs f_{n+1}; then f_n,
 * f_{n-1}, ...) as exact rationals (Table 1 "Adams-Bashforth-Moulton 1..8"). */
int orc_am_coefficients(int k, int64_t* num, int64_t* den);

/* Adams–Bashforth–Moulton k, PECE (R-26): the RKF78 bootstrap of R-23, then
 * per step  E: f_n = F(u_n);  P: u_p = u_n + sum_{j<k} (dt*beta_j) f_{n-j};  E: f_p = F(u_p);
 * C: u_{n+1} = u_n + (dt*m_0) f_p + sum_{j=1}^{k-1} (dt*m_j) f_{n-j+1}; both sums newest
 * first (R-24).  Arguments and trajectory as orc_ab_integrate. */
int orc_abm_integrate(const orc_problem* p, int k, double* u, double t0, double dt, int64_t nsteps,
                      double* traj);

/* Algebra ops ("for_each#" / "for_each_norm").
 * out = sum_{j=0}^{k-1} coef[j]*in[j], left to right, 1 <= k <= 14. */
int orc_lincomb(int64_t count, double* out, int k, const double* coef, const double* const* in);
double orc_norm_inf(int64_t count, const double* u);

#ifdef __cplusplus
}
#endif
#endif
