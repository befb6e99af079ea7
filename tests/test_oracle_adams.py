"""Pins of the oracle's Adams–Bashforth k = 1..8 (Table 1 multi-step row; Fig. 2c/d,
P:L215 "convergence orders between 1 and 8" -- SURVEY §8 f2).

* the published coefficients equal the definition beta_j = int_0^1 prod_{m != j}
  (s + m)/(m - j) ds (Lagrange interpolation of f on t_n, t_{n-1}, ...), in exact rationals;
* on u' = lambda*u the method is an exact linear recurrence (RKF78 bootstrap: R78(z), then
  u_{n+1} = u_n + z sum_j beta_j u_{n-j}) which the oracle must reproduce to rounding;
* trajectory-max convergence order k on Eq. 1b and on the decay problem.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import rk_inputs

EPS = np.finfo(np.float64).eps


def lagrange_ab(k):
    out = []
    for j in range(k):
        poly, den = [Fraction(1)], Fraction(1)
        for m in range(k):
            if m == j:
                continue
            new = [Fraction(0)] * (len(poly) + 1)
            for i, c in enumerate(poly):
                new[i] += c * m
                new[i + 1] += c
            poly, den = new, den * (m - j)
        out.append(sum(c / (i + 1) for i, c in enumerate(poly)) / den)
    return out


@pytest.mark.parametrize("k", range(1, 9))
def test_coefficients_are_the_lagrange_integrals(k):
    assert oracle.ab_coefficients(k) == lagrange_ab(k)
    assert sum(oracle.ab_coefficients(k)) == 1


def _R_tableau(tab, z):
    A, b, s = tab["a"], tab["b"], tab["s"]
    v, out = [Fraction(1)] * s, Fraction(1)
    for kk in range(1, s + 1):
        out += sum(b[i] * v[i] for i in range(s)) * z ** kk
        v = [sum(A[i][j] * v[j] for j in range(s)) for i in range(s)]
    return out


@pytest.mark.parametrize("k", range(1, 9))
def test_linear_recurrence(k):
    lam, dt, n = -1.0, 0.0625, 40  # inside every AB-k stability interval
    z = Fraction(lam) * Fraction(dt)
    R78 = _R_tableau(oracle.tableau(oracle.RKF78), z)
    beta = lagrange_ab(k)
    u0 = np.array([1.0, -0.4])
    got = oracle.ab_integrate(oracle.exp_problem(2, lam), k, u0, 0.0, dt, n)
    for i in range(2):
        seq = [Fraction(u0[i])]
        for m in range(n):
            if m < k - 1:
                seq.append(seq[-1] * R78)
            else:
                seq.append(seq[-1] + z * sum(beta[j] * seq[m - j] for j in range(k)))
        exact = seq[-1]
        assert abs(Fraction(got[i]) - exact) <= 8 * n * k * EPS * abs(float(u0[i])), (k, i)


def _traj_err(p, k, u0, t0, dt, n, exact):
    _, tr = oracle.ab_integrate(p, k, u0, t0, dt, n, trajectory=True)
    ts = t0 + dt * np.arange(1, n + 1)
    return float(np.max(np.abs(tr - np.stack([exact(t) for t in ts]))))


def _orders_ok(errs, k, floor, tol=0.3):
    ords = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    good = [abs(o - k) <= tol and errs[i + 1] > floor for i, o in enumerate(ords)]
    return any(good[i] and good[i + 1] for i in range(len(good) - 1)), ords


@pytest.mark.parametrize("k", range(1, 8))
def test_orders_logistic(k):
    p = oracle.logistic_problem(1)
    ex = lambda t: np.array([1.0 / (1.0 + math.exp(-t))])
    errs = [_traj_err(p, k, ex(-5.0), -5.0, 0.5 * 2.0 ** -m, int(20 * 2 ** m), ex) for m in range(8)]
    ok, ords = _orders_ok(errs, k, 1e-13)
    assert ok, (k, ords, errs)


@pytest.mark.parametrize("k", [6, 7, 8])
def test_orders_exp_family(k):
    """The paper's Fig. 2c problem (Eq. 1a, A = x*y, t in [-5, 5])."""
    u0 = rk_inputs.exp_family_u0(4, -5.0)
    A = u0 * math.exp(5.0)
    p = oracle.exp_problem(u0.size, 1.0)
    ex = lambda t: A * math.exp(t)
    errs = [_traj_err(p, k, u0, -5.0, 0.5 * 2.0 ** -m, int(20 * 2 ** m), ex) for m in range(7)]
    ok, ords = _orders_ok(errs, k, 1e-11)
    assert ok, (k, ords, errs)


# ---------------------------------------------------------------------------------------
# Adams–Bashforth–Moulton k = 1..8, PECE (Table 1; R-26)
# ---------------------------------------------------------------------------------------
def lagrange_am(k):
    """m_j = int_0^1 L_j(s) ds, L_j the Lagrange basis on the nodes s = 1, 0, -1, ..., 2-k
    (f_{n+1}, f_n, ..., f_{n-k+2}); computed here from the definition in exact rationals."""
    nodes = [Fraction(1 - j) for j in range(k)]
    out = []
    for j in range(k):
        poly, den = [Fraction(1)], Fraction(1)
        for m in range(k):
            if m == j:
                continue
            new = [Fraction(0)] * (len(poly) + 1)
            for i, c in enumerate(poly):  # poly * (s - x_m)
                new[i] -= c * nodes[m]
                new[i + 1] += c
            poly, den = new, den * (nodes[j] - nodes[m])
        out.append(sum(c / (i + 1) for i, c in enumerate(poly)) / den)
    return out


@pytest.mark.parametrize("k", range(1, 9))
def test_am_coefficients_are_the_lagrange_integrals(k):
    assert oracle.am_coefficients(k) == lagrange_am(k)
    assert sum(oracle.am_coefficients(k)) == 1


def test_am_textbook_rows():
    """Trapezoid rule (k=2) and the 4-term corrector 9/24, 19/24, -5/24, 1/24."""
    assert oracle.am_coefficients(2) == [Fraction(1, 2), Fraction(1, 2)]
    assert oracle.am_coefficients(4) == [Fraction(9, 24), Fraction(19, 24), Fraction(-5, 24),
                                         Fraction(1, 24)]


@pytest.mark.parametrize("k", range(1, 9))
def test_abm_linear_recurrence(k):
    """On u' = lambda*u, PECE is the exact recurrence p = u_n + z sum beta_j u_{n-j},
    u_{n+1} = u_n + z m_0 p + z sum_{j>=1} m_j u_{n-j+1} after the R78(z) bootstrap."""
    lam, dt, n = -1.0, 0.0625, 40
    z = Fraction(lam) * Fraction(dt)
    R78 = _R_tableau(oracle.tableau(oracle.RKF78), z)
    beta, mo = lagrange_ab(k), lagrange_am(k)
    u0 = np.array([1.0, -0.4])
    got = oracle.abm_integrate(oracle.exp_problem(2, lam), k, u0, 0.0, dt, n)
    for i in range(2):
        seq = [Fraction(u0[i])]
        for m in range(n):
            if m < k - 1:
                seq.append(seq[-1] * R78)
            else:
                p = seq[-1] + z * sum(beta[j] * seq[m - j] for j in range(k))
                seq.append(seq[-1] + z * mo[0] * p + z * sum(mo[j] * seq[m - j + 1] for j in range(1, k)))
        assert abs(Fraction(got[i]) - seq[-1]) <= 16 * n * k * EPS * abs(float(u0[i])), (k, i)


def test_abm_first_steps_are_the_bootstrap():
    """The first k-1 steps equal Adams–Bashforth's (both are the RKF78 start-up, R-23)."""
    p = oracle.logistic_problem(3)
    u0 = np.array([0.1, 0.5, 0.9])
    for k in (2, 5, 8):
        a = oracle.abm_integrate(p, k, u0, 0.0, 0.1, k - 1)
        b = oracle.ab_integrate(p, k, u0, 0.0, 0.1, k - 1)
        assert np.array_equal(a, b)


def _abm_traj_err(p, k, u0, t0, dt, n, exact):
    _, tr = oracle.abm_integrate(p, k, u0, t0, dt, n, trajectory=True)
    ts = t0 + dt * np.arange(1, n + 1)
    return float(np.max(np.abs(tr - np.stack([exact(t) for t in ts]))))


@pytest.mark.parametrize("k", range(1, 8))
def test_abm_orders_logistic(k):
    p = oracle.logistic_problem(1)
    ex = lambda t: np.array([1.0 / (1.0 + math.exp(-t))])
    errs = [_abm_traj_err(p, k, ex(-5.0), -5.0, 0.5 * 2.0 ** -m, int(20 * 2 ** m), ex) for m in range(8)]
    ok, ords = _orders_ok(errs, k, 1e-13)
    assert ok, (k, ords, errs)


@pytest.mark.parametrize("k", [6, 7, 8])
def test_abm_orders_decay(k):
    """u' = -u on [0, 4] (Eq. 1a with lambda = -1): trajectory-max order k down to ~1e-14
    (on the growing exponential family the high orders reach the roundoff floor first)."""
    p = oracle.exp_problem(1, -1.0)
    ex = lambda t: np.array([math.exp(-t)])
    errs = [_abm_traj_err(p, k, ex(0.0), 0.0, 0.5 * 2.0 ** -m, int(8 * 2 ** m), ex) for m in range(6)]
    ok, ords = _orders_ok(errs, k, 1e-14)
    assert ok, (k, ords, errs)
