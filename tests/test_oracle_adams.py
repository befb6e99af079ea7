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
