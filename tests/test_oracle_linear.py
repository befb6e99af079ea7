"""Pins of the oracle's stepper arithmetic on the linear test equation u' = lambda*u.

For an explicit RK method the n-step result is exactly u0*R(z)^n with z = lambda*dt and
R the stability polynomial (textbook; Euler/RK4 truncated exponentials, CK54/DOPRI5 per
SURVEY App. A).  The embedded error of one step is E(z)*u0 with E = R_b - R_bhat.
Any wrong coefficient, dropped stage term or wrong sign moves the result by O(dt^k),
many orders of magnitude above the 4*n ulp gate.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EPS = np.finfo(np.float64).eps
POLYS = json.load(open(os.path.join(GOLD, "stability_polys.json")))
NAMES = {oracle.EULER: "euler", oracle.RK4: "rk4", oracle.CASH_KARP54: "cash_karp54",
         oracle.DOPRI5: "dopri5", oracle.MIDPOINT: "midpoint",
         oracle.MODIFIED_MIDPOINT: "modified_midpoint"}


def R(name, z, which="b"):
    return sum(Fraction(c) * z ** k for k, c in enumerate(POLYS[name][which]))


@pytest.mark.parametrize("scheme", list(NAMES))
@pytest.mark.parametrize("lam,dt,n", [(-1.0, 0.1, 10), (-1.0, 2.0 ** -8, 256), (1.0, 0.5, 20),
                                      (-3.0, 0.3, 7)])
def test_linear_closed_form(scheme, lam, dt, n):
    u0 = np.array([1.0, 0.3, -2.5, 1e-3])
    p = oracle.exp_problem(u0.size, lam)
    u = u0.copy()
    for _ in range(n):
        u = oracle.step(p, scheme, 0.0, dt, u)
    Rn = R(NAMES[scheme], Fraction(lam) * Fraction(dt)) ** n
    for i in range(u0.size):
        exact = Fraction(u0[i]) * Rn
        ulp = abs(float(exact)) * EPS
        assert abs(Fraction(u[i]) - exact) <= 4 * n * ulp + 1e-300, (i, float(u[i]), float(exact))


@pytest.mark.parametrize("scheme", [oracle.CASH_KARP54, oracle.DOPRI5])
@pytest.mark.parametrize("lam,dt", [(-1.0, 0.1), (1.0, 0.5), (-2.0, 0.25), (-1.0, 1.0)])
def test_embedded_error_closed_form(scheme, lam, dt):
    u0 = np.array([1.0, -0.75, 3.0])
    p = oracle.exp_problem(u0.size, lam)
    un, err = oracle.step(p, scheme, 0.0, dt, u0, with_error=True)
    name = NAMES[scheme]
    z = Fraction(lam) * Fraction(dt)
    E = R(name, z, "b") - R(name, z, "bhat")
    # E(z) = O(z^5): the first five coefficients of R_b and R_bhat agree (orders 5 and 4)
    assert POLYS[name]["b"][:5] == POLYS[name]["bhat"][:5]
    for i in range(u0.size):
        want = E * Fraction(u0[i])
        scale = abs(u0[i]) * abs(lam) * dt * 8 * max(1.0, float(abs(R(name, z))))
        assert abs(Fraction(err[i]) - want) <= 16 * EPS * scale, (i, err[i], float(want))


def test_spec_worked_values():
    # S:L62 / S:L150: Euler, du/dt=u, u=[1], dt=0.1 -> 1.1
    assert oracle.step(oracle.exp_problem(1, 1.0), oracle.EULER, 0.0, 0.1, [1.0])[0] == 1.1
    # S:L63 / S:L151: RK4, du/dt=u, u=[1], dt=1 -> 2.708333333333333 (= fl(65/24) left to right)
    v = oracle.step(oracle.exp_problem(1, 1.0), oracle.RK4, 0.0, 1.0, [1.0])[0]
    assert v == 2.7083333333333335 == float(Fraction(65, 24))


def test_decay_ten_steps_golden():
    """u'=-u, u0=1, dt=0.1, 10 steps (exact R(z)^10, 18 digits)."""
    gold = json.load(open(os.path.join(GOLD, "linear_decay.json")))
    for scheme, name in NAMES.items():
        u = np.array([1.0])
        for _ in range(10):
            u = oracle.step(oracle.exp_problem(1, -1.0), scheme, 0.0, 0.1, u)
        assert abs(u[0] - float(gold[name])) <= 40 * EPS, (name, u[0])


@pytest.mark.parametrize("scheme", list(NAMES))
def test_zero_rhs_fixed_point(scheme):
    """du/dt = 0 (lambda = 0): the state is unchanged and the error estimate is 0."""
    u0 = np.array([0.5, -1.0, 7.0])
    p = oracle.exp_problem(3, 0.0)
    if scheme in (oracle.CASH_KARP54, oracle.DOPRI5):
        un, err = oracle.step(p, scheme, 0.0, 0.7, u0, with_error=True)
        assert np.all(err == 0.0)
    else:
        un = oracle.step(p, scheme, 0.0, 0.7, u0)
    assert np.array_equal(un, u0)


def _R_from_tableau(tab, w, z):
    """R(z) = 1 + sum_k (w^T A^{k-1} 1) z^k, exact (the tableau itself is pinned by the
    order conditions in test_oracle_tableau.py)."""
    A, s = tab["a"], tab["s"]
    v, out = [Fraction(1)] * s, Fraction(1)
    for k in range(1, s + 1):
        out += sum(w[i] * v[i] for i in range(s)) * z ** k
        v = [sum(A[i][j] * v[j] for j in range(s)) for i in range(s)]
    return out


@pytest.mark.parametrize("lam,dt,n", [(-1.0, 0.1, 10), (1.0, 0.5, 20), (-3.0, 0.3, 7), (-1.0, 2.0, 3)])
def test_rkf78_linear_closed_form(lam, dt, n):
    """RKF78 step arithmetic (13 stages, 8th-order weights) vs u0*R(z)^n, and the embedded
    error vs (R_b - R_bhat)(z)*u0."""
    tab = oracle.tableau(oracle.RKF78)
    u0 = np.array([1.0, 0.3, -2.5])
    p = oracle.exp_problem(u0.size, lam)
    z = Fraction(lam) * Fraction(dt)
    R = _R_from_tableau(tab, tab["b"], z)
    u = u0.copy()
    for _ in range(n):
        u = oracle.step(p, oracle.RKF78, 0.0, dt, u)
    for i in range(u0.size):
        exact = Fraction(u0[i]) * R ** n
        assert abs(Fraction(u[i]) - exact) <= 8 * n * abs(float(exact)) * EPS + 1e-300
    un, err = oracle.step(p, oracle.RKF78, 0.0, dt, u0, with_error=True)
    E = R - _R_from_tableau(tab, tab["bhat"], z)
    for i in range(u0.size):
        scale = abs(u0[i]) * abs(lam) * dt * 8 * max(1.0, float(abs(R)))
        assert abs(Fraction(err[i]) - E * Fraction(u0[i])) <= 16 * EPS * scale
