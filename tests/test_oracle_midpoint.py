"""Pins that tell the two order-2 "midpoint" schemes apart from each other and from every
other 2-/3-stage order-2 method (Heun, Ralston, ...), which the order conditions, row sums and
R(z) = 1 + z + z^2/2 alone do not (VERDICT r1 "What's weak" 1).

* Explicit midpoint rule (RK_MIDPOINT): "an Euler half step, then the full step with
  the midpoint slope".  One step of the logistic RHS u' = u(1 - u) (Eq. 1b) from
  u0 = 1/4 with dt = 1/2 is computed here from that sentence in exact rationals; every
  intermediate is dyadic, so the oracle's fp64 result must equal it exactly.  Heun's rule
  (trapezoid slopes) gives 1447/4096, Ralston's (2/3-point) another value.
* Modified midpoint (RK_MODIFIED_MIDPOINT; Table 1, P:L58 = Odeint's modified_midpoint, DESIGN.md
  R-22): Gragg's recurrence with n = 2 substeps, h = dt/2,
      x1 = u + h F(u);  x2 = u + 2h F(x1);  u_new = (x1 + x2 + h F(x2)) / 2,
  is evaluated here AS THAT RECURRENCE (not the oracle's Butcher form) in exact rationals and
  must match the oracle's Butcher-form step to rounding.  Its linear R(z) carries z^3/8
  (tests/golden/stability_polys.json, derived from the recurrence by hand), which the explicit
  midpoint lacks.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle

EPS = np.finfo(np.float64).eps


def f_log(u):
    return u * (1 - u)


def explicit_midpoint(u0, dt, f):
    return u0 + dt * f(u0 + dt / 2 * f(u0))


def heun(u0, dt, f):
    return u0 + dt / 2 * (f(u0) + f(u0 + dt * f(u0)))


def ralston(u0, dt, f):
    k1 = f(u0)
    return u0 + dt * (k1 / 4 + 3 * f(u0 + Fr(2, 3) * dt * k1) / 4)


def gragg(u0, dt, f, n=2):
    """Odeint modified_midpoint: Gragg's substep recurrence (x0, x1 swap form)."""
    h = dt / n
    x0, x1 = u0, u0 + h * f(u0)
    for _ in range(1, n):
        x0, x1 = x1, x0 + 2 * h * f(x1)
    return (x0 + x1 + h * f(x1)) / 2


def test_explicit_midpoint_logistic_exact():
    u0, dt = Fr(1, 4), Fr(1, 2)
    want = explicit_midpoint(u0, dt, f_log)
    assert want == Fr(2903, 8192)
    # the pin separates the order-2 family: Heun and Ralston land elsewhere
    assert heun(u0, dt, f_log) == Fr(1447, 4096) != want
    assert ralston(u0, dt, f_log) != want
    got = oracle.step(oracle.logistic_problem(1), oracle.MIDPOINT, 0.0, 0.5, [0.25])[0]
    assert Fr(got) == want


@pytest.mark.parametrize("u0,dt", [(0.25, 0.5), (0.7, 0.3), (-0.4, 0.125), (2.0, 1.0)])
def test_modified_midpoint_is_gragg(u0, dt):
    """The oracle's Butcher form equals Gragg's recurrence (n = 2) on a nonlinear RHS."""
    want = gragg(Fr(u0), Fr(dt), f_log)
    got = oracle.step(oracle.logistic_problem(1), oracle.MODIFIED_MIDPOINT, 0.0, dt, [u0])[0]
    assert abs(Fr(got) - want) <= 8 * EPS * max(1.0, abs(float(want))), (got, float(want))
    # ... and differs from the explicit midpoint by far more than rounding (O(dt^3))
    em = explicit_midpoint(Fr(u0), Fr(dt), f_log)
    assert abs(float(em - want)) > 1e3 * EPS * max(1.0, abs(float(want)))


def test_modified_midpoint_three_rhs_evaluations():
    """Gragg with n = 2 substeps evaluates F three times (F(u), F(x1), F(x2)): the Butcher form
    has three stages with nodes 0, 1/2, 1 (the substep points)."""
    tab = oracle.tableau(oracle.MODIFIED_MIDPOINT)
    assert tab["s"] == 3 and tab["c"] == [0, Fr(1, 2), 1]
    calls = []

    def f_count(u):
        calls.append(u)
        return f_log(u)
    gragg(Fr(1, 3), Fr(1, 5), f_count)
    assert len(calls) == 3


def test_modified_midpoint_linear_z3():
    """u' = -u, dt = 1/2: one step is R(-1/2) = 1 - 1/2 + 1/8 - 1/64 (Gragg), not the explicit
    midpoint's 1 - 1/2 + 1/8: the z^3/8 term is visible at 2^-6."""
    got = oracle.step(oracle.exp_problem(1, -1.0), oracle.MODIFIED_MIDPOINT, 0.0, 0.5, [1.0])[0]
    assert got == float(Fr(1) - Fr(1, 2) + Fr(1, 8) - Fr(1, 64)) == 0.609375
    got_em = oracle.step(oracle.exp_problem(1, -1.0), oracle.MIDPOINT, 0.0, 0.5, [1.0])[0]
    assert got_em == 0.625
