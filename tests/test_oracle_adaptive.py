"""Pins of the oracle's error control ("If the tolerance is violated, the step is
rejected and the step size is reduced. This is repeated until the step is accepted. For
error estimations below the tolerance, the step size is increased.").

The controller constants are Odeint's defaults as read in DESIGN.md R-12 -- the paper
delegates them to Odeint, so this part is "parity unpinned" against Odeint itself.  It
is pinned internally by (i) the accept/reject counts of an independent replay
(tests/golden/adaptive_counts.json), (ii) the closed-form tie-breaks
below, (iii) the tolerance actually achieved against the Eq. 1a/1b closed forms.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import rk_inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "adaptive_counts.json")))


@pytest.mark.parametrize("run", GOLD["runs"], ids=[r["name"] for r in GOLD["runs"]])
def test_adaptive_counts_golden(run):
    n, t0, t1 = run["n"], run["t0"], run["t1"]
    if run["problem"] == "logistic":
        u0 = rk_inputs.logistic_u0(n, t0, run["shifted"])
        s = rk_inputs.logistic_shift(n) if run["shifted"] else np.zeros(n)
        p, exact = oracle.logistic_problem(n), 1.0 / (1.0 + np.exp(-(t1 - s)))
    else:
        u0 = np.ones(n)
        p, exact = oracle.exp_problem(n, -1.0), np.full(n, math.exp(-(t1 - t0)))
    u, acc, rej, rc = oracle.integrate_adaptive(p, oracle.SCHEMES[run["scheme"]], u0, t0, t1,
                                                run["dt0"], run["tol"], run["tol"])
    assert rc == oracle.OK
    assert (acc, rej) == (run["accepted"], run["rejected"])
    err = float(np.max(np.abs(u - exact)))
    assert 0.9 * run["final_err"] <= err <= 1.1 * run["final_err"]
    assert err <= 100 * run["tol"]  # final error <= 100*rtol


def test_controller_tie_breaks():
    """DESIGN.md R-14: E == 1 accepts; E == 0.5 leaves dt; E == 0 clamps to 5^-5 (x4.5)."""
    assert oracle.controller(1.0, 0.5) == (True, 0.5)   # accepted, no growth at E >= 0.5
    assert oracle.controller(0.5, 0.5) == (True, 0.5)
    acc, dt = oracle.controller(0.0, 1.0)
    assert acc and abs(dt - 4.5) < 1e-14            # 0.9 * (5^-5)^(-1/5) = 0.9 * 5
    acc, dt = oracle.controller(1.0 + 2 ** -52, 1.0)
    assert not acc and dt < 1.0                      # rejected, decreased
    acc, dt = oracle.controller(1e6, 1.0)
    assert not acc and dt == 0.2                     # shrink floor 1/5


@pytest.mark.parametrize("E", [1e-9, 0.01, 0.3, 0.49])
def test_accept_grows(E):
    acc, dt = oracle.controller(E, 1.0)
    assert acc and 1.0 < dt <= 4.5 + 1e-14
    assert abs(dt - 0.9 * max(E, 5.0 ** -5) ** (-0.2)) < 1e-12


@pytest.mark.parametrize("E", [1.5, 10.0, 300.0])
def test_reject_shrinks(E):
    acc, dt = oracle.controller(E, 1.0)
    assert not acc and 0.2 <= dt < 0.9
    assert abs(dt - max(0.9 * E ** (-1.0 / 3.0), 0.2)) < 1e-15


def test_error_ratio_formula_pins():
    """r = |e| / (atol + rtol*(|u| + dt*|k1|)): zero error -> 0; boundary values."""
    assert oracle.error_ratio_max([0.0], [5.0], [1.0], 0.1, 1e-6, 1e-6) == 0.0
    # e = 1e-6, u = k1 = 0, rtol = 0 -> exactly 1 (S:L82 analogue)
    assert oracle.error_ratio_max([1e-6], [0.0], [0.0], 0.5, 1e-6, 0.0) == 1.0
    # the k1 term: u = 0, k1 = 1, dt = 1, atol tiny: r = |e| / (rtol*dt*|k1|)
    r = oracle.error_ratio_max([2e-4], [0.0], [1.0], 1.0, 1e-300, 1e-4)
    assert abs(r - 2.0) < 1e-12
    assert math.isnan(oracle.error_ratio_max([1.0, float("nan")], [0.0, 0.0], [0.0, 0.0],
                                             1.0, 1.0, 1.0))


def test_adaptive_rejects_diverged_state():
    """A NaN error ratio is a divergence (R-14), not an accepted step."""
    p = oracle.logistic_problem(2)
    u, acc, rej, rc = oracle.integrate_adaptive(p, oracle.DOPRI5, [0.5, float("nan")], 0.0, 1.0,
                                                0.1, 1e-8, 1e-8)
    assert rc == oracle.ERR_DIVERGED and acc == 0


def test_adaptive_unsupported_for_fixed_schemes():
    p = oracle.logistic_problem(1)
    for s in (oracle.EULER, oracle.RK4):
        assert oracle.integrate_adaptive(p, s, [0.5], 0.0, 1.0, 0.1, 1e-8, 1e-8)[3] == \
            oracle.ERR_UNSUPPORTED


def test_zero_rhs_one_step():
    """du/dt = 0: one accepted step of size t1 - t0 when dt0 already covers it."""
    p = oracle.exp_problem(3, 0.0)
    u, acc, rej, rc = oracle.integrate_adaptive(p, oracle.DOPRI5, [1.0, 2.0, 3.0], 0.0, 1.0, 2.0,
                                                1e-8, 1e-8)
    assert rc == 0 and (acc, rej) == (1, 0) and list(u) == [1.0, 2.0, 3.0]


def test_adaptive_hits_t1_exactly():
    """Last step truncated to t1 (R-16): decay solved to t1 = 1 within tolerance."""
    p = oracle.exp_problem(1, -1.0)
    for dt0 in (0.013, 0.37, 5.0):
        u, acc, rej, rc = oracle.integrate_adaptive(p, oracle.DOPRI5, [1.0], 0.0, 1.0, dt0,
                                                    1e-10, 1e-10)
        assert rc == 0 and abs(u[0] - math.exp(-1.0)) < 1e-8


def test_rkf78_adaptive_meets_tolerance():
    """RKF78 error-controlled (stepper order 8, error order 7, R-12) on Eq. 1b:
    reaches t1 exactly, final error <= 100*tol, rejections recover."""
    u0 = rk_inputs.logistic_u0(1, -5.0, shifted=False)
    for tol in (1e-6, 1e-8, 1e-10):
        u, acc, rej, rc = oracle.integrate_adaptive(oracle.logistic_problem(1), oracle.RKF78, u0,
                                                    -5.0, 5.0, 0.1, tol, tol)
        assert rc == oracle.OK and acc > 0
        assert abs(u[0] - 1.0 / (1.0 + math.exp(-5.0))) <= 100 * tol


def _cr_pow(x: float, y: float) -> float:
    """x^y correctly rounded to double: Python's decimal computes non-integral powers
    correctly rounded at the context precision (60 digits here), float() rounds once more."""
    from decimal import Decimal, localcontext
    with localcontext() as c:
        c.prec = 60
        return float(Decimal(x) ** Decimal(y))


def test_controller_pow_correctly_rounded():
    """DESIGN.md R-27: the controller's pow is the correctly rounded x^y (the oracle evaluates
    it in binary128 and rounds once; the library in double-double).  Every dt the oracle
    proposes equals the one built from 60-digit decimal powers with the same fp64 steps
    (fac = 0.9 * x^y, clamps, dt * fac).  glibc's pow misses ~0.1 % of these arguments by an
    ulp, so this pin separates the two readings."""
    rng = np.random.default_rng(27)
    Es = list(10.0 ** rng.uniform(-12, 4, 3000)) + [0.3, 0.49, 1.5, 10.0, 5.0 ** -5, 1e-300]
    emin = _cr_pow(5.0, -5.0)
    for E in Es:
        E = float(E)
        for dt0 in (1.0, 0.1):
            acc, dt = oracle.controller(E, dt0)
            if E > 1.0:
                want = dt0 * max(0.9 * _cr_pow(E, -1.0 / 3.0), 0.2)
            elif E < 0.5:
                want = dt0 * (0.9 * _cr_pow(max(E, emin), -1.0 / 5.0))
            else:
                want = dt0
            assert acc == (E <= 1.0) and dt == want, (E, dt0, dt, want)
            acc_s, dt_s = oracle.controller_spec(E, dt0, 5)
            if E <= 1.0:
                want_s = dt0 * min(5.0, max(0.2, 0.9 * _cr_pow(E, -1.0 / 5.0)))
            else:
                want_s = dt0 * max(0.2, 0.9 * _cr_pow(E, -1.0 / 4.0))
            assert acc_s == (E <= 1.0) and dt_s == want_s, (E, dt0, dt_s, want_s)


def test_dt_underflow_floor():
    """DESIGN.md R-29: with an unattainable tolerance every try is rejected with the
    1/5 shrink floor (E ~ 1e290 >> 4.5^3), so dt_k = dt0 * 0.2^k (fp64 products) until the first
    dt below 16 eps max(|t|, 1); that try is not taken: RK_ERR_DT_UNDERFLOW after exactly k
    rejections, u untouched.  (An error ratio that is not huge would shrink by less than 5x.)"""
    n = 8
    u0 = rk_inputs.logistic_u0(n)
    dt, k = 0.1, 0
    while not dt < 16 * np.finfo(float).eps * max(abs(-5.0), 1.0):
        dt, k = dt * 0.2, k + 1
    u, acc, rej, rc = oracle.integrate_adaptive(oracle.logistic_problem(n), oracle.DOPRI5, u0, -5.0, 5.0, 0.1,
                                                1e-300, 1e-300)
    assert rc == oracle.ERR_DT_UNDERFLOW and acc == 0 and rej == k and k == 19
    assert np.array_equal(u, u0)
