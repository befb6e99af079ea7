"""Pins of the oracle's alternative controller reading (R-28): SPEC's elementary
controller with SPEC's elementwise error ratio.

The paper only fixes the semantics ("If the tolerance is violated, the step is
rejected and the step size is reduced. This is repeated until the step is accepted. For
error estimations below the tolerance, the step size is increased.") and delegates the
constants to Odeint; SURVEY Z12 ships Odeint's reading (R-12) and keeps SPEC's
behind an option.  This reading is pinned by
  (i)   SPEC's printed examples (S:L79-82 ratio, S:L231-232 controller),
  (ii)  the accept/reject counts of the survey's independent replay (SURVEY Z12 [calc]:
        logistic DOPRI5 tol 1e-8 dt0 0.1 accepts 46 and rejects 3 under SPEC's reading),
  (iii) a closed-form replay on the linear test equation u' = u, where one DOPRI5 try gives
        u_new = R(z) u and e = E(z) u exactly up to rounding (SURVEY App. A polynomials,
        tests/golden/stability_polys.json), so the ratio of every try is known without the
        oracle's stage arithmetic; u grows, so max(|u_old|, |u_new|) = |u_new| there and a
        ratio built on |u_old| alone fails it,
  (iv)  SPEC's invariants (dt_next within [0.2 dt, 5 dt]; rejected tries leave u).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import rk_inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "adaptive_counts.json")))
POLY = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "stability_polys.json")))


def test_spec_ratio_examples():
    """zero error -> 0; e = atol, u = 0, rtol = 0 -> 1; 2e-4/(1e-4 + 1e-4*1) -> 1."""
    assert oracle.error_ratio_max_spec([0.0], [3.0], [4.0], 1e-6, 1e-6) == 0.0
    assert oracle.error_ratio_max_spec([1e-6], [0.0], [0.0], 1e-6, 0.0) == 1.0
    assert oracle.error_ratio_max_spec([2e-4], [1.0], [1.0], 1e-4, 1e-4) == 1.0


def test_spec_ratio_uses_larger_magnitude():
    """The denominator takes max(|u_old|, |u_new|), either side, signs stripped."""
    assert oracle.error_ratio_max_spec([3.0], [-1.0], [2.0], 1e-300, 1.0) == 1.5
    assert oracle.error_ratio_max_spec([3.0], [-2.0], [1.0], 1e-300, 1.0) == 1.5
    assert oracle.error_ratio_max_spec([-6.0, 1.0], [2.0, 1.0], [-3.0, 1.0], 1e-300, 1.0) == 2.0
    assert math.isnan(oracle.error_ratio_max_spec([1.0, float("nan")], [1.0, 1.0], [1.0, 1.0],
                                                  1.0, 1.0))


def test_spec_controller_examples():
    """err = 0 -> accepted, dt_next = grow_cap*dt = 5 dt.
    S:L232: err = 1 -> accepted, dt_next = 0.9 dt (safety-adjusted, smaller)."""
    assert oracle.controller_spec(0.0, 1.0) == (True, 5.0)
    acc, dt = oracle.controller_spec(1.0, 1.0)
    assert acc and dt == 0.9
    acc, dt = oracle.controller_spec(1.0 + 2 ** -52, 1.0)
    assert not acc and dt <= 0.9
    assert oracle.controller_spec(1e30, 1.0) == (False, 0.2)   # shrink floor
    assert oracle.controller_spec(1e-30, 1.0) == (True, 5.0)   # grow cap


def test_spec_controller_always_rescales():
    """Unlike Odeint (dt kept for 0.5 <= E <= 1), SPEC rescales on every accept."""
    acc, dt = oracle.controller_spec(0.75, 1.0)
    assert acc and dt < 1.0
    assert oracle.controller(0.75, 1.0) == (True, 1.0)


def test_spec_dt_bounds_invariant():
    """dt_next in [shrink_floor*dt, grow_cap*dt] always; accept iff E <= 1."""
    rng = np.random.default_rng(7)
    for E in np.concatenate([10.0 ** rng.uniform(-12, 12, 400), [0.0, 1.0, 0.5, 2.0]]):
        for p in (5, 8):
            acc, dt = oracle.controller_spec(float(E), 2.0, p)
            assert acc == (E <= 1.0)
            assert 0.4 <= dt <= 10.0


def test_spec_counts_golden():
    """SURVEY Z12 [calc]: the independent replay of SPEC's reading on the logistic, DOPRI5,
    tol 1e-8, dt0 0.1 accepts 46 steps and rejects 3 (Odeint's reading: 46 / 6)."""
    run = GOLD["spec_runs"][0]
    u0 = rk_inputs.logistic_u0(1, run["t0"], False)
    u, acc, rej, rc = oracle.integrate_adaptive_ctrl(
        oracle.logistic_problem(1), oracle.SCHEMES[run["scheme"]], u0, run["t0"], run["t1"],
        run["dt0"], run["tol"], run["tol"], oracle.CTRL_SPEC)
    assert rc == oracle.OK and (acc, rej) == (run["accepted"], run["rejected"])
    exact = 1.0 / (1.0 + math.exp(-run["t1"]))
    assert abs(u[0] - exact) <= 100 * run["tol"]


def _poly(coefs, z):
    return sum(Fraction(c) * z ** k for k, c in enumerate(coefs))


def _closed_form_replay(scheme, p, t0, t1, dt0, tol):
    """SPEC's loop on u' = u with u0 = 1, each try's u_new and e taken from the
    closed-form stability polynomials in exact rationals; only t, dt and the controller
    arithmetic are floats.  Returns (accepted, rejected, u)."""
    b, bh = POLY[scheme]["b"], POLY[scheme]["bhat"]
    u, t, dt = Fraction(1), t0, dt0
    acc = rej = 0
    while t1 - t > 2.0 ** -52:
        if (t + dt) - t1 > 2.0 ** -52:
            dt = t1 - t
        while True:
            z = Fraction(dt)
            un = _poly(b, z) * u
            e = (_poly(b, z) - _poly(bh, z)) * u
            E = float(abs(e) / (Fraction(tol) + Fraction(tol) * max(abs(u), abs(un))))
            if E <= 1.0:
                fac = min(5.0, max(0.2, 0.9 * E ** (-1.0 / p)))
                u, t, dt = un, t + dt, dt * fac
                acc += 1
                break
            dt = dt * max(0.2, 0.9 * E ** (-1.0 / (p - 1)))
            rej += 1
    return acc, rej, float(u)


@pytest.mark.parametrize("scheme,tol,dt0", [("dopri5", 1e-8, 2.0), ("dopri5", 1e-6, 1.0),
                                            ("cash_karp54", 1e-8, 2.0),
                                            ("cash_karp54", 1e-10, 1.0)])
def test_spec_linear_closed_form_replay(scheme, tol, dt0):
    acc_r, rej_r, u_r = _closed_form_replay(scheme, 5, 0.0, 5.0, dt0, tol)
    u, acc, rej, rc = oracle.integrate_adaptive_ctrl(oracle.exp_problem(1, 1.0),
                                                     oracle.SCHEMES[scheme], [1.0], 0.0, 5.0,
                                                     dt0, tol, tol, oracle.CTRL_SPEC)
    assert rc == oracle.OK
    assert (acc, rej) == (acc_r, rej_r) and rej > 0
    assert abs(u[0] - u_r) <= 1e-12 * abs(u_r)
    assert abs(u[0] - math.exp(5.0)) <= 1e3 * tol * math.exp(5.0)


def test_spec_rejected_try_leaves_state_and_hits_t1():
    """rejected steps never mutate u; du/dt = 0 reaches t1 exactly with cap-limited
    growth: from dt0 = 0.1 on [0, 10]: 0.1, 0.5, 2.5, then 6.9 (truncated)."""
    p = oracle.exp_problem(3, 0.0)
    u, acc, rej, rc = oracle.integrate_adaptive_ctrl(p, oracle.DOPRI5, [1.0, -2.0, 3.0], 0.0, 10.0,
                                                     0.1, 1e-8, 1e-8, oracle.CTRL_SPEC)
    assert rc == 0 and (acc, rej) == (4, 0) and list(u) == [1.0, -2.0, 3.0]


def test_spec_stall_and_divergence():
    p = oracle.logistic_problem(1)
    u, acc, rej, rc = oracle.integrate_adaptive_ctrl(p, oracle.DOPRI5, [0.5], 0.0, 1.0, 0.1,
                                                     1e-30, 0.0, oracle.CTRL_SPEC, max_tries=3)
    assert rc == oracle.ERR_STALL and acc == 0 and rej == 3
    u, acc, rej, rc = oracle.integrate_adaptive_ctrl(p, oracle.DOPRI5, [float("nan")], 0.0, 1.0,
                                                     0.1, 1e-8, 1e-8, oracle.CTRL_SPEC)
    assert rc == oracle.ERR_DIVERGED


def test_odeint_ctrl_entry_is_the_default_driver():
    """integrate_adaptive_ctrl(ODEINT) is bit for bit the default driver."""
    u0 = rk_inputs.logistic_u0(64, -5.0, True)
    a = oracle.integrate_adaptive(oracle.logistic_problem(64), oracle.DOPRI5, u0, -5.0, 5.0, 0.1,
                                  1e-8, 1e-8)
    b = oracle.integrate_adaptive_ctrl(oracle.logistic_problem(64), oracle.DOPRI5, u0, -5.0, 5.0,
                                       0.1, 1e-8, 1e-8, oracle.CTRL_ODEINT)
    assert a[1:] == b[1:] and np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64))
