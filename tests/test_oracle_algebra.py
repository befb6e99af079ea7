"""Pins of the oracle's algebra ops (P:L133-135 for_each#/for_each_norm)."""
import numpy as np
import pytest

import oracle
import rk_inputs


def test_lincomb_spec_examples():
    assert list(oracle.lincomb([1.0], [[2.0, 3.0]])) == [2.0, 3.0]
    assert list(oracle.lincomb([1.0, 0.1], [[1.0, 1.0], [1.0, 1.0]])) == [1.1, 1.1]
    # RK4 update with k from du/dt = u, dt = 1: k1=1, k2=1.5, k3=1.75, k4=2.75
    v = oracle.lincomb([1.0, 1 / 6, 2 / 6, 2 / 6, 1 / 6], [[1.0], [1.0], [1.5], [1.75], [2.75]])
    assert abs(v[0] - 2.708333333333333) < 1e-15


def test_lincomb_arity_limits():
    x = rk_inputs.random_state(5, 1)
    for k in (1, 7, 14):
        oracle.lincomb(np.ones(k), [x] * k)
    with pytest.raises(ValueError):
        oracle.lincomb(np.ones(15), [x] * 15)


def test_lincomb_is_exact_for_dyadic_data():
    """Dyadic inputs/coefficients with small exponent range: every partial sum is exact,
    so the result equals the exact rational sum (independent of evaluation order)."""
    rng = np.random.default_rng(5)
    k, n = 14, 64
    ins = [rng.integers(-2 ** 20, 2 ** 20, size=n) / 2.0 ** 10 for _ in range(k)]
    coef = rng.integers(-64, 64, size=k) / 8.0
    got = oracle.lincomb(coef, ins)
    want = sum(int(c * 8) * np.round(x * 2 ** 10).astype(np.int64) for c, x in zip(coef, ins))
    assert np.array_equal(got, want / 2.0 ** 13)


def test_norm_inf_spec_examples():
    assert oracle.norm_inf([-3.0, 2.0, 0.5]) == 3.0
    assert oracle.norm_inf([0.0, 0.0, 0.0, 0.0]) == 0.0
    assert oracle.norm_inf([1e-16, -2e-16]) == 2e-16
    x = rk_inputs.random_state(1000, 9)
    assert oracle.norm_inf(-2.0 * x) == 2.0 * oracle.norm_inf(x)
