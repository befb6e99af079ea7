"""Pins for the oracle's Butcher tableaux (Table 1): exact-rational order
conditions from Butcher's rooted-tree theory, consistency (row sums, sum b = 1) and the
stability polynomials.  A mistyped coefficient breaks at least one order condition.
"""
import json
import os
from fractions import Fraction
from math import factorial

import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rooted_trees(n):
    """All rooted trees with n vertices, as sorted tuples of child subtrees."""
    memo = {1: [()]}

    def trees(m):
        if m in memo:
            return memo[m]
        out = set()
        # children multisets with total order m-1, built from non-increasing subtree picks
        def build(rem, max_key, acc):
            if rem == 0:
                out.add(tuple(sorted(acc)))
                return
            for k in range(min(rem, m - 1), 0, -1):
                for t in trees(k):
                    key = (k, t)
                    if max_key is not None and key > max_key:
                        continue
                    build(rem - k, key, acc + [t])
        build(m - 1, None, [])
        memo[m] = sorted(out)
        return memo[m]

    return trees(n)


def order_of(t):
    return 1 + sum(order_of(c) for c in t)


def gamma(t):
    g = order_of(t)
    for c in t:
        g *= gamma(c)
    return g


_G_CACHE = {}


def elementary_weight(tab, w, t):
    """Phi(t) = sum_i w_i * prod_{children c} (A g(c))_i, with g(leaf) = 1."""
    A, s = tab["a"], tab["s"]
    key = id(tab)

    def g(tree):
        ck = (key, tree)
        if ck in _G_CACHE:
            return _G_CACHE[ck]
        vec = [Fraction(1)] * s
        for c in tree:
            gc = g(c)
            Agc = [sum(A[i][j] * gc[j] for j in range(s) if A[i][j]) for i in range(s)]
            vec = [vec[i] * Agc[i] for i in range(s)]
        _G_CACHE[ck] = vec
        return vec

    gv = g(t)
    return sum(w[i] * gv[i] for i in range(s))


def test_tree_counts():
    # number of rooted trees of order 1..5 is 1, 1, 2, 4, 9 (OEIS A000081)
    assert [len(rooted_trees(n)) for n in range(1, 6)] == [1, 1, 2, 4, 9]


SCHEMES = [("euler", oracle.EULER, 1, None), ("rk4", oracle.RK4, 4, None),
           ("cash_karp54", oracle.CASH_KARP54, 5, 4), ("dopri5", oracle.DOPRI5, 5, 4),
           ("rkf78", oracle.RKF78, 8, 7), ("midpoint", oracle.MIDPOINT, 2, None),
           ("modified_midpoint", oracle.MODIFIED_MIDPOINT, 2, None)]


def test_tree_counts_to_order_9():
    # 1, 1, 2, 4, 9, 20, 48, 115, 286 (OEIS A000081): 200 conditions for order 8
    assert [len(rooted_trees(n)) for n in range(1, 10)] == [1, 1, 2, 4, 9, 20, 48, 115, 286]


@pytest.mark.parametrize("name,scheme,p,q", SCHEMES)
def test_order_conditions(name, scheme, p, q):
    tab = oracle.tableau(scheme)
    assert tab["order"] == p
    n_checked = 0
    for m in range(1, p + 1):
        for t in rooted_trees(m):
            assert elementary_weight(tab, tab["b"], t) == Fraction(1, gamma(t)), (name, t)
            n_checked += 1
    assert n_checked == {1: 1, 2: 2, 4: 8, 5: 17, 8: 200}[p]
    # the method is NOT of order p+1 (some tree of order p+1 fails): the order is exact
    assert any(elementary_weight(tab, tab["b"], t) != Fraction(1, gamma(t))
               for t in rooted_trees(p + 1))
    if q is not None:
        assert tab["err_order"] == q
        for m in range(1, q + 1):
            for t in rooted_trees(m):
                assert elementary_weight(tab, tab["bhat"], t) == Fraction(1, gamma(t)), (name, t)
        assert any(elementary_weight(tab, tab["bhat"], t) != Fraction(1, gamma(t))
                   for t in rooted_trees(q + 1))


@pytest.mark.parametrize("name,scheme,p,q", SCHEMES)
def test_consistency(name, scheme, p, q):
    tab = oracle.tableau(scheme)
    s = tab["s"]
    for i in range(s):
        assert sum(tab["a"][i]) == tab["c"][i]          # row-sum condition
        assert all(tab["a"][i][j] == 0 for j in range(i, s))  # explicit
    assert sum(tab["b"]) == 1                             # consistency
    if q is not None:
        assert sum(tab["bhat"]) == 1


def test_dopri5_fsal_row():
    """DOPRI5 is FSAL: its last row equals b, c_7 = 1, b_7 = 0 (Dormand & Prince)."""
    tab = oracle.tableau(oracle.DOPRI5)
    assert tab["a"][6][:6] == tab["b"][:6] and tab["b"][6] == 0 and tab["c"][6] == 1


def stability_poly(tab, w):
    """R(z) = 1 + sum_k (w^T A^{k-1} 1) z^k, coefficients k = 0..s."""
    A, s = tab["a"], tab["s"]
    coeffs = [Fraction(1)]
    v = [Fraction(1)] * s
    for _ in range(s):
        coeffs.append(sum(w[i] * v[i] for i in range(s)))
        v = [sum(A[i][j] * v[j] for j in range(s)) for i in range(s)]
    return coeffs


def test_stability_polynomials_golden():
    """Against SURVEY App. A (exact [calc] values, tests/golden/stability_polys.json)."""
    gold = json.load(open(os.path.join(GOLD, "stability_polys.json")))
    for name, scheme, p, q in SCHEMES:
        tab = oracle.tableau(scheme)
        R = stability_poly(tab, tab["b"])
        # order p => the first p+1 coefficients are 1/k!
        assert R[:p + 1] == [Fraction(1, factorial(k)) for k in range(p + 1)]
        if name not in gold:  # RKF78: no published polynomial in SURVEY; order pin above only
            continue
        want = [Fraction(c) for c in gold[name]["b"]]
        assert R[:len(want)] == want and all(c == 0 for c in R[len(want):]), name
        if q is not None:
            Rh = stability_poly(tab, tab["bhat"])
            want = [Fraction(c) for c in gold[name]["bhat"]]
            assert Rh[:len(want)] == want and all(c == 0 for c in Rh[len(want):]), name
