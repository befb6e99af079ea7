"""Pins of the oracle's Gray–Scott RHS (Eq. 3 / Listing 2) with the
7-point periodic Laplacian of DESIGN.md R-3, and of stepper+stencil together.

Closed forms used:
  * (C0, C1) = (1, 0) is a steady state -> RHS exactly 0.
  * Linear reductions: with C1 = 0, v = C0 - 1 obeys v' = d1*Lap v - F v; with F = 0 and
    C0 = 0, C1' = d2*Lap C1 - K C1.  A Fourier mode prod_a cos(2 pi m_a i_a / n_a) is an
    eigenvector of the discrete Laplacian with eigenvalue -(4/h^2) sum_a sin^2(pi m_a/n_a),
    so after n RK steps the amplitude is exactly R(z)^n with z = (d*lambda - rate)*dt.
  * Reaction coupling: with d = F = K = 0 the homogeneous system is C0' = -C0 C1^2,
    C1' = +C0 C1^2; C0 + C1 = A is conserved and G(C1) = -1/(A C1) + ln(C1/(A-C1))/A^2
    satisfies G(C1(t)) - G(C1(0)) = t (separable ODE, integrated by partial fractions).
  * The discrete Laplacian telescopes: sum over the periodic grid is 0.
  * Second-order consistency of the stencil on sin(2 pi x / L).
Non-cubic grids with distinct mode numbers catch transposed axes.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import rk_inputs

POLYS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "stability_polys.json")))
NAMES = {oracle.EULER: "euler", oracle.RK4: "rk4", oracle.CASH_KARP54: "cash_karp54",
         oracle.DOPRI5: "dopri5"}


def R(scheme, z):
    return float(sum(Fraction(c) * Fraction(z) ** k for k, c in enumerate(POLYS[NAMES[scheme]]["b"])))


def mode(nx, ny, nz, m):
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return (np.cos(2 * np.pi * m[0] * x / nx) * np.cos(2 * np.pi * m[1] * y / ny)
            * np.cos(2 * np.pi * m[2] * z / nz))


def lam(nx, ny, nz, m, h):
    return -(4.0 / h ** 2) * sum(math.sin(math.pi * mi / ni) ** 2 for mi, ni in zip(m, (nx, ny, nz)))


def pack(c0, c1):
    """[z][y][x] fields -> [z][c][y][x] state."""
    return np.ascontiguousarray(np.stack([c0, c1], axis=1))


def test_steady_state_exact_zero():
    p = oracle.gray_scott_problem(7, 5, 4)
    u = pack(np.ones((4, 5, 7)), np.zeros((4, 5, 7)))
    assert np.all(oracle.rhs(p, u) == 0.0)


def test_homogeneous_reaction_values():
    """Constant fields: the stencil is exactly 0 in difference form (R-3), so the
    RHS reduces to the reaction terms; at C0=1 the F terms cancel exactly: f0 = -C1^2."""
    p = oracle.gray_scott_problem(3, 4, 5, F=0.014, K=0.053)
    for c1 in (0.0, 0.25, 0.5, 1.0):
        u = pack(np.ones((5, 4, 3)), np.full((5, 4, 3), c1))
        f = oracle.rhs(p, u).reshape(5, 2, 4, 3)
        assert np.all(f[:, 0] == -(c1 * c1))


@pytest.mark.parametrize("scheme", [oracle.EULER, oracle.RK4, oracle.CASH_KARP54, oracle.DOPRI5])
@pytest.mark.parametrize("dims,m", [((16, 12, 10), (1, 2, 3)), ((10, 16, 12), (3, 0, 1)),
                                    ((12, 10, 16), (0, 1, 5))])
def test_fourier_mode_c0(scheme, dims, m):
    nx, ny, nz = dims
    h, d1, F, dt, n, eps = 2.5 / 64, 2e-4, 0.014, 1.0, 12, 1e-3
    p = oracle.gray_scott_problem(nx, ny, nz, d1=d1, d2=1e-4, F=F, K=0.053, h=h)
    md = mode(nx, ny, nz, m)
    u = pack(1.0 + eps * md, np.zeros_like(md))
    for _ in range(n):
        u = oracle.step(p, scheme, 0.0, dt, u)
    amp = R(scheme, (d1 * lam(nx, ny, nz, m, h) - F) * dt) ** n
    got = u.reshape(nz, 2, ny, nx)
    assert np.max(np.abs(got[:, 0] - (1.0 + eps * amp * md))) < 1e-14
    assert np.all(got[:, 1] == 0.0)


@pytest.mark.parametrize("scheme", [oracle.RK4, oracle.DOPRI5])
def test_fourier_mode_c1(scheme):
    nx, ny, nz, m = 12, 14, 16, (2, 1, 3)
    h, d2, K, dt, n, eps = 2.5 / 64, 1e-4, 0.053, 1.0, 15, 1e-2
    p = oracle.gray_scott_problem(nx, ny, nz, d1=2e-4, d2=d2, F=0.0, K=K, h=h)
    md = mode(nx, ny, nz, m)
    u = pack(np.zeros_like(md), eps * md)
    for _ in range(n):
        u = oracle.step(p, scheme, 0.0, dt, u)
    amp = R(scheme, (d2 * lam(nx, ny, nz, m, h) - K) * dt) ** n
    got = u.reshape(nz, 2, ny, nx)
    assert np.all(got[:, 0] == 0.0)
    assert np.max(np.abs(got[:, 1] - eps * amp * md)) < 1e-15


def test_reaction_coupling_closed_form():
    p = oracle.gray_scott_problem(2, 2, 2, d1=0.0, d2=0.0, F=0.0, K=0.0)
    s, T, dt = 0.5, 2.0, 1.0 / 256
    A = 1.0 + s
    u = pack(np.ones((2, 2, 2)), np.full((2, 2, 2), s))
    for _ in range(int(T / dt)):
        u = oracle.step(p, oracle.RK4, 0.0, dt, u)
    c = u.reshape(2, 2, 2, 2)
    c0, c1 = float(c[0, 0, 0, 0]), float(c[0, 1, 0, 0])
    G = lambda x: -1.0 / (A * x) + math.log(x / (A - x)) / A ** 2
    assert abs(G(c1) - G(s) - T) < 1e-10
    assert abs(c0 + c1 - A) < 1e-14


def test_mass_identity_random_fields():
    """sum_cells f = sum_cells reaction (Laplacian telescopes); and the reaction's C0*C1^2
    terms cancel in f0 + f1 (mass exchange between the species)."""
    rng = np.random.default_rng(7)
    nz, ny, nx = 5, 6, 8
    u = rng.uniform(0.0, 1.0, size=(nz, 2, ny, nx))
    p_lap = oracle.gray_scott_problem(nx, ny, nz, d1=1.0, d2=1.0, F=0.0, K=0.0)
    p_rx = oracle.gray_scott_problem(nx, ny, nz, d1=0.0, d2=0.0, F=0.0, K=0.0)
    lap_part = oracle.rhs(p_lap, u) - oracle.rhs(p_rx, u)
    scale = np.max(np.abs(lap_part))
    assert abs(lap_part.reshape(nz, 2, -1)[:, 0].sum()) < 1e-11 * scale * u.size
    assert abs(lap_part.reshape(nz, 2, -1)[:, 1].sum()) < 1e-11 * scale * u.size
    F, K = 0.014, 0.053
    p = oracle.gray_scott_problem(nx, ny, nz, d1=0.0, d2=0.0, F=F, K=K)
    f = oracle.rhs(p, u).reshape(nz, 2, ny, nx)
    c0, c1 = u[:, 0], u[:, 1]
    assert np.max(np.abs(f[:, 0] + f[:, 1] - (F * (1 - c0) - (F + K) * c1))) < 1e-15


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_stencil_second_order(axis):
    """Lap sin(2 pi x/L) -> -(2 pi/L)^2 sin, error x4 per halving of h."""
    L = 2.5
    errs = []
    for n in (16, 32, 64):
        dims = [4, 4, 4]
        dims[axis] = n
        nx, ny, nz = dims
        h = L / n
        idx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")[2 - axis]
        v = np.sin(2 * np.pi * idx * h / L)
        p = oracle.gray_scott_problem(nx, ny, nz, d1=1.0, d2=0.0, F=0.0, K=0.0, h=h)
        f = oracle.rhs(p, pack(v, np.zeros_like(v))).reshape(nz, 2, ny, nx)[:, 0]
        errs.append(np.max(np.abs(f + (2 * np.pi / L) ** 2 * v)))
    for a, b in zip(errs, errs[1:]):
        assert 3.2 < a / b < 4.8, errs


def test_translation_equivariance_bitwise():
    """The periodic stencil commutes exactly with periodic shifts of the grid."""
    rng = np.random.default_rng(3)
    nz, ny, nx = 4, 5, 6
    u = rng.uniform(0, 1, size=(nz, 2, ny, nx))
    p = oracle.gray_scott_problem(nx, ny, nz)
    f = oracle.rhs(p, u).reshape(nz, 2, ny, nx)
    us = np.ascontiguousarray(np.roll(u, shift=(1, 2, 3), axis=(0, 2, 3)))
    fs = oracle.rhs(p, us).reshape(nz, 2, ny, nx)
    assert np.array_equal(fs, np.roll(f, shift=(1, 2, 3), axis=(0, 2, 3)))


def test_config3_bounded_and_patterned():
    """64^3, RK4, dt=1, t in [0,20]: fields stay within [0,1] (
    SPEC bound [-0.05, 1.3]) and the seeded cube spreads."""
    n = 64
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    p = oracle.gray_scott_problem(n, n, n)
    u, steps = oracle.integrate_const(p, oracle.RK4, u0, 0.0, 20.0, 1.0)
    assert steps == 20
    c = u.reshape(n, 2, n, n)
    assert c.min() >= 0.0 and c.max() <= 1.0
    assert np.count_nonzero(c[:, 1] > 1e-6) > np.count_nonzero(u0.reshape(n, 2, n, n)[:, 1] > 0)
