"""ctypes wrapper of the plain-C fp64 oracle (oracle/rk_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline legs (``cpu_baseline``, ``--impl reference``) may import this module.  The
product package ``paper_2309_05331_b200`` never imports it and shares no code with it.

Every function here is argument marshalling for the C oracle; the arithmetic lives in
rk_oracle.c, each function of which cites the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rk_oracle.c")
_HDR = os.path.join(_HERE, "rk_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

EULER, RK4, CASH_KARP54, DOPRI5, RKF78, MIDPOINT, MODIFIED_MIDPOINT = 0, 1, 2, 3, 4, 5, 6
SCHEMES = {"euler": EULER, "rk4": RK4, "cash_karp54": CASH_KARP54, "dopri5": DOPRI5,
           "rkf78": RKF78, "midpoint": MIDPOINT, "modified_midpoint": MODIFIED_MIDPOINT}
RHS_EXP, RHS_LOGISTIC, RHS_GRAY_SCOTT = 0, 1, 2
OK, ERR_ARG, ERR_UNSUPPORTED, ERR_DIVERGED, ERR_STALL, ERR_DT_UNDERFLOW = 0, 1, 2, 3, 4, 5

# -O2 -ffp-contract=off: no FMA contraction; no -ffast-math: IEEE division, no FTZ/DAZ.
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree (gcc).  Returns the library path."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(f) > os.path.getmtime(_LIB) for f in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lquadmath", "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Problem(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int), ("ncomp", ctypes.c_int), ("n", ctypes.c_int64),
        ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
        ("lam", ctypes.c_double), ("d1", ctypes.c_double), ("d2", ctypes.c_double),
        ("F", ctypes.c_double), ("K", ctypes.c_double), ("h", ctypes.c_double),
    ]

    @property
    def count(self) -> int:
        return int(self.n) * int(self.ncomp)


def exp_problem(n: int, lam: float) -> Problem:
    """du/dt = lam*u on n independent elements (Eq. 1a; R-9)."""
    return Problem(RHS_EXP, 1, n, 0, 0, 0, lam, 0.0, 0.0, 0.0, 0.0, 0.0)


def logistic_problem(n: int) -> Problem:
    """du/dt = u(1-u) on n independent elements (Eq. 1b)."""
    return Problem(RHS_LOGISTIC, 1, n, 0, 0, 0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0)


def gray_scott_problem(nx, ny, nz, d1=2e-4, d2=1e-4, F=0.014, K=0.053, h=2.5 / 64) -> Problem:
    """3D Gray–Scott, Listing 2, periodic grid, layout [z][c][y][x]."""
    return Problem(RHS_GRAY_SCOTT, 2, nx * ny * nz, nx, ny, nz, 0.0, d1, d2, F, K, h)


_lib = None


def lib():
    global _lib
    if _lib is None:
        # ORACLE_LIB: an alternative build of the same source (the sanitizer test's ASan/UBSan build)
        L = ctypes.CDLL(os.environ.get("ORACLE_LIB") or build())
        P = ctypes.POINTER(Problem)
        dp = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.orc_tableau.argtypes = [ctypes.c_int] + [i64p] * 8 + [ctypes.POINTER(ctypes.c_int)] * 2
        L.orc_tableau.restype = ctypes.c_int
        L.orc_rhs.argtypes = [P, dp, dp]
        L.orc_rhs.restype = None
        L.orc_step.argtypes = [P, ctypes.c_int, ctypes.c_double, ctypes.c_double, dp, dp, dp]
        L.orc_step.restype = ctypes.c_int
        L.orc_error_ratio_max.argtypes = [ctypes.c_int64, dp, dp, dp, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_double]
        L.orc_error_ratio_max.restype = ctypes.c_double
        L.orc_controller.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int, dp]
        L.orc_controller.restype = ctypes.c_int
        L.orc_integrate_const.argtypes = [P, ctypes.c_int, dp, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, i64p]
        L.orc_integrate_const.restype = ctypes.c_int
        L.orc_integrate_adaptive.argtypes = [P, ctypes.c_int, dp, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                             i64p, i64p]
        L.orc_integrate_adaptive.restype = ctypes.c_int
        L.orc_error_ratio_max_spec.argtypes = [ctypes.c_int64, dp, dp, dp, ctypes.c_double,
                                               ctypes.c_double]
        L.orc_error_ratio_max_spec.restype = ctypes.c_double
        L.orc_controller_spec.argtypes = [ctypes.c_double, ctypes.c_int, dp]
        L.orc_controller_spec.restype = ctypes.c_int
        L.orc_integrate_adaptive_ctrl.argtypes = [P, ctypes.c_int, dp, ctypes.c_double,
                                                  ctypes.c_double, ctypes.c_double,
                                                  ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                                  ctypes.c_int, i64p, i64p]
        L.orc_integrate_adaptive_ctrl.restype = ctypes.c_int
        L.orc_lincomb.argtypes = [ctypes.c_int64, dp, ctypes.c_int, dp, ctypes.POINTER(dp)]
        L.orc_lincomb.restype = ctypes.c_int
        L.orc_norm_inf.argtypes = [ctypes.c_int64, dp]
        L.orc_norm_inf.restype = ctypes.c_double
        L.orc_ab_coefficients.argtypes = [ctypes.c_int, i64p, i64p]
        L.orc_ab_coefficients.restype = ctypes.c_int
        L.orc_ab_integrate.argtypes = [P, ctypes.c_int, dp, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_int64, dp]
        L.orc_ab_integrate.restype = ctypes.c_int
        L.orc_am_coefficients.argtypes = [ctypes.c_int, i64p, i64p]
        L.orc_am_coefficients.restype = ctypes.c_int
        L.orc_abm_integrate.argtypes = [P, ctypes.c_int, dp, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_int64, dp]
        L.orc_abm_integrate.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _arr(u) -> np.ndarray:
    return np.ascontiguousarray(u, dtype=np.float64)


def tableau(scheme: int) -> dict:
    """The oracle's Butcher tableau as exact Fractions (for the order-condition pins)."""
    S = 13
    bufs = [(ctypes.c_int64 * (S * S))() for _ in range(2)] + \
           [(ctypes.c_int64 * S)() for _ in range(6)]
    order, err_order = ctypes.c_int(), ctypes.c_int()
    s = lib().orc_tableau(scheme, *bufs, ctypes.byref(order), ctypes.byref(err_order))
    if s < 0:
        raise ValueError(f"bad scheme {scheme}")
    an, ad, bn, bd, hn, hd, cn, cd = bufs
    return {
        "s": s,
        "a": [[Fraction(an[i * s + j], ad[i * s + j]) for j in range(s)] for i in range(s)],
        "b": [Fraction(bn[i], bd[i]) for i in range(s)],
        "bhat": [Fraction(hn[i], hd[i]) for i in range(s)],
        "c": [Fraction(cn[i], cd[i]) for i in range(s)],
        "order": order.value,
        "err_order": err_order.value,
    }


def rhs(p: Problem, u) -> np.ndarray:
    u = _arr(u)
    assert u.size == p.count
    f = np.empty_like(u)
    lib().orc_rhs(ctypes.byref(p), _ptr(u), _ptr(f))
    return f


def step(p: Problem, scheme: int, t: float, dt: float, u, with_error: bool = False):
    """One textbook RK step.  Returns u_new, or (u_new, err) if with_error."""
    u = _arr(u)
    assert u.size == p.count
    un = np.empty_like(u)
    er = np.empty_like(u) if with_error else None
    rc = lib().orc_step(ctypes.byref(p), scheme, t, dt, _ptr(u), _ptr(un),
                        _ptr(er) if with_error else None)
    if rc != OK:
        raise RuntimeError(f"orc_step failed rc={rc}")
    return (un, er) if with_error else un


def error_ratio_max(err, u, k1, dt, atol, rtol) -> float:
    err, u, k1 = _arr(err), _arr(u), _arr(k1)
    return lib().orc_error_ratio_max(err.size, _ptr(err), _ptr(u), _ptr(k1), dt, atol, rtol)


def controller(E: float, dt: float, p: int = 5, q: int = 4):
    """Returns (accepted, dt_next)."""
    d = ctypes.c_double(dt)
    acc = lib().orc_controller(E, p, q, ctypes.byref(d))
    return bool(acc), d.value


def error_ratio_max_spec(err, u_old, u_new, atol, rtol) -> float:
    """SPEC's elementwise_err_ratio (R-28)."""
    err, u_old, u_new = _arr(err), _arr(u_old), _arr(u_new)
    return lib().orc_error_ratio_max_spec(err.size, _ptr(err), _ptr(u_old), _ptr(u_new), atol, rtol)


def controller_spec(E: float, dt: float, p: int = 5):
    """SPEC's elementary controller (R-28).  Returns (accepted, dt_next)."""
    d = ctypes.c_double(dt)
    acc = lib().orc_controller_spec(E, p, ctypes.byref(d))
    return bool(acc), d.value


def integrate_const(p: Problem, scheme: int, u, t0: float, t1: float, dt: float):
    """Returns (u_final, steps)."""
    u = _arr(u).copy()
    n = ctypes.c_int64()
    rc = lib().orc_integrate_const(ctypes.byref(p), scheme, _ptr(u), t0, t1, dt, ctypes.byref(n))
    if rc != OK:
        raise RuntimeError(f"orc_integrate_const rc={rc}")
    return u, n.value


def integrate_adaptive(p: Problem, scheme: int, u, t0, t1, dt0, atol, rtol):
    """Returns (u_final, accepted, rejected, rc)."""
    u = _arr(u).copy()
    a, r = ctypes.c_int64(), ctypes.c_int64()
    rc = lib().orc_integrate_adaptive(ctypes.byref(p), scheme, _ptr(u), t0, t1, dt0, atol, rtol,
                                      ctypes.byref(a), ctypes.byref(r))
    return u, a.value, r.value, rc


CTRL_ODEINT, CTRL_SPEC = 0, 1


def integrate_adaptive_ctrl(p: Problem, scheme: int, u, t0, t1, dt0, atol, rtol,
                            controller: int = CTRL_ODEINT, max_tries: int = 500):
    """integrate_adaptive with the controller reading of choice (R-12 Odeint, R-28 SPEC).
    Returns (u_final, accepted, rejected, rc)."""
    u = _arr(u).copy()
    a, r = ctypes.c_int64(), ctypes.c_int64()
    rc = lib().orc_integrate_adaptive_ctrl(ctypes.byref(p), scheme, _ptr(u), t0, t1, dt0, atol,
                                           rtol, controller, max_tries, ctypes.byref(a),
                                           ctypes.byref(r))
    return u, a.value, r.value, rc


def lincomb(coef, inputs) -> np.ndarray:
    ins = [_arr(x) for x in inputs]
    k = len(ins)
    out = np.empty_like(ins[0])
    c = np.ascontiguousarray(coef, dtype=np.float64)
    arr = (ctypes.POINTER(ctypes.c_double) * k)(*[_ptr(x) for x in ins])
    rc = lib().orc_lincomb(out.size, _ptr(out), k, _ptr(c), arr)
    if rc != OK:
        raise ValueError("lincomb arity must be 1..14")
    return out


def norm_inf(u) -> float:
    u = _arr(u)
    return lib().orc_norm_inf(u.size, _ptr(u))


def ab_coefficients(k: int) -> list:
    """Adams–Bashforth k-step coefficients beta_0..beta_{k-1} (newest first), Fractions."""
    num, den = (ctypes.c_int64 * 8)(), (ctypes.c_int64 * 8)()
    if lib().orc_ab_coefficients(k, num, den) != k:
        raise ValueError("k must be 1..8")
    return [Fraction(num[j], den[j]) for j in range(k)]


def ab_integrate(p: Problem, k: int, u, t0: float, dt: float, nsteps: int,
                 trajectory: bool = False):
    """Adams–Bashforth k, nsteps fixed steps (RKF78 bootstrap).  Returns the final state, or
    (final, trajectory[nsteps, count]) if trajectory."""
    u = _arr(u).copy()
    tr = np.empty((nsteps, u.size)) if trajectory else None
    rc = lib().orc_ab_integrate(ctypes.byref(p), k, _ptr(u), t0, dt, nsteps,
                                _ptr(tr) if trajectory else None)
    if rc != OK:
        raise RuntimeError(f"orc_ab_integrate rc={rc}")
    return (u, tr) if trajectory else u


def am_coefficients(k: int) -> list:
    """Adams–Moulton k-term corrector coefficients m_0..m_{k-1} (m_0 weighs f_{n+1}), Fractions."""
    num, den = (ctypes.c_int64 * 8)(), (ctypes.c_int64 * 8)()
    if lib().orc_am_coefficients(k, num, den) != k:
        raise ValueError("k must be 1..8")
    return [Fraction(num[j], den[j]) for j in range(k)]


def abm_integrate(p: Problem, k: int, u, t0: float, dt: float, nsteps: int,
                  trajectory: bool = False):
    """Adams–Bashforth–Moulton k (PECE), nsteps fixed steps after the RKF78 bootstrap.
    Returns the final state, or (final, trajectory[nsteps, count]) if trajectory."""
    u = _arr(u).copy()
    tr = np.empty((nsteps, u.size)) if trajectory else None
    rc = lib().orc_abm_integrate(ctypes.byref(p), k, _ptr(u), t0, dt, nsteps,
                                 _ptr(tr) if trajectory else None)
    if rc != OK:
        raise RuntimeError(f"orc_abm_integrate rc={rc}")
    return (u, tr) if trajectory else u
