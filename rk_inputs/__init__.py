"""Seeded synthetic input generators shared by the tests, bench.py and smoke().

This module holds NO arithmetic of the method (no stage values, RHS, steppers or
controller).  It only builds initial states, so the oracle (oracle/) and the CUDA path
(paper_2309_05331_b200/) can be fed bit-identical inputs without sharing code.
The recipes are stated in DESIGN.md §"Input recipe" with their PAPER.md readings.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_uniform(seed: int, gidx: np.ndarray, comp: int) -> np.ndarray:
    """xi in [0,1): splitmix64 of seed + (2*gidx + comp + 1)*golden."""
    with np.errstate(over="ignore"):
        g = np.asarray(gidx, dtype=np.uint64)
        z = np.uint64(seed) + (np.uint64(2) * g + np.uint64(comp + 1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def cube_range(n: int) -> tuple[int, int]:
    """Centred cube of side n/8 along one axis: indices [7n/16, 9n/16)."""
    lo, hi = (7 * n) // 16, (9 * n) // 16
    if hi <= lo:  # tiny grids: keep one seeded cell
        hi = lo + 1
    return lo, hi


def gray_scott_ic(nx: int, ny: int, nz: int, seed: int = 42, z0: int = 0, nzl: int | None = None,
                  zblocks: int = 1) -> np.ndarray:
    """Gray–Scott initial state, planes [z0, z0+nzl) of the global nx*ny*nz grid.

    Layout [z][c][y][x] (fp64), c=0 is C0, c=1 is C1 (Listing 2).
    Recipe (R-6; the paper gives no IC): C0=1, C1=0 everywhere except
    one centred cube of side n/8 per z-block of nz/zblocks planes, where
    C0 = 0.5*(1+0.02*(xi0-0.5)), C1 = 0.25*(1+0.02*(xi1-0.5)), xi from splitmix64 of the
    global cell index.  zblocks>1 stacks one cube per block (weak scaling).
    """
    if nzl is None:
        nzl = nz - z0
    u = np.zeros((nzl, 2, ny, nx), dtype=np.float64)
    u[:, 0] = 1.0
    assert nz % zblocks == 0
    nzb = nz // zblocks
    xlo, xhi = cube_range(nx)
    ylo, yhi = cube_range(ny)
    zlo_b, zhi_b = cube_range(nzb)
    for b in range(zblocks):
        zlo, zhi = b * nzb + zlo_b, b * nzb + zhi_b
        a, e = max(zlo, z0), min(zhi, z0 + nzl)
        if a >= e:
            continue
        zz, yy, xx = np.meshgrid(np.arange(a, e, dtype=np.int64), np.arange(ylo, yhi, dtype=np.int64),
                                 np.arange(xlo, xhi, dtype=np.int64), indexing="ij")
        gidx = (zz * ny + yy) * nx + xx
        xi0 = splitmix64_uniform(seed, gidx, 0)
        xi1 = splitmix64_uniform(seed, gidx, 1)
        u[a - z0:e - z0, 0, ylo:yhi, xlo:xhi] = 0.5 * (1.0 + 0.02 * (xi0 - 0.5))
        u[a - z0:e - z0, 1, ylo:yhi, xlo:xhi] = 0.25 * (1.0 + 0.02 * (xi1 - 0.5))
    return u


def exp_decay_u0(n: int) -> np.ndarray:
    """Config 1 (BASELINE.json configs[0]): u_i(0) = (i+1)/N (R-9)."""
    return (np.arange(n, dtype=np.float64) + 1.0) / float(n)


def logistic_shift(n: int) -> np.ndarray:
    """Config 2 per-element time shift s_i = -1 + 2i/(N-1) (R-10); 0 for N=1."""
    if n == 1:
        return np.zeros(1)
    return -1.0 + 2.0 * np.arange(n, dtype=np.float64) / float(n - 1)


def logistic_u0(n: int, t0: float = -5.0, shifted: bool = True) -> np.ndarray:
    """u_i(t0) = 1/(1+exp(-(t0 - s_i))): the Eq. 1b solution sampled at t0."""
    s = logistic_shift(n) if shifted else np.zeros(n)
    return 1.0 / (1.0 + np.exp(-(t0 - s)))


def exp_family_u0(n_side: int, t0: float = -5.0) -> np.ndarray:
    """Paper's exponential family: A(x,y)=x*y on an n_side^2 node grid
    of [0,1]^2 (x_i = i/(n-1)), u(t0) = A*e^{t0}.  Flattened row-major (y, x)."""
    x = np.arange(n_side, dtype=np.float64) / float(n_side - 1)
    A = np.outer(x, x).ravel()
    return A * np.exp(t0)


def random_state(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Seeded uniform test vector (algebra-op conformance inputs)."""
    return np.random.default_rng(seed).uniform(lo, hi, size=n)


def slab_partition(nz: int, world: int) -> list[tuple[int, int]]:
    """(z0, nzl) per rank; remainder planes go to the lowest ranks."""
    base, rem = divmod(nz, world)
    out, z = [], 0
    for r in range(world):
        nzl = base + (1 if r < rem else 0)
        out.append((z, nzl))
        z += nzl
    return out
