"""The seeded input generators (rk_inputs) are decomposition-independent and follow the
recipe in DESIGN.md (R-6, R-9, R-10)."""
import numpy as np

import rk_inputs


def test_gs_ic_far_field_and_cube():
    u = rk_inputs.gray_scott_ic(32, 32, 32, seed=42)
    assert u.shape == (32, 2, 32, 32)
    lo, hi = rk_inputs.cube_range(32)
    assert (lo, hi) == (14, 18)
    mask = np.zeros((32, 32, 32), bool)
    mask[lo:hi, lo:hi, lo:hi] = True
    c0, c1 = u[:, 0], u[:, 1]
    assert np.all(c0[~mask] == 1.0) and np.all(c1[~mask] == 0.0)
    assert np.all(np.abs(c0[mask] / 0.5 - 1.0) <= 0.01) and np.all(np.abs(c1[mask] / 0.25 - 1.0) <= 0.01)
    assert np.unique(c1[mask]).size == mask.sum()          # seeded perturbation breaks symmetry


def test_gs_ic_slabs_concatenate_bitwise():
    full = rk_inputs.gray_scott_ic(16, 12, 40, seed=3, zblocks=2)
    for world in (2, 3, 8):
        parts = [rk_inputs.gray_scott_ic(16, 12, 40, seed=3, z0=z0, nzl=nzl, zblocks=2)
                 for z0, nzl in rk_inputs.slab_partition(40, world)]
        assert np.array_equal(np.concatenate(parts, axis=0), full)


def test_gs_ic_weak_scaling_blocks():
    u = rk_inputs.gray_scott_ic(16, 16, 48, seed=1, zblocks=3)
    assert sum(np.count_nonzero(u[b * 16:(b + 1) * 16, 1]) for b in range(3)) == 3 * 2 * 2 * 2
    assert all(np.count_nonzero(u[b * 16:(b + 1) * 16, 1]) == 8 for b in range(3))


def test_slab_partition_remainder_rule():
    assert rk_inputs.slab_partition(8, 2) == [(0, 4), (4, 4)]
    assert rk_inputs.slab_partition(7, 2) == [(0, 4), (4, 3)]
    p = rk_inputs.slab_partition(512, 24)
    assert sum(1 for _, n in p if n == 22) == 8 and sum(n for _, n in p) == 512


def test_vector_inputs():
    assert list(rk_inputs.exp_decay_u0(4)) == [0.25, 0.5, 0.75, 1.0]
    s = rk_inputs.logistic_shift(5)
    assert list(s) == [-1.0, -0.5, 0.0, 0.5, 1.0]
    assert abs(rk_inputs.logistic_u0(1, -5.0, shifted=False)[0] - 0.0066928509242848554) < 1e-18
    u = rk_inputs.exp_family_u0(16, 0.0)
    assert u[-1] == 1.0 and u[0] == 0.0
