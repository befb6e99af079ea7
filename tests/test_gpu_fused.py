"""GPU parity of K6 (rk_fused.cu) and K7 (rk_fused2.cu, warp-specialised): a whole fixed RK4 /
explicit- / modified-midpoint step of Gray–Scott in one launch (temporal blocking across the
stages, RK_OPT_FUSED_STEP = 1 / 2).  Gate: bitwise equality
with the fp64 oracle (R-17/R-18) on seeded inputs, at sizes spanning several 32x16
tiles and z chunks with ragged tails, degenerate grids (1..5 cells per axis, where the
L-cell periodic margin wraps several times), every z-chunk length, and 512^3 sampled cells in
bench.py's launch configuration."""
import numpy as np
import pytest

import oracle
import rk_inputs

pytestmark = pytest.mark.gpu

OS = oracle.SCHEMES
FUSED = ["rk4", "midpoint", "modified_midpoint"]


@pytest.fixture(scope="module")
def ctx():
    import paper_2309_05331_b200 as rk
    c = rk.Context(0, 1, 0)
    yield c
    c.close()


def bitwise(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture(params=[1, 2], ids=["k6", "k7"])
def mode(request):
    return request.param


def fused_state(ctx, nx, ny, nz, u0, mode=1):
    import paper_2309_05331_b200 as rk
    st = ctx.grid(nx, ny, nz, 2)
    st.set_rhs_gray_scott()
    st.set(u0)
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    st.set_option(rk.OPT_FUSED_STEP, mode)
    return st


def perturbed_ic(nx, ny, nz, seed=42):
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=seed)
    return u0 + 0.01 * rk_inputs.random_state(u0.size, 5).reshape(u0.shape)


GRIDS = [(4, 4, 4), (8, 8, 8), (16, 16, 16), (33, 17, 9), (64, 40, 12), (1, 1, 3), (2, 3, 1),
         (5, 1, 2), (70, 9, 20), (96, 48, 40), (130, 35, 70)]


@pytest.mark.parametrize("scheme", FUSED)
@pytest.mark.parametrize("dims", GRIDS, ids=lambda d: "x".join(map(str, d)))
def test_fused_steps_bitwise(ctx, mode, scheme, dims):
    nx, ny, nz = dims
    u0 = perturbed_ic(nx, ny, nz)
    st = fused_state(ctx, nx, ny, nz, u0, mode)
    p = oracle.gray_scott_problem(nx, ny, nz)
    u = u0
    before = st.stats()
    for k in range(3):
        st.do_step(scheme, float(k), 1.0)
        u = oracle.step(p, OS[scheme], float(k), 1.0, u)
        assert bitwise(st.get(), u), (scheme, dims, k)
    after = st.stats()
    assert after["stage_launches"] - before["stage_launches"] == 3  # one launch per step


@pytest.mark.parametrize("fz", [1, 2, 3, 5, 8, 64])
@pytest.mark.parametrize("scheme", FUSED)
def test_fused_zchunks_bitwise(ctx, mode, scheme, fz, monkeypatch):
    """Every z-chunk length gives the same bits (the chunk's L-plane z margin is recomputed)."""
    monkeypatch.setenv("RKB_FZ", str(fz))
    nx, ny, nz = 40, 20, 23
    u0 = perturbed_ic(nx, ny, nz, seed=7)
    st = fused_state(ctx, nx, ny, nz, u0, mode)
    st.do_step(scheme, 0.0, 0.5)
    st.do_step(scheme, 0.5, 0.5)
    p = oracle.gray_scott_problem(nx, ny, nz)
    u = oracle.step(p, OS[scheme], 0.0, 0.5, u0)
    u = oracle.step(p, OS[scheme], 0.5, 0.5, u)
    assert bitwise(st.get(), u), fz


def test_fused_config3_integrate_const(ctx, mode):
    """BASELINE configs[2] through K6: 64^3, RK4, dt = 1, t in [0, 20] (20 launches)."""
    n = 64
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = fused_state(ctx, n, n, n, u0, mode)
    steps = st.integrate_const("rk4", 0.0, 20.0, 1.0)
    uo, so = oracle.integrate_const(oracle.gray_scott_problem(n, n, n), OS["rk4"], u0, 0.0, 20.0, 1.0)
    assert steps == so == 20
    assert bitwise(st.get(), uo)


@pytest.mark.parametrize("scheme", FUSED)
def test_fused_graph_replay(ctx, mode, scheme):
    import paper_2309_05331_b200 as rk
    nx, ny, nz = 48, 33, 17
    u0 = perturbed_ic(nx, ny, nz, seed=3)
    st = fused_state(ctx, nx, ny, nz, u0, mode)
    st.set_option(rk.OPT_USE_GRAPH, 1)
    steps = st.integrate_const(scheme, 0.0, 7.0, 1.0)
    uo, so = oracle.integrate_const(oracle.gray_scott_problem(nx, ny, nz), OS[scheme], u0, 0.0, 7.0, 1.0)
    assert steps == so == 7
    assert bitwise(st.get(), uo)


@pytest.mark.parametrize("scheme", FUSED)
def test_fused_equals_stage_kernels(ctx, mode, scheme):
    """K6 and the stage-by-stage K3 path agree bit for bit on a multi-tile grid."""
    import paper_2309_05331_b200 as rk
    nx, ny, nz = 200, 130, 50
    u0 = perturbed_ic(nx, ny, nz, seed=11)
    a = fused_state(ctx, nx, ny, nz, u0, mode)
    b = fused_state(ctx, nx, ny, nz, u0, mode)
    b.set_option(rk.OPT_FUSED_STEP, 0)
    for k in range(2):
        a.do_step(scheme, float(k), 1.0)
        b.do_step(scheme, float(k), 1.0)
    assert bitwise(a.get(), b.get())


def _sample_block(u, z, y, x, r):
    nz, _, ny, nx = u.shape
    zi = np.arange(z - r, z + r + 1) % nz
    yi = np.arange(y - r, y + r + 1) % ny
    xi = np.arange(x - r, x + r + 1) % nx
    return np.ascontiguousarray(u[zi][:, :, yi][:, :, :, xi])


@pytest.mark.parametrize("scheme", FUSED)
def test_fused_512_sampled_parity(ctx, mode, scheme):
    """One K6 step at 512^3 exactly as bench.py runs it; sampled cells (tile corners, domain
    edges and corners, the IC cube's faces) recomputed by the oracle on their periodic
    neighbourhood."""
    n = 512
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = fused_state(ctx, n, n, n, u0, mode)
    st.do_step(scheme, 0.0, 1.0)
    g = st.get()
    lo, hi = rk_inputs.cube_range(n)
    rng = np.random.default_rng(1)
    pts = [(lo, lo, lo), (hi - 1, hi, lo - 1), (0, 0, 0), (511, 511, 511), (0, 511, 0), (511, 0, 31),
           (lo + 3, 255, 256), (lo, lo + 15, 31), (hi, lo, 32), (lo, 16, 0), (lo + 1, 15, 511),
           (31, lo, lo), (32, hi, hi)] + [tuple(rng.integers(lo - 6, hi + 6, 3)) for _ in range(12)]
    r = 6
    p = oracle.gray_scott_problem(2 * r + 1, 2 * r + 1, 2 * r + 1)
    for (z, y, x) in pts:
        blk = _sample_block(u0, z, y, x, r)
        out = oracle.step(p, OS[scheme], 0.0, 1.0, blk).reshape(blk.shape)
        assert bitwise(g[z, :, y, x], out[r, :, r, r]), (z, y, x)
