"""GPU parity: the CUDA path through the C-ABI against the fp64 oracle on the same seeded
inputs (rk_inputs).  Design target and gate: bitwise identity (R-17/R-18), which
implies the BASELINE north_star tolerances (1e-12 per step, 1e-9 final, identical
accepted/rejected counts).  Sizes span several tiles (32x8 xy tiles, z chunks) with ragged
tails, plus degenerate grids (1..4 cells per axis)."""
import math

import numpy as np
import pytest

import oracle
import rk_inputs

pytestmark = pytest.mark.gpu

SCHEMES = ["euler", "rk4", "cash_karp54", "dopri5", "rkf78", "midpoint", "modified_midpoint"]
OS = oracle.SCHEMES


@pytest.fixture(scope="module")
def ctx():
    import paper_2309_05331_b200 as rk
    c = rk.Context(0, 1, 0)
    yield c
    c.close()


def bitwise(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def gs_state(ctx, nx, ny, nz, u0, coop=False, **prm):
    """A Gray–Scott state.  coop=False pins fixed steps to the stage-by-stage TMA stencil
    path (K3: no K5, no K8 stage pairs); coop=True leaves the persistent small-grid path (K5)
    on (library default).  K8 has its own tests (test_gpu_pair.py)."""
    import paper_2309_05331_b200 as rk
    st = ctx.grid(nx, ny, nz, 2)
    st.set_rhs_gray_scott(**prm)
    st.set(u0)
    if not coop:
        st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
        st.set_option(rk.OPT_FUSED_STEP, 0)
    return st


# ---------------------------------------------------------------------------------------
# pointwise (exp / logistic) vector path
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("n", [1, 2, 3, 1000, 100001])
@pytest.mark.parametrize("rhs", ["exp", "logistic"])
def test_pointwise_do_step_bitwise(ctx, scheme, n, rhs):
    u0 = rk_inputs.logistic_u0(n) if rhs == "logistic" else rk_inputs.exp_decay_u0(n)
    st = ctx.vector(n)
    if rhs == "exp":
        st.set_rhs_exponential(-1.0)
        p = oracle.exp_problem(n, -1.0)
    else:
        st.set_rhs_logistic()
        p = oracle.logistic_problem(n)
    st.set(u0)
    u = u0
    for k in range(3):
        st.do_step(scheme, 0.0, 0.1 * (k + 1))
        u = oracle.step(p, OS[scheme], 0.0, 0.1 * (k + 1), u)
        assert bitwise(st.get(), u), (scheme, n, k)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_config1_exp_decay_integrate_const(ctx, scheme):
    """BASELINE configs[0]: du/dt=-u, N=1e5, t in [0,1]; multi-step in-register kernel."""
    n = 100000
    u0 = rk_inputs.exp_decay_u0(n)
    st = ctx.vector(n)
    st.set_rhs_exponential(-1.0)
    for dt in (0.1, 2.0 ** -5):
        st.set(u0)
        steps = st.integrate_const(scheme, 0.0, 1.0, dt)
        uo, so = oracle.integrate_const(oracle.exp_problem(n, -1.0), OS[scheme], u0, 0.0, 1.0, dt)
        assert steps == so == round(1.0 / dt)
        g = st.get()
        assert bitwise(g, uo)
        order = {"euler": 1, "rk4": 4, "cash_karp54": 5, "dopri5": 5, "rkf78": 8,
                 "midpoint": 2, "modified_midpoint": 2}[scheme]
        err = np.max(np.abs(g - u0 * math.exp(-1.0)))
        assert err < 2 * dt ** order


@pytest.mark.parametrize("scheme,tol,acc_rej", [("dopri5", 1e-8, (51, 2)), ("cash_karp54", 1e-8, None)])
def test_config2_logistic_adaptive(ctx, scheme, tol, acc_rej):
    """BASELINE configs[1]: logistic N=1e6 adaptive (atol = rtol = 1e-8): accepted and
    rejected counts identical to the oracle, final state bitwise."""
    n = 1000000
    u0 = rk_inputs.logistic_u0(n)
    st = ctx.vector(n)
    st.set_rhs_logistic()
    st.set(u0)
    a, r = st.integrate_adaptive(scheme, -5.0, 5.0, 0.1, tol, tol)
    uo, ao, ro, rc = oracle.integrate_adaptive(oracle.logistic_problem(n), OS[scheme], u0, -5.0,
                                               5.0, 0.1, tol, tol)
    assert rc == 0 and (a, r) == (ao, ro)
    if acc_rej:
        assert (a, r) == acc_rej
    assert bitwise(st.get(), uo)


def test_try_step_rejection_leaves_state(ctx):
    n = 4096
    u0 = rk_inputs.logistic_u0(n)
    st = ctx.vector(n)
    st.set_rhs_logistic()
    st.set(u0)
    acc, E, dtn = st.try_step("dopri5", -5.0, 8.0, 1e-12, 1e-12)
    assert not acc and E > 1 and dtn < 8.0
    assert bitwise(st.get(), u0)
    accepted, Eo = oracle.controller(E, 8.0)
    assert (acc, dtn) == (accepted, Eo)


# ---------------------------------------------------------------------------------------
# Gray–Scott grid path
# ---------------------------------------------------------------------------------------
GRIDS = [(4, 4, 4), (8, 8, 8), (16, 16, 16), (33, 17, 9), (64, 40, 12), (1, 1, 3), (2, 3, 1),
         (5, 1, 2), (70, 9, 20)]


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("dims", GRIDS, ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("coop", [False, True], ids=["k3", "k5"])
def test_gs_steps_bitwise(ctx, scheme, dims, coop):
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=42)
    # perturb so every cell is non-trivial (the IC is mostly the (1,0) steady state)
    u0 = u0 + 0.01 * rk_inputs.random_state(u0.size, 5).reshape(u0.shape)
    st = gs_state(ctx, nx, ny, nz, u0, coop=coop)
    p = oracle.gray_scott_problem(nx, ny, nz)
    u = u0
    for k in range(3):
        st.do_step(scheme, float(k), 1.0)
        u = oracle.step(p, OS[scheme], float(k), 1.0, u)
        assert bitwise(st.get(), u), (scheme, dims, k)


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("dims", [(16, 16, 16), (33, 17, 9), (8, 8, 1), (8, 8, 2), (8, 8, 3)],
                         ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("overlap", [1, 0])
def test_gs_halo_loopback_bitwise(ctx, scheme, dims, overlap):
    """The multi-GPU code path (pack -> exchange -> interior + boundary launches, ghost
    planes) on one GPU with a self-exchange: bitwise equal to the oracle."""
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=1) + 0.01 * rk_inputs.random_state(
        2 * nx * ny * nz, 9).reshape(nz, 2, ny, nx)
    st = gs_state(ctx, nx, ny, nz, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, 1)
    st.set_option(rk.OPT_HALO_OVERLAP, overlap)
    p = oracle.gray_scott_problem(nx, ny, nz)
    u = u0
    for k in range(2):
        st.do_step(scheme, 0.0, 1.0)
        u = oracle.step(p, OS[scheme], 0.0, 1.0, u)
        assert bitwise(st.get(), u)
    assert st.stats()["halo_exchanges"] > 0


@pytest.mark.parametrize("coop", [False, True], ids=["k3", "k5"])
def test_config3_gray_scott_64_rk4(ctx, coop):
    """BASELINE configs[2]: 64^3 periodic, RK4, dt=1, t in [0,20]: bitwise after every step,
    through the stage-by-stage stencil path (k3) and the persistent one-launch path (k5)."""
    n = 64
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = gs_state(ctx, n, n, n, u0, coop=coop)
    p = oracle.gray_scott_problem(n, n, n)
    u = u0
    for k in range(20):
        st.do_step("rk4", float(k), 1.0)
        u = oracle.step(p, oracle.RK4, float(k), 1.0, u)
        assert bitwise(st.get(), u), k
    st.set(u0)
    assert st.integrate_const("rk4", 0.0, 20.0, 1.0) == 20
    assert bitwise(st.get(), u)


@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54", "rkf78"])
@pytest.mark.parametrize("tol", [1e-6, 1e-8])
def test_gs_adaptive_counts_and_state(ctx, scheme, tol):
    n = 32
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = gs_state(ctx, n, n, n, u0)
    a, r = st.integrate_adaptive(scheme, 0.0, 20.0, 1.0, tol, tol)
    uo, ao, ro, rc = oracle.integrate_adaptive(oracle.gray_scott_problem(n, n, n), OS[scheme],
                                               u0, 0.0, 20.0, 1.0, tol, tol)
    assert rc == 0 and (a, r) == (ao, ro) and a > 0
    assert bitwise(st.get(), uo)


def test_gs_try_step_matches_oracle_ratio(ctx):
    n = 24
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=3) + 0.05 * rk_inputs.random_state(
        2 * n ** 3, 4).reshape(n, 2, n, n)
    p = oracle.gray_scott_problem(n, n, n)
    for scheme in ("dopri5", "cash_karp54", "rkf78"):
        st = gs_state(ctx, n, n, n, u0)
        for dt in (4.0, 1.0, 0.25):
            st.set(u0)
            acc, E, dtn = st.try_step(scheme, 0.0, dt, 1e-7, 1e-7)
            un, err = oracle.step(p, OS[scheme], 0.0, dt, u0, with_error=True)
            Eo = oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), dt, 1e-7, 1e-7)
            assert E == Eo
            assert bitwise(st.get(), un if acc else u0)


# ---------------------------------------------------------------------------------------
# full BASELINE size (512^3), launch configuration of bench.py, sampled outputs
# ---------------------------------------------------------------------------------------
def _sample_block(u, z, y, x, r=8):
    """(2r+1)^3 periodic neighbourhood of cell (z,y,x) from a [z][c][y][x] array."""
    nz, _, ny, nx = u.shape
    zi = np.arange(z - r, z + r + 1) % nz
    yi = np.arange(y - r, y + r + 1) % ny
    xi = np.arange(x - r, x + r + 1) % nx
    return np.ascontiguousarray(u[zi][:, :, yi][:, :, :, xi])


@pytest.mark.parametrize("scheme,adaptive", [("rk4", False), ("dopri5", True), ("dopri5", False),
                                             ("cash_karp54", True), ("euler", False), ("midpoint", False),
                                             ("rkf78", False), ("rkf78", True)])
def test_512_sampled_parity(ctx, scheme, adaptive):
    """One step (or one adaptive try) at 512^3 exactly as bench.py runs it; every sampled
    cell's new value is recomputed by the oracle on its periodic neighbourhood of radius
    (#stages + 1) (a cell's new value depends on cells at most #stages away), and must
    match bitwise."""
    n = 512
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = gs_state(ctx, n, n, n, u0)
    dt = 1.0
    if adaptive:  # as bench.py: tries until accepted; a rejected try leaves u untouched
        for _ in range(10):
            acc, E, dtn = st.try_step(scheme, 0.0, dt, 1e-6, 1e-6)
            if acc:
                break
            assert E > 1.0 and dtn < dt
            dt = dtn
        assert acc and 0.0 <= E <= 1.0
    else:
        st.do_step(scheme, 0.0, dt)
    g = st.get()
    lo, hi = rk_inputs.cube_range(n)
    rng = np.random.default_rng(0)
    pts = [(lo, lo, lo), (hi - 1, hi, lo - 1), (0, 0, 0), (511, 511, 511), (lo + 3, 255, 256),
           (lo, lo + 5, 31), (hi, lo, 32)] + [tuple(rng.integers(lo - 4, hi + 4, 3)) for _ in range(12)]
    r = 14 if scheme == "rkf78" else 8
    p = oracle.gray_scott_problem(2 * r + 1, 2 * r + 1, 2 * r + 1)
    for (z, y, x) in pts:
        blk = _sample_block(u0, z, y, x, r)
        out = oracle.step(p, OS[scheme], 0.0, dt, blk).reshape(blk.shape)
        assert bitwise(g[z, :, y, x], out[r, :, r, r]), (z, y, x)


@pytest.mark.parametrize("method", ["ab2", "abm2", "ab4"])
def test_512_sampled_parity_adams(ctx, method):
    """Adams steps at 512^3 in bench.py's launch configuration: RKF78 start-up then Adams
    steps; sampled cells against the oracle on their periodic neighbourhoods."""
    n = 512
    k = int(method.lstrip("abm"))
    nsteps = k  # k-1 start-up steps + 1 Adams step
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = gs_state(ctx, n, n, n, u0)
    for m in range(nsteps):
        st.do_step(method, float(m), 1.0)
    g = st.get()
    lo, hi = rk_inputs.cube_range(n)
    rng = np.random.default_rng(1)
    pts = [(lo, lo, lo), (hi - 1, hi, lo - 1), (0, 0, 0), (511, 511, 511)] + \
          [tuple(rng.integers(lo - 4, hi + 4, 3)) for _ in range(6)]
    r = 14 * (k - 1) + 4
    p = oracle.gray_scott_problem(2 * r + 1, 2 * r + 1, 2 * r + 1)
    run = oracle.abm_integrate if method.startswith("abm") else oracle.ab_integrate
    for (z, y, x) in pts:
        blk = _sample_block(u0, z, y, x, r)
        out = run(p, k, blk, 0.0, 1.0, nsteps).reshape(blk.shape)
        assert bitwise(g[z, :, y, x], out[r, :, r, r]), (z, y, x)


# ---------------------------------------------------------------------------------------
# algebra ops and error conventions
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("k", [1, 2, 5, 14])
def test_lincomb_bitwise(ctx, k):
    n = 10007
    ins = [rk_inputs.random_state(n, 100 + j) for j in range(k)]
    coef = list(rk_inputs.random_state(k, 7))
    sts = []
    for x in ins:
        s = ctx.vector(n)
        s.set(x)
        sts.append(s)
    out = ctx.vector(n)
    out.lincomb(coef, sts)
    assert bitwise(out.get(), oracle.lincomb(coef, ins))
    sts[0].lincomb(coef, sts)  # aliasing: out is an input
    assert bitwise(sts[0].get(), oracle.lincomb(coef, ins))


def test_norm_inf(ctx):
    x = rk_inputs.random_state(123457, 3)
    st = ctx.vector(x.size)
    st.set(x)
    assert st.norm_inf() == oracle.norm_inf(x)
    x[777] = -5.0
    st.set(x)
    assert st.norm_inf() == 5.0
    x[5] = np.nan
    st.set(x)
    assert math.isnan(st.norm_inf())


def test_error_conventions(ctx):
    import paper_2309_05331_b200 as rk
    v = ctx.vector(10)
    with pytest.raises(rk.RKError) as e:
        v.do_step("rk4", 0.0, 0.1)
    assert e.value.status == "RK_ERR_STATE"          # RHS unset
    v.set_rhs_logistic()
    with pytest.raises(rk.RKError) as e:
        v.integrate_adaptive("rk4", 0.0, 1.0, 0.1, 1e-6, 1e-6)
    assert e.value.status == "RK_ERR_UNSUPPORTED"
    for bad in (0.0, -1.0, math.inf, math.nan):
        with pytest.raises(rk.RKError) as e:
            v.do_step("rk4", 0.0, bad)
        assert e.value.status == "RK_ERR_ARG"
    with pytest.raises(rk.RKError) as e:
        v.set_rhs_gray_scott()
    assert e.value.status == "RK_ERR_STATE"
    with pytest.raises(rk.RKError) as e:
        v.lincomb([1.0] * 15, [v] * 15)
    assert e.value.status == "RK_ERR_CONTRACT"
    w = ctx.vector(11)
    with pytest.raises(rk.RKError) as e:
        v.lincomb([1.0], [w])
    assert e.value.status == "RK_ERR_CONTRACT"
    x = np.full(10, 0.5)
    x[3] = np.nan
    v.set(x)
    with pytest.raises(rk.RKError) as e:
        v.integrate_adaptive("dopri5", 0.0, 1.0, 0.1, 1e-6, 1e-6)
    assert e.value.status == "RK_ERR_DIVERGED"


def test_comm_timeout_option(ctx):
    """RK_OPT_COMM_TIMEOUT_MS (failure detection): >= 0 accepted; on one GPU there
    is no communicator, so results are unchanged; a negative deadline is an argument error."""
    import paper_2309_05331_b200 as rk
    v = ctx.vector(1001)
    v.set_rhs_logistic()
    u0 = rk_inputs.logistic_u0(1001)
    v.set(u0)
    v.set_option(rk.OPT_COMM_TIMEOUT_MS, 5000)
    a, r = v.integrate_adaptive("dopri5", -5.0, 5.0, 0.1, 1e-8, 1e-8)
    uo, ao, ro, rc = oracle.integrate_adaptive(oracle.logistic_problem(1001), OS["dopri5"], u0, -5.0, 5.0, 0.1,
                                               1e-8, 1e-8)
    assert (a, r) == (ao, ro) and bitwise(v.get(), uo)
    with pytest.raises(rk.RKError) as e:
        v.set_option(rk.OPT_COMM_TIMEOUT_MS, -1)
    assert e.value.status == "RK_ERR_ARG"
    v.set_option(rk.OPT_COMM_TIMEOUT_MS, 0)


def test_stats_count_launches(ctx):
    n = 16
    st = gs_state(ctx, n, n, n, rk_inputs.gray_scott_ic(n, n, n))
    st.reset_stats()
    st.do_step("rk4", 0.0, 1.0)
    s = st.stats()
    assert s["rhs_evals"] == 4 and s["stage_launches"] == 4 and s["kernel_launches"] >= 4


# ---------------------------------------------------------------------------------------
# Adams–Bashforth k = 1..8: RKF78 bootstrap + one fused launch per step
# ---------------------------------------------------------------------------------------
def _odeint_steps(t0, t1, dt):
    n, t = 0, t0
    while (t + dt) - t1 <= np.finfo(float).eps:
        n += 1
        t = t0 + n * dt
    return n


@pytest.mark.parametrize("k", range(1, 9))
@pytest.mark.parametrize("rhs", ["exp", "logistic"])
def test_ab_vector_bitwise(ctx, k, rhs):
    n = 10001
    if rhs == "exp":
        u0 = rk_inputs.exp_decay_u0(n)
        p = oracle.exp_problem(n, -1.0)
    else:
        u0 = rk_inputs.logistic_u0(n)
        p = oracle.logistic_problem(n)
    st = ctx.vector(n)
    st.set_rhs_exponential(-1.0) if rhs == "exp" else st.set_rhs_logistic()
    st.set(u0)
    dt = 2.0 ** -5
    steps = st.integrate_const(f"ab{k}", 0.0, 1.0, dt)
    assert steps == _odeint_steps(0.0, 1.0, dt)
    assert bitwise(st.get(), oracle.ab_integrate(p, k, u0, 0.0, dt, steps))
    # do_step continues the same history (no re-bootstrap)
    for _ in range(3):
        st.do_step(f"ab{k}", 0.0, dt)
    assert bitwise(st.get(), oracle.ab_integrate(p, k, u0, 0.0, dt, steps + 3))


@pytest.mark.parametrize("k", [1, 2, 4, 8])
@pytest.mark.parametrize("dims", [(16, 12, 10), (33, 17, 9)], ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("loopback", [0, 1])
def test_ab_grid_bitwise(ctx, k, dims, loopback):
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=7) + 0.01 * rk_inputs.random_state(
        2 * nx * ny * nz, 11).reshape(nz, 2, ny, nx)
    st = gs_state(ctx, nx, ny, nz, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, loopback)
    p = oracle.gray_scott_problem(nx, ny, nz)
    nsteps = k + 4
    for m in range(nsteps):
        st.do_step(f"ab{k}", float(m), 1.0)
    assert bitwise(st.get(), oracle.ab_integrate(p, k, u0, 0.0, 1.0, nsteps))


def test_ab_history_restarts(ctx):
    """A new dt (or set / another scheme) restarts the bootstrap, as documented."""
    n = 64
    u0 = rk_inputs.logistic_u0(n)
    p = oracle.logistic_problem(n)
    st = ctx.vector(n)
    st.set_rhs_logistic()
    st.set(u0)
    for _ in range(5):
        st.do_step("ab3", 0.0, 0.1)
    mid = oracle.ab_integrate(p, 3, u0, 0.0, 0.1, 5)
    assert bitwise(st.get(), mid)
    for _ in range(4):
        st.do_step("ab3", 0.0, 0.05)
    assert bitwise(st.get(), oracle.ab_integrate(p, 3, mid, 0.0, 0.05, 4))


# ---------------------------------------------------------------------------------------
# f4: rk_eval_rhs and the unfused "native" RK4 ablation
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("dims", [(16, 16, 16), (33, 17, 9), (1, 1, 3), (70, 9, 20)],
                         ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("loopback", [0, 1])
def test_eval_rhs_grid_bitwise(ctx, dims, loopback):
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=3) + 0.01 * rk_inputs.random_state(
        2 * nx * ny * nz, 4).reshape(nz, 2, ny, nx)
    st = gs_state(ctx, nx, ny, nz, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, loopback)
    out = ctx.grid(nx, ny, nz, 2)
    st.eval_rhs(out)
    assert bitwise(out.get(), oracle.rhs(oracle.gray_scott_problem(nx, ny, nz), u0))
    assert bitwise(st.get(), u0)  # input untouched


@pytest.mark.parametrize("rhs", ["exp", "logistic"])
def test_eval_rhs_vector_bitwise(ctx, rhs):
    n = 100003
    u0 = rk_inputs.logistic_u0(n) if rhs == "logistic" else rk_inputs.exp_decay_u0(n)
    st = ctx.vector(n)
    if rhs == "exp":
        st.set_rhs_exponential(-0.7)
        p = oracle.exp_problem(n, -0.7)
    else:
        st.set_rhs_logistic()
        p = oracle.logistic_problem(n)
    st.set(u0)
    out = ctx.vector(n)
    st.eval_rhs(out)
    assert bitwise(out.get(), oracle.rhs(p, u0))


def test_eval_rhs_errors(ctx):
    import paper_2309_05331_b200 as rk
    a, b = ctx.vector(10), ctx.vector(11)
    with pytest.raises(rk.RKError) as e:
        a.eval_rhs(a)
    assert e.value.status == "RK_ERR_ARG"
    a.set_rhs_logistic()
    with pytest.raises(rk.RKError) as e:
        a.eval_rhs(b)
    assert e.value.status == "RK_ERR_CONTRACT"
    c = ctx.vector(10)
    with pytest.raises(rk.RKError) as e:
        c.eval_rhs(a)  # no RHS on the input
    assert e.value.status == "RK_ERR_STATE"


@pytest.mark.parametrize("dims", [(33, 17, 9), (64, 64, 64)], ids=lambda d: "x".join(map(str, d)))
def test_native_rk4_equals_fused_grid(ctx, dims):
    """The unfused RK4 (eval_rhs + lincomb per stage) and the fused stage kernels evaluate the
    same expression trees (R-17): bitwise equal to each other and to the oracle."""
    from paper_2309_05331_b200.ablation import NativeRK4
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=42) + 0.01 * rk_inputs.random_state(
        2 * nx * ny * nz, 5).reshape(nz, 2, ny, nx)
    fused = gs_state(ctx, nx, ny, nz, u0)
    native = gs_state(ctx, nx, ny, nz, u0)
    nat = NativeRK4(native)
    p = oracle.gray_scott_problem(nx, ny, nz)
    u = u0
    for k in range(3):
        fused.do_step("rk4", float(k), 1.0)
        nat.step(1.0)
        u = oracle.step(p, oracle.RK4, float(k), 1.0, u)
        assert bitwise(native.get(), fused.get()) and bitwise(native.get(), u), k
    nat.close()


def test_native_rk4_equals_fused_vector(ctx):
    from paper_2309_05331_b200.ablation import NativeRK4
    n = 262144  # the exponential-family 512^2 workload
    u0 = rk_inputs.exp_family_u0(512)  # du/dt = u, u = A(x,y) e^t
    fused, native = ctx.vector(n), ctx.vector(n)
    for s in (fused, native):
        s.set_rhs_exponential(1.0)
        s.set(u0)
    nat = NativeRK4(native)
    for k in range(4):
        fused.do_step("rk4", 0.0, 0.01)
        nat.step(0.01)
    assert bitwise(native.get(), fused.get())
    nat.close()


# ---------------------------------------------------------------------------------------
# Adams–Bashforth–Moulton k = 1..8, PECE (Table 1; R-26)
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("k", range(1, 9))
@pytest.mark.parametrize("rhs", ["exp", "logistic"])
def test_abm_vector_bitwise(ctx, k, rhs):
    n = 10001
    if rhs == "exp":
        u0 = rk_inputs.exp_decay_u0(n)
        p = oracle.exp_problem(n, -1.0)
    else:
        u0 = rk_inputs.logistic_u0(n)
        p = oracle.logistic_problem(n)
    st = ctx.vector(n)
    st.set_rhs_exponential(-1.0) if rhs == "exp" else st.set_rhs_logistic()
    st.set(u0)
    dt = 2.0 ** -5
    steps = st.integrate_const(f"abm{k}", 0.0, 1.0, dt)
    assert steps == _odeint_steps(0.0, 1.0, dt)
    assert bitwise(st.get(), oracle.abm_integrate(p, k, u0, 0.0, dt, steps))
    for _ in range(3):
        st.do_step(f"abm{k}", 0.0, dt)
    assert bitwise(st.get(), oracle.abm_integrate(p, k, u0, 0.0, dt, steps + 3))


@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dims", [(16, 12, 10), (33, 17, 9), (8, 8, 1)], ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("loopback", [0, 1])
def test_abm_grid_bitwise(ctx, k, dims, loopback):
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=8) + 0.01 * rk_inputs.random_state(
        2 * nx * ny * nz, 12).reshape(nz, 2, ny, nx)
    st = gs_state(ctx, nx, ny, nz, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, loopback)
    p = oracle.gray_scott_problem(nx, ny, nz)
    nsteps = k + 3
    for m in range(nsteps):
        st.do_step(f"abm{k}", float(m), 1.0)
    assert bitwise(st.get(), oracle.abm_integrate(p, k, u0, 0.0, 1.0, nsteps))
    st.set(u0)
    assert st.integrate_const(f"abm{k}", 0.0, float(nsteps), 1.0) == nsteps
    assert bitwise(st.get(), oracle.abm_integrate(p, k, u0, 0.0, 1.0, nsteps))


def test_abm_stats_two_rhs_per_step(ctx):
    n = 16
    st = gs_state(ctx, n, n, n, rk_inputs.gray_scott_ic(n, n, n))
    for _ in range(3):  # bootstrap of k = 4
        st.do_step("abm4", 0.0, 1.0)
    st.reset_stats()
    st.do_step("abm4", 0.0, 1.0)
    s = st.stats()
    assert s["rhs_evals"] == 2 and s["stage_launches"] == 2


# ---------------------------------------------------------------------------------------
# f3: device-resident adaptive loop (RK_OPT_DEVICE_LOOP; R-27)
# ---------------------------------------------------------------------------------------
def _adaptive_vec(ctx, rhs, n, u0, scheme, t0, t1, dt0, tol, device_loop, max_tries=None):
    import paper_2309_05331_b200 as rk
    st = ctx.vector(n)
    st.set_rhs_exponential(-1.0) if rhs == "exp" else st.set_rhs_logistic()
    st.set(u0)
    st.set_option(rk.OPT_DEVICE_LOOP, 1 if device_loop else 0)
    if max_tries:
        st.set_option(rk.OPT_MAX_TRIES, max_tries)
    a, r = st.integrate_adaptive(scheme, t0, t1, dt0, tol, tol)
    s = st.stats()
    return st.get(), a, r, s


@pytest.mark.parametrize("scheme,tol,acc_rej", [("dopri5", 1e-8, (51, 2)), ("cash_karp54", 1e-8, None),
                                                ("rkf78", 1e-10, None)])
def test_device_loop_config2(ctx, scheme, tol, acc_rej):
    """Config 2 through the one-launch device loop: counts and final state identical to the
    oracle (and to the host-driven loop)."""
    n = 1000000
    u0 = rk_inputs.logistic_u0(n)
    g, a, r, s = _adaptive_vec(ctx, "logistic", n, u0, scheme, -5.0, 5.0, 0.1, tol, True)
    uo, ao, ro, rc = oracle.integrate_adaptive(oracle.logistic_problem(n), OS[scheme], u0, -5.0,
                                               5.0, 0.1, tol, tol)
    assert rc == 0 and (a, r) == (ao, ro)
    if acc_rej:
        assert (a, r) == acc_rej
    assert bitwise(g, uo)
    assert s["kernel_launches"] == 1 and s["tries"] == a + r


@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54", "rkf78"])
@pytest.mark.parametrize("tol", [1e-3, 1e-5, 1e-7, 1e-9, 1e-11, 1e-13])
@pytest.mark.parametrize("rhs", ["exp", "logistic"])
def test_device_loop_matches_host_loop(ctx, scheme, tol, rhs):
    """Many controller evaluations (rejections included, dt0 too large on purpose): the device
    controller's double-double pow reproduces the host's libm pow on every call."""
    n = 30001
    u0 = rk_inputs.logistic_u0(n) if rhs == "logistic" else rk_inputs.exp_decay_u0(n)
    t0, t1 = (-5.0, 5.0) if rhs == "logistic" else (0.0, 3.0)
    gd, ad, rd, sd = _adaptive_vec(ctx, rhs, n, u0, scheme, t0, t1, 2.0, tol, True)
    gh, ah, rh, sh = _adaptive_vec(ctx, rhs, n, u0, scheme, t0, t1, 2.0, tol, False)
    assert (ad, rd) == (ah, rh)
    assert bitwise(gd, gh)
    assert sd["last_dt"] == sh["last_dt"]


@pytest.mark.parametrize("n", [1, 2, 7, 262145, 3000001])
def test_device_loop_sizes(ctx, n):
    """The device loop from 1 element to more elements than the cooperative grid has threads
    (grid-stride tries, odd tails): equal to the host loop bit for bit."""
    u0 = rk_inputs.logistic_u0(n) if n > 1 else np.array([0.25])
    gd, ad, rd, sd = _adaptive_vec(ctx, "logistic", n, u0, "dopri5", -5.0, 5.0, 0.5, 1e-7, True)
    gh, ah, rh, sh = _adaptive_vec(ctx, "logistic", n, u0, "dopri5", -5.0, 5.0, 0.5, 1e-7, False)
    assert (ad, rd) == (ah, rh)
    assert bitwise(gd, gh)


def test_device_loop_errors(ctx):
    import paper_2309_05331_b200 as rk
    n = 1000
    x = np.full(n, 0.5)
    x[7] = np.nan
    with pytest.raises(rk.RKError) as e:
        _adaptive_vec(ctx, "logistic", n, x, "dopri5", 0.0, 1.0, 0.1, 1e-6, True)
    assert e.value.status == "RK_ERR_DIVERGED"
    with pytest.raises(rk.RKError) as e:  # dt0 = 50 needs several rejections: stall at 1 try
        _adaptive_vec(ctx, "logistic", n, rk_inputs.logistic_u0(n), "dopri5", -5.0, 50.0, 50.0, 1e-10, True,
                      max_tries=1)
    assert e.value.status == "RK_ERR_STALL"


@pytest.mark.parametrize("scheme,nsteps", [("rk4", 20), ("dopri5", 7), ("euler", 6), ("rkf78", 5)])
def test_graph_replay_integrate_const(ctx, scheme, nsteps):
    """RK_OPT_USE_GRAPH: the fixed steps replayed from a captured CUDA graph give the oracle's
    state bitwise, and the same counters as launching them one by one."""
    import paper_2309_05331_b200 as rk
    n = 64
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42) + 0.01 * rk_inputs.random_state(2 * n ** 3, 6).reshape(n, 2, n, n)
    p = oracle.gray_scott_problem(n, n, n)
    uo, so = oracle.integrate_const(p, OS[scheme], u0, 0.0, float(nsteps), 1.0)
    stats = []
    for graph in (1, 0):
        st = gs_state(ctx, n, n, n, u0)
        st.set_option(rk.OPT_USE_GRAPH, graph)
        assert st.integrate_const(scheme, 0.0, float(nsteps), 1.0) == so == nsteps
        assert bitwise(st.get(), uo), graph
        s = st.stats()
        stats.append({k: s[k] for k in ("steps", "rhs_evals", "stage_launches", "kernel_launches", "stage_bytes")})
        st.close()
    assert stats[0] == stats[1]


def test_graph_replay_on_torch_stream():
    """The ctx stream may be torch's current (legacy default) stream, which cannot be captured:
    the graph is captured on a private stream and replayed on the ctx stream."""
    import torch
    import paper_2309_05331_b200 as rk
    c = rk.Context(0, 1, 0, torch.cuda.current_stream())
    n = 32
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=1)
    st = gs_state(c, n, n, n, u0)
    st.set_option(rk.OPT_USE_GRAPH, 1)
    assert st.integrate_const("rk4", 0.0, 9.0, 1.0) == 9
    uo, _ = oracle.integrate_const(oracle.gray_scott_problem(n, n, n), oracle.RK4, u0, 0.0, 9.0, 1.0)
    assert bitwise(st.get(), uo)
    c.close()


# ---------------------------------------------------------------------------------------
# f3: peer-to-peer halo stores with the flag handshake (RK_OPT_HALO_P2P), loopback on 1 GPU
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("scheme", ["rk4", "dopri5", "rkf78", "ab3", "abm2"])
@pytest.mark.parametrize("dims", [(16, 16, 16), (33, 17, 9), (8, 8, 1), (8, 8, 2), (8, 8, 3)],
                         ids=lambda d: "x".join(map(str, d)))
def test_gs_halo_p2p_loopback_bitwise(ctx, scheme, dims):
    """The P2P path (pack stores into the neighbours' double-buffered ghost planes, ready/ack
    flags, interior + boundary launches) with this rank as both neighbours: bitwise equal to
    the oracle over several stages and steps (both ghost parities, flag sequence > 2)."""
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=2) + 0.01 * rk_inputs.random_state(
        2 * nx * ny * nz, 10).reshape(nz, 2, ny, nx)
    st = gs_state(ctx, nx, ny, nz, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, 1)
    st.set_option(rk.OPT_HALO_P2P, 1)
    p = oracle.gray_scott_problem(nx, ny, nz)
    nsteps = 4
    for m in range(nsteps):
        st.do_step(scheme, float(m), 1.0)
    if scheme.startswith("abm"):
        ref = oracle.abm_integrate(p, int(scheme[3:]), u0, 0.0, 1.0, nsteps)
    elif scheme.startswith("ab"):
        ref = oracle.ab_integrate(p, int(scheme[2:]), u0, 0.0, 1.0, nsteps)
    else:
        ref = u0
        for m in range(nsteps):
            ref = oracle.step(p, OS[scheme], float(m), 1.0, ref)
    assert bitwise(st.get(), ref)
    s = st.stats()
    assert s["halo_exchanges"] >= 4


def test_gs_halo_p2p_adaptive_counts(ctx):
    import paper_2309_05331_b200 as rk
    n = 24
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = gs_state(ctx, n, n, n, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, 1)
    st.set_option(rk.OPT_HALO_P2P, 1)
    a, r = st.integrate_adaptive("dopri5", 0.0, 20.0, 1.0, 1e-6, 1e-6)
    uo, ao, ro, rc = oracle.integrate_adaptive(oracle.gray_scott_problem(n, n, n), oracle.DOPRI5, u0,
                                               0.0, 20.0, 1.0, 1e-6, 1e-6)
    assert rc == 0 and (a, r) == (ao, ro)
    assert bitwise(st.get(), uo)
    out = ctx.grid(n, n, n, 2)
    st.set(u0)
    st.eval_rhs(out)
    assert bitwise(out.get(), oracle.rhs(oracle.gray_scott_problem(n, n, n), u0))


# ---------------------------------------------------------------------------------------
# RK_OPT_CONTROLLER = 1: SPEC's elementary controller and ratio (R-28)
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54", "rkf78"])
@pytest.mark.parametrize("device_loop", [0, 1])
def test_spec_controller_vector(ctx, scheme, device_loop):
    """Config 2 input under SPEC's reading: counts identical to the oracle's, final state
    bitwise, for the host-driven try loop and the device-resident loop."""
    import paper_2309_05331_b200 as rk
    n = 200001
    u0 = rk_inputs.logistic_u0(n)
    st = ctx.vector(n)
    st.set_rhs_logistic()
    st.set(u0)
    st.set_option(rk.OPT_CONTROLLER, rk.CTRL_SPEC)
    st.set_option(rk.OPT_DEVICE_LOOP, device_loop)
    a, r = st.integrate_adaptive(scheme, -5.0, 5.0, 2.0, 1e-8, 1e-8)
    uo, ao, ro, rc = oracle.integrate_adaptive_ctrl(oracle.logistic_problem(n), OS[scheme], u0,
                                                    -5.0, 5.0, 2.0, 1e-8, 1e-8, oracle.CTRL_SPEC)
    assert rc == 0 and (a, r) == (ao, ro) and r > 0
    assert bitwise(st.get(), uo)


def test_spec_controller_vector_golden(ctx):
    """SURVEY Z12 [calc]: the paper's single logistic curve, DOPRI5 tol 1e-8: 46 / 3."""
    import paper_2309_05331_b200 as rk
    st = ctx.vector(1)
    st.set_rhs_logistic()
    st.set(rk_inputs.logistic_u0(1, -5.0, False))
    st.set_option(rk.OPT_CONTROLLER, rk.CTRL_SPEC)
    assert st.integrate_adaptive("dopri5", -5.0, 5.0, 0.1, 1e-8, 1e-8) == (46, 3)


@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54", "rkf78"])
@pytest.mark.parametrize("loopback", [0, 1])
def test_spec_controller_gray_scott(ctx, scheme, loopback):
    """Gray–Scott under SPEC's reading (the SPEC ratio epilogue of the fused stage kernel,
    DOPRI5's 2-slot FSAL tail): counts and final state bitwise vs the oracle."""
    import paper_2309_05331_b200 as rk
    nx, ny, nz = 33, 17, 12
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=5) + 0.02 * rk_inputs.random_state(
        2 * nx * ny * nz, 9).reshape(nz, 2, ny, nx)
    st = gs_state(ctx, nx, ny, nz, u0)
    st.set_option(rk.OPT_CONTROLLER, rk.CTRL_SPEC)
    st.set_option(rk.OPT_HALO_LOOPBACK, loopback)
    a, r = st.integrate_adaptive(scheme, 0.0, 20.0, 4.0, 1e-6, 1e-6)
    uo, ao, ro, rc = oracle.integrate_adaptive_ctrl(oracle.gray_scott_problem(nx, ny, nz),
                                                    OS[scheme], u0, 0.0, 20.0, 4.0, 1e-6, 1e-6,
                                                    oracle.CTRL_SPEC)
    assert rc == 0 and (a, r) == (ao, ro) and a > 0
    assert bitwise(st.get(), uo)


def test_spec_try_step_ratio(ctx):
    """One SPEC try: E equals the oracle's max |e|/(atol + rtol max(|u|, |u_new|))."""
    import paper_2309_05331_b200 as rk
    n = 24
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=3) + 0.05 * rk_inputs.random_state(
        2 * n ** 3, 4).reshape(n, 2, n, n)
    p = oracle.gray_scott_problem(n, n, n)
    for scheme in ("dopri5", "cash_karp54", "rkf78"):
        st = gs_state(ctx, n, n, n, u0)
        st.set_option(rk.OPT_CONTROLLER, rk.CTRL_SPEC)
        for dt in (4.0, 1.0, 0.25):
            st.set(u0)
            acc, E, dtn = st.try_step(scheme, 0.0, dt, 1e-7, 1e-7)
            un, err = oracle.step(p, OS[scheme], 0.0, dt, u0, with_error=True)
            assert E == oracle.error_ratio_max_spec(err, u0, un, 1e-7, 1e-7)
            assert (acc, dtn) == oracle.controller_spec(E, dt, 8 if scheme == "rkf78" else 5)
            assert bitwise(st.get(), un if acc else u0)


# ---------------------------------------------------------------------------------------
# RK_OPT_CHECK_FINITE: a non-finite state is RK_ERR_DIVERGED carrying t
# ---------------------------------------------------------------------------------------
def test_check_finite_grid(ctx):
    import paper_2309_05331_b200 as rk
    n = 16
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=1)
    st = gs_state(ctx, n, n, n, u0)
    st.set_option(rk.OPT_CHECK_FINITE, 1)
    assert st.integrate_const("rk4", 0.0, 5.0, 1.0) == 5           # finite: no error
    st.set_rhs_gray_scott(d1=1e6)                                  # explicit RK blows up
    with pytest.raises(rk.RKError) as e:
        st.integrate_const("rk4", 0.0, 400.0, 1.0)
    assert e.value.status == "RK_ERR_DIVERGED"
    t = st.stats()["diverged_t"]
    assert 1.0 <= t < 400.0 and t == int(t)
    assert not np.all(np.isfinite(st.get()))


def test_check_finite_vector_and_default_off(ctx):
    import paper_2309_05331_b200 as rk
    st = ctx.vector(1000)
    st.set_rhs_exponential(1.0)
    st.set(np.full(1000, 1.0))
    assert st.integrate_const("rk4", 0.0, 1000.0, 1.0) == 1000      # overflows, unchecked
    assert not np.all(np.isfinite(st.get()))
    st.set(np.full(1000, 1.0))
    st.set_option(rk.OPT_CHECK_FINITE, 64)
    with pytest.raises(rk.RKError) as e:
        st.integrate_const("rk4", 0.0, 1000.0, 1.0)
    assert e.value.status == "RK_ERR_DIVERGED"
    assert st.stats()["diverged_t"] in [64.0 * j for j in range(1, 16)]
    st.set(np.full(1000, 1.0))
    with pytest.raises(rk.RKError) as e:
        for i in range(1000):
            st.do_step("rk4", float(i), 1.0)
    assert e.value.status == "RK_ERR_DIVERGED"


# ---------------------------------------------------------------------------------------
# K5: persistent cooperative small-grid steps (RK_OPT_COOP_MAX_CELLS, rk_smallgrid.cu)
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("dims", [(64, 64, 64), (33, 17, 9), (1, 1, 3), (70, 9, 20)],
                         ids=lambda d: "x".join(map(str, d)))
def test_coop_integrate_const_one_launch(ctx, scheme, dims):
    """integrate_const through K5: one launch for all steps (odd and even counts, so the final
    state sits in either ping-pong buffer), bitwise equal to the oracle, counters as K3's."""
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=8) + 0.01 * rk_inputs.random_state(
        2 * nx * ny * nz, 3).reshape(nz, 2, ny, nx)
    p = oracle.gray_scott_problem(nx, ny, nz)
    for nsteps in (5, 6):
        uo, so = oracle.integrate_const(p, OS[scheme], u0, 0.0, float(nsteps), 1.0)
        stats = []
        for coop in (True, False):
            st = gs_state(ctx, nx, ny, nz, u0, coop=coop)
            assert st.integrate_const(scheme, 0.0, float(nsteps), 1.0) == so == nsteps
            assert bitwise(st.get(), uo), (coop, nsteps)
            s = st.stats()
            stats.append(s)
            st.close()
        assert stats[0]["kernel_launches"] == 2  # ring fill of set() + one K5 launch
        for k in ("steps", "rhs_evals", "stage_bytes"):
            assert stats[0][k] == stats[1][k], k


def test_coop_threshold_and_mixing(ctx):
    """Above RK_OPT_COOP_MAX_CELLS the stage path runs; K5 steps, K3 steps and adaptive tries
    interleave on one state (FSAL k1 invalidated by K5 steps) with the oracle's results."""
    import paper_2309_05331_b200 as rk
    n = 24
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=2)
    p = oracle.gray_scott_problem(n, n, n)
    st = gs_state(ctx, n, n, n, u0, coop=True)
    st.set_option(rk.OPT_COOP_MAX_CELLS, n ** 3 - 1)
    st.do_step("rk4", 0.0, 1.0)
    assert st.stats()["kernel_launches"] == 1 + 4  # ring fill of set() + 4 stage launches
    st.set_option(rk.OPT_COOP_MAX_CELLS, n ** 3)
    st.do_step("rk4", 1.0, 1.0)
    acc, E, dtn = st.try_step("dopri5", 2.0, 1.0, 1e-6, 1e-6)
    st.do_step("dopri5", 3.0, 0.5)
    acc2, E2, _ = st.try_step("dopri5", 3.5, 0.5, 1e-6, 1e-6)
    u = oracle.step(p, oracle.RK4, 0.0, 1.0, u0)
    u = oracle.step(p, oracle.RK4, 1.0, 1.0, u)
    un, err = oracle.step(p, oracle.DOPRI5, 2.0, 1.0, u, with_error=True)
    assert E == oracle.error_ratio_max(err, u, oracle.rhs(p, u), 1.0, 1e-6, 1e-6)
    u = un if acc else u
    u = oracle.step(p, oracle.DOPRI5, 3.0, 0.5, u)
    un, err = oracle.step(p, oracle.DOPRI5, 3.5, 0.5, u, with_error=True)
    assert E2 == oracle.error_ratio_max(err, u, oracle.rhs(p, u), 0.5, 1e-6, 1e-6)
    assert bitwise(st.get(), un if acc2 else u)


# ---------------------------------------------------------------------------------------
# K5 device loop on a grid: the whole integrate_adaptive in one cooperative launch
# (RK_OPT_DEVICE_LOOP within RK_OPT_COOP_MAX_CELLS; R-27)
# ---------------------------------------------------------------------------------------
def _gs_adaptive(ctx, dims, u0, scheme, dt0, tol, device_loop, ctrl=0, max_tries=None):
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    st = gs_state(ctx, nx, ny, nz, u0, coop=True)
    st.set_option(rk.OPT_DEVICE_LOOP, device_loop)
    st.set_option(rk.OPT_CONTROLLER, ctrl)
    if max_tries:
        st.set_option(rk.OPT_MAX_TRIES, max_tries)
    st.reset_stats()
    try:
        a, r = st.integrate_adaptive(scheme, 0.0, 20.0, dt0, tol, tol)
        return st.get(), a, r, st.stats()
    finally:
        st.close()


@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54", "rkf78"])
@pytest.mark.parametrize("ctrl", [0, 1], ids=["odeint", "spec"])
@pytest.mark.parametrize("dims", [(32, 32, 32), (33, 17, 9)], ids=lambda d: "x".join(map(str, d)))
def test_device_loop_grid_bitwise(ctx, scheme, ctrl, dims):
    """Accepted / rejected counts equal the oracle's, in one kernel launch, with rejections
    (dt0 = 4 is too large on purpose), and the final state is bitwise equal.  The controller's
    pow is the correctly rounded x^y everywhere (R-27: double-double on the device and
    in the host loop, binary128 in the oracle); this input (33x17x9 / Odeint / DOPRI5) used to
    hit one of the ~0.1 % of arguments where glibc's pow is an ulp off."""
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=4) + 0.02 * rk_inputs.random_state(
        2 * nx * ny * nz, 5).reshape(nz, 2, ny, nx)
    g, a, r, s = _gs_adaptive(ctx, dims, u0, scheme, 4.0, 1e-6, 1, ctrl)
    uo, ao, ro, rc = oracle.integrate_adaptive_ctrl(oracle.gray_scott_problem(nx, ny, nz), OS[scheme], u0,
                                                    0.0, 20.0, 4.0, 1e-6, 1e-6, ctrl)
    assert rc == 0 and (a, r) == (ao, ro) and r > 0
    assert s["kernel_launches"] == 1 and s["tries"] == a + r
    assert bitwise(g, uo)
    gh, ah, rh, sh = _gs_adaptive(ctx, dims, u0, scheme, 4.0, 1e-6, 0, ctrl)
    assert (ah, rh) == (a, r) and bitwise(gh, g) and sh["last_dt"] == s["last_dt"]


def test_device_loop_grid_errors(ctx):
    import paper_2309_05331_b200 as rk
    n = 16
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=1)
    bad = u0.copy()
    bad[3, 1, 4, 5] = np.nan
    with pytest.raises(rk.RKError) as e:
        _gs_adaptive(ctx, (n, n, n), bad, "dopri5", 1.0, 1e-6, 1)
    assert e.value.status == "RK_ERR_DIVERGED"
    with pytest.raises(rk.RKError) as e:  # dt0 = 20 needs rejections: stall at one try
        _gs_adaptive(ctx, (n, n, n), u0 + 0.05 * rk_inputs.random_state(2 * n ** 3, 2).reshape(n, 2, n, n),
                     "dopri5", 20.0, 1e-10, 1, max_tries=1)
    assert e.value.status == "RK_ERR_STALL"


@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54", "rkf78"])
@pytest.mark.parametrize("p2p", [0, 1], ids=["nccl_path", "p2p"])
@pytest.mark.parametrize("overlap", [1, 0])
@pytest.mark.parametrize("dims", [(24, 24, 24), (33, 17, 3), (16, 8, 2), (16, 8, 1)],
                         ids=lambda d: "x".join(map(str, d)))
def test_gs_halo_loopback_adaptive(ctx, scheme, p2p, overlap, dims):
    """Error-controlled runs through the multi-GPU stage path on one GPU (pack, ghost planes,
    interior + boundary launches; the write-ahead stage's Y_F is what the final stage's pack
    ships): counts and final state bitwise vs the oracle, incl. slabs of 1..3 planes."""
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=6) + 0.02 * rk_inputs.random_state(
        2 * nx * ny * nz, 8).reshape(nz, 2, ny, nx)
    st = gs_state(ctx, nx, ny, nz, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, 1)
    st.set_option(rk.OPT_HALO_P2P, p2p)
    st.set_option(rk.OPT_HALO_OVERLAP, overlap)
    a, r = st.integrate_adaptive(scheme, 0.0, 10.0, 4.0, 1e-6, 1e-6)
    uo, ao, ro, rc = oracle.integrate_adaptive(oracle.gray_scott_problem(nx, ny, nz), OS[scheme], u0,
                                               0.0, 10.0, 4.0, 1e-6, 1e-6)
    assert rc == 0 and (a, r) == (ao, ro) and r > 0
    assert bitwise(st.get(), uo)


def test_max_size_1024_cubed_rk4(ctx):
    """Maximum size: a 1024^3 grid (2^31 values per array, 16 GiB; five arrays for RK4 fill
    ~81 GiB of HBM), so padded offsets of the upper planes exceed int32.  One RK4 step in the
    default launch configuration; sampled cells (incl. the last planes and the periodic
    corners) bitwise against the oracle on their radius-5 neighbourhoods."""
    import gc
    gc.collect()
    n = 1024
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = gs_state(ctx, n, n, n, u0)
    st.do_step("rk4", 0.0, 1.0)
    g = st.get()
    st.close()
    lo, hi = rk_inputs.cube_range(n)
    pts = [(1023, 1023, 1023), (1023, 0, 511), (1022, 1023, 0), (0, 0, 0), (lo, lo, lo),
           (hi - 1, hi, lo - 1), (hi, 700, hi - 1), (900, lo + 3, hi)]
    r = 5
    p = oracle.gray_scott_problem(2 * r + 1, 2 * r + 1, 2 * r + 1)
    for (z, y, x) in pts:
        blk = _sample_block(u0, z, y, x, r)
        out = oracle.step(p, oracle.RK4, 0.0, 1.0, blk).reshape(blk.shape)
        assert bitwise(g[z, :, y, x], out[r, :, r, r]), (z, y, x)
    del g, u0
    gc.collect()


@pytest.mark.parametrize("coop", [True, False], ids=["k5", "k3"])
def test_gs32_20000_steps_bitwise_golden(ctx, coop):
    """20000 RK4 steps of Gray–Scott 32^3 (S:L515 run length): the final state's SHA-256 equals
    the oracle's (tests/golden/gs32_rk4_20000.json, written by make_gs32_longrun.py from oracle/
    only).  C1 decays into fp64 denormals on the way, so this pins FTZ-free arithmetic."""
    import hashlib
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "gs32_rk4_20000.json")))
    n = 32
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = gs_state(ctx, n, n, n, u0, coop=coop)
    steps = st.integrate_const("rk4", 0.0, float(gold["steps"]), 1.0)
    assert steps == gold["steps"]
    g = np.ascontiguousarray(st.get(), dtype="<f8")
    assert float(g[:, 1].min()) == gold["c1_min"] and float(g[:, 0].max()) == gold["c0_max"]
    assert hashlib.sha256(g.tobytes()).hexdigest() == gold["sha256_final"]


def test_checkpoint_resume_bitwise(ctx):
    """Checkpoint = rk_state_get (+ t, dt), resume = rk_state_set on a NEW state: the resumed
    run equals the uninterrupted one bit for bit -- fixed RK4 through integrate_const, and
    error-controlled DOPRI5 through try_step (same accepted dt sequence; the resumed state
    recomputes k1 = F(u), the same value FSAL would have carried)."""
    nx, ny, nz = 40, 24, 20
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=8) + 0.01 * rk_inputs.random_state(2 * nx * ny * nz, 2).reshape(nz, 2, ny, nx)
    a = gs_state(ctx, nx, ny, nz, u0)
    a.integrate_const("rk4", 0.0, 10.0, 1.0)
    b = gs_state(ctx, nx, ny, nz, u0)
    b.integrate_const("rk4", 0.0, 5.0, 1.0)
    c = gs_state(ctx, nx, ny, nz, b.get())
    c.integrate_const("rk4", 5.0, 10.0, 1.0)
    assert bitwise(a.get(), c.get())

    def accepted_steps(st, t, dt, n):
        seq = []
        while len(seq) < n:
            ok, E, dtn = st.try_step("dopri5", t, dt, 1e-6, 1e-6)
            if ok:
                seq.append(dt)
                t += dt
            dt = dtn
        return t, dt, seq

    full = gs_state(ctx, nx, ny, nz, u0)
    _, _, seq_full = accepted_steps(full, 0.0, 1.0, 8)
    part = gs_state(ctx, nx, ny, nz, u0)
    t, dt, seq1 = accepted_steps(part, 0.0, 1.0, 3)
    ck = part.get()
    res = gs_state(ctx, nx, ny, nz, ck)
    _, _, seq2 = accepted_steps(res, t, dt, 5)
    assert seq1 + seq2 == seq_full
    assert bitwise(full.get(), res.get())
