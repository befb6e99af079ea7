"""GPU parity of the device-resident try loop for grids beyond the K5 size (RK_OPT_DEVICE_LOOP,
SURVEY f3; rk_runtime.cu graph_adaptive_loop): the whole rk_integrate_adaptive runs as one
CUDA-graph launch (conditional WHILE over SWITCH-selected try bodies and a controller kernel),
with no host round trip per try.  Gate: accepted / rejected counts identical to the oracle and
the final state bitwise equal (R-17, R-27), equal to the host-driven loop too.
RK_OPT_COOP_MAX_CELLS = 0 sends small grids down this path (K5 would take them otherwise)."""
import numpy as np
import pytest

import oracle
import rk_inputs

pytestmark = pytest.mark.gpu
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


def make(ctx, dims, u0, device_loop=1, ctrl=0, max_tries=None):
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    st = ctx.grid(nx, ny, nz, 2)
    st.set_rhs_gray_scott()
    st.set(u0)
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    st.set_option(rk.OPT_DEVICE_LOOP, device_loop)
    st.set_option(rk.OPT_CONTROLLER, ctrl)
    if max_tries:
        st.set_option(rk.OPT_MAX_TRIES, max_tries)
    return st


def ic(dims, seed=4, amp=0.02):
    nx, ny, nz = dims
    return rk_inputs.gray_scott_ic(nx, ny, nz, seed=seed) + amp * rk_inputs.random_state(
        2 * nx * ny * nz, seed + 1).reshape(nz, 2, ny, nx)


@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54", "rkf78"])
@pytest.mark.parametrize("ctrl", [0, 1], ids=["odeint", "spec"])
@pytest.mark.parametrize("dims", [(32, 32, 32), (33, 17, 9), (70, 9, 20)], ids=lambda d: "x".join(map(str, d)))
def test_graph_loop_bitwise(ctx, scheme, ctrl, dims):
    nx, ny, nz = dims
    u0 = ic(dims)
    st = make(ctx, dims, u0, 1, ctrl)
    st.reset_stats()
    a, r = st.integrate_adaptive(scheme, 0.0, 20.0, 4.0, 1e-6, 1e-6)  # dt0 = 4: rejections
    s = st.stats()
    uo, ao, ro, rc = oracle.integrate_adaptive_ctrl(oracle.gray_scott_problem(nx, ny, nz), OS[scheme], u0,
                                                    0.0, 20.0, 4.0, 1e-6, 1e-6, ctrl)
    assert rc == 0 and (a, r) == (ao, ro) and r > 0
    assert s["tries"] == a + r
    g = st.get()
    assert bitwise(g, uo)
    h = make(ctx, dims, u0, 0, ctrl)  # host-driven loop: same counts, same bits, same last dt
    ah, rh = h.integrate_adaptive(scheme, 0.0, 20.0, 4.0, 1e-6, 1e-6)
    assert (ah, rh) == (a, r) and bitwise(h.get(), g)
    assert h.stats()["last_dt"] == s["last_dt"] and h.stats()["last_err_ratio"] == s["last_err_ratio"]
    st.close()
    h.close()


@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54"])
def test_graph_loop_reuse_and_continuation(ctx, scheme):
    """The captured graph is reused across calls whatever buffer holds u (odd / even accepted
    counts flip the parity), and stepping continues correctly after it (FSAL k1 included)."""
    dims = (40, 24, 20)
    nx, ny, nz = dims
    u0 = ic(dims, seed=9)
    p = oracle.gray_scott_problem(nx, ny, nz)
    st = make(ctx, dims, u0)
    u = u0
    t = 0.0
    for t1 in (3.0, 7.5, 8.0, 15.0):
        a, r = st.integrate_adaptive(scheme, t, t1, 1.0, 1e-6, 1e-6)
        u, ao, ro, rc = oracle.integrate_adaptive(p, OS[scheme], u, t, t1, 1.0, 1e-6, 1e-6)
        assert rc == 0 and (a, r) == (ao, ro)
        assert bitwise(st.get(), u), t1
        t = t1
    # a try_step and a fixed step after the graph loop see the right u (and, for DOPRI5, k1)
    acc, E, dtn = st.try_step(scheme, t, 0.5, 1e-6, 1e-6)
    un, err = oracle.step(p, OS[scheme], t, 0.5, u, with_error=True)
    assert E == oracle.error_ratio_max(err, u, oracle.rhs(p, u), 0.5, 1e-6, 1e-6)
    u = un if acc else u
    assert bitwise(st.get(), u)
    st.do_step("rk4", t, 1.0)
    assert bitwise(st.get(), oracle.step(p, oracle.RK4, t, 1.0, u))
    st.close()


def test_graph_loop_errors(ctx):
    import paper_2309_05331_b200 as rk
    dims = (16, 16, 16)
    u0 = ic(dims, seed=1, amp=0.0)
    bad = u0.copy()
    bad[3, 1, 4, 5] = np.nan
    st = make(ctx, dims, bad)
    with pytest.raises(rk.RKError) as e:
        st.integrate_adaptive("dopri5", 0.0, 20.0, 1.0, 1e-6, 1e-6)
    assert e.value.status == "RK_ERR_DIVERGED"
    st.close()
    st = make(ctx, dims, ic(dims, seed=1, amp=0.05), max_tries=1)
    with pytest.raises(rk.RKError) as e:  # dt0 = 20 needs rejections: stall at one try
        st.integrate_adaptive("dopri5", 0.0, 20.0, 20.0, 1e-10, 1e-10)
    assert e.value.status == "RK_ERR_STALL"
    st.close()


def test_graph_loop_one_launch_per_integration(ctx):
    """No host work per try: a whole integration is one graph launch, the try count and the
    launch accounting come back from the device state."""
    dims = (48, 32, 24)
    u0 = ic(dims, seed=12)
    st = make(ctx, dims, u0)
    st.integrate_adaptive("dopri5", 0.0, 20.0, 1.0, 1e-6, 1e-6)  # build + first run
    st.set(u0)
    st.reset_stats()
    a, r = st.integrate_adaptive("dopri5", 0.0, 20.0, 1.0, 1e-6, 1e-6)
    s = st.stats()
    assert s["tries"] == a + r and s["stage_launches"] == 6 * (a + r) + 1  # FSAL: k1 once
    st.close()
