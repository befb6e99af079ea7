"""GPU parity at production launch configurations, mixed-scheme state transitions, and the NCCL
calls of the one-GPU loopback path.

* Full-array parity at 256x256x100 (VERDICT r1 "What's weak" 3): at this size pick_zchunk keeps
  the production z chunks (48 planes for heavy stages, 16 for light two-row stages, 8 for
  Y-direct stages), the last chunk of every launch is ragged (100 = 2*48 + 4 = 6*16 + 4 =
  12*8 + 4) and the Y-direct mbarrier ring (R = 6 planes) wraps -- unlike the <= 64^3 grids
  of test_gpu_parity.py.  Every element is compared with the oracle, bitwise, through the
  one-GPU path and through the multi-GPU stage path (loopback: NCCL self send/recv).
* Adams steps between Runge-Kutta steps on the same state: k1 must not survive
  a change of u made by an Adams step.
* The loopback path runs NCCL (a 1-rank communicator): NCCL_DEBUG=INFO shows it.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import rk_inputs

pytestmark = pytest.mark.gpu
OS = oracle.SCHEMES
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctx():
    import paper_2309_05331_b200 as rk
    c = rk.Context(0, 1, 0)
    yield c
    c.close()


def bitwise(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def first_mismatch(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    bad = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
    return (bad.size, bad[:4], a[bad[:4]], b[bad[:4]]) if bad.size else None


def gs_state(ctx, dims, u0, loopback=0):
    import paper_2309_05331_b200 as rk
    nx, ny, nz = dims
    st = ctx.grid(nx, ny, nz, 2)
    st.set_rhs_gray_scott()
    st.set(u0)
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    st.set_option(rk.OPT_HALO_LOOPBACK, loopback)
    return st


_U0 = {}
_ORACLE = {}


def prod_u0(dims):
    if dims not in _U0:
        nx, ny, nz = dims
        # the R-6 IC plus a small seeded perturbation, so every cell is non-trivial
        _U0[dims] = rk_inputs.gray_scott_ic(nx, ny, nz, seed=42) + 0.01 * rk_inputs.random_state(
            2 * nx * ny * nz, 13).reshape(nz, 2, ny, nx)
    return _U0[dims]


def oracle_result(dims, case):
    """(state, extra) of one case on the oracle, computed once per module."""
    key = (dims, case)
    if key not in _ORACLE:
        u0 = prod_u0(dims)
        p = oracle.gray_scott_problem(*dims)
        kind, name = case
        if kind == "step":
            _ORACLE[key] = (oracle.step(p, OS[name], 0.0, 1.0, u0), None)
        elif kind == "try":  # one error-controlled try at dt = 1, tol 1e-6 (bench's first try)
            un, err = oracle.step(p, OS[name], 0.0, 1.0, u0, with_error=True)
            E = oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), 1.0, 1e-6, 1e-6)
            _ORACLE[key] = (un, E)
        elif kind == "ab":  # k+1 Adams-Bashforth steps (k-1 RKF78 bootstrap steps first)
            k = int(name[2:])
            _ORACLE[key] = (oracle.ab_integrate(p, k, u0, 0.0, 1.0, k + 1), None)
    return _ORACLE[key]


PROD = (256, 256, 100)
CASES = [("try", "dopri5"), ("try", "cash_karp54"), ("step", "rk4"), ("step", "rkf78"), ("ab", "ab4"),
         ("step", "modified_midpoint")]


@pytest.mark.parametrize("loopback", [0, 1], ids=["one_gpu", "halo_path"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}")
def test_production_chunks_full_array(ctx, case, loopback):
    dims = PROD
    u0 = prod_u0(dims)
    want, E_o = oracle_result(dims, case)
    st = gs_state(ctx, dims, u0, loopback)
    kind, name = case
    try:
        if kind == "step":
            st.do_step(name, 0.0, 1.0)
            got = st.get()
        elif kind == "try":
            acc, E, _ = st.try_step(name, 0.0, 1.0, 1e-6, 1e-6)
            assert E == E_o, (E, E_o)
            got = st.get()
            if not acc:  # a rejected try leaves u; compare the proposal through u_new instead
                want = u0
        else:
            k = int(name[2:])
            for m in range(k + 1):
                st.do_step(name, float(m), 1.0)
            got = st.get()
        assert bitwise(got, want), first_mismatch(got, want)
        if loopback:
            assert st.stats()["halo_exchanges"] > 0
    finally:
        st.close()


@pytest.mark.parametrize("case", [("try", "dopri5"), ("step", "rk4")], ids=lambda c: c[1])
def test_production_chunks_ragged_tiles(ctx, case):
    """Same production chunks with ragged x and y tiles (250 = 7*32 + 26, 254 = 31*8 + 6)."""
    dims = (250, 254, 100)
    u0 = prod_u0(dims)
    want, E_o = oracle_result(dims, case)
    st = gs_state(ctx, dims, u0)
    try:
        if case[0] == "step":
            st.do_step(case[1], 0.0, 1.0)
        else:
            acc, E, _ = st.try_step(case[1], 0.0, 1.0, 1e-6, 1e-6)
            assert E == E_o
            if not acc:
                want = u0
        got = st.get()
        assert bitwise(got, want), first_mismatch(got, want)
    finally:
        st.close()


@pytest.mark.parametrize("loopback", [0, 1])
@pytest.mark.parametrize("dims", [(24, 16, 12), (33, 17, 9)], ids=lambda d: "x".join(map(str, d)))
def test_adams_between_rk_steps(ctx, dims, loopback):
    """DOPRI5 try (accepted: k1 <- k7 = F(u_new) via FSAL), then AB1 and ABM1 steps (no
    bootstrap, no stored k), then RK4 and another DOPRI5 try: every state and E equal the
    oracle's -- the RK steps after an Adams step must recompute k1 = F(u)."""
    nx, ny, nz = dims
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=21) + 0.01 * rk_inputs.random_state(
        2 * nx * ny * nz, 22).reshape(nz, 2, ny, nx)
    p = oracle.gray_scott_problem(nx, ny, nz)
    st = gs_state(ctx, dims, u0, loopback)

    def try_dopri(u, t):
        acc, E, dtn = st.try_step("dopri5", t, 1.0, 1e-3, 1e-3)
        un, err = oracle.step(p, oracle.DOPRI5, t, 1.0, u, with_error=True)
        assert E == oracle.error_ratio_max(err, u, oracle.rhs(p, u), 1.0, 1e-3, 1e-3)
        assert acc, E
        assert bitwise(st.get(), un)
        return un

    u = try_dopri(u0, 0.0)
    st.do_step("ab1", 1.0, 1.0)
    u = oracle.ab_integrate(p, 1, u, 1.0, 1.0, 1)
    assert bitwise(st.get(), u)
    st.do_step("abm1", 2.0, 1.0)
    u = oracle.abm_integrate(p, 1, u, 2.0, 1.0, 1)
    assert bitwise(st.get(), u)
    st.do_step("rk4", 3.0, 1.0)
    u = oracle.step(p, oracle.RK4, 3.0, 1.0, u)
    assert bitwise(st.get(), u)
    u = try_dopri(u, 4.0)
    st.do_step("abm1", 5.0, 1.0)
    u = oracle.abm_integrate(p, 1, u, 5.0, 1.0, 1)
    u = try_dopri(u, 6.0)
    st.close()


_NCCL_PROBE = r"""
import numpy as np, sys
sys.path.insert(0, sys.argv[1])
import paper_2309_05331_b200 as rk, rk_inputs
ctx = rk.Context(0, 1, 0)
st = ctx.grid(16, 16, 8, 2)
st.set_rhs_gray_scott()
st.set(rk_inputs.gray_scott_ic(16, 16, 8, seed=42))
st.set_option(rk.OPT_HALO_LOOPBACK, 1)
acc, E, dtn = st.try_step("dopri5", 0.0, 1.0, 1e-6, 1e-6)
s = st.stats()
print("probe", acc, E, s["halo_exchanges"], s["halo_bytes"], flush=True)
st.close(); ctx.close()
"""


def test_loopback_runs_nccl():
    """The loopback halo path executes real NCCL calls: a 1-rank communicator is created and
    the self send/recv + allreduce run (NCCL_DEBUG=INFO lines on stderr)."""
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,P2P,COLL")
    r = subprocess.run([sys.executable, "-c", _NCCL_PROBE, ROOT], capture_output=True, text=True,
                       timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    out = r.stdout + r.stderr
    assert "probe True" in out or "probe False" in out
    assert "NCCL INFO" in out, out[-3000:]
    assert "nranks 1" in out, out[-3000:]
    lines = [ln for ln in out.splitlines() if "NCCL INFO" in ln]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "nccl_loopback_info.txt"), "w") as f:
        f.write("\n".join(lines[:200]) + "\n")


@pytest.mark.parametrize("kind", ["grid", "vector"])
def test_error_spike_forces_rejection(ctx, kind):
    """RK_OPT_ERROR_SPIKE (S:L519 criterion 8): the spiked try is rejected, leaves u bitwise
    unchanged, and shrinks dt by at least the safety factor (here to the 1/5 floor: E >= 1e6);
    the next tries proceed normally (the host loop and the oracle agree again)."""
    import paper_2309_05331_b200 as rk
    if kind == "grid":
        dims = (24, 16, 12)
        u0 = rk_inputs.gray_scott_ic(*dims, seed=3) + 0.01 * rk_inputs.random_state(2 * 24 * 16 * 12, 4).reshape(12, 2, 16, 24)
        st = gs_state(ctx, dims, u0)
        p = oracle.gray_scott_problem(*dims)
        dt = 1.0
    else:
        n = 1000
        u0 = rk_inputs.logistic_u0(n)
        st = ctx.vector(n)
        st.set_rhs_logistic()
        st.set(u0)
        p = oracle.logistic_problem(n)
        dt = 0.1
    st.set_option(rk.OPT_ERROR_SPIKE, 1)
    acc, E, dtn = st.try_step("dopri5", 0.0, dt, 1e-6, 1e-6)
    assert not acc and E >= 1e6
    assert bitwise(st.get(), u0)
    assert dtn <= 0.9 * dt and dtn == dt * 0.2
    acc, E, dtn2 = st.try_step("dopri5", 0.0, dtn, 1e-6, 1e-6)  # spike consumed: normal try
    un, err = oracle.step(p, oracle.DOPRI5, 0.0, dtn, u0, with_error=True)
    assert E == oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), dtn, 1e-6, 1e-6)
    assert bitwise(st.get(), un if acc else u0)
    # inside integrate_adaptive: the spiked 2nd try is rejected on top of the natural rejections
    st.set(u0)
    a0, r0 = st.integrate_adaptive("dopri5", 0.0, 10 * dt, dt, 1e-6, 1e-6)
    assert a0 + r0 >= 2
    st.set(u0)
    st.set_option(rk.OPT_ERROR_SPIKE, 2)
    st.reset_stats()
    a1, r1 = st.integrate_adaptive("dopri5", 0.0, 10 * dt, dt, 1e-6, 1e-6)
    assert r1 >= r0 + 1 and a1 >= 1 and st.stats()["rejected"] == r1
    st.close()


@pytest.mark.parametrize("scheme", ["euler", "rk4", "cash_karp54", "dopri5", "rkf78", "midpoint", "modified_midpoint"])
@pytest.mark.parametrize("loopback", [0, 1])
def test_unfused_kernels_fixed_bitwise(ctx, scheme, loopback):
    """RK_OPT_FUSED_KERNELS = 0 (the Odeint-like unfused dataflow): every stage value
    and k_j through HBM, the same sums -- bitwise equal to the oracle (and so to the fused path)."""
    import paper_2309_05331_b200 as rk
    dims = (33, 17, 9)
    u0 = rk_inputs.gray_scott_ic(*dims, seed=5) + 0.01 * rk_inputs.random_state(2 * 33 * 17 * 9, 6).reshape(9, 2, 17, 33)
    st = gs_state(ctx, dims, u0, loopback)
    st.set_option(rk.OPT_FUSED_KERNELS, 0)
    p = oracle.gray_scott_problem(*dims)
    u = u0
    for k in range(2):
        st.do_step(scheme, float(k), 1.0)
        u = oracle.step(p, OS[scheme], float(k), 1.0, u)
        assert bitwise(st.get(), u), (scheme, k)
    st.close()


@pytest.mark.parametrize("scheme", ["dopri5", "cash_karp54", "rkf78"])
@pytest.mark.parametrize("ctrl", [0, 1], ids=["odeint", "spec"])
@pytest.mark.parametrize("kind", ["grid", "grid_loopback", "vector"])
def test_unfused_kernels_adaptive(ctx, scheme, ctrl, kind):
    import paper_2309_05331_b200 as rk
    if kind == "vector":
        n = 5000
        u0 = rk_inputs.logistic_u0(n)
        st = ctx.vector(n)
        st.set_rhs_logistic()
        st.set(u0)
        p, t0, t1, dt0, tol = oracle.logistic_problem(n), -5.0, 5.0, 0.1, 1e-8
    else:
        dims = (24, 16, 12)
        u0 = rk_inputs.gray_scott_ic(*dims, seed=7) + 0.02 * rk_inputs.random_state(2 * 24 * 16 * 12, 8).reshape(12, 2, 16, 24)
        st = gs_state(ctx, dims, u0, 1 if kind == "grid_loopback" else 0)
        p, t0, t1, dt0, tol = oracle.gray_scott_problem(*dims), 0.0, 12.0, 4.0, 1e-6
    st.set_option(rk.OPT_FUSED_KERNELS, 0)
    st.set_option(rk.OPT_CONTROLLER, ctrl)
    a, r = st.integrate_adaptive(scheme, t0, t1, dt0, tol, tol)
    uo, ao, ro, rc = oracle.integrate_adaptive_ctrl(p, OS[scheme], u0, t0, t1, dt0, tol, tol, ctrl)
    assert rc == 0 and (a, r) == (ao, ro)
    assert bitwise(st.get(), uo)
    st.close()


@pytest.mark.parametrize("kind", ["vector", "grid"])
@pytest.mark.parametrize("device_loop", [0, 1])
def test_dt_underflow_parity(ctx, kind, device_loop):
    """RK_ERR_DT_UNDERFLOW (R-29) at the same try as the oracle: with an unattainable
    tolerance every try is rejected until dt < 16 eps max(|t|, 1); u is left untouched."""
    import paper_2309_05331_b200 as rk
    if kind == "vector":
        n = 64
        u0 = rk_inputs.logistic_u0(n)
        st = ctx.vector(n)
        st.set_rhs_logistic()
        p, t0, t1, dt0 = oracle.logistic_problem(n), -5.0, 5.0, 0.1
    else:
        dims = (16, 8, 6)
        u0 = rk_inputs.gray_scott_ic(*dims, seed=2) + 0.01 * rk_inputs.random_state(2 * 16 * 8 * 6, 3).reshape(6, 2, 8, 16)
        st = gs_state(ctx, dims, u0)
        p, t0, t1, dt0 = oracle.gray_scott_problem(*dims), 0.0, 20.0, 1.0
    st.set(u0)
    st.set_option(rk.OPT_DEVICE_LOOP, device_loop)
    st.reset_stats()
    uo, ao, ro, rc = oracle.integrate_adaptive(p, oracle.DOPRI5, u0, t0, t1, dt0, 1e-300, 1e-300)
    assert rc == oracle.ERR_DT_UNDERFLOW and ao == 0 and ro > 0
    with pytest.raises(rk.RKError) as e:
        st.integrate_adaptive("dopri5", t0, t1, dt0, 1e-300, 1e-300)
    assert e.value.status == "RK_ERR_DT_UNDERFLOW"
    s = st.stats()
    assert (s["accepted"], s["rejected"]) == (ao, ro)
    assert bitwise(st.get(), uo) and bitwise(uo, u0)
    st.close()


def test_torch_allocator_hook():
    """rk_ctx_set_allocator: with allocator="torch" the state arrays come from
    torch's caching allocator (torch.cuda.memory_allocated grows by them and shrinks back on
    close) and results are unchanged."""
    import torch

    import paper_2309_05331_b200 as rk
    dims = (40, 24, 10)
    u0 = rk_inputs.gray_scott_ic(*dims, seed=11)
    p = oracle.gray_scott_problem(*dims)
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_allocated(0)
    c = rk.Context(0, 1, 0, allocator="torch")
    st = c.grid(*dims, 2)
    st.set_rhs_gray_scott()
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    st.set(u0)
    st.do_step("rk4", 0.0, 1.0)
    acc, E, dtn = st.try_step("dopri5", 1.0, 1.0, 1e-6, 1e-6)
    u = oracle.step(p, oracle.RK4, 0.0, 1.0, u0)
    un, err = oracle.step(p, oracle.DOPRI5, 1.0, 1.0, u, with_error=True)
    assert bitwise(st.get(), un if acc else u)
    arr = (dims[1] + 2) * (dims[0] + 2 + (dims[0] % 2)) * 2 * dims[2] * 8  # one padded array
    assert torch.cuda.memory_allocated(0) - m0 >= 8 * arr  # u, u_new, k1..k6 at least
    st.close()
    c.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated(0) == m0


def test_comm_deadline_counts_progress_not_backlog(ctx):
    """RK_OPT_COMM_TIMEOUT_MS runs from the last collective PROGRESS.  A 128^3 RK4
    integrate_const through the loopback halo path (NCCL 1-rank communicator) enqueues ~40 ms of
    stages and exchanges without a host wait; a 2 ms deadline must not abort it (every exchange
    completes within a stage), nor may it abort plain compute of another state on the same
    context once no collective is outstanding; results stay bitwise."""
    import paper_2309_05331_b200 as rk
    dims = (128, 128, 128)
    u0 = rk_inputs.gray_scott_ic(*dims, seed=42)
    st = gs_state(ctx, dims, u0, loopback=1)
    st.set_option(rk.OPT_COMM_TIMEOUT_MS, 2)
    n = st.integrate_const("rk4", 0.0, 60.0, 1.0)
    assert n == 60
    ref = gs_state(ctx, dims, u0)
    ref.integrate_const("rk4", 0.0, 60.0, 1.0)
    assert bitwise(st.get(), ref.get())
    st.set_option(rk.OPT_COMM_TIMEOUT_MS, 0)
    st.close()
    ref.close()


def test_512_full_array_parity(ctx):
    """The headline configuration in full (configs[3], 512^3, bench.py's launch configuration):
    DOPRI5 error-controlled tries as integrate_adaptive takes them from the IC (dt0 = 1 is
    rejected; the controller's dt is accepted) -- E, the decision and the proposed dt equal,
    u unchanged after the rejection and the accepted new state equal -- and one RK4 step, EVERY
    element bitwise against the oracle's single-domain run (~70 s of oracle time, ~25 GB of
    host memory)."""
    import gc
    n = 512
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    p = oracle.gray_scott_problem(n, n, n)
    st = gs_state(ctx, (n, n, n), u0)
    k1 = oracle.rhs(p, u0)
    dt = 1.0
    for _ in range(2):  # the bench's first try (rejected at dt0 = 1), then the controller's dt
        acc, E, dtn = st.try_step("dopri5", 0.0, dt, 1e-6, 1e-6)
        un, err = oracle.step(p, oracle.DOPRI5, 0.0, dt, u0, with_error=True)
        Eo = oracle.error_ratio_max(err, u0, k1, dt, 1e-6, 1e-6)
        del err
        gc.collect()
        assert E == Eo, (E, Eo)
        acc_o, dt_o = oracle.controller(Eo, dt)
        assert (acc, dtn) == (acc_o, dt_o)
        got = st.get()
        want = un if acc else u0
        assert bitwise(got, want), first_mismatch(got, want)
        del un, got, want
        gc.collect()
        if acc:
            break
        dt = dtn
    assert acc  # the accepted try's full new state was compared
    del k1
    st.set(u0)
    st.do_step("rk4", 0.0, 1.0)
    got = st.get()
    want = oracle.step(p, oracle.RK4, 0.0, 1.0, u0)
    assert bitwise(got, want), first_mismatch(got, want)
    st.close()
    del got, want, u0
    gc.collect()

