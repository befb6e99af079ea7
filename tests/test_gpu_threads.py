"""API calls from host threads that have made no CUDA call of their own (a serving thread pool,
the e2e pipeline's workers): every entry point binds its context's device first (DeviceGuard in
rk_runtime.cu), so the driver-API calls behind it (TMA descriptor encoding) find a current
context.  Without that, the first K8 launch from a fresh thread failed with "invalid argument"
in cuTensorMapEncodeTiled.  Results are compared bitwise with the oracle (R-17)."""
import threading

import numpy as np
import pytest

import oracle
import rk_inputs

pytestmark = pytest.mark.gpu


def bitwise(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def in_thread(fn):
    out = {}

    def run():
        try:
            out["value"] = fn()
        except BaseException as e:  # noqa: BLE001 -- re-raised in the test thread
            out["error"] = e

    t = threading.Thread(target=run)
    t.start()
    t.join()
    if "error" in out:
        raise out["error"]
    return out["value"]


DIMS = (64, 32, 9)  # tile-aligned: the DOPRI5 try runs the K8 head and tail pairs


def test_state_from_main_thread_used_in_fresh_thread():
    import paper_2309_05331_b200 as rk
    u0 = rk_inputs.gray_scott_ic(*DIMS, seed=3)
    p = oracle.gray_scott_problem(*DIMS)
    ctx = rk.Context(0, 1, 0)
    st = ctx.grid(*DIMS, 2)
    st.set_rhs_gray_scott()
    st.set(u0)
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    acc, E, _ = in_thread(lambda: st.try_step("dopri5", 0.0, 1.0, 1e-6, 1e-6))
    un, err = oracle.step(p, oracle.DOPRI5, 0.0, 1.0, u0, with_error=True)
    assert E == oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), 1.0, 1e-6, 1e-6)
    assert bitwise(in_thread(st.get), un if acc else u0)
    st.set(u0)
    in_thread(lambda: st.do_step("rk4", 0.0, 1.0))
    assert bitwise(st.get(), oracle.step(p, oracle.RK4, 0.0, 1.0, u0))
    st.close()
    ctx.close()


def test_context_and_state_created_in_fresh_thread():
    import paper_2309_05331_b200 as rk
    u0 = rk_inputs.gray_scott_ic(*DIMS, seed=4)
    p = oracle.gray_scott_problem(*DIMS)

    def work():
        ctx = rk.Context(0, 1, 0)
        st = ctx.grid(*DIMS, 2)
        st.set_rhs_gray_scott()
        st.set(u0)
        st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
        acc, rej = st.integrate_adaptive("dopri5", 0.0, 5.0, 1.0, 1e-6, 1e-6)
        got = st.get()
        st.close()
        ctx.close()
        return acc, rej, got

    acc, rej, got = in_thread(work)
    want, a_o, r_o, rc = oracle.integrate_adaptive(p, oracle.DOPRI5, u0, 0.0, 5.0, 1.0, 1e-6, 1e-6)
    assert rc == 0 and (acc, rej) == (a_o, r_o)
    assert bitwise(got, want)
