"""Repro for write-ahead stage issues: a few adaptive / fixed Gray–Scott runs vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, rk_inputs
import paper_2309_05331_b200 as rk

ctx = rk.Context(0, 1, 0)
n = 32
u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
for scheme in sys.argv[1:] or ["cash_karp54"]:
    st = ctx.grid(n, n, n, 2)
    st.set_rhs_gray_scott()
    st.set(u0)
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    try:
        a, r = st.integrate_adaptive(scheme, 0.0, 20.0, 1.0, 1e-6, 1e-6)
        uo, ao, ro, rc = oracle.integrate_adaptive(oracle.gray_scott_problem(n, n, n), oracle.SCHEMES[scheme], u0, 0.0, 20.0, 1.0, 1e-6, 1e-6)
        print(scheme, (a, r), (ao, ro), np.array_equal(st.get().view(np.uint64), uo.ravel().view(np.uint64)))
    except Exception as e:
        print(scheme, "ERROR", e)
    st.close()
