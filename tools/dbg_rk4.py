import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, rk_inputs, paper_2309_05331_b200 as rk
ctx = rk.Context(0, 1, 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
scheme = sys.argv[2] if len(sys.argv) > 2 else "rk4"
u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
st = ctx.grid(n, n, n, 2); st.set_rhs_gray_scott(); st.set(u0)
st.do_step(scheme, 0.0, 1.0)
g = st.get()
want = oracle.step(oracle.gray_scott_problem(n, n, n), oracle.SCHEMES[scheme], 0.0, 1.0, u0).reshape(u0.shape)
print(n, scheme, "mismatch", np.count_nonzero(g != want))
