import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, rk_inputs, paper_2309_05331_b200 as rk
ctx = rk.Context(0, 1, 0)
for n in (24, 16, 32, 20, 25):
    for pert in (0, 1):
        u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
        if pert:
            u0 = u0 + 0.01 * rk_inputs.random_state(u0.size, 5).reshape(u0.shape)
        st = ctx.grid(n, n, n, 2); st.set_rhs_gray_scott(); st.set(u0)
        st.do_step(rk.RK4, 0.0, 1.0)
        p = oracle.gray_scott_problem(n, n, n)
        want = oracle.step(p, oracle.RK4, 0.0, 1.0, u0).reshape(u0.shape)
        got = st.get()
        bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
        print(n, pert, "mismatches", len(bad), bad[:5].tolist(), flush=True)
        if len(bad):
            z,c,y,x = bad[0]
            print("  got", got[z,c,y,x], "want", want[z,c,y,x], "diff", got[z,c,y,x]-want[z,c,y,x])
        st.close()
