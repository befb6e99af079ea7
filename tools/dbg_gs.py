import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, rk_inputs, paper_2309_05331_b200 as rk
ctx = rk.Context(0, 1, 0)
for dims in [(4,4,4), (8,8,8), (6,4,4), (4,6,4), (4,4,6), (64,8,4)]:
    nx, ny, nz = dims
    u0 = np.ones((nz,2,ny,nx)); u0[:,1] = 0
    u0[:, 0] += np.arange(nx)[None,None,:] * 1e-3 + np.arange(ny)[None,:,None] * 1e-2 + np.arange(nz)[:,None,None]*1e-1
    st = ctx.grid(nx, ny, nz, 2); st.set_rhs_gray_scott(d1=1.0, d2=0.0, F=0.0, K=0.0, h=1.0); st.set(u0)
    g0 = st.get()
    print(dims, "roundtrip ok", np.array_equal(g0, u0))
    st.do_step("euler", 0.0, 1.0)
    p = oracle.gray_scott_problem(nx, ny, nz, d1=1.0, d2=0.0, F=0.0, K=0.0, h=1.0)
    want = oracle.step(p, oracle.EULER, 0.0, 1.0, u0).reshape(u0.shape)
    got = st.get()
    d = got - want
    bad = np.argwhere(d != 0)
    print("  mismatches", len(bad))
    for b in bad[:8]:
        z,c,y,x = b; print("   ", b.tolist(), "diff(lap err)", d[z,c,y,x])
