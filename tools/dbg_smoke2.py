import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
def mt(p): return time.ctime(os.path.getmtime(p)) if os.path.exists(p) else None
for f in ["paper_2309_05331_b200/librkb200.so", "oracle/liboracle.so", "oracle/rk_oracle.c", "build/rkb200/rk_runtime.o"]:
    print(f, mt(os.path.join(ROOT, f)))
import __graft_entry__ as ge
from paper_2309_05331_b200 import build as b
print("rk stale?", b._stale(b.LIB, [os.path.join(b.BUILD, s.replace('.cu','.o')) for s in b.SOURCES]))
ge.build()
for f in ["paper_2309_05331_b200/librkb200.so", "oracle/liboracle.so"]:
    print(f, mt(os.path.join(ROOT, f)))
import oracle, rk_inputs, paper_2309_05331_b200 as rk
n = 24
u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
ctx = rk.Context(0, 1, 0)
st = ctx.grid(n, n, n, 2); st.set_rhs_gray_scott(); st.set(u0)
st.do_step(rk.RK4, 0.0, 1.0)
p = oracle.gray_scott_problem(n, n, n)
want = oracle.step(p, oracle.RK4, 0.0, 1.0, u0).reshape(u0.shape)
got = st.get()
bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
print("mismatch", len(bad), bad[:4].tolist())
if len(bad):
    z,c,y,x = bad[0]; print(got[z,c,y,x], want[z,c,y,x])
