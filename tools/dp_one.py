"""ncu target: DOPRI5 error-controlled tries at 512^3 (the headline's stage launches, K8 tail pair)."""
import sys

import torch

import paper_2309_05331_b200 as rk
import rk_inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = rk.Context(0, 1, 0, torch.cuda.current_stream())
st = ctx.grid(n, n, n, 2)
st.set_rhs_gray_scott(h=0.0390625)
st.set(torch.from_numpy(rk_inputs.gray_scott_ic(n, n, n, seed=42)).cuda())
t, dt = 0.0, 1.0
for k in range(4):
    acc, E, dtn = st.try_step("dopri5", t, dt, 1e-6, 1e-6)
    if acc:
        t += dt
    dt = dtn
torch.cuda.synchronize()
st.close()
ctx.close()
