"""Developer: configs[1] (logistic N = 1e6, DOPRI5 tol 1e-8) through the device loop (ncu target)."""
import torch

import paper_2309_05331_b200 as rk
import rk_inputs

n = 1000000
ctx = rk.Context(0, 1, 0, torch.cuda.current_stream())
st = ctx.vector(n)
st.set_rhs_logistic()
st.set_option(rk.OPT_DEVICE_LOOP, 1)
for _ in range(2):
    st.set(rk_inputs.logistic_u0(n))
    print(st.integrate_adaptive("dopri5", -5.0, 5.0, 0.1, 1e-8, 1e-8))
torch.cuda.synchronize()
