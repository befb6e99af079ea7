"""ncu target: K8 pair launches at 512^3 (RK4 and explicit midpoint steps after warm-up)."""
import sys

import torch

import paper_2309_05331_b200 as rk
import rk_inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = rk.Context(0, 1, 0, torch.cuda.current_stream())
st = ctx.grid(n, n, n, 2)
st.set_rhs_gray_scott(h=0.0390625)
st.set(torch.from_numpy(rk_inputs.gray_scott_ic(n, n, n, seed=42)).cuda())
st.set_option(rk.OPT_FUSED_STEP, 3)
for scheme in ("rk4", "midpoint"):
    for k in range(3):
        st.do_step(scheme, float(k), 1.0)
torch.cuda.synchronize()
st.close()
ctx.close()
