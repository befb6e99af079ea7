"""Developer: a few K6 steps at 512^3 (ncu target)."""
import sys

import torch

import paper_2309_05331_b200 as rk
import rk_inputs

scheme = sys.argv[1] if len(sys.argv) > 1 else "rk4"
n = 512
ctx = rk.Context(0, 1, 0, torch.cuda.current_stream())
st = ctx.grid(n, n, n, 2)
st.set_rhs_gray_scott()
st.set(rk_inputs.gray_scott_ic(n, n, n, seed=42))
st.set_option(rk.OPT_FUSED_STEP, 1)
for _ in range(3):
    st.do_step(scheme, 0.0, 1.0)
torch.cuda.synchronize()
