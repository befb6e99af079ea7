"""ncu target: a few K7 RK4 steps at 512^3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_05331_b200 as rk  # noqa: E402
import rk_inputs  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = rk.Context(0, 1, 0, torch.cuda.current_stream())
st = ctx.grid(512, 512, 512, 2)
st.set_rhs_gray_scott()
st.set(rk_inputs.gray_scott_ic(512, 512, 512, seed=42))
st.set_option(rk.OPT_FUSED_STEP, mode)
for _ in range(3):
    st.do_step("rk4", 0.0, 1.0)
torch.cuda.synchronize()
print("done")
