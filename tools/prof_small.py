"""configs[2] (64^3 Gray–Scott RK4) launch-bound study: a few integrate_const steps, for ncu."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_05331_b200 as rk  # noqa: E402
import rk_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = rk.Context(0, 1, 0)
g = ctx.grid(n, n, n, 2)
g.set_rhs_gray_scott()
if os.environ.get("K3"):  # force the stage-by-stage TMA path
    g.set_option(rk.OPT_COOP_MAX_CELLS, 0)
g.set(rk_inputs.gray_scott_ic(n, n, n, seed=42))
g.integrate_const("rk4", 0.0, float(steps), 1.0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
g.integrate_const("rk4", 0.0, 20.0, 1.0)
e1.record()
torch.cuda.synchronize()
print(f"{'K3' if os.environ.get('K3') else 'K5'} {os.environ.get('RKB_K5_MINB', '')} {n}^3 rk4: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/step")
g.close()
ctx.close()
