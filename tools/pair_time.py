"""Per-role launch times of DOPRI5 tries at 512^3 (RK_OPT_TIMING), independent of the results
(for timing experiments whose arithmetic is deliberately incomplete).  python tools/pair_time.py [n] [tries]"""
import sys

import torch

import paper_2309_05331_b200 as rk
import rk_inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
tries = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ctx = rk.Context(0, 1, 0, torch.cuda.current_stream())
st = ctx.grid(n, n, n, 2)
st.set_rhs_gray_scott(h=0.0390625)
st.set(torch.from_numpy(rk_inputs.gray_scott_ic(n, n, n, seed=42)).cuda())
for _ in range(2):
    try:
        st.try_step("dopri5", 0.0, 1.0, 1e-6, 1e-6)
    except Exception as e:  # noqa: BLE001
        print("warm-up:", e)
st.set_option(rk.OPT_TIMING, 1)
st.reset_stats()
for _ in range(tries):
    try:
        st.try_step("dopri5", 0.0, 1.0, 1e-6, 1e-6)
    except Exception as e:  # noqa: BLE001
        print("try:", e)
torch.cuda.synchronize()
s = st.stats()
h = s["head_kernel_ms"] / max(1, s["head_launches"])
m = s.get("mid_kernel_ms", 0.0) / max(1, s.get("mid_launches", 0))
t = (s["pair_kernel_ms"] - s["head_kernel_ms"] - s.get("mid_kernel_ms", 0.0)) / max(1, tries)
k3 = (s["stage_kernel_ms"] - s["pair_kernel_ms"]) / max(1, tries)
print(f"per try: head {h:.3f} mid {m:.3f} tail {t:.3f} k3 {k3:.3f} ms  (stage total {s['stage_kernel_ms'] / tries:.3f})")
st.close()
ctx.close()
