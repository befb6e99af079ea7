"""Developer timing: K6 / K7 fused whole-step vs K3 stage-by-stage at 512^3 (RK4, midpoints)."""
import os
import sys

import torch

import paper_2309_05331_b200 as rk
import rk_inputs


def run(scheme, fused, n=512, steps=10, fz=None):
    if fz:
        os.environ["RKB_FZ"] = str(fz)
        os.environ["RKB_PZ"] = str(fz)
    ctx = rk.Context(0, 1, 0, torch.cuda.current_stream())
    st = ctx.grid(n, n, n, 2)
    st.set_rhs_gray_scott()
    st.set(rk_inputs.gray_scott_ic(n, n, n, seed=42))
    st.set_option(rk.OPT_FUSED_STEP, fused)
    for _ in range(3):
        st.do_step(scheme, 0.0, 1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        st.do_step(scheme, 0.0, 1.0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    st.close()
    ctx.close()
    os.environ.pop("RKB_FZ", None)
    os.environ.pop("RKB_PZ", None)
    return ms


if __name__ == "__main__":
    for scheme in sys.argv[1:] or ["rk4", "midpoint"]:
        k3 = run(scheme, 0)
        print(f"{scheme} K3 stage-by-stage: {k3:.3f} ms/step  {512**3 / k3 / 1e6:.3e} cell-updates/s", flush=True)
        for mode in [int(m) for m in os.environ.get("FT_MODES", "1,2").split(",")]:
            for fz in [int(f) for f in os.environ.get("FT_FZ", "32,64,128").split(",")]:
                f = run(scheme, mode, fz=fz)
                print(f"{scheme} K{5 + mode} fused fz={fz}: {f:.3f} ms/step  {512**3 / f / 1e6:.3e} cell-updates/s  "
                      f"x{k3 / f:.2f}", flush=True)
