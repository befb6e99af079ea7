"""Developer timing: small Gray-Scott grids, RK4 integrate_const over 20 steps -- K5 (persistent
cooperative launch) vs K8 stage pairs (launched per step, and replayed from a CUDA graph)."""
import statistics

import torch

import paper_2309_05331_b200 as rk
import rk_inputs

ctx = rk.Context(0, 1, 0, torch.cuda.current_stream())
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for n in (32, 48, 64, 96, 128):
    g = ctx.grid(n, n, n, 2)
    g.set_rhs_gray_scott(h=2.5 / 64)
    u = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    res = {}
    for mode in ("k5", "k8", "k8_graph", "k3"):
        g.set_option(rk.OPT_COOP_MAX_CELLS, n ** 3 if mode == "k5" else 0)
        g.set_option(rk.OPT_FUSED_STEP, 0 if mode == "k3" else 3)
        g.set_option(rk.OPT_USE_GRAPH, 1 if mode == "k8_graph" else 0)
        g.set(u)
        g.integrate_const("rk4", 0.0, 20.0, 1.0)
        ms = []
        for _ in range(5):
            g.set(u)
            torch.cuda.synchronize()
            ev0.record()
            g.integrate_const("rk4", 0.0, 20.0, 1.0)
            ev1.record()
            torch.cuda.synchronize()
            ms.append(ev0.elapsed_time(ev1))
        res[mode] = statistics.median(ms) / 20 * 1e3
    print(f"{n}^3 RK4 us/step: " + ", ".join(f"{k} {v:.1f}" for k, v in res.items()), flush=True)
    g.close()
ctx.close()
