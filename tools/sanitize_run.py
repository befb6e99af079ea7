"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every scheme on a ragged 40x12x10 grid (K5) and 40x21x13 (K3, K6), the loopback multi-GPU halo path
(NCCL and P2P, incl. the P2P allreduce), adaptive tries, the device-resident graph loop, the
unfused dataflow, Adams-Bashforth and the algebra ops.
Run:  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2309_05331_b200 as rk  # noqa: E402
import rk_inputs  # noqa: E402

ctx = rk.Context(0, 1, 0)
# SAN_NO_NCCL=1: skip the NCCL loopback sections (compute-sanitizer racecheck and NCCL's own
# kernels / proxy thread do not mix; every other section runs)
NO_NCCL = os.environ.get("SAN_NO_NCCL") == "1"
# SAN_SECTIONS: comma list of sections to run (default all): base, k3k6, r2, k8, vector
SECTIONS = set(os.environ.get("SAN_SECTIONS", "base,k3k6,r2,k8,vector").split(","))


def mark(msg):
    print("section", msg, flush=True)

nx, ny, nz = 40, 12, 10
u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=3) + 0.01 * rk_inputs.random_state(2 * nx * ny * nz, 1).reshape(nz, 2, ny, nx)
for loop in ((0,) if NO_NCCL else (0, 1)) if "base" in SECTIONS else ():
    mark(f"base loopback={loop}")
    st = ctx.grid(nx, ny, nz, 2)
    st.set_rhs_gray_scott()
    st.set_option(rk.OPT_HALO_LOOPBACK, loop)
    st.set(u0)
    for s in ("euler", "midpoint", "modified_midpoint", "rk4", "cash_karp54", "dopri5", "rkf78", "ab3"):
        st.do_step(s, 0.0, 1.0)
    for s in ("cash_karp54", "dopri5", "rkf78"):
        st.try_step(s, 0.0, 0.5, 1e-6, 1e-6)
    st.get()
    st.close()
# the stage-by-stage kernels on a small grid (K5 off) and K6 (whole-step fusion, several z chunks)
os.environ["RKB_FZ"] = "3"
for fused in (0, 1) if "k3k6" in SECTIONS else ():
    mark(f"k3k6 fused={fused}")
    st = ctx.grid(nx, ny + 9, nz + 3, 2)
    st.set_rhs_gray_scott()
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    st.set_option(rk.OPT_FUSED_STEP, fused)
    st.set(rk_inputs.gray_scott_ic(nx, ny + 9, nz + 3, seed=4))
    for s in ("midpoint", "modified_midpoint", "rk4", "dopri5"):
        st.do_step(s, 0.0, 1.0)
    st.get()
    st.close()
# round 2 paths: P2P loopback under error control (device stage counter + P2P allreduce), the
# device-resident graph loop (plain and over P2P), the unfused dataflow, chunk groups (z chunks)
# SAN_NO_GRAPH=1 skips the device-resident graph loop (conditional graph nodes crash the
# racecheck tool's host side; memcheck / synccheck / initcheck run them)
R2 = ((1, 0, 1), (1, 1, 1), (0, 1, 1), (0, 0, 0))
NO_GRAPH = os.environ.get("SAN_NO_GRAPH") == "1"
if NO_GRAPH:
    R2 = tuple(v for v in R2 if v[1] == 0)
for p2p, dl, fk in R2 if "r2" in SECTIONS else ():
    mark(f"r2 p2p={p2p} device_loop={dl} fused_kernels={fk}")
    st = ctx.grid(nx, ny + 9, nz + 3, 2)
    st.set_rhs_gray_scott()
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    st.set_option(rk.OPT_HALO_LOOPBACK, p2p)
    st.set_option(rk.OPT_HALO_P2P, p2p)
    st.set_option(rk.OPT_DEVICE_LOOP, dl)
    st.set_option(rk.OPT_FUSED_KERNELS, fk)
    st.set(rk_inputs.gray_scott_ic(nx, ny + 9, nz + 3, seed=5))
    st.integrate_adaptive("dopri5", 0.0, 6.0, 2.0, 1e-6, 1e-6)
    st.integrate_adaptive("cash_karp54", 6.0, 8.0, 1.0, 1e-6, 1e-6)
    st.get()
    st.close()
# K8 stage pairs (tile-aligned grid: RK4 pairs, the explicit midpoint pair, Gragg's pair, the
# DOPRI5 head and tail pairs inside error-controlled tries and the device-resident try loop), several z chunks so chunk edges and the edge-CTA patch list run
if "k8" in SECTIONS:
    mark("k8")
    os.environ["RKB_PZ"] = "5"
    st = ctx.grid(64, 32, 11, 2)
    st.set_rhs_gray_scott()
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    st.set(rk_inputs.gray_scott_ic(64, 32, 11, seed=6))
    for s in ("rk4", "midpoint", "modified_midpoint", "rk4"):
        st.do_step(s, 0.0, 1.0)
    for k in range(3):  # the head pair (stages 2 + 3) and the tail pair (6 + 7) of every try
        st.try_step("dopri5", float(k), 0.5, 1e-6, 1e-6)
    if not NO_GRAPH:  # the device-resident graph try loop: the pairs' device-dt (DTP) variants
        st.set_option(rk.OPT_DEVICE_LOOP, 1)
        st.integrate_adaptive("dopri5", 0.0, 2.0, 0.5, 1e-6, 1e-6)
        st.set_option(rk.OPT_DEVICE_LOOP, 0)
    st.get()
    st.close()
    if not NO_NCCL:  # the pairs on the slab path: ghost planes through the 1-rank NCCL loopback
        mark("k8 loopback")
        st = ctx.grid(64, 32, 11, 2)
        st.set_rhs_gray_scott()
        st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
        st.set_option(rk.OPT_HALO_LOOPBACK, 1)
        st.set(rk_inputs.gray_scott_ic(64, 32, 11, seed=7))
        for s in ("rk4", "midpoint"):
            st.do_step(s, 0.0, 1.0)
        for k in range(2):
            st.try_step("dopri5", float(k), 0.5, 1e-6, 1e-6)
        st.get()
        st.close()
    os.environ.pop("RKB_PZ")
mark("vector")
v = ctx.vector(1001)
v.set_rhs_logistic()
v.set(rk_inputs.logistic_u0(1001))
v.integrate_adaptive("dopri5", -5.0, 5.0, 0.1, 1e-8, 1e-8)
v.integrate_const("ab4", 0.0, 1.0, 0.05)
w = ctx.vector(1001)
w.lincomb([1.0, 2.0], [v, v])
print("norm", w.norm_inf())
ctx.close()
print("sanitize workload done")
