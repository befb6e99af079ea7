"""Multi-process check of the P2P transport WITHOUT NCCL on ONE GPU (tests/test_shared_gpu.py):
torchrun starts `world` ranks that all use cuda:0 (NCCL refuses that), a gloo process group
carries only the CUDA IPC handle exchange (rk_p2p_export / rk_p2p_import) and the result
gathering.  Every rank owns a z-slab of a Gray–Scott grid; the pack kernels store Y_i's
boundary planes into the z-neighbours' ghost planes in ANOTHER process through CUDA IPC
mappings, the error ratio is reduced by atomicMax into every rank's mapped flag block (no
NCCL anywhere).  Checked bitwise against the fp64 oracle's single-domain run: RK4 steps, DOPRI5
error control through the host try loop and through the device-resident graph loop, a
logistic vector under DOPRI5 error control, norm_inf, and NaN propagation to every rank.  The
P2P exchange is timed (pack-kernel stores, CUDA events).  Exit code 0 = pass."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

import oracle
import paper_2309_05331_b200 as rk
import rk_inputs


def main():
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = rk.Context.from_torch_distributed(0, None, transport="p2p")
    nx, ny, nz = 40, 24, 5 * world + 2  # ragged slabs (remainder planes on the low ranks)
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=42)
    u0 = u0 + 0.01 * rk_inputs.random_state(u0.size, 5).reshape(u0.shape)
    p = oracle.gray_scott_problem(nx, ny, nz)
    failures, info = [], {}

    def gather(st):
        parts = [None] * world
        dist.all_gather_object(parts, (st.begin, np.ascontiguousarray(st.get())))
        return np.concatenate([a for _, a in sorted(parts, key=lambda x: x[0])], axis=0)

    def same(a, b):
        return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))

    for overlap in (1, 0):
        st = ctx.grid(nx, ny, nz, 2)
        st.set_rhs_gray_scott()
        st.set_option(rk.OPT_HALO_OVERLAP, overlap)
        st.set(np.ascontiguousarray(u0[st.begin:st.begin + st.local]))
        st.set_option(rk.OPT_TIMING, 1)
        for k in range(3):
            st.do_step("rk4", float(k), 1.0)
        s = st.stats()
        st.set_option(rk.OPT_TIMING, 0)
        if overlap:
            info["halo_exchanges"] = s["halo_exchanges"]
            info["ms_per_exchange"] = s["halo_ms"] / max(1, s["halo_exchanges"])
            info["bytes_per_exchange"] = s["halo_bytes"] / max(1, s["halo_exchanges"])
        g = gather(st)
        ref = u0
        for k in range(3):
            ref = oracle.step(p, oracle.RK4, float(k), 1.0, ref)
        if rank == 0 and not same(g, ref):
            failures.append(f"rk4 overlap={overlap}")
        ro, ao, jo, rc = oracle.integrate_adaptive(p, oracle.DOPRI5, u0, 0.0, 6.0, 2.0, 1e-6, 1e-6)
        for dl in (0, 1):
            st.set(np.ascontiguousarray(u0[st.begin:st.begin + st.local]))
            st.set_option(rk.OPT_DEVICE_LOOP, dl)
            st.reset_stats()
            acc, rej = st.integrate_adaptive("dopri5", 0.0, 6.0, 2.0, 1e-6, 1e-6)
            g = gather(st)
            if rank == 0 and ((acc, rej) != (ao, jo) or not same(g, ro)):
                failures.append(f"dopri5 device_loop={dl} overlap={overlap}: {(acc, rej)} vs {(ao, jo)}")
            if dl:
                info["graph_loop_tries"] = st.stats()["tries"]
        st.set_option(rk.OPT_DEVICE_LOOP, 0)
        m = st.norm_inf()
        if rank == 0 and m != float(np.max(np.abs(g))):
            failures.append(f"norm_inf {m}")
        st.close()
    # a logistic vector under error control: the E allreduce through the P2P flag blocks
    n = 1001
    v = ctx.vector(n)
    v.set_rhs_logistic()
    ul = rk_inputs.logistic_u0(n)
    v.set(np.ascontiguousarray(ul[v.begin:v.begin + v.local]))
    acc, rej = v.integrate_adaptive("dopri5", -5.0, 5.0, 0.1, 1e-8, 1e-8)
    parts = [None] * world
    dist.all_gather_object(parts, (v.begin, v.get().ravel().copy()))
    gv = np.concatenate([a for _, a in sorted(parts, key=lambda x: x[0])])
    uo, ao, jo, rc = oracle.integrate_adaptive(oracle.logistic_problem(n), oracle.DOPRI5, ul, -5.0, 5.0, 0.1,
                                               1e-8, 1e-8)
    if rank == 0 and ((acc, rej) != (ao, jo) or not same(gv, uo)):
        failures.append(f"logistic vector: {(acc, rej)} vs {(ao, jo)}")
    v.close()
    # NaN on the last rank only: every rank must report divergence (host loop and graph loop)
    for dl in (0, 1):
        st = ctx.grid(nx, ny, nz, 2)
        st.set_rhs_gray_scott()
        st.set_option(rk.OPT_DEVICE_LOOP, dl)
        blk = np.ascontiguousarray(u0[st.begin:st.begin + st.local]).copy()
        if rank == world - 1:
            blk[0, 0, 0, 0] = np.nan
        st.set(blk)
        try:
            st.integrate_adaptive("dopri5", 0.0, 2.0, 1.0, 1e-6, 1e-6)
            diverged = False
        except rk.RKError as e:
            diverged = "DIVERGED" in str(e).upper()
        flags = [None] * world
        dist.all_gather_object(flags, diverged)
        if rank == 0 and not all(flags):
            failures.append(f"NaN propagation (device_loop={dl}): {flags}")
        st.close()
    # RK_OPT_CHECK_ARGS: identical arguments pass; a rank calling with another dt makes every
    # rank return RK_ERR_CONTRACT before any collective work
    st = ctx.grid(nx, ny, nz, 2)
    st.set_rhs_gray_scott()
    st.set(np.ascontiguousarray(u0[st.begin:st.begin + st.local]))
    st.set_option(rk.OPT_CHECK_ARGS, 1)
    st.do_step("rk4", 0.0, 1.0)
    try:
        st.do_step("rk4", 1.0, 0.5 if rank == world - 1 else 1.0)
        status = "ok"
    except rk.RKError as e:
        status = e.status
    flags = [None] * world
    dist.all_gather_object(flags, status)
    if rank == 0 and flags != ["RK_ERR_CONTRACT"] * world:
        failures.append(f"collective argument check: {flags}")
    st.close()
    ctx.close()
    dist.destroy_process_group()
    if rank == 0:
        print("INFO:", json.dumps(info), flush=True)
        print("FAILURES:", failures if failures else "none", flush=True)
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
