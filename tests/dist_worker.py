"""Multi-GPU check of the halo path (SURVEY §4 tests/dist): launched by torchrun with one rank
per GPU (tests/test_dist_nccl.py; skipped on a one-GPU box).  Every rank owns a z-slab of a
Gray–Scott grid; after RK4 steps, an error-controlled DOPRI5 integration (allreduce(max) of
the error norm every try) and with both halo transports (NCCL send/recv; P2P stores over
NVLink), the gathered state must equal the fp64 oracle's single-domain run bit for bit (so
every ghost plane was fresh every stage), and a NaN on one rank must stop every rank
with RK_ERR_DIVERGED (allreduce NaN propagation).  Exit code 0 = pass."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

import oracle
import paper_2309_05331_b200 as rk
import rk_inputs


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    stream = torch.cuda.current_stream()
    ctx = rk.Context.from_torch_distributed(local, stream)
    # failure detection on: host waits poll NCCL's async error state (10-minute deadline)
    nx, ny, nz = 40, 24, 7 * world + 3  # ragged slabs (remainder planes on the low ranks)
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=42)
    u0 = u0 + 0.01 * rk_inputs.random_state(u0.size, 5).reshape(u0.shape)
    p = oracle.gray_scott_problem(nx, ny, nz)
    failures = []

    def gather(st):
        parts = [None] * world
        dist.all_gather_object(parts, (st.begin, np.ascontiguousarray(st.get())))
        return np.concatenate([a for _, a in sorted(parts, key=lambda x: x[0])], axis=0)

    for p2p in (0, 1):
        for overlap in (1, 0):
            st = ctx.grid(nx, ny, nz, 2)
            st.set_rhs_gray_scott()
            st.set_option(rk.OPT_COMM_TIMEOUT_MS, 600000)
            if world == 1:  # one GPU: the same halo code path through the loopback exchange
                st.set_option(rk.OPT_HALO_LOOPBACK, 1)
            st.set_option(rk.OPT_HALO_OVERLAP, overlap)
            st.set_option(rk.OPT_HALO_P2P, p2p)
            st.set(np.ascontiguousarray(u0[st.begin:st.begin + st.local]))
            for k in range(3):
                st.do_step("rk4", float(k), 1.0)
            g = gather(st)
            ref = u0
            for k in range(3):
                ref = oracle.step(p, oracle.RK4, float(k), 1.0, ref)
            if rank == 0 and not np.array_equal(g.view(np.uint64), ref.view(np.uint64)):
                failures.append(f"rk4 p2p={p2p} overlap={overlap}")
            st.set(np.ascontiguousarray(u0[st.begin:st.begin + st.local]))
            acc, rej = st.integrate_adaptive("dopri5", 0.0, 6.0, 1.0, 1e-6, 1e-6)
            g = gather(st)
            ro, ao, jo, rc = oracle.integrate_adaptive(p, oracle.DOPRI5, u0, 0.0, 6.0, 1.0, 1e-6, 1e-6)
            if rank == 0 and ((acc, rej) != (ao, jo) or not np.array_equal(g.view(np.uint64), ro.view(np.uint64))):
                failures.append(f"dopri5 p2p={p2p} overlap={overlap}: {(acc, rej)} vs {(ao, jo)}")
            st.close()
    # NaN on the last rank only: every rank must report divergence
    st = ctx.grid(nx, ny, nz, 2)
    st.set_rhs_gray_scott()
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
        failures.append(f"NaN propagation: {flags}")
    st.close()
    ctx.close()
    dist.destroy_process_group()
    if rank == 0:
        print("FAILURES:", failures if failures else "none", flush=True)
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
