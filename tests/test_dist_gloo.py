"""Multi-rank host logic on CPU (gloo, world 2..4): the NCCL unique-id broadcast used by
rk_ctx_create, the z-slab partition, and the library's per-stage halo exchange plan
(rk_halo_plan_get) executed with real point-to-point messages between processes: every
rank's ghost planes must receive its periodic z-neighbours' boundary planes (P:L168, P:L176
ghost_get).  The device path runs the same plan with NCCL send/recv."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nz, plane_shape, q):
    import torch
    import torch.distributed as dist

    import paper_2309_05331_b200 as rk
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        uid = rk.api.broadcast_unique_id()
        uids = [None] * world
        dist.all_gather_object(uids, uid)
        z0, nzl = rk.partition(nz, world, rank)
        # a plane is tagged with its global z index in every value
        send = torch.stack([torch.full(plane_shape, float(z0), dtype=torch.float64),
                            torch.full(plane_shape, float(z0 + nzl - 1), dtype=torch.float64)])
        ghost = torch.full((2,) + plane_shape, -1.0, dtype=torch.float64)
        plan = rk.halo_plan(world, rank)
        reqs = []
        for m in plan["msgs"]:
            buf = ghost if m["recv"] else send
            view = buf[m["slot"]:m["slot"] + m["nplanes"]].contiguous()
            if m["recv"]:
                reqs.append((dist.irecv(view, src=m["peer"]), view, m["slot"]))
            else:
                reqs.append((dist.isend(view, dst=m["peer"]), None, None))
        for r, view, slot in reqs:
            r.wait()
            if view is not None:
                ghost[slot:slot + view.shape[0]] = view
        q.put((rank, uid, uids, z0, nzl, plan, float(ghost[0].min()), float(ghost[0].max()),
               float(ghost[1].min()), float(ghost[1].max())))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world,nz", [(2, 8), (2, 7), (3, 13), (4, 9), (4, 4)])
def test_halo_plan_gloo(world, nz):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nz, (3, 5), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res = sorted(res, key=lambda r: r[0])
    for r in res:
        assert len(r) > 2, r
    parts = [(r[3], r[4]) for r in res]
    assert sum(n for _, n in parts) == nz and all(n >= 1 for _, n in parts)
    for rank, uid, uids, z0, nzl, plan, hi_min, hi_max, lo_min, lo_max in res:
        assert len(uid) == 128 and all(u == uids[0] for u in uids)     # same NCCL id everywhere
        assert plan["up"] == (rank + 1) % world and plan["down"] == (rank - 1) % world
        # ghost slot 0 = plane z0+nzl (periodic), slot 1 = plane z0-1 (periodic)
        assert hi_min == hi_max == float((z0 + nzl) % nz)
        assert lo_min == lo_max == float((z0 - 1) % nz)


def _pair_worker(rank, world, port, nz, plane_shape, q):
    import torch
    import torch.distributed as dist

    import paper_2309_05331_b200 as rk
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        z0, nzl = rk.partition(nz, world, rank)
        # the slab's planes, every value tagged with the global z index (source: z, base: 1000 + z)
        src = torch.stack([torch.full(plane_shape, float(z0 + i), dtype=torch.float64) for i in range(nzl)])
        base = src + 1000.0
        g2 = torch.full((4,) + plane_shape, -1.0, dtype=torch.float64)   # [-2, -1 | nzl, nzl+1]
        g1 = torch.full((2,) + plane_shape, -1.0, dtype=torch.float64)   # [-1 | nzl]
        plan = rk.pair_ghost_plan(world, rank, True)
        reqs = []
        for m in plan["msgs"]:
            n = m["nplanes"]
            if m["recv"]:
                g = g2 if m["array"] == 0 else g1
                off = n if m["side"] else 0
                view = torch.empty((n,) + plane_shape, dtype=torch.float64)
                reqs.append((dist.irecv(view, src=m["peer"]), view, g, off))
            else:
                a = src if m["array"] == 0 else base
                view = (a[nzl - n:] if m["side"] else a[:n]).contiguous()
                reqs.append((dist.isend(view, dst=m["peer"]), None, None, None))
        for r, view, g, off in reqs:
            r.wait()
            if view is not None:
                g[off:off + view.shape[0]] = view
        q.put((rank, z0, nzl, [float(g2[i].mean()) for i in range(4)], [float(g1[i].mean()) for i in range(2)],
               [float(g2[i].std()) for i in range(4)]))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world,nz", [(2, 8), (2, 5), (3, 13), (4, 9), (4, 8)])
def test_pair_ghost_plan_gloo(world, nz):
    """The K8 pairs' ghost exchange (rk_pair_ghost_plan, posting order as on NCCL) executed with
    real point-to-point messages: every rank's 2-deep source ghosts and 1-deep base ghosts hold
    its periodic z-neighbours' boundary planes, also at world 2 where one peer is both."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pair_worker, args=(r, world, port, nz, (3, 5), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in sorted(res, key=lambda r: r[0]):
        assert len(r) > 2, r
        rank, z0, nzl, g2, g1, sd = r
        assert nzl >= 2
        assert g2 == [float((z0 - 2) % nz), float((z0 - 1) % nz), float((z0 + nzl) % nz), float((z0 + nzl + 1) % nz)]
        assert g1 == [1000.0 + (z0 - 1) % nz, 1000.0 + (z0 + nzl) % nz]
        assert max(sd) == 0.0
