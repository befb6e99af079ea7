"""Thin Python API over librkb200.so (include/rk_b200.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; PyTorch supplies the
CUDA stream, device tensors for set/get, and the process group that broadcasts the NCCL
unique id.  Names follow the C-ABI (and the paper's Odeint vocabulary: do_step,
integrate_const, integrate_adaptive).
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _native
from ._native import Stats, call

EULER, RK4, CASH_KARP54, DOPRI5, FEHLBERG78, MIDPOINT, MODIFIED_MIDPOINT = 0, 1, 2, 3, 4, 5, 6
EXPLICIT_MIDPOINT = MIDPOINT
SCHEMES = {"euler": EULER, "rk4": RK4, "cash_karp54": CASH_KARP54, "dopri5": DOPRI5,
           "rkf78": FEHLBERG78, "midpoint": MIDPOINT, "explicit_midpoint": MIDPOINT,
           "modified_midpoint": MODIFIED_MIDPOINT}
SCHEMES.update({f"ab{k}": 10 + k for k in range(1, 9)})  # Adams–Bashforth k (rk_b200.h)
SCHEMES.update({f"abm{k}": 20 + k for k in range(1, 9)})  # Adams–Bashforth–Moulton k (PECE)


def _scheme(s) -> int:
    return SCHEMES[s] if isinstance(s, str) else int(s)


def _stream_handle(stream) -> int | None:
    """None -> the library creates its own stream; a torch stream (or raw handle) is used
    as is; torch's default stream (handle 0) maps to cudaStreamLegacy (0x1), since a NULL
    handle means "create one" in rk_ctx_create."""
    if stream is None:
        return None
    h = stream if isinstance(stream, int) else int(stream.cuda_stream)
    return h if h != 0 else 1


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


def _torch_allocator(device: int):
    """ctypes callbacks routing the library's state arrays through torch's caching allocator
    (plumbing only: the library still owns what it computes)."""
    import torch

    def alloc(nbytes, stream, _user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device, stream or 0)
        except Exception:  # noqa: BLE001  (an exception must not cross the C ABI: NULL = OOM)
            return None

    def free(ptr, _stream, _user):
        torch.cuda.caching_allocator_delete(ptr)

    return _ALLOC_FN(alloc), _FREE_FN(free)


def _order_after_torch(t) -> None:
    """The library copies on the ctx stream, which need not be torch's current stream: let the
    torch work already queued on `t` (writes before set, reads before get) finish first."""
    if t.is_cuda:
        import torch
        torch.cuda.current_stream(t.device).synchronize()


def broadcast_unique_id(group=None, device: int | None = None) -> bytes:
    """Rank 0 creates the NCCL unique id (rk_nccl_unique_id); every rank of the torch process
    group receives the same 128 bytes (plumbing for rk_ctx_create, world > 1)."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(_native.UNIQUE_ID_BYTES, dtype=torch.uint8)
    if dist.get_rank(group) == 0:
        t[:] = torch.frombuffer(bytearray(Context.nccl_unique_id()), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda(device)
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().numpy().tobytes())


class Context:
    """One per rank (one process per device).  world > 1 with NCCL needs the NCCL
    unique id, which ``Context.from_torch_distributed`` broadcasts over the torch process group;
    world > 1 without one is a P2P-only context (rk_ctx_create): every state exchanges its CUDA
    IPC handles over ``p2p_group`` (a torch process group, e.g. gloo) when it is created."""

    def __init__(self, rank: int = 0, world: int = 1, device: int = 0, stream=None,
                 unique_id: bytes | None = None, p2p_group=None, allocator: str | None = None):
        L = _native.lib()
        h = ctypes.c_void_p()
        uid = None
        if world > 1 and unique_id is not None:
            if len(unique_id) != _native.UNIQUE_ID_BYTES:
                raise ValueError("the NCCL unique id has 128 bytes")
            uid = ctypes.create_string_buffer(bytes(unique_id), _native.UNIQUE_ID_BYTES)
        elif world > 1 and p2p_group is None:
            raise ValueError("world > 1 needs the NCCL unique id or a process group for the P2P handles")
        self._p2p_group = p2p_group if uid is None and world > 1 else None
        sh = _stream_handle(stream)
        call("rk_ctx_create", rank, world, device, uid, ctypes.c_void_p(sh) if sh else None,
             ctypes.byref(h))
        self._h = h
        self._L = L
        self._states = weakref.WeakSet()
        self.rank, self.world, self.device = rank, world, device
        self._alloc_cbs = None
        if allocator == "torch":  # state arrays from torch's caching allocator (rk_ctx_set_allocator)
            self._alloc_cbs = _torch_allocator(device)
            call("rk_ctx_set_allocator", h, ctypes.cast(self._alloc_cbs[0], ctypes.c_void_p),
                 ctypes.cast(self._alloc_cbs[1], ctypes.c_void_p), None)
        elif allocator is not None:
            raise ValueError("allocator: None (cudaMalloc) or 'torch'")

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(_native.UNIQUE_ID_BYTES)
        call("rk_nccl_unique_id", buf)
        return buf.raw

    @classmethod
    def from_torch_distributed(cls, device: int, stream=None, group=None, transport: str = "nccl") -> "Context":
        """transport "nccl": NCCL communicator (unique id broadcast over `group`); "p2p": no NCCL,
        every state's IPC handles are all-gathered over `group` (works for several ranks on
        one GPU, which NCCL refuses)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if transport == "p2p" and world > 1:
            return cls(rank, world, device, stream, None, p2p_group=group if group is not None else dist.group.WORLD)
        uid = broadcast_unique_id(group, device) if world > 1 else None
        return cls(rank, world, device, stream, uid)

    def _connect(self, st: "State") -> "State":
        if self._p2p_group is not None:  # P2P-only context: exchange the IPC handles (collective)
            st.p2p_connect(self._p2p_group)
        return st

    def grid(self, nx: int, ny: int, nz: int, ncomp: int = 2) -> "State":
        h = ctypes.c_void_p()
        call("rk_state_create_grid", self._h, nx, ny, nz, ncomp, ctypes.byref(h))
        st = State(self, h, grid=True, dims=(nx, ny, nz), ncomp=ncomp)
        self._states.add(st)
        return self._connect(st)

    def vector(self, n: int, ncomp: int = 1) -> "State":
        h = ctypes.c_void_p()
        call("rk_state_create_vector", self._h, n, ncomp, ctypes.byref(h))
        st = State(self, h, grid=False, dims=(n,), ncomp=ncomp)
        self._states.add(st)
        return self._connect(st)

    def close(self):
        if getattr(self, "_h", None):
            for st in list(self._states):  # states first: they live on this ctx
                st.close()
            self._L.rk_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class State:
    """A distributed state: z-slab grid [z][c][y][x] or block vector [c][i] (rk_b200.h)."""

    def __init__(self, ctx: Context, h, grid: bool, dims, ncomp: int):
        self.ctx, self._h, self.grid, self.dims, self.ncomp = ctx, h, grid, dims, ncomp
        self._rhs = None  # (setter name, args) of the last set_rhs_* call
        b, c, n = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        call("rk_state_local_range", h, ctypes.byref(b), ctypes.byref(c))
        call("rk_state_local_size", h, ctypes.byref(n))
        self.begin, self.local, self.size = b.value, c.value, n.value

    @property
    def local_shape(self) -> tuple:
        if self.grid:
            nx, ny, _ = self.dims
            return (self.local, self.ncomp, ny, nx)
        return (self.ncomp, self.local)

    # ---- data movement -------------------------------------------------------------
    def set(self, src) -> None:
        """src: numpy array (host) or torch tensor (host or on this device), fp64."""
        if hasattr(src, "data_ptr"):  # torch
            assert src.dtype.__repr__() == "torch.float64" and src.is_contiguous()
            assert src.numel() == self.size
            _order_after_torch(src)
            call("rk_state_set", self._h, ctypes.c_void_p(src.data_ptr()), 1 if src.is_cuda else 0)
        else:
            a = np.ascontiguousarray(src, dtype=np.float64)
            assert a.size == self.size, (a.size, self.size)
            call("rk_state_set", self._h, a.ctypes.data_as(ctypes.c_void_p), 0)

    def get(self, out=None):
        """Returns a numpy array of local_shape, or fills `out` (numpy / torch)."""
        if out is None:
            out = np.empty(self.local_shape, dtype=np.float64)
        if hasattr(out, "data_ptr"):
            assert out.numel() == self.size and out.is_contiguous()
            _order_after_torch(out)
            call("rk_state_get", self._h, ctypes.c_void_p(out.data_ptr()), 1 if out.is_cuda else 0)
        else:
            assert out.size == self.size and out.flags.c_contiguous and out.dtype == np.float64
            call("rk_state_get", self._h, out.ctypes.data_as(ctypes.c_void_p), 0)
        return out

    # ---- RHS / options -------------------------------------------------------------
    def set_rhs_exponential(self, lam: float) -> None:
        call("rk_set_rhs_exponential", self._h, lam)
        self._rhs = ("set_rhs_exponential", (lam,))

    def set_rhs_logistic(self) -> None:
        call("rk_set_rhs_logistic", self._h)
        self._rhs = ("set_rhs_logistic", ())

    def set_rhs_gray_scott(self, d1=2e-4, d2=1e-4, F=0.014, K=0.053, h=2.5 / 64) -> None:
        call("rk_set_rhs_gray_scott", self._h, d1, d2, F, K, h)
        self._rhs = ("set_rhs_gray_scott", (d1, d2, F, K, h))

    def copy_rhs_from(self, other: "State") -> None:
        """Give this state the right-hand side last set on `other`."""
        if other._rhs is not None:
            getattr(self, other._rhs[0])(*other._rhs[1])

    def set_option(self, key: int, value: int) -> None:
        call("rk_set_option", self._h, key, value)

    # ---- stepping ------------------------------------------------------------------
    def do_step(self, scheme, t: float, dt: float) -> None:
        call("rk_do_step", self._h, _scheme(scheme), t, dt)

    def try_step(self, scheme, t: float, dt: float, atol: float, rtol: float):
        """Returns (accepted, err_ratio, dt_next)."""
        a, e, d = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        call("rk_try_step", self._h, _scheme(scheme), t, dt, atol, rtol, ctypes.byref(a),
             ctypes.byref(e), ctypes.byref(d))
        return bool(a.value), e.value, d.value

    def integrate_const(self, scheme, t0: float, t1: float, dt: float) -> int:
        n = ctypes.c_int64()
        call("rk_integrate_const", self._h, _scheme(scheme), t0, t1, dt, ctypes.byref(n))
        return n.value

    def integrate_adaptive(self, scheme, t0, t1, dt0, atol, rtol):
        """Returns (accepted, rejected)."""
        a, r = ctypes.c_int64(), ctypes.c_int64()
        call("rk_integrate_adaptive", self._h, _scheme(scheme), t0, t1, dt0, atol, rtol,
             ctypes.byref(a), ctypes.byref(r))
        return a.value, r.value

    def p2p_connect(self, group=None) -> None:
        """P2P transport without NCCL: all-gather this state's CUDA IPC handles over the torch
        process group and map the peers (rk_p2p_export / rk_p2p_import; collective)."""
        import torch.distributed as dist
        n = ctypes.c_int64()
        call("rk_p2p_export", self._h, None, 0, ctypes.byref(n))
        buf = ctypes.create_string_buffer(n.value)
        call("rk_p2p_export", self._h, buf, n.value, ctypes.byref(n))
        parts = [None] * dist.get_world_size(group)
        dist.all_gather_object(parts, buf.raw[:n.value], group=group)
        blob = b"".join(parts)
        call("rk_p2p_import", self._h, ctypes.create_string_buffer(blob, len(blob)), n.value)

    # ---- algebra -------------------------------------------------------------------
    def lincomb(self, coef, states) -> None:
        """self = sum_j coef[j] * states[j] (1 <= k <= 14)."""
        k = len(states)
        c = (ctypes.c_double * max(k, 1))(*coef)
        hs = (ctypes.c_void_p * max(k, 1))(*[s._h for s in states])
        call("rk_lincomb", self._h, k, c, hs)

    def eval_rhs(self, out: "State") -> None:
        """out = F(self) with self's right-hand side (rk_eval_rhs)."""
        call("rk_eval_rhs", self._h, out._h)

    def norm_inf(self) -> float:
        d = ctypes.c_double()
        call("rk_norm_inf", self._h, ctypes.byref(d))
        return d.value

    def stats(self) -> dict:
        s = Stats()
        call("rk_get_stats", self._h, ctypes.byref(s))
        return s.as_dict()

    def reset_stats(self) -> None:
        call("rk_reset_stats", self._h)

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().rk_state_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- host-only helpers (no GPU) ------------------------------------------------------
def partition(n_global: int, world: int, rank: int) -> tuple[int, int]:
    b, c = ctypes.c_int64(), ctypes.c_int64()
    call("rk_partition", n_global, world, rank, ctypes.byref(b), ctypes.byref(c))
    return b.value, c.value


def tableau(scheme) -> dict:
    S = 13
    a, b, e, c = (ctypes.c_double * (S * S))(), (ctypes.c_double * S)(), (ctypes.c_double * S)(), \
        (ctypes.c_double * S)()
    s, o, eo = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    call("rk_tableau", _scheme(scheme), a, b, e, c, ctypes.byref(s), ctypes.byref(o), ctypes.byref(eo))
    n = s.value
    return {"s": n, "a": [[a[i * n + j] for j in range(n)] for i in range(n)], "b": list(b[:n]),
            "e": list(e[:n]), "c": list(c[:n]), "order": o.value, "err_order": eo.value}


def halo_plan(world: int, rank: int) -> dict:
    """The library's per-stage halo exchange plan for `rank` (rk_halo_plan_get)."""
    p = _native.HaloPlan()
    call("rk_halo_plan_get", world, rank, ctypes.byref(p))
    return {"up": p.up, "down": p.down,
            "msgs": [{"recv": bool(m.recv), "peer": m.peer, "slot": m.slot, "nplanes": m.nplanes}
                     for m in p.msg[:p.nmsg]]}


def pair_ghost_plan(world: int, rank: int, with_base: bool) -> dict:
    """The ghost exchange of a K8 stage pair on the multi-GPU slab (rk_pair_ghost_plan)."""
    p = _native.PairPlan()
    call("rk_pair_ghost_plan", world, rank, 1 if with_base else 0, ctypes.byref(p))
    return {"up": p.up, "down": p.down,
            "msgs": [{"recv": bool(m.recv), "peer": m.peer, "array": m.array, "side": m.side,
                      "nplanes": m.nplanes} for m in p.msg[:p.nmsg]]}


def controller(scheme, E: float, dt: float, kind: int = 0):
    """Library's host step adjuster (kind 0: Odeint R-12, 1: SPEC R-28): (accepted, dt_next)."""
    d, a = ctypes.c_double(dt), ctypes.c_int()
    if kind == 0:
        call("rk_controller", _scheme(scheme), E, ctypes.byref(d), ctypes.byref(a))
    else:
        call("rk_step_adjust", _scheme(scheme), kind, E, ctypes.byref(d), ctypes.byref(a))
    return bool(a.value), d.value
