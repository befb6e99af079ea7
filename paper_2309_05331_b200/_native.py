"""ctypes declarations of librkb200.so (include/rk_b200.h).  Argument marshalling only.

There is no fallback: if the shared library is missing or fails to load, importing the
package's compute API raises.  Build it with ``python -m paper_2309_05331_b200.build``.
"""
from __future__ import annotations

import ctypes
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librkb200.so")

RK_OK = 0
STATUS = {0: "RK_OK", 1: "RK_ERR_ARG", 2: "RK_ERR_CONTRACT", 3: "RK_ERR_UNSUPPORTED",
          4: "RK_ERR_STATE", 5: "RK_ERR_DIVERGED", 6: "RK_ERR_DT_UNDERFLOW", 7: "RK_ERR_STALL",
          8: "RK_ERR_CUDA", 9: "RK_ERR_NCCL", 10: "RK_ERR_OOM"}
OPT_HALO_OVERLAP, OPT_HALO_LOOPBACK, OPT_MAX_TRIES, OPT_TIMING, OPT_USE_GRAPH, OPT_DEVICE_LOOP, OPT_HALO_P2P = 1, 2, 3, 4, 5, 6, 7
OPT_CONTROLLER, OPT_CHECK_FINITE, OPT_COOP_MAX_CELLS = 8, 9, 10
OPT_FUSED_STEP, OPT_COMM_TIMEOUT_MS, OPT_ERROR_SPIKE, OPT_CHECK_ARGS, OPT_FUSED_KERNELS = 11, 12, 13, 14, 15
CTRL_ODEINT, CTRL_SPEC = 0, 1
ABI_VERSION = 5
UNIQUE_ID_BYTES = 128


class RKError(RuntimeError):
    def __init__(self, code: int, func: str, msg: str):
        self.code = code
        self.status = STATUS.get(code, str(code))
        super().__init__(f"{func} -> {self.status}: {msg}")


class Stats(ctypes.Structure):
    _fields_ = [("rhs_evals", ctypes.c_int64), ("steps", ctypes.c_int64), ("tries", ctypes.c_int64),
                ("accepted", ctypes.c_int64), ("rejected", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("halo_exchanges", ctypes.c_int64),
                ("halo_bytes", ctypes.c_int64), ("stage_launches", ctypes.c_int64),
                ("stage_kernel_ms", ctypes.c_double), ("halo_ms", ctypes.c_double),
                ("last_err_ratio", ctypes.c_double), ("last_dt", ctypes.c_double),
                ("stage_bytes", ctypes.c_int64), ("diverged_t", ctypes.c_double),
                ("pair_launches", ctypes.c_int64), ("pair_kernel_ms", ctypes.c_double),
                ("pair_bytes", ctypes.c_int64), ("head_launches", ctypes.c_int64),
                ("head_kernel_ms", ctypes.c_double), ("head_bytes", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class HaloMsg(ctypes.Structure):
    _fields_ = [("recv", ctypes.c_int), ("peer", ctypes.c_int), ("slot", ctypes.c_int),
                ("nplanes", ctypes.c_int)]


class HaloPlan(ctypes.Structure):
    _fields_ = [("up", ctypes.c_int), ("down", ctypes.c_int), ("nmsg", ctypes.c_int),
                ("msg", HaloMsg * 4)]


class PairMsg(ctypes.Structure):
    _fields_ = [("recv", ctypes.c_int), ("peer", ctypes.c_int), ("array", ctypes.c_int), ("side", ctypes.c_int),
                ("nplanes", ctypes.c_int)]


class PairPlan(ctypes.Structure):
    _fields_ = [("up", ctypes.c_int), ("down", ctypes.c_int), ("nmsg", ctypes.c_int), ("msg", PairMsg * 8)]


_v, _p, _i, _i64, _d = ctypes.c_void_p, ctypes.POINTER, ctypes.c_int, ctypes.c_int64, ctypes.c_double
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_ip = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); every function declared in include/rk_b200.h
SIGNATURES = {
    "rk_abi_version": (_i, []),
    "rk_last_error": (ctypes.c_char_p, []),
    "rk_partition": (_i, [_i64, _i, _i, _i64p, _i64p]),
    "rk_tableau": (_i, [_i, _dp, _dp, _dp, _dp, _ip, _ip, _ip]),
    "rk_controller": (_i, [_i, _d, _dp, _ip]),
    "rk_step_adjust": (_i, [_i, _i, _d, _dp, _ip]),
    "rk_halo_plan_get": (_i, [_i, _i, _p(HaloPlan)]),
    "rk_pair_ghost_plan": (_i, [_i, _i, _i, _p(PairPlan)]),
    "rk_nccl_unique_id": (_i, [_v]),
    "rk_ctx_create": (_i, [_i, _i, _i, _v, _v, _p(_v)]),
    "rk_ctx_destroy": (_i, [_v]),
    "rk_ctx_set_allocator": (_i, [_v, _v, _v, _v]),
    "rk_state_create_grid": (_i, [_v, _i64, _i64, _i64, _i, _p(_v)]),
    "rk_state_create_vector": (_i, [_v, _i64, _i, _p(_v)]),
    "rk_state_destroy": (_i, [_v]),
    "rk_state_local_range": (_i, [_v, _i64p, _i64p]),
    "rk_state_local_size": (_i, [_v, _i64p]),
    "rk_state_set": (_i, [_v, _v, _i]),
    "rk_state_get": (_i, [_v, _v, _i]),
    "rk_set_rhs_exponential": (_i, [_v, _d]),
    "rk_set_rhs_logistic": (_i, [_v]),
    "rk_set_rhs_gray_scott": (_i, [_v, _d, _d, _d, _d, _d]),
    "rk_set_option": (_i, [_v, _i, _i64]),
    "rk_do_step": (_i, [_v, _i, _d, _d]),
    "rk_try_step": (_i, [_v, _i, _d, _d, _d, _d, _ip, _dp, _dp]),
    "rk_integrate_const": (_i, [_v, _i, _d, _d, _d, _i64p]),
    "rk_integrate_adaptive": (_i, [_v, _i, _d, _d, _d, _d, _d, _i64p, _i64p]),
    "rk_lincomb": (_i, [_v, _i, _dp, _p(_v)]),
    "rk_norm_inf": (_i, [_v, _dp]),
    "rk_eval_rhs": (_i, [_v, _v]),
    "rk_p2p_export": (_i, [_v, _v, _i64, _i64p]),
    "rk_p2p_import": (_i, [_v, _v, _i64]),
    "rk_get_stats": (_i, [_v, _p(Stats)]),
    "rk_reset_stats": (_i, [_v]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load librkb200.so (in-tree).  Raises if it is missing: no CPU fallback exists."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2309_05331_b200.build` "
                              "(there is no CPU fallback for the CUDA path)")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.rk_abi_version() != ABI_VERSION:
            raise ImportError("librkb200.so ABI version mismatch")
        _lib = L
    return _lib


def check(code: int, func: str) -> None:
    if code != RK_OK:
        raise RKError(code, func, lib().rk_last_error().decode(errors="replace"))


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
