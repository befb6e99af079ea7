"""paper_2309_05331_b200 — B200-native explicit Runge–Kutta time stepping of a
block-distributed fp64 state (the hot path of arxiv 2309.05331, OpenFPM + Odeint).

The compute path is librkb200.so (hand-written sm_100a CUDA behind the C-ABI in
include/rk_b200.h); this package is its thin ctypes binding.  There is no CPU fallback.
"""
from .api import (CASH_KARP54, DOPRI5, EULER, EXPLICIT_MIDPOINT, FEHLBERG78, MIDPOINT, MODIFIED_MIDPOINT,
                  RK4, SCHEMES, Context, State, controller, halo_plan, pair_ghost_plan, partition, tableau)
from ._native import (CTRL_ODEINT, CTRL_SPEC, OPT_CHECK_FINITE, OPT_CONTROLLER, OPT_COOP_MAX_CELLS,
                      OPT_FUSED_STEP, OPT_COMM_TIMEOUT_MS, OPT_ERROR_SPIKE, OPT_CHECK_ARGS, OPT_FUSED_KERNELS,
                      OPT_DEVICE_LOOP,
                      OPT_HALO_LOOPBACK, OPT_HALO_OVERLAP, OPT_HALO_P2P, OPT_MAX_TRIES, OPT_TIMING,
                      OPT_USE_GRAPH, RKError, lib)

__all__ = ["Context", "State", "EULER", "RK4", "CASH_KARP54", "DOPRI5", "FEHLBERG78", "MIDPOINT",
           "EXPLICIT_MIDPOINT", "MODIFIED_MIDPOINT", "SCHEMES", "RKError",
           "partition", "tableau", "controller", "halo_plan", "pair_ghost_plan", "lib", "OPT_HALO_OVERLAP", "OPT_HALO_LOOPBACK",
           "OPT_MAX_TRIES", "OPT_TIMING", "OPT_USE_GRAPH", "OPT_DEVICE_LOOP", "OPT_HALO_P2P",
           "OPT_CONTROLLER", "OPT_CHECK_FINITE", "OPT_COOP_MAX_CELLS", "OPT_FUSED_STEP", "OPT_COMM_TIMEOUT_MS", "OPT_ERROR_SPIKE", "OPT_CHECK_ARGS", "OPT_FUSED_KERNELS", "CTRL_ODEINT", "CTRL_SPEC"]
