"""Unfused ("native") Runge–Kutta stepping — the ablation of SURVEY.md f4.

The paper compares Odeint's RK4 (stages computed on the fly inside the algebra) with OpenFPM's
hand-written "native" RK4, which evaluates each stage into its own array (P:L253, P:L255,
P:L271).  The GPU analogue is the library's RK_OPT_FUSED_KERNELS = 0 mode: per stage one
lincomb launch writes Y_i and one RHS launch k_i = F(Y_i), then the final combination (and,
under error control, the error estimate and the ratio max) -- every intermediate through HBM,
against the fused stage kernels of the default mode.  Both evaluate R-17's sums in the same
order, so the two paths are bitwise identical; only the traffic differs.  All
arithmetic runs in the library's kernels; this module only sets the option and calls do_step.
"""
from . import _native, api


class NativeRK4:
    """Unfused RK4 steps on `st` (RK_OPT_FUSED_KERNELS = 0 while this object is open)."""

    def __init__(self, st: "api.State"):
        self.st = st
        st.set_option(_native.OPT_FUSED_KERNELS, 0)

    def step(self, dt: float) -> None:
        """u <- u + dt*(k1/6 + k2/3 + k3/3 + k4/6): 4 RHS + 4 lincomb launches (the RHS is
        autonomous, so the time argument is immaterial)."""
        self.st.do_step("rk4", 0.0, dt)

    def close(self) -> None:
        if self.st is not None and getattr(self.st, "_h", None):
            self.st.set_option(_native.OPT_FUSED_KERNELS, 1)
        self.st = None
