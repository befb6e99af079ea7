"""Unfused ("native") RK4 built from the library's separate ops — the ablation of SURVEY.md f4.

The paper compares Odeint's RK4 (stages computed on the fly inside the algebra) with OpenFPM's
hand-written "native" RK4, which evaluates each stage into its own array (P:L253, P:L255,
P:L271).  The GPU analogue: one rk_eval_rhs launch per stage plus one rk_lincomb launch per
stage value and for the final combination, every intermediate going through HBM, against the
fused stage kernels of rk_do_step.  Both orders of operations are R-17's, so the two paths are
bitwise identical; only the traffic differs.  All arithmetic runs in the
library's kernels; this module only sequences C-ABI calls.
"""
from . import api


class NativeRK4:
    """Work arrays for unfused RK4 on states shaped like `st` (k1..k4 and the stage value Y)."""

    def __init__(self, st: "api.State"):
        self.st = st
        mk = (lambda: st.ctx.grid(*st.dims, st.ncomp)) if st.grid else (lambda: st.ctx.vector(st.dims[0], st.ncomp))
        self.k = [mk() for _ in range(4)]
        self.y = mk()
        self.y.copy_rhs_from(st)
        tab = api.tableau("rk4")
        self.a = tab["a"]
        self.b = tab["b"]

    def step(self, dt: float) -> None:
        """u <- u + dt*(k1/6 + k2/3 + k3/3 + k4/6), one launch per op (4 RHS + 4 lincomb)."""
        u, k, y, a = self.st, self.k, self.y, self.a
        u.eval_rhs(k[0])                                  # k1 = F(u)
        for i in range(1, 4):
            y.lincomb([1.0, dt * a[i][i - 1]], [u, k[i - 1]])  # Y_i = u + (dt a_i,i-1) k_{i-1}
            y.eval_rhs(k[i])                              # k_i = F(Y_i)
        u.lincomb([1.0] + [dt * bj for bj in self.b], [u] + k)  # u + sum (dt b_j) k_j

    def close(self) -> None:
        for s in self.k + [self.y]:
            s.close()
