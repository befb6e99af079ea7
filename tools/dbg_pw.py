"""Time the pointwise DOPRI5 try kernel (host loop) and the device-loop kernel on configs[1]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2309_05331_b200 as rk
import rk_inputs

c = rk.Context(0, 1, 0)
n = 1000000
v = c.vector(n)
v.set_rhs_logistic()
u0 = rk_inputs.logistic_u0(n)
for dl in (0, 1, 0, 1):
    v.set_option(rk.OPT_DEVICE_LOOP, dl)
    v.set(u0)
    v.reset_stats()
    t = time.perf_counter()
    a, r = v.integrate_adaptive("dopri5", -5.0, 5.0, 0.1, 1e-8, 1e-8)
    dtm = time.perf_counter() - t
    print("device_loop", dl, a, r, "%.3f ms" % (dtm * 1e3), "%.1f us/try" % (dtm * 1e6 / (a + r)))
for k in range(3):
    v.set(u0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(100):
        v.try_step("dopri5", -5.0, 0.01, 1e-8, 1e-8)
    print("try_step x100: %.1f us/try" % ((time.perf_counter() - t) * 1e4))
    t = time.perf_counter()
    v.integrate_const("dopri5", 0.0, 1.0, 0.01)
    torch.cuda.synchronize()
    print("integrate_const 100 steps in registers: %.1f us/step" % ((time.perf_counter() - t) * 1e4))
