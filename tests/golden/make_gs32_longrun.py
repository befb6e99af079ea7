"""Writes gs32_rk4_20000.json: the fp64 oracle (only oracle/ and the shared seeded inputs) on
Gray–Scott 32^3 (R-1..R-6 parameters, IC seed 42), classic RK4, dt = 1, t in
[0, 20000] -- the run length of SPEC.md acceptance criterion 5.  Records the SHA-256
of the final state's bytes ([z][c][y][x] little-endian fp64), per-component min / max and the
variance of C1 at t = 0 and t = 20000.  With this IC the perturbation decays to the (1, 0)
steady state and C1 ends in fp64 denormals, so the GPU test built on it pins 20000 steps of
bitwise arithmetic including denormals (no flush-to-zero, R-17).  The oracle takes
~6 minutes (denormal arithmetic is slow on the CPU).  Run: python tests/golden/make_gs32_longrun.py"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import rk_inputs  # noqa: E402

n, steps = 32, 20000
u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
t = time.time()
u, k = oracle.integrate_const(oracle.gray_scott_problem(n, n, n), oracle.RK4, u0, 0.0, float(steps), 1.0)
sec = time.time() - t
assert k == steps
u = np.ascontiguousarray(u, dtype="<f8")
out = {
    "source": "oracle.integrate_const(gray_scott_problem(32,32,32), RK4, gray_scott_ic(32,32,32,seed=42), 0, 20000, 1)",
    "cite": "SPEC.md acceptance criterion 5 (S:L515); parameters DESIGN.md R-1..R-6",
    "steps": steps,
    "sha256_final": hashlib.sha256(u.tobytes()).hexdigest(),
    "c0_min": float(u[:, 0].min()), "c0_max": float(u[:, 0].max()),
    "c1_min": float(u[:, 1].min()), "c1_max": float(u[:, 1].max()),
    "c1_var_initial": float(u0[:, 1].var()), "c1_var_final": float(u[:, 1].var()),
    "oracle_seconds": round(sec, 1),
}
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gs32_rk4_20000.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
