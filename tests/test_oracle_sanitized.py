"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer: oracle/rk_oracle.c
is rebuilt with -fsanitize=address,undefined into a temporary library and a workload over
every entry point (all schemes on a small periodic grid, adaptive runs with rejections,
Adams-Bashforth(-Moulton), the algebra ops, the controllers) runs in a subprocess with the
ASan runtime preloaded; any sanitizer report fails the test.  Results must also equal the
regular build's bit for bit (the sanitizers change no arithmetic)."""
import os
import shutil
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKLOAD = r'''
import hashlib, numpy as np, oracle, rk_inputs
h = hashlib.sha256()
p = oracle.gray_scott_problem(9, 7, 5)
u0 = rk_inputs.gray_scott_ic(9, 7, 5, seed=3) + 0.01 * rk_inputs.random_state(2 * 9 * 7 * 5, 4).reshape(5, 2, 7, 9)
for name, s in sorted(oracle.SCHEMES.items()):
    u = oracle.step(p, s, 0.0, 0.5, u0)
    h.update(np.ascontiguousarray(u).tobytes())
for s in (oracle.CASH_KARP54, oracle.DOPRI5, oracle.RKF78):
    u, acc, rej, rc = oracle.integrate_adaptive(oracle.logistic_problem(101), s, rk_inputs.logistic_u0(101), -5.0, 5.0, 3.0, 1e-9, 1e-9)
    h.update(np.ascontiguousarray(u).tobytes()); h.update(bytes([acc % 256, rej % 256, rc % 256]))
    u, acc, rej, rc = oracle.integrate_adaptive(p, s, u0, 0.0, 4.0, 2.0, 1e-7, 1e-7)
    h.update(np.ascontiguousarray(u).tobytes())
u, n = oracle.integrate_const(oracle.exp_problem(33, -1.0), oracle.RK4, rk_inputs.exp_decay_u0(33), 0.0, 1.0, 0.1)
h.update(np.ascontiguousarray(u).tobytes())
for k in (1, 3, 8):
    u = oracle.ab_integrate(oracle.logistic_problem(17), k, rk_inputs.logistic_u0(17), -5.0, 0.05, 12)
    h.update(np.ascontiguousarray(u).tobytes())
    u = oracle.abm_integrate(oracle.logistic_problem(17), k, rk_inputs.logistic_u0(17), -5.0, 0.05, 12)
    h.update(np.ascontiguousarray(u).tobytes())
x = rk_inputs.random_state(1000, 9)
h.update(np.ascontiguousarray(oracle.lincomb([0.5, -2.0, 3.0], [x, x * 2, x * 3])).tobytes())
h.update(repr(oracle.norm_inf(x)).encode())
h.update(repr(oracle.controller(1.7, 0.3)).encode() + repr(oracle.controller(0.01, 0.3)).encode())
print("DIGEST", h.hexdigest())
'''


def _run(env):
    r = subprocess.run([sys.executable, "-c", WORKLOAD], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    return r


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_oracle_asan_ubsan():
    libasan = subprocess.run(["gcc", "-print-file-name=libasan.so"], capture_output=True, text=True).stdout.strip()
    if not os.path.isabs(libasan) or not os.path.exists(libasan):
        pytest.skip("libasan not available")
    tmp = tempfile.mkdtemp(prefix="oracle_asan_")
    lib = os.path.join(tmp, "liboracle.so")
    b = subprocess.run(["gcc", "-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
                        "-fno-sanitize-recover=undefined", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                        "-std=c11", os.path.join(ROOT, "oracle", "rk_oracle.c"), "-o", lib, "-lquadmath", "-lm"],
                       capture_output=True, text=True)
    assert b.returncode == 0, b.stderr
    base = dict(os.environ, PYTHONPATH=ROOT)
    ref = _run(base)
    assert ref.returncode == 0, ref.stderr[-2000:]
    env = dict(base, ORACLE_LIB=lib, LD_PRELOAD=libasan,
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=0:halt_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    r = _run(env)
    assert r.returncode == 0, r.stderr[-4000:]
    assert "AddressSanitizer" not in r.stderr and "runtime error" not in r.stderr, r.stderr[-4000:]
    assert ref.stdout.split()[-1] == r.stdout.split()[-1]  # same bits with the sanitized build
