"""Multi-GPU halo path over NCCL / NVLink (SURVEY §4 tests/dist): torchrun with G ranks, one
per GPU, G in {2, 4, 8} up to the visible GPUs; tests/dist_worker.py asserts bitwise equality
with the oracle's single-domain run for RK4 and error-controlled DOPRI5 (NCCL and P2P
transports, overlap on and off) and NaN propagation through the allreduce.  world = 1 runs the
same script through the one-GPU loopback exchange; larger worlds are skipped when fewer GPUs
are visible."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_multi_gpu_bitwise(world):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs, {_ngpus()} visible")
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(ROOT, "tests", "dist_worker.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "FAILURES: none" in r.stdout
