"""The P2P transport across PROCESSES on one GPU (tests/shared_gpu_worker.py): world 2 (one
peer is both z-neighbours) and world 3 (distinct neighbours, ragged slabs), no NCCL -- the
halo stores, the ready/ack flag handshake and the allreduce(max) atomics cross process
boundaries through CUDA IPC mappings exactly as they cross GPUs on an 8-GPU box."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_transport_across_processes(world):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(ROOT, "tests", "shared_gpu_worker.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "FAILURES: none" in r.stdout, r.stdout[-3000:]
    info = json.loads(r.stdout.split("INFO:", 1)[1].splitlines()[0])
    assert info["halo_exchanges"] > 0 and info["ms_per_exchange"] > 0
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"shared_gpu_w{world}.json"), "w") as f:
        json.dump(info, f)
