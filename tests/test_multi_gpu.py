"""Multi-GPU ghost exchange over NCCL (one process per GPU via torchrun):
N-rank results bitwise equal to the single-GPU run and within tolerance of the
oracle, with and without the boundary-first overlap.  Needs >= 2 GPUs."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


_PORT_BUSY = ("Address already in use", "EADDRINUSE", "failed to listen", "address in use")


def _torchrun(n, script, *args, timeout=600):
    """torchrun on 127.0.0.1 with a free port; a port taken between the probe and
    the rendezvous (another process, NCCL's bootstrap sockets) is retried."""
    for attempt in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()),
               os.path.join(ROOT, "tests", script), *args]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
        busy = r.returncode != 0 and any(m in r.stdout + r.stderr for m in _PORT_BUSY)
        if not busy:
            break
    print(r.stdout[-6000:], r.stderr[-6000:])
    return r


@pytest.mark.parametrize("n", [2, 4])
def test_nccl_exchange_matches_single_gpu(n):
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "mgpu_worker.py").returncode == 0


@pytest.mark.parametrize("n,config", [(2, "weak"), (4, "weak"), (2, "strong"), (2, "patchy"), (2, "aa"),
                                      (4, "patchy")])
def test_full_size_bitwise_vs_one_gpu(n, config):
    """BASELINE weak-scaling config (384^3 fp64 per GPU) and strong-scaling config
    (768^3 in 8 patches of 384^3) at full size, 10 steps: N-GPU samples across
    every process cut equal the one-GPU run bitwise (tests/mgpu_fullsize_worker.py)."""
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "mgpu_fullsize_worker.py", config, timeout=900).returncode == 0


def test_peer_timeout_reports_error():
    """A peer that stops stepping makes the fused exchange report an error
    (LBM_ERR_INTERNAL from lbm_step after LBM_PEER_TIMEOUT_S) -- never a hang."""
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    assert _torchrun(2, "mgpu_timeout_worker.py", timeout=300).returncode == 0
