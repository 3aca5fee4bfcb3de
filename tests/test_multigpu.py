"""Multi-GPU parity (W = 2, 4, 8 over NCCL/NVLink): launches tests/mgpu_worker.py under
torchrun on all visible GPUs (and on 2 when more are visible).  Skipped with < 2 GPUs."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _counts():
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    return sorted({c for c in (2, n) if 2 <= c <= n})


@pytest.mark.parametrize("nproc", _counts() or [2])
def test_mgpu_worker(nproc):
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mgpu_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert out.count("OK") >= nproc, out[-2000:]
