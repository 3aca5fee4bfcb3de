"""Cross-process P2P parity on one GPU: tests/hostcoll_worker.py under torchrun with N
processes sharing cuda:0 (host-collective mesh, no NCCL; see the worker's docstring).  This
is the multi-process protocol of the default W > 1 path — CUDA IPC symmetric buffers,
device-epoch handshakes between processes, push / pull / store kernels on other processes'
buffers, HSDP's world reduce-scatter, graph replays, the handshake timeout — run where only
one GPU is available (the NVLink link itself is covered by tests/test_multigpu.py)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_hostcoll_worker_one_gpu(nproc):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "hostcoll_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT, env=env)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert out.count("hostcoll OK") == nproc, out[-2000:]
