import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (launched via torchrun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    """The tests load the in-tree CUDA library; build it (nvcc cross-compiles without a GPU)
    if this checkout has none yet.  An existing library is used as is."""
    lib = os.path.join(ROOT, "paper_2410_06511_b200", "libfsdp_b200.so")
    if not os.path.exists(lib):
        import subprocess
        subprocess.run([sys.executable, os.path.join(ROOT, "paper_2410_06511_b200", "build.py")], check=False,
                       timeout=1800)
