"""Builds libfsdp_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; no fast math, IEEE
division, no flush-to-zero (bit-exact casts and the ÷W pre-division depend on it).
NCCL is the 2.28 copy shipped in the venv's nvidia/nccl wheel — the same libnccl.so.2
torch loads, so one NCCL lives in the process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libfsdp_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # noqa: F401  (namespace package of the nvidia-nccl wheel)
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "fsdp_b200.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    inc, lib = nccl_dirs()
    import time
    t_start = time.time()   # the library is stamped with this: sources edited during the build stay newer
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC",
           "-prec-div=true", "-prec-sqrt=true", "-ftz=false", "-Xptxas", "-v",
           *os.environ.get("FSDP_B200_NVCC_EXTRA", "").split(),   # experiments only (e.g. -D...)
           "-I", INCLUDE, "-I", CSRC, "-I", inc, *sources(),
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}", "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(res.stderr)
    os.replace(tmp, LIB)
    os.utime(LIB, (t_start, t_start))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
