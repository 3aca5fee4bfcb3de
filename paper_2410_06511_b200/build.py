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
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(INCLUDE, "fsdp_b200.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compiles every source to an object in parallel (one nvcc per file), then links."""
    if not force and not _stale():
        return LIB
    inc, lib = nccl_dirs()
    import time
    from concurrent.futures import ThreadPoolExecutor
    t_start = time.time()   # the library is stamped with this: sources edited during the build stay newer
    tmp = LIB + ".tmp"
    objdir = os.path.join(HERE, ".obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-prec-div=true", "-prec-sqrt=true", "-ftz=false", "-Xptxas", "-v",
             *os.environ.get("FSDP_B200_NVCC_EXTRA", "").split(),   # experiments only (e.g. -D...)
             "-I", INCLUDE, "-I", CSRC, "-I", inc]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *flags, "-c", src, "-o", obj]
        return obj, cmd, subprocess.run(cmd, capture_output=True, text=True)

    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, srcs))
    link = [NVCC, *ARCH, "--shared", "-Xcompiler", "-fPIC", *[o for o, _, _ in results],
            "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}", "-o", tmp]
    res_link = None
    if all(r.returncode == 0 for _, _, r in results):
        res_link = subprocess.run(link, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        for _, cmd, r in results:
            f.write(" ".join(cmd) + "\n\n" + r.stdout + r.stderr + "\n")
        if res_link is not None:
            f.write(" ".join(link) + "\n\n" + res_link.stdout + res_link.stderr)
    if res_link is None or res_link.returncode != 0:
        for _, _, r in results:
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
        if res_link is not None:
            sys.stderr.write(res_link.stdout + res_link.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        for _, _, r in results:
            sys.stdout.write(r.stderr)
    os.replace(tmp, LIB)
    os.utime(LIB, (t_start, t_start))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
