"""Build libmeerkat.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2305_17813_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmeerkat.so")
ROOT = os.path.dirname(HERE)

def _nccl_include() -> str:
    """nccl.h for the types and prototypes of part.cu (libnccl.so.2 itself is opened at run time):
    the one next to torch's NCCL when present, else the system's."""
    try:
        import nvidia.nccl as m   # noqa: PLC0415
        for p in m.__path__:
            if os.path.exists(os.path.join(p, "include", "nccl.h")):
                return os.path.join(p, "include")
    except Exception:
        pass
    return "/usr/include"


NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v", "-I" + _nccl_include(), "-ldl",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "meerkat.h")]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Build OUT (or `out`, with extra -D `defines`, for A/B experiments)."""
    if out is not None:
        cmd = [os.environ.get("NVCC", "nvcc"), *NVCC_FLAGS, *[f"-D{d}" for d in defines], *sources(), "-o", out]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed")
        return out
    if not force and not stale():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = OUT + ".tmp"
    cmd = [nvcc, *NVCC_FLAGS, *sources(), "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(tmp, OUT)
    if verbose:
        sys.stdout.write(r.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
