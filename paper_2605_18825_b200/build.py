"""Build libsae.so (sm_100a) in-tree with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsae.so")
SOURCES = ["sae.cu"]
DEPS = ["sae.cu", "replay_impl.cuh", "dmath.cuh", "xxh64.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "--fmad=false",            # no FMA contraction anywhere (SURVEY c.4); the policy code also uses RN intrinsics
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "sae.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile csrc/ into libsae.so (or `out`, with extra -D`defines`, e.g. a debug build)."""
    if out is None and not force and not stale():
        return OUT
    dst = out or OUT
    tmp = dst + ".tmp%d" % os.getpid()
    cmd = [nvcc(), *NVCC_FLAGS, *["-D" + d for d in defines], "-I", os.path.join(ROOT, "include"), "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, dst)
    return dst


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
