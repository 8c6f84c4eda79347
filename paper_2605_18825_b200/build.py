"""Build libsae.so (sm_100a) in-tree with nvcc: each translation unit of csrc/ is compiled to
an object (rebuilt when it or a header it includes is newer), then linked into one shared
library."""
from __future__ import annotations

import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsae.so")
OBJ = os.path.join(HERE, "build")
# translation unit -> the files it includes
SOURCES = {
    "sae.cu": ["sae.cu", "replay_impl.cuh", "dmath.cuh", "xxh64.cuh"],
    "predictor.cu": ["predictor.cu"],
}

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    *ARCH,
    "-lineinfo", "-O3", "-std=c++17",
    "--fmad=false",            # no FMA contraction anywhere (SURVEY c.4); the policy code also uses RN intrinsics
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def _hdr() -> str:
    return os.path.join(ROOT, "include", "sae.h")


def _newer(dst: str, deps) -> bool:
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(p) > t for p in deps)


def stale() -> bool:
    deps = [os.path.join(CSRC, f) for fs in SOURCES.values() for f in fs] + [_hdr()]
    return _newer(OUT, deps)


def _run(cmd, verbose):
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed: " + " ".join(cmd[-3:]))
    if verbose:
        sys.stderr.write(r.stderr)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile csrc/ into libsae.so (or `out`, with extra -D`defines`, e.g. a debug build)."""
    if out is None and not force and not stale():
        return OUT
    dst = out or OUT
    tag = ("_" + "_".join(d.replace("=", "-") for d in defines)) if defines else ""
    os.makedirs(OBJ, exist_ok=True)
    objs = []
    t_first = None
    for tu, deps in SOURCES.items():
        o = os.path.join(OBJ, tu.replace(".cu", tag + ".o"))
        if force or _newer(o, [os.path.join(CSRC, f) for f in deps] + [_hdr()]):
            tmp = o + ".tmp%d" % os.getpid()
            t0 = time.time()
            t_first = t0 if t_first is None else min(t_first, t0)
            _run([nvcc(), *NVCC_FLAGS, *["-D" + d for d in defines], "-I", os.path.join(ROOT, "include"),
                  "-c", "-o", tmp, os.path.join(CSRC, tu)], verbose)
            os.replace(tmp, o)
            os.utime(o, (t0, t0))     # a source edited during the compile stays newer: rebuilt next time
        objs.append(o)
    tmp = dst + ".tmp%d" % os.getpid()
    _run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs], verbose)
    os.replace(tmp, dst)
    if t_first is not None:
        os.utime(dst, (t_first, t_first))
    return dst


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
