"""Build the in-tree CUDA library libbimine_b200.so for sm_100a.

    python -m paper_1512_01641_b200.build

One nvcc invocation over csrc/abi.cu (which includes every kernel
header) and csrc/host_text.cpp; and the small CPython extension _pyhost
(csrc/pyhost.c, gcc against the interpreter's headers).  Both are written
next to this file so they travel to the GPU box with the repository
snapshot; the product loads the library with ctypes and fails loudly when
it is absent (see _native.py).
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbimine_b200.so")
SOURCES = ["abi.cu", "host_text.cpp"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".inc", ".h")))
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "bimine_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


PYHOST_SRC = os.path.join(CSRC, "pyhost.c")
PYHOST = os.path.join(HERE, "_pyhost" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def build_pyhost(force: bool = False) -> str:
    if not force and os.path.exists(PYHOST) and os.path.getmtime(PYHOST) >= os.path.getmtime(PYHOST_SRC):
        return PYHOST
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-Wall", "-shared", "-fPIC", "-I" + sysconfig.get_paths()["include"],
           PYHOST_SRC, "-o", PYHOST + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("gcc failed building _pyhost")
    os.replace(PYHOST + ".tmp", PYHOST)
    return PYHOST


def build(force: bool = False, verbose: bool = False) -> str:
    build_pyhost(force)
    if not force and not stale():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libbimine_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
