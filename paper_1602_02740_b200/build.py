"""Build libtoomgpu.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1602_02740_b200.build [--force]

Steps: (1) regenerate csrc/generated/toom_programs.cuh from gen/toomgen.py
(the generator proves every program exact before emitting it), (2) nvcc the
C-ABI library with -gencode arch=compute_100a,code=sm_100a -lineinfo.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
GEN_OUT = os.path.join(CSRC, "generated", "toom_programs.cuh")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libtoomgpu.so")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")

NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
]


def _sources():
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cu")]
    return srcs


def _deps():
    deps = _sources() + [os.path.join(PKG, "gen", "toomgen.py"), os.path.join(INCLUDE, "toomgpu.h")]
    for root, _, files in os.walk(CSRC):
        deps += [os.path.join(root, f) for f in files if f.endswith((".cuh", ".h"))]
    return deps


def generate():
    sys.path.insert(0, os.path.join(PKG, "gen"))
    try:
        import toomgen
    finally:
        sys.path.pop(0)
    code, _ = toomgen.generate_all()
    os.makedirs(os.path.dirname(GEN_OUT), exist_ok=True)
    old = open(GEN_OUT).read() if os.path.exists(GEN_OUT) else None
    if old != code:
        with open(GEN_OUT, "w") as f:
            f.write(code)


def build(force: bool = False, verbose: bool = False) -> str:
    generate()
    newest = max(os.path.getmtime(p) for p in _deps() if os.path.exists(p))
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = ["nvcc", *NVCC_FLAGS, "-I", INCLUDE, "-o", tmp, *_sources()]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
