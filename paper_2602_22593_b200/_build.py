"""Build libflykv.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "lib", "libflykv.so")
SOURCES = [os.path.join(CSRC, f) for f in ("flykv_host.cpp", "flykv_vmm.cpp", "flykv_nvls.cpp", "flykv_kernels.cu",
                                                 "flykv_decode.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "flykv_internal.h"), os.path.join(INCLUDE, "flykv.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
    "-cudart", "static",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tmp = LIB + f".tmp{os.getpid()}"
    extra = os.environ.get("FLYKV_NVCC_EXTRA", "").split()   # experiment knobs (-D...), never set by build()
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-shared", "-I", INCLUDE, "-I", CSRC, *SOURCES, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libflykv.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


EXAMPLE_SRC = os.path.join(ROOT, "examples", "c_switch_demo.c")
EXAMPLE_BIN = os.path.join(ROOT, "examples", "bin", "c_switch_demo")
EXAMPLE_MP_SRC = os.path.join(ROOT, "examples", "c_multiproc_demo.c")
EXAMPLE_MP_BIN = os.path.join(ROOT, "examples", "bin", "c_multiproc_demo")


def build_example() -> str:
    """Plain C (gcc -std=c99) programs against include/flykv.h + libflykv.so:
    the single-process demo (returned) and the multi-process one."""
    os.makedirs(os.path.dirname(EXAMPLE_BIN), exist_ok=True)
    cuda = os.path.dirname(os.path.dirname(nvcc())) if os.path.isabs(nvcc()) else "/usr/local/cuda"
    for src, out in ((EXAMPLE_SRC, EXAMPLE_BIN), (EXAMPLE_MP_SRC, EXAMPLE_MP_BIN)):
        cmd = ["gcc", "-std=c99", "-Wall", "-O2", "-o", out, src, "-I", INCLUDE,
               "-I", os.path.join(cuda, "include"), "-L", os.path.dirname(LIB), "-lflykv",
               "-L", os.path.join(cuda, "lib64"), "-lcudart", "-Wl,-rpath,$ORIGIN/../../paper_2602_22593_b200/lib",
               "-Wl,-rpath," + os.path.join(cuda, "lib64")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"gcc failed building {os.path.relpath(out, ROOT)}")
    return EXAMPLE_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
