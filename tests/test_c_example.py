"""The C ABI from plain C: examples/c_switch_demo.c (gcc -std=c99, no Python,
no torch) allocates pools with cudaMalloc, switches DP2 -> TP2 -> DP2 and
checks the round trip byte for byte; examples/c_multiproc_demo.c does the
same with one forked process per pool (CUDA IPC, kv_switch_range with the
device-side group barrier when every process has its own GPU, else
kv_switch_range_host with a host barrier)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bin(mp=False):
    from paper_2602_22593_b200 import _build
    b = _build.EXAMPLE_MP_BIN if mp else _build.EXAMPLE_BIN
    deps = [_build.EXAMPLE_SRC, _build.EXAMPLE_MP_SRC, os.path.join(_build.INCLUDE, "flykv.h"), _build.LIB]
    if not os.path.exists(b) or any(os.path.getmtime(d) > os.path.getmtime(b) for d in deps):
        _build.build_example()
    return b


def test_c_example_builds():
    assert os.access(_bin(), os.X_OK)
    assert os.access(_bin(mp=True), os.X_OK)


@pytest.mark.gpu
def test_c_example_runs():
    r = subprocess.run([_bin()], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "round-trip byte-exact" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 4])
def test_c_multiproc_example_runs(n):
    """examples/c_multiproc_demo.c: n forked processes, one pool each, CUDA
    IPC peer pools, one call per switch (push + barrier + remap; on one GPU
    kv_switch_range_host with a host barrier) DP_n -> TP_n -> DP_n, round
    trip byte-exact -- the multi-process path with no Python anywhere."""
    r = subprocess.run([_bin(mp=True), str(n)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "multi-process round-trip byte-exact" in r.stdout
