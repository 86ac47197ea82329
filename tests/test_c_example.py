"""The C ABI from plain C: examples/c_switch_demo.c (gcc -std=c99, no Python,
no torch) allocates pools with cudaMalloc, switches DP2 -> TP2 -> DP2 and
checks the round trip byte for byte."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bin():
    from paper_2602_22593_b200 import _build
    b = _build.EXAMPLE_BIN
    deps = [_build.EXAMPLE_SRC, os.path.join(_build.INCLUDE, "flykv.h"), _build.LIB]
    if not os.path.exists(b) or any(os.path.getmtime(d) > os.path.getmtime(b) for d in deps):
        _build.build_example()
    return b


def test_c_example_builds():
    assert os.access(_bin(), os.X_OK)


@pytest.mark.gpu
def test_c_example_runs():
    r = subprocess.run([_bin()], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "round-trip byte-exact" in r.stdout
