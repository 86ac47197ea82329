"""bench.py's multi-rank path on one B200: `bench.py --gpus N` outside
torchrun launches N ranks itself (one process per GPU; here, with
FLYKV_SAME_DEVICE=1, all on cuda:0 with gloo plumbing and the host barrier,
since spinning device barriers of different processes must not share a
GPU).  Rank 0 prints one JSON line for the whole job."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,config", [(2, "tiny"), (4, "c2")])
def test_bench_self_launched_ranks(n, config):
    env = dict(os.environ, FLYKV_SAME_DEVICE="1")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--config", config, "--requests", "8",
                        "--steps", "3", "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["barrier"].startswith("host")
    assert d["e2e"]["api"].startswith("flykv.kv_switch_range_host")


def test_bench_decode_line():
    """bench.py --decode (N3): one decode step over every (pool, layer),
    captured in a CUDA graph, before and after the forward switch; one JSON
    line with the roofline of kv_paged_decode."""
    r = subprocess.run([sys.executable, "bench.py", "--decode", "--config", "tiny", "--q-heads", "16", "--steps", "3",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert d["roofline"]["kernel"] == "flykv_paged_decode_kernel" and d["roofline"]["bound"] == "hbm"
    assert d["value"] > 0 and d["dp_layout"]["GBps"] > 0 and d["gpu_launches"] == 3 * 2 * 2
