"""Host logic of bench.py (CPU only): the NVLink/HBM roofline model of
SURVEY 8(d), the reference arm's JSON contract (the oracle on host cores),
its rank-0-only rule under torchrun, and the all-cores oracle figure."""
import json
import os
import subprocess
import sys

import numpy as np

import bench
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_nvlink_roofline_closed_form():
    """2 GPUs: GPU0 keeps 4 GB and sends 2 GB to GPU1; GPU1 sends 1 GB to GPU0."""
    m = np.array([[4e9, 2e9], [1e9, 0.0]])
    t, eg, ing, hbm = bench.nvlink_roofline(m, hbm_gbs=8000.0, link_gbs=1000.0)
    assert list(eg) == [2e9, 1e9] and list(ing) == [1e9, 2e9]
    assert list(hbm) == [4e9 + 2e9 + 4e9 + 1e9, 1e9 + 0 + 2e9 + 0]   # reads (row) + writes (column)
    assert t == max(2e9 / 1e12, 11e9 / 8e12)


def _run_reference(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--steps", "2",
                        "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_reference_arm_json_contract():
    lines = _run_reference({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]


def test_reference_arm_other_ranks_print_nothing():
    assert _run_reference({"WORLD_SIZE": "2", "RANK": "1"}) == []


def test_all_cores_oracle_figure():
    gbs, threads, info = bench.cpu_oracle_parallel(synth.WORKLOADS["tiny"](), reqs_per_thread=2, steps=2)
    assert gbs > 0 and 1 <= threads <= 4 and "threads" in info


def test_bench_has_no_undefined_names():
    """bench.py's GPU paths cannot run here; at least every name they load is
    bound somewhere (a crude pyflakes: catches typos in rarely-run branches)."""
    import ast
    import builtins
    for path in ("bench.py", "__graft_entry__.py", os.path.join("paper_2602_22593_b200", "engine.py"),
                 os.path.join("paper_2602_22593_b200", "comm.py")):
        tree = ast.parse(open(os.path.join(ROOT, path)).read())
        bound = set(dir(builtins)) | {"__file__"}
        for node in ast.walk(tree):
            if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
                bound.add(node.name)
            elif isinstance(node, ast.arg):
                bound.add(node.arg)
            elif isinstance(node, ast.Name) and isinstance(node.ctx, (ast.Store, ast.Del)):
                bound.add(node.id)
            elif isinstance(node, (ast.Import, ast.ImportFrom)):
                bound.update((a.asname or a.name).split(".")[0] for a in node.names)
            elif isinstance(node, ast.ExceptHandler) and node.name:
                bound.add(node.name)
        loaded = {n.id for n in ast.walk(tree) if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Load)}
        assert loaded <= bound, f"{path}: undefined {sorted(loaded - bound)}"


def test_gpus_n_self_launches_n_ranks():
    """bench.py --gpus 2 outside torchrun re-runs itself under
    torch.distributed.run with 2 ranks (the multi-rank path): the reference
    arm's line, printed by rank 0 alone, reports n_gpus = 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--gpus", "2",
                        "--steps", "1", "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


def test_main_dispatch(monkeypatch):
    """--gpus N > 1 without WORLD_SIZE -> self_launch; under torchrun
    (WORLD_SIZE > 1) -> run_multi; otherwise run_single.  Default workload:
    the north_star headline c4 (Llama-3-70B 8 x DP1 -> TP8)."""
    calls = []
    monkeypatch.setattr(bench, "self_launch", lambda a: calls.append(("self", a.gpus)) or 0)
    monkeypatch.setattr(bench, "run_multi", lambda a: calls.append(("multi", a.gpus)) or 0)
    monkeypatch.setattr(bench, "run_single", lambda a: calls.append(("single", a.config)) or 0)
    for k in ("WORLD_SIZE", "RANK"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    bench.main()
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("RANK", "0")
    bench.main()
    monkeypatch.delenv("WORLD_SIZE")
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    bench.main()
    assert calls == [("self", 4), ("multi", 4), ("single", "c4")]


def test_process_matrix_of_virtual_ranks():
    """8 engines on 2 GPUs (4 virtual ranks each): bytes between pools of one
    process stay in its HBM; the rest crosses NVLink."""
    m = np.arange(64, dtype=np.float64).reshape(8, 8)
    pm = bench.proc_matrix(m, 4)
    assert pm.shape == (2, 2) and pm.sum() == m.sum()
    assert pm[0, 1] == m[:4, 4:].sum() and pm[1, 0] == m[4:, :4].sum()


def test_weak_series_keeps_per_gpu_bytes():
    """--config weak (synth.weak_merge): two DP engines per GPU merged into TP
    groups of min(2N, 8); every GPU sources the same requests at every N."""
    import synth
    per_gpu = set()
    for n in (1, 2, 4, 8):
        w = synth.weak_merge(n)
        assert w.n_gpus == 2 * n and len(w.T) == 16 * n
        assert all(d[1] == min(2 * n, 8) and d[0] % d[1] == 0 for d in w.dst)
        for g in range(0, w.n_gpus, 2):   # GPU g // 2 owns engines g, g + 1
            per_gpu.add(tuple(sorted(T for T, s in zip(w.T, w.src) if s[0] in (g, g + 1))))
    assert len(per_gpu) == 1
