#!/usr/bin/env python
"""bench.py -- DP<->TP KV re-layout throughput (GB/s, % roofline) + switch latency.

Metric (BASELINE.json): "DP<->TP KV re-layout GB/s (% HBM/NVLink roofline) +
switch latency ms".  A *step* is one whole live switch of the workload: the
host planner (validation, allocation, segment index, descriptor upload), the
reshard kernel over every atom, and the per-GPU block-table remap kernels
(a1-a7).  Steps alternate direction (DP4 -> TP2x2, then
back), so every step moves the full payload with fresh allocations.

N=1 (default): BASELINE configs[1] (Llama-3.1-8B-shaped cache, 64 requests,
DP4 -> TP2x2) with the 4 engines as virtual ranks (4 pools) on one B200; the
bound is HBM (read + write of every byte).  N>1 (torchrun, one process per
GPU): DP_N -> TP_N merge of the same geometry with 16 requests per GPU, every
GPU pushing its atoms into peer pools over NVLink (IPC-mapped), bound by
NVLink per-direction bandwidth ("weak" scaling).

`value`  = payload bytes of the K timed steps / device time (CUDA events on
           the switch stream; max over ranks), pools resident in HBM.
`e2e`    = the same steps through the public API with the request tables
           coming from host memory (descriptor H2D inside the step) and the new
           block tables read back to host each step, host wall clock.
--impl reference runs the oracle (plain C, host cores) on a bounded sample of
the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

FALLBACK_HBM_GBS = 6650.0       # B200_PROFILING.md fallback (copy), "of fallback"
FALLBACK_NVLINK_GBS = 770.0     # measured peer copy per direction (B200_PROFILING.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", help="workload key of synth.WORKLOADS (N=1)")
    ap.add_argument("--cpu-sample-reqs", type=int, default=6, help="oracle sample per --impl reference step")
    ap.add_argument("--cpu-baseline-reqs", type=int, default=16, help="oracle sample for cpu_baseline")
    ap.add_argument("--cpu-baseline-steps", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run N steps only, no JSON")
    ap.add_argument("--no-fill", action="store_true", help="skip the content hash fill (profiling runs)")
    ap.add_argument("--requests", type=int, default=0, help="use only the first N requests (profiling)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm, src = FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"
    if os.path.exists(path):
        try:
            d = json.load(open(path))
            for k in ("hbm_gbs", "hbm_GBs", "hbm_copy_gbs"):
                if k in d:
                    hbm, src = float(d[k]), "measured (MEASURED_PEAKS.json)"
                    break
        except Exception:
            pass
    return hbm, src


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() in ("active", "1", "yes"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------- workload
def build_workload(args, world: int, rank: int):
    if world == 1:
        w = synth.WORKLOADS[args.config]()
    else:
        w = synth.dp_to_tp(world, 16 * world)
    if args.requests:
        w = synth.Workload(w.name + f" first{args.requests}", w.L, w.H, w.d, w.B, w.e, w.n_gpus,
                           w.T[:args.requests], w.src[:args.requests], w.dst[:args.requests])
    return w


def src_tables_product(w, nb):
    from paper_2602_22593_b200 import flykv as F
    g = F.geometry(w.L, w.H, w.d, w.B, w.e)
    counts = [F.kv_blocks_for(g, T, s[1]) for T, s in zip(w.T, w.src)]
    return synth.source_tables(w, counts, nb)


# --------------------------------------------------------------- reference arm
def cpu_oracle_run(w, n_sample: int, steps: int, warmup: int):
    """Time the oracle (plain C, one host thread) on the first n_sample
    requests of the workload; each step is one switch of the sample (the
    direction alternates).  Returns (GB/s, seconds per step, sample info)."""
    from oracle import oracle as O
    sub = synth.Workload(w.name + " sample", w.L, w.H, w.d, w.B, w.e, w.n_gpus, w.T[:n_sample], w.src[:n_sample],
                         w.dst[:n_sample])
    og = O.Geom(w.L, w.H, w.d, w.B, w.e)
    nb = synth.pool_blocks(sub)
    M = O.block_bytes(og)
    pools = [np.full(w.L * n * M, 0x5A, dtype=np.uint8) for n in nb]
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    counts = [O.num_blocks(og, T, s[1]) for T, s in zip(sub.T, sub.src)]
    tabs = synth.source_tables(sub, counts, nb)
    reqs = []
    for T, s, d, ids in zip(sub.T, sub.src, sub.dst, tabs):
        for r in range(s[1]):
            held[s[0] + r][ids] = 1
        reqs.append(O.Req(T, s, list(ids), d))
    payload = 0
    for T, s, d in zip(sub.T, sub.src, sub.dst):
        if tuple(s) != tuple(d):
            payload += 2 * w.L * w.H * (-(-T // w.B)) * w.B * w.d * w.e * O.replicas(og, d[1])
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        st, new = O.switch(og, pools, held, reqs)
        t1 = time.perf_counter()
        assert st == 0
        reqs = [O.Req(r.T, r.dst, list(t), r.src) for r, t in zip(reqs, new)]
        if it >= warmup:
            times.append(t1 - t0)
    sec = sum(times) / len(times)
    info = (f"first {n_sample} of {len(w.T)} requests ({payload / 1e9:.3f} GB payload per switch), "
            f"oracle kv_oracle.c, 1 thread, {steps} timed switches")
    return payload / sec / 1e9, sec, info, payload


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = build_workload(args, world, rank)
    gbs, sec, info, payload = cpu_oracle_run(w, args.cpu_sample_reqs, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": "DP<->TP KV re-layout GB/s", "value": round(gbs, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": w.name, "sample": info},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": info},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm, N = 1
def run_single(args):
    import torch

    from paper_2602_22593_b200 import flykv as F
    from paper_2602_22593_b200.engine import KVSwitchEngine

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    w = build_workload(args, 1, 0)
    g = F.geometry(w.L, w.H, w.d, w.B, w.e)
    nb = synth.pool_blocks(w)
    eng = KVSwitchEngine(g, nb, dev, tp_degrees=(2, 4, 8))
    if not args.no_fill:
        for i, t in enumerate(eng.pools.tensors):
            synth.fill_hash_torch(t, i)
    tabs = src_tables_product(w, nb)
    for s, ids in zip(w.src, tabs):
        eng.cache.reserve(s, ids)
    state = {"reqs": [(i, T, s, ids, d) for i, (T, s, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]}
    stream = eng.stream

    def next_requests(plan):
        new = plan.dst_tables()
        return [(rid, T, d, t, s) for (rid, T, s, _, d), t in zip(state["reqs"], new)]

    ev_pairs = []

    def step(timed_kernel=False):
        plan = eng.plan(state["reqs"])
        plan.upload(stream)
        if timed_kernel:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        F.kv_reshard(plan, -1, stream)
        if timed_kernel:
            e1.record(stream)
            ev_pairs.append((e0, e1))
        tables = eng.alloc_tables(plan, range(eng.n_gpus))
        for gg, t in tables.items():
            F.kv_remap_block_tables(plan, gg, t.req_ptr, t.block_ids, t.meta, stream)
        state["reqs"] = next_requests(plan)
        return plan, tables

    with torch.cuda.stream(stream):
        plan0 = eng.plan(state["reqs"])
        stats, bytes_matrix = plan0.stats()
        plan0.destroy()
        if args.profile_steps:
            for _ in range(args.profile_steps):
                step()
            torch.cuda.synchronize()
            return 0
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        # ------------------------------------------------ device-timed region
        n_launch0 = F.launch_count()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as clk:
            torch.cuda.synchronize()
            start.record(stream)
            plans = []
            for _ in range(args.steps):
                plans.append(step(timed_kernel=True))
            end.record(stream)
            torch.cuda.synchronize()
        launches = F.launch_count() - n_launch0
        total_ms = start.elapsed_time(end)
        kern_ms = [a.elapsed_time(b) for a, b in ev_pairs]
        plans.clear()
        clocks = clk.summary()
        # ------------------------------------------------ end-to-end region
        e2e = None
        lat_ms = []
        if not args.no_e2e:
            h2d = d2h = 0
            for it in range(args.steps):
                t0 = time.perf_counter()
                plan, tables, host = eng.switch(state["reqs"], read_back=True)
                t1 = time.perf_counter()
                lat_ms.append((t1 - t0) * 1e3)
                st_, _ = plan.stats()
                h2d += st_["h2d_bytes"]
                d2h += sum(int(x.numel()) * 4 for v in host.values() for x in v)
                state["reqs"] = next_requests(plan)
            e2e = {"value": round(stats["payload_bytes"] * len(lat_ms) / (sum(lat_ms) / 1e3) / 1e9, 3), "unit": "GB/s",
                   "h2d_bytes_per_step": int(h2d // len(lat_ms)), "d2h_bytes_per_step": int(d2h // len(lat_ms)),
                   "switch_latency_ms_p50": round(statistics.median(lat_ms), 3),
                   "switch_latency_ms_p99": round(float(np.percentile(lat_ms, 99)), 3)}

    payload = stats["payload_bytes"]
    value = payload * args.steps / (total_ms / 1e3) / 1e9
    kmean = sum(kern_ms) / len(kern_ms)
    algo_bytes = (stats["n_atoms"] + stats["n_atom_writes"]) * stats["atom_bytes"]  # read + write, all local HBM
    hbm_peak, peak_src = peaks()
    achieved = algo_bytes / (kmean / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if not args.no_cpu_baseline:
        gbs, sec, info, _ = cpu_oracle_run(w, args.cpu_baseline_reqs, args.cpu_baseline_steps, 0)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": info}
    line = {
        "metric": "DP<->TP KV re-layout GB/s", "value": round(value, 3), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": w.name + " (4 virtual ranks on 1 GPU)" if w.n_gpus > 1 else w.name,
                   "layers": w.L, "kv_heads": w.H, "head_dim": w.d, "block_base": w.B, "requests": len(w.T),
                   "tokens": w.tokens(), "payload_bytes_per_step": payload,
                   "l2": "inputs larger than L2 (payload >> 126 MB), no flush needed",
                   "step": "plan + descriptor upload + reshard + remap (alternating direction)"},
        "switch_latency_ms": round(total_ms / args.steps, 4),
        "reshard_kernel_ms": round(kmean, 4),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "kernel": "flykv_reshard_kernel", "algorithmic_bytes_per_launch": algo_bytes},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        from paper_2602_22593_b200 import comm
        return comm.run_bench_multi(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
