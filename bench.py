#!/usr/bin/env python
"""bench.py -- DP<->TP KV re-layout throughput (GB/s, % roofline) + switch latency.

Metric (BASELINE.json): "DP<->TP KV re-layout GB/s (% HBM/NVLink roofline) +
switch latency ms".  A *step* is one whole live switch of the workload: the
host planner (validation, allocation, segment index, descriptor upload), the
reshard kernel over every atom, and the block-table remap (DESIGN.md section
1, a1-a7).  Steps alternate direction (DP -> TP, then back), so every step
moves the full payload with fresh allocations.

N=1 (default): the north_star headline, BASELINE configs[3] (Llama-3-70B-
shaped cache, 64 requests, 8 x DP1 -> TP8) with the 8 engines as virtual
ranks (8 pools) on one B200; the bound is HBM (read + write of every byte).
--config picks another workload (synth.WORKLOADS).  N>1: `bench.py --gpus N`
outside torchrun launches N ranks itself (one process per GPU); the same
switch runs with its engines mapped onto the N GPUs as blocks of 8/N virtual
ranks ("strong" scaling), every GPU pushing its atoms into peer pools over
NVLink (IPC-mapped), then the group barrier (device-side kv_group_barrier;
the host barrier when FLYKV_SAME_DEVICE=1 puts every rank on cuda:0, a
correctness mode, not an NVLink number).

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
import gc
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

DEBUG = bool(os.environ.get("FLYKV_BENCH_DEBUG"))
FALLBACK_HBM_GBS = 6650.0       # B200_PROFILING.md fallback (copy), "of fallback"
FALLBACK_NVLINK_GBS = 770.0     # measured peer copy per direction (B200_PROFILING.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4",
                    help="workload key of synth.WORKLOADS; default c4 = the north_star headline (Llama-3-70B "
                         "8 x DP1 -> TP8), its 8 engines mapped onto the N GPUs as 8/N virtual ranks each "
                         "(strong scaling); 'weak' = synth.weak_merge(N): two engines per GPU, per-GPU bytes fixed")
    ap.add_argument("--cpu-sample-reqs", type=int, default=4,
                    help="oracle sample (first N requests) per step of --impl reference and of cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-parallel", action="store_true", help="skip the all-cores oracle figure")
    ap.add_argument("--pieces", action="store_true",
                    help="memory-bounded waves that may split a request into block-aligned token pieces (R20)")
    ap.add_argument("--long-last", action="store_true", help="move the longest request to the end of the order")
    ap.add_argument("--lifo", action="store_true",
                    help="each switch moves the requests in the reverse order of the previous one (undo order)")
    ap.add_argument("--nvls", action="store_true",
                    help="N>1, GQA replication: NVLS multicast teams for the replicas (pools in shareable VMM memory, "
                         "one multimem store per atom per team); reports why when the box cannot")
    ap.add_argument("--a2a", action="store_true",
                    help="N>1 comparator: kv_pack -> all_to_all_single -> kv_unpack instead of the P2P-push kernel")
    ap.add_argument("--frag", type=float, default=1.25, help="source placement window / source need")
    ap.add_argument("--pool-slack", type=float, default=1.05, help="pool room beyond the window / max need")
    ap.add_argument("--placement", default="fragmented", choices=["fragmented", "contiguous"],
                    help="source block placement: seeded permutation (default) or ascending IDs")
    ap.add_argument("--waves", action="store_true", help="memory-bounded waves (kv_plan_waves) per switch")
    ap.add_argument("--rank-ids", default="identity", choices=["identity", "suggest"],
                    help="destination rank-ID assignment (P:291): identity (R3) or kv_suggest_rank_ids (N2)")
    ap.add_argument("--work-order", type=int, default=None, choices=[0, 1],
                    help="kernel work order (kv_cache_set_work_order): 1 mixed, 0 plan order; default 0 at N=1 "
                         "(all pools on one device) and 1 with one process per GPU")
    ap.add_argument("--clock-ms", type=int, default=200, help="nvidia-smi sampling period in the timed region (0: off)")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run N steps only, no JSON")
    ap.add_argument("--no-fill", action="store_true", help="skip the content hash fill (profiling runs)")
    ap.add_argument("--requests", type=int, default=0, help="use only the first N requests (profiling)")
    ap.add_argument("--decode", action="store_true",
                    help="N3 consumer: time kv_paged_decode over every layer of every pool after the forward "
                         "switch (and on the DP layout before it); its own JSON line")
    ap.add_argument("--q-heads", type=int, default=64, help="--decode: query heads of the model (Llama-3-70B: 64)")
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
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region.

    A background `nvidia-smi --query-gpu=timestamp,... -lms <period>` is
    started before the warm-up (its NVML start-up stalls the driver, which
    must not land in the timed region) and stopped after the region; only the
    samples stamped inside [begin, end] (plus the nearest one on each side)
    are summarised (B200_PROFILING.md clocks line)."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 200):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self._p = None
        self.t0 = self.t1 = None

    def start(self):
        if self.period_ms <= 0:
            return self
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                        "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._p = None
        return self

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()
        if self._p is not None:
            time.sleep(self.period_ms / 1000.0 + 0.05)  # one sample after the region
        self.stop()

    def stop(self):
        if self._p is None:
            return
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        self._p = None
        rows = []
        for line in out.splitlines():
            r = [x.strip() for x in line.split(",")]
            if len(r) < 10:
                continue
            try:
                import datetime
                r[0] = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except Exception:
                continue
            rows.append(r)
        if self.t0 is not None and rows:
            inside = [r for r in rows if self.t0 <= r[0] <= (self.t1 or r[0])]
            before = [r for r in rows if r[0] < self.t0][-1:]
            after = [r for r in rows if self.t1 is not None and r[0] > self.t1][:1]
            rows = before + inside + after
        self.rows = rows

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(r[2]) for r in self.rows) if v is not None]
        mx = [v for v in (num(r[3]) for r in self.rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for n, v in zip(names, r[6:10]):
                if v.strip().lower() in ("active", "1", "yes"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------- workload
def build_workload(args, world: int, rank: int):
    """The same workload at every N (strong scaling): its engines are mapped
    onto the N GPUs as consecutive blocks of engines/N virtual ranks."""
    # "weak": the weak-scaling series (per-GPU bytes fixed, engines = 2 x GPUs); the others are fixed workloads
    w = synth.weak_merge(world) if args.config == "weak" else synth.WORKLOADS[args.config]()
    if args.requests:
        w = synth.Workload(w.name + f" first{args.requests}", w.L, w.H, w.d, w.B, w.e, w.n_gpus,
                           w.T[:args.requests], w.src[:args.requests], w.dst[:args.requests])
    if getattr(args, "long_last", False):  # scheduling order (R8: requests move in caller order)
        k = int(np.argmax(w.T))
        idx = [i for i in range(len(w.T)) if i != k] + [k]
        w = synth.Workload(w.name + " long-last", w.L, w.H, w.d, w.B, w.e, w.n_gpus, [w.T[i] for i in idx],
                           [w.src[i] for i in idx], [w.dst[i] for i in idx])
    return w


def pools_and_tables(w, frag: float = 1.25, slack: float = 1.05, contiguous: bool = False):
    """Pool sizes + fragmented source tables; block counts from the product's
    own kv_blocks_for (Eq.2)."""
    from paper_2602_22593_b200 import flykv as F
    g = F.geometry(w.L, w.H, w.d, w.B, w.e)
    n0 = [F.kv_blocks_for(g, T, s[1]) for T, s in zip(w.T, w.src)]
    n1 = [F.kv_blocks_for(g, T, d[1]) for T, d in zip(w.T, w.dst)]
    return synth.realistic_pools(w, n0, n1, frag=frag, slack=slack, contiguous=contiguous)


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


def _mem_available_bytes() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_oracle_parallel(w, reqs_per_thread: int = 2, steps: int = 3, max_threads: int = 64):
    """The same oracle, unchanged, run as independent switches on every host
    core at once (SURVEY 8(d) asks for a single-thread and an all-cores
    figure): thread k owns requests [k*r, (k+1)*r) of the workload and its own
    pools, and alternates their direction `steps` times.  ctypes releases the
    GIL around each or_switch call, so the threads run in parallel.  Thread
    count is bounded by the cores this process may use, the workload's request
    count and a quarter of the host's available memory.  Returns (GB/s over the
    wall time of all threads, threads, info)."""
    import threading

    from oracle import oracle as O
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    og = O.Geom(w.L, w.H, w.d, w.B, w.e)
    M = O.block_bytes(og)
    subs = []
    for k in range(min(cores, max_threads, len(w.T) // reqs_per_thread)):
        a, b = k * reqs_per_thread, (k + 1) * reqs_per_thread
        subs.append(synth.Workload(w.name, w.L, w.H, w.d, w.B, w.e, w.n_gpus, w.T[a:b], w.src[a:b], w.dst[a:b]))
    budget = _mem_available_bytes() // 4
    need = 0
    for i, sub in enumerate(subs):
        need += sum(synth.pool_blocks(sub)) * w.L * M
        if budget and need > budget:
            subs = subs[:max(i, 1)]
            break
    work = []
    for sub in subs:
        nb = synth.pool_blocks(sub)
        pools = [np.full(w.L * n * M, 0x5A, dtype=np.uint8) for n in nb]
        held = [np.zeros(n, dtype=np.uint8) for n in nb]
        counts = [O.num_blocks(og, T, s_[1]) for T, s_ in zip(sub.T, sub.src)]
        tabs = synth.source_tables(sub, counts, nb)
        reqs = []
        for T, s_, d, ids in zip(sub.T, sub.src, sub.dst, tabs):
            for r in range(s_[1]):
                held[s_[0] + r][ids] = 1
            reqs.append(O.Req(T, s_, list(ids), d))
        work.append([pools, held, reqs, 0])
    start = threading.Barrier(len(work) + 1)

    def run(item):
        pools, held, reqs, _ = item
        start.wait()
        moved = 0
        for _ in range(steps):
            st, new = O.switch(og, pools, held, reqs)
            assert st == 0
            for r in reqs:
                if tuple(r.src) != tuple(r.dst):
                    moved += 2 * w.L * w.H * (-(-r.T // w.B)) * w.B * w.d * w.e * O.replicas(og, r.dst[1])
            reqs = [O.Req(r.T, r.dst, list(t), r.src) for r, t in zip(reqs, new)]
        item[3] = moved

    threads = [threading.Thread(target=run, args=(it,)) for it in work]
    for t in threads:
        t.start()
    start.wait()
    t0 = time.perf_counter()
    for t in threads:
        t.join()
    sec = time.perf_counter() - t0
    payload = sum(it[3] for it in work)
    info = (f"{len(work)} threads x {reqs_per_thread} requests each (requests 0..{len(work) * reqs_per_thread - 1}), "
            f"{steps} switches per thread, {payload / 1e9:.2f} GB moved in {sec:.2f} s wall")
    return payload / sec / 1e9, len(work), info


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_of(w, args, parallel: bool = True) -> dict:
    """The oracle as it stands, one host thread, on the same bounded sample
    and with the same --steps/--warmup in both arms (cpu_baseline of our
    line and the value of the --impl reference line are one measurement
    procedure), plus the all-cores figure."""
    gbs, sec, info, _ = cpu_oracle_run(w, args.cpu_sample_reqs, args.steps, args.warmup)
    out = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": info,
           "cpu_model": cpu_model(), "ms_per_switch": round(sec * 1e3, 3)}
    if parallel:
        pg, nt, pinfo = cpu_oracle_parallel(w)
        out["all_cores"] = {"value": round(pg, 4), "unit": "GB/s", "cores": nt, "sample": pinfo}
    return out


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = build_workload(args, world, rank)
    cpu = cpu_baseline_of(w, args, parallel=False)
    gbs = cpu["value"]
    line = {
        "impl": "reference", "metric": "DP<->TP KV re-layout GB/s", "value": gbs, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["ms_per_switch"],
        "higher_is_better": True, "scaling": "weak" if args.config == "weak" else "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": w.name + (f" ({w.n_gpus} engines)" if w.n_gpus > 1 else ""),
                   "layers": w.L, "kv_heads": w.H, "head_dim": w.d, "block_base": w.B, "requests": len(w.T),
                   "tokens": w.tokens(), "sample": cpu["sample"]},
        "cpu_baseline": cpu,
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
    nb, tabs = pools_and_tables(w, args.frag, args.pool_slack, args.placement == "contiguous")
    eng = KVSwitchEngine(g, nb, dev, tp_degrees=(2, 4, 8))
    if args.work_order is None:
        args.work_order = 0
    eng.cache.set_work_order(args.work_order)
    if not args.no_fill:
        for i, t in enumerate(eng.pools.tensors):
            synth.fill_hash_torch(t, i)
    for s, ids in zip(w.src, tabs):
        eng.cache.reserve(s, ids)
    reqs0 = [(i, T, s, ids, d, None, None) for i, (T, s, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]
    rank_ids = {}
    if args.rank_ids == "suggest":  # N2: one assignment per destination group (R19)
        for grp in sorted(set(tuple(d) for d in w.dst)):
            if grp[1] > 1:
                rank_ids[grp] = F.kv_suggest_rank_ids(eng.cache, reqs0, grp)
        reqs0 = [r[:6] + (rank_ids.get(tuple(r[4])),) for r in reqs0]
    state = {"reqs": reqs0, "n": 0}   # n: switches run so far (even before a forward switch)
    stream = eng.stream

    def flipped(reqs, plan):
        new = plan.dst_tables()
        return [(rid, T, d, t, s, drid, srid) for (rid, T, s, _, d, srid, drid), t in zip(reqs, new)]

    ev_pairs = []      # per step: [(e0, e1) per wave] around the reshard launches
    kern_fwd = []      # per timed step: did it start from the workload's initial layout
    step_stats = []    # per step: summed plan statistics over its waves
    n_waves = []

    def waves_of(reqs):
        """The switch of `reqs` as waves: [(plan requests, [(request index,
        tok0, tok1) per plan request])].  One wave by default; --waves:
        request-granular memory-bounded waves (N1); --pieces: waves that may
        split a request into block-aligned token pieces (R20)."""
        if args.pieces:
            return [([F.piece_request(g, reqs[i], t0, t1) for i, t0, t1 in wv], wv)
                    for wv in F.kv_plan_pieces(eng.cache, reqs)]
        ranges = F.kv_plan_waves(eng.cache, reqs) if args.waves else [(0, len(reqs))]
        return [(reqs[a:b], [(i, 0, reqs[i][1]) for i in range(a, b)]) for a, b in ranges]

    def flip_all(reqs, ws, plans_):
        """The requests after a switch run as waves ws by plans_: every request
        from its destination (concatenated piece tables) back to its source."""
        parts = [[] for _ in reqs]
        for (_, owners), plan in zip(ws, plans_):
            for (i, _, _), t in zip(owners, plan.dst_tables()):
                parts[i].append(t)
        out = [(rid, T, d, np.concatenate(parts[i]).astype(np.int32), s, drid, srid)
               for i, (rid, T, s, _, d, srid, drid) in enumerate(reqs)]
        return out[::-1] if args.lifo else out   # --lifo: undo a switch in the reverse request order

    def step(timed_kernel=False, read_back=False):
        """One whole switch (all waves).  Returns (tables, host copies)."""
        state["n"] += 1
        reqs = state["reqs"]
        pairs, agg, host, plans_ = [], None, {}, []
        ws = waves_of(reqs)
        dbg = [time.perf_counter()] if read_back and DEBUG else None
        for k, (sub, _) in enumerate(ws):
            plan = eng.plan(sub)
            dbg is not None and dbg.append(time.perf_counter())
            plan.upload(stream)
            dbg is not None and dbg.append(time.perf_counter())
            st_, _ = plan.stats()
            agg = dict(st_) if agg is None else {k_: (agg[k_] if k_ == "atom_bytes" else agg[k_] + st_[k_]) for k_ in agg}
            if timed_kernel:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            F.kv_reshard(plan, -1, stream)
            if timed_kernel:
                e1.record(stream)
                pairs.append((e0, e1))
            dbg is not None and dbg.append(time.perf_counter())
            views, packed = eng.alloc_packed(plan)            # every pool's table, one launch
            dbg is not None and dbg.append(time.perf_counter())
            F.kv_remap_block_tables(plan, -1, packed[0], packed[1], packed[2], stream)
            dbg is not None and dbg.append(time.perf_counter())
            if read_back:                                     # three D2H copies for all pools
                host[k] = tuple(x.to("cpu", non_blocking=True) for x in packed)
            dbg is not None and dbg.append(time.perf_counter())
            plans_.append(plan)
            dbg is not None and dbg.append(time.perf_counter())
        state["reqs"] = flip_all(reqs, ws, plans_)
        if dbg is not None:
            d = [(y - x) * 1e3 for x, y in zip(dbg, dbg[1:])]
            if sum(d) > 3:
                sys.stderr.write("slow enqueue: plan %.2f upload %.2f stats+reshard %.2f alloc %.2f remap %.2f d2h %.2f "
                                 "flip %.2f\n" % tuple(d[:7]))
        if timed_kernel:
            ev_pairs.append(pairs)
            kern_fwd.append(state["n"] % 2 == 1)
            step_stats.append(agg)
            n_waves.append(len(ws))
        return agg, host

    def step_switch():
        """One whole switch through kv_switch (plan, upload, reshard, remap,
        one table read-back, sync), or kv_switch_multi for several waves (one
        C call, one sync).  A single-wave
        switch that reverses the previous one is kv_switch_back: the inverse
        request list is built inside the library, nothing is marshalled.
        Returns (aggregated stats, device->host bytes)."""
        state["n"] += 1
        chain = state.setdefault("chain", [])
        if not (args.waves or args.pieces) and chain:
            plans_ = [F.kv_switch_back(eng.cache, chain[-1][2][0], stream)]
            chain.append((None, None, plans_))
        else:
            settle_switches()
            reqs = state["reqs"]
            if (args.waves or args.pieces) and os.environ.get("FLYKV_MULTI_WAVE", "1") == "1":
                # schedule + every wave in one C call, one sync (kv_switch_waves)
                wv, plans_ = F.kv_switch_waves(eng.cache, reqs, split=args.pieces, stream=stream)
                ws = [(None, owners) for owners in wv]
            else:  # FLYKV_MULTI_WAVE=0 (A/B): one kv_switch per wave
                ws = waves_of(reqs)
                plans_ = [F.kv_switch(eng.cache, sub, stream) for sub, _ in ws]
            state["chain"] = [(reqs, ws, plans_)]
        agg, d2h_b = None, 0
        for plan in plans_:
            st_, _ = plan.stats()
            agg = dict(st_) if agg is None else {k: (agg[k] if k == "atom_bytes" else agg[k] + st_[k]) for k in agg}
            n_res, n_ids = plan.resident(-1)
            d2h_b += 4 * (n_res + w.n_gpus + n_ids + 4 * n_res)
        return agg, d2h_b

    def settle_switches():
        """Replay the request tuples through the switches step_switch ran
        (outside the timed region), so state["reqs"] matches the cache."""
        for reqs_, ws, plans_ in state.pop("chain", []):
            reqs = state["reqs"]
            if ws is None:  # kv_switch_back of a single-wave, unsplit switch
                ws = [(reqs, [(i, 0, r[1]) for i, r in enumerate(reqs)])]
            state["reqs"] = flip_all(reqs, ws, plans_)

    class _Tables:
        """A finished plan's destination tables, kept after the plan is destroyed."""

        def __init__(self, plan):
            self.tabs = plan.dst_tables()

        def dst_tables(self):
            return self.tabs

    def compact_chain():
        """Between timed e2e steps: keep only the last switch's plan alive (the
        next kv_switch_back needs it); older ones keep their tables and are
        destroyed, so the library recycles their host buffers."""
        chain = state.get("chain", [])
        for k in range(len(chain) - 1):
            r_, ws_, plans_ = chain[k]
            if plans_ and not isinstance(plans_[0], _Tables):
                done = [_Tables(p) for p in plans_]
                for p in plans_:
                    p.destroy()
                chain[k] = (r_, ws_, done)

    with torch.cuda.stream(stream):
        if args.profile_steps:
            for _ in range(args.profile_steps):
                step()
            torch.cuda.synchronize()
            return 0
        p0_ = eng.plan(waves_of(state["reqs"])[0][0])
        fwd_matrix = p0_.stats()[1]
        p0_.destroy()
        fwd_rows = None
        if w.n_gpus > 1:  # the forward plan in the mixed order an N-GPU run would use (link model)
            eng.cache.set_work_order(1)
            p0_ = eng.plan(waves_of(state["reqs"])[0][0])
            fwd_rows = [p0_.work_order(x) for x in range(w.n_gpus)]
            p0_.destroy()
            eng.cache.set_work_order(args.work_order)
        clk = ClockSampler(torch.cuda.current_device(), args.clock_ms).start()
        stats = None
        for _ in range(max(args.warmup, 1)):
            st_w, _ = step()
            stats = stats or st_w            # forward-direction statistics
        torch.cuda.synchronize()
        # ------------------------------------------------ device-timed region
        # per-step events; when the payload fits in L2 a 512 MiB buffer is
        # rewritten between steps, outside the step events (L2 flush)
        flush = None
        if 2 * stats["payload_bytes"] < 4 * 126 * 2 ** 20:
            flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
        n_launch0 = F.launch_count()
        step_ev = []
        torch.cuda.synchronize()
        gc.collect()
        gc.disable()   # no collector pauses inside the timed regions
        clk.begin()
        plans = []
        for _ in range(args.steps):
            if flush is not None:
                flush.fill_(1)
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            plans.append(step(timed_kernel=True))
            b_.record(stream)
            step_ev.append((a_, b_))
        torch.cuda.synchronize()
        clk.end()
        launches = F.launch_count() - n_launch0
        total_ms = sum(a_.elapsed_time(b_) for a_, b_ in step_ev)
        kern_ms = [sum(a.elapsed_time(b) for a, b in pairs) for pairs in ev_pairs]
        plans.clear()
        clocks = clk.summary()
        # context for the roofline: a torch device copy (a library kernel,
        # not ours) run back to back for about as long as the timed region,
        # on this box in this process -- the sustained copy rate next to
        # MEASURED_PEAKS.json's burst figure (best of 10 short copies)
        sustained = None
        try:
            n_cp = 2 ** 32
            ca = torch.empty(n_cp, dtype=torch.uint8, device=dev)
            cb = torch.empty(n_cp, dtype=torch.uint8, device=dev)
            with torch.cuda.stream(stream):
                for _ in range(3):
                    cb.copy_(ca)
                reps = max(8, int(total_ms / (2 * n_cp / 6.4e12 * 1e3)))
                c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                c0.record(stream)
                for _ in range(reps):
                    cb.copy_(ca)
                c1.record(stream)
            torch.cuda.synchronize()
            sustained = {"value": round(2 * n_cp * reps / (c0.elapsed_time(c1) / 1e3) / 1e9, 1), "unit": "GB/s",
                         "how": f"torch copy_ of 4 GiB x {reps} back to back (read + write bytes), CUDA events"}
            del ca, cb
        except RuntimeError:
            sustained = None
        # ------------------------------------------------ end-to-end region
        e2e = None
        lat_ms = []
        if not args.no_e2e:
            h2d = d2h = 0
            e2e_payload = 0
            plan_ms = []
            enq_ms = []
            phases = []
            lat_fwd = []
            for _ in range(max(args.warmup, 1)):   # untimed end-to-end warm-up switches
                step_switch()
                stream.synchronize()
                compact_chain()
            for it in range(args.steps):
                t0 = time.perf_counter()
                if DEBUG:  # the same switch through the torch-plumbing engine, with enqueue timings
                    st_, host = step(read_back=True)
                    d2h_b = sum(int(x.numel()) * 4 for v in host.values() for x in v)
                else:      # the C ABI's one-call switch: returns with the tables on the host
                    st_, d2h_b = step_switch()
                te = time.perf_counter()
                stream.synchronize()
                t1 = time.perf_counter()
                if DEBUG and (t1 - te) * 1e3 > 8:
                    sys.stderr.write("slow sync: %.2f ms\n" % ((t1 - te) * 1e3))
                lat_ms.append((t1 - t0) * 1e3)
                lat_fwd.append(state["n"] % 2 == 1)   # this switch started from the workload's initial layout
                if not DEBUG:
                    compact_chain()                   # outside the step's timed window
                enq_ms.append((te - t0) * 1e3)
                h2d += st_["h2d_bytes"]
                e2e_payload += st_["payload_bytes"]
                d2h += d2h_b
                plan_ms.append(0.0)
                if not DEBUG:   # the library's own phase clock of this switch (kv_plan_stats t_*_ns)
                    phases.append([st_[k] / 1e6 for k in ("t_plan_ns", "t_enqueue_ns", "t_wait_ns", "t_read_ns")])
            gc.enable()
            settle_switches()
            if os.environ.get("FLYKV_BENCH_DEBUG"):
                sys.stderr.write("e2e per-step ms: " + " ".join(f"{x:.2f}" for x in lat_ms) + "\n")
                sys.stderr.write("e2e enqueue ms: " + " ".join(f"{x:.2f}" for x in enq_ms) + "\n")
            # host planning time alone (kv_plan_switch), measured on plans that are then abandoned
            for it in range(min(args.steps, 10)):
                sub0 = waves_of(state["reqs"])[0][0]
                t0 = time.perf_counter()
                p_ = eng.plan(sub0)
                plan_ms[it] = (time.perf_counter() - t0) * 1e3
                p_.destroy()
            plan_ms = plan_ms[:min(args.steps, 10)]
            tail = None
            if phases:  # attribute the latency tail: phases of the median step vs the slowest step
                order = np.argsort(lat_ms)
                med, worst = int(order[len(order) // 2]), int(order[-1])

                def split(k):
                    ph = phases[k]
                    return {"wall": round(lat_ms[k], 3), "plan": round(ph[0], 3), "enqueue": round(ph[1], 3),
                            "device_wait": round(ph[2], 3), "table_copy": round(ph[3], 3),
                            "python": round(lat_ms[k] - sum(ph), 3)}
                tail = {"median_step": split(med), "slowest_step": split(worst),
                        "device_wait_ms_p50_max": [round(float(np.percentile([p[2] for p in phases], 50)), 3),
                                                   round(max(p[2] for p in phases), 3)],
                        "note": "per-step host phases from the library (kv_plan_stats t_*_ns); python = wall minus "
                                "the library's phases (marshalling, ctypes, the stream sync already done)"}
            e2e = {"value": round(e2e_payload / (sum(lat_ms) / 1e3) / 1e9, 3), "unit": "GB/s",
                   "h2d_bytes_per_step": int(h2d // len(lat_ms)), "d2h_bytes_per_step": int(d2h // len(lat_ms)),
                   "value_at_p50": round(e2e_payload / len(lat_ms) / (statistics.median(lat_ms) / 1e3) / 1e9, 3),
                   "switch_latency_ms_p50": round(statistics.median(lat_ms), 3),
                   "switch_latency_ms_p99": round(float(np.percentile(lat_ms, 99)), 3),
                   # directions alternate; under GQA replication they move different bytes, so the
                   # pooled p50 can fall between them: the p50 of each direction
                   "switch_latency_ms_p50_forward_reverse": [
                       round(statistics.median([x for x, f in zip(lat_ms, lat_fwd) if f]), 3) if any(lat_fwd) else None,
                       round(statistics.median([x for x, f in zip(lat_ms, lat_fwd) if not f]), 3)
                       if not all(lat_fwd) else None],
                   "host_plan_ms_p50": round(statistics.median(plan_ms), 3),
                   "latency_breakdown": tail,
                   "api": ("KVSwitchEngine.switch(read_back=True)" if DEBUG else
                           "flykv.kv_switch / kv_switch_back: one C-ABI call per switch (plan, upload, "
                           "reshard, remap, one table read-back, sync); several waves: kv_switch_waves, one call "
                           "(schedule + every wave) and one sync")}

    # per-step statistics: directions alternate, and under GQA replication the
    # two directions move different byte counts (TP>H writes p/H replicas)
    payload_sum = sum(x["payload_bytes"] for x in step_stats)
    payload = payload_sum / len(step_stats)
    value = payload_sum / (total_ms / 1e3) / 1e9
    kmean = sum(kern_ms) / len(kern_ms)
    # read once + write every replica, all local HBM (virtual ranks share one device)
    algo_bytes = sum((x["n_atoms"] + x["n_atom_writes"]) * x["atom_bytes"] for x in step_stats) / len(step_stats)
    hbm_peak, peak_src = peaks()
    achieved = algo_bytes / (kmean / 1e3) / 1e9
    # What the same plan would be bound by if the virtual ranks were real
    # GPUs on NVSwitch: SURVEY 8(d) t_min from the forward plan's byte matrix
    # (a model, not a measurement).
    modeled = None
    if w.n_gpus > 1:
        t_min, eg, ing, hb = nvlink_roofline(fwd_matrix, hbm_peak)
        off = fwd_matrix.sum() - np.trace(fwd_matrix)
        modeled = {"n_gpus": w.n_gpus, "t_min_ms": round(t_min * 1e3, 3),
                   "max_egress_GB": round(float(eg.max()) / 1e9, 3), "max_ingress_GB": round(float(ing.max()) / 1e9, 3),
                   "local_fraction": round(float(np.trace(fwd_matrix) / max(fwd_matrix.sum(), 1)), 4),
                   "t_model_mixed_order_ms": round(ordered_link_model(fwd_rows, hbm_peak) * 1e3, 3),
                   "rank_ids": args.rank_ids, "link_GBps": FALLBACK_NVLINK_GBS,
                   "note": "model of an N-GPU run of the forward plan, not measured: t_min from its byte matrix, "
                           "t_model_mixed_order_ms from bench.ordered_link_model of its mixed kernel order"}
        del off
    # DRAM bytes of one forward launch from a committed ncu --set full capture
    # (plus that launch's algorithmic bytes: under GQA the two directions of
    # a step move different byte counts, so compare the ratio)
    traffic = traffic_ratio = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tpath) and not args.requests:
        try:
            tj = json.load(open(tpath))
            traffic, traffic_ratio = tj.get("dram_bytes_per_launch"), tj.get("traffic_over_algorithmic")
        except Exception:
            traffic = traffic_ratio = None
    cpu = None if args.no_cpu_baseline else cpu_baseline_of(w, args, parallel=not args.no_cpu_parallel)
    line = {
        "metric": "DP<->TP KV re-layout GB/s", "value": round(value, 3), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak" if args.config == "weak" else "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": w.name + (f" ({w.n_gpus} virtual ranks on 1 GPU)" if w.n_gpus > 1 else ""),
                   "layers": w.L, "kv_heads": w.H, "head_dim": w.d, "block_base": w.B, "requests": len(w.T),
                   "tokens": w.tokens(), "payload_bytes_per_step": int(payload),
                   "payload_bytes_forward": stats["payload_bytes"],
                   "placement": args.placement,
                   "work_order": ["plan", "mixed"][args.work_order],
                   "waves_per_switch": (round(sum(n_waves) / len(n_waves), 2) if (args.waves or args.pieces) else 1),
                   "pieces": bool(args.pieces), "long_last": bool(args.long_last), "lifo": bool(args.lifo),
                   "pool_bytes": int(eng.pools.nbytes()),
                   "l2": ("L2 flushed between steps (512 MiB rewrite, outside the step events)" if flush is not None
                          else "inputs larger than L2 (payload >> 126 MB), no flush needed"),
                   "step": "plan + descriptor upload + reshard + remap (alternating direction)"},
        "switch_latency_ms": round(total_ms / args.steps, 4),
        "reshard_kernel_ms": round(kmean, 4),
        "reshard_kernel_ms_steps": [round(x, 3) for x in kern_ms],   # per timed step (directions alternate)
        "reshard_kernel_ms_forward_reverse": [
            round(statistics.mean([x for x, f in zip(kern_ms, kern_fwd) if f]), 4) if any(kern_fwd) else None,
            round(statistics.mean([x for x, f in zip(kern_ms, kern_fwd) if not f]), 4) if not all(kern_fwd) else None],
        "reshard_kernel_ms_p50_p90": [round(float(np.percentile(kern_ms, 50)), 4),
                                      round(float(np.percentile(kern_ms, 90)), 4)],
        "modeled_nvlink": modeled,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                     "traffic_over_algorithmic_forward_launch": traffic_ratio, "peak_source": peak_src,
                     "kernel": ("flykv_reshard_tma_kernel (>= 4 replicas, forward) / flykv_reshard_kernel"
                                if max(max(d[1], s_[1]) for d, s_ in zip(w.dst, w.src)) >= 4 * w.H
                                and os.environ.get("FLYKV_REP_TMA", "1") != "0" else "flykv_reshard_kernel"),
                     "algorithmic_bytes_per_launch": int(algo_bytes),
                     "sustained_copy_same_box": sustained,
                     "frac_of_sustained_copy": (round(achieved / sustained["value"], 4) if sustained else None)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    return 0


def nvlink_roofline(bytes_matrix, hbm_gbs, link_gbs=FALLBACK_NVLINK_GBS):
    """t_min of SURVEY 8(d): max over GPUs of egress/link, ingress/link,
    (reads + writes)/HBM, in seconds; plus the per-GPU byte vectors."""
    m = np.asarray(bytes_matrix, dtype=np.float64)
    n = m.shape[0]
    off = m * (1 - np.eye(n))
    egress = off.sum(1)
    ingress = off.sum(0)
    hbm = m.sum(1) + m.sum(0)          # source reads + destination writes
    t = np.maximum(np.maximum(egress, ingress) / (link_gbs * 1e9), hbm / (hbm_gbs * 1e9))
    return float(t.max()), egress, ingress, hbm


def ordered_link_model(pieces, hbm_gbs, link_gbs=FALLBACK_NVLINK_GBS):
    """Completion time (s) of an N-GPU push in which every GPU works through
    its pieces in kernel order (flykv Plan.work_order: per piece the bytes
    written to each GPU, last column the bytes read), all GPUs at once.
    Fluid model: each sender moves its current piece's bytes in the piece's
    destination mix; rates are max-min fair (progressive filling, bytes
    written per second) under sender egress <= link, receiver ingress <=
    link (remote writes only) and per-GPU HBM (reads of its pieces + every
    write landing on it) <= hbm.  Unlike t_min (nvlink_roofline), which
    assumes each GPU's traffic is spread evenly over the whole switch, this
    charges senders that push into the same receiver at the same time
    (ingress hot-spots) -- a model, not a measurement."""
    n = len(pieces)
    cap = np.concatenate([np.full(n, link_gbs * 1e9), np.full(n, link_gbs * 1e9), np.full(n, hbm_gbs * 1e9)])
    idx = [0] * n
    rem = np.ones(n)
    t = 0.0
    eye = np.eye(n, dtype=bool)
    while True:
        act = [g for g in range(n) if idx[g] < len(pieces[g])]
        if not act:
            return t
        A = np.zeros((3 * n, n))      # resource use per byte/s written by sender g
        W = np.zeros(n)
        for g in act:
            row = pieces[g][idx[g]].astype(np.float64)
            v, r = row[:n], row[n]
            W[g] = v.sum()
            if W[g] <= 0:
                continue
            remote = np.where(eye[g], 0.0, v)
            A[g, g] = remote.sum() / W[g]             # egress of g
            A[n:2 * n, g] = remote / W[g]             # ingress of each receiver
            A[2 * n:, g] = v / W[g]                   # writes landing in each HBM
            A[2 * n + g, g] += r / W[g]               # reads of g
        zero = [g for g in act if W[g] <= 0]
        if zero:                                      # all-hole pieces take no time
            for g in zero:
                idx[g] += 1
                rem[g] = 1.0
            continue
        y = np.zeros(n)
        free = np.zeros(n, dtype=bool)
        free[act] = True
        load = np.zeros(3 * n)
        while free.any():
            s = A[:, free].sum(1)
            ok = s > 1e-15
            if not ok.any():
                break
            slack = (cap[ok] - load[ok]) / s[ok]
            d = max(float(slack.min()), 0.0)
            y[free] += d
            load += d * s
            sat = np.where(ok)[0][slack <= d * (1 + 1e-9) + 1e-300]
            for c in sat:
                free &= ~(A[c] > 1e-15)
        dt = min(rem[g] * W[g] / y[g] for g in act if y[g] > 0)
        t += dt
        for g in act:
            if y[g] > 0:
                rem[g] -= dt * y[g] / W[g]
                if rem[g] <= 1e-9:
                    idx[g] += 1
                    rem[g] = 1.0


def proc_matrix(bytes_matrix, v: int):
    """Pool-level byte matrix -> process-level (process r owns pools
    [r*v, (r+1)*v)): bytes between pools of one process stay in its HBM."""
    m = np.asarray(bytes_matrix, dtype=np.float64)
    n = m.shape[0] // v
    return m.reshape(n, v, n, v).sum(axis=(1, 3))


def run_multi(args):
    """One process per GPU (torchrun; bench.py --gpus N self-launches it).
    The workload's engines (8 for the default c4) are mapped onto the N
    processes as consecutive blocks of v = engines/N virtual ranks, so the
    same switch runs at every N (strong scaling).  Each process pushes the
    atoms its pools hold into every destination pool (local, or a peer GPU's
    through CUDA IPC over NVLink), then the device-side group barrier (a5,
    kv_group_barrier), then remaps its own pools' tables."""
    import torch
    import torch.distributed as dist

    from paper_2602_22593_b200 import comm
    from paper_2602_22593_b200 import flykv as F

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    same_dev = os.environ.get("FLYKV_SAME_DEVICE") == "1"   # test mode: all ranks on cuda:0, gloo plumbing
    if not same_dev and torch.cuda.device_count() < world:
        sys.stderr.write(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPU(s); "
                         "set FLYKV_SAME_DEVICE=1 to run every rank on cuda:0 (test mode)\n")
        return 2
    dev = torch.device("cuda", 0 if same_dev else local)
    torch.cuda.set_device(dev)
    nccl = not same_dev
    if nccl:   # NCCL init lines on stderr (the driver checks the rank count)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    w = build_workload(args, world, rank)
    if w.n_gpus % world:
        if rank == 0:
            sys.stderr.write(f"bench.py: workload {w.name} has {w.n_gpus} engines, not divisible by {world} GPUs\n")
        dist.destroy_process_group()
        return 2
    v = w.n_gpus // world
    mine = range(rank * v, (rank + 1) * v)
    degrees = [p for p in (2, 4, 8) if p <= world and world % p == 0]
    cpool = comm.CommunicatorPool(world, degrees, backend="nccl" if nccl else "gloo")   # eager
    world_key = tuple(range(world))
    barrier = comm.make_barrier(rank, world, list(dict.fromkeys(list(cpool.keys) + [world_key])), dev)
    host_bar = isinstance(barrier, comm.HostBarrier)
    bar_kind = "host" if host_bar else "device"
    bar_desc = ("host: stream sync + process-group barrier (ranks share one GPU, where spinning launches of "
                "different processes are not co-scheduled)" if host_bar
                else "kv_group_barrier (device-side, IPC counters)")
    g = F.geometry(w.L, w.H, w.d, w.B, w.e)
    _, _, M = F.kv_layout(g, 1)
    nb, tabs = pools_and_tables(w, args.frag, args.pool_slack, args.placement == "contiguous")
    nvls = None
    if args.nvls:   # N2: NVLS multicast teams for GQA replicas, when the box allows
        teams = sorted({d[1] // w.H for d in w.dst if d[1] > w.H})
        reason, gran = None, 0
        if v != 1:
            reason = "needs one pool per GPU (engines == GPUs)"
        elif same_dev:
            reason = "ranks share one device; a multicast team needs distinct GPUs"
        elif not teams:
            reason = f"no GQA replication in this workload (destination degrees <= H_kv = {w.H})"
        else:
            ok, gran, why = F.mc_supported(max(teams), w.L * nb[0] * M)
            reason = None if ok else why
        nvls = {"requested": True, "enabled": reason is None, "reason": reason, "team_sizes": teams}
    mcs = []
    if nvls and nvls["enabled"]:
        pool_mem, bases, nbs, imported_vmm = comm.exchange_pools_vmm(w.L * nb[0] * M, rank, world, w.L, M, nb[0],
                                                                   dev.index, gran)
        local_pools = pool_mem.tensor((1, w.L, nb[0], M))
        imported = []
    else:
        pool_mem, imported_vmm = None, []
        local_pools = torch.empty((v, w.L, nb[0], M), dtype=torch.uint8, device=dev)
    if not args.no_fill:
        for k, gp in enumerate(mine):
            synth.fill_hash_torch(local_pools[k], gp)
    torch.cuda.synchronize()
    if pool_mem is None:
        bases, nbs, imported = comm.exchange_pools(local_pools, rank, world, w.L, M)
    cache = F.KVCache(g, nbs, bases, tuple(p for p in (2, 4, 8) if p <= w.n_gpus))
    if pool_mem is not None:
        for r_ in nvls["team_sizes"]:
            mcs.append(comm.setup_multicast_teams(cache, pool_mem, rank, world, r_, w.L, M, nb[0], dev.index))
    if args.work_order is None:
        args.work_order = 0 if (same_dev or world == 1) else 1
    cache.set_work_order(args.work_order)
    for s_, ids in zip(w.src, tabs):
        cache.reserve(s_, ids)
    stream = torch.cuda.Stream(dev)
    reqs0 = [(i, T, s_, ids, d, None, None) for i, (T, s_, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]
    if args.rank_ids == "suggest":  # N2 (R19): identical on every rank (deterministic)
        rank_ids = {grp: F.kv_suggest_rank_ids(cache, reqs0, grp) for grp in sorted(set(tuple(d) for d in w.dst))
                    if grp[1] > 1}
        reqs0 = [r[:6] + (rank_ids.get(tuple(r[4])),) for r in reqs0]
    state = {"reqs": reqs0}
    ev_pairs = []

    def barrier_key(reqs):
        """Processes whose pools the switch touches: those of the smallest
        pooled group covering every source and destination (R12)."""
        if not reqs:
            return world_key
        lo = min(min(r[2][0], r[4][0]) for r in reqs)
        hi = max(max(r[2][0] + r[2][1], r[4][0] + r[4][1]) for r in reqs)
        key = cpool.covering([(lo // v, 1), ((hi - 1) // v, 1)])
        return key if key in barrier.slot else world_key

    step_stats = []
    out_bufs = {}

    def step(timed=False, read_back=False):
        plan = F.kv_plan_switch(cache, state["reqs"])
        plan.upload(stream)
        if timed:
            step_stats.append(plan.stats())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        if args.a2a:  # comparator: per-destination chunks through NCCL all_to_all_single (gloo: host copies)
            if v != 1:
                raise SystemExit("--a2a needs one pool per process")
            _, mat = plan.stats()
            send_off, recv_off = F.a2a_offsets(plan)
            n_send, n_recv = int(mat[rank].sum()), int(mat[:, rank].sum())
            send = torch.empty(max(n_send, 16), dtype=torch.uint8, device=dev)
            recv = torch.empty(max(n_recv, 16), dtype=torch.uint8, device=dev)
            F.kv_pack(plan, rank, send, send_off[rank], stream)
            with torch.cuda.stream(stream):
                outs, ins = [int(x) for x in mat[:, rank]], [int(x) for x in mat[rank]]
                if nccl:
                    dist.all_to_all_single(recv[:n_recv], send[:n_send], outs, ins)
                else:
                    stream.synchronize()
                    rh = torch.empty(n_recv, dtype=torch.uint8)
                    dist.all_to_all_single(rh, send[:n_send].cpu(), outs, ins)
                    recv[:n_recv].copy_(rh)
            F.kv_unpack(plan, rank, recv, recv_off[rank], stream)
        else:
            F.kv_reshard_range(plan, mine.start, mine.stop, stream)
        if timed:
            e1.record(stream)
            ev_pairs.append((e0, e1))
        barrier.wait(barrier_key(state["reqs"]), stream)   # a5
        host_bytes = 0
        for gp in mine:
            n_res, n_ids = plan.resident(gp)
            key = (gp, n_res, n_ids)
            if key not in out_bufs:
                out_bufs[key] = (torch.empty(n_res + 1, dtype=torch.int32, device=dev),
                                 torch.empty(max(n_ids, 1), dtype=torch.int32, device=dev),
                                 torch.empty((max(n_res, 1), 4), dtype=torch.int32, device=dev))
            rp, ids, meta = out_bufs[key]
            F.kv_remap_block_tables(plan, gp, rp, ids, meta, stream)
            if read_back:
                with torch.cuda.stream(stream):
                    h = [rp.to("cpu", non_blocking=True), ids[:n_ids].to("cpu", non_blocking=True),
                         meta[:n_res].to("cpu", non_blocking=True)]
                host_bytes += sum(int(x.numel()) * 4 for x in h)
        if read_back:
            stream.synchronize()
        new = plan.dst_tables()
        state["reqs"] = [(rid, T, d, t, s_, drid, srid)
                         for (rid, T, s_, _, d, srid, drid), t in zip(state["reqs"], new)]
        return plan, host_bytes

    clk = ClockSampler(dev.index, args.clock_ms).start()
    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    barrier.check()
    dist.barrier()
    n_launch0 = F.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    keep = []
    clk.begin()
    start.record(stream)
    for _ in range(args.steps):
        keep.append(step(timed=True))
    end.record(stream)
    torch.cuda.synchronize()
    clk.end()
    barrier.check()
    dist.barrier()
    launches = F.launch_count() - n_launch0
    my_ms = start.elapsed_time(end)
    kern = [a.elapsed_time(b) for a, b in ev_pairs]
    my_kern = sum(kern) / len(kern)
    keep.clear()
    lat = []
    h2d = d2h = 0
    e2e_payload = 0
    def step_one_call():
        """One switch through the public one-call API for this process's
        share (kv_switch_range: plan, upload, push, device barrier, remap of
        the owned pools, one read-back, sync)."""
        reqs = state["reqs"]
        plan = F.kv_switch_range(cache, reqs, mine.start, mine.stop, barrier.arm(barrier_key(reqs)), stream)
        _, tot = plan.packed_offsets()
        new = plan.dst_tables()
        state["reqs"] = [(rid, T, d, t, s_, drid, srid) for (rid, T, s_, _, d, srid, drid), t in zip(reqs, new)]
        return plan, 4 * int(tot.sum())

    e2e_step = step_one_call if not args.a2a else (lambda: step(read_back=True))
    if not args.no_e2e:
        for _ in range(max(args.warmup, 1)):   # untimed end-to-end warm-up switches
            e2e_step()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            dist.barrier()
            t0 = time.perf_counter()
            plan, hb = e2e_step()
            lat.append((time.perf_counter() - t0) * 1e3)
            h2d += plan.stats()[0]["h2d_bytes"]
            e2e_payload += plan.stats()[0]["payload_bytes"]
            d2h += hb
        barrier.check()
    red = torch.tensor([my_ms, my_kern, (sum(lat) / len(lat)) if lat else 0.0,
                        statistics.median(lat) if lat else 0.0, float(np.percentile(lat, 99)) if lat else 0.0],
                       dtype=torch.float64, device=dev if nccl else "cpu")
    dist.all_reduce(red, op=dist.ReduceOp.MAX)
    total_ms, kern_ms, lat_mean, lat_p50, lat_p99 = [float(x) for x in red.tolist()]
    n_l = torch.tensor([float(launches), float(d2h)], dtype=torch.float64, device=dev if nccl else "cpu")
    dist.all_reduce(n_l, op=dist.ReduceOp.SUM)   # every rank's kernels / read-backs count toward the job
    launches_all, d2h_all = int(n_l[0].item()), int(n_l[1].item())
    pool_cost = {"backend": "nccl" if nccl else "gloo", "groups": len(cpool.keys),
                 "init_seconds": round(cpool.init_seconds, 4),
                 "host_bytes_per_group": (int(cpool.host_bytes_per_group)
                                          if cpool.host_bytes_per_group is not None else None)}
    barrier.close()
    comm.close_pools(imported)
    torch.cuda.synchronize()
    dist.barrier()
    for m_ in mcs:
        m_.free()
    for pm_ in imported_vmm:
        pm_.free()
    if rank == 0:
        payload_sum = sum(x[0]["payload_bytes"] for x in step_stats)
        payload = payload_sum / len(step_stats)
        hbm_peak, peak_src = peaks()
        t_min = busiest = 0.0
        for _, m in step_stats:
            t, eg, ing, _ = nvlink_roofline(proc_matrix(m, v), hbm_peak)
            t_min += t / len(step_stats)
            busiest += float(max(eg.max(), ing.max())) / len(step_stats)
        achieved = busiest / (kern_ms / 1e3) / 1e9
        hbm_algo = sum((x[0]["n_atoms"] + x[0]["n_atom_writes"]) * x[0]["atom_bytes"] for x in step_stats) / len(step_stats)
        if same_dev:   # every rank on cuda:0: one HBM does all the reads and writes
            a_ = hbm_algo / (total_ms / args.steps / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": round(a_, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(a_ / hbm_peak, 4), "traffic": None, "peak_source": peak_src,
                    "kernel": "flykv_reshard_kernel of every rank sharing cuda:0; per-step time (incl. the device "
                              "barrier) as the denominator since the ranks' launches overlap"}
        else:
            roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": FALLBACK_NVLINK_GBS,
                    "unit": "GB/s", "frac": round(achieved / FALLBACK_NVLINK_GBS, 4), "traffic": None,
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md 770 GB/s)",
                    "t_min_ms": round(t_min * 1e3, 4), "frac_of_t_min": round(t_min * 1e3 / kern_ms, 4),
                    "work_order": ["plan", "mixed"][args.work_order],
                    "kernel": "flykv_reshard_kernel (busiest GPU's egress/ingress per launch)"}
        line = {
            "metric": "DP<->TP KV re-layout GB/s", "value": round(payload_sum / (total_ms / 1e3) / 1e9, 3),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True, "scaling": "weak" if args.config == "weak" else "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": w.name + (f" ({v} virtual ranks per GPU)" if v > 1 else "") +
                       (" (ranks share cuda:0, gloo plumbing)" if same_dev else "") +
                       (" [pack -> all_to_all_single -> unpack comparator]" if args.a2a else ""),
                       "engines": w.n_gpus, "pools_per_gpu": v, "layers": w.L,
                       "work_order": ["plan", "mixed"][args.work_order],
                       "kv_heads": w.H, "head_dim": w.d, "block_base": w.B, "requests": len(w.T),
                       "tokens": w.tokens(), "payload_bytes_per_step": int(payload),
                       "l2": "inputs larger than L2, no flush needed",
                       "barrier": bar_desc,
                       "step": (f"plan + upload + pack + all_to_all_single + unpack + {bar_kind} barrier + remap"
                                if args.a2a else
                                f"plan + upload + reshard (P2P push) + {bar_kind} barrier + remap")},
            "switch_latency_ms": round(total_ms / args.steps, 4),
            "reshard_kernel_ms": round(kern_ms, 4),
            "roofline": roof,
            "cpu_baseline": None,
            "e2e": ({"value": round(e2e_payload / len(lat) / (lat_mean / 1e3) / 1e9, 3), "unit": "GB/s",
                     "h2d_bytes_per_step": int(h2d // max(len(lat), 1)),
                     "d2h_bytes_per_step": int(d2h_all // max(len(lat), 1)),
                     "switch_latency_ms_p50": round(lat_p50, 3), "switch_latency_ms_p99": round(lat_p99, 3),
                     "switch_latency_ms_mean": round(lat_mean, 3),
                     "api": (f"flykv.{'kv_switch_range_host' if host_bar else 'kv_switch_range'}: one C-ABI call "
                             f"per rank per switch (plan, upload, push, {bar_kind} barrier, remap of the owned "
                             "pools, one table read-back, sync)" if not args.a2a
                             else f"plan, kv_pack, all_to_all_single, kv_unpack, {bar_kind} barrier, remap, read-back"),
                     "note": "per-rank wall clock from a host barrier to its tables on the host; max over ranks"}
                    if lat else None),
            "comm_pool": pool_cost,
            "nvls": nvls,
            "gpu_launches": launches_all,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    del local_pools
    if pool_mem is not None:
        pool_mem.free()
    dist.destroy_process_group()
    return 0


def run_decode(args):
    """N3 consumer measurement: paged decode attention (kv_paged_decode) reads
    the cache through the tables the remap produced.  One *pass* = one decode
    step of every resident request on every pool, every layer (L x pools
    launches, one per (pool, layer) as a model's attention layers would issue
    them).  Timed on the DP layout (before the switch) and on the TP layout
    (after the forward switch): algorithmic bytes = every K/V byte of every
    resident (request, local KV head) once, plus q and out; HBM-bound."""
    import torch

    from paper_2602_22593_b200 import flykv as F
    from paper_2602_22593_b200.engine import KVSwitchEngine

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    w = build_workload(args, 1, 0)
    g = F.geometry(w.L, w.H, w.d, w.B, w.e)
    nb, tabs = pools_and_tables(w, args.frag, args.pool_slack, args.placement == "contiguous")
    eng = KVSwitchEngine(g, nb, dev, tp_degrees=(2, 4, 8))
    eng.cache.set_work_order(0)
    for i, t in enumerate(eng.pools.tensors):   # finite bf16 contents: hash bytes with exponent bit 7 cleared
        synth.fill_hash_torch(t, i)
        t.view(torch.int16).bitwise_and_(-16385)
    for s_, ids in zip(w.src, tabs):
        eng.cache.reserve(s_, ids)
    hbm, hbm_src = peaks()
    stream = torch.cuda.Stream(dev)   # decode stream (graph capture needs a non-default stream)
    Hq = args.q_heads
    scale = 1.0 / float(np.sqrt(w.d))
    gen = torch.Generator(device=dev).manual_seed(5)

    def prepare(plan, views, host, req_of_layout):
        """Per pool: (pool, table views, seq_lens, q, out, q_local, algorithmic bytes per layer)."""
        items = []
        for gp in range(w.n_gpus):
            n_res, _ = plan.resident(gp)
            if n_res == 0:
                continue
            meta = host[gp][2].numpy()
            deg = req_of_layout(int(meta[0, 0]))   # every request of a pool has one degree here
            q_local = Hq // deg
            lens = torch.as_tensor([w.T[int(i)] for i in meta[:, 0]], dtype=torch.int32, device=dev)
            q = torch.randn((n_res, q_local, w.d), generator=gen, device=dev).to(torch.bfloat16)
            out = torch.empty((n_res, q_local, w.d), dtype=torch.float32, device=dev)
            kv = sum(int(w.T[int(i)]) * int(meta[k, 2]) for k, i in enumerate(meta[:, 0])) * 2 * w.d * w.e
            items.append((gp, views[gp], lens, q, out, q_local, kv + q.numel() * 2 + out.numel() * 4))
        return items

    def one_pass(items, after=True):
        """after: KV_DECODE_AFTER_DECODE on every launch -- the kernel before each is a decode launch (or, for
        the first, one of this library's kernels, none of which lets its dependents start early)."""
        for gp, t, lens, q, out, q_local, _ in items:
            base = eng.pools.tensors[gp]
            for l in range(w.L):
                F.kv_paged_decode(g, base[l].data_ptr(), t.meta.shape[0], t.req_ptr, t.block_ids, t.meta, lens,
                                  q_local, q, out, scale, max(w.T), stream, after_decode=after)

    def timed(items, after=True):
        """One pass captured in a CUDA graph (the 80-layer decode step is
        launch-bound from Python: 640 launches), replayed `steps` times
        between CUDA events; plus the same passes launched eagerly."""
        for _ in range(max(args.warmup, 3)):   # warm-up also sizes the decode workspace (no allocation in capture)
            one_pass(items, after)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            one_pass(items, after)
        torch.cuda.synchronize()
        for _ in range(max(args.warmup, 3)):
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk.begin()
        n0 = F.launch_count()
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        clk.end()
        ms = e0.elapsed_time(e1) / args.steps
        n_launch = (len(items) * w.L) * args.steps   # kernels inside the replayed graph (none launched by the host)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            one_pass(items, after)
        f1.record(stream)
        torch.cuda.synchronize()
        eager_ms = f0.elapsed_time(f1) / args.steps
        nbytes = sum(it[6] for it in items) * w.L
        del graph
        return ms, nbytes, n_launch, eager_ms

    clk = ClockSampler(0, args.clock_ms).start()
    # DP layout: a no-op plan lists every request in its DP engine's table
    noop = [(i, T, s_, ids, s_) for i, (T, s_, ids) in enumerate(zip(w.T, w.src, tabs))]
    plan0, views0, host0 = eng.switch(noop, read_back=True)
    torch.cuda.synchronize()
    dp_items = prepare(plan0, views0, host0, lambda i: w.src[i][1])
    dp_ms, dp_bytes, dp_launch, dp_eager = timed(dp_items)
    dp_ms_serial = timed(dp_items, after=False)[0]   # every launch waits for the previous one
    # forward switch, then the TP layout
    move = [(i, T, s_, ids_, d_) for i, (T, s_, ids_, d_) in enumerate(zip(w.T, w.src, tabs, w.dst))]
    plan1, views1, host1 = eng.switch(move, read_back=True)
    torch.cuda.synchronize()
    tp_items = prepare(plan1, views1, host1, lambda i: w.dst[i][1])
    tp_ms, tp_bytes, tp_launch, tp_eager = timed(tp_items)
    tp_ms_serial = timed(tp_items, after=False)[0]
    clk.stop()
    gbs = tp_bytes / tp_ms / 1e6
    line = {
        "metric": "paged decode attention GB/s (N3 consumer of the re-laid-out cache)",
        "value": round(gbs, 1), "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": round(tp_ms, 4), "higher_is_better": True, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": w.name + " after the forward switch", "layers": w.L, "kv_heads": w.H,
                   "q_heads": Hq, "head_dim": w.d, "requests": len(w.T), "tokens": w.tokens(),
                   "step": f"one decode step: kv_paged_decode for every (pool, layer), {tp_launch // args.steps} "
                           "launches back to back (programmatic dependent launch overlaps each launch's tiles "
                           "with the previous one's tail), captured once in a CUDA graph and replayed",
                   "l2": "inputs larger than L2 (KV bytes per pass >> 126 MB), no flush needed"},
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(gbs / hbm, 4), "traffic": None, "peak_source": hbm_src,
                     "kernel": "flykv_paged_decode_kernel", "algorithmic_bytes_per_step": int(tp_bytes),
                     "algorithmic_bytes": "every K/V byte of every resident (request, local KV head) + q + out"},
        "serialized": {"ms_per_step": round(tp_ms_serial, 4), "GBps": round(tp_bytes / tp_ms_serial / 1e6, 1),
                       "frac": round(tp_bytes / tp_ms_serial / 1e6 / hbm, 4),
                       "note": "flags 0: every launch starts after the previous one completed (as when a model's "
                               "other layer kernels sit between two attention launches); value/roofline use "
                               "KV_DECODE_AFTER_DECODE, consecutive decode launches overlapped"},
        "eager_ms_per_step": round(tp_eager, 4),
        "eager_note": "the same step launched from Python (640 ctypes calls): host-bound, context only",
        "dp_layout": {"ms_per_step": round(dp_ms, 4), "GBps": round(dp_bytes / dp_ms / 1e6, 1),
                      "eager_ms_per_step": round(dp_eager, 4),
                      "serialized_frac": round(dp_bytes / dp_ms_serial / 1e6 / hbm, 4),
                      "frac": round(dp_bytes / dp_ms / 1e6 / hbm, 4), "bytes_per_step": int(dp_bytes),
                      "launches_per_step": dp_launch // args.steps},
        "gpu_launches": tp_launch,
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    return 0


def self_launch(args) -> int:
    """bench.py --gpus N (N > 1) outside torchrun: re-run this script under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:   # not under torchrun: launch the N ranks ourselves
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.decode:
        return run_decode(args)
    if world > 1:
        return run_multi(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
