#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (run here, no GPU needed).

  python scripts/ncu_summary.py full  <report.ncu-rep> <out.json> [algorithmic_bytes]
  python scripts/ncu_summary.py launches <launches.csv> <out.json>
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "dram__cycles_elapsed.avg.per_second", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "smsp__cycles_active.avg"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def full(rep, out, algo=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        m = {"kernel": d.get("Kernel Name", ("", ""))[1]}
        for k in KEYS:
            if k in d:
                u, v = d[k]
                try:
                    f = float(v.replace(",", ""))
                except ValueError:
                    m[k] = v
                    continue
                m[k] = {"value": f, "unit": u}
        rb = m.get("dram__bytes_read.sum")
        wb = m.get("dram__bytes_write.sum")
        t = m.get("gpu__time_duration.sum")
        if isinstance(rb, dict) and isinstance(wb, dict):
            traffic = rb["value"] * SCALE.get(rb["unit"], 1) + wb["value"] * SCALE.get(wb["unit"], 1)
            m["dram_bytes_per_launch"] = traffic
            if isinstance(t, dict):
                m["dram_GBps_under_ncu"] = traffic / (t["value"] * SCALE.get(t["unit"], 1)) / 1e9
            if algo:
                m["algorithmic_bytes_per_launch"] = float(algo)
                m["traffic_over_algorithmic"] = traffic / float(algo)
        res.append(m)
    json.dump({"report": rep, "launches": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r and r[0] != "ID" and len(r) > 14]
    by = collections.defaultdict(list)
    for r in rows:
        if r[12] == "gpu__time_duration.sum":
            by[r[4]].append(float(r[14]) * SCALE.get(r[13], 1e-9))
    tot = sum(sum(v) for v in by.values())
    summ = {k: {"launches": len(v), "mean_ms": 1e3 * sum(v) / len(v), "total_ms": 1e3 * sum(v),
                "share": sum(v) / tot} for k, v in by.items()}
    json.dump({"source": path, "kernels": summ, "note": "ncu serialised cold-cache launch times; compare shares"},
              open(out, "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
