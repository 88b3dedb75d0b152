#!/usr/bin/env python3
"""Summarise ncu output for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches gpurun_out/launches.csv      # launch list -> shares
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep [--key K] # --set full metrics
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size"]


def short(name):
    n = name.split("(")[0]
    n = n.replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return n.strip()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        t = float(r[vi].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    total = sum(v[1] for v in agg.values())
    out = []
    for k, (n, t) in agg.items():
        out.append({"kernel": k, "launches": n, "total_ns": t, "avg_ns": t / n,
                    "share": t / total if total else 0.0})
    return out


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m in FULL:
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                d[m] = v
                d[m + "_unit"] = units[hdr.index(m)]
        res.append(d)
    return res


def main():
    mode, path = sys.argv[1], sys.argv[2]
    data = launches(path) if mode == "launches" else full(path)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
