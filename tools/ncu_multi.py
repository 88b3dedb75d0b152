#!/usr/bin/env python3
"""Per-kernel summary of a multi-kernel ncu --set full report:
    python tools/ncu_multi.py report.ncu-rep [--json out.json]
time, DRAM bytes read+write, registers, warps active, issue activity, top stalls."""
import csv
import io
import json
import subprocess
import sys

STALLS = ["barrier", "branch_resolving", "dispatch_stall", "drain", "imc_miss", "lg_throttle",
          "long_scoreboard", "math_pipe_throttle", "membar", "mio_throttle", "misc",
          "no_instruction", "not_selected", "selected", "short_scoreboard", "sleeping",
          "tex_throttle", "wait"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: k for k, h in enumerate(hdr)}

    def g(r, name):
        k = col.get(name)
        if k is None or r[k] in ("", "n/a"):
            return None
        try:
            return float(r[k].replace(",", ""))
        except ValueError:
            return r[k]
    res = []
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        t = g(r, "gpu__time_duration.sum")
        tu = units[col["gpu__time_duration.sum"]]
        rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
        bu = units[col["dram__bytes_read.sum"]]
        inst = g(r, "smsp__average_warp_latency_issue_stalled_barrier") or 0
        st = {}
        for s in STALLS:
            v = g(r, f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")
            if v:
                st[s] = round(v, 2)
        st = dict(sorted(st.items(), key=lambda kv: -kv[1])[:6])
        res.append(dict(kernel=name, time=t, time_unit=tu, dram_read=rd, dram_write=wr,
                        dram_unit=bu, regs=g(r, "launch__registers_per_thread"),
                        grid=g(r, "launch__grid_size"), block=g(r, "launch__block_size"),
                        warps_active_pct=g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                        issue_pct=g(r, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
                        dram_pct=g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                        l2_hit=g(r, "lts__t_sector_hit_rate.pct"),
                        stalls_per_issue=st))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    for d in res:
        print(json.dumps(d))


if __name__ == "__main__":
    main()
