#!/usr/bin/env python3
"""Summarise `ncu -i REP --page raw --csv` exports (written on the GPU box, so
the multi-GB .ncu-rep files never travel) into one JSON list for profiles/.

    python tools/ncu_csv_summary.py out.json name=raw.csv [name=raw.csv ...]

Per launch: kernel, duration, DRAM bytes, registers, occupancy, issue
activity, L1 / L2 hit rates, global load sectors per request and the top
stall reasons (warp-latency samples per issued instruction)."""
import csv
import json
import sys

MET = {
    "time_us": ("gpu__time_duration.sum", 1),
    "dram_read_gb": ("dram__bytes_read.sum", None),
    "dram_write_gb": ("dram__bytes_write.sum", None),
    "regs": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    "dram_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "ld_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 1),
    "ld_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 1),
    "st_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", 1),
    "st_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", 1),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "warp_inst": ("smsp__inst_executed.sum", 1),
}
STALL = "smsp__average_warps_issue_stalled_"


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def to_gb(v, unit):
    f = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(unit, None)
    return round(v * f, 4) if f is not None else v


def parse(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units = rows[hi], rows[hi + 1]
    out = []
    for r in rows[hi + 2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "?").split("(")[0].replace("void ", "")}
        for k, (m, scale) in MET.items():
            v = num(d.get(m, ""))
            if v is None:
                continue
            if scale is None:
                rec[k] = to_gb(v, u.get(m, ""))
            elif k == "time_us":
                f = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                     "msecond": 1e3}[u.get(m, "us")]
                rec[k] = round(v * f, 3)
            else:
                rec[k] = round(v, 3)
        if rec.get("ld_requests"):
            rec["ld_sectors_per_req"] = round(rec["ld_sectors"] / rec["ld_requests"], 2)
        if rec.get("st_requests"):
            rec["st_sectors_per_req"] = round(rec["st_sectors"] / rec["st_requests"], 2)
        st = {}
        for k, v in d.items():
            if k.startswith(STALL) and k.endswith("_per_issue_active.ratio"):
                x = num(v)
                if x and "selected" not in k:
                    st[k[len(STALL):-len("_per_issue_active.ratio")]] = round(x, 2)
        rec["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:6])
        out.append(rec)
    return out


def main():
    res = []
    for arg in sys.argv[2:]:
        name, path = arg.split("=", 1)
        for rec in parse(path):
            res.append({"case": name, **rec})
    with open(sys.argv[1], "w") as fh:
        json.dump(res, fh, indent=1)
    for r in res:
        print(r["case"], r["kernel"], r.get("time_us"), r.get("dram_read_gb"), r.get("dram_write_gb"),
              "L1", r.get("l1_hit_pct"), "L2", r.get("l2_hit_pct"), "ld s/r", r.get("ld_sectors_per_req"),
              "warps", r.get("warps_active_pct"), "issue", r.get("issue_pct"), r["stalls_per_issue"])


if __name__ == "__main__":
    main()
