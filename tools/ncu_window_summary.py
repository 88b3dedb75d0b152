"""Summarise ncu --set full captures (AoS window or any kernels) into markdown:
per report the kernel, time, DRAM bytes, registers, issue/warp activity, the
main stall reasons and the top source lines (needs -lineinfo, --import-source).
usage: python tools/ncu_window_summary.py out.md name=report.ncu-rep ..."""
import csv
import io
import os
import subprocess
import sys

MET = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
       "sm__inst_issued.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}


def lines(rep, top):
    out = subprocess.run([sys.executable, __file__.replace("ncu_window_summary", "src_hist"), rep,
                          "", str(top)], capture_output=True, text=True).stdout
    return out.strip().splitlines()


def main():
    dst = sys.argv[1]
    title = os.environ.get("NCU_SUMMARY_TITLE",
                           "AoS window kernels, ncu --set full (C1 256^3 channel, fp64, one launch each)")
    md = ["# " + title, ""]
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        d = raw(rep)
        kern = d.get("Kernel Name", ("", "?"))[1]
        md.append(f"## {name}: `{kern[:90]}`")
        md.append("")
        for m in MET:
            if m in d:
                md.append(f"* {m}: {d[m][1]} {d[m][0]}")
        stalls = []
        for h, (u, v) in d.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    x = float(v)
                except ValueError:
                    continue
                if x >= 0.1:
                    stalls.append((x, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        md.append("* stalls per issued instruction: " +
                  ", ".join(f"{n} {x:.2f}" for x, n in sorted(stalls, reverse=True)))
        md.append("")
        md.append("```")
        md.extend(lines(rep, 12))
        md.append("```")
        md.append("")
    open(dst, "w").write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
