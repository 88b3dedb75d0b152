"""Per-source-line warp instructions and stall samples from an ncu report
(needs -lineinfo and --import-source on).
usage: python tools/src_hist.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if len(sys.argv) > 2 and sys.argv[2]:
        cmd += ["-k", "regex:" + sys.argv[2]]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    fname, hdr, lines = "?", None, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            ci = hdr.index("Instructions Executed")
            cs = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        try:
            lines.append((int(r[ci] or 0), int(r[cs] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except ValueError:  # a source line whose quotes broke the CSV
            continue
    ti = sum(x[0] for x in lines) or 1
    ts = sum(x[1] for x in lines) or 1
    print(f"total warp instructions {ti}  stall samples {ts}")
    for i, s, loc, src in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{100 * i / ti:6.2f}% inst {100 * s / ts:6.2f}% stall  {loc:24s} {src}")


if __name__ == "__main__":
    main()
