#!/usr/bin/env python3
"""Per-source-line warp instructions and stall samples from an exported
`ncu -i REP --page source --csv --print-source cuda,sass` file (see
tools/ncu_one.sh), for the functions matching a regex.

    python tools/src_csv_hist.py src.csv [function-regex] [top]"""
import csv
import re
import sys


def main():
    path = sys.argv[1]
    rx = re.compile(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    fname, func, hdr, lines = "?", "", None, []
    for r in csv.reader(open(path)):
        if len(r) >= 2 and r[0] == "File Path":
            fname, hdr = r[1].rsplit("/", 1)[-1], None
            continue
        if len(r) >= 2 and r[0] == "Function Name":
            func = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ci = hdr.index("Instructions Executed")
            cs = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        if rx and not rx.search(func):
            continue
        try:
            lines.append((int(r[ci] or 0), int(r[cs] or 0), f"{fname}:{r[0]}", r[1].strip()[:80]))
        except ValueError:
            continue
    ti = sum(x[0] for x in lines) or 1
    ts = sum(x[1] for x in lines) or 1
    print(f"total warp instructions {ti}  stall samples {ts}")
    print("-- by instructions")
    for i, s, loc, src in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{100 * i / ti:6.2f}% inst {100 * s / ts:6.2f}% stall  {loc:26s} {src}")
    print("-- by stall samples")
    for i, s, loc, src in sorted(lines, key=lambda x: -x[1])[:top]:
        print(f"{100 * i / ti:6.2f}% inst {100 * s / ts:6.2f}% stall  {loc:26s} {src}")


if __name__ == "__main__":
    main()
