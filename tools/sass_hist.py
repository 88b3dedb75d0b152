"""Histogram of an ncu report's SASS page: warp instructions executed and
stall samples per opcode, plus the total per launch.
usage: python tools/sass_hist.py report.ncu-rep [kernel-regex]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if len(sys.argv) > 2:
        cmd += ["-k", "regex:" + sys.argv[2]]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    inst = defaultdict(int)
    stall = defaultdict(int)
    for r in rows:
        if len(r) > 3 and r[0] == "Address":
            hdr = r
            ci = hdr.index("Instructions Executed")
            cs = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        op = r[1].split()[0] if r[1].split() else "?"
        if op.startswith("@"):
            op = r[1].split()[1]
        op = op.split(".")[0]
        inst[op] += int(r[ci] or 0)
        stall[op] += int(r[cs] or 0)
    tot_i, tot_s = sum(inst.values()), sum(stall.values())
    print(f"total warp instructions {tot_i}  stall samples {tot_s}")
    for op in sorted(inst, key=lambda o: -inst[o])[:40]:
        print(f"{op:12s} {inst[op]:12d} {100 * inst[op] / tot_i:6.2f}%  stall {100 * stall[op] / max(tot_s, 1):6.2f}%")


if __name__ == "__main__":
    main()
