"""Compact view of sweep JSON lines: scheme addressing layout dtype frac MFLUP/s.
usage: python tools/jsum.py file.jsonl [file2.jsonl ...]"""
import json
import sys

for fn in sys.argv[1:]:
    for ln in open(fn):
        if not ln.strip():
            continue
        r = json.loads(ln)
        print(f'{r["config"]} {r["scheme"]:13s} {r["addressing"]:8s} {r["layout"]} {r["dtype"]} '
              f'{r["frac"]:.3f} {r["mflups"]:9.1f}')
