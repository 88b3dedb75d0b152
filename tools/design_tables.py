#!/usr/bin/env python3
"""Rewrite the four sweep tables of DESIGN.md section 5 from profiles/r02_sweep_<cfg>.jsonl
(tools/md_table.py format). usage: python tools/design_tables.py"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADS = {"c1": "C1 (256³ channel", "c4": "C4 (200³ periodic", "c2": "C2 (porous 256³",
         "c0": "C0 (128³ periodic"}


def main():
    path = os.path.join(ROOT, "DESIGN.md")
    text = open(path).read()
    for cfg, head in HEADS.items():
        table = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "md_table.py"),
                                os.path.join(ROOT, "profiles", f"r02_sweep_{cfg}.jsonl")],
                               capture_output=True, text=True, check=True).stdout.rstrip("\n")
        i = text.index(head)
        m = re.compile(r"(\| scheme \| addr \|.*?\n)((?:\|.*\n)+)").search(text, i)
        text = text[:m.start()] + table + "\n" + text[m.end():]
    open(path, "w").write(text)


if __name__ == "__main__":
    main()
