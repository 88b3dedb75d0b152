"""Markdown table (DESIGN.md §5 format) from a tools/sweep.py JSON-lines file:
one row per (scheme, addressing), columns SoA f64 / SoA f32 / AoS f64 / AoS f32,
cells "MFLUP/s (fraction of the roofline)".
usage: python tools/md_table.py profiles/r01_sweep_c4_final5.jsonl"""
import json
import sys

ORDER = ["ts", "os-push", "os-pull", "osnt-pull-1s", "osnt-pull-2s", "cg", "swap-push",
         "swap-pull", "aap", "et"]
COLS = [("soa", "f64"), ("soa", "f32"), ("aos", "f64"), ("aos", "f32")]


def main():
    cells, keys = {}, []
    for ln in open(sys.argv[1]):
        if not ln.strip():
            continue
        r = json.loads(ln)
        k = (r["scheme"], r["addressing"])
        if k not in keys:
            keys.append(k)
        cells[k + (r["layout"], r["dtype"])] = f'{r["mflups"]:.0f} ({r["frac"]:.2f})'
    keys.sort(key=lambda k: (k[1] != "direct", ORDER.index(k[0]) if k[0] in ORDER else 99))
    print("| scheme | addr | SoA f64 | SoA f32 | AoS f64 | AoS f32 |")
    print("|---|---|---|---|---|---|")
    for k in keys:
        row = [cells.get(k + c, "—") for c in COLS]
        print(f"| {k[0]} | {k[1]} | " + " | ".join(row) + " |")


if __name__ == "__main__":
    main()
