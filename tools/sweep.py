#!/usr/bin/env python3
"""Propagation-scheme sweep (BASELINE.json configs[4] and friends) on one B200.

    python tools/sweep.py [--config c4] [--steps 50] [--out profiles/sweep.jsonl]

For every implemented (scheme, addressing) x {SoA, AoS} x {fp64, fp32}: MFLUP/s
from CUDA events on the launching stream (warm-up first), the algorithmic
bytes/FLUP of SURVEY.md 8(d), achieved GB/s and the fraction of the measured
HBM copy peak. One JSON object per line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1111_0922_b200 as L  # noqa: E402
from paper_1111_0922_b200.geometry import gen_random_spheres  # noqa: E402

SCHEMES = ["ts", "os-push", "os-pull", "osnt-pull-1s", "osnt-pull-2s", "cg", "swap-push",
           "swap-pull", "aap", "et"]
IND = ["os-push", "os-pull", "osnt-pull-1s", "osnt-pull-2s", "aap", "et"]
EXT = ["ts", "swap-push", "swap-pull"]


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def run_one(geo, flow, scheme, addr, layout, prec, steps, warmup, init, tag):
    ext = addr == "indirect" and scheme in EXT
    st = L.create_stepper(scheme, addr, geo, flow,
                          L.StepperOptions(layout=layout, precision=prec, extensions=ext))
    st.init_field(init, seed=2011)
    st.step_n(warmup)
    st.synchronize()
    ms = st.step_timed(steps)
    n = st.node_count()
    bpl = L.gpu_bytes_per_lup(scheme, addr, prec)
    mflups = n * steps / (ms * 1e-3) / 1e6
    gbs = mflups * 1e6 * bpl / 1e9
    P = peak()
    rec = dict(config=tag, scheme=scheme, addressing=addr, layout=layout,
               dtype="f64" if prec == 8 else "f32", nodes=n, steps=steps,
               ms_per_step=ms / steps, mflups=round(mflups, 1), bytes_per_flup=bpl,
               gbs=round(gbs, 1), frac=round(gbs / P, 4),
               roofline_mflups=round(P * 1e9 / bpl / 1e6, 1),
               launches_per_step=st.launches_per_step())
    st.close()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=["c4", "c1", "c2", "c0"])
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--out", default=None)
    ap.add_argument("--schemes", default=None)
    ap.add_argument("--layouts", default="soa,aos")
    ap.add_argument("--precisions", default="8,4")
    args = ap.parse_args()

    if args.config == "c4":
        geo = L.GridGeometry(200, 200, 200)
        flow, init = L.bgk(1.0), "taylor_green"
        pairs = [(s, "direct") for s in SCHEMES] + [(s, "indirect") for s in IND + EXT]
    elif args.config == "c0":
        geo = L.GridGeometry(128, 128, 128)
        flow, init = L.bgk(1.0), "taylor_green"
        pairs = [("os-push", "direct"), ("os-pull", "direct")]
    elif args.config == "c1":
        geo = L.GridGeometry(256, 256, 256, ("periodic", "periodic", "wall"))
        flow, init = L.bgk(1.7, (1e-6, 0, 0)), "rest"
        pairs = [(s, "direct") for s in SCHEMES]
    else:
        geo = gen_random_spheres(256, 256, 256, 8.0, 0.40, seed=2011)
        flow, init = L.bgk(1.7, (1e-6, 0, 0)), "rest"
        pairs = [("os-pull", "indirect"), ("os-push", "indirect"), ("aap", "indirect"),
                 ("et", "indirect")]
    if args.schemes:
        keep = set(args.schemes.split(","))
        pairs = [p for p in pairs if p[0] in keep]
    out = open(args.out, "a") if args.out else None
    for scheme, addr in pairs:
        for layout in args.layouts.split(","):
            for prec in [int(p) for p in args.precisions.split(",")]:
                rec = run_one(geo, flow, scheme, addr, layout, prec, args.steps, args.warmup,
                              init, args.config)
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()


if __name__ == "__main__":
    main()
