#!/usr/bin/env python3
"""Phase breakdown of the AoS window kernels (experiments; needs a library
built with -DLBM_WIN_TRACE, e.g. tools/build_variant.sh trace -DLBM_WIN_TRACE):

    LBMGPU_LIBRARY=build/variants/trace/liblbmgpu.so python tools/win_trace.py [--prec 8]

Runs C1 (256^3 channel) AoS sweeps and prints, per scheme, the share of the
window blocks' cycles (thread 0, summed over blocks) in each phase of the
plane loop."""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1111_0922_b200 as L  # noqa: E402

PH = ["prologue", "barrier_prev", "issue_prefetch", "wait_plane", "compute", "barrier_compute",
      "writeback"]

ap = argparse.ArgumentParser()
ap.add_argument("--prec", type=int, default=8)
ap.add_argument("--schemes", default="aap,os-pull,et,os-push")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
fn = L._L.lbmgpu_debug_win_trace
fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
geo = L.GridGeometry(256, 256, 256, ("periodic", "periodic", "wall"))
flow = L.bgk(1.7, (1e-6, 0, 0))
for s in a.schemes.split(","):
    st = L.create_stepper(s, "direct", geo, flow, L.StepperOptions(layout="aos", precision=a.prec))
    st.step_n(4)
    st.synchronize()
    buf = (C.c_ulonglong * 16)()
    fn(buf, 1)
    ms = st.step_timed(a.steps)
    fn(buf, 1)
    tot = sum(buf[:7]) or 1
    rows = buf[12] or 1
    print(json.dumps({"scheme": s, "prec": a.prec, "ms_per_step": round(ms / a.steps, 4),
                      **{PH[k]: round(buf[k] / tot, 3) for k in range(7)},
                      "row_copies": rows,
                      "cyc_per_row": {n: round(buf[k] / rows, 1) for n, k in
                                      (("head_tail_cp_async", 8), ("cp_async_mbar_arrive", 9),
                                       ("arrive_tx", 10), ("bulk_issue", 11))}}), flush=True)
    st.close()
