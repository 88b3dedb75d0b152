#!/usr/bin/env python3
"""Drive every direct scheme on C1 (256^3 channel) for a few steps so that one
ncu pass can record each kernel's DRAM bytes and time (run under ncu):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --clock-control none --csv --log-file gpurun_out/schemes.csv \\
        python tools/ncu_schemes.py [soa|aos] [scheme,scheme,...] [8|4]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1111_0922_b200 as L  # noqa: E402

SCHEMES = ["ts", "os-push", "os-pull", "osnt-pull-1s", "cg", "swap-push", "aap", "et"]


def main():
    layout = sys.argv[1] if len(sys.argv) > 1 else "soa"
    schemes = sys.argv[2].split(",") if len(sys.argv) > 2 else SCHEMES
    prec = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    geo = L.GridGeometry(256, 256, 256, ("periodic", "periodic", "wall"))
    flow = L.bgk(1.7, (1e-6, 0.0, 0.0))
    for s in schemes:
        st = L.create_stepper(s, "direct", geo, flow,
                              L.StepperOptions(layout=layout, precision=prec))
        st.init_field("rest")
        st.step_n(4)
        st.synchronize()
        st.close()


if __name__ == "__main__":
    main()
