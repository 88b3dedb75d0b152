#!/usr/bin/env python3
"""Run a few steps of one or more steppers so ncu can capture their kernels:

    ncu ... python tools/ncu_drive.py CONFIG SCHEME[,SCHEME..] ADDR LAYOUT PREC [STEPS]

CONFIG: c1 (256^3 channel), c2 (porous 256^3), c4 (200^3 periodic). Every
stepper is created, started (rest / Taylor-Green) and stepped STEPS times."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1111_0922_b200 as L  # noqa: E402


def main():
    cfg, schemes, addr, layout, prec = sys.argv[1:6]
    steps = int(sys.argv[6]) if len(sys.argv) > 6 else 4
    if cfg == "c1":
        geo, flow, init = L.GridGeometry(256, 256, 256, ("periodic", "periodic", "wall")), \
            L.bgk(1.7, (1e-6, 0, 0)), "rest"
    elif cfg == "c2":
        from paper_1111_0922_b200.geometry import gen_random_spheres
        geo, flow, init = gen_random_spheres(256, 256, 256), L.bgk(1.7, (1e-6, 0, 0)), "rest"
    else:
        geo, flow, init = L.GridGeometry(200, 200, 200), L.bgk(1.0), "taylor_green"
    for s in schemes.split(","):
        ext = addr == "indirect" and s in ("ts", "swap-push", "swap-pull")
        st = L.create_stepper(s, addr, geo, flow, L.StepperOptions(layout=layout,
                                                                   precision=int(prec),
                                                                   extensions=ext))
        st.init_field(init, seed=2011)
        st.step_n(steps)
        st.synchronize()
        st.close()


if __name__ == "__main__":
    main()
