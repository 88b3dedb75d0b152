"""scratch: C2 porous indirect stepping for ncu"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_0922_b200 as L
from paper_1111_0922_b200.geometry import gen_random_spheres
geo = gen_random_spheres(256, 256, 256, 8.0, 0.40, seed=2011)
scheme = sys.argv[1] if len(sys.argv) > 1 else "aap"
st = L.create_stepper(scheme, "indirect", geo, L.bgk(1.7, (1e-6, 0, 0)), L.StepperOptions(precision=8))
st.init_field("rest"); st.step_n(6); st.synchronize()
ms = st.step_timed(20) / 20
print(scheme, "ms/step", ms, "MFLUP/s", st.node_count() / ms / 1e3)
