import os, sys, json
sys.path.insert(0, "/root/repo")
import paper_1111_0922_b200 as L
for env in sys.argv[1:]:
    for kv in env.split(";"):
        if kv:
            k, v = kv.split("="); os.environ[k] = v
    for cfg in ("c1", "c4"):
        if cfg == "c1":
            geo = L.GridGeometry(256, 256, 256, ("periodic", "periodic", "wall")); flow = L.bgk(1.7, (1e-6, 0, 0))
        else:
            geo = L.GridGeometry(200, 200, 200); flow = L.bgk(1.0)
        for prec in (8, 4):
            st = L.create_stepper("swap-push", "direct", geo, flow, L.StepperOptions(precision=prec))
            st.init_field("rest"); st.step_n(4); st.synchronize()
            ms = st.step_timed(30) / 30
            n = st.node_count()
            print(json.dumps(dict(env=env, cfg=cfg, prec=prec, ms=round(ms, 4), frac=round(n * 38 * prec / ms / 1e6 / 6462.7, 3))), flush=True)
            st.close()
