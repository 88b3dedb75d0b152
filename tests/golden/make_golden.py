"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the development container (needs oracle/_ref/libref.so, i.e. the
unmodified reference compiled from /root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Every array below is produced by the reference library's own public API
(create_stepper / load_natural / step / extract_natural / build_sparse /
TrtOperator::collide / traffic / verify_suite) through oracle/ref_capi.cpp.
The GPU box has no /root/reference; the tests read these committed files.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

R = oracle.RefLib()
O = oracle.Oracle()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ts_run(dims, policy, mask, le, magic, g, f0, steps, record=()):
    st = R.create("ts", 0, dims, policy, mask, le, magic, g)
    st.load(f0)
    out = {}
    for t in range(1, steps + 1):
        st.step(1)
        if t in record or t == steps:
            out[t] = st.extract()
    return out


def main():
    cases = {}

    # (1) the reference's own equivalence setting: make_seeded_geometry(42),
    # default FlowParams (TRT, lambda_e = 1/0.9, magic 3/16, g = 1e-5 x),
    # random_field(4242) (p/tests/test_schemes.cpp:145-183)
    dims, pol, mask = R.make_seeded_geometry(42)
    n = int(mask.sum())
    f0 = O.random_field(4242, n)
    res = ts_run(dims, pol, mask, 1 / 0.9, 3 / 16, [1e-5, 0, 0], f0, 10, record=(1, 2, 3))
    cases["seeded42"] = dict(dims=dims, policy=pol, mask=mask, lambda_even=1 / 0.9,
                             magic=3 / 16, force=[1e-5, 0, 0], f0=f0, steps=10,
                             f1=res[1], f2=res[2], f3=res[3], f10=res[10])

    # (2) config-1 miniature: channel periodic x/y, walls z, BGK omega=1.7,
    # g = 1e-6 x, rest start (f_i = w_i), 24 steps (even count)
    dims = (16, 12, 10)
    pol = np.array([0, 0, 1], np.uint8)
    st = R.create("aap", 0, dims, pol, None, 1.7, (1 / 1.7 - 0.5) ** 2, [1e-6, 0, 0])
    f0 = st.extract()
    res = ts_run(dims, pol, None, 1.7, (1 / 1.7 - 0.5) ** 2, [1e-6, 0, 0], f0, 24, record=(1,))
    cases["channel_c1"] = dict(dims=dims, policy=pol, mask=np.ones(np.prod(dims), np.uint8),
                               lambda_even=1.7, magic=(1 / 1.7 - 0.5) ** 2,
                               force=[1e-6, 0, 0], f0=f0, steps=24, f1=res[1], f24=res[24])

    # (3) config-0 miniature: fully periodic 12x10x8, BGK omega = 1 (magic 1/4),
    # g = 0, seeded random start, 16 steps
    dims = (12, 10, 8)
    pol = np.array([0, 0, 0], np.uint8)
    f0 = O.random_field(777, int(np.prod(dims)))
    res = ts_run(dims, pol, None, 1.0, 0.25, [0, 0, 0], f0, 16, record=(1,))
    cases["periodic_c0"] = dict(dims=dims, policy=pol, mask=np.ones(np.prod(dims), np.uint8),
                                lambda_even=1.0, magic=0.25, force=[0, 0, 0], f0=f0,
                                steps=16, f1=res[1], f16=res[16])

    # (4) porous miniature: 20x16x12 all-periodic box with seeded random solid
    # spheres (config-2 shape), g = 1e-6 x, omega = 1.7, 12 steps
    dims = (20, 16, 12)
    pol = np.array([0, 0, 0], np.uint8)
    rng = np.random.default_rng(2024)
    X, Y, Z = np.meshgrid(np.arange(dims[0]), np.arange(dims[1]), np.arange(dims[2]),
                          indexing="ij")
    solid = np.zeros(dims, bool)
    for _ in range(6):
        c = rng.uniform(0, dims)
        d2 = sum(np.minimum(np.abs(a - ci), dims[k] - np.abs(a - ci)) ** 2
                 for k, (a, ci) in enumerate(zip((X + 0.5, Y + 0.5, Z + 0.5), c)))
        solid |= d2 < 3.0 ** 2
    mask = (~solid).transpose(2, 1, 0).ravel().astype(np.uint8)  # x-fastest
    n = int(mask.sum())
    f0 = O.random_field(99, n)
    res = ts_run(dims, pol, mask, 1.7, (1 / 1.7 - 0.5) ** 2, [1e-6, 0, 0], f0, 12, record=(1,))
    cases["porous_c2"] = dict(dims=dims, policy=pol, mask=mask, lambda_even=1.7,
                              magic=(1 / 1.7 - 0.5) ** 2, force=[1e-6, 0, 0], f0=f0, steps=12,
                              f1=res[1], f12=res[12])

    # (5) closed box (all walls) for conservation (p/tests/test_schemes.cpp:416-436)
    dims = (8, 8, 8)
    pol = np.array([1, 1, 1], np.uint8)
    f0 = O.random_field(88, 512)
    res = ts_run(dims, pol, None, 1 / 0.9, 3 / 16, [0, 0, 0], f0, 20, record=(1,))
    cases["closed_box"] = dict(dims=dims, policy=pol, mask=np.ones(512, np.uint8),
                               lambda_even=1 / 0.9, magic=3 / 16, force=[0, 0, 0], f0=f0,
                               steps=20, f1=res[1], f20=res[20])

    for name, c in cases.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                            **{k: np.asarray(v) for k, v in c.items()})

    # IDX: build_sparse on seeded masks (p/tests/test_geometry.cpp:16-27 shape)
    idx = {}
    for seed in (1, 42, 1234):
        dims, pol, mask = R.make_seeded_geometry(seed)
        adj, node_of = R.build_sparse(*dims, pol, mask)
        idx[f"seed{seed}_mask"] = mask
        idx[f"seed{seed}_adjacency"] = adj
        idx[f"seed{seed}_node_of"] = node_of
    d = cases["porous_c2"]
    adj, node_of = R.build_sparse(*d["dims"], d["policy"], d["mask"])
    idx["porous_adjacency"] = adj
    idx["porous_node_of"] = node_of
    rem, nmail = O.et_rem(adj)
    idx["porous_et_rem"] = rem
    idx["porous_et_mail"] = np.array(nmail)
    np.savez_compressed(os.path.join(HERE, "idx.npz"), **idx)

    # collision known answers (TrtOperator::collide on 64 seeded nodes)
    f = O.random_field(7, 64)
    col = dict(f_in=f,
               trt=R.collide(f, 1 / 0.9, R.L.ref_lambda_odd(1 / 0.9, 3 / 16), [1e-4, -2e-4, 3e-4]),
               bgk17=R.collide(f, 1.7, 1.7, [1e-6, 0, 0]),
               bgk10=R.collide(f, 1.0, 1.0, [0, 0, 0]),
               zero=R.collide(f, 0.0, 0.0, [0, 0, 0]),
               lambda_odd_default=np.array(R.L.ref_lambda_odd(1 / 0.9, 3 / 16)),
               flops=np.array(R.L.ref_flops_per_update()))
    c, w, o = R.stencil()
    col.update(c=c, w=w, opposite=o)
    tr = np.array([[*R.traffic(fam, a)[0], R.traffic(fam, a)[1]] for fam in range(7)
                   for a in range(2)])
    col["traffic"] = tr
    ids, mr, ap = R.verify_suite(42, 10)
    col["verify_ids"] = ids
    col["verify_max_rel"] = mr
    np.savez_compressed(os.path.join(HERE, "collision_traffic.npz"), **col)

    # LBMGEO1 file written by the reference's save_geo (p/src/geometry.cpp:123-135)
    dims, pol, mask = R.make_seeded_geometry(42)
    R.save_geo(dims, pol, mask, os.path.join(HERE, "seeded42.lbmgeo"))

    with open(os.path.join(HERE, "SHA256SUMS"), "w") as fh:
        for name in sorted(os.listdir(HERE)):
            if name.endswith(".npz"):
                with np.load(os.path.join(HERE, name)) as z:
                    for k in sorted(z.files):
                        fh.write(f"{name}:{k} {sha(z[k])}\n")
        with open(os.path.join(HERE, "seeded42.lbmgeo"), "rb") as g:
            fh.write(f"seeded42.lbmgeo:bytes {hashlib.sha256(g.read()).hexdigest()}\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
