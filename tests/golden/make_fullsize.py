"""Full-size parity digests of the BASELINE configurations, made by the REFERENCE.

Run in the development container (needs oracle/_ref/libref.so, the unmodified
reference compiled from /root/reference by oracle/Makefile); takes about an
hour on 8 cores:

    python tests/golden/make_fullsize.py [c0 c1 c2 c4]

For every config the reference's own public API runs the BASELINE.json size
and step count: create_stepper (p/src/stepper.cpp:155-180) -> load_natural ->
step() x steps -> extract_natural (p/include/lbmlab/stepper.hpp:70-106), with
workers = 0 (all host threads, p/src/stepper.cpp:197-205). Several reference
schemes run per config and must agree bit for bit (the reference's own
equivalence contract, p/src/bench.cpp:314-329, p/tests/acceptance.cpp:128-136).

Written (the GPU box has no /root/reference; tests/test_gpu_fullsize_parity.py
reads these):
  fullsize.json          per config: inputs, the SHA-256 of the canonical start
                         snapshot, of the final one and of a few intermediate
                         ones (odd t included), the sample stride
  fullsize_<cfg>.npy     the final snapshot's values [::1009] (fp32 checks)

Inputs: C0/C4 start from the seeded Taylor-Green field of DESIGN.md section 8
(oracle orc_init_field, also the product's device init); C1/C2 from rest
(f_i = w_i, the reference's default start). C2's mask is
paper_1111_0922_b200.geometry.gen_random_spheres(256, 256, 256) (its SHA-256 is
recorded, so the GPU side checks it uses the same medium).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

STRIDE = 1009
SEED = 2011

# name -> BASELINE.json configs[k] at full size and step count
CONFIGS = {
    "c0": dict(dims=(128, 128, 128), policy=(0, 0, 0), omega=1.0, force=(0.0, 0.0, 0.0),
               init="taylor_green", steps=100, record=(1, 99),
               runs=[("os-push", 0), ("os-pull", 0)]),
    "c1": dict(dims=(256, 256, 256), policy=(0, 0, 1), omega=1.7, force=(1e-6, 0.0, 0.0),
               init="rest", steps=1000, record=(1, 999),
               runs=[("aap", 0), ("et", 0), ("os-pull", 0)]),
    "c2": dict(dims=(256, 256, 256), policy=(0, 0, 0), omega=1.7, force=(1e-6, 0.0, 0.0),
               init="rest", steps=500, record=(1, 499), porous=True,
               runs=[("os-pull", 1), ("aap", 1), ("os-push", 1)]),
    "c4": dict(dims=(200, 200, 200), policy=(0, 0, 0), omega=1.0, force=(0.0, 0.0, 0.0),
               init="taylor_green", steps=200, record=(1, 199),
               runs=[("aap", 0), ("os-pull", 0), ("et", 1)]),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def magic_for(omega: float) -> float:
    # BGK as TRT with lambda_odd == lambda_even
    return (1.0 / omega - 0.5) ** 2


def main(names):
    R = oracle.RefLib()
    O = oracle.Oracle()
    path = os.path.join(HERE, "fullsize.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        cfg = CONFIGS[name]
        dims, pol = cfg["dims"], np.array(cfg["policy"], np.uint8)
        mask = None
        entry = dict(dims=list(dims), policy=list(cfg["policy"]), omega=cfg["omega"],
                     magic=magic_for(cfg["omega"]), force=list(cfg["force"]),
                     init=cfg["init"], seed=SEED, steps=cfg["steps"], stride=STRIDE)
        if cfg.get("porous"):
            from paper_1111_0922_b200.geometry import gen_random_spheres
            mask = gen_random_spheres(*dims).mask
            entry["mask_sha256"] = hashlib.sha256(mask.tobytes()).hexdigest()
        f0 = O.init_field(cfg["init"], dims, pol, mask, seed=SEED)
        entry["nodes"] = f0.size // 19
        entry["start_sha256"] = sha(f0)
        recs = []
        for scheme, addr in cfg["runs"]:
            t0 = time.time()
            st = R.create(scheme, addr, dims, pol, mask, cfg["omega"], magic_for(cfg["omega"]),
                          cfg["force"], workers=0)
            st.load(f0)
            digests, t = {}, 0
            for tr in sorted(cfg["record"]) + [cfg["steps"]]:
                st.step(tr - t)
                t = tr
                f = st.extract()
                digests[str(t)] = sha(f)
            recs.append(dict(scheme=scheme, addressing=["direct", "indirect"][addr],
                             sha256=digests, seconds=round(time.time() - t0, 1)))
            print(f"{name} {scheme}/{addr}: {digests} ({time.time() - t0:.0f} s)", flush=True)
            del st
        first = recs[0]["sha256"]
        for r in recs[1:]:
            if r["sha256"] != first:
                raise SystemExit(f"{name}: reference schemes disagree: {recs}")
        entry["sha256"] = first
        entry["reference_runs"] = recs
        np.save(os.path.join(HERE, f"fullsize_{name}.npy"), f[::STRIDE].copy())
        out[name] = entry
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:] or ["c0", "c4", "c2", "c1"]))
