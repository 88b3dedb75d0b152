"""CPU: the inputs of the full-size parity digests are pinned.

* the oracle's seeded Taylor-Green start (orc_init_field, also the device
  init) is equilibrium(rho, u) of the reference itself (p/src/collision.cpp:38-45,
  called through oracle/_ref) plus the documented noise, bit for bit;
* the starts the reference was run from (tests/golden/fullsize.json) are
  reproduced by the oracle at full size (C0 128^3, C4 200^3), and C2's
  porous mask by the geometry generator.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libref.so")
FULL = json.load(open(os.path.join(GOLDEN, "fullsize.json")))


def _splitmix_pm1(seed, stream):
    m = (1 << 64) - 1
    z = (seed + 0x9e3779b97f4a7c15 * (stream + 1)) & m
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & m
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & m
    z ^= z >> 31
    return float(z >> 11) * 2.0 ** -52 - 1.0


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
def test_taylor_green_is_reference_equilibrium_plus_noise():
    import oracle
    R, O = oracle.RefLib(), oracle.Oracle()
    dims, seed = (6, 5, 4), 2011
    f = O.init_field("taylor_green", dims, seed=seed).reshape(-1, 19)
    two_pi = 6.283185307179586476925286766559
    n = 0
    for z in range(dims[2]):
        for y in range(dims[1]):
            for x in range(dims[0]):
                cell = x + dims[0] * (y + dims[1] * z)
                X, Y, Z = (two_pi * x / dims[0], two_pi * y / dims[1], two_pi * z / dims[2])
                rho = 1.0 + 1e-3 * _splitmix_pm1(seed, cell * 20 + 19)
                u = [0.01 * math.sin(X) * math.cos(Y) * math.cos(Z),
                     -0.01 * math.cos(X) * math.sin(Y) * math.cos(Z), 0.0]
                for i in range(19):
                    want = R.L.ref_equilibrium(rho, np.array(u), i) + \
                        1e-4 * _splitmix_pm1(seed, cell * 20 + i)
                    assert f[n, i] == want, (x, y, z, i)
                n += 1


@pytest.mark.parametrize("name", ["c0", "c4"])
def test_fullsize_start_reproduced_by_oracle(name):
    import oracle
    e = FULL[name]
    f0 = oracle.Oracle().init_field(e["init"], tuple(e["dims"]), e["policy"], seed=e["seed"])
    assert hashlib.sha256(f0.tobytes()).hexdigest() == e["start_sha256"]


def test_fullsize_porous_mask_reproduced():
    from paper_1111_0922_b200.geometry import gen_random_spheres
    e = FULL["c2"]
    g = gen_random_spheres(*e["dims"])
    assert hashlib.sha256(g.mask.tobytes()).hexdigest() == e["mask_sha256"]
    assert g.fluid_count() == e["nodes"]


def test_fullsize_reference_runs_agree():
    """every reference scheme run per config gave the same digests"""
    for name, e in FULL.items():
        for r in e["reference_runs"]:
            assert r["sha256"] == e["sha256"], (name, r["scheme"])
        assert str(e["steps"]) in e["sha256"]
