"""CPU: the C-ABI library loads, exports every entry point include/lbmgpu.h
declares, and its host-side logic (no GPU needed) matches the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_case


def _declared():
    txt = open(os.path.join(ROOT, "include", "lbmgpu.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|double|const char\*)\s+(lbmgpu_\w+)\s*\(",
                                 txt, re.M)))


def test_library_exports_every_declared_symbol(lbm):
    names = _declared()
    assert len(names) >= 30
    # RTLD_NOW: every symbol the library references must resolve at load time
    lib = ctypes.CDLL(lbm.LIBRARY_PATH, mode=os.RTLD_NOW | os.RTLD_LOCAL)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_native():
    """the fatbin carries sm_100a SASS (cuobjdump lists the cubin arch)"""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_1111_0922_b200",
                                                                 "liblbmgpu.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_traffic_matches_reference_table(lbm):
    z = load_case("collision_traffic")
    rows = []
    for fam in lbm.FAMILIES:
        for a in ("direct", "indirect"):
            cnt, b = lbm.traffic(fam, a)
            rows.append([cnt[0], cnt[1], cnt[2], cnt[3], cnt[4], cnt[5], b])
    assert np.array_equal(np.array(rows, float), z["traffic"])
    # fp32 halves the PDF bytes
    assert lbm.traffic("aap", "direct", 4)[1] == 152
    assert lbm.gpu_bytes_per_lup("aap", "direct") == 304
    assert lbm.gpu_bytes_per_lup("aap", "indirect") == 340
    assert lbm.gpu_bytes_per_lup("os-pull", "indirect") == 376
    assert lbm.gpu_bytes_per_lup("ts", "direct") == 608
    assert lbm.gpu_bytes_per_lup("aap", "indirect", 4) == 188


def test_kernel_availability_matrix(lbm):
    """p/src/stepper.cpp:140-153: 10 direct + 6 indirect"""
    n = sum(lbm.kernel_available(s, a) for s in lbm.SCHEMES for a in lbm.ADDRESSINGS)
    assert n == 16
    for s in ("ts", "cg", "swap-push", "swap-pull"):
        assert not lbm.kernel_available(s, "indirect")
    assert lbm.kernel_available("ts", "indirect", extensions=True)
    assert not lbm.kernel_available("cg", "indirect", extensions=True)


def test_lambda_odd_and_bgk(lbm):
    z = load_case("collision_traffic")
    assert lbm.lambda_odd(lbm.FlowParams()) == float(z["lambda_odd_default"])
    assert lbm.bgk(1.7).magic_lambda == (1 / 1.7 - 0.5) ** 2
    assert lbm.lambda_odd(lbm.bgk(1.0)) == 1.0


def test_argument_errors_before_device_access(lbm):
    g = lbm.gen_channel(4, 4, 4)
    with pytest.raises(ValueError, match="kernel not implemented; traffic model only"):
        lbm.create_stepper("cg", "indirect", g)
    with pytest.raises(ValueError, match="workers must be >= 0"):
        lbm.create_stepper("aap", "direct", g, options=lbm.StepperOptions(workers=-1))
    with pytest.raises(ValueError, match="chunk_length must be >= 1"):
        lbm.create_stepper("osnt-pull-2s", "direct", g,
                           options=lbm.StepperOptions(chunk_length=0))
    with pytest.raises(ValueError, match="unknown scheme"):
        lbm.create_stepper("warp", "direct", g)
    with pytest.raises(ValueError, match="zero dimension"):
        lbm.gen_channel(0, 4, 4)


def test_geometry_generators():
    from paper_1111_0922_b200.geometry import gen_packed_bed, gen_random_spheres
    # frozen count of the reference's calibrated bed (p/tests/test_geometry.cpp:100-105)
    assert gen_packed_bed(500, 100, 100, 4.65, 9.0).fluid_count() == 2103037
    assert gen_packed_bed(8, 8, 8, 0.0, 10.0).fluid_count() == 512
    with pytest.raises(ValueError, match="overlapping spheres"):
        gen_packed_bed(8, 8, 8, 11.0, 10.0)
    g = gen_random_spheres(48, 40, 32, radius=4.0, porosity=0.4, seed=5)
    phi = g.fluid_count() / g.cells()
    assert 0.37 < phi <= 0.40
    g2 = gen_random_spheres(48, 40, 32, radius=4.0, porosity=0.4, seed=5)
    assert np.array_equal(g.mask, g2.mask)
