"""CPU: LBMGEO1 geometry IO (p/src/geometry.cpp:123-171) — our writer
produces the reference's bytes, and the reader applies its checks/messages."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_case


def test_save_geo_matches_reference_bytes(tmp_path):
    import paper_1111_0922_b200 as L
    from paper_1111_0922_b200.geometry import save_geo
    z = load_case("idx")
    g = L.GridGeometry(16, 8, 8, ("periodic", "wall", "periodic"), z["seed42_mask"])
    p = tmp_path / "g.lbmgeo"
    save_geo(g, str(p))
    with open(os.path.join(GOLDEN, "seeded42.lbmgeo"), "rb") as fh:
        assert p.read_bytes() == fh.read()


def test_load_geo_round_trip_and_reference_file(tmp_path):
    from paper_1111_0922_b200.geometry import load_geo, save_geo
    g = load_geo(os.path.join(GOLDEN, "seeded42.lbmgeo"))
    z = load_case("idx")
    assert (g.nx, g.ny, g.nz) == (16, 8, 8)
    assert tuple(g.axis_policy) == ("periodic", "wall", "periodic")
    assert np.array_equal(g.mask, z["seed42_mask"])
    p = tmp_path / "rt.lbmgeo"
    save_geo(g, str(p))
    r = load_geo(str(p))
    assert np.array_equal(r.mask, g.mask) and tuple(r.axis_policy) == tuple(g.axis_policy)


def test_load_geo_errors(tmp_path):
    from paper_1111_0922_b200.geometry import load_geo
    with pytest.raises(RuntimeError, match="cannot open ./no_such_geometry_file.bin"):
        load_geo("./no_such_geometry_file.bin")
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTGEO!!garbage")
    with pytest.raises(RuntimeError, match="not a geometry file"):
        load_geo(str(bad))
    good = open(os.path.join(GOLDEN, "seeded42.lbmgeo"), "rb").read()
    cut = tmp_path / "cut.bin"
    cut.write_bytes(good[:-10])
    with pytest.raises(RuntimeError, match="short read"):
        load_geo(str(cut))
    zero = tmp_path / "zero.bin"
    zero.write_bytes(good[:8] + b"\0" * 12 + good[20:])
    with pytest.raises(RuntimeError, match="dimension overflow"):
        load_geo(str(zero))
