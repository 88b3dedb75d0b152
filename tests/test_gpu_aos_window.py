"""GPU: the AoS window kernels (kernels_aos.cu: 32x8 tiles marching through
z chunks with a shared-memory plane ring) against the SoA kernels of the same
scheme and against the oracle's two-step stepper (SWAP's link exchange and
CG's plane groups run through the same windows). Sizes are chosen so the
in-place AA / SWAP windows apply (periodic nx >= 34, ny >= 10) and tiles are
partial in x and y, with walls, solids and several z chunks; fp64 and fp32
must both be bit-identical to SoA (same arithmetic, different data path)."""
import numpy as np
import pytest

from conftest import bitwise_equal

pytestmark = pytest.mark.gpu

WINDOW_SCHEMES = ["ts", "os-push", "os-pull", "osnt-pull-1s", "aap", "swap-push", "swap-pull", "cg",
                  "et"]
GEOMS = {
    "periodic": ((40, 12, 10), ("periodic", "periodic", "periodic"), None),
    "channel_z": ((45, 17, 11), ("periodic", "periodic", "wall"), None),
    "walls_xy": ((36, 10, 9), ("wall", "wall", "periodic"), None),
    "porous": ((41, 13, 12), ("periodic", "periodic", "periodic"), 0.2),
    "tall": ((35, 10, 70), ("periodic", "periodic", "periodic"), None),
}


def _geo(L, name):
    dims, pol, solid = GEOMS[name]
    mask = None
    if solid:
        rng = np.random.default_rng(7)
        mask = (rng.random(dims[0] * dims[1] * dims[2]) >= solid).astype(np.uint8)
    return L.GridGeometry(*dims, pol, mask)


@pytest.mark.parametrize("precision", [8, 4])
@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("scheme", WINDOW_SCHEMES)
def test_aos_window_equals_soa(gpu, scheme, geom, precision):
    L = gpu
    geo = _geo(L, geom)
    flow = L.FlowParams(1.0 / 0.8, 3.0 / 16.0, (2e-5, -1e-5, 5e-6), 1.0)
    st = {lay: L.create_stepper(scheme, "direct", geo, flow,
                                L.StepperOptions(layout=lay, precision=precision))
          for lay in ("soa", "aos")}
    for s in st.values():
        s.init_field("random", seed=5)
    for steps in (1, 2, 4):  # t = 1 (odd), 3, 7
        for s in st.values():
            s.step_n(steps)
            s.synchronize()
        a, b = st["soa"].extract_natural(), st["aos"].extract_natural()
        assert bitwise_equal(a, b), (scheme, geom, precision, st["soa"].time_step())


@pytest.mark.parametrize("geom", ["channel_z", "porous"])
@pytest.mark.parametrize("scheme", WINDOW_SCHEMES)
def test_aos_window_matches_oracle(gpu, scheme, geom):
    import oracle
    L = gpu
    geo = _geo(L, geom)
    nx, ny, nz = geo.nx, geo.ny, geo.nz
    pol = [1 if p == "wall" else 0 for p in geo.axis_policy]
    g = (2e-5, -1e-5, 5e-6)
    O = oracle.Oracle()
    f0 = O.random_field(99, geo.fluid_count())
    # BGK omega = 1.7: lambda_odd == lambda_even exactly (L.bgk checks it)
    st = L.create_stepper(scheme, "direct", geo, L.bgk(1.7, g), L.StepperOptions(layout="aos"))
    le = lo = 1.7
    st.load_natural(f0)
    st.step_n(5)
    st.synchronize()
    want = O.ts_run(nx, ny, nz, pol, geo.mask, le, lo, g, f0, 5)
    assert bitwise_equal(st.extract_natural(), want)


def test_aos_window_large_c4_shape(gpu):
    """C4's 200^3 shape class (partial x tile of 8, 25 y tiles, many z
    chunks) at 200x40x48: AoS AA/OS pull/OS push equal SoA after an odd and
    an even step count."""
    L = gpu
    geo = L.GridGeometry(200, 40, 48)
    for scheme in ("aap", "os-pull", "os-push", "et"):
        st = {lay: L.create_stepper(scheme, "direct", geo, L.bgk(1.0),
                                    L.StepperOptions(layout=lay)) for lay in ("soa", "aos")}
        for s in st.values():
            s.init_field("taylor_green", seed=3, u0=0.05)
        for steps in (3, 3):
            for s in st.values():
                s.step_n(steps)
                s.synchronize()
            assert bitwise_equal(st["soa"].extract_natural(), st["aos"].extract_natural()), scheme


@pytest.mark.parametrize("geom", ["periodic", "walls_xy"])
def test_aos_window_swap_deferred_fixup(gpu, geom):
    """SWAP push with deferred seam fix-ups (p/src/scheme_swap.cpp:86-95): the
    window exchanges the non-wrapped links, the pending list the seam links;
    extraction in between (swap_partial phase) equals SoA bit for bit"""
    L = gpu
    geo = _geo(L, geom)
    flow = L.bgk(1.7, (1e-5, 0.0, 2e-6))
    st = {lay: L.create_stepper("swap-push", "direct", geo, flow,
                                L.StepperOptions(layout=lay, swap_deferred_fixup=True))
          for lay in ("soa", "aos")}
    for s in st.values():
        s.init_field("random", seed=12)
    for steps in (1, 2, 3):
        for s in st.values():
            s.step_n(steps)
            s.synchronize()
        assert st["soa"].layout_phase() == st["aos"].layout_phase()
        assert bitwise_equal(st["soa"].extract_natural(), st["aos"].extract_natural()), steps


@pytest.mark.parametrize("zchunk", [5, 9, 23])
@pytest.mark.parametrize("precision", [8, 4])
@pytest.mark.parametrize("scheme", WINDOW_SCHEMES)
def test_aos_window_long_z_chunks(gpu, monkeypatch, scheme, precision, zchunk):
    """z chunks longer than the plane ring (the ring slots and their barrier
    phases wrap several times per block) on a box small enough to compare."""
    L = gpu
    monkeypatch.setenv("LBMGPU_AOS_ZCHUNK", str(zchunk))
    geo = L.GridGeometry(40, 14, 48, ("periodic", "periodic", "periodic"))
    flow = L.FlowParams(1.0 / 0.8, 3.0 / 16.0, (2e-5, -1e-5, 5e-6), 1.0)
    st = {lay: L.create_stepper(scheme, "direct", geo, flow,
                                L.StepperOptions(layout=lay, precision=precision))
          for lay in ("soa", "aos")}
    for s in st.values():
        s.init_field("random", seed=9)
    for steps in (1, 2):
        for s in st.values():
            s.step_n(steps)
            s.synchronize()
        assert bitwise_equal(st["soa"].extract_natural(), st["aos"].extract_natural()), \
            (scheme, precision, zchunk, st["soa"].time_step())
