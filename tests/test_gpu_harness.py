"""GPU harness (p/src/bench.cpp, p/tests/acceptance.cpp) on the B200:
verify_suite, run_bench + CSV columns, and the acceptance gate's physics
criterion 5 (force-driven channel reaches the analytic Poiseuille profile with
the walls half a link beyond the outermost nodes, rel Linf <= 1e-6)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_verify_suite_matches_reference_shape(gpu):
    """verify_suite(42, 10): 15 pairs, all bitwise (p/tests/test_bench.cpp:52-65)"""
    ents, ok = gpu.verify_suite(42, 10)
    assert ok and len(ents) == 15
    assert all(e.bitwise and e.max_rel_linf == 0.0 for e in ents)


def test_verify_suite_all_layouts_and_precisions(gpu):
    ents, ok = gpu.verify_suite(7, 6, all_variants=True)
    assert ok and len(ents) == 16 * 4 - 1
    for e in ents:
        if e.dtype == "f64":
            assert e.bitwise, e
        else:
            assert e.max_rel_linf <= 1e-5, e


def test_run_bench_record_and_csv(gpu):
    """run_bench record fields (p/tests/test_bench.cpp:67-103)"""
    L = gpu
    g = L.gen_channel(64, 32, 32)
    r = L.run_bench("aap", "direct", g, L.FlowParams(), steps=20, warmup=2, timed_runs=3,
                    hbm_gbs=6552.3, geometry_name="channel:64x32x32")
    assert r.fluid_count == 64 * 32 * 32 and r.steps == 20
    assert r.seconds > 0 and r.mlups > 0
    assert r.bytes_per_lup == 304 and r.gpu_bytes_per_lup == 304
    assert abs(r.predicted_mlups - 6552.3e3 / 304) < 1e-6
    assert not r.model_violated
    csv = L.to_csv([r])
    assert csv.splitlines()[0] == L.CSV_COLUMNS
    assert csv.splitlines()[1].startswith("aap,direct,soa,f64,channel:64x32x32,65536,20,")
    with pytest.raises(ValueError, match="steps must be at least 1"):
        L.run_bench("aap", "direct", g, steps=0)


@pytest.mark.parametrize("scheme,addr", [("aap", "direct"), ("et", "indirect"),
                                         ("os-pull", "direct")])
def test_poiseuille_acceptance_criterion_5(gpu, scheme, addr):
    """p/tests/acceptance.cpp:173-230: 16x32x4, walls in y, TRT defaults
    (tau 0.9, magic 3/16, g = 1e-5 x); run to a steady y-profile (change
    < 1e-12); compare u_x with g/(2 nu) (h^2/4 - yc^2), h = ny."""
    L = gpu
    g = L.GridGeometry(16, 32, 4, ("periodic", "wall", "periodic"))
    p = L.FlowParams()
    st = L.create_stepper(scheme, addr, g, p)

    def profile():
        _, u = L.macroscopic_fields(st, p)
        return u[:, 0].reshape(4, 32, 16).mean(axis=(0, 2))

    prev = profile()
    change = 1.0
    for _ in range(400):
        st.step_n(500)  # even: AA ends in natural layout
        cur = profile()
        change = np.max(np.abs(cur - prev)) / np.max(np.abs(cur))
        prev = cur
        if change < 1e-12:
            break
    assert change < 1e-12
    nu = (1.0 / p.lambda_even - 0.5) / 3.0
    h = 32.0
    yc = np.arange(32) + 0.5 - h / 2
    ana = p.body_force[0] / (2 * nu) * (h * h / 4 - yc * yc)
    assert np.max(np.abs(prev - ana)) / np.max(np.abs(ana)) <= 1e-6


def test_shared_reciprocal_division_is_ddiv_rn(gpu):
    """the collision's three divisions by rho share one reciprocal
    (dev::rcp_prep / div_by, fp64 and fp32); bit patterns must equal
    __ddiv_rn's / __fdiv_rn's on 2^26 seeded inputs incl. signed zeros,
    denormals, infinities and NaNs"""
    assert gpu.selftest_division(1 << 26, seed=20251019) == 0


def test_macroscopic_fields_vacuum_node(gpu):
    """moments' std::domain_error("vacuum node") (p/src/collision.cpp:31) as
    DomainError, through the Python mirror's macroscopic_fields."""
    L = gpu
    st = L.create_stepper("aap", "direct", L.GridGeometry(8, 6, 4), L.bgk(1.0))
    f = st.extract_natural().reshape(-1, 19)
    f[2] = 0.0
    st.load_natural(f.ravel())
    with pytest.raises(L.DomainError, match="vacuum node"):
        L.macroscopic_fields(st, L.bgk(1.0))
