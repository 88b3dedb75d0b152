"""GPU parity at BASELINE.json's full sizes through size-independent
properties (the oracle is too slow there):

* cross-scheme bit equality — every scheme of the reference yields the same
  canonical state bit for bit (the reference's own equivalence property,
  p/src/bench.cpp:314-329); at full size a mismatch anywhere in 10^8 values
  shows up;
* IDX: full-size porous build_sparse bit-identical to the C oracle's, and
  reciprocal;
* multi-GPU decomposition: 8 z-slabs of config 3 bit-identical to one domain;
* conservation: total mass to 1e-12 (no sources);
* fp32 vs fp64 at config 4 after 200 steps within the 1e-5 tolerance.
"""
import numpy as np
import pytest

from conftest import bitwise_equal, max_rel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _run(L, scheme, addr, geo, flow, steps, init, layout="soa", precision=8, seed=2011):
    st = L.create_stepper(scheme, addr, geo, flow,
                          L.StepperOptions(layout=layout, precision=precision))
    if isinstance(init, np.ndarray):
        st.load_natural(init)
    else:
        st.init_field(init, seed=seed)
    st.step_n(steps)
    st.synchronize()
    out = st.extract_natural()
    st.close()
    return out


def test_config1_channel_all_schemes_bitwise(gpu):
    """C1: 256^3 channel, walls z, BGK 1.7, g = 1e-6 x; 40 steps from a
    perturbed start; AA / ET / OS push / OS pull / OSNT / TS / SWAP / CG, SoA,
    plus AA and ET AoS: one canonical state."""
    L = gpu
    geo = L.GridGeometry(256, 256, 256, ("periodic", "periodic", "wall"))
    flow = L.bgk(1.7, (1e-6, 0, 0))
    st = L.create_stepper("aap", "direct", geo, flow)
    st.init_field("taylor_green", seed=7, u0=0.02)
    f0 = st.extract_natural()
    st.close()
    want = _run(L, "aap", "direct", geo, flow, 40, f0)
    assert abs(want.sum() - f0.sum()) / f0.sum() <= 1e-12
    for scheme, layout in [("et", "soa"), ("os-pull", "soa"), ("os-push", "soa"),
                           ("osnt-pull-2s", "soa"), ("ts", "soa"), ("swap-push", "soa"),
                           ("cg", "soa"), ("aap", "aos"), ("et", "aos")]:
        got = _run(L, scheme, "direct", geo, flow, 40, f0, layout=layout)
        assert bitwise_equal(got, want), (scheme, layout, max_rel(got, want))


def test_config2_porous_idx_and_schemes(gpu):
    """C2: 256^3 box, random r=8 spheres to porosity 0.40 (N ~ 6.7 M): the
    GPU IDX equals the oracle's build_sparse bit for bit and is reciprocal;
    OS pull / AA / ET indirect and AA direct (masked) agree bitwise."""
    import oracle
    from paper_1111_0922_b200.geometry import gen_random_spheres
    L = gpu
    geo = gen_random_spheres(256, 256, 256, 8.0, 0.40, seed=2011)
    n, adj, node_of = L.build_sparse(geo, node_of=True)
    assert n == geo.fluid_count() and 0.39 < n / geo.cells() <= 0.40
    O = oracle.Oracle()
    want_adj, want_nof = O.build_sparse(256, 256, 256, [0, 0, 0], geo.mask)
    assert np.array_equal(adj, want_adj) and np.array_equal(node_of, want_nof)
    opp = [0, 2, 1, 4, 3, 6, 5, 18, 17, 16, 15, 14, 13, 12, 11, 10, 9, 8, 7]
    ids = np.arange(n, dtype=np.uint32)
    for i in range(1, 19):
        m = adj[:, i - 1]
        real = m != ids
        assert np.array_equal(adj[m[real], opp[i] - 1], ids[real])
    flow = L.bgk(1.7, (1e-6, 0, 0))
    want = _run(L, "os-pull", "indirect", geo, flow, 20, "random")
    for scheme, addr in [("aap", "indirect"), ("et", "indirect"), ("aap", "direct"),
                         ("os-push", "indirect")]:
        got = _run(L, scheme, addr, geo, flow, 20, "random")
        assert bitwise_equal(got, want), (scheme, addr, max_rel(got, want))


def test_config3_eight_slabs_bitwise_one_domain(gpu):
    """C3: 512x512x1024 periodic AA, Taylor-Green; 8 z-slabs (in-process
    transport, the NCCL plan) vs one 40.8 GB domain, at even and odd t."""
    L = gpu
    dims = (512, 512, 1024)
    flow = L.bgk(1.0)
    one = L.create_stepper("aap", "direct", L.GridGeometry(*dims), flow)
    one.init_field("taylor_green", seed=3)
    slabs = [L.create_stepper("aap", "direct", L.GridGeometry(*dims), flow,
                              L.StepperOptions(z_begin=k * 128, z_end=(k + 1) * 128))
             for k in range(8)]
    for s in slabs:
        s.init_field("taylor_green", seed=3)
    per = 512 * 512 * 128
    for steps in (4, 1):
        one.step_n(steps)
        one.synchronize()
        L.slab_group_step(slabs, steps)
        if one.time_step() % 2:
            L.slab_group_sync_ghosts(slabs)
        for k, s in enumerate(slabs):
            assert bitwise_equal(s.extract_natural(), one.extract_natural_range(k * per, per)), \
                (k, one.time_step())


def test_config4_fp32_within_tolerance(gpu):
    """C4: 200^3 periodic Taylor-Green, 200 steps: fp32 AA / OS pull / ET
    (SoA and AoS) within max relative 1e-5 of the fp64 result."""
    L = gpu
    geo = L.GridGeometry(200, 200, 200)
    flow = L.bgk(1.0)
    st = L.create_stepper("aap", "direct", geo, flow)
    st.init_field("taylor_green", seed=5)
    f0 = st.extract_natural()
    st.close()
    want = _run(L, "aap", "direct", geo, flow, 200, f0)
    for scheme, layout in [("aap", "soa"), ("os-pull", "soa"), ("et", "soa"), ("aap", "aos")]:
        got = _run(L, scheme, "direct", geo, flow, 200, f0, layout=layout, precision=4)
        assert max_rel(got, want) <= 1e-5, (scheme, layout, max_rel(got, want))
