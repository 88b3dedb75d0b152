"""GPU parity: every (scheme, addressing, layout, precision) of liblbmgpu.so,
driven through the C ABI (paper_1111_0922_b200 -> include/lbmgpu.h), against
the reference's own results (tests/golden/, made by make_golden.py from the
compiled reference) and against the C oracle at larger sizes.

Bar: fp64 bit-for-bit (memcmp), like the reference's cross-scheme check
(p/src/bench.cpp:314-329); fp32 max relative error <= 1e-5 (north_star).
"""
import numpy as np
import pytest

from conftest import bitwise_equal, load_case, max_rel

pytestmark = pytest.mark.gpu

SCHEMES = ["ts", "os-push", "os-pull", "osnt-pull-1s", "osnt-pull-2s", "cg", "swap-push",
           "swap-pull", "aap", "et"]
PAIRS = [(s, "direct") for s in SCHEMES] + [
    (s, "indirect") for s in ["os-push", "os-pull", "osnt-pull-1s", "osnt-pull-2s", "aap", "et"]]
EXT_PAIRS = [("ts", "indirect"), ("swap-push", "indirect"), ("swap-pull", "indirect")]
CASES = ["seeded42", "channel_c1", "periodic_c0", "porous_c2", "closed_box"]
FP32_TOL = 1e-5


def geometry(L, c):
    pol = ["wall" if p else "periodic" for p in c["policy"]]
    mask = c["mask"] if not c["mask"].all() else None
    return L.GridGeometry(*[int(v) for v in c["dims"]], pol, mask)


def make(L, c, scheme, addr, layout="soa", precision=8, **kw):
    flow = L.FlowParams(float(c["lambda_even"]), float(c["magic"]), tuple(c["force"]), 1.0)
    opts = L.StepperOptions(layout=layout, precision=precision,
                            extensions=(scheme, addr) in EXT_PAIRS, **kw)
    return L.create_stepper(scheme, addr, geometry(L, c), flow, opts)


def check(got, want, precision):
    if precision == 8:
        assert bitwise_equal(got, want), f"max rel {max_rel(got, want):.3e}"
    else:
        assert max_rel(got, want) <= FP32_TOL


@pytest.mark.parametrize("precision", [8, 4])
@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("scheme,addr", PAIRS + EXT_PAIRS)
@pytest.mark.parametrize("case", CASES)
def test_scheme_matches_reference(gpu, case, scheme, addr, layout, precision):
    c = load_case(case)
    st = make(gpu, c, scheme, addr, layout, precision)
    assert st.node_count() == c["f0"].size // 19
    st.load_natural(c["f0"])
    assert st.time_step() == 0
    st.step()
    check(st.extract_natural(), c["f1"], precision)
    steps = int(c["steps"])
    st.step_n(steps - 1)
    st.synchronize()
    assert st.time_step() == steps
    check(st.extract_natural(), c[f"f{steps}"], precision)


@pytest.mark.parametrize("scheme,addr", PAIRS)
def test_every_step_tracks_reference_seeded42(gpu, scheme, addr):
    """the reference's equivalence test: extract after EVERY step
    (p/tests/test_schemes.cpp:145-183) — here against steps 1,2,3,10."""
    c = load_case("seeded42")
    st = make(gpu, c, scheme, addr)
    st.load_natural(c["f0"])
    for t in range(1, 11):
        st.step()
        if f"f{t}" in c:
            assert bitwise_equal(st.extract_natural(), c[f"f{t}"]), t


@pytest.mark.parametrize("scheme,addr", PAIRS + EXT_PAIRS)
def test_load_then_extract_is_identity(gpu, scheme, addr):
    """p/tests/test_schemes.cpp:210-224"""
    c = load_case("seeded42")
    st = make(gpu, c, scheme, addr)
    st.step()
    st.load_natural(c["f0"])
    assert st.time_step() == 0
    assert bitwise_equal(st.extract_natural(), c["f0"])


@pytest.mark.parametrize("scheme,addr", PAIRS + EXT_PAIRS)
def test_equilibrium_start_agrees(gpu, scheme, addr):
    """p/tests/test_schemes.cpp:185-208: the default start is w_i*rho0"""
    c = load_case("seeded42")
    st = make(gpu, c, scheme, addr)
    n = st.node_count()
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    assert bitwise_equal(st.extract_natural(), np.tile(w, n))


def test_pure_streaming_is_a_permutation(gpu):
    """p/tests/test_schemes.cpp:226-245"""
    c = load_case("seeded42")
    for scheme, addr in PAIRS:
        st = make(gpu, c, scheme, addr, zero_collision=True)
        st.load_natural(c["f0"])
        s0 = np.sort(c["f0"])
        for _ in range(4):
            st.step()
            assert bitwise_equal(np.sort(st.extract_natural()), s0), scheme


def test_two_zero_collision_aa_steps_equal_double_streaming(gpu):
    """p/tests/test_schemes.cpp:247-266"""
    c = load_case("seeded42")
    for addr in ("direct", "indirect"):
        aa = make(gpu, c, "aap", addr, zero_collision=True)
        ts = make(gpu, c, "ts", "direct", zero_collision=True)
        aa.load_natural(c["f0"])
        ts.load_natural(c["f0"])
        aa.step(), aa.step(), ts.step(), ts.step()
        assert bitwise_equal(aa.extract_natural(), ts.extract_natural())


def test_chunk_length_and_streaming_stores_do_not_change_results(gpu):
    """p/tests/test_schemes.cpp:268-307"""
    c = load_case("seeded42")
    for scheme in ("osnt-pull-1s", "osnt-pull-2s"):
        for addr in ("direct", "indirect"):
            outs = []
            for chunk, nt in ((1, True), (150, True), (922, False)):
                st = make(gpu, c, scheme, addr, chunk_length=chunk, streaming_stores=nt)
                st.load_natural(c["f0"])
                st.step_n(5)
                outs.append(st.extract_natural())
            assert bitwise_equal(outs[0], outs[1]) and bitwise_equal(outs[0], outs[2])


def test_swap_fixup_timing_does_not_change_state(gpu):
    """p/tests/test_schemes.cpp:309-330"""
    c = load_case("seeded42")
    for scheme in ("swap-push", "swap-pull"):
        x = make(gpu, c, scheme, "direct", swap_deferred_fixup=False)
        y = make(gpu, c, scheme, "direct", swap_deferred_fixup=True)
        x.load_natural(c["f0"])
        y.load_natural(c["f0"])
        for _ in range(6):
            x.step(), y.step()
            assert bitwise_equal(x.extract_natural(), y.extract_natural())


def test_layout_phases(gpu):
    """p/tests/test_schemes.cpp:358-396"""
    L = gpu
    g = L.gen_channel(8, 4, 4)

    def phase(scheme, steps, deferred=False):
        st = L.create_stepper(scheme, "direct", g, L.FlowParams(),
                              L.StepperOptions(swap_deferred_fixup=deferred))
        for _ in range(steps):
            st.step()
        return st.layout_phase()

    for s in ("ts", "os-push", "os-pull", "osnt-pull-1s"):
        assert all(phase(s, t) == "natural" for t in (0, 1, 2))
    assert [phase("aap", t) for t in (0, 1, 2)] == ["natural", "opposed", "natural"]
    assert phase("cg", 1) == "shifted_even" and phase("cg", 2) == "shifted_odd"
    assert phase("swap-push", 1) == "opposed"
    assert phase("swap-push", 1, True) == "swap_partial"
    assert phase("swap-pull", 2) == "natural"
    assert [phase("et", t) for t in (0, 1, 2)] == ["natural", "twisted", "natural"]


def test_et_handle_exchange_is_an_involution(gpu):
    """p/tests/test_schemes.cpp:398-414"""
    L = gpu
    g = L.gen_channel(8, 4, 4)
    for addr in ("direct", "indirect"):
        et = L.create_stepper("et", addr, g)
        before = et.extract_natural()
        assert et.layout_phase() == "natural"
        assert et.exchange_opposite_handles()
        assert et.layout_phase() == "twisted"
        assert et.exchange_opposite_handles()
        assert bitwise_equal(et.extract_natural(), before)
    assert not L.create_stepper("ts", "direct", g).exchange_opposite_handles()


@pytest.mark.parametrize("scheme,addr", PAIRS + EXT_PAIRS)
def test_closed_box_conserves_mass(gpu, scheme, addr):
    """p/tests/test_schemes.cpp:416-436 (100 steps, 1e-12)"""
    c = load_case("closed_box")
    st = make(gpu, c, scheme, addr)
    st.load_natural(c["f0"])
    m0 = c["f0"].sum()
    st.step_n(100)
    assert abs(st.extract_natural().sum() - m0) / m0 <= 1e-12


@pytest.mark.parametrize("seed", [1, 42, 1234])
def test_build_sparse_bitwise(gpu, seed):
    z = load_case("idx")
    L = gpu
    g = L.GridGeometry(16, 8, 8, ("periodic", "wall", "periodic"), z[f"seed{seed}_mask"])
    n, adj, node_of = L.build_sparse(g, node_of=True)
    assert n == int(z[f"seed{seed}_mask"].sum())
    assert np.array_equal(adj, z[f"seed{seed}_adjacency"])
    assert np.array_equal(node_of, z[f"seed{seed}_node_of"])


def test_build_sparse_porous_and_et_rem(gpu):
    z = load_case("idx")
    c = load_case("porous_c2")
    L = gpu
    g = geometry(L, c)
    n, adj, _ = L.build_sparse(g)
    assert np.array_equal(adj, z["porous_adjacency"])
    rem, nmail = L.build_et_rem(g)
    assert np.array_equal(rem, z["porous_et_rem"]) and nmail == int(z["porous_et_mail"])


def test_build_sparse_edge_cases(gpu):
    L = gpu
    n, adj, _ = L.build_sparse(L.GridGeometry(4, 4, 4))
    assert n == 64 and (adj != np.arange(64)[:, None]).all()
    n, adj, _ = L.build_sparse(L.GridGeometry(1, 1, 1, ("wall",) * 3))
    assert n == 1 and (adj == 0).all()
    n, adj, _ = L.build_sparse(L.GridGeometry(3, 3, 3, mask=np.zeros(27, np.uint8)))
    assert n == 0 and adj.size == 0


def test_unsupported_pairs_and_option_errors(gpu):
    L = gpu
    g = L.gen_channel(4, 4, 4)
    for s in ("ts", "cg", "swap-push", "swap-pull"):
        with pytest.raises(ValueError, match="kernel not implemented; traffic model only"):
            L.create_stepper(s, "indirect", g)
    with pytest.raises(ValueError, match="kernel not implemented; traffic model only"):
        L.create_stepper("cg", "indirect", g, options=L.StepperOptions(extensions=True))
    with pytest.raises(ValueError, match="workers must be >= 0"):
        L.create_stepper("aap", "direct", g, options=L.StepperOptions(workers=-1))
    with pytest.raises(ValueError, match="chunk_length must be >= 1"):
        L.create_stepper("osnt-pull-1s", "direct", g, options=L.StepperOptions(chunk_length=0))


@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("scheme,addr", PAIRS + EXT_PAIRS)
def test_degenerate_geometries(gpu, scheme, addr, layout):
    """No fluid node at all, and one fluid node walled in by solids: stepping
    works, the snapshot has the fluid count's length, and the lone node (every
    link bounces back onto itself) evolves like the oracle's 1-node box."""
    import oracle
    L = gpu
    opts = L.StepperOptions(layout=layout, extensions=(scheme, addr) in EXT_PAIRS)
    empty = L.GridGeometry(3, 3, 3, ("periodic",) * 3, np.zeros(27, np.uint8))
    st = L.create_stepper(scheme, addr, empty, L.bgk(1.0), opts)
    st.step_n(3)
    st.synchronize()
    assert st.node_count() == 0 and st.extract_natural().size == 0
    mask = np.zeros(27, np.uint8)
    mask[13] = 1  # the centre of a 3^3 box
    lone = L.GridGeometry(3, 3, 3, ("periodic",) * 3, mask)
    st = L.create_stepper(scheme, addr, lone, L.bgk(1.7, (1e-4, 0.0, 0.0)), opts)
    O = oracle.Oracle()
    f0 = O.random_field(5, 1)
    st.load_natural(f0)
    st.step_n(4)
    st.synchronize()
    want = O.ts_run(1, 1, 1, [1, 1, 1], None, 1.7, 1.7, [1e-4, 0.0, 0.0], f0, 4)
    assert bitwise_equal(st.extract_natural(), want)


def test_index_range_guards(gpu):
    """build_sparse's guard (p/src/geometry.cpp:177-179): 2^31 fluid nodes are
    refused with the reference's text before any device allocation; a grid of
    2^32 cells exceeds the 32-bit storage index of the direct kernels."""
    L = gpu
    with pytest.raises(RuntimeError, match="fluid count exceeds 32-bit index range"):
        L.create_stepper("aap", "indirect", L.GridGeometry(2048, 1024, 1024))
    with pytest.raises(RuntimeError, match="grid exceeds 32-bit cell index range"):
        L.create_stepper("aap", "direct", L.GridGeometry(4096, 1024, 1024))


def test_cg_sweeps_back_to_back_per_thread_aos(gpu):
    """CG's plane groups are chained with programmatic dependent launch; a
    sweep's first group must not let the next group start loading before the
    previous sweep's stores landed. Many sweeps queued back to back on the
    per-thread kernels (AoS windows off, in a subprocess: the switch is read
    once per process), bitwise = the oracle."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_1111_0922_b200 as L, oracle\n"
        "O = oracle.Oracle(); dims = (35, 10, 70)\n"
        "geo = L.GridGeometry(*dims)\n"
        "f0 = O.random_field(99, geo.fluid_count())\n"
        "for lay in ('aos', 'soa'):\n"
        "    st = L.create_stepper('cg', 'direct', geo, L.bgk(1.7, (2e-5, 0.0, 0.0)),"
        " L.StepperOptions(layout=lay))\n"
        "    st.load_natural(f0); st.step_n(12); st.synchronize()\n"
        "    want = O.ts_run(*dims, [0, 0, 0], None, 1.7, 1.7, [2e-5, 0.0, 0.0], f0, 12)\n"
        "    assert (st.extract_natural().view(np.uint64) == want.view(np.uint64)).all(), lay\n"
        "print('ok')\n" % ROOT)
    env = dict(os.environ, LBMGPU_AOS_WINDOW="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("zpipe", ["1", "0"])
def test_cg_aos_plane_groups_z_pipeline(gpu, zpipe):
    """AoS CG plane groups through the z-pipeline push (k_win_zp over [z0, z1)
    with the saved wrap planes; default for fp32, LBMGPU_AOS_ZPIPE_CG=1 forces
    it for fp64) and through the k_win gather windows (= 0): fp64 bitwise =
    the oracle, fp32 bitwise = the SoA fp32 stepper; small plane groups and a
    ragged z chunk, periodic and walled z, a porous mask. In a subprocess:
    the switches are read once per process."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_1111_0922_b200 as L, oracle\n"
        "O = oracle.Oracle()\n"
        "rng = np.random.default_rng(3)\n"
        "for dims, pol, porous in (((45, 17, 23), (0, 0, 0), False), ((35, 10, 70), (0, 0, 1), False),"
        " ((40, 12, 21), (0, 1, 0), True)):\n"
        "    names = tuple('wall' if w else 'periodic' for w in pol)\n"
        "    mask = (rng.random(dims[0] * dims[1] * dims[2]) > 0.25).astype(np.uint8) if porous else None\n"
        "    geo = L.GridGeometry(*dims, names, mask)\n"
        "    f0 = O.random_field(7, geo.fluid_count())\n"
        "    flow = L.bgk(1.7, (2e-5, 1e-6, -3e-6))\n"
        "    want = O.ts_run(*dims, list(pol), mask, 1.7, 1.7, [2e-5, 1e-6, -3e-6], f0, 9)\n"
        "    out = {}\n"
        "    for prec in (8, 4):\n"
        "        for lay in ('aos', 'soa'):\n"
        "            st = L.create_stepper('cg', 'direct', geo, flow,"
        " L.StepperOptions(layout=lay, precision=prec))\n"
        "            st.load_natural(f0); st.step_n(9); st.synchronize()\n"
        "            out[prec, lay] = st.extract_natural()\n"
        "    assert (out[8, 'aos'].view(np.uint64) == want.view(np.uint64)).all(), (dims, 'f64')\n"
        "    assert (out[4, 'aos'].view(np.uint64) == out[4, 'soa'].view(np.uint64)).all(), (dims, 'f32')\n"
        "print('ok')\n" % ROOT)
    env = dict(os.environ, LBMGPU_AOS_ZPIPE_CG=zpipe, LBMGPU_CG_PLANES="5", LBMGPU_AOS_ZCHUNK="3")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("dims,policy", [
    ((5, 7, 6), ("periodic", "periodic", "periodic")),
    ((33, 9, 5), ("periodic", "periodic", "wall")),
    ((300, 3, 4), ("periodic", "wall", "periodic")),
    ((512, 2, 3), ("wall", "periodic", "periodic")),
    ((40, 40, 12), ("periodic", "periodic", "wall")),
    ((24, 19, 9), "porous"),
])
@pytest.mark.parametrize("precision", [8, 4])
@pytest.mark.parametrize("scheme", ["swap-push", "swap-pull"])
def test_swap_one_sweep_equals_two_passes(gpu, monkeypatch, dims, policy, precision, scheme):
    """kernels_swap.cu (collisions + exchanges in one launch, tiles of full x
    rows ordered by flags) against the collide pass + exchange pass: bitwise,
    over tile shapes (several rows per tile, one row, a ragged last tile,
    nx = 512), wall axes, a porous mask, and the deferred seam fix-up."""
    rng = np.random.default_rng(11)
    mask = None
    if policy == "porous":
        mask = (rng.random(dims[::-1]) > 0.3).astype(np.uint8).reshape(-1)
        policy = ("periodic", "periodic", "periodic")
    geo = gpu.GridGeometry(*dims, policy, mask)
    flow = gpu.bgk(1.7, body_force=(1e-6, 2e-7, -1e-7))
    outs = []
    for fused in ("1", "0"):
        monkeypatch.setenv("LBMGPU_SWAP_FUSED", fused)
        for deferred in (False, True):
            st = gpu.create_stepper(scheme, "direct", geo, flow,
                                    gpu.StepperOptions(precision=precision,
                                                       swap_deferred_fixup=deferred))
            st.init_field("taylor_green", seed=5)
            st.step_n(5)
            st.synchronize()
            outs.append(st.extract_natural())
    for o in outs[1:]:
        assert bitwise_equal(o, outs[0])


@pytest.mark.parametrize("aos_window", ["0", "1"])
def test_cg_all_solid_plane_groups(gpu, aos_window):
    """CG plane groups with no fluid cell (a solid band thicker than a group,
    LBMGPU_CG_PLANES=2): every thread of such a group still waits for the group
    ahead before it exits, so the chain of programmatic dependent launches
    keeps its order. Many sweeps back to back, bitwise = the oracle (SoA and
    AoS; per-thread AoS kernels and the tile windows)."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_1111_0922_b200 as L, oracle\n"
        "O = oracle.Oracle(); dims = (24, 16, 40)\n"
        "mask = np.ones(dims[::-1], np.uint8); mask[10:21] = 0; mask[30:33, 4:9] = 0\n"
        "mask = mask.reshape(-1)\n"
        "geo = L.GridGeometry(*dims, ('periodic',) * 3, mask)\n"
        "f0 = O.random_field(7, geo.fluid_count())\n"
        "want = O.ts_run(*dims, [0, 0, 0], mask, 1.7, 1.7, [2e-5, 0.0, 0.0], f0, 15)\n"
        "for lay in ('soa', 'aos'):\n"
        "    st = L.create_stepper('cg', 'direct', geo, L.bgk(1.7, (2e-5, 0.0, 0.0)),"
        " L.StepperOptions(layout=lay))\n"
        "    st.load_natural(f0); st.step_n(15); st.synchronize()\n"
        "    assert (st.extract_natural().view(np.uint64) == want.view(np.uint64)).all(), lay\n"
        "print('ok')\n" % ROOT)
    env = dict(os.environ, LBMGPU_AOS_WINDOW=aos_window, LBMGPU_CG_PLANES="2")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("dims,policy", [
    ((5, 7, 6), ("periodic", "periodic", "periodic")),
    ((70, 20, 30), ("periodic", "periodic", "periodic")),
    ((33, 9, 17), ("periodic", "periodic", "wall")),
    ((45, 19, 11), ("wall", "wall", "periodic")),
    ((64, 16, 9), ("wall", "periodic", "wall")),
    ((40, 17, 12), "porous"),
])
@pytest.mark.parametrize("zchunk", ["", "3"])
@pytest.mark.parametrize("precision", [8, 4])
@pytest.mark.parametrize("scheme", ["swap-push", "swap-pull"])
def test_swap_single_pass_equals_two_passes(gpu, monkeypatch, dims, policy, zchunk, precision,
                                            scheme):
    """kernels_swap1.cu (one sweep; links between blocks through face buffers
    of alternating parity) against the collide pass + exchange pass: bitwise
    after odd and even step counts, across extractions (push flushes its face
    values into the field) and reloads, over ragged tiles, several z chunks
    (LBMGPU_SWAP1_ZCHUNK), wall axes, a porous mask and the deferred seam
    fix-up."""
    rng = np.random.default_rng(13)
    mask = None
    if policy == "porous":
        mask = (rng.random(dims[::-1]) > 0.3).astype(np.uint8).reshape(-1)
        policy = ("periodic", "periodic", "periodic")
    geo = gpu.GridGeometry(*dims, policy, mask)
    flow = gpu.bgk(1.7, body_force=(1e-6, 2e-7, -1e-7))
    monkeypatch.setenv("LBMGPU_SWAP1_ZCHUNK", zchunk)
    f0 = None
    for deferred in (False, True):
        outs = []
        for single in ("1", "0"):
            monkeypatch.setenv("LBMGPU_SWAP_SINGLE", single)
            st = gpu.create_stepper(scheme, "direct", geo, flow,
                                    gpu.StepperOptions(precision=precision,
                                                       swap_deferred_fixup=deferred))
            st.init_field("taylor_green", seed=5)
            if f0 is None:
                f0 = st.extract_natural()
            got = []
            for n in (3, 4):
                st.step_n(n)
                got.append(st.extract_natural())
            st.load_natural(f0)
            st.step_n(5)
            got.append(st.extract_natural())
            outs.append(got)
        for a, b in zip(outs[0], outs[1]):
            assert bitwise_equal(a, b), (deferred,)


@pytest.mark.parametrize("dims,policy", [
    ((5, 7, 6), ("periodic", "periodic", "periodic")),
    ((70, 20, 30), ("periodic", "periodic", "periodic")),
    ((33, 9, 17), ("periodic", "periodic", "wall")),
    ((45, 19, 11), ("wall", "wall", "periodic")),
    ((40, 17, 12), "porous"),
])
@pytest.mark.parametrize("zchunk", ["", "3"])
@pytest.mark.parametrize("precision", [8, 4])
@pytest.mark.parametrize("scheme", ["swap-push", "swap-pull"])
def test_swap_single_pass_aos(gpu, monkeypatch, dims, policy, zchunk, precision, scheme):
    """kernels_swap1.cu k_swap1_aos (AoS records staged in shared memory,
    links between blocks through the face buffers) against the AoS two-pass
    SWAP: bitwise over odd and even steps, extractions and a reload."""
    rng = np.random.default_rng(17)
    mask = None
    if policy == "porous":
        mask = (rng.random(dims[::-1]) > 0.3).astype(np.uint8).reshape(-1)
        policy = ("periodic", "periodic", "periodic")
    geo = gpu.GridGeometry(*dims, policy, mask)
    flow = gpu.bgk(1.7, body_force=(1e-6, 2e-7, -1e-7))
    monkeypatch.setenv("LBMGPU_SWAP1_ZCHUNK", zchunk)
    outs, f0 = [], None
    deferred = zchunk == "3"  # the deferred seam fix-up on half the cases
    for single in ("1", "0"):
        monkeypatch.setenv("LBMGPU_SWAP_SINGLE_AOS", single)  # 0: two-pass windows
        st = gpu.create_stepper(scheme, "direct", geo, flow,
                                gpu.StepperOptions(precision=precision, layout="aos",
                                                   swap_deferred_fixup=deferred))
        st.init_field("taylor_green", seed=5)
        if f0 is None:
            f0 = st.extract_natural()
        got = []
        for n in (3, 4):
            st.step_n(n)
            got.append(st.extract_natural())
        st.load_natural(f0)
        st.step_n(5)
        got.append(st.extract_natural())
        outs.append(got)
    for a, b in zip(outs[0], outs[1]):
        assert bitwise_equal(a, b)
