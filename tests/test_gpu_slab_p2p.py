"""GPU: the peer-memory ("p2p") transport of AA z-slabs. The face planes' odd
sweep (kernels_direct.cu k_aa_odd_face) reads and rewrites the neighbour
slab's face slots in place through peer pointers; there is no ghost exchange.
P slabs must reproduce the single-domain AA stepper bit for bit at odd and
even t (in one process: slabs on this device ordered by step events; one rank:
the multi-process path with its flag-word barrier, connected to itself)."""
import numpy as np
import pytest

from conftest import bitwise_equal

pytestmark = pytest.mark.gpu


def _slabs(L, dims, pol, flow, bounds, precision=8):
    geo = L.GridGeometry(*dims, pol)
    return [L.create_stepper("aap", "direct", geo, flow,
                             L.StepperOptions(z_begin=int(a), z_end=int(b), precision=precision))
            for a, b in bounds]


@pytest.mark.parametrize("precision", [8, 4])
@pytest.mark.parametrize("pol", [("periodic", "periodic", "periodic"), ("wall", "periodic", "periodic"),
                                 ("periodic", "wall", "periodic")])
@pytest.mark.parametrize("nslab", [1, 2, 3, 4])
def test_p2p_group_matches_single_domain(gpu, nslab, pol, precision):
    L = gpu
    dims = (24, 20, 16)
    cuts = np.linspace(0, dims[2], nslab + 1).astype(int)
    bounds = list(zip(cuts[:-1], cuts[1:]))
    flow = L.FlowParams(1.0 / 0.8, 3.0 / 16.0, (2e-5, -1e-5, 5e-6), 1.0)
    ref = L.create_stepper("aap", "direct", L.GridGeometry(*dims, pol), flow,
                           L.StepperOptions(precision=precision))
    ref.init_field("taylor_green", seed=11, u0=0.05)
    slabs = _slabs(L, dims, pol, flow, bounds, precision)
    for s in slabs:
        s.init_field("taylor_green", seed=11, u0=0.05)
    L.slab_group_connect_p2p(slabs)
    for steps in (1, 4, 3, 2):  # t = 1, 5 (odd), 8, 10 (even)
        ref.step_n(steps)
        ref.synchronize()
        L.slab_group_step(slabs, steps)
        if ref.time_step() % 2:
            L.slab_group_sync_ghosts(slabs)
        got = np.concatenate([s.extract_natural() for s in slabs])
        assert bitwise_equal(got, ref.extract_natural()), (nslab, pol, ref.time_step())


def test_p2p_group_uneven_split_and_reload(gpu):
    L = gpu
    dims = (20, 18, 13)
    pol = ("periodic", "periodic", "periodic")
    flow = L.bgk(1.7, (1e-5, 0.0, 0.0))
    ref = L.create_stepper("aap", "direct", L.GridGeometry(*dims), flow)
    slabs = _slabs(L, dims, pol, flow, [(0, 2), (2, 9), (9, 13)])
    rng = np.random.default_rng(3)
    f0 = (1.0 / 19.0) * (1.0 + 0.01 * rng.standard_normal((dims[0] * dims[1] * dims[2], 19)))
    ref.load_natural(f0)
    plane = dims[0] * dims[1]
    for s, (a, b) in zip(slabs, [(0, 2), (2, 9), (9, 13)]):
        s.load_natural(f0[a * plane:b * plane])
    L.slab_group_connect_p2p(slabs)
    for _ in range(2):  # a reload keeps the transport
        ref.step_n(7)
        L.slab_group_step(slabs, 7)
        L.slab_group_sync_ghosts(slabs)
        got = np.concatenate([s.extract_natural() for s in slabs])
        assert bitwise_equal(got, ref.extract_natural())
        ref.load_natural(f0)
        for s, (a, b) in zip(slabs, [(0, 2), (2, 9), (9, 13)]):
            s.load_natural(f0[a * plane:b * plane])


@pytest.mark.parametrize("precision", [8, 4])
def test_p2p_single_rank_ipc_path(gpu, precision):
    """The one-rank-per-process path (flag barrier kernel on the side stream,
    face planes over the connected pointers) with the ring closed on itself."""
    L = gpu
    dims = (24, 20, 16)
    flow = L.bgk(1.0)
    ref = L.create_stepper("aap", "direct", L.GridGeometry(*dims), flow,
                           L.StepperOptions(precision=precision))
    ref.init_field("taylor_green", seed=5, u0=0.05)
    (s,) = _slabs(L, dims, ("periodic",) * 3, flow, [(0, dims[2])], precision)
    s.init_field("taylor_green", seed=5, u0=0.05)
    blob = s.slab_p2p_export()
    assert len(blob) == L.P2P_BLOB_BYTES and blob[:7] == b"LBMP2P1"
    s.slab_p2p_connect(blob, blob, 1, 0)
    for steps in (1, 6, 3):
        ref.step_n(steps)
        ref.synchronize()
        s.step_n(steps)
        if ref.time_step() % 2:
            s.slab_sync_ghosts()
        assert bitwise_equal(s.extract_natural(), ref.extract_natural()), ref.time_step()


def test_p2p_errors(gpu):
    L = gpu
    dims = (16, 12, 8)
    flow = L.bgk(1.0)
    geo = L.GridGeometry(*dims)
    os_slabs = [L.create_stepper("os-pull", "direct", geo, flow, L.StepperOptions(z_begin=a, z_end=b))
                for a, b in [(0, 4), (4, 8)]]
    with pytest.raises(ValueError, match="AA on direct"):
        L.slab_group_connect_p2p(os_slabs)
    thin = [L.create_stepper("aap", "direct", geo, flow, L.StepperOptions(z_begin=a, z_end=a + 1))
            for a in range(8)]
    with pytest.raises(ValueError, match="at least 2 planes"):
        L.slab_group_connect_p2p(thin)
    (s,) = _slabs(L, dims, ("periodic",) * 3, flow, [(0, 8)])
    with pytest.raises(ValueError, match="not a p2p blob"):
        s.slab_p2p_connect(bytes(L.P2P_BLOB_BYTES), bytes(L.P2P_BLOB_BYTES), 1, 0)
