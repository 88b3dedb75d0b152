"""GPU: z-slab steppers (the multi-GPU decomposition: AA, ET, OS push/pull,
OSNT) driven in one process with the in-process transport (same halo plan as
the NCCL transport). P slabs must reproduce the single-domain stepper of the
same scheme bit for bit, at even and odd steps; the slab snapshots are
contiguous ranges of the global one."""
import numpy as np
import pytest

from conftest import bitwise_equal

pytestmark = pytest.mark.gpu


def _slabs(L, dims, flow, bounds, precision=8, scheme="aap"):
    geo = L.GridGeometry(*dims, ("periodic", "periodic", "periodic"))
    return [L.create_stepper(scheme, "direct", geo, flow,
                             L.StepperOptions(z_begin=a, z_end=b, precision=precision))
            for a, b in bounds]


def _needs_ghosts(scheme, t):
    return (scheme == "aap" and t % 2 == 1) or "pull" in scheme or scheme == "et"


def _ext(scheme):  # TS / SWAP indirect are GPU extensions (the reference's are direct-only)
    return scheme in ("ts", "swap-push", "swap-pull")


@pytest.mark.parametrize("scheme", ["aap", "os-pull", "os-push", "osnt-pull-2s", "et", "ts",
                                    "swap-push", "swap-pull", "cg"])
@pytest.mark.parametrize("nslab", [1, 2, 3, 4])
def test_slabs_match_single_domain(gpu, nslab, scheme):
    L = gpu
    dims = (24, 20, 16)
    nz = dims[2]
    cuts = np.linspace(0, nz, nslab + 1).astype(int)
    bounds = list(zip(cuts[:-1], cuts[1:]))
    flow = L.bgk(1.0)
    ref = L.create_stepper(scheme, "direct", L.GridGeometry(*dims), flow)
    ref.init_field("taylor_green", seed=11, u0=0.05)
    slabs = _slabs(L, dims, flow, bounds, scheme=scheme)
    for s in slabs:
        s.init_field("taylor_green", seed=11, u0=0.05)
    # device-side init is keyed by the global cell: the slabs start identical
    assert bitwise_equal(np.concatenate([s.extract_natural() for s in slabs]),
                         ref.extract_natural())
    for steps in (1, 4, 3):  # ends at t = 1 (odd), 5 (odd), 8 (even)
        ref.step_n(steps)
        ref.synchronize()
        L.slab_group_step(slabs, steps)
        if _needs_ghosts(scheme, ref.time_step()):
            L.slab_group_sync_ghosts(slabs)
        got = np.concatenate([s.extract_natural() for s in slabs])
        assert bitwise_equal(got, ref.extract_natural()), (nslab, ref.time_step())


@pytest.mark.parametrize("scheme", ["aap", "et", "os-pull"])
def test_slab_load_and_uneven_split(gpu, scheme):
    L = gpu
    dims = (16, 12, 10)
    flow = L.bgk(1.7, (1e-6, 0, 0))
    ref = L.create_stepper(scheme, "direct", L.GridGeometry(*dims), flow)
    ref.init_field("random", seed=3)
    f0 = ref.extract_natural()
    bounds = [(0, 1), (1, 4), (4, 10)]
    slabs = _slabs(L, dims, flow, bounds, scheme=scheme)
    per = dims[0] * dims[1] * 19
    for s, (a, b) in zip(slabs, bounds):
        s.load_natural(f0[a * per:b * per])
    ref.step_n(6)
    ref.synchronize()
    L.slab_group_step(slabs, 6)
    if _needs_ghosts(scheme, 6):
        L.slab_group_sync_ghosts(slabs)
    assert bitwise_equal(np.concatenate([s.extract_natural() for s in slabs]),
                         ref.extract_natural())


def test_slab_errors(gpu):
    L = gpu
    geo = L.GridGeometry(8, 8, 8)
    with pytest.raises(ValueError, match="supports every scheme"):
        L.create_stepper("aap", "direct", geo,
                         options=L.StepperOptions(z_begin=0, z_end=4, layout="aos"))
    with pytest.raises(ValueError, match="swap_deferred_fixup"):
        L.create_stepper("swap-push", "direct", geo,
                         options=L.StepperOptions(z_begin=0, z_end=4, swap_deferred_fixup=True))
    with pytest.raises(ValueError, match="periodic z"):
        L.create_stepper("aap", "direct", L.gen_channel(8, 8, 8),
                         options=L.StepperOptions(z_begin=0, z_end=4))
    with pytest.raises(ValueError, match="ET z-slabs need periodic x and y"):
        L.create_stepper("et", "direct", L.GridGeometry(8, 8, 8, ("wall", "periodic", "periodic")),
                         options=L.StepperOptions(z_begin=0, z_end=4))
    s = L.create_stepper("aap", "direct", geo, options=L.StepperOptions(z_begin=0, z_end=4))
    with pytest.raises(RuntimeError, match="no transport"):
        s.step()


@pytest.mark.parametrize("scheme", ["aap", "os-pull", "os-push", "et", "ts", "swap-push",
                                    "swap-pull", "cg"])
def test_nccl_transport_single_rank_ring(gpu, scheme):
    """The NCCL transport itself (liblbmgpu.so dlopens libnccl): one rank whose
    ring neighbours are itself, the overlapped interior/boundary schedule, the
    phase-0/phase-1 groups — bitwise equal to the periodic single domain."""
    L = gpu
    dims = (32, 24, 20)
    flow = L.bgk(1.0)
    ref = L.create_stepper(scheme, "direct", L.GridGeometry(*dims), flow)
    ref.init_field("taylor_green", seed=9, u0=0.05)
    s = L.create_stepper(scheme, "direct", L.GridGeometry(*dims), flow,
                         L.StepperOptions(z_begin=0, z_end=dims[2]))
    s.slab_connect_nccl(L.nccl_unique_id(), 1, 0)
    s.init_field("taylor_green", seed=9, u0=0.05)
    for steps in (6, 3):
        ref.step_n(steps)
        ref.synchronize()
        s.step_n(steps)
        s.synchronize()
        if _needs_ghosts(scheme, s.time_step()):
            s.slab_sync_ghosts()
        assert bitwise_equal(s.extract_natural(), ref.extract_natural()), s.time_step()


def _porous(L, dims, solid=0.25, seed=5):
    rng = np.random.default_rng(seed)
    mask = (rng.random(dims[0] * dims[1] * dims[2]) >= solid).astype(np.uint8)
    return L.GridGeometry(*dims, ("periodic", "periodic", "periodic"), mask)


@pytest.mark.parametrize("scheme", ["aap", "os-pull", "os-push", "osnt-pull-2s", "ts", "et",
                                    "swap-push", "swap-pull"])
@pytest.mark.parametrize("bounds", [[(0, 12)], [(0, 5), (5, 12)], [(0, 1), (1, 7), (7, 12)]])
def test_indirect_slabs_match_single_domain(gpu, scheme, bounds):
    """indirect z-slabs: each slab numbers its fluid nodes over its planes plus
    one ghost plane per face, the exchanges move node ranges; porous box,
    bitwise = the single-domain indirect stepper"""
    L = gpu
    dims = (20, 16, 12)
    geo = _porous(L, dims)
    flow = L.bgk(1.3, (1e-5, 2e-6, 0.0))
    ext = _ext(scheme)
    ref = L.create_stepper(scheme, "indirect", geo, flow, L.StepperOptions(extensions=ext))
    ref.init_field("random", seed=4)
    slabs = [L.create_stepper(scheme, "indirect", geo, flow,
                              L.StepperOptions(z_begin=a, z_end=b, extensions=ext))
             for a, b in bounds]
    for s in slabs:
        s.init_field("random", seed=4)
    assert sum(s.node_count() for s in slabs) == ref.node_count()
    assert bitwise_equal(np.concatenate([s.extract_natural() for s in slabs]),
                         ref.extract_natural())
    for steps in (1, 4, 3):
        ref.step_n(steps)
        ref.synchronize()
        L.slab_group_step(slabs, steps)
        if _needs_ghosts(scheme, ref.time_step()):
            L.slab_group_sync_ghosts(slabs)
        got = np.concatenate([s.extract_natural() for s in slabs])
        assert bitwise_equal(got, ref.extract_natural()), (bounds, ref.time_step())


def test_indirect_slab_host_load(gpu):
    L = gpu
    dims = (16, 12, 10)
    geo = _porous(L, dims, 0.3, seed=9)
    flow = L.bgk(1.7, (1e-6, 0, 0))
    ref = L.create_stepper("aap", "indirect", geo, flow)
    ref.init_field("random", seed=3)
    f0 = ref.extract_natural()
    bounds = [(0, 3), (3, 10)]
    slabs = [L.create_stepper("aap", "indirect", geo, flow, L.StepperOptions(z_begin=a, z_end=b))
             for a, b in bounds]
    k = 0
    for s in slabs:
        n = s.node_count()
        s.load_natural(f0[k * 19:(k + n) * 19])
        k += n
    ref.step_n(5)
    ref.synchronize()
    L.slab_group_step(slabs, 5)
    L.slab_group_sync_ghosts(slabs)
    assert bitwise_equal(np.concatenate([s.extract_natural() for s in slabs]),
                         ref.extract_natural())


@pytest.mark.parametrize("scheme", ["aap", "os-pull", "os-push", "et"])
def test_indirect_nccl_single_rank_ring(gpu, scheme):
    L = gpu
    dims = (24, 20, 14)
    geo = _porous(L, dims, 0.2, seed=2)
    flow = L.bgk(1.0)
    ref = L.create_stepper(scheme, "indirect", geo, flow)
    ref.init_field("taylor_green", seed=9, u0=0.05)
    s = L.create_stepper(scheme, "indirect", geo, flow, L.StepperOptions(z_begin=0, z_end=dims[2]))
    s.slab_connect_nccl(L.nccl_unique_id(), 1, 0)
    s.init_field("taylor_green", seed=9, u0=0.05)
    for steps in (6, 3):
        ref.step_n(steps)
        ref.synchronize()
        s.step_n(steps)
        s.synchronize()
        if _needs_ghosts(scheme, s.time_step()):
            s.slab_sync_ghosts()
        assert bitwise_equal(s.extract_natural(), ref.extract_natural()), s.time_step()


@pytest.mark.parametrize("scheme", ["aap", "os-push", "os-pull", "ts", "swap-push", "swap-pull",
                                    "cg"])
def test_direct_slabs_with_xy_walls(gpu, scheme):
    """x/y walls: an owner node whose link towards the neighbour slab bounces
    writes that face slot itself, so phase 1 merges instead of copying"""
    L = gpu
    dims = (20, 14, 12)
    geo = L.GridGeometry(*dims, ("wall", "wall", "periodic"))
    flow = L.bgk(1.7, (1e-5, 0, 2e-6))
    ref = L.create_stepper(scheme, "direct", geo, flow)
    ref.init_field("random", seed=8)
    bounds = [(0, 4), (4, 9), (9, 12)]
    slabs = [L.create_stepper(scheme, "direct", geo, flow, L.StepperOptions(z_begin=a, z_end=b))
             for a, b in bounds]
    for s in slabs:
        s.init_field("random", seed=8)
    for steps in (1, 4, 3):
        ref.step_n(steps)
        ref.synchronize()
        L.slab_group_step(slabs, steps)
        if _needs_ghosts(scheme, ref.time_step()):
            L.slab_group_sync_ghosts(slabs)
        assert bitwise_equal(np.concatenate([s.extract_natural() for s in slabs]),
                             ref.extract_natural()), ref.time_step()
