"""CPU, multi-process (gloo, world_size 2): the z-slab halo plans that
liblbmgpu.so's NCCL transport executes (lbmgpu_scheme_halo_plan) drive numpy
restatements of the AA pattern, the one-step push/pull scheme and the
esoteric twist on two ranks; the gathered state must equal the single-domain two-step oracle bit
for bit, at even and odd steps."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

DIMS = (6, 4, 8)  # nx, ny, nz (periodic); two slabs of 4 planes
STEPS = 7
FORCE = (1e-4, -2e-5, 3e-5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _initial(nodes):
    import oracle
    return oracle.Oracle().random_field(20251019, nodes)


def _worker(rank, world, port, scheme, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle.aa_numpy import AaSlab, EtSlab, OsSlab, trt
    import paper_1111_0922_b200 as L

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz = DIMS
    nzl = nz // world
    op = trt(1.3, 1.3, FORCE)
    if scheme == "aap":
        slab = AaSlab(nx, ny, nzl, op)
        plane_of = lambda grid, slot, plane: slab.plane(slot, plane)  # noqa: E731
    elif scheme == "et":
        slab = EtSlab(nx, ny, nzl, op)
        plane_of = lambda grid, slot, plane: slab.plane(slot, plane)  # noqa: E731
    else:
        slab = OsSlab(nx, ny, nzl, op, pull=scheme == "os-pull")
        plane_of = slab.plane
    f0 = _initial(nx * ny * nz)
    per = nx * ny * nzl * 19
    slab.load(f0[rank * per:(rank + 1) * per])
    plan = L.halo_plan(nzl, scheme)

    def phase(ph, grid):
        reqs = []
        for (p, send, peer, plane, slot) in plan:
            if p != ph or not send:
                continue
            dst = (rank + peer) % world
            t = torch.from_numpy(np.ascontiguousarray(plane_of(grid, slot, plane)))
            reqs.append(dist.isend(t, dst=dst, tag=int(slot) + 32 * ph))
        for (p, send, peer, plane, slot) in plan:
            if p != ph or send:
                continue
            src = (rank + peer) % world
            t = torch.empty(ny, nx, dtype=torch.float64)
            dist.recv(t, src=src, tag=int(slot) + 32 * ph)
            plane_of(grid, slot, plane)[...] = t.numpy()
        for r in reqs:
            r.wait()

    results = {}
    if scheme == "et":
        phase(1, 0)  # the fill parks boundary cells' remote slots in the ghosts
    for t in range(1, STEPS + 1):
        if scheme == "et":
            phase(0, 0)
            slab.step_local()
            phase(1, 0)  # with the sweep's handles
            slab.swap_handles()
        elif scheme == "aap":
            odd = slab.t % 2 == 1
            if odd:
                phase(0, 0)
            slab.step_local()
            if odd:
                phase(1, 0)
        elif scheme == "os-pull":
            slab.precollide()
            phase(0, slab.active)
            slab.step_local()
        else:
            slab.step_local()
            phase(1, slab.active)  # the grid just written
        if t in (STEPS - 1, STEPS):
            if scheme == "aap" and slab.t % 2 == 1:
                phase(0, 0)  # fresh ghosts for the odd-time gather
            if scheme == "et":
                phase(0, 0)  # the gather reads remote slots under the new handles
            if scheme == "os-pull":
                phase(0, slab.active ^ 1)  # the idle grid the extraction streams
            results[t] = slab.extract()
    out = {}
    for t, v in results.items():
        parts = [torch.zeros(per, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(v))
        out[t] = np.concatenate([p.numpy() for p in parts])
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_halo_plan_shape():
    import paper_1111_0922_b200 as L
    plan = L.halo_plan(5)
    assert plan.shape == (40, 5)
    for ph in (0, 1):
        rows = plan[plan[:, 0] == ph]
        assert (rows[:, 1] == 1).sum() == 10 and (rows[:, 1] == 0).sum() == 10
    # crossing slot sets: cz=-1 {6,8,11,13,16}, cz=+1 {5,9,12,14,17}
    assert set(plan[(plan[:, 3] == -1)][:, 4]) == {6, 8, 11, 13, 16}
    assert set(plan[(plan[:, 3] == 5)][:, 4]) == {5, 9, 12, 14, 17}
    pull = L.halo_plan(5, "os-pull")
    assert pull.shape == (20, 5) and (pull[:, 0] == 0).all()
    assert set(pull[pull[:, 3] == -1][:, 4]) == {5, 9, 12, 14, 17}
    push = L.halo_plan(5, "os-push")
    assert push.shape == (20, 5) and (push[:, 0] == 1).all()
    assert np.array_equal(L.halo_plan(5, "osnt-pull-2s"), pull)
    assert np.array_equal(L.halo_plan(5, "ts"), pull)  # TS streams by pulling from B
    sw = L.halo_plan(5, "swap-pull")  # one-way per face: lower ghost <-> lower neighbour's top
    assert sw.shape == (20, 5) and np.array_equal(sw, L.halo_plan(5, "swap-push"))
    assert set(sw[:, 3]) == {-1, 4} and set(sw[:, 4]) == {5, 9, 12, 14, 17}
    et = L.halo_plan(5, "et")
    assert et.shape == (20, 5)
    assert set(et[et[:, 3] == 5][:, 4]) == {6, 16, 13}  # upper ghost
    assert set(et[et[:, 3] == -1][:, 4]) == {17, 14}  # lower ghost
    assert np.array_equal(L.halo_plan(5, "cg"), push)  # CG's face pushes land in padding planes
    with pytest.raises(ValueError):
        L.halo_plan(5, "d3q27")


@pytest.mark.parametrize("scheme", ["aap", "os-pull", "os-push", "et"])
def test_two_rank_gloo_slabs_match_single_domain(scheme):
    import torch.multiprocessing as mp
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, scheme, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nx, ny, nz = DIMS
    f0 = _initial(nx * ny * nz)
    O = oracle.Oracle()
    for t in (STEPS - 1, STEPS):
        want = O.ts_run(nx, ny, nz, [0, 0, 0], None, 1.3, 1.3, FORCE, f0, t)
        assert np.array_equal(out[t].view(np.uint64), want.view(np.uint64)), (scheme, t)
