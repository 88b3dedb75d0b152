"""GPU: the one-rank-per-process peer-memory transport (slabs.cu
connect_p2p_ipc with nranks >= 2) in 2 and 4 separate processes on device 0.

Each process owns one z-slab, publishes its field through a CUDA IPC handle
(lbmgpu_slab_p2p_export), opens its neighbours' handles
(cudaIpcOpenMemHandle) and sweeps its face planes through those mappings.
The ranks share ONE GPU here, and kernels of different processes that spin on
each other's flag words are not guaranteed to run concurrently (B200_PROFILING:
Xid 109), so the ranks connect host-ordered (LBMGPU_P2P_HOST_ORDERED): after
every step each rank synchronizes its stream and the ranks meet at a gloo
barrier instead of the flag-word kernel. Everything else — the IPC mappings,
the neighbour face-slot addressing of another process's blob, the odd face
sweep over the mapped memory, ghost sync for extraction at odd t — is the
multi-GPU code path. The gathered slabs must equal the single-domain AA
stepper bit for bit at odd and even t.

Run by pytest; the same file is the per-rank worker (``--rank``)."""
import argparse
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DIMS = (24, 20, 16)
CHECKS = (1, 5, 8, 11)  # t after which the slabs are compared (odd and even)


def _worker(rank, world, port, precision, out):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1111_0922_b200 as L

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cuts = np.linspace(0, DIMS[2], world + 1).astype(int)
    geo = L.GridGeometry(*DIMS)
    flow = L.FlowParams(1.0 / 0.8, 3.0 / 16.0, (2e-5, -1e-5, 5e-6), 1.0)
    s = L.create_stepper("aap", "direct", geo, flow,
                         L.StepperOptions(z_begin=int(cuts[rank]), z_end=int(cuts[rank + 1]),
                                          precision=precision))
    s.init_field("taylor_green", seed=11, u0=0.05)
    blobs = [None] * world
    dist.all_gather_object(blobs, s.slab_p2p_export())
    s.slab_p2p_connect(blobs[(rank - 1) % world], blobs[(rank + 1) % world], world, rank,
                       host_ordered=True)
    dist.barrier()
    snaps = {}
    t = 0
    while t < CHECKS[-1]:
        s.step_n(1)
        s.synchronize()
        dist.barrier()
        t += 1
        if t in CHECKS:
            if t % 2:
                s.slab_sync_ghosts()
                s.synchronize()
                dist.barrier()
            parts = [None] * world
            dist.all_gather_object(parts, s.extract_natural())
            snaps[t] = np.concatenate(parts)
    dist.barrier()
    if rank == 0:
        ref = L.create_stepper("aap", "direct", geo, flow, L.StepperOptions(precision=precision))
        ref.init_field("taylor_green", seed=11, u0=0.05)
        bad = []
        for t in CHECKS:
            ref.step_n(t - ref.time_step())
            ref.synchronize()
            want = ref.extract_natural()
            if not np.array_equal(np.ascontiguousarray(snaps[t]).view(np.uint8),
                                  np.ascontiguousarray(want).view(np.uint8)):
                bad.append(t)
        with open(out, "w") as fh:
            fh.write("ok\n" if not bad else f"mismatch at t={bad}\n")
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [8, 4])
@pytest.mark.parametrize("world", [2, 4])
def test_p2p_ipc_ranks_in_separate_processes(gpu, world, precision, tmp_path):
    port = _free_port()
    out = str(tmp_path / "result.txt")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen([sys.executable, os.path.abspath(__file__), "--rank", str(r),
                               "--world", str(world), "--port", str(port), "--precision",
                               str(precision), "--out", out], env=env, cwd=ROOT)
             for r in range(world)]
    codes = []
    for p in procs:
        try:
            codes.append(p.wait(timeout=240))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    assert codes == [0] * world, codes
    with open(out) as fh:
        assert fh.read().strip() == "ok"


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--port", type=int, required=True)
    ap.add_argument("--precision", type=int, default=8)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    _worker(a.rank, a.world, a.port, a.precision, a.out)
