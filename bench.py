#!/usr/bin/env python3
"""Benchmark of the B200-native D3Q19 collide+propagate step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one LBM time step (one collide+propagate sweep of the whole
lattice). The workload at every N is BASELINE.json configs[3] ("C3", the
config its 1/2/4/8-GPU metric is quoted on): a 512x512x1024 periodic box,
BGK omega=1.0, seeded Taylor-Green start, AA pattern, direct addressing, SoA,
fp64 (40.8 GB; it fits one B200). N=1 runs the single-domain stepper; under
torchrun (N>1) the box is split into z-slabs, one per rank (DESIGN.md
section 6). Strong scaling: the box is fixed. value = fluid nodes x K / device
time (MFLUP/s), max over ranks. `--gpus N` outside torchrun relaunches itself
under torch.distributed.run with N ranks.

Prints ONE JSON line (rank 0). See DESIGN.md section 7 for every key.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MFLUP/s and achieved HBM GB/s as % of bytes/FLUP roofline, 1/2/4/8 B200"

CONFIGS = {
    # BASELINE.json configs[1]
    "c1": dict(dims=(256, 256, 256), policy=("periodic", "periodic", "wall"), omega=1.7,
               force=(1e-6, 0.0, 0.0), init="rest",
               desc="C1: 256^3 channel, periodic x/y, bounce-back walls z=0/255, BGK omega=1.7, "
                    "g=1e-6 x, rest start"),
    # BASELINE.json configs[0]
    "c0": dict(dims=(128, 128, 128), policy=("periodic",) * 3, omega=1.0, force=(0.0, 0.0, 0.0),
               init="taylor_green",
               desc="C0: 128^3 periodic, BGK omega=1.0, Taylor-Green + 1e-4 noise"),
    # BASELINE.json configs[4]
    "c4": dict(dims=(200, 200, 200), policy=("periodic",) * 3, omega=1.0, force=(0.0, 0.0, 0.0),
               init="taylor_green", desc="C4: 200^3 periodic, BGK omega=1.0, Taylor-Green"),
    # BASELINE.json configs[2] (porous, indirect); over z-slabs with --slabs / N>1
    "c2": dict(dims=(256, 256, 256), policy=("periodic",) * 3, omega=1.7,
               force=(1e-6, 0.0, 0.0), init="rest", porous=True,
               desc="C2: 256^3 periodic, random r=8 spheres to porosity 0.40 (seed 2011), "
                    "indirect, BGK omega=1.7, g=1e-6 x, rest start"),
    # BASELINE.json configs[3] (multi-GPU z-slabs)
    "c3": dict(dims=(512, 512, 1024), policy=("periodic",) * 3, omega=1.0,
               force=(0.0, 0.0, 0.0), init="taylor_green",
               desc="C3: 512x512x1024 periodic, BGK omega=1.0, Taylor-Green, z-slabs"),
}


def config_dict(name, args, ws, nodes):
    """The `config` object, identical in both arms for the same invocation."""
    cfg = CONFIGS[name]
    pdf = 8 if args.precision == 8 else 4
    field = nodes * 19 * pdf * (1 if args.scheme in ("aap", "et", "cg", "swap-push", "swap-pull")
                                else 2)
    return {"workload": cfg["desc"], "scheme": args.scheme, "addressing": args.addressing,
            "layout": args.layout, "precision": "f64" if pdf == 8 else "f32",
            "dims": list(cfg["dims"]), "fluid_nodes": int(nodes),
            "parallelism": "single domain" if ws == 1 else f"z-slabs x{ws}",
            "l2": f"inputs larger than L2 ({field / 1e9:.2f} GB of PDFs vs 126 MB L2), "
                  "no flush needed"}


def fluid_nodes(name):
    cfg = CONFIGS[name]
    nx, ny, nz = cfg["dims"]
    if cfg.get("porous"):
        from paper_1111_0922_b200.geometry import gen_random_spheres
        return gen_random_spheres(nx, ny, nz).fluid_count()
    return nx * ny * nz


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _one(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=5).stdout.strip()
            if out:
                self.rows.append([v.strip() for v in out.split(",")])
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._one()
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            self._one()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > k + 2 and r[k + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws == 1:
        return 1, 0, 0, None
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    return ws, rank, local, dist


def reduce_max(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def traffic_from_profiles(kernel_key):
    """dram bytes read+write per launch from the committed ncu --set full capture"""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(kernel_key)
    except Exception:
        return None


# ---------------------------------------------------------------------------
def cpu_reference_sample(cfg, scheme, budget_s=20.0, max_steps=None):
    """The UNMODIFIED reference (oracle/_ref/libref.so, built from /root/reference)
    through its own run_bench (p/src/bench.cpp:155-198) with every host core."""
    import oracle
    R = oracle.RefLib()
    dims = tuple(cfg["dims"])
    sub = ""
    if dims[0] * dims[1] * dims[2] > (1 << 25):
        # bounded sample: the same per-node work on a z-truncated box (MFLUP/s is a
        # per-node rate); the full C3 lattice would need 41 GB of host memory
        nzs = max(2, (1 << 25) // (dims[0] * dims[1]))
        sub = f" [bounded sample: {dims[0]}x{dims[1]}x{nzs} sub-box of {dims[0]}x{dims[1]}x{dims[2]}]"
        dims = (dims[0], dims[1], nzs)
    pol = [1 if p == "wall" else 0 for p in cfg["policy"]]
    om = cfg["omega"]
    magic = (1.0 / om - 0.5) ** 2
    addr, mask = 0, None
    if cfg.get("porous"):  # C2: the same seeded spheres, the reference's indirect path
        from paper_1111_0922_b200.geometry import gen_random_spheres
        mask = gen_random_spheres(*dims).mask
        addr = 1
    # one probe step sizes the sample to the budget
    s1, _, _ = R.run_bench(scheme, addr, dims, pol, mask, om, magic, cfg["force"], 1, workers=0,
                           warmup=0, timed_runs=1)
    steps = max(2, int(budget_s / 3.0 / max(s1, 1e-6)))
    if max_steps:
        steps = min(steps, max_steps)
    sec, mlups, workers = R.run_bench(scheme, addr, dims, pol, mask, om, magic, cfg["force"],
                                      steps, workers=0, warmup=1, timed_runs=3)
    return dict(value=mlups, unit="MFLUP/s", cores=workers, kind="reference",
                sample=f"{cfg['desc']}{sub}; reference {scheme}/{'indirect' if addr else 'direct'} "
                       f"run_bench, {steps} steps x 3 "
                       f"runs (median) after 1 warm-up step, workers=0 -> {workers} threads, "
                       f"nproc={os.cpu_count()}, OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND', 'unset')}")


def run_reference_arm(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if ws > 1:
        # torchrun sets OMP_NUM_THREADS=1 per rank; the lone reference rank
        # takes every host core (read when the reference's OpenMP starts)
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    cfg = CONFIGS[args.config]
    n_gpus = max(ws, args.gpus)
    budget = float(os.environ.get("LBM_REF_BUDGET_S", "90"))
    base = cpu_reference_sample(cfg, args.scheme, budget_s=budget, max_steps=args.steps)
    nodes = fluid_nodes(args.config)
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "MFLUP/s",
        "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": nodes / (base["value"] * 1e6) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json config; seeded start)",
        "config": config_dict(args.config, args, n_gpus, nodes),
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "MFLUP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def live_peaks(L, device, field_bytes):
    """In-place and copy streaming probes on this GPU (lbmgpu_stream_bandwidth),
    over 4 GiB (or the field size if smaller), best of 10: the second
    denominator beside MEASURED_PEAKS.json (whose copy is torch's)."""
    nb = int(min(4 << 30, max(1 << 28, field_bytes)))
    return {"inplace_gbs": round(L.stream_bandwidth(nb, True, 10, device), 1),
            "copy_gbs": round(L.stream_bandwidth(nb, False, 10, device), 1),
            "bytes": nb, "how": "lbmgpu_stream_bandwidth: 16-B vector grid-stride kernel, "
                                "read+write bytes, best of 10, CUDA events"}


def make_geometry(L, name, args):
    cfg = CONFIGS[name]
    if cfg.get("porous"):
        from paper_1111_0922_b200.geometry import gen_random_spheres
        args.addressing = "indirect"
        return gen_random_spheres(*cfg["dims"])
    return L.GridGeometry(*cfg["dims"], cfg["policy"])


def run_ours(args):
    ws, rank, local, dist = dist_setup()
    import paper_1111_0922_b200 as L
    if L.device_count() < 1:
        raise SystemExit("no CUDA device visible")
    if ws > 1 or args.slabs:
        return run_slabs(args, ws, rank, local, dist, L)

    cfg = CONFIGS[args.config]
    dims = cfg["dims"]
    geo = make_geometry(L, args.config, args)
    flow = L.bgk(cfg["omega"], body_force=cfg["force"])
    opts = L.StepperOptions(layout=args.layout, precision=args.precision, device=local,
                            extensions=args.scheme in ("ts", "swap-push", "swap-pull")
                            and args.addressing == "indirect")
    st = L.create_stepper(args.scheme, args.addressing, geo, flow, opts)
    st.init_field(cfg["init"], seed=2011)
    nodes = st.node_count()
    pdf = 8 if args.precision == 8 else 4

    # warm-up, then K steps between CUDA events on the launching stream
    st.step_n(args.warmup)
    st.synchronize()
    barrier(dist)
    with ClockSampler(local) as clk:
        ms = st.step_timed(args.steps)
    ms = reduce_max(dist, ms)
    launches = st.launches_per_step()
    value = nodes * args.steps / (ms * 1e-3) / 1e6

    peak, peak_src = load_peaks()
    bpl = L.gpu_bytes_per_lup(args.scheme, args.addressing, pdf)
    per_launch_ms = ms / (args.steps * launches)
    # dominant kernel: one launch updates every node once for AA/ET/OS/CG (bytes
    # per launch = bytes/FLUP x N); two-launch schemes split the step
    achieved = bpl * nodes / launches / (per_launch_ms * 1e-3) / 1e9
    kern = {"aap": "k_local+k_aa_odd", "et": "k_et", "os-pull": "k_os_pull",
            "os-push": "k_os_push", "osnt-pull-1s": "k_os_pull", "osnt-pull-2s": "k_os_pull",
            "cg": "k_cg", "ts": "k_local+k_ts_stream", "swap-push": "k_local+k_swap",
            "swap-pull": "k_swap+k_local"}[args.scheme]
    key = f"{args.config}:{args.scheme}:{args.addressing}:{args.layout}:{pdf}"
    live = live_peaks(L, local, st.storage_bytes()[0]) if not args.no_live_peak else None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic_from_profiles(key),
                "traffic_key": key, "algorithmic_bytes_per_flup": bpl,
                "algorithmic_bytes_per_launch": bpl * nodes / launches, "kernel": kern,
                "per_launch_ms": round(per_launch_ms, 5), "peak_source": peak_src,
                "model_mflups": round(peak * 1e9 / bpl / 1e6, 1)}
    if live:
        roofline["live_peak"] = live
        roofline["frac_vs_live_inplace"] = round(achieved / live["inplace_gbs"], 4)

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "MFLUP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if pdf == 8 else "f32",
        "data": "synthetic (BASELINE.json config; seeded start)",
        "config": config_dict(args.config, args, 1, nodes),
        "roofline": roofline,
        "gpu_launches": args.steps * launches,
        "clocks": clk.summary(),
    }

    if not args.no_e2e:
        line["e2e"] = e2e_run(L, st, args, nodes)
    if not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_reference_sample(cfg, args.scheme, budget_s=20.0)
        except Exception as e:  # reference library absent on this box
            line["cpu_baseline"] = {"value": None, "unit": "MFLUP/s", "cores": 0,
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    return 0


def e2e_run(L, st, args, nodes):
    """Same metric through the public API with HOST buffers: load the canonical
    snapshot from pinned host memory, K steps, extract it back into the same
    pinned buffer, all inside the timed region (wall clock around synchronous
    calls). One pinned buffer (C3: 40.8 GB)."""
    n = nodes * 19
    buf = L.PinnedArray(n)
    st.extract_natural(buf.array)  # a valid state to start from
    st.synchronize()
    t0 = time.perf_counter()
    st.load_natural(buf.array)
    st.step_n(args.steps)
    st.extract_natural(buf.array)
    t = time.perf_counter() - t0
    del buf
    return {"value": round(nodes * args.steps / t / 1e6, 2), "unit": "MFLUP/s",
            "h2d_bytes_per_step": n * 8 / args.steps, "d2h_bytes_per_step": n * 8 / args.steps,
            "seconds": round(t, 4),
            "note": "load_natural(pinned host) + K steps + extract_natural(pinned host)"}


def run_slabs(args, ws, rank, local, dist, L):
    """BASELINE.json configs[3] over z-slabs: the box is split into ws slabs, one
    per rank (GPU); AA pattern with the NCCL halo exchange of the 5 crossing slot
    planes per face before and after every odd sweep, overlapped with the
    interior planes. Strong scaling: the whole box is fixed."""
    cfg = CONFIGS[args.config]
    nx, ny, nz = cfg["dims"]
    if nz % ws:
        raise SystemExit(f"nz={nz} not divisible by {ws} ranks")
    if args.layout != "soa":
        raise SystemExit("z-slabs are SoA only (--layout soa)")
    z0, z1 = rank * nz // ws, (rank + 1) * nz // ws
    geo = make_geometry(L, args.config, args)
    flow = L.bgk(cfg["omega"], body_force=cfg["force"])
    pdf = 8 if args.precision == 8 else 4
    st = L.create_stepper(args.scheme, args.addressing, geo, flow,
                          L.StepperOptions(device=local, z_begin=z0, z_end=z1,
                                           precision=args.precision, layout=args.layout))
    comm = None
    if args.transport == "p2p":
        # peer-memory AA: face planes read/rewrite the neighbours' slots in
        # place (CUDA IPC pointers), steps ordered by flag words; no NCCL
        blobs = [st.slab_p2p_export()]
        if dist is not None:
            blobs = [None] * ws
            dist.all_gather_object(blobs, st.slab_p2p_export())
        st.slab_p2p_connect(blobs[(rank - 1) % ws], blobs[(rank + 1) % ws], ws, rank)
        barrier(dist)
        comm = {"transport": "p2p (CUDA IPC peer pointers, flag words)"}
    else:
        uid = [L.nccl_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(uid, src=0)
        st.slab_connect_nccl(uid[0], ws, rank)
        comm = dict(st.slab_comm_info(), transport="nccl (halo send/recv, comm stream)")
    st.init_field(cfg["init"], seed=2011)
    nodes_local = st.node_count()
    nodes = int(reduce_sum(dist, nodes_local))
    st.step_n(args.warmup)
    st.synchronize()
    barrier(dist)
    with ClockSampler(local) as clk:
        ms_local = st.step_timed(args.steps)
    ms = reduce_max(dist, ms_local)
    value = nodes * args.steps / (ms * 1e-3) / 1e6
    peak, peak_src = load_peaks()
    bpl = L.gpu_bytes_per_lup(args.scheme, args.addressing, pdf)
    achieved = bpl * nodes_local / (ms / args.steps * 1e-3) / 1e9
    launches = st.launches_per_step()
    halo = 2 * 2 * 5 * nx * ny * pdf  # bytes per rank per exchange (all-fluid planes)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "MFLUP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if pdf == 8 else "f32",
        "data": "synthetic (BASELINE.json config; seeded start)",
        "config": config_dict(args.config, args, ws, nodes),
        "comm": comm,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic_from_profiles(
                         f"{args.config}:{args.scheme}:{args.addressing}:{args.layout}:{pdf}"),
                     "algorithmic_bytes_per_flup": bpl,
                     "kernel": f"{args.scheme} sweep (per rank, slowest rank's step)",
                     "peak_source": peak_src,
                     "halo_bytes_per_exchange_per_rank": halo},
        "gpu_launches": args.steps * launches,
        "clocks": clk.summary(),
    }
    if not args.no_e2e:
        line["e2e"] = e2e_slabs(L, st, args, dist, nodes_local, nodes)
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier(dist)
    return 0


def e2e_slabs(L, st, args, dist, nodes_local, nodes):
    """e2e on the slab path: every rank loads its slab's canonical snapshot
    from pinned host memory, runs K steps (halo exchanges included), brings
    its ghosts up to date and extracts back to host; the max over ranks of the
    wall time between two barriers. One pinned buffer per rank (the extract
    overwrites the loaded snapshot)."""
    n = nodes_local * 19
    buf = L.PinnedArray(n)
    st.slab_sync_ghosts()  # collective: the extraction may read ghost planes
    st.extract_natural(buf.array)
    barrier(dist)
    t0 = time.perf_counter()
    st.load_natural(buf.array)
    st.step_n(args.steps)
    st.slab_sync_ghosts()
    st.extract_natural(buf.array)
    t = reduce_max(dist, time.perf_counter() - t0)
    total = nodes * 19 * (8 if args.precision == 8 else 4)
    return {"value": round(nodes * args.steps / t / 1e6, 2), "unit": "MFLUP/s",
            "h2d_bytes_per_step": total / args.steps, "d2h_bytes_per_step": total / args.steps,
            "seconds": round(t, 4),
            "note": "per rank: load_natural(pinned host) + K steps + slab_sync_ghosts + "
                    "extract_natural(pinned host); bytes are whole-job"}


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n):
    """`--gpus N` (N > 1) outside torchrun: re-exec this command with N ranks,
    exactly as the driver launches it."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, LBM_BENCH_RELAUNCHED="1")
    os.execvpe(cmd[0], cmd, env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS),
                    help="BASELINE.json config (default c3, the metric's config, at every N)")
    ap.add_argument("--scheme", default="aap")
    ap.add_argument("--addressing", default="direct")
    ap.add_argument("--layout", default="soa")
    ap.add_argument("--precision", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-live-peak", action="store_true")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="z-slab exchange: NCCL halo phases, or p2p (AA direct: face planes "
                         "read and rewrite the neighbours' slots through peer pointers)")
    ap.add_argument("--slabs", action="store_true",
                    help="run the z-slab/NCCL path even at N=1 (one rank, ring to itself)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if CONFIGS[args.config].get("porous"):
        args.addressing = "indirect"
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference_arm(args)
    if ws == 0 and args.gpus > 1:
        if os.environ.get("LBM_BENCH_RELAUNCHED"):
            raise SystemExit("relaunch under torch.distributed.run did not set WORLD_SIZE")
        relaunch_under_torchrun(args.gpus)
    if ws > 0 and ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: refusing to report a "
                         "different GPU count than requested")
    if os.environ.get("LBM_BENCH_DRYRUN"):
        # launch check only (tests/test_bench_contract.py): report the rank layout
        print(json.dumps({"dryrun": True, "rank": int(os.environ.get("RANK", "0")),
                          "world_size": max(ws, 1), "gpus": args.gpus}), flush=True)
        return 0
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
