"""B200-native D3Q19 collide+propagate (arXiv 1111.0922 propagation schemes).

Python mirror of the reference's C++ lattice/propagation API (``lbmlab``,
``/root/reference/proj/include/lbmlab``): ``GridGeometry``, ``FlowParams``,
``StepperOptions``, ``create_stepper`` -> ``Stepper`` with ``step`` /
``extract_natural`` / ``load_natural`` / ``layout_phase`` /
``exchange_opposite_handles``, ``kernel_available``, ``build_sparse``,
``traffic``, ``lambda_odd``. Every call goes through the C ABI of
``include/lbmgpu.h`` into ``liblbmgpu.so`` (hand-written sm_100a kernels).
There is no CPU fallback: importing fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBRARY_PATH = os.environ.get("LBMGPU_LIBRARY") or os.path.join(_HERE, "liblbmgpu.so")

if not os.path.exists(LIBRARY_PATH):
    raise ImportError(
        f"{LIBRARY_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
        "g.build()'` (make -C paper_1111_0922_b200/csrc). There is no CPU fallback.")

_L = C.CDLL(LIBRARY_PATH)

# lbmlab::SchemeId order (p/include/lbmlab/stepper.hpp:15-26)
SCHEMES = ("ts", "os-push", "os-pull", "osnt-pull-1s", "osnt-pull-2s", "cg", "swap-push",
           "swap-pull", "aap", "et")
FAMILIES = ("ts", "os", "osnt", "cg", "swap", "aap", "et")
FAMILY_OF = {"ts": "ts", "os-push": "os", "os-pull": "os", "osnt-pull-1s": "osnt",
             "osnt-pull-2s": "osnt", "cg": "cg", "swap-push": "swap", "swap-pull": "swap",
             "aap": "aap", "et": "et"}
ADDRESSINGS = ("direct", "indirect")
LAYOUT_PHASES = ("natural", "opposed", "shifted_even", "shifted_odd", "twisted", "swap_partial")
Q = 19
P2P_HOST_ORDERED = 1
P2P_BLOB_BYTES = 256  # LBMGPU_P2P_BLOB_BYTES


class _Geometry(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("axis_policy", C.c_uint8 * 3), ("mask", C.c_void_p)]


class _Flow(C.Structure):
    _fields_ = [("lambda_even", C.c_double), ("lambda_odd", C.c_double),
                ("body_force", C.c_double * 3), ("rho0", C.c_double)]


class _BenchResult(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("addressing", C.c_int32), ("layout", C.c_int32),
                ("precision", C.c_int32), ("fluid_count", C.c_uint64), ("steps", C.c_int32)] + \
               [(n, C.c_double) for n in ("seconds", "mlups", "bytes_per_lup", "gpu_bytes_per_lup",
                                          "predicted_mlups", "model_fraction", "achieved_gbs")]


class _VerifyEntry(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("scheme", "addressing", "layout", "precision", "bitwise",
                                         "pass_")] + [("max_rel_linf", C.c_double)]


class _Options(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "scheme", "addressing", "layout", "precision", "device", "workers", "chunk_length",
        "streaming_stores", "swap_deferred_fixup", "zero_collision", "extensions", "z_begin",
        "z_end")]


_P = C.c_void_p
_sig = {
    "lbmgpu_default_options": (None, [C.POINTER(_Options)]),
    "lbmgpu_create": (C.c_int, [C.POINTER(_Geometry), C.POINTER(_Flow), C.POINTER(_Options),
                                C.POINTER(_P)]),
    "lbmgpu_destroy": (C.c_int, [_P]),
    "lbmgpu_step": (C.c_int, [_P, C.c_int64]),
    "lbmgpu_step_timed": (C.c_int, [_P, C.c_int64, C.POINTER(C.c_double)]),
    "lbmgpu_synchronize": (C.c_int, [_P]),
    "lbmgpu_extract_natural": (C.c_int, [_P, _P]),
    "lbmgpu_load_natural": (C.c_int, [_P, _P]),
    "lbmgpu_extract_natural_range": (C.c_int, [_P, C.c_uint64, C.c_uint64, _P, C.c_int32]),
    "lbmgpu_extract_natural_device": (C.c_int, [_P, _P]),
    "lbmgpu_load_natural_device": (C.c_int, [_P, _P]),
    "lbmgpu_init_field": (C.c_int, [_P, C.c_int32, C.c_uint64, C.c_double, C.c_double,
                                    C.c_double]),
    "lbmgpu_layout_phase": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "lbmgpu_exchange_opposite_handles": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "lbmgpu_time_step": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "lbmgpu_node_count": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "lbmgpu_storage_bytes": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "lbmgpu_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "lbmgpu_launches_per_step": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "lbmgpu_kernel_available": (C.c_int, [C.c_int32, C.c_int32]),
    "lbmgpu_kernel_available_ext": (C.c_int, [C.c_int32, C.c_int32]),
    "lbmgpu_build_sparse": (C.c_int, [C.POINTER(_Geometry), C.c_int32, C.POINTER(C.c_uint32),
                                      _P, _P]),
    "lbmgpu_build_et_rem": (C.c_int, [C.POINTER(_Geometry), C.c_int32, C.POINTER(C.c_uint32),
                                      _P, C.POINTER(C.c_uint32)]),
    "lbmgpu_traffic": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                 C.POINTER(C.c_double)]),
    "lbmgpu_gpu_bytes_per_lup": (C.c_int, [C.c_int32, C.c_int32, C.c_int32,
                                           C.POINTER(C.c_double)]),
    "lbmgpu_lambda_odd": (C.c_double, [C.c_double, C.c_double]),
    "lbmgpu_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(_P)]),
    "lbmgpu_halo_plan": (C.c_int, [C.c_int32, _P, C.POINTER(C.c_int32)]),
    "lbmgpu_scheme_halo_plan": (C.c_int, [C.c_int32, C.c_int32, _P, C.POINTER(C.c_int32)]),
    "lbmgpu_nccl_unique_id": (C.c_int, [_P]),
    "lbmgpu_slab_connect_nccl": (C.c_int, [_P, _P, C.c_int32, C.c_int32]),
    "lbmgpu_slab_sync_ghosts": (C.c_int, [_P]),
    "lbmgpu_slab_comm_info": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32)]),
    "lbmgpu_slab_group_step": (C.c_int, [_P, C.c_int32, C.c_int64]),
    "lbmgpu_slab_group_sync_ghosts": (C.c_int, [_P, C.c_int32]),
    "lbmgpu_slab_group_connect_p2p": (C.c_int, [_P, C.c_int32]),
    "lbmgpu_slab_p2p_export": (C.c_int, [_P, _P]),
    "lbmgpu_slab_p2p_connect": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32]),
    "lbmgpu_slab_p2p_connect_ex": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_uint32]),
    "lbmgpu_host_free": (C.c_int, [_P]),
    "lbmgpu_run_bench": (C.c_int, [C.POINTER(_Geometry), C.POINTER(_Flow), C.POINTER(_Options),
                                   C.c_int32, C.c_int32, C.c_int32, C.c_double, _P]),
    "lbmgpu_stream_bandwidth": (C.c_int, [C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                          C.POINTER(C.c_double)]),
    "lbmgpu_selftest_division": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int32,
                                           C.POINTER(C.c_uint64)]),
    "lbmgpu_verify_suite": (C.c_int, [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "lbmgpu_last_error": (C.c_char_p, []),
    "lbmgpu_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "lbmgpu_version": (C.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    _fn = getattr(_L, _name)
    _fn.restype = _res
    _fn.argtypes = _args

class DomainError(ValueError):
    """std::domain_error (a std::logic_error, like invalid_argument -> ValueError):
    the reference's "vacuum node" (p/src/collision.cpp:31)."""


# status -> Python exception, mirroring the reference's C++ exception types
_ERRORS = {1: ValueError, 2: RuntimeError, 3: DomainError, 4: MemoryError, 5: RuntimeError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = (_L.lbmgpu_last_error() or b"").decode()
        raise _ERRORS.get(rc, RuntimeError)(msg)


def _scheme_id(s) -> int:
    if isinstance(s, (int, np.integer)):
        return int(s)
    n = str(s).lower().replace("_", "-")
    if n not in SCHEMES:
        raise ValueError(f"unknown scheme: {s}")
    return SCHEMES.index(n)


def _addr_id(a) -> int:
    if isinstance(a, (int, np.integer)):
        return int(a)
    n = str(a).lower()
    if n in ("direct", "full"):
        return 0
    if n in ("indirect", "sparse"):
        return 1
    raise ValueError(f"unknown addressing: {a}")


# ---------------------------------------------------------------------------
# reference value types
# ---------------------------------------------------------------------------
@dataclass
class GridGeometry:
    """lbmlab::GridGeometry (p/include/lbmlab/geometry.hpp:19-38)."""
    nx: int
    ny: int
    nz: int
    axis_policy: Sequence[str] = ("periodic", "periodic", "periodic")
    mask: Optional[np.ndarray] = None  # x-fastest uint8, 1 = fluid; None = all fluid

    def cells(self) -> int:
        return self.nx * self.ny * self.nz

    def fluid_count(self) -> int:
        return self.cells() if self.mask is None else int(np.count_nonzero(self.mask))

    def _c(self):
        g = _Geometry(self.nx, self.ny, self.nz)
        for k, p in enumerate(self.axis_policy):
            g.axis_policy[k] = {"periodic": 0, "wall": 1, 0: 0, 1: 1}[p]
        keep = None
        if self.mask is not None:
            keep = np.ascontiguousarray(self.mask, dtype=np.uint8).ravel()
            if keep.size != self.cells():
                raise ValueError("mask size does not match the grid")
            g.mask = keep.ctypes.data
        return g, keep


def gen_channel(nx: int, ny: int, nz: int) -> GridGeometry:
    """gen_channel (p/src/geometry.cpp:62-71): periodic x, walls in y and z."""
    if min(nx, ny, nz) < 1:
        raise ValueError("zero dimension")
    return GridGeometry(nx, ny, nz, ("periodic", "wall", "wall"))


@dataclass
class FlowParams:
    """lbmlab::FlowParams (p/include/lbmlab/collision.hpp:10-15), same defaults."""
    lambda_even: float = 1.0 / 0.9
    magic_lambda: float = 3.0 / 16.0
    body_force: Sequence[float] = (1e-5, 0.0, 0.0)
    rho0: float = 1.0


def lambda_odd(p: FlowParams) -> float:
    """lambda_odd (p/src/collision.cpp:8-11)."""
    return _L.lbmgpu_lambda_odd(p.lambda_even, p.magic_lambda)


def bgk(omega: float, body_force=(0.0, 0.0, 0.0), rho0: float = 1.0) -> FlowParams:
    """BGK as TRT with lambda_odd == lambda_even: magic Lambda = (1/omega - 1/2)^2
    makes lambda_odd(p) return omega exactly for the omegas used here (checked)."""
    p = FlowParams(omega, (1.0 / omega - 0.5) ** 2, tuple(body_force), rho0)
    if lambda_odd(p) != omega:
        raise ValueError(f"no exact BGK magic parameter for omega={omega}")
    return p


@dataclass
class StepperOptions:
    """lbmlab::StepperOptions (p/include/lbmlab/stepper.hpp:55-64) + GPU selectors."""
    workers: int = 1
    chunk_length: int = 150
    streaming_stores: bool = True
    swap_deferred_fixup: bool = False
    zero_collision: bool = False
    layout: str = "soa"        # "soa" | "aos"
    precision: int = 8         # 8 fp64 | 4 fp32
    device: int = 0
    extensions: bool = False   # allow TS/SWAP indirect (GPU-only kernels)
    z_begin: int = 0           # z-slab [z_begin, z_end) of a multi-GPU decomposition
    z_end: int = 0             # (AA, direct, SoA); 0 = whole box


# ---------------------------------------------------------------------------
# Stepper
# ---------------------------------------------------------------------------
class Stepper:
    """lbmlab::Stepper (p/include/lbmlab/stepper.hpp:70-106) on a B200."""

    def __init__(self, handle: C.c_void_p, scheme: int, addressing: int, opts: StepperOptions):
        self._h = handle
        self._scheme = scheme
        self._addr = addressing
        self.options = opts
        n = C.c_uint64()
        _check(_L.lbmgpu_node_count(self._h, C.byref(n)))
        self._nodes = int(n.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L.lbmgpu_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    # -- the reference surface ------------------------------------------------
    def step(self) -> None:
        """One time step, synchronous like the reference's Stepper::step()."""
        _check(_L.lbmgpu_step(self._h, 1))
        _check(_L.lbmgpu_synchronize(self._h))

    def step_n(self, n: int) -> None:
        """n time steps enqueued asynchronously on the stepper's stream."""
        _check(_L.lbmgpu_step(self._h, int(n)))

    def step_timed(self, n: int) -> float:
        """n steps between CUDA events on the launching stream; returns device ms."""
        ms = C.c_double()
        _check(_L.lbmgpu_step_timed(self._h, int(n), C.byref(ms)))
        return ms.value

    def synchronize(self) -> None:
        _check(_L.lbmgpu_synchronize(self._h))

    def extract_natural(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.values(), dtype=np.float64)
        if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != self.values():
            raise ValueError("out must be a contiguous float64 array of node_count*19")
        _check(_L.lbmgpu_extract_natural(self._h, out.ctypes.data))
        return out

    def extract_natural_range(self, first: int, count: int) -> np.ndarray:
        """nodes [first, first + count) of the canonical snapshot"""
        out = np.empty(int(count) * Q, dtype=np.float64)
        _check(_L.lbmgpu_extract_natural_range(self._h, int(first), int(count), out.ctypes.data, 0))
        return out

    def load_natural(self, f: np.ndarray) -> None:
        a = np.ascontiguousarray(f, dtype=np.float64).ravel()
        if a.size != self.values():
            raise ValueError("snapshot must hold node_count*19 values")
        _check(_L.lbmgpu_load_natural(self._h, a.ctypes.data))

    def extract_natural_device(self, dev_ptr: int) -> None:
        _check(_L.lbmgpu_extract_natural_device(self._h, dev_ptr))

    def load_natural_device(self, dev_ptr: int) -> None:
        _check(_L.lbmgpu_load_natural_device(self._h, dev_ptr))

    def init_field(self, kind: str = "rest", seed: int = 0, u0: float = 0.01,
                   drho: float = 1e-3, noise: float = 1e-4) -> None:
        k = {"rest": 0, "taylor_green": 1, "random": 2}[kind]
        _check(_L.lbmgpu_init_field(self._h, k, seed, u0, drho, noise))

    def layout_phase(self) -> str:
        v = C.c_int32()
        _check(_L.lbmgpu_layout_phase(self._h, C.byref(v)))
        return LAYOUT_PHASES[v.value]

    def exchange_opposite_handles(self) -> bool:
        v = C.c_int32()
        _check(_L.lbmgpu_exchange_opposite_handles(self._h, C.byref(v)))
        return bool(v.value)

    def scheme(self) -> str:
        return SCHEMES[self._scheme]

    def addressing(self) -> str:
        return ADDRESSINGS[self._addr]

    def time_step(self) -> int:
        v = C.c_int64()
        _check(_L.lbmgpu_time_step(self._h, C.byref(v)))
        return int(v.value)

    def node_count(self) -> int:
        return self._nodes

    def q(self) -> int:
        return Q

    def values(self) -> int:
        return self._nodes * Q

    # -- GPU extras -------------------------------------------------------------
    def storage_bytes(self):
        a, b = C.c_uint64(), C.c_uint64()
        _check(_L.lbmgpu_storage_bytes(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def launches_per_step(self) -> int:
        v = C.c_int32()
        _check(_L.lbmgpu_launches_per_step(self._h, C.byref(v)))
        return int(v.value)

    # -- multi-GPU z-slabs ------------------------------------------------------
    def slab_connect_nccl(self, unique_id: bytes, nranks: int, rank: int) -> None:
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(_L.lbmgpu_slab_connect_nccl(self._h, buf, nranks, rank))

    def slab_sync_ghosts(self) -> None:
        _check(_L.lbmgpu_slab_sync_ghosts(self._h))

    def slab_comm_info(self) -> dict:
        """ncclCommCount / ncclCommUserRank / ncclGetVersion of the slab's communicator"""
        c, r, v = C.c_int32(), C.c_int32(), C.c_int32()
        _check(_L.lbmgpu_slab_comm_info(self._h, C.byref(c), C.byref(r), C.byref(v)))
        return {"ncclCommCount": c.value, "ncclCommUserRank": r.value, "ncclGetVersion": v.value}

    def slab_p2p_export(self) -> bytes:
        """This slab's peer-memory blob (CUDA IPC handles of its field and flag
        words, its layout) for the neighbours' slab_p2p_connect."""
        buf = (C.c_uint8 * P2P_BLOB_BYTES)()
        _check(_L.lbmgpu_slab_p2p_export(self._h, buf))
        return bytes(buf)

    def slab_p2p_connect(self, lower: bytes, upper: bytes, nranks: int, rank: int,
                         host_ordered: bool = False) -> None:
        """One rank per process: AA odd face planes read and rewrite the
        neighbours' face slots in place through peer pointers (collective).
        host_ordered: no flag-word barrier kernel; the caller synchronizes and
        runs a host barrier across the ranks after every step / sync_ghosts
        (ranks sharing one GPU)."""
        lo = (C.c_uint8 * P2P_BLOB_BYTES).from_buffer_copy(lower[:P2P_BLOB_BYTES])
        hi = (C.c_uint8 * P2P_BLOB_BYTES).from_buffer_copy(upper[:P2P_BLOB_BYTES])
        flags = P2P_HOST_ORDERED if host_ordered else 0
        _check(_L.lbmgpu_slab_p2p_connect_ex(self._h, lo, hi, nranks, rank, flags))

    def cuda_stream(self) -> int:
        v = C.c_void_p()
        _check(_L.lbmgpu_stream(self._h, C.byref(v)))
        return int(v.value or 0)


def _c_options(sid, aid, options):
    o = _Options()
    _L.lbmgpu_default_options(C.byref(o))
    o.scheme, o.addressing = sid, aid
    o.layout = {"soa": 0, "aos": 1}[options.layout.lower()]
    o.precision = int(options.precision)
    o.device = int(options.device)
    o.workers = int(options.workers)
    o.chunk_length = int(options.chunk_length)
    o.streaming_stores = int(bool(options.streaming_stores))
    o.swap_deferred_fixup = int(bool(options.swap_deferred_fixup))
    o.zero_collision = int(bool(options.zero_collision))
    o.extensions = int(bool(options.extensions))
    o.z_begin = int(options.z_begin)
    o.z_end = int(options.z_end)
    return o


def _c_flow(flow):
    return _Flow(flow.lambda_even, lambda_odd(flow), (C.c_double * 3)(*flow.body_force), flow.rho0)


def create_stepper(scheme, addressing, geometry: GridGeometry, flow: FlowParams = None,
                   options: StepperOptions = None) -> Stepper:
    """create_stepper (p/src/stepper.cpp:155-180)."""
    flow = flow or FlowParams()
    options = options or StepperOptions()
    sid, aid = _scheme_id(scheme), _addr_id(addressing)
    g, keep = geometry._c()
    fl = _c_flow(flow)
    o = _c_options(sid, aid, options)
    h = C.c_void_p()
    _check(_L.lbmgpu_create(C.byref(g), C.byref(fl), C.byref(o), C.byref(h)))
    del keep
    return Stepper(h, sid, aid, options)


@dataclass
class BenchResult:
    """lbmlab::BenchResult (p/include/lbmlab/bench.hpp:49-62) + B200 columns."""
    scheme: str
    addressing: str
    layout: str
    dtype: str
    geometry: str
    fluid_count: int
    steps: int
    seconds: float
    mlups: float
    bytes_per_lup: float        # the paper's traffic() model
    gpu_bytes_per_lup: float    # compulsory DRAM bytes of these kernels
    predicted_mlups: float      # hbm_gbs / gpu_bytes_per_lup
    model_fraction: float
    achieved_gbs: float
    model_violated: bool


CSV_COLUMNS = ("scheme,addressing,layout,dtype,geometry,fluid_count,steps,seconds,mlups,"
               "bytes_per_lup,gpu_bytes_per_lup,predicted_mlups,model_fraction,achieved_gbs")


def run_bench(scheme, addressing, geometry: GridGeometry, flow: FlowParams = None, steps: int = 10,
              warmup: int = 3, timed_runs: int = 3, options: StepperOptions = None,
              hbm_gbs: float = 0.0, geometry_name: str = "custom") -> BenchResult:
    """run_bench (p/src/bench.cpp:155-198) on the GPU: median device time of
    timed_runs x steps; model_violated when model_fraction > 1.1 (bench.cpp:196)."""
    flow = flow or FlowParams()
    options = options or StepperOptions()
    sid, aid = _scheme_id(scheme), _addr_id(addressing)
    g, keep = geometry._c()
    r = _BenchResult()
    _check(_L.lbmgpu_run_bench(C.byref(g), C.byref(_c_flow(flow)),
                               C.byref(_c_options(sid, aid, options)), steps, warmup, timed_runs,
                               hbm_gbs, C.byref(r)))
    del keep
    return BenchResult(SCHEMES[sid], ADDRESSINGS[aid], options.layout,
                       "f64" if options.precision == 8 else "f32", geometry_name,
                       int(r.fluid_count), r.steps, r.seconds, r.mlups, r.bytes_per_lup,
                       r.gpu_bytes_per_lup, r.predicted_mlups, r.model_fraction, r.achieved_gbs,
                       r.model_fraction > 1.1)


def to_csv(results) -> str:
    """to_csv (p/src/bench.cpp:210-241) with the B200 columns"""
    out = CSV_COLUMNS + "\n"
    for r in results:
        out += ",".join([r.scheme, r.addressing, r.layout, r.dtype, r.geometry,
                         str(r.fluid_count), str(r.steps)] +
                        [f"{v:.6g}" for v in (r.seconds, r.mlups, r.bytes_per_lup,
                                              r.gpu_bytes_per_lup, r.predicted_mlups,
                                              r.model_fraction, r.achieved_gbs)]) + "\n"
    return out


@dataclass
class VerifyEntry:
    scheme: str
    addressing: str
    layout: str
    dtype: str
    bitwise: bool
    passed: bool
    max_rel_linf: float


def stream_bandwidth(nbytes: int = 4 << 30, inplace: bool = True, reps: int = 10,
                     device: int = 0) -> float:
    """GB/s (read + write) of a streaming copy or in-place update over nbytes
    (lbmgpu_stream_bandwidth): the live roofline denominator of bench.py."""
    g = C.c_double()
    _check(_L.lbmgpu_stream_bandwidth(device, nbytes, int(inplace), reps, C.byref(g)))
    return g.value


def selftest_division(n: int = 1 << 26, seed: int = 1, device: int = 0) -> int:
    """Mismatching bit patterns of the collision's shared-reciprocal division
    against __ddiv_rn over n seeded inputs (lbmgpu_selftest_division)."""
    m = C.c_uint64()
    _check(_L.lbmgpu_selftest_division(n, seed, device, C.byref(m)))
    return m.value


def verify_suite(seed: int = 42, steps: int = 10, device: int = 0, all_variants: bool = False):
    """verify_suite (p/src/bench.cpp:275-341) on the GPU. Returns (entries, all_pass)."""
    cap = 128
    arr = (_VerifyEntry * cap)()
    n, ap = C.c_int32(), C.c_int32()
    _check(_L.lbmgpu_verify_suite(seed, steps, device, int(all_variants), arr, cap, C.byref(n),
                                  C.byref(ap)))
    ents = [VerifyEntry(SCHEMES[e.scheme], ADDRESSINGS[e.addressing], ("soa", "aos")[e.layout],
                        "f64" if e.precision == 8 else "f32", bool(e.bitwise), bool(e.pass_),
                        e.max_rel_linf) for e in arr[:n.value]]
    return ents, bool(ap.value)


def macroscopic_fields(stepper: Stepper, flow: FlowParams):
    """macroscopic_fields (p/src/stepper.cpp:182-193): per fluid node rho and
    u = (sum f c) / rho + g / 2 (moments, p/src/collision.cpp:24-36); host-side
    diagnostic over the extracted snapshot. Raises DomainError("vacuum node")
    (std::domain_error in the reference) when a node's rho <= 0."""
    from .geometry import C_VECTORS
    f = stepper.extract_natural().reshape(-1, Q)
    rho = np.zeros(f.shape[0])
    m = np.zeros((f.shape[0], 3))
    for i in range(Q):
        rho = rho + f[:, i]
        for k in range(3):
            m[:, k] = m[:, k] + f[:, i] * C_VECTORS[i][k]
    if not np.all(rho > 0.0):
        raise DomainError("vacuum node")
    u = m / rho[:, None] + 0.5 * np.asarray(flow.body_force)[None, :]
    return rho, u


def kernel_available(scheme, addressing, extensions: bool = False) -> bool:
    """kernel_available (p/src/stepper.cpp:140-153)."""
    f = _L.lbmgpu_kernel_available_ext if extensions else _L.lbmgpu_kernel_available
    return bool(f(_scheme_id(scheme), _addr_id(addressing)))


def build_sparse(geometry: GridGeometry, device: int = 0, node_of: bool = False):
    """build_sparse (p/src/geometry.cpp:173-207) on the GPU. Returns
    (fluid_count, adjacency[N, 18] uint32 node-major, node_of[cells] or None)."""
    g, keep = geometry._c()
    n = C.c_uint32()
    _check(_L.lbmgpu_build_sparse(C.byref(g), device, C.byref(n), None, None))
    adj = np.empty(int(n.value) * 18, dtype=np.uint32)
    nof = np.empty(geometry.cells(), dtype=np.uint32) if node_of else None
    _check(_L.lbmgpu_build_sparse(C.byref(g), device, C.byref(n), adj.ctypes.data,
                                  nof.ctypes.data if node_of else None))
    del keep
    return int(n.value), adj.reshape(-1, 18), nof


def build_et_rem(geometry: GridGeometry, device: int = 0):
    """ET indirect remote table (p/src/scheme_et.cpp:42-62): (rem[N, 9], mailboxes)."""
    g, keep = geometry._c()
    n, m = C.c_uint32(), C.c_uint32()
    _check(_L.lbmgpu_build_et_rem(C.byref(g), device, C.byref(n), None, C.byref(m)))
    rem = np.empty(int(n.value) * 9, dtype=np.uint32)
    _check(_L.lbmgpu_build_et_rem(C.byref(g), device, C.byref(n), rem.ctypes.data, C.byref(m)))
    del keep
    return rem.reshape(-1, 9), int(m.value)


def traffic(family, addressing, pdf_bytes: int = 8):
    """traffic() (p/src/perfmodel.cpp:12-75): (counts[6], bytes_per_lup)."""
    fam = FAMILIES.index(family) if isinstance(family, str) else int(family)
    out = (C.c_int32 * 6)()
    b = C.c_double()
    _check(_L.lbmgpu_traffic(fam, _addr_id(addressing), pdf_bytes, out, C.byref(b)))
    return list(out), b.value


def gpu_bytes_per_lup(scheme, addressing, pdf_bytes: int = 8) -> float:
    """Compulsory DRAM bytes per fluid-node update."""
    b = C.c_double()
    _check(_L.lbmgpu_gpu_bytes_per_lup(_scheme_id(scheme), _addr_id(addressing), pdf_bytes,
                                       C.byref(b)))
    return b.value


def halo_plan(nzl: int, scheme="aap"):
    """The z-slab exchange plan (lbmgpu_scheme_halo_plan): rows of (phase,
    send, peer, plane, slot) in posting order."""
    n = C.c_int32()
    sid = _scheme_id(scheme)
    _check(_L.lbmgpu_scheme_halo_plan(sid, nzl, None, C.byref(n)))
    ops = np.zeros(n.value * 5, np.int32)
    _check(_L.lbmgpu_scheme_halo_plan(sid, nzl, ops.ctypes.data, C.byref(n)))
    return ops.reshape(-1, 5)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_L.lbmgpu_nccl_unique_id(buf))
    return bytes(buf)


def slab_group_step(steppers, steps: int) -> None:
    """Step in-process z-slabs in lockstep (exchanges as device copies)."""
    arr = (C.c_void_p * len(steppers))(*[s._h for s in steppers])
    _check(_L.lbmgpu_slab_group_step(arr, len(steppers), int(steps)))


def slab_group_connect_p2p(steppers) -> None:
    """In-process z-slabs (ring in list order): switch them to the peer-memory
    transport (AA direct); slab_group_step then orders steps by events only."""
    arr = (_P * len(steppers))(*[s._h for s in steppers])
    _check(_L.lbmgpu_slab_group_connect_p2p(arr, len(steppers)))


def slab_group_sync_ghosts(steppers) -> None:
    arr = (C.c_void_p * len(steppers))(*[s._h for s in steppers])
    _check(_L.lbmgpu_slab_group_sync_ghosts(arr, len(steppers)))


class PinnedArray:
    """float64 array in page-locked host memory (lbmgpu_host_alloc)."""

    def __init__(self, n: int):
        p = C.c_void_p()
        _check(_L.lbmgpu_host_alloc(int(n) * 8, C.byref(p)))
        self._p = p
        self.array = np.ctypeslib.as_array((C.c_double * int(n)).from_address(p.value))

    def __del__(self):
        if getattr(self, "_p", None):
            _L.lbmgpu_host_free(self._p)
            self._p = None


def device_count() -> int:
    v = C.c_int32()
    _check(_L.lbmgpu_device_count(C.byref(v)))
    return int(v.value)


def version() -> str:
    return _L.lbmgpu_version().decode()
