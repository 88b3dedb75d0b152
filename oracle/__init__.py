"""TEST INFRASTRUCTURE ONLY — the CPU oracle and the reference library.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs may import this package, and only as the checker. The
product (``paper_1111_0922_b200``) never imports it.

* ``Oracle``  — ctypes view of ``_lib/liboracle.so``, the plain-C restatement
  of the reference D3Q19 path (``lbm_oracle.c``; each function cites the
  reference file:line it follows).
* ``RefLib``  — ctypes view of ``_ref/libref.so``: the UNMODIFIED reference
  library compiled from ``/root/reference/proj/src`` by ``oracle/Makefile``
  plus the thin C shim ``ref_capi.cpp``. Present only where it was built (it
  is built in the development container and travels to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "_lib", "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libref.so")

# SchemeId order (p/include/lbmlab/stepper.hpp:15-26)
SCHEMES = ["ts", "os-push", "os-pull", "osnt-pull-1s", "osnt-pull-2s", "cg",
           "swap-push", "swap-pull", "aap", "et"]
FAMILIES = ["ts", "os", "osnt", "cg", "swap", "aap", "et"]
FAMILY_OF = {"ts": 0, "os-push": 1, "os-pull": 1, "osnt-pull-1s": 2, "osnt-pull-2s": 2,
             "cg": 3, "swap-push": 4, "swap-pull": 4, "aap": 5, "et": 6}

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """Compile the oracle (and the reference library when /root/reference exists)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class _Geom(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("policy", C.c_uint8 * 3), ("mask", C.c_void_p)]


def _geom(nx, ny, nz, policy, mask):
    g = _Geom(nx, ny, nz)
    for k in range(3):
        g.policy[k] = int(policy[k])
    g._mask_keep = None
    if mask is not None:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        g._mask_keep = m
        g.mask = m.ctypes.data
    else:
        g.mask = None
    return g


class Oracle:
    """The C restatement (lbm_oracle.c)."""

    def __init__(self, path: str = LIB_ORACLE):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.orc_lambda_odd.restype = C.c_double
        L.orc_lambda_odd.argtypes = [C.c_double, C.c_double]
        L.orc_collide.argtypes = [C.c_void_p, _f64p]
        L.orc_trt_init.argtypes = [C.c_void_p, C.c_double, C.c_double, _f64p]
        L.orc_equilibrium.restype = C.c_double
        L.orc_equilibrium.argtypes = [C.c_double, _f64p, C.c_int]
        L.orc_fluid_count.restype = C.c_size_t
        L.orc_fluid_count.argtypes = [C.c_void_p]
        L.orc_build_sparse.argtypes = [C.c_void_p, _u32p, C.c_void_p]
        L.orc_et_rem.restype = C.c_uint32
        L.orc_et_rem.argtypes = [C.c_uint32, _u32p, _u32p]
        L.orc_ts_run.argtypes = [C.c_void_p, C.c_double, C.c_double, _f64p, _f64p,
                                 C.c_longlong, _f64p, C.c_int]
        L.orc_traffic.argtypes = [C.c_int, C.c_int, _i32p, C.POINTER(C.c_double)]
        L.orc_make_seeded_geometry.argtypes = [C.c_uint64, _u8p, _u8p]
        L.orc_random_field.argtypes = [C.c_uint64, C.c_size_t, C.c_double, _f64p]
        L.orc_stencil.argtypes = [_i32p, _f64p, _i32p]
        L.orc_flops_per_update.restype = C.c_int
        L.orc_init_field.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_uint64, C.c_double, C.c_double, C.c_double,
                                     C.c_double, _f64p]

    # -- physics -------------------------------------------------------------
    def stencil(self):
        c = np.zeros(57, np.int32)
        w = np.zeros(19)
        o = np.zeros(19, np.int32)
        self.L.orc_stencil(c, w, o)
        return c.reshape(19, 3), w, o

    def lambda_odd(self, lambda_even, magic):
        return self.L.orc_lambda_odd(lambda_even, magic)

    def collide(self, f, lambda_even, lambda_odd, g):
        f = np.array(f, dtype=np.float64).reshape(-1, 19)
        op = C.create_string_buffer(8 * 64)
        self.L.orc_trt_init(op, lambda_even, lambda_odd, np.asarray(g, np.float64))
        for n in range(f.shape[0]):
            row = np.ascontiguousarray(f[n])
            self.L.orc_collide(op, row)
            f[n] = row
        return f

    def equilibrium(self, rho, u, i):
        return self.L.orc_equilibrium(rho, np.asarray(u, np.float64), i)

    def flops_per_update(self):
        return self.L.orc_flops_per_update()

    # -- geometry ------------------------------------------------------------
    def fluid_count(self, nx, ny, nz, policy, mask=None):
        return int(self.L.orc_fluid_count(C.byref(_geom(nx, ny, nz, policy, mask))))

    def build_sparse(self, nx, ny, nz, policy, mask=None):
        g = _geom(nx, ny, nz, policy, mask)
        n = int(self.L.orc_fluid_count(C.byref(g)))
        adj = np.zeros(n * 18, np.uint32)
        node_of = np.zeros(nx * ny * nz, np.uint32)
        rc = self.L.orc_build_sparse(C.byref(g), adj, node_of.ctypes.data)
        if rc != 0:
            raise RuntimeError("fluid count exceeds 32-bit index range")
        return adj.reshape(n, 18), node_of

    def et_rem(self, adjacency):
        n = adjacency.shape[0]
        rem = np.zeros(n * 9, np.uint32)
        nmail = self.L.orc_et_rem(n, np.ascontiguousarray(adjacency, np.uint32).ravel(), rem)
        return rem.reshape(n, 9), int(nmail)

    def init_field(self, kind, dims, policy=(0, 0, 0), mask=None, seed=0, rho0=1.0,
                   u0=0.01, drho=1e-3, noise=1e-4, gdims=None, z0=0):
        """Canonical start snapshot of the BASELINE configs (lbm_oracle.c
        orc_init_field): kind 'rest' | 'taylor_green' | 'random'; gdims/z0
        place a z-slab inside a global box."""
        k = {"rest": 0, "taylor_green": 1, "random": 2}[kind]
        nx, ny, nz = dims
        gnx, gny, gnz = gdims or dims
        g = _geom(nx, ny, nz, policy, mask)
        n = int(self.L.orc_fluid_count(C.byref(g)))
        out = np.empty(n * 19)
        if self.L.orc_init_field(C.byref(g), k, gnx, gny, gnz, z0, seed, rho0, u0, drho, noise,
                                 out) != 0:
            raise MemoryError("oracle allocation failed")
        return out

    def make_seeded_geometry(self, seed):
        mask = np.zeros(16 * 8 * 8, np.uint8)
        pol = np.zeros(3, np.uint8)
        self.L.orc_make_seeded_geometry(seed, mask, pol)
        return (16, 8, 8), pol, mask

    def random_field(self, seed, nodes, scale=1.0):
        f = np.zeros(nodes * 19)
        self.L.orc_random_field(seed, nodes, scale, f)
        return f

    # -- stepping ------------------------------------------------------------
    def ts_run(self, nx, ny, nz, policy, mask, lambda_even, lambda_odd, g, f_in, steps,
               threads=None):
        geo = _geom(nx, ny, nz, policy, mask)
        f_in = np.ascontiguousarray(f_in, np.float64).ravel()
        out = np.zeros_like(f_in)
        rc = self.L.orc_ts_run(C.byref(geo), lambda_even, lambda_odd,
                               np.asarray(g, np.float64), f_in, steps, out,
                               threads or os.cpu_count() or 1)
        if rc != 0:
            raise MemoryError("oracle allocation failed")
        return out

    def traffic(self, family, addressing):
        out = np.zeros(6, np.int32)
        b = C.c_double()
        if self.L.orc_traffic(family, addressing, out, C.byref(b)) != 0:
            raise ValueError("unknown scheme")
        return out, b.value


class RefLib:
    """The unmodified reference library (oracle/_ref/libref.so)."""

    def __init__(self, path: str = LIB_REF):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_lambda_odd.restype = C.c_double
        L.ref_lambda_odd.argtypes = [C.c_double, C.c_double]
        L.ref_collide.argtypes = [C.c_double, C.c_double, _f64p, _f64p, C.c_longlong]
        L.ref_equilibrium.restype = C.c_double
        L.ref_equilibrium.argtypes = [C.c_double, _f64p, C.c_int]
        L.ref_stencil.argtypes = [_i32p, _f64p, _i32p]
        L.ref_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, C.c_void_p,
                                 C.c_double, C.c_double, _f64p, C.c_double, C.c_int, C.c_int,
                                 C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_step.argtypes = [C.c_void_p, C.c_longlong]
        L.ref_extract.argtypes = [C.c_void_p, _f64p]
        L.ref_load.argtypes = [C.c_void_p, _f64p]
        L.ref_time_step.restype = C.c_longlong
        L.ref_time_step.argtypes = [C.c_void_p]
        L.ref_node_count.restype = C.c_ulonglong
        L.ref_node_count.argtypes = [C.c_void_p]
        L.ref_layout_phase.argtypes = [C.c_void_p]
        L.ref_exchange_opposite_handles.argtypes = [C.c_void_p]
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_build_sparse.argtypes = [C.c_int, C.c_int, C.c_int, _u8p, C.c_void_p,
                                       C.POINTER(C.c_uint), C.c_void_p, C.c_void_p]
        L.ref_make_seeded_geometry.argtypes = [C.c_ulonglong, _u8p, _u8p]
        L.ref_traffic.argtypes = [C.c_int, C.c_int, _i32p, C.POINTER(C.c_double)]
        L.ref_run_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u8p,
                                    C.c_void_p, C.c_double, C.c_double, _f64p, C.c_double,
                                    C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int)]
        L.ref_verify_suite.argtypes = [C.c_ulonglong, C.c_int, _i32p, _f64p,
                                       C.POINTER(C.c_int)]
        L.ref_flops_per_update.restype = C.c_int
        L.ref_save_geo.argtypes = [C.c_int, C.c_int, C.c_int, _u8p, C.c_void_p, C.c_char_p]
        L.ref_kernel_available.argtypes = [C.c_int, C.c_int]

    def error(self):
        return self.L.ref_last_error().decode()

    def stencil(self):
        c = np.zeros(57, np.int32)
        w = np.zeros(19)
        o = np.zeros(19, np.int32)
        self.L.ref_stencil(c, w, o)
        return c.reshape(19, 3), w, o

    def collide(self, f, lambda_even, lambda_odd, g):
        f = np.array(f, dtype=np.float64).ravel().copy()
        self.L.ref_collide(lambda_even, lambda_odd, np.asarray(g, np.float64), f, f.size // 19)
        return f.reshape(-1, 19)

    def create(self, scheme, addressing, dims, policy, mask, lambda_even, magic, g,
               rho0=1.0, workers=1, chunk_length=150, streaming_stores=True,
               swap_deferred_fixup=False, zero_collision=False):
        h = C.c_void_p()
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        rc = self.L.ref_create(SCHEMES.index(scheme) if isinstance(scheme, str) else scheme,
                               addressing, dims[0], dims[1], dims[2],
                               np.asarray(policy, np.uint8),
                               None if m is None else m.ctypes.data, lambda_even, magic,
                               np.asarray(g, np.float64), rho0, workers, chunk_length,
                               int(streaming_stores), int(swap_deferred_fixup),
                               int(zero_collision), C.byref(h))
        if rc != 0:
            raise RuntimeError(f"ref_create failed ({rc}): {self.error()}")
        return RefStepper(self, h)

    def build_sparse(self, nx, ny, nz, policy, mask=None):
        cells = nx * ny * nz
        n = C.c_uint()
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        pol = np.asarray(policy, np.uint8)
        rc = self.L.ref_build_sparse(nx, ny, nz, pol, None if m is None else m.ctypes.data,
                                     C.byref(n), None, None)
        if rc != 0:
            raise RuntimeError(self.error())
        adj = np.zeros(n.value * 18, np.uint32)
        node_of = np.zeros(cells, np.uint32)
        self.L.ref_build_sparse(nx, ny, nz, pol, None if m is None else m.ctypes.data,
                                C.byref(n), adj.ctypes.data, node_of.ctypes.data)
        return adj.reshape(-1, 18), node_of

    def make_seeded_geometry(self, seed):
        mask = np.zeros(1024, np.uint8)
        pol = np.zeros(3, np.uint8)
        self.L.ref_make_seeded_geometry(seed, mask, pol)
        return (16, 8, 8), pol, mask

    def save_geo(self, dims, policy, mask, path):
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        if self.L.ref_save_geo(dims[0], dims[1], dims[2], np.asarray(policy, np.uint8),
                               None if m is None else m.ctypes.data, path.encode()) != 0:
            raise RuntimeError(self.error())

    def traffic(self, family, addressing):
        out = np.zeros(6, np.int32)
        b = C.c_double()
        self.L.ref_traffic(family, addressing, out, C.byref(b))
        return out, b.value

    def run_bench(self, scheme, addressing, dims, policy, mask, lambda_even, magic, g,
                  steps, workers=0, warmup=1, timed_runs=3, rho0=1.0):
        s, ml, wu = C.c_double(), C.c_double(), C.c_int()
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        rc = self.L.ref_run_bench(SCHEMES.index(scheme) if isinstance(scheme, str) else scheme,
                                  addressing, dims[0], dims[1], dims[2],
                                  np.asarray(policy, np.uint8),
                                  None if m is None else m.ctypes.data, lambda_even, magic,
                                  np.asarray(g, np.float64), rho0, steps, workers, warmup,
                                  timed_runs, C.byref(s), C.byref(ml), C.byref(wu))
        if rc != 0:
            raise RuntimeError(self.error())
        return s.value, ml.value, wu.value

    def verify_suite(self, seed, steps):
        ids = np.zeros(64 * 4, np.int32)
        mr = np.zeros(64)
        ap = C.c_int()
        n = self.L.ref_verify_suite(seed, steps, ids, mr, C.byref(ap))
        if n < 0:
            raise RuntimeError(self.error())
        return ids[: 4 * n].reshape(n, 4), mr[:n], bool(ap.value)


class RefStepper:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h
        self.nodes = int(lib.L.ref_node_count(h))

    def step(self, n=1):
        if self.lib.L.ref_step(self.h, n) != 0:
            raise RuntimeError(self.lib.error())

    def extract(self):
        out = np.zeros(self.nodes * 19)
        if self.lib.L.ref_extract(self.h, out) != 0:
            raise RuntimeError(self.lib.error())
        return out

    def load(self, f):
        if self.lib.L.ref_load(self.h, np.ascontiguousarray(f, np.float64).ravel()) != 0:
            raise RuntimeError(self.lib.error())

    def time_step(self):
        return int(self.lib.L.ref_time_step(self.h))

    def layout_phase(self):
        return int(self.lib.L.ref_layout_phase(self.h))

    def exchange_opposite_handles(self):
        return bool(self.lib.L.ref_exchange_opposite_handles(self.h))

    def __del__(self):
        try:
            self.lib.L.ref_destroy(self.h)
        except Exception:
            pass
