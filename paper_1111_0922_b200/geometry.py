"""Host-side geometry generators (input data for the path, not the hot path).

* ``gen_random_spheres`` — BASELINE.json configs[2] porous medium: seeded random
  overlapping spheres placed until the porosity reaches the target. The
  reference has no such generator (its ``gen_packed_bed``, p/src/geometry.cpp:73-121,
  is a deterministic staggered lattice); the same mask is handed to both the
  GPU and the CPU reference, so parity does not depend on it.
* ``gen_packed_bed`` — restatement of the reference's staggered sphere bed.
"""
from __future__ import annotations

import math
import struct

import numpy as np

from . import GridGeometry

# D3Q19 lattice vectors in canonical order (p/src/stencil.cpp:18-57)
C_VECTORS = ((0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1),
             (-1, -1, 0), (-1, 0, -1), (-1, 0, 1), (-1, 1, 0), (0, -1, -1), (0, -1, 1),
             (0, 1, -1), (0, 1, 1), (1, -1, 0), (1, 0, -1), (1, 0, 1), (1, 1, 0))

_MAGIC = b"LBMGEO1\0"


def save_geo(g: GridGeometry, path: str) -> None:
    """save_geo (p/src/geometry.cpp:123-135): 8-byte magic, u32 nx/ny/nz
    little-endian, 3 axis-policy bytes, nx*ny*nz mask bytes (x-fastest)."""
    mask = np.ones(g.cells(), np.uint8) if g.mask is None else np.asarray(g.mask, np.uint8)
    pol = [{"periodic": 0, "wall": 1, 0: 0, 1: 1}[p] for p in g.axis_policy]
    try:
        fh = open(path, "wb")
    except OSError:
        raise RuntimeError(f"cannot open {path}")
    with fh:
        fh.write(_MAGIC + struct.pack("<III", g.nx, g.ny, g.nz) + bytes(pol) + mask.tobytes())


def load_geo(path: str) -> GridGeometry:
    """load_geo (p/src/geometry.cpp:137-171), same checks and messages."""
    try:
        fh = open(path, "rb")
    except OSError:
        raise RuntimeError(f"cannot open {path}")
    with fh:
        magic = fh.read(8)
        if len(magic) != 8 or magic != _MAGIC:
            raise RuntimeError("not a geometry file")
        dims = fh.read(12)
        if len(dims) != 12:
            raise RuntimeError("short read")
        nx, ny, nz = struct.unpack("<III", dims)
        if (nx == 0 or ny == 0 or nz == 0 or max(nx, ny, nz) > 0x7FFFFFFF
                or nx * ny * nz > (1 << 40)):
            raise RuntimeError("dimension overflow")
        pol = fh.read(3)
        if len(pol) != 3:
            raise RuntimeError("short read")
        if any(p > 1 for p in pol):
            raise RuntimeError("not a geometry file")
        mask = np.frombuffer(fh.read(nx * ny * nz), np.uint8)
        if mask.size != nx * ny * nz:
            raise RuntimeError("short read")
    policy = tuple("wall" if p else "periodic" for p in pol)
    return GridGeometry(nx, ny, nz, policy, (mask != 0).astype(np.uint8))


def gen_random_spheres(nx: int, ny: int, nz: int, radius: float = 8.0, porosity: float = 0.40,
                       seed: int = 2011, periodic: bool = True) -> GridGeometry:
    """A cell is solid when its centre lies within `radius` of a sphere centre
    (minimum-image distance on periodic axes). Centres are drawn uniformly in
    the box from numpy's PCG64(seed); spheres are added until the fluid
    fraction is <= porosity. Returns an all-periodic GridGeometry (x-fastest mask)."""
    rng = np.random.default_rng(seed)
    solid = np.zeros((nz, ny, nx), dtype=bool)
    r = int(math.ceil(radius)) + 1
    off = np.arange(-r, r + 1)
    target_solid = int(math.ceil((1.0 - porosity) * nx * ny * nz))
    nsolid = 0
    while nsolid < target_solid:
        c = rng.uniform(0.0, 1.0, 3) * np.array([nx, ny, nz])
        ix = (np.floor(c[0]).astype(int) + off)
        iy = (np.floor(c[1]).astype(int) + off)
        iz = (np.floor(c[2]).astype(int) + off)
        dx = (ix + 0.5 - c[0]) ** 2
        dy = (iy + 0.5 - c[1]) ** 2
        dz = (iz + 0.5 - c[2]) ** 2
        inside = (dz[:, None, None] + dy[None, :, None] + dx[None, None, :]) < radius * radius
        zz, yy, xx = np.nonzero(inside)
        gx, gy, gz = ix[xx], iy[yy], iz[zz]
        if periodic:
            gx, gy, gz = gx % nx, gy % ny, gz % nz
        else:
            keep = (gx >= 0) & (gx < nx) & (gy >= 0) & (gy < ny) & (gz >= 0) & (gz < nz)
            gx, gy, gz = gx[keep], gy[keep], gz[keep]
        new = ~solid[gz, gy, gx]
        solid[gz[new], gy[new], gx[new]] = True
        nsolid += int(np.count_nonzero(new))
    mask = (~solid).astype(np.uint8).ravel()  # (z, y, x) C-order = x-fastest
    return GridGeometry(nx, ny, nz, ("periodic",) * 3, mask)


def gen_packed_bed(nx: int, ny: int, nz: int, radius: float, pitch: float) -> GridGeometry:
    """gen_packed_bed (p/src/geometry.cpp:73-121): layers of a square sphere grid
    of spacing `pitch` at z = k*pitch, odd layers offset by pitch/2 in x and y;
    periodic x, walls y/z. Vectorised per layer; same cell classification."""
    if min(nx, ny, nz) < 1:
        raise ValueError("zero dimension")
    if radius < 0.0:
        raise ValueError("radius must be non-negative")
    if not pitch > 0.0:
        raise ValueError("pitch must be positive")
    if radius > pitch:
        raise ValueError("overlapping spheres")
    solid = np.zeros((nz, ny, nx), dtype=bool)
    if radius > 0.0:
        r2 = radius * radius
        cx = np.arange(nx) + 0.5
        cy = np.arange(ny) + 0.5
        for z in range(nz):
            czv = z + 0.5
            klo = int(math.floor((czv - radius) / pitch))
            khi = int(math.ceil((czv + radius) / pitch))
            for k in range(klo, khi + 1):
                o = 0.5 * pitch if (k & 1) else 0.0
                dz2 = (czv - k * pitch) ** 2
                # nearest sphere centres along x and y for this layer
                ix = np.round((cx - o) / pitch)
                iy = np.round((cy - o) / pitch)
                best = None
                for di in (-1, 0, 1):
                    dx2 = (cx - ((ix + di) * pitch + o)) ** 2
                    for dj in (-1, 0, 1):
                        dy2 = (cy - ((iy + dj) * pitch + o)) ** 2
                        d = dy2[:, None] + dx2[None, :]
                        best = d if best is None else np.minimum(best, d)
                solid[z] |= (best + dz2) < r2
    mask = (~solid).astype(np.uint8).ravel()
    return GridGeometry(nx, ny, nz, ("periodic", "wall", "wall"), mask)
