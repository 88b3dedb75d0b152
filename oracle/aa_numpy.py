"""TEST INFRASTRUCTURE ONLY — numpy restatements of the AA pattern and the
one-step push/pull scheme on one z-slab with ghost planes, used to check the
multi-GPU halo plans on CPU.

Vectorised over cells with the reference's exact operation order (numpy
float64 ufuncs round like the -ffp-contract=off C code), so it is bitwise equal
to lbm_oracle.c / the reference:
  collide      TrtOperator::collide   p/src/collision.cpp:95-139
  even sweep   AapStepper::sweep_even p/src/scheme_aap.cpp:114-131
  odd sweep    sweep_odd_direct       p/src/scheme_aap.cpp:133-173 (x/y periodic,
               z neighbours through the ghost planes)
"""
import numpy as np

C = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1],
              [-1, -1, 0], [-1, 0, -1], [-1, 0, 1], [-1, 1, 0], [0, -1, -1], [0, -1, 1],
              [0, 1, -1], [0, 1, 1], [1, -1, 0], [1, 0, -1], [1, 0, 1], [1, 1, 0]])
OPP = [0, 2, 1, 4, 3, 6, 5, 18, 17, 16, 15, 14, 13, 12, 11, 10, 9, 8, 7]
PI = [1, 3, 5, 7, 8, 9, 10, 11, 12]
PJ = [2, 4, 6, 18, 17, 16, 15, 14, 13]
W = [1.0 / 3.0] + [1.0 / 18.0] * 6 + [1.0 / 36.0] * 12


def trt(lambda_even, lambda_odd, g):
    """TrtOperator::build (p/src/collision.cpp:64-93)"""
    w2, f3w = [], []
    for p in range(9):
        i = PI[p]
        cg = 0.0
        for k in range(3):
            if C[i][k] != 0:
                cg += C[i][k] * g[k]
        w2.append(2.0 * W[i])
        f3w.append(3.0 * W[i] * cg)
    return dict(le=lambda_even, le_half=0.5 * lambda_even, lo_half=0.5 * lambda_odd, w0=W[0],
                w2=w2, f3w=f3w)


def collide(op, f):
    """f: list of 19 arrays (same shape); returns the 19 post-collision arrays"""
    f = list(f)
    fsum = [f[PI[p]] + f[PJ[p]] for p in range(9)]
    fdif = [f[PI[p]] - f[PJ[p]] for p in range(9)]
    rho = f[0]
    for p in range(9):
        rho = rho + fsum[p]
    u = []
    for k in range(3):
        m = np.zeros_like(rho)
        for p in range(9):
            ck = C[PI[p]][k]
            if ck > 0:
                m = m + fdif[p]
            elif ck < 0:
                m = m + (-fdif[p])
        u.append(m / rho)
    usq = u[0] * u[0]
    usq = usq + u[1] * u[1]
    usq = usq + u[2] * u[2]
    base = 1.0 - 1.5 * usq
    wr0 = op["w0"] * rho
    e0 = wr0 * base
    f[0] = f[0] - op["le"] * (f[0] - e0)
    for p in range(9):
        i, j = PI[p], PJ[p]
        cu = None
        for k in range(3):
            ck = C[i][k]
            if ck == 0:
                continue
            t = u[k] if ck > 0 else -u[k]
            cu = t if cu is None else cu + t
        cu3 = 3.0 * cu
        cusq45 = 0.5 * (cu3 * cu3)
        wr2 = op["w2"][p] * rho
        esum = wr2 * (base + cusq45)
        edif = wr2 * cu3
        dp = op["le_half"] * (fsum[p] - esum)
        dm = op["lo_half"] * (fdif[p] - edif)
        dmf = dm - op["f3w"][p] * rho
        f[i] = f[i] - dp - dmf
        f[j] = f[j] - dp + dmf
    return f


class AaSlab:
    """AA pattern on local planes [z0, z1) of an nx*ny*nz periodic box;
    F[19, nzl + 2, ny, nx] with ghost storage planes 0 and nzl + 1."""

    def __init__(self, nx, ny, nzl, op):
        self.nx, self.ny, self.nzl, self.op = nx, ny, nzl, op
        self.F = np.zeros((19, nzl + 2, ny, nx))
        self.t = 0

    def load(self, snap):  # canonical snapshot of the slab's nodes, x-fastest
        s = snap.reshape(self.nzl, self.ny, self.nx, 19)
        for i in range(19):
            self.F[i, 1:-1] = s[..., i]
        self.t = 0

    def plane(self, slot, plane):  # view of one slot plane (local plane index)
        return self.F[slot, plane + 1]

    def step_local(self):
        n = self.nzl
        if self.t % 2 == 0:
            tmp = collide(self.op, [self.F[i, 1:n + 1] for i in range(19)])
            for i in range(19):
                self.F[OPP[i], 1:n + 1] = tmp[i]
        else:
            src = [self.F[0, 1:n + 1]]
            for i in range(1, 19):
                cx, cy, cz = C[i]
                rolled = np.roll(self.F[OPP[i]], (cy, cx), axis=(1, 2))
                src.append(rolled[1 - cz:n + 1 - cz])
            tmp = collide(self.op, src)
            self.F[0, 1:n + 1] = tmp[0]
            for j in range(1, 19):
                cx, cy, cz = C[j]
                self.F[j, 1 + cz:n + 1 + cz] = np.roll(tmp[j], (cy, cx), axis=(1, 2))
        self.t += 1

    def extract(self):
        n = self.nzl
        out = np.zeros((n, self.ny, self.nx, 19))
        if self.t % 2 == 0:
            for i in range(19):
                out[..., i] = self.F[i, 1:n + 1]
        else:  # p/src/scheme_aap.cpp:57-75 (needs fresh ghosts)
            out[..., 0] = self.F[0, 1:n + 1]
            for i in range(1, 19):
                cx, cy, cz = C[i]
                rolled = np.roll(self.F[OPP[i]], (cy, cx), axis=(1, 2))
                out[..., i] = rolled[1 - cz:n + 1 - cz]
        return out.ravel()


class OsSlab:
    """One-step two-grid scheme on a slab (p/src/scheme_os.cpp): pull gathers
    A[i][X - c_i] (after a first precollide, :79-102, 141-174), push scatters
    to B[i][X + c_i] (:104-139); x/y periodic, z through ghost planes."""

    def __init__(self, nx, ny, nzl, op, pull):
        self.nx, self.ny, self.nzl, self.op, self.pull = nx, ny, nzl, op, pull
        self.G = [np.zeros((19, nzl + 2, ny, nx)), np.zeros((19, nzl + 2, ny, nx))]
        self.active = 0
        self.fresh = pull
        self.t = 0

    def load(self, snap):
        s = snap.reshape(self.nzl, self.ny, self.nx, 19)
        for i in range(19):
            self.G[self.active][i, 1:-1] = s[..., i]
        self.t = 0
        self.fresh = self.pull

    def plane(self, grid, slot, plane):
        return self.G[grid][slot, plane + 1]

    def precollide(self):
        if self.pull and self.fresh:
            n, A = self.nzl, self.G[self.active]
            tmp = collide(self.op, [A[i, 1:n + 1] for i in range(19)])
            for i in range(19):
                A[i, 1:n + 1] = tmp[i]
            self.fresh = False

    def step_local(self):
        n, A, B = self.nzl, self.G[self.active], self.G[self.active ^ 1]
        if self.pull:
            src = [A[0, 1:n + 1]]
            for i in range(1, 19):
                cx, cy, cz = C[i]
                src.append(np.roll(A[i], (cy, cx), axis=(1, 2))[1 - cz:n + 1 - cz])
            tmp = collide(self.op, src)
            for i in range(19):
                B[i, 1:n + 1] = tmp[i]
        else:
            tmp = collide(self.op, [A[i, 1:n + 1] for i in range(19)])
            B[0, 1:n + 1] = tmp[0]
            for i in range(1, 19):
                cx, cy, cz = C[i]
                B[i, 1 + cz:n + 1 + cz] = np.roll(tmp[i], (cy, cx), axis=(1, 2))
        self.active ^= 1
        self.t += 1

    def extract(self):
        n = self.nzl
        out = np.zeros((n, self.ny, self.nx, 19))
        if not self.pull or self.fresh:
            for i in range(19):
                out[..., i] = self.G[self.active][i, 1:n + 1]
        else:  # gather_out_direct from the idle grid (p/src/stepper.cpp:228-252)
            I = self.G[self.active ^ 1]
            out[..., 0] = I[0, 1:n + 1]
            for i in range(1, 19):
                cx, cy, cz = C[i]
                out[..., i] = np.roll(I[i], (cy, cx), axis=(1, 2))[1 - cz:n + 1 - cz]
        return out.ravel()


class EtSlab:
    """Esoteric twist on a slab (p/src/scheme_et.cpp): one grid, handle table
    b[] swapped pairwise after every sweep (:191-239), fill with identity
    handles (:152-169), natural extraction (:83-109); x/y periodic, z through
    ghost planes. plane(slot, plane) maps the logical slot through b[]."""

    def __init__(self, nx, ny, nzl, op):
        self.nx, self.ny, self.nzl, self.op = nx, ny, nzl, op
        self.F = np.zeros((19, nzl + 2, ny, nx))
        self.b = list(range(19))
        self.t = 0

    def _remote(self, slot, i):  # F[slot][X + c_i] over the local planes
        cx, cy, cz = C[i]
        n = self.nzl
        return np.roll(self.F[slot], (-cy, -cx), axis=(1, 2))[1 + cz:n + 1 + cz]

    def _put_remote(self, slot, i, v):
        cx, cy, cz = C[i]
        n = self.nzl
        self.F[slot, 1 + cz:n + 1 + cz] = np.roll(v, (cy, cx), axis=(1, 2))

    def load(self, snap):
        s = snap.reshape(self.nzl, self.ny, self.nx, 19)
        self.b = list(range(19))
        self.F[0, 1:-1] = s[..., 0]
        for p in range(9):
            i, j = PI[p], PJ[p]
            self.F[i, 1:-1] = s[..., i]
            self._put_remote(j, i, s[..., j])
        self.t = 0

    def plane(self, slot, plane):
        return self.F[self.b[slot], plane + 1]

    def step_local(self):
        """one sweep with the current handles; swap_handles() afterwards"""
        n, b = self.nzl, self.b
        f = [None] * 19
        f[0] = self.F[0, 1:n + 1].copy()
        for p in range(9):
            i, j = PI[p], PJ[p]
            f[i] = self.F[b[i], 1:n + 1].copy()
            f[j] = self._remote(b[j], i).copy()
        f = collide(self.op, f)
        self.F[0, 1:n + 1] = f[0]
        for p in range(9):
            i, j = PI[p], PJ[p]
            self.F[b[i], 1:n + 1] = f[j]
            self._put_remote(b[j], i, f[i])
        self.t += 1

    def swap_handles(self):
        for p in range(9):
            i, j = PI[p], PJ[p]
            self.b[i], self.b[j] = self.b[j], self.b[i]

    def extract(self):
        n, b = self.nzl, self.b
        out = np.zeros((n, self.ny, self.nx, 19))
        out[..., 0] = self.F[0, 1:n + 1]
        for p in range(9):
            i, j = PI[p], PJ[p]
            out[..., i] = self.F[b[i], 1:n + 1]
            out[..., j] = self._remote(b[j], i)
        return out.ravel()
