"""GPU: the device collision (dev::collide) against the reference's collision
tests (p/tests/test_collision.cpp). On a 1x1x1 periodic lattice every link of
the single node leads back to itself, so one OS-push step is exactly one
collision: f' = collide(f).
  known answers: bitwise equal to the oracle's restatement (and through it
    to the compiled reference, tests/test_oracle.py)   test_collision.cpp:39-53
  parity equivariance is exact without forcing         :116-130
  zero-rate operator is the exact identity             :132-139
  equal rates reduce to plain BGK (1e-14)              :152-173
  equilibrium is a fixed point without forcing (1e-13) :103-114
"""
import numpy as np
import pytest

from conftest import bitwise_equal

pytestmark = pytest.mark.gpu

OPP = [0, 2, 1, 4, 3, 6, 5, 18, 17, 16, 15, 14, 13, 12, 11, 10, 9, 8, 7]


def _collider(L, flow, precision=8, zero=False):
    st = L.create_stepper("os-push", "direct", L.GridGeometry(1, 1, 1), flow,
                          L.StepperOptions(precision=precision, zero_collision=zero))

    def collide(f):
        st.load_natural(np.ascontiguousarray(f, np.float64))
        st.step()
        return st.extract_natural()
    return collide


def _samples(n, seed):
    import oracle
    return oracle.Oracle().random_field(seed, n).reshape(n, 19)


def test_device_collision_equals_oracle_bitwise(gpu):
    import oracle
    L = gpu
    O = oracle.Oracle()
    flows = [L.FlowParams(1 / 0.9, 3 / 16, (1e-4, -2e-4, 3e-4), 1.0),  # TRT, magic 3/16
             L.bgk(1.7, (1e-6, 0.0, 0.0)), L.bgk(1.0)]
    for flow in flows:
        collide = _collider(L, flow)
        le, lo, g = flow.lambda_even, L.lambda_odd(flow), list(flow.body_force)
        for f in _samples(8, 17):
            assert bitwise_equal(collide(f), O.collide(f, le, lo, g)[0])


def test_parity_equivariance_exact(gpu):
    L = gpu
    collide = _collider(L, L.FlowParams(1 / 0.9, 3 / 16, (0.0, 0.0, 0.0), 1.0))
    for f in _samples(8, 11):
        rf = np.empty(19)
        rf[OPP] = f
        a, b = collide(f), collide(rf)
        assert bitwise_equal(b[OPP], a)


def test_zero_rates_are_identity(gpu):
    L = gpu
    collide = _collider(L, L.FlowParams(1 / 0.9, 3 / 16, (1e-4, 0.0, 0.0), 1.0), zero=True)
    for f in _samples(4, 3):
        assert bitwise_equal(collide(f), f)


def test_equal_rates_reduce_to_bgk(gpu):
    import oracle
    L = gpu
    O = oracle.Oracle()
    c, w, _ = O.stencil()
    g = np.array([2e-5, -1e-5, 3e-6])
    collide = _collider(L, L.bgk(1.0, tuple(g)))
    lam = 1.0
    for f in _samples(8, 11):
        rho = f.sum()
        u = (f[:, None] * c).sum(0) / rho
        feq = np.array([O.equilibrium(rho, list(u), i) for i in range(19)])
        want = f - lam * (f - feq) + 3.0 * w * (c @ g) * rho
        got = collide(f)
        assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-14


def test_equilibrium_is_fixed_point(gpu):
    import oracle
    L = gpu
    O = oracle.Oracle()
    collide = _collider(L, L.FlowParams(1 / 0.9, 3 / 16, (0.0, 0.0, 0.0), 1.0))
    for rho, u in [(1.0, [0.0, 0.0, 0.0]), (1.05, [0.03, -0.02, 0.01]), (0.97, [-0.05, 0.04, 0.0])]:
        feq = np.array([O.equilibrium(rho, u, i) for i in range(19)])
        got = collide(feq)
        assert np.max(np.abs(got - feq) / np.abs(feq)) <= 1e-13


def test_fp32_collision_within_tolerance(gpu):
    import oracle
    L = gpu
    O = oracle.Oracle()
    flow = L.bgk(1.7, (1e-6, 0.0, 0.0))
    collide = _collider(L, flow, precision=4)
    for f in _samples(8, 23):
        want = O.collide(f, 1.7, 1.7, [1e-6, 0.0, 0.0])[0]
        assert np.max(np.abs(collide(f) - want) / np.abs(want)) <= 1e-5
