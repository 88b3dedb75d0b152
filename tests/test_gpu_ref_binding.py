"""GPU: the reference-side binding (include/lbmgpu/lbmlab_gpu.hpp) —
`GpuStepper : lbmlab::Stepper` — driven by the reference's own callers.

build/ref_binding (tests/cpp/ref_binding.cpp) is compiled in the development
container against the UNMODIFIED reference headers and library (oracle/_ref,
built from /root/reference) and travels to the GPU box prebuilt. It runs
verify_suite's loop against the reference's CPU two-step stepper (all 16
pairs x SoA/AoS x fp64/fp32, memcmp after every step), acceptance criteria 4
(1000-step closed box), 5 (channel profile through the reference's
macroscopic_fields) and 8 (chunk invariance), the reference's exception texts
(incl. domain_error "vacuum node") and run_bench's timing loop.
"""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "build", "ref_binding")


@pytest.mark.parametrize("check", ["verify", "conserve", "channel", "chunks", "errors", "bench"])
def test_reference_callers_through_binding(gpu, check):
    assert os.path.exists(BIN), "build/ref_binding missing: run __graft_entry__.build() " \
                                "where /root/reference exists"
    r = subprocess.run([BIN, check], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, OMP_NUM_THREADS=str(min(16, os.cpu_count() or 1))))
    print(r.stdout)
    assert r.returncode == 0 and f"[PASS] {check}" in r.stdout, r.stdout + r.stderr
