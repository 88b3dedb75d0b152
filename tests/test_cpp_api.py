"""GPU: the C++ drop-in mirror (include/lbmgpu/lbmgpu.hpp) runs the reference's
scheme-equivalence scenario (tests/cpp/test_api.cpp, built by build())."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_mirror_runs_reference_scenarios(gpu):
    exe = os.path.join(ROOT, "build", "test_api")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
