"""CPU: bench.py's driver contract on the arm that needs no GPU. The
reference arm (`--impl reference`) times the reference's own CPU stepping
path (oracle/_ref, built from /root/reference) and must print exactly one JSON
line with the keys the driver reads; under torchrun only rank 0 prints.
The GPU arm's line is checked by tests/test_gpu_harness.py."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libref.so")


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ, LBM_REF_BUDGET_S="1", OMP_NUM_THREADS="4")
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                          env=env, capture_output=True, text=True, timeout=timeout)


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
def test_reference_arm_prints_one_contract_line():
    r = _run(["--impl", "reference", "--config", "c0", "--scheme", "os-push", "--steps", "3",
              "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["unit"] == "MFLUP/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C0")


def test_reference_arm_other_ranks_exit_silently():
    r = _run(["--impl", "reference", "--config", "c0", "--steps", "3"],
             env_extra={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"}, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""
