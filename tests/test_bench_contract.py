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
    assert d["scaling"] == "strong"


def test_reference_arm_other_ranks_exit_silently():
    r = _run(["--impl", "reference", "--config", "c0", "--steps", "3"],
             env_extra={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"}, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_gpus_flag_relaunches_n_ranks():
    """`bench.py --gpus 2` outside torchrun re-execs itself under
    torch.distributed.run with two ranks (never a silent one-GPU line)."""
    r = _run(["--gpus", "2", "--steps", "3"], env_extra={"LBM_BENCH_DRYRUN": "1"}, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world_size"] == 2 and d["gpus"] == 2 for d in lines)


def test_gpus_flag_must_match_world_size():
    r = _run(["--gpus", "4", "--steps", "3"],
             env_extra={"LBM_BENCH_DRYRUN": "1", "WORLD_SIZE": "2", "RANK": "0"}, timeout=120)
    assert r.returncode != 0
    assert "WORLD_SIZE=2" in r.stderr


def test_reference_arm_config_matches_ours_shape():
    """Both arms build `config` with bench.config_dict, so the driver's
    same-config check compares like with like (C3 default at every N)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)

    class A:
        scheme, addressing, layout, precision = "aap", "direct", "soa", 8
    c = b.config_dict("c3", A, 1, 512 * 512 * 1024)
    assert c["workload"].startswith("C3") and c["dims"] == [512, 512, 1024]
    assert c["parallelism"] == "single domain"
    assert b.config_dict("c3", A, 8, 512 * 512 * 1024)["parallelism"] == "z-slabs x8"
