"""bench.py's reference arm on CPU (the tiny config): the contract keys, the same workload
config the GPU arm prints, and the reference's own invoke being what was timed."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    from oracle import ref_step

    if not ref_step.available():
        pytest.skip("oracle/_ref not built (oracle/build_ref.sh)")
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "tiny",
                          "--steps", "3", "--warmup", "5"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["cpu_baseline"]["samples_timed"] == 3
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    sys.path.insert(0, REPO)
    import bench

    class A:
        config, batch, seq, remat, moe_routing = "tiny", 8, 256, "save_all", "router"

    assert line["config"] == bench.workload_config(A, 1)
