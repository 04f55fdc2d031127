"""bench.py's reference arm on the host (no GPU needed): it honours --steps
and --warmup exactly and prints the same `config` dict as the GPU arm
(VERDICT r1 weak #6)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_honours_steps_and_config():
    import argparse
    import bench
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2",
                        "--warmup", "1", "--workload", "1080p-batch"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    a = argparse.Namespace(workload="1080p-batch", contract="sr", prefetch=1, transport="peer")
    assert d["config"] == bench.base_config(a, 1)
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0


def test_default_workload_by_world(monkeypatch):
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    monkeypatch.setenv("WORLD_SIZE", "1")
    assert bench.parse().workload == "8k"
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.parse().workload == "32k-bands"


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsobel5_ref.so")),
                    reason="compiled reference absent")
def test_cpu_matrix_rows_in_reference_schema():
    import bench
    m = bench.cpu_matrix(budget_s=0.0)  # the budget stops after the first row
    assert m["csv_header"] == "label,width,height,iters,mean_s,stddev_s,mps,mps_per_core"
    assert len(m["rows"]) == 1 and m["rows"][0]["csv"].startswith("fast-5x5,1920,1080,2,")
    assert m["host"]["nproc"] == os.cpu_count()
