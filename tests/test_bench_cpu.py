"""bench.py's CPU-side contract: the reference arm (the unmodified reference,
oracle/_ref, on the host) prints one JSON line with the keys the driver reads,
and the roofline traffic figure comes from the committed ncu launch list."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsfref_mt.so")):
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "plans_per_sec" and line["unit"] == "plans/s"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["steps"] == 2
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "plans/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_committed_launch_list_traffic():
    sys.path.insert(0, ROOT)
    import bench
    t = bench.committed_dram_bytes(bench.LATENCY_KERNEL, "(16, 1, 1)")
    assert t is not None and 1e4 < t < 1e7             # bytes per config-2 launch
    assert bench.committed_dram_bytes("no_such_kernel", "(1, 1, 1)") is None
