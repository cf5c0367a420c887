"""bench.py's reference arm runs on CPU: it must print one JSON line with the driver's
contract keys (impl=reference, metric/value/unit, cpu_baseline, e2e)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libflowbb_ref.so")),
                    reason="reference not compiled here")
def test_reference_arm_explore_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--target", "4096",
              "--ref-seconds", "2"])
    assert d["impl"] == "reference" and d["unit"] == "bounded subproblems/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert all(r[2] > 0 for r in d["rounds"])


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libflowbb_ref.so")),
                    reason="reference not compiled here")
def test_reference_arm_bound_line():
    d = _run(["--impl", "reference", "--mode", "bound", "--instance", "ta021", "--ref-seconds", "1"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert "random_node" in d["cpu_baseline"]["sample"]
