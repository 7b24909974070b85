"""bench.py's reference arm on the host (no GPU): the reference build (oracle/_ref) runs the bench
step in a subprocess of its own (OpenMP active wait, bound threads, no torch in that process), and
`--impl reference` prints the contract's JSON line with the arm's own e2e / cpu_baseline objects."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref_lib  # noqa: E402

pytestmark = pytest.mark.skipif(not ref_lib.available(), reason="oracle/_ref not built")


def test_reference_worker_times_the_bench_step():
    import bench
    times, cores = bench.reference_step_times(2, 0)
    assert len(times) == 2 and all(t > 0 for t in times)
    assert cores >= 1


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--no-pfasst"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "reference" and "own process" in line["cpu_baseline"]["sample"]
    assert line["config"]["workload"].startswith("rhs_eval T255")
