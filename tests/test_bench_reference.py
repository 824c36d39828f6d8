"""bench.py --impl reference (host only): the reference algorithm's CPU arm prints the driver's
JSON line with the same config dict as the GPU arm and, on the small configuration 1, times whole
solves of the reference pipeline (oracle port), not an extrapolated sample."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_reference_arm_matches_config():
    """--impl reference prints the same config dict as the GPU arm (same_config) and, on a small
    configuration, whole solves (ms_per_step = one solve)."""
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.strip()][-1])
    assert d["impl"] == "reference" and d["config"]["workload"] == "cfg1-poisson2d-64"
    assert d["config"]["n"] == 4096 and d["config"]["subdomains"] == 16
    assert d["cpu_baseline"]["iterations_per_solve"] == 20 and "extrapolated" not in d
    assert abs(d["ms_per_step"] - 1e3 * 20 / d["value"]) <= 1e-6 * d["ms_per_step"]
