"""bench.py keeps the driver contract: one JSON line on stdout with the required keys, on the
smallest configuration (fast)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--config", "1", "--steps", "3",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
              "clocks", "cpu_baseline", "loop_roofline"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    assert d["results"]["true_rel_residual"] <= 1.01 * d["config"]["tol"]
    # configuration 1 is small: the CPU baseline runs the whole reference pipeline, not a sample
    assert d["cpu_baseline"]["extrapolated"] is False and d["cpu_baseline"]["iterations_per_solve"] == 20
    assert "value_1thread" in d["cpu_baseline"] and d["cpu_baseline"]["setup_s"] > 0

